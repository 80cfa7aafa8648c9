// Multi-GPU plumbing for a C++ host (SURVEY §8(b) "a multi-GPU communicator setup", §8(e)):
// an NCCL communicator plus the collectives the row-sharded sketches and PCG need --
// all-reduce of the m x m Gram-type partials, all-gather, and the column <-> row block
// transposes (grouped send / recv over NVLink).  NCCL is resolved at run time with dlopen
// ("libnccl.so.2": the copy torch already loaded, else the system one), so the library has
// no link-time NCCL dependency and the Python side keeps using torch.distributed.
#include <dlfcn.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

namespace w4 {
void set_last_error(const std::string& msg);
}

using namespace w4;

namespace {

// the subset of nccl.h used here (ABI-stable across NCCL 2.x)
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclSuccess = 0 };
enum { ncclDouble = 8 };
enum { ncclSum = 0 };

struct Nccl {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        n.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!n.h) return;
        auto sym = [](const char* name) { return dlsym(n.h, name); };
        n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
        n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
        n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
        n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
        n.AllGather = reinterpret_cast<decltype(n.AllGather)>(sym("ncclAllGather"));
        n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
        n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
        n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
        n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
        n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    });
    if (!n.h || !n.GetUniqueId || !n.CommInitRank || !n.AllReduce || !n.Send || !n.GroupEnd)
        throw DeviceError("NCCL (libnccl.so.2) is not available");
    return n;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw DeviceError(std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error"));
}

// balanced partition of `total` into `size` parts: part r = [off(r), off(r + 1))
int64_t part_off(int64_t total, int size, int r) { return total * r / size; }

}  // namespace

struct wc4dvar_comm {
    ncclComm_t comm = nullptr;
    int rank = 0, size = 1, device = 0;
    DevBuf pack, unpack;
};

#define W4_COMM_BEGIN try {
#define W4_COMM_END                        \
    return WC4DVAR_OK;                     \
    }                                      \
    catch (const w4::InvalidArgument& e) { \
        w4::set_last_error(e.what());      \
        return WC4DVAR_INVALID_ARGUMENT;   \
    }                                      \
    catch (const std::exception& e) {      \
        w4::set_last_error(e.what());      \
        return WC4DVAR_DEVICE;             \
    }

extern "C" {

int wc4dvar_gpu_comm_unique_id(unsigned char* id128) {
    W4_COMM_BEGIN
    require(id128 != nullptr, "comm_unique_id: null buffer");
    ncclUniqueId u;
    check(nccl().GetUniqueId(&u), "ncclGetUniqueId");
    std::memcpy(id128, u.internal, 128);
    W4_COMM_END
}

int wc4dvar_gpu_comm_create(const unsigned char* id128, int rank, int size, int device, wc4dvar_comm** out) {
    W4_COMM_BEGIN
    require(id128 && out && size >= 1 && rank >= 0 && rank < size, "comm_create: bad arguments");
    DeviceGuard g(device);
    ncclUniqueId u;
    std::memcpy(u.internal, id128, 128);
    std::unique_ptr<wc4dvar_comm> c(new wc4dvar_comm());
    check(nccl().CommInitRank(&c->comm, size, u, rank), "ncclCommInitRank");
    c->rank = rank;
    c->size = size;
    c->device = device;
    *out = c.release();
    W4_COMM_END
}

int wc4dvar_gpu_comm_destroy(wc4dvar_comm* c) {
    W4_COMM_BEGIN
    if (!c) return WC4DVAR_OK;
    {
        DeviceGuard g(c->device);
        if (c->comm) nccl().CommDestroy(c->comm);
    }
    delete c;
    W4_COMM_END
}

int wc4dvar_gpu_comm_allreduce_sum(wc4dvar_comm* c, double* buf, int64_t count, void* stream) {
    W4_COMM_BEGIN
    require(c && (buf || count == 0) && count >= 0, "comm_allreduce_sum: bad arguments");
    DeviceGuard g(c->device);
    check(nccl().AllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, c->comm, static_cast<cudaStream_t>(stream)),
          "ncclAllReduce");
    W4_COMM_END
}

int wc4dvar_gpu_comm_allgather(wc4dvar_comm* c, const double* send, int64_t count, double* recv, void* stream) {
    W4_COMM_BEGIN
    require(c && send && recv && count >= 0, "comm_allgather: bad arguments");
    DeviceGuard g(c->device);
    check(nccl().AllGather(send, recv, (size_t)count, ncclDouble, c->comm, static_cast<cudaStream_t>(stream)),
          "ncclAllGather");
    W4_COMM_END
}

// Column shard -> row shard (SURVEY §8(e) transpose).  Rank r holds columns
// [coff(r), coff(r+1)) of an nrows x ncols block (cols: nrows x mr, ld nrows) and receives rows
// [roff(r), roff(r+1)) of all ncols columns (rows: Rr x ncols, ld Rr).  Balanced partitions.
int wc4dvar_gpu_comm_cols_to_rows(wc4dvar_comm* c, const double* cols, int64_t nrows, int64_t ncols, double* rows,
                                  void* stream) {
    W4_COMM_BEGIN
    require(c && nrows >= 0 && ncols >= 0, "comm_cols_to_rows: bad arguments");
    DeviceGuard g(c->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int G = c->size, r = c->rank;
    const int64_t mr = part_off(ncols, G, r + 1) - part_off(ncols, G, r);
    const int64_t Rr = part_off(nrows, G, r + 1) - part_off(nrows, G, r);
    // pack: block for rank s = rows [roff(s), roff(s+1)) of my mr columns, contiguous
    double* pk = c->pack.get<double>((size_t)std::max<int64_t>(nrows * mr, 1));
    for (int s = 0; s < G; ++s) {
        const int64_t r0 = part_off(nrows, G, s), rs = part_off(nrows, G, s + 1) - r0;
        if (rs * mr)
            W4_CUDA(cudaMemcpy2DAsync(pk + r0 * mr, rs * sizeof(double), cols + r0, nrows * sizeof(double),
                                      rs * sizeof(double), mr, cudaMemcpyDeviceToDevice, st));
    }
    check(nccl().GroupStart(), "ncclGroupStart");
    for (int s = 0; s < G; ++s) {
        const int64_t r0 = part_off(nrows, G, s), rs = part_off(nrows, G, s + 1) - r0;
        const int64_t c0 = part_off(ncols, G, s), ms = part_off(ncols, G, s + 1) - c0;
        if (rs * mr) check(nccl().Send(pk + r0 * mr, (size_t)(rs * mr), ncclDouble, s, c->comm, st), "ncclSend");
        // source s's block is an Rr x ms column-major slab: columns [c0, c0 + ms) of `rows`
        if (Rr * ms) check(nccl().Recv(rows + c0 * Rr, (size_t)(Rr * ms), ncclDouble, s, c->comm, st), "ncclRecv");
    }
    check(nccl().GroupEnd(), "ncclGroupEnd");
    W4_COMM_END
}

// Row shard -> column shard, the inverse of comm_cols_to_rows.
int wc4dvar_gpu_comm_rows_to_cols(wc4dvar_comm* c, const double* rows, int64_t nrows, int64_t ncols, double* cols,
                                  void* stream) {
    W4_COMM_BEGIN
    require(c && nrows >= 0 && ncols >= 0, "comm_rows_to_cols: bad arguments");
    DeviceGuard g(c->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int G = c->size, r = c->rank;
    const int64_t mr = part_off(ncols, G, r + 1) - part_off(ncols, G, r);
    const int64_t Rr = part_off(nrows, G, r + 1) - part_off(nrows, G, r);
    double* up = c->unpack.get<double>((size_t)std::max<int64_t>(nrows * mr, 1));
    check(nccl().GroupStart(), "ncclGroupStart");
    for (int s = 0; s < G; ++s) {
        const int64_t r0 = part_off(nrows, G, s), rs = part_off(nrows, G, s + 1) - r0;
        const int64_t c0 = part_off(ncols, G, s), ms = part_off(ncols, G, s + 1) - c0;
        if (Rr * ms) check(nccl().Send(rows + c0 * Rr, (size_t)(Rr * ms), ncclDouble, s, c->comm, st), "ncclSend");
        if (rs * mr) check(nccl().Recv(up + r0 * mr, (size_t)(rs * mr), ncclDouble, s, c->comm, st), "ncclRecv");
    }
    check(nccl().GroupEnd(), "ncclGroupEnd");
    for (int s = 0; s < G; ++s) {
        const int64_t r0 = part_off(nrows, G, s), rs = part_off(nrows, G, s + 1) - r0;
        if (rs * mr)
            W4_CUDA(cudaMemcpy2DAsync(cols + r0, nrows * sizeof(double), up + r0 * mr, rs * sizeof(double),
                                      rs * sizeof(double), mr, cudaMemcpyDeviceToDevice, st));
    }
    W4_COMM_END
}

}  // extern "C"
