// C-ABI entry points (include/wc4dvar_gpu.h).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <sstream>
#include <vector>

#include "l96.cuh"
#include "lanczos.cuh"
#include "lmp_pcg.cuh"
#include "ops.cuh"
#include "pcg.cuh"
#include "sketch.cuh"

namespace w4 {
void gaussian_fill(int64_t count, uint64_t seed, double* out);
double probe_dmma_tflops();
}

using namespace w4;

#define W4_API_BEGIN try {
#define W4_API_END                         \
    return WC4DVAR_OK;                     \
    }                                      \
    catch (const w4::InvalidArgument& e) { \
        w4::set_last_error(e.what());      \
        return WC4DVAR_INVALID_ARGUMENT;   \
    }                                      \
    catch (const w4::NumericalError& e) {  \
        w4::set_last_error(e.what());      \
        return WC4DVAR_NUMERICAL;          \
    }                                      \
    catch (const std::exception& e) {      \
        w4::set_last_error(e.what());      \
        return WC4DVAR_DEVICE;             \
    }

namespace w4 {
void gaussian_block_dev(int64_t n_total, int64_t row0, int64_t rows, int64_t col0, int64_t cols,
                        uint64_t seed, double* out, int64_t ldo, bool raw, cudaStream_t st);
}

namespace {

thread_local SketchTiming g_sketch_timing;

template <class T>
T* dev_upload(const T* host, size_t count, cudaStream_t st) {
    T* d = nullptr;
    W4_CUDA(cudaMalloc(&d, sizeof(T) * std::max<size_t>(count, 1)));
    if (count) W4_CUDA(cudaMemcpyAsync(d, host, sizeof(T) * count, cudaMemcpyHostToDevice, st));
    return d;
}

// Copy a host col-major (rows x cols, ld) block into a contiguous device buffer.
void h2d_block(double* dst, const double* src, int64_t rows, int64_t cols, int64_t ld,
               cudaStream_t st) {
    if (rows * cols == 0) return;
    W4_CUDA(cudaMemcpy2DAsync(dst, rows * sizeof(double), src, ld * sizeof(double),
                              rows * sizeof(double), cols, cudaMemcpyHostToDevice, st));
}
void d2h_block(double* dst, int64_t ld, const double* src, int64_t rows, int64_t cols,
               cudaStream_t st) {
    if (rows * cols == 0) return;
    W4_CUDA(cudaMemcpy2DAsync(dst, ld * sizeof(double), src, rows * sizeof(double),
                              rows * sizeof(double), cols, cudaMemcpyDeviceToHost, st));
}

bool overlaps(const double* a, int64_t lda, int64_t ma, const double* b, int64_t ldb, int64_t mb,
              int64_t rows) {
    if (!a || !b || ma == 0 || mb == 0) return false;
    const double* ae = a + (ma - 1) * lda + rows;
    const double* be = b + (mb - 1) * ldb + rows;
    return a < be && b < ae;
}

cudaStream_t pick(wc4dvar_op* op, void* s) {
    return s ? static_cast<cudaStream_t>(s) : op->stream;
}

}  // namespace

extern "C" {

const char* wc4dvar_gpu_last_error(void) { return w4::last_error_cstr(); }

const char* wc4dvar_gpu_version(void) { return "wc4dvar-b200 0.1 (sm_100a, fp64 DMMA)"; }

int wc4dvar_gpu_hessian_create(const wc4dvar_model_desc* model, const wc4dvar_network_desc* net,
                               const wc4dvar_cov_desc* bh, const wc4dvar_cov_desc* qh,
                               double sigma_obs, int device, wc4dvar_op** out) {
    W4_API_BEGIN
    require(model && net && bh && qh && out, "HessianOperator: null descriptor");
    *out = nullptr;
    // HessianOperator ctor checks (operators.cpp:64-77)
    require(sigma_obs > 0.0, "HessianOperator: sigma_obs must be positive");
    require(model->n >= 1 && model->N >= 0, "HessianOperator: bad window");
    require(model->substeps >= 1, "HessianOperator: substeps must be >= 1");
    require(bh->half != nullptr, "HessianOperator: background factor mismatch");
    require(qh->half != nullptr, "HessianOperator: model-error factor mismatch");
    require(bh->kind == qh->kind, "HessianOperator: factors must share a representation");
    require(net->n == model->n && net->N == model->N, "HessianOperator: network/window mismatch");
    require(model->kind >= WC4DVAR_MODEL_IDENTITY && model->kind <= WC4DVAR_MODEL_LORENZ96,
            "HessianOperator: unknown model kind");
    require(model->kind != WC4DVAR_MODEL_LORENZ96 || ((model->stages || model->trajectory) && model->dt > 0.0),
            "Lorenz96Linearized: stages (or the trajectory) and dt are required");
    require(model->kind != WC4DVAR_MODEL_LORENZ96 || model->stages || model->ld_trajectory >= model->n,
            "Lorenz96Linearized: ld_trajectory < n");
    require(model->kind != WC4DVAR_MODEL_LORENZ96 || model->n >= 4, "Lorenz96Model: n must be >= 4");
    require(bh->kind == WC4DVAR_COV_DENSE || bh->kind == WC4DVAR_COV_CIRCULANT,
            "HessianOperator: unknown covariance representation");
    const int64_t n = model->n;
    const int N = model->N;
    for (int a = 0; a < net->n_times; ++a) {
        require(net->times[a] >= 0 && net->times[a] <= N, "ObservationNetwork: time out of window");
        if (a) require(net->times[a] > net->times[a - 1], "ObservationNetwork: times must ascend");
    }
    for (int b = 0; b < net->n_points; ++b) {
        require(net->points[b] >= 0 && net->points[b] < n, "ObservationNetwork: point outside grid");
        if (b) require(net->points[b] > net->points[b - 1], "ObservationNetwork: points must ascend");
    }
    DeviceGuard g(device);
    std::unique_ptr<HessianOp> h(new HessianOp());
    h->init_common(device, n * (N + 1));
    cudaStream_t st = h->stream;
    h->n = n;
    h->N = N;
    h->sigma_obs = sigma_obs;
    h->cov_kind = bh->kind;
    h->md.kind = model->kind;
    h->md.n = n;
    h->md.N = N;
    h->md.s = model->substeps;
    h->md.c = model->courant;
    h->md.d = model->diffusion;
    h->md.dt = model->dt;
    if (model->kind == WC4DVAR_MODEL_LORENZ96) {
        const int64_t nst = (int64_t)N * model->substeps;
        if (model->stages) {
            h->d_stages = dev_upload(model->stages, (size_t)nst * 4 * n, st);
        } else {
            // Lorenz96Linearized ctor (operators.cpp:44-51): stages of trajectory columns
            // 0 .. N s - 1, computed on the device
            W4_CUDA(cudaMalloc(&h->d_stages, sizeof(double) * std::max<size_t>((size_t)nst * 4 * n, 1)));
            const double* tr = model->trajectory;
            int64_t ldt = model->ld_trajectory;
            double* tmp = nullptr;
            if (!model->trajectory_on_device) {
                W4_CUDA(cudaMalloc(&tmp, sizeof(double) * (size_t)n * (nst + 1)));
                h2d_block(tmp, model->trajectory, n, nst + 1, ldt, st);
                tr = tmp;
                ldt = n;
            }
            l96_stages_dev(n, model->forcing, model->dt, tr, ldt, nst, h->d_stages, st);
            if (tmp) {
                W4_CUDA(cudaStreamSynchronize(st));
                cudaFree(tmp);
            }
        }
        h->md.stages = h->d_stages;
    }
    h->times.assign(net->times, net->times + net->n_times);
    h->points.assign(net->points, net->points + net->n_points);
    std::vector<int> slot(N + 1, -1), pmap(n, -1);
    for (int a = 0; a < net->n_times; ++a) slot[net->times[a]] = a;
    for (int b = 0; b < net->n_points; ++b) pmap[net->points[b]] = b;
    h->d_slot = dev_upload(slot.data(), slot.size(), st);
    h->d_pmap = dev_upload(pmap.data(), pmap.size(), st);
    h->d_times = dev_upload(h->times.data(), h->times.size(), st);
    h->d_points = dev_upload(h->points.data(), h->points.size(), st);
    h->nd.n_times = net->n_times;
    h->nd.n_points = net->n_points;
    h->nd.q = (int64_t)net->n_times * net->n_points;
    h->nd.slot = h->d_slot;
    h->nd.pmap = h->d_pmap;
    {  // regular spatial network (models.cpp:159-176): points = 0, sx, 2 sx, ... < n
        const int np = net->n_points;
        int sx = np >= 2 ? net->points[1] - net->points[0] : (np == 1 ? (int)n : 0);
        bool reg = np >= 1 && net->points[0] == 0 && sx >= 1 && (int64_t)np == (n + sx - 1) / sx;
        for (int b = 0; reg && b < np; ++b) reg = net->points[b] == b * sx;
        h->nd.sx = reg ? sx : 0;
    }
    if (bh->kind == WC4DVAR_COV_CIRCULANT) {
        h->circ = new CirculantPlan();
        h->circ->init(n, bh->half, qh->half, bh->half_inv, qh->half_inv, st);
        h->setup_spectral(st);
        W4_CUDA(cudaStreamSynchronize(st));
        *out = h.release();
        return WC4DVAR_OK;
    }
    const size_t fsz = (size_t)n * n;
    // sym_sqrt symmetrises its factors exactly (covariance.cpp:101-102); when a factor is
    // bitwise symmetric the D^{1/2} GEMM may read its columns as rows.
    auto is_sym = [n](const double* F) {
        if (!F) return false;
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = j + 1; i < n; ++i)
                if (F[i + j * n] != F[j + i * n]) return false;
        return true;
    };
    h->sym[0] = is_sym(bh->half);
    h->sym[1] = is_sym(qh->half);
    h->sym[2] = is_sym(bh->half_inv);
    h->sym[3] = is_sym(qh->half_inv);
    h->b_half = dev_upload(bh->half, fsz, st);
    h->q_half = dev_upload(qh->half, fsz, st);
    if (bh->half_inv) h->b_half_inv = dev_upload(bh->half_inv, fsz, st);
    if (qh->half_inv) h->q_half_inv = dev_upload(qh->half_inv, fsz, st);
    W4_CUDA(cudaStreamSynchronize(st));
    *out = h.release();
    W4_API_END
}

int wc4dvar_gpu_dense_create(int64_t n, const double* A, int64_t lda, int device,
                             wc4dvar_op** out) {
    W4_API_BEGIN
    require(out && A && n >= 0 && lda >= n, "DenseOperator: bad arguments");
    *out = nullptr;
    DeviceGuard g(device);
    std::unique_ptr<DenseOp> d(new DenseOp());
    d->init_common(device, n);
    W4_CUDA(cudaMalloc(&d->A, sizeof(double) * std::max<int64_t>(n * n, 1)));
    h2d_block(d->A, A, n, n, lda, d->stream);
    W4_CUDA(cudaStreamSynchronize(d->stream));
    *out = d.release();
    W4_API_END
}

int wc4dvar_gpu_op_destroy(wc4dvar_op* op) {
    W4_API_BEGIN
    delete op;
    W4_API_END
}

int64_t wc4dvar_gpu_op_dim(const wc4dvar_op* op) { return op ? op->dim : -1; }
int64_t wc4dvar_gpu_op_apply_count(const wc4dvar_op* op) { return op ? op->applies.load() : -1; }
void wc4dvar_gpu_op_reset_apply_count(wc4dvar_op* op) {
    if (op) op->applies.store(0);
}
int wc4dvar_gpu_op_device(const wc4dvar_op* op) { return op ? op->device : -1; }

int wc4dvar_gpu_op_release_workspaces(wc4dvar_op* op) {
    W4_API_BEGIN
    require(op != nullptr, "release_workspaces: null operator");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    W4_CUDA(cudaStreamSynchronize(op->stream));
    op->release_workspaces();
    W4_API_END
}

int wc4dvar_gpu_op_apply_block(wc4dvar_op* op, const double* V, int64_t ldv, int64_t m,
                               double* out, int64_t ldo) {
    W4_API_BEGIN
    require(op != nullptr, "apply_block: null operator");
    require(m >= 0 && ldv >= op->dim && ldo >= op->dim,
            "LinearOperator::apply_block: dimension mismatch");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    op->applies += m;
    if (m == 0 || op->dim == 0) return WC4DVAR_OK;
    cudaStream_t st = op->stream;
    // Copy/compute pipeline for wide blocks: the columns go through a two-slot device ring
    // in `nch` chunks; chunk c+1's host->device copy and chunk c-1's device->host copy run
    // on their own streams while chunk c computes.  Each column's arithmetic is unchanged
    // (bitwise), and the device staging stays bounded (2 x 2 slots of <= kStageBytes) for
    // blocks far larger than HBM headroom (C4: n_A x 256 = 34.8 GB each way, PCIe-bound:
    // 48 GB/s per direction with both directions busy, tools/pcie_probe.py).
    // WC4DVAR_PIPELINE_CHUNKS (default 2; 1 = off) is the chunk count below that bound.
    static const int chunks_env = [] {
        const char* e = std::getenv("WC4DVAR_PIPELINE_CHUNKS");
        return e ? std::atoi(e) : 2;
    }();
    // WC4DVAR_PIPELINE_STAGE_MB: device bytes per chunk slot (default 512; C4 k = 256 e2e step
    // 840 / 778 / 749 ms at 4096 / 1024 / 512 MB against a 722 ms PCIe floor): small enough that
    // the ramp (first H2D) and the tail (last compute + D2H) are short against a step of
    // full-duplex PCIe traffic, large enough that every chunk fills the GPU (C4: 2 columns)
    static const size_t kStageBytes = [] {
        const char* e = std::getenv("WC4DVAR_PIPELINE_STAGE_MB");
        return (size_t)(e ? std::max(64, std::atoi(e)) : 512) << 20;
    }();
    int64_t cmax = std::max<int64_t>(1, (int64_t)(kStageBytes / (sizeof(double) * (size_t)op->dim)));
    if (cmax > 1 && (cmax & 1)) --cmax;  // even chunks: the Fourier-space apply packs columns in pairs
    int64_t nch = cdiv(m, cmax);
    if (nch == 1 && m >= 32 && chunks_env > 1) nch = std::min<int64_t>(chunks_env, 4);
    if (op->prof && m <= cmax) nch = 1;  // stage timers see one apply
    if (nch > 1) {
        op->ensure_pipeline();
        op->reset_status(st);
        const int64_t cw = cdiv(m, nch);
        double* din = op->in_buf.get<double>((size_t)op->dim * cw * 2);
        double* dout = op->out_buf.get<double>((size_t)op->dim * cw * 2);
        cudaEvent_t* in_ready = op->pipe_ev;       // [0, 2)
        cudaEvent_t* computed = op->pipe_ev + 2;   // [2, 4)
        cudaEvent_t* drained = op->pipe_ev + 4;    // [4, 6)
        for (int64_t c = 0; c < nch; ++c) {
            const int slot = (int)(c & 1);
            const int64_t c0 = m * c / nch, w = m * (c + 1) / nch - c0;
            double* di = din + (size_t)slot * op->dim * cw;
            double* dq = dout + (size_t)slot * op->dim * cw;
            if (c >= 2) W4_CUDA(cudaStreamWaitEvent(op->pipe_in, computed[slot], 0));
            h2d_block(di, V + c0 * ldv, op->dim, w, ldv, op->pipe_in);
            W4_CUDA(cudaEventRecord(in_ready[slot], op->pipe_in));
            W4_CUDA(cudaStreamWaitEvent(st, in_ready[slot], 0));
            if (c >= 2) W4_CUDA(cudaStreamWaitEvent(st, drained[slot], 0));
            op->apply_block_dev(di, op->dim, w, dq, op->dim, st);
            W4_CUDA(cudaEventRecord(computed[slot], st));
            W4_CUDA(cudaStreamWaitEvent(op->pipe_out, computed[slot], 0));
            d2h_block(out + c0 * ldo, ldo, dq, op->dim, w, op->pipe_out);
            W4_CUDA(cudaEventRecord(drained[slot], op->pipe_out));
        }
        W4_CUDA(cudaStreamSynchronize(op->pipe_out));
        op->check_status(st);
        return WC4DVAR_OK;
    }
    double* din = op->in_buf.get<double>((size_t)op->dim * m);
    double* dout = op->out_buf.get<double>((size_t)op->dim * m);
    h2d_block(din, V, op->dim, m, ldv, st);
    op->reset_status(st);
    op->apply_block_dev(din, op->dim, m, dout, op->dim, st);
    d2h_block(out, ldo, dout, op->dim, m, st);
    op->check_status(st);
    W4_API_END
}

int wc4dvar_gpu_op_apply(wc4dvar_op* op, const double* in, double* out) {
    return wc4dvar_gpu_op_apply_block(op, in, op ? op->dim : 0, 1, out, op ? op->dim : 0);
}

int wc4dvar_gpu_op_apply_block_dev(wc4dvar_op* op, const double* V, int64_t ldv, int64_t m,
                                   double* out, int64_t ldo, void* stream) {
    W4_API_BEGIN
    require(op != nullptr, "apply_block: null operator");
    require(m >= 0 && ldv >= op->dim && ldo >= op->dim,
            "LinearOperator::apply_block: dimension mismatch");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    op->applies += m;
    if (m == 0 || op->dim == 0) return WC4DVAR_OK;
    cudaStream_t st = pick(op, stream);
    const double* src = V;
    int64_t lds = ldv;
    if (overlaps(V, ldv, m, out, ldo, m, op->dim)) {
        double* tmp = op->in_buf.get<double>((size_t)op->dim * m);
        W4_CUDA(cudaMemcpy2DAsync(tmp, op->dim * 8, V, ldv * 8, op->dim * 8, m,
                                  cudaMemcpyDeviceToDevice, st));
        src = tmp;
        lds = op->dim;
    }
    op->reset_status(st);
    op->apply_block_dev(src, lds, m, out, ldo, st);
    op->check_status(st);
    W4_API_END
}

int wc4dvar_gpu_hessian_piece_dev(wc4dvar_op* op, int which, const double* V, int64_t ldv,
                                  int64_t m, double* out, int64_t ldo, void* stream) {
    W4_API_BEGIN
    HessianOp* h = dynamic_cast<HessianOp*>(op);
    require(h != nullptr, "hessian piece: operator is not a HessianOperator");
    static const char* names[] = {"apply_Linv", "apply_LinvT", "apply_D_half", "apply_D_half_inv", "sweeps"};
    require(which >= 0 && which <= 4, "hessian piece: unknown selector");
    require(m >= 0 && ldv >= op->dim && ldo >= op->dim,
            std::string(names[which]) + ": window length mismatch");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    if (m == 0) return WC4DVAR_OK;
    cudaStream_t st = pick(op, stream);
    const double* src = V;
    int64_t lds = ldv;
    if (overlaps(V, ldv, m, out, ldo, m, op->dim)) {
        double* tmp = op->in_buf.get<double>((size_t)op->dim * m);
        W4_CUDA(cudaMemcpy2DAsync(tmp, op->dim * 8, V, ldv * 8, op->dim * 8, m,
                                  cudaMemcpyDeviceToDevice, st));
        src = tmp;
        lds = op->dim;
    }
    op->reset_status(st);
    h->piece_dev(which, src, lds, m, out, ldo, st);
    if (which == WC4DVAR_SWEEPS) op->check_status(st);  // the apply's stage-tagged finite checks
    else W4_CUDA(cudaStreamSynchronize(st));
    W4_API_END
}

int wc4dvar_gpu_factor_apply_dev(wc4dvar_op* op, int which, int inv, const double* X, int64_t ldx, int64_t c,
                                 double* out, int64_t ldo, void* stream) {
    W4_API_BEGIN
    HessianOp* h = dynamic_cast<HessianOp*>(op);
    require(h != nullptr, "factor apply: operator is not a HessianOperator");
    require(which == 0 || which == 1, "factor apply: which must be 0 (B) or 1 (Q)");
    require(c >= 0 && ldx >= h->n && ldo >= h->n && (c == 0 || (X && out)), "factor apply: bad arguments");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    cudaStream_t st = pick(op, stream);
    const double* src = X;
    if (overlaps(X, ldx, c, out, ldo, c, h->n)) {
        double* tmp = op->in_buf.get<double>((size_t)h->n * c);
        W4_CUDA(cudaMemcpy2DAsync(tmp, h->n * 8, X, ldx * 8, h->n * 8, c, cudaMemcpyDeviceToDevice, st));
        src = tmp;
        ldx = h->n;
    }
    h->factor_apply(which, inv != 0, src, ldx, c, out, ldo, st);
    W4_CUDA(cudaStreamSynchronize(st));
    W4_API_END
}

int wc4dvar_gpu_observe_dev(wc4dvar_op* op, const double* traj, double* y, void* stream) {
    W4_API_BEGIN
    HessianOp* h = dynamic_cast<HessianOp*>(op);
    require(h != nullptr, "observe: operator is not a HessianOperator");
    require(traj && (y || h->nd.q == 0), "observe: null argument");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    h->observe_dev(traj, y, pick(op, stream));
    W4_API_END
}

int wc4dvar_gpu_observe(wc4dvar_op* op, const double* traj, double* y) {
    W4_API_BEGIN
    HessianOp* h = dynamic_cast<HessianOp*>(op);
    require(h != nullptr, "observe: operator is not a HessianOperator");
    require(traj && (y || h->nd.q == 0), "observe: null argument");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    const int64_t q = h->nd.q;
    if (q == 0) return WC4DVAR_OK;
    double* dt = op->in_buf.get<double>((size_t)op->dim);
    double* dy = op->out_buf.get<double>((size_t)q);
    W4_CUDA(cudaMemcpyAsync(dt, traj, sizeof(double) * op->dim, cudaMemcpyHostToDevice, op->stream));
    h->observe_dev(dt, dy, op->stream);
    W4_CUDA(cudaMemcpyAsync(y, dy, sizeof(double) * q, cudaMemcpyDeviceToHost, op->stream));
    W4_CUDA(cudaStreamSynchronize(op->stream));
    W4_API_END
}

int wc4dvar_gpu_observation_range_dev(wc4dvar_op* op, double* W, int64_t ldw, void* stream) {
    W4_API_BEGIN
    HessianOp* h = dynamic_cast<HessianOp*>(op);
    require(h != nullptr, "observation_range: operator is not a HessianOperator");
    require(ldw >= op->dim && (W || h->nd.q == 0), "observation_range: bad output");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    cudaStream_t st = pick(op, stream);
    op->reset_status(st);
    h->observation_range_dev(W, ldw, st);
    op->check_status(st);
    W4_API_END
}

int wc4dvar_gpu_observation_range(wc4dvar_op* op, double* W, int64_t ldw) {
    W4_API_BEGIN
    HessianOp* h = dynamic_cast<HessianOp*>(op);
    require(h != nullptr, "observation_range: operator is not a HessianOperator");
    require(ldw >= op->dim && (W || h->nd.q == 0), "observation_range: bad output");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    const int64_t q = h->nd.q;
    if (q == 0) return WC4DVAR_OK;
    double* dw = op->out_buf.get<double>((size_t)op->dim * q);
    const int rc = wc4dvar_gpu_observation_range_dev(op, dw, op->dim, nullptr);
    if (rc != WC4DVAR_OK) return rc;
    d2h_block(W, ldw, dw, op->dim, q, op->stream);
    W4_CUDA(cudaStreamSynchronize(op->stream));
    W4_API_END
}

int wc4dvar_gpu_clustered_spectrum(wc4dvar_op* op, const wc4dvar_lmp* precond, const double* obs_range,
                                   int64_t ldw, double* nonunit, int64_t* n_nonunit, int64_t* unit_multiplicity) {
    W4_API_BEGIN
    HessianOp* h = dynamic_cast<HessianOp*>(op);
    require(h != nullptr, "clustered_spectrum: operator is not a HessianOperator");
    require(nonunit && n_nonunit && unit_multiplicity, "clustered_spectrum: null output");
    require(!obs_range || ldw >= op->dim, "clustered_spectrum: observation range mismatch");
    require(!precond || precond->n == op->dim, "clustered_spectrum: preconditioner dimension mismatch");
    require(!precond || precond->device == op->device, "clustered_spectrum: preconditioner on another device");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    cudaStream_t st = op->stream;
    const int64_t n = op->dim, q = h->nd.q;
    const int64_t k = precond ? precond->k : 0;  // identity LMP: k = 0 (spectrum.cpp:36)
    double* W = op->in_buf.get<double>((size_t)n * std::max<int64_t>(q, 1));
    if (obs_range) {
        h2d_block(W, obs_range, n, q, ldw, st);
    } else {
        op->reset_status(st);
        h->observation_range_dev(W, n, st);
        op->check_status(st);
    }
    if (precond && k) W4_CUDA(cudaStreamSynchronize(precond->stream));  // U / T built on the LMP stream
    double* vals = op->out_buf.get<double>((size_t)std::max<int64_t>(q + k, 1));
    double* Ucol = nullptr;  // the spectrum's tall GEMMs take U column-major
    if (k) {
        W4_CUDA(cudaMallocAsync(&Ucol, sizeof(double) * n * k, st));
        lmp_unblock_U(n, (int)k, precond->U, Ucol, n, st);
    }
    clustered_spectrum_dev(*op, W, q, Ucol, k, precond ? precond->T : nullptr, vals, st);
    if (Ucol) W4_CUDA(cudaFreeAsync(Ucol, st));
    W4_CUDA(cudaMemcpyAsync(nonunit, vals, sizeof(double) * (q + k), cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    *n_nonunit = q + k;
    *unit_multiplicity = n - (q + k);
    W4_API_END
}

int wc4dvar_gpu_hessian_piece(wc4dvar_op* op, int which, const double* V, int64_t ldv, int64_t m,
                              double* out, int64_t ldo) {
    W4_API_BEGIN
    require(op != nullptr, "hessian piece: null operator");
    require(m >= 0 && ldv >= op->dim && ldo >= op->dim, "hessian piece: window length mismatch");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    if (m == 0) return WC4DVAR_OK;
    double* din = op->in_buf.get<double>((size_t)op->dim * m);
    double* dout = op->out_buf.get<double>((size_t)op->dim * m);
    h2d_block(din, V, op->dim, m, ldv, op->stream);
    const int rc = wc4dvar_gpu_hessian_piece_dev(op, which, din, op->dim, m, dout, op->dim, nullptr);
    if (rc != WC4DVAR_OK) return rc;
    d2h_block(out, ldo, dout, op->dim, m, op->stream);
    W4_CUDA(cudaStreamSynchronize(op->stream));
    W4_API_END
}

int wc4dvar_gpu_op_spectral(wc4dvar_op* op, int mode, int* active) {
    W4_API_BEGIN
    require(op != nullptr, "op_spectral: null operator");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    HessianOp* h = dynamic_cast<HessianOp*>(op);
    if (mode >= 0) {
        require(h != nullptr || mode == 0, "op_spectral: not a HessianOperator");
        if (h) {
            require(mode == 0 || h->d_mhat != nullptr,
                    "op_spectral: operator is not eligible (needs a periodic stencil model, circulant "
                    "factors with a fused transform and a regular network whose stride divides n)");
            h->spectral = mode != 0;
        }
    }
    if (active) *active = (h && h->spectral) ? 1 : 0;
    W4_API_END
}

int wc4dvar_gpu_op_profile(wc4dvar_op* op, int enable) {
    W4_API_BEGIN
    require(op != nullptr, "op_profile: null operator");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    if (enable && !op->pev[0])
        for (auto& e : op->pev) W4_CUDA(cudaEventCreate(&e));
    op->prof = enable != 0;
    op->prof_pending = false;
    op->prof_ms[0] = op->prof_ms[1] = op->prof_ms[2] = 0;
    op->prof_calls = 0;
    W4_API_END
}

int wc4dvar_gpu_op_profile_read(wc4dvar_op* op, double* ms3, int64_t* calls) {
    W4_API_BEGIN
    require(op && ms3 && calls, "op_profile_read: null argument");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    for (int i = 0; i < 3; ++i) ms3[i] = op->prof_ms[i];
    *calls = op->prof_calls;
    W4_API_END
}

int wc4dvar_gpu_probe_dmma_peak(int device, double* tflops) {
    W4_API_BEGIN
    require(tflops != nullptr, "probe_dmma_peak: null");
    DeviceGuard g(device);
    *tflops = w4::probe_dmma_tflops();
    W4_API_END
}

int wc4dvar_gpu_l96_trajectory_dev(int64_t n, double forcing, double dt, const double* x0, int64_t spinup,
                                   int64_t steps, double* traj, int64_t ldt, int device, void* stream) {
    W4_API_BEGIN
    require(n >= 4, "lorenz96_rhs: n must be >= 4");
    require(spinup >= 0 && steps >= 0 && ldt >= n && x0 && traj, "l96_trajectory: bad arguments");
    DeviceGuard g(device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    DevBuf work;
    l96_trajectory_dev(n, forcing, dt, x0, spinup, steps, traj, ldt, spinup > 1 ? work.get<double>(n) : nullptr, st);
    W4_CUDA(cudaStreamSynchronize(st));  // work is released on return
    W4_API_END
}

int wc4dvar_gpu_l96_trajectory(int64_t n, double forcing, double dt, const double* x0, int64_t spinup,
                               int64_t steps, double* traj, int64_t ldt, int device) {
    W4_API_BEGIN
    require(n >= 4, "lorenz96_rhs: n must be >= 4");
    require(spinup >= 0 && steps >= 0 && ldt >= n && x0 && traj, "l96_trajectory: bad arguments");
    DeviceGuard g(device);
    cudaStream_t st = nullptr;
    W4_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::unique_ptr<CUstream_st, void (*)(cudaStream_t)> sguard(st, [](cudaStream_t s) { cudaStreamDestroy(s); });
    DevBuf dx0, dtraj, work;
    double* x = dx0.get<double>(n);
    double* tr = dtraj.get<double>((size_t)n * (steps + 1));
    W4_CUDA(cudaMemcpyAsync(x, x0, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    l96_trajectory_dev(n, forcing, dt, x, spinup, steps, tr, n, spinup > 1 ? work.get<double>(n) : nullptr, st);
    d2h_block(traj, ldt, tr, n, steps + 1, st);
    W4_CUDA(cudaStreamSynchronize(st));
    W4_API_END
}

int wc4dvar_gpu_l96_integrate_p(int64_t n, int32_t N, int32_t substeps, double forcing, double dt, const double* p,
                                double* traj, int64_t ldt, int device) {
    W4_API_BEGIN
    require(n >= 4, "lorenz96_rhs: n must be >= 4");
    require(N >= 0 && substeps >= 1 && ldt >= n && p && traj, "integrate_p: bad arguments");
    DeviceGuard g(device);
    cudaStream_t st = nullptr;
    W4_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::unique_ptr<CUstream_st, void (*)(cudaStream_t)> sguard(st, [](cudaStream_t s) { cudaStreamDestroy(s); });
    const int64_t cols = (int64_t)N * substeps + 1;
    DevBuf dp, dtraj, dstat;
    double* pd = dp.get<double>((size_t)n * (N + 1));
    double* tr = dtraj.get<double>((size_t)n * cols);
    unsigned* stat = dstat.get<unsigned>(std::max(N, 1));
    W4_CUDA(cudaMemsetAsync(stat, 0, sizeof(unsigned) * std::max(N, 1), st));
    W4_CUDA(cudaMemcpyAsync(pd, p, sizeof(double) * n * (N + 1), cudaMemcpyHostToDevice, st));
    l96_integrate_p_dev(n, N, substeps, forcing, dt, pd, tr, n, stat, st);
    std::vector<unsigned> hs(std::max(N, 1));
    W4_CUDA(cudaMemcpyAsync(hs.data(), stat, sizeof(unsigned) * hs.size(), cudaMemcpyDeviceToHost, st));
    d2h_block(traj, ldt, tr, n, cols, st);
    W4_CUDA(cudaStreamSynchronize(st));
    for (int i = 0; i < N; ++i)
        if (hs[i]) throw NumericalError("integrate_p: non-finite trajectory at step " + std::to_string(i + 1));
    W4_API_END
}

int wc4dvar_gpu_gaussian_matrix(int64_t rows, int64_t cols, uint64_t seed, double* out) {
    W4_API_BEGIN
    require(rows >= 0 && cols >= 0 && (out || rows * cols == 0), "gaussian_matrix: bad arguments");
    w4::gaussian_fill(rows * cols, seed, out);
    W4_API_END
}

int wc4dvar_gpu_sketch_dev(wc4dvar_op* op, const wc4dvar_sketch_config* cfg,
                           const double* omega_dev, double* U_dev, int64_t ldu, double* theta_dev,
                           int64_t* k_out, void* stream) {
    W4_API_BEGIN
    require(op && cfg && omega_dev && U_dev && theta_dev && k_out, "sketch: null argument");
    require(ldu >= op->dim, "sketch: ldu < dim");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    g_sketch_timing = SketchTiming{};
    *k_out = sketch_dev(*op, *cfg, omega_dev, U_dev, ldu, theta_dev, pick(op, stream),
                        &g_sketch_timing);
    W4_API_END
}

int wc4dvar_gpu_sketch(wc4dvar_op* op, const wc4dvar_sketch_config* cfg, const double* omega,
                       double* U, int64_t ldu, double* theta, int64_t* k_out) {
    W4_API_BEGIN
    require(op && cfg && U && theta && k_out, "sketch: null argument");
    require(ldu >= op->dim, "sketch: ldu < dim");
    // SketchConfig::validate before drawing (randevd.cpp:63)
    require(cfg->target_rank >= 1, "SketchConfig: target rank must be >= 1");
    require(cfg->oversample >= 0, "SketchConfig: oversampling must be >= 0");
    const int64_t m = (int64_t)cfg->target_rank + cfg->oversample;
    require(m <= op->dim, "SketchConfig: k + l exceeds operator dimension");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    const int64_t n = op->dim;
    cudaStream_t st = op->stream;
    double* dom = op->in_buf.get<double>((size_t)n * m);
    double* dU = op->out_buf.get<double>((size_t)n * cfg->target_rank + cfg->target_rank);
    double* dth = dU + (size_t)n * cfg->target_rank;
    if (omega) {
        h2d_block(dom, omega, n, m, n, st);
    } else {  // gaussian_matrix(dim, k + l, seed) drawn on the device (jump-ahead NormalStream)
        w4::gaussian_block_dev(n, 0, n, 0, m, cfg->seed, dom, n, false, st);
    }
    g_sketch_timing = SketchTiming{};
    const int64_t kk = sketch_dev(*op, *cfg, dom, dU, n, dth, st, &g_sketch_timing);
    d2h_block(U, ldu, dU, n, kk, st);
    W4_CUDA(cudaMemcpyAsync(theta, dth, sizeof(double) * kk, cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    *k_out = kk;
    W4_API_END
}

int wc4dvar_gpu_rayleigh_ritz(wc4dvar_op* op, const double* Z, int64_t ldz, int64_t m, double* U,
                              int64_t ldu, double* theta) {
    W4_API_BEGIN
    require(op && Z && U && theta, "rayleigh_ritz: null argument");
    require(ldz >= op->dim && ldu >= op->dim, "rayleigh_ritz: dimension mismatch");
    require(m >= 1 && m <= 512, "rayleigh_ritz: 1 <= m <= 512");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    const int64_t n = op->dim;
    cudaStream_t st = op->stream;
    double* dz = op->in_buf.get<double>((size_t)n * m);
    double* dU = op->out_buf.get<double>((size_t)n * m + m);
    double* dth = dU + (size_t)n * m;
    h2d_block(dz, Z, n, m, ldz, st);
    rayleigh_ritz_dev(*op, dz, n, m, dU, n, dth, st);
    d2h_block(U, ldu, dU, n, m, st);
    W4_CUDA(cudaMemcpyAsync(theta, dth, sizeof(double) * m, cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    W4_API_END
}

int wc4dvar_gpu_last_sketch_timing(double* ms5) {
    W4_API_BEGIN
    require(ms5 != nullptr, "last_sketch_timing: null");
    ms5[0] = g_sketch_timing.apply_ms;
    ms5[1] = g_sketch_timing.orth_ms;
    ms5[2] = g_sketch_timing.small_ms;
    ms5[3] = g_sketch_timing.gemm_ms;
    ms5[4] = g_sketch_timing.total_ms;
    W4_API_END
}

// ----------------------------------------------------------------------------- LMP
static int lmp_build_impl(int64_t n, int64_t k, const double* U, int64_t ldu, const double* theta,
                          int device, bool dev_ptrs, wc4dvar_lmp** out) {
    W4_API_BEGIN
    require(out != nullptr && n >= 0 && k >= 0, "build_spectral_lmp: bad arguments");
    *out = nullptr;
    DeviceGuard g(device);
    std::unique_ptr<wc4dvar_lmp> f(new wc4dvar_lmp());
    f->device = device;
    f->n = n;
    f->k = (int)k;
    W4_CUDA(cudaStreamCreateWithFlags(&f->stream, cudaStreamNonBlocking));
    W4_CUDA(cudaMalloc(&f->counter, 4 * sizeof(unsigned)));
    W4_CUDA(cudaMemset(f->counter, 0, 4 * sizeof(unsigned)));
    if (k == 0) {  // LmpFactor::identity (lmp.cpp:28-33, :36)
        *out = f.release();
        return WC4DVAR_OK;
    }
    require(ldu >= n && U && theta, "build_spectral_lmp: bad arguments");
    cudaStream_t st = f->stream;
    std::vector<double> th(k);
    if (dev_ptrs)
        W4_CUDA(cudaMemcpy(th.data(), theta, sizeof(double) * k, cudaMemcpyDeviceToHost));
    else
        std::memcpy(th.data(), theta, sizeof(double) * k);
    const double mn = *std::min_element(th.begin(), th.end());
    if (!(mn > 0.0)) {  // lmp.cpp:37-41
        std::ostringstream m;
        m << "build_spectral_lmp: nonpositive Ritz value " << mn;
        throw NumericalError(m.str());
    }
    // U is kept in the row-tile blocked layout of the PCG row passes (lmp_block_U); a
    // column-major device copy (the caller's, or a staging upload) feeds U^T U and the
    // blocking kernel.
    W4_CUDA(cudaMalloc(&f->U, sizeof(double) * lmp_blocked_size(n, (int)k)));
    W4_CUDA(cudaMalloc(&f->theta, sizeof(double) * k));
    W4_CUDA(cudaMalloc(&f->T, sizeof(double) * k * k));
    const double* Ucol = U;
    int64_t ldc = ldu;
    double* staged = nullptr;
    if (!dev_ptrs) {
        W4_CUDA(cudaMallocAsync(&staged, sizeof(double) * n * k, st));
        W4_CUDA(cudaMemcpy2DAsync(staged, n * 8, U, ldu * 8, n * 8, k, cudaMemcpyHostToDevice, st));
        Ucol = staged;
        ldc = n;
    }
    lmp_block_U(n, (int)k, Ucol, ldc, f->U, st);
    W4_CUDA(cudaMemcpyAsync(f->theta, th.data(), sizeof(double) * k, cudaMemcpyHostToDevice, st));
    double* S = f->tmp.get<double>((size_t)k * k + 1);
    gemm_tn(n, k, k, Ucol, ldc, Ucol, ldc, 1.0, S, k, f->partial, st);
    if (staged) W4_CUDA(cudaFreeAsync(staged, st));
    double* dd = S + k * k;
    defect_max((int)k, S, dd, st);
    double defect = 0;
    W4_CUDA(cudaMemcpyAsync(&defect, dd, sizeof(double), cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    if (!(defect <= 1e-8)) {  // lmp.cpp:42-47
        std::ostringstream m;
        m << "build_spectral_lmp: Ritz vectors not orthonormal (defect " << defect << ")";
        throw NumericalError(m.str());
    }
    lmp_build_T((int)k, S, f->theta, f->T, st);
    W4_CUDA(cudaStreamSynchronize(st));
    *out = f.release();
    W4_API_END
}

int wc4dvar_gpu_lmp_build(int64_t n, int64_t k, const double* U, int64_t ldu, const double* theta,
                          int device, wc4dvar_lmp** out) {
    return lmp_build_impl(n, k, U, ldu, theta, device, false, out);
}

int wc4dvar_gpu_lmp_build_dev(int64_t n, int64_t k, const double* U, int64_t ldu,
                              const double* theta, int device, wc4dvar_lmp** out) {
    return lmp_build_impl(n, k, U, ldu, theta, device, true, out);
}

int wc4dvar_gpu_lmp_destroy(wc4dvar_lmp* f) {
    W4_API_BEGIN
    delete f;
    W4_API_END
}

int wc4dvar_gpu_lmp_apply(wc4dvar_lmp* f, int transpose, const double* v, double* out) {
    W4_API_BEGIN
    require(f && v && out, "LmpFactor::apply: null argument");
    std::lock_guard<std::mutex> lk(f->mu);
    DeviceGuard g(f->device);
    const int64_t n = f->n;
    cudaStream_t st = f->stream;
    if (f->k == 0) {
        std::memmove(out, v, sizeof(double) * n);
        return WC4DVAR_OK;
    }
    double* buf = f->tmp.get<double>((size_t)2 * n + f->k + 1);
    double* dv = buf;
    double* dout = buf + n;
    double* gk = buf + 2 * n;
    W4_CUDA(cudaMemcpyAsync(dv, v, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    RowPassCtx c;
    c.n = n;
    c.k = f->k;
    c.U = f->U;
    c.ldu = n;
    c.blk_rb = lmp_tile_rows(f->k);
    c.T = f->T;
    c.partial = f->partial.get<double>((size_t)std::min<int64_t>(cdiv(n, 32) + 1, 2048) * (f->k + 1));
    c.counter = f->counter;
    rowpass_utv(c, dv, nullptr, nullptr, gk, st);
    rowpass_apply(c, transpose != 0, dv, gk, dout, st);
    W4_CUDA(cudaMemcpyAsync(out, dout, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    W4_API_END
}

// ----------------------------------------------------------------------------- cost
int wc4dvar_gpu_cost_create(wc4dvar_op* op, const double* b, const double* d, wc4dvar_cost** out) {
    W4_API_BEGIN
    HessianOp* h = dynamic_cast<HessianOp*>(op);
    require(h && b && out, "QuadraticCost: bad arguments");
    *out = nullptr;
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    std::unique_ptr<wc4dvar_cost> c(new wc4dvar_cost());
    c->op = h;
    const int64_t n = op->dim, q = h->nd.q;
    cudaStream_t st = op->stream;
    double* db = op->in_buf.get<double>((size_t)n);
    W4_CUDA(cudaMemcpyAsync(db, b, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    W4_CUDA(cudaMalloc(&c->b_tilde, sizeof(double) * n));
    h->piece_dev(WC4DVAR_D_HALF_INV, db, n, 1, c->b_tilde, n, st);  // assimilation.cpp:131
    c->d = dev_upload(d ? d : b, d ? (size_t)q : 0, st);
    W4_CUDA(cudaMalloc(&c->counter, 4 * sizeof(unsigned)));
    W4_CUDA(cudaMemsetAsync(c->counter, 0, 4 * sizeof(unsigned), st));
    W4_CUDA(cudaMalloc(&c->d_val, 2 * sizeof(double)));
    W4_CUDA(cudaStreamSynchronize(st));
    *out = c.release();
    W4_API_END
}

int wc4dvar_gpu_cost_destroy(wc4dvar_cost* c) {
    W4_API_BEGIN
    delete c;
    W4_API_END
}

int wc4dvar_gpu_cost_eval(wc4dvar_cost* c, const double* x, double* value) {
    W4_API_BEGIN
    require(c && x && value, "QuadraticCost: null argument");
    wc4dvar_op* op = c->op;
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    double* dx = op->in_buf.get<double>((size_t)op->dim);
    W4_CUDA(cudaMemcpyAsync(dx, x, sizeof(double) * op->dim, cudaMemcpyHostToDevice, op->stream));
    *value = c->eval_dev(dx, op->stream);
    W4_API_END
}

int wc4dvar_gpu_cost_rhs(wc4dvar_cost* c, double* rhs) {
    W4_API_BEGIN
    require(c && rhs, "QuadraticCost: null argument");
    HessianOp* h = c->op;
    std::lock_guard<std::recursive_mutex> lk(h->mu);
    DeviceGuard g(h->device);
    const int64_t n = h->dim;
    cudaStream_t st = h->stream;
    double* s = h->in_buf.get<double>((size_t)2 * n);
    double* u = s + n;
    // rhs = b~ + r_inv D^{1/2} L^{-T} H^T d  (assimilation.cpp:142-146)
    SweepArgs a;
    a.Y = c->d;
    a.S = s;
    a.lds = n;
    a.do_adj = true;
    a.adj_obs = h->nd.q > 0;
    a.m = 1;
    h->reset_status(st);
    sweep(h->md, h->nd, a, h->d_status, st, &h->sweep_ws);
    h->piece_dev(WC4DVAR_D_HALF, s, n, 1, u, n, st);
    const double r_inv = 1.0 / (h->sigma_obs * h->sigma_obs);
    axpby(n, 1.0, c->b_tilde, r_inv, u, u, st);
    W4_CUDA(cudaMemcpyAsync(rhs, u, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    W4_API_END
}

// ----------------------------------------------------------------------------- PCG
int wc4dvar_gpu_pcg(wc4dvar_op* op, const double* b, wc4dvar_lmp* pre, const double* x0,
                    const wc4dvar_pcg_options* opts, wc4dvar_cost* cost, double* x,
                    wc4dvar_pcg_history* hist) {
    W4_API_BEGIN
    require(op && b && opts && x, "pcg_split: null argument");
    require(!pre || pre->k == 0 || pre->n == op->dim, "pcg_split: preconditioner dimension mismatch");
    require(!cost || cost->op == op, "pcg_split: cost belongs to another operator");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    const int64_t n = op->dim;
    cudaStream_t st = op->stream;
    double* buf = op->out_buf.get<double>((size_t)3 * n);
    double* db = buf;
    double* dx0 = x0 ? buf + n : nullptr;
    double* dx = buf + 2 * n;
    W4_CUDA(cudaMemcpyAsync(db, b, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    if (x0) W4_CUDA(cudaMemcpyAsync(dx0, x0, sizeof(double) * n, cudaMemcpyHostToDevice, st));
    PcgRecord rec;
    pcg_dev(*op, db, pre, dx0, *opts, cost, dx, rec, st);
    W4_CUDA(cudaMemcpyAsync(x, dx, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    if (hist) {
        for (size_t i = 0; i < rec.alphas.size(); ++i) {
            if (hist->alphas) hist->alphas[i] = rec.alphas[i];
            if (hist->betas) hist->betas[i] = rec.betas[i];
        }
        for (size_t i = 0; i < rec.residual_norms.size(); ++i)
            if (hist->residual_norms) hist->residual_norms[i] = rec.residual_norms[i];
        for (size_t i = 0; i < rec.costs.size(); ++i)
            if (hist->quadratic_costs) hist->quadratic_costs[i] = rec.costs[i];
        hist->iterations = rec.iterations;
        hist->converged = rec.converged ? 1 : 0;
        hist->stop_reason = rec.stop_reason;
        hist->n_residuals = 0;
        if (hist->normalized_residuals && rec.nf) {
            require(hist->ld_residuals >= n, "pcg_split: ld_residuals < dim");
            d2h_block(hist->normalized_residuals, hist->ld_residuals, rec.F, n, rec.nf, st);
            W4_CUDA(cudaStreamSynchronize(st));
            hist->n_residuals = rec.nf;
        }
    }
    W4_API_END
}

int wc4dvar_gpu_lanczos_eigenpairs(wc4dvar_op* op, int64_t k, const wc4dvar_lanczos_options* opts, double* U,
                                   int64_t ldu, double* values, int64_t* steps) {
    W4_API_BEGIN
    require(op && opts && U && values, "lanczos_eigenpairs: null argument");
    require(ldu >= op->dim, "lanczos_eigenpairs: ldu < dim");
    std::lock_guard<std::recursive_mutex> lk(op->mu);
    DeviceGuard g(op->device);
    cudaStream_t st = op->stream;
    const int64_t n = op->dim;
    require(k >= 1 && k <= n, "lanczos_eigenpairs: k out of range");
    double* dU = op->out_buf.get<double>((size_t)n * k);
    const int64_t m = lanczos_eigenpairs_dev(*op, k, opts->max_iter, opts->tol, opts->seed, dU, n, values, st);
    d2h_block(U, ldu, dU, n, k, st);
    W4_CUDA(cudaStreamSynchronize(st));
    if (steps) *steps = m;
    W4_API_END
}

int wc4dvar_gpu_ritz_from_tridiagonal(int64_t n, int64_t j, const double* gammas, const double* taus,
                                      const double* residual_basis, int64_t ldf, int64_t k, double* U, int64_t ldu,
                                      double* values, int device) {
    W4_API_BEGIN
    require(j >= 1 && gammas && (j == 1 || taus), "ritz_from_tridiagonal: empty tridiagonal");
    require(k >= 1 && k <= j, "ritz_from_tridiagonal: k out of range");
    require(residual_basis && ldf >= n && n >= 1, "ritz_from_tridiagonal: residual basis shorter than T");
    require(U && values && ldu >= n, "ritz_from_tridiagonal: bad output");
    DeviceGuard g(device);
    cudaStream_t st = nullptr;
    W4_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::unique_ptr<CUstream_st, void (*)(cudaStream_t)> sguard(st, [](cudaStream_t s) { cudaStreamDestroy(s); });
    DevBuf fb, ub;
    double* F = fb.get<double>((size_t)n * j);
    double* dU = ub.get<double>((size_t)n * k);
    h2d_block(F, residual_basis, n, j, ldf, st);
    ritz_from_tridiagonal_dev(n, j, gammas, taus, F, n, k, dU, n, values, st);
    d2h_block(U, ldu, dU, n, k, st);
    W4_CUDA(cudaStreamSynchronize(st));
    W4_API_END
}

}  // extern "C"
