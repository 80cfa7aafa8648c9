// C-ABI of the tall-skinny building blocks used by the row-sharded (multi-GPU) sketches
// (include/wc4dvar_gpu.h, "Row-sharded building blocks").  Each entry is the LOCAL half of
// one dense step of randevd.cpp; the caller all-reduces the m x m results between them
// (paper_2101_07249_b200/distributed.py).  They run the same kernels as the single-GPU
// sketches (sketch.cu), so at world size 1 the distributed methods reproduce sketch_dev.
#include <algorithm>
#include <string>

#include "gemm.cuh"
#include "smallla.cuh"

using namespace w4;

namespace w4 {
void set_last_error(const std::string& msg);
}

#define W4_LA_BEGIN try {
#define W4_LA_END                          \
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

namespace {

// Per-thread, per-device scratch (split-GEMM partials, small-LA workspace, info words).
struct Scratch {
    DevBuf gemm, small, ints;
    PinBuf h;
};
constexpr int kMaxDev = 16;
thread_local Scratch t_scratch[kMaxDev];

Scratch& scratch(int device) {
    require(device >= 0 && device < kMaxDev, "device index out of range");
    return t_scratch[device];
}

int read_int(Scratch& s, const int* d, cudaStream_t st) {
    int* h = s.h.get<int>(2);
    W4_CUDA(cudaMemcpyAsync(h, d, sizeof(int), cudaMemcpyDeviceToHost, st));
    W4_CUDA(cudaStreamSynchronize(st));
    return *h;
}

}  // namespace

extern "C" {

int wc4dvar_gpu_la_gram_dev(int device, int64_t rows, int64_t m1, int64_t m2, const double* A,
                            int64_t lda, const double* B, int64_t ldb, double* G, int64_t ldg,
                            void* stream) {
    W4_LA_BEGIN
    require(rows >= 0 && m1 >= 0 && m2 >= 0, "gram: negative size");
    require(lda >= std::max<int64_t>(rows, 1) && ldb >= std::max<int64_t>(rows, 1) &&
                ldg >= std::max<int64_t>(m1, 1),
            "gram: leading dimension too small");
    DeviceGuard g(device);
    auto st = static_cast<cudaStream_t>(stream);
    if (m1 == 0 || m2 == 0) return WC4DVAR_OK;
    if (rows == 0) {
        W4_CUDA(cudaMemset2DAsync(G, ldg * sizeof(double), 0, m1 * sizeof(double), m2, st));
        return WC4DVAR_OK;
    }
    gemm_tn(rows, m1, m2, A, lda, B, ldb, 1.0, G, ldg, scratch(device).gemm, st);
    W4_LA_END
}

int wc4dvar_gpu_la_tall_times_small_dev(int device, int64_t rows, int64_t k, int64_t ncols,
                                        const double* A, int64_t lda, const double* W, int64_t ldw,
                                        double* C, int64_t ldc, void* stream) {
    W4_LA_BEGIN
    require(rows >= 0 && k >= 1 && ncols >= 0, "tall_times_small: bad size");
    require(lda >= std::max<int64_t>(rows, 1) && ldw >= k && ldc >= std::max<int64_t>(rows, 1),
            "tall_times_small: leading dimension too small");
    require(C != A, "tall_times_small: output must not alias the input");
    DeviceGuard g(device);
    if (rows == 0 || ncols == 0) return WC4DVAR_OK;
    GemmPass p;
    p.A = A;
    p.lda = lda;
    p.M = rows;
    p.K = k;
    p.ncols = ncols;
    p.in = ColMap::plain(W, ldw);
    p.out = ColMap::plain(C, ldc);
    gemm_nn(&p, 1, nullptr, static_cast<cudaStream_t>(stream));
    W4_LA_END
}

int wc4dvar_gpu_la_chol_upper_dev(int device, int64_t m, const double* G, double* R, void* stream) {
    W4_LA_BEGIN
    require(m >= 1 && m <= 512, "chol_upper: m must be in [1, 512]");
    DeviceGuard g(device);
    auto st = static_cast<cudaStream_t>(stream);
    Scratch& s = scratch(device);
    int* info = s.ints.get<int>(4);
    chol_upper((int)m, G, R, info, s.small, st);
    const int bad = read_int(s, info, st);
    if (bad) throw NumericalError("chol_upper: matrix is not positive definite (pivot " +
                                  std::to_string(bad - 1) + ")");
    W4_LA_END
}

int wc4dvar_gpu_la_chol_inv_upper_dev(int device, int64_t m, const double* G, double* R,
                                      double* Rinv, void* stream) {
    W4_LA_BEGIN
    require(m >= 1 && m <= 512, "chol_inv_upper: m must be in [1, 512]");
    DeviceGuard g(device);
    auto st = static_cast<cudaStream_t>(stream);
    Scratch& s = scratch(device);
    int* info = s.ints.get<int>(4);
    chol_inv_upper((int)m, G, R, Rinv, info, s.small, st);
    const int bad = read_int(s, info, st);
    if (bad) throw NumericalError("chol_inv_upper: matrix is not positive definite (pivot " +
                                  std::to_string(bad - 1) + ")");
    W4_LA_END
}

int wc4dvar_gpu_la_tri_inv_upper_dev(int device, int64_t m, const double* R, double* Rinv,
                                     void* stream) {
    W4_LA_BEGIN
    require(m >= 1 && m <= 512, "tri_inv_upper: m must be in [1, 512]");
    DeviceGuard g(device);
    tri_inv_upper((int)m, R, Rinv, static_cast<cudaStream_t>(stream));
    W4_LA_END
}

int wc4dvar_gpu_la_pivoted_rank_dev(int device, int64_t m, const double* G, double tol_rel,
                                    int64_t* rank, int32_t* perm, void* stream) {
    W4_LA_BEGIN
    require(m >= 1 && m <= 512, "pivoted_rank: m must be in [1, 512]");
    require(rank != nullptr && perm != nullptr, "pivoted_rank: null output");
    DeviceGuard g(device);
    auto st = static_cast<cudaStream_t>(stream);
    Scratch& s = scratch(device);
    int* r = s.ints.get<int>(4);
    pivoted_chol_rank((int)m, G, tol_rel, r, perm, s.small, st);
    *rank = read_int(s, r, st);
    W4_LA_END
}

int wc4dvar_gpu_la_sym_evd_dev(int device, int64_t m, const double* K, double* vals, double* W,
                               void* stream) {
    W4_LA_BEGIN
    require(m >= 1 && m <= 512, "sym_evd: m must be in [1, 512]");
    DeviceGuard g(device);
    sym_evd_desc((int)m, K, vals, W, scratch(device).small, static_cast<cudaStream_t>(stream));
    W4_LA_END
}

int wc4dvar_gpu_la_svd_left_dev(int device, int64_t m, const double* X, double* sigma, double* U,
                                void* stream) {
    W4_LA_BEGIN
    require(m >= 1 && m <= 512, "svd_left: m must be in [1, 512]");
    DeviceGuard g(device);
    svd_left_desc((int)m, X, sigma, U, scratch(device).small, static_cast<cudaStream_t>(stream));
    W4_LA_END
}

int wc4dvar_gpu_la_small_gemm_dev(int device, int32_t trans_a, int32_t trans_b, int64_t M,
                                  int64_t N, int64_t K, double alpha, const double* A, int64_t lda,
                                  const double* B, int64_t ldb, double beta, double* C, int64_t ldc,
                                  void* stream) {
    W4_LA_BEGIN
    require(M >= 0 && N >= 0 && K >= 0 && M <= 4096 && N <= 4096 && K <= 4096,
            "small_gemm: sizes must be in [0, 4096]");
    DeviceGuard g(device);
    if (M == 0 || N == 0) return WC4DVAR_OK;
    small_gemm(trans_a != 0, trans_b != 0, (int)M, (int)N, (int)K, alpha, A, (int)lda, B, (int)ldb,
               beta, C, (int)ldc, static_cast<cudaStream_t>(stream));
    W4_LA_END
}

int wc4dvar_gpu_la_gather_cols_dev(int device, int64_t rows, int64_t r, const double* in,
                                   int64_t ldi, const int32_t* perm, double* out, int64_t ldo,
                                   void* stream) {
    W4_LA_BEGIN
    require(rows >= 0 && r >= 0 && ldi >= rows && ldo >= rows, "gather_cols: bad size");
    DeviceGuard g(device);
    if (rows == 0 || r == 0) return WC4DVAR_OK;
    gather_cols(rows, (int)r, in, ldi, perm, out, ldo, static_cast<cudaStream_t>(stream));
    W4_LA_END
}

}  // extern "C"
