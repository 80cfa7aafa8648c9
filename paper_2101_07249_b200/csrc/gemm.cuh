// fp64 tensor-core (DMMA) GEMMs for sm_100a.
//
// tcgen05/UMMA has no f64 kind, so fp64 tensor work on B200 goes through
// mma.sync.m16n8k8.f64 (SASS: DMMA.8x8x4).  Two kernel families:
//   * gemm_nn: C[:, c] = alpha * A * B[:, c] (+ add[:, c]) with column maps, used for the
//     block-diagonal D^{1/2} apply of HessianOperator (operators.cpp:103-113) -- the whole
//     n_A x m block is viewed as an n x (N+1)m matrix of n-columns -- and for tall x small
//     products (Y R^{-1}, Z W) of the sketches (randevd.cpp:57,105,133).
//   * gemm_tn: C = A^T B for tall-skinny A, B (Gram matrices, Z^T A Z, Z^T E1), split over
//     rows with a fixed-order reduction so results are bitwise reproducible.
#pragma once

#include "common.cuh"

namespace w4 {

// Column c of a "column-mapped" matrix lives at
//   base + (c / per) * ld_outer + (off + c % per) * stride.
struct ColMap {
    const double* base = nullptr;
    int64_t ld_outer = 0;
    int64_t stride = 0;
    int32_t per = 1;
    int32_t off = 0;
    __host__ __device__ const double* col(int64_t c) const {
        return base + (c / per) * ld_outer + (off + c % per) * stride;
    }
    static ColMap plain(const double* p, int64_t ld) {
        ColMap m;
        m.base = p;
        m.ld_outer = ld;
        m.stride = 0;
        m.per = 1;
        m.off = 0;
        return m;
    }
};

struct GemmPass {
    const double* A = nullptr;  // M x K col-major
    int64_t lda = 0;
    int64_t M = 0, K = 0, ncols = 0;
    double alpha = 1.0;
    ColMap in;    // K-long columns
    ColMap out;   // M-long columns
    ColMap add;   // optional addend (base == nullptr: none)
    bool symA = false;  // A == A^T bitwise (enables the k-contiguous LDS.128 kernel)
    bool upper_tri = false;  // B (the `in` columns) is upper triangular: column c has zeros
                             // below row c, so an output tile of columns [n0, n0 + BN) stops
                             // its k loop at n0 + BN (whole zero k-tiles skipped: the same
                             // bits, Y R^{-1} at about 3/4 of the flops)
};

// Launch one or two passes in a single kernel.  status (optional) gets
// ST_OUT_NONFINITE if any stored value is non-finite.
void gemm_nn(const GemmPass* passes, int npass, unsigned* status, cudaStream_t stream);

// C (m1 x m2, ldc) = alpha * A^T B, A: R x m1 (lda), B: R x m2 (ldb).
// work: scratch device buffer (grown as needed).  When B == A (same pointer, m2 == m1,
// ldb == lda) the product is a Gram matrix: only the tiles on and above the diagonal are
// computed and the reduction mirrors them (bitwise the full product: the DMMA sums of
// (r, c) and (c, r) multiply the same pairs in the same k order).
// sym_result: the caller knows A^T B is symmetric (Y^T (A Y) for the symmetric operator A): only
// the upper-triangle tiles are computed and mirrored, as for a Gram A^T A.
void gemm_tn(int64_t R, int64_t m1, int64_t m2, const double* A, int64_t lda, const double* B,
             int64_t ldb, double alpha, double* C, int64_t ldc, DevBuf& work, cudaStream_t stream, bool sym_result = false);

}  // namespace w4
