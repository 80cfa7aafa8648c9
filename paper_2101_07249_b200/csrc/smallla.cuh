// Small dense (m x m, m <= a few hundred) factorizations on device, one CTA each.
// They replace the Eigen calls of the sketches on the k+l dimension
// (randevd.cpp:38 SelfAdjointEigenSolver, :97 LLT, :105 triangular solve, :106 BDCSVD)
// and the rank probe of ColPivHouseholderQR (randevd.cpp:67,89).
#pragma once

#include "common.cuh"

namespace w4 {

// info codes written to *info (device int): 0 ok, j+1 = breakdown at pivot j.
// R = upper Cholesky factor of sym(G): R^T R = 0.5 (G + G^T)   (Eigen::LLT on the
// symmetric part; randevd.cpp:96-102).  G, R: m x m col-major (ld m); may alias.
void chol_upper(int m, const double* G, double* R, int* info, DevBuf& work, cudaStream_t st);

// R = chol_upper(G) and Rinv = R^{-1} together (one register-resident kernel for m <= 128).
// R, Rinv: m x m (ld m); R may alias G.  *info as chol_upper.
void chol_inv_upper(int m, const double* G, double* R, double* Rinv, int* info, DevBuf& work,
                    cudaStream_t st);
// Diagonally pivoted Cholesky rank probe of a Gram matrix: rank = number of pivots
// above tol_rel * max(diag).  perm[0..m) = pivot order (device ints).
void pivoted_chol_rank(int m, const double* G, double tol_rel, int* rank, int* perm, DevBuf& work,
                       cudaStream_t st);

// Rinv = R^{-1} for upper-triangular R (m x m).
void tri_inv_upper(int m, const double* R, double* Rinv, cudaStream_t st);

// Symmetric EVD of sym(K) by parallel cyclic Jacobi; values decreasing,
// W columns the matching eigenvectors (randevd.cpp:37-43).
void sym_evd_desc(int m, const double* K, double* vals, double* W, DevBuf& work, cudaStream_t st);

// One-sided Jacobi SVD of X (m x m): sigma decreasing and left singular vectors U.
void svd_left_desc(int m, const double* X, double* sigma, double* U, DevBuf& work,
                   cudaStream_t st);

// C (M x N) = alpha * op(A) op(B) + beta * C for small matrices (one thread per entry).
void small_gemm(bool ta, bool tb, int M, int N, int K, double alpha, const double* A, int lda,
                const double* B, int ldb, double beta, double* C, int ldc, cudaStream_t st);

// Gather columns: out[:, j] = in[:, perm[j]] for j < r (rows R).
void gather_cols(int64_t R, int r, const double* in, int64_t ldi, const int* perm, double* out,
                 int64_t ldo, cudaStream_t st);

}  // namespace w4
