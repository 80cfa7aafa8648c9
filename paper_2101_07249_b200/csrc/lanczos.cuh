// Lanczos eigenpairs and CG-Lanczos Ritz recovery on the device (see lanczos.cu).
#pragma once

#include "ops.cuh"

namespace w4 {

// lanczos_eigenpairs (krylov.cpp:178-278): top-k pairs of op; U_out device (n x k, ld n),
// values_out host (k, decreasing).  max_iter 0 = min(n, 8k + 120).  Returns the Krylov
// dimension used.  Counts one apply per step.
int64_t lanczos_eigenpairs_dev(wc4dvar_op& op, int64_t k, int max_iter, double tol, uint64_t seed,
                               double* U_out, int64_t ldu, double* values_out, cudaStream_t st);

// ritz_from_tridiagonal (krylov.cpp:136-176): T = (gammas, taus) host (j, j-1); F device
// (n x j, ldf) the normalised CG residuals f_0..f_{j-1}.  U_out device (n x k), values host.
int64_t ritz_from_tridiagonal_dev(int64_t n, int64_t j, const double* gammas, const double* taus, const double* F,
                                  int64_t ldf, int64_t k, double* U_out, int64_t ldu, double* values_out,
                                  cudaStream_t st);

}  // namespace w4
