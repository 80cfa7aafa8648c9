// Randomized eigenpairs on device: REVD, Nystrom, ritzit (randevd.cpp:47-148).
#pragma once

#include "ops.cuh"

namespace w4 {

struct SketchTiming {
    double apply_ms = 0, orth_ms = 0, small_ms = 0, gemm_ms = 0, total_ms = 0;
};

// Omega: dim x m device (ld dim).  U_out: dim x k (ldu), theta_out: k (device).
// Returns the number of pairs produced.  Counts operator applies like the reference.
int64_t sketch_dev(wc4dvar_op& op, const wc4dvar_sketch_config& cfg, const double* omega,
                   double* U_out, int64_t ldu, double* theta_out, cudaStream_t st,
                   SketchTiming* timing);

// Rayleigh-Ritz on an orthonormal Z (dim x m): all m pairs, decreasing.
void rayleigh_ritz_dev(wc4dvar_op& op, const double* Z, int64_t ldz, int64_t m, double* U_out,
                       int64_t ldu, double* theta_out, cudaStream_t st);

// clustered_spectrum (spectrum.cpp:31-64): eigenvalues (decreasing, q + k of them) of
// C^T A C on an orthonormal basis Q of span([W | U]) -- W the observation range (dim x q),
// U / T the LMP's vectors and compact-WY factor (k = 0: no preconditioner).  The remaining
// dim - (q + k) eigenvalues are exactly 1.  vals_out: device, q + k.  Counts q + k applies.
void clustered_spectrum_dev(wc4dvar_op& op, const double* W, int64_t q, const double* U, int64_t k,
                            const double* T, double* vals_out, cudaStream_t st);

}  // namespace w4
