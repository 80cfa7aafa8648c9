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

}  // namespace w4
