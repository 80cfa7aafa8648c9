// Split-preconditioned CG on device (krylov.cpp:22-99).
#pragma once

#include <vector>

#include "ops.cuh"

namespace w4 {

struct PcgRecord {
    std::vector<double> alphas, betas, residual_norms, costs;
    int iterations = 0;
    bool converged = false;
    int stop_reason = 2;
    const double* F = nullptr;  // device: the stored normalised residuals (n x nf, ld n)
    int nf = 0;
};

// b, x0 (nullable), x: device vectors of length op.dim on op's device.
void pcg_dev(wc4dvar_op& op, const double* b, wc4dvar_lmp* pre, const double* x0,
             const wc4dvar_pcg_options& opts, wc4dvar_cost* cost, double* x, PcgRecord& rec,
             cudaStream_t st);

}  // namespace w4
