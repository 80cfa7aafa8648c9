// Batched tangent-linear / adjoint window sweeps (L^{-1}, L^{-T}) with the observation
// operator fused in (HessianOperator::apply_Linv / apply_LinvT / observe / observe_adjoint,
// operators.cpp:79-101, models.cpp:184-201).
#pragma once

#include "common.cuh"

namespace w4 {

struct ModelDev {
    int kind = WC4DVAR_MODEL_IDENTITY;
    int64_t n = 0;
    int N = 0;
    int s = 1;
    double c = 0.0, d = 0.0, dt = 0.0;
    const double* stages = nullptr;  // device, L96: (N*s) x 4n
};

// The s-fold power of a radius-1 TL (or adjoint) step as one (2s+1)-tap periodic stencil:
// y_j = sum_k t[k] x_{j-s+k}.  The step is linear with constant coefficients (advection /
// advection-diffusion, models.cpp:27-45), so one interval of s sub-steps is a single
// convolution -- (2s+1) FMAs per point instead of 3s, and no per-sub-step halo recompute.
// Rounding differs from s sequential steps at the 1e-16 level (all taps are >= 0 for a
// stable step, so the sum has no cancellation).
constexpr int kMaxFusedS = 10;
struct StencilTaps {
    double t[2 * kMaxFusedS + 1];
};
StencilTaps stencil_power(int kind, double c, double d, int s, bool adjoint);

struct NetDev {
    int n_times = 0, n_points = 0;
    int64_t q = 0;
    const int* slot = nullptr;  // N+1: observation slot of time t, or -1
    const int* pmap = nullptr;  // n: index of grid point j in points[], or -1
    int sx = 0;  // > 0: points are exactly {0, sx, 2 sx, ...} (ObservationNetwork::build), so
                 // pmap[g] = g % sx ? -1 : g / sx without a table lookup
};

struct SweepArgs {
    // forward sweep (x_0 = X_0, x_{i+1} = M_i x_i + X_{i+1})
    const double* X = nullptr;
    int64_t ldx = 0;
    double* traj = nullptr;  // optional: every x_i
    int64_t ldtraj = 0;
    double* Y = nullptr;  // q x m obs (ld q): forward writes scale_fwd * H x, adjoint reads it
    double scale_fwd = 1.0;
    bool do_fwd = false;
    bool fwd_obs = false;
    // adjoint sweep (s_N = v_N + H_N^T y, s_i = v_i + H_i^T y + M_i^T s_{i+1})
    const double* V = nullptr;  // optional addend v
    int64_t ldv = 0;
    double* S = nullptr;
    int64_t lds = 0;
    bool do_adj = false;
    bool adj_obs = false;
    int64_t m = 0;
};

// Max grid points handled by the resident (whole state in shared memory) sweep.
int64_t sweep_resident_max_n();
// ws: scratch for the tiled path's launch-boundary states (grown as needed).
void sweep(const ModelDev& model, const NetDev& net, const SweepArgs& a, unsigned* status,
           cudaStream_t stream, DevBuf* ws = nullptr);
// Tiled window sweeps (large n, Lorenz-96); see sweep_tiled.cu.
// tile_override > 0 forces tiled mode with that tile size (tests).
void sweep_tiled(const ModelDev& model, const NetDev& net, const SweepArgs& a, unsigned* status,
                 cudaStream_t stream, DevBuf& ws, int tile_override = 0);

}  // namespace w4
