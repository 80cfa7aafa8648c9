// Lorenz-96 nonlinear model on the device: the linearisation trajectory
// and the stored RK4 stages that every TL / adjoint sweep reads.
//
//   lorenz96_rhs  models.cpp:59-70      d_j = -x_{j-2} x_{j-1} + x_{j-1} x_{j+1} - x_j + F
//   lorenz96_step models.cpp:72-78      RK4
//   Lorenz96Stages::at models.cpp:80-87 [x1 | x2 | x3 | x4] of one step
//   Lorenz96Linearized ctor operators.cpp:44-51 (stages of every trajectory column)
//   AssimilationSystem::integrate_p assimilation.cpp:21-33 (x_{i+1} = M(x_i) + p_{i+1})
//
// One fused kernel advances one RK4 step: a CTA stages x on its tile plus the RK4 halo
// (8 points left, 4 right) in SMEM, evaluates the four right-hand sides on shrinking
// ranges, and writes x_{next} and / or the four stages of the step.  Every operation is an
// explicitly rounded __dmul_rn / __dadd_rn in the reference's evaluation order, so the
// trajectory and the stages are bitwise equal to the reference's (non-FMA x86) arithmetic.
#include "common.cuh"
#include "l96.cuh"

#include <algorithm>

namespace w4 {
namespace {

constexpr int kT = 1024;      // tile points per CTA
constexpr int kHL = 8, kHR = 4;  // RK4 halo: 4 rhs evaluations of radius (2, 1)
constexpr int kR = kT + kHL + kHR;
constexpr int kThreads = 256;

// d_j = -x_{j-2} x_{j-1} + x_{j-1} x_{j+1} - x_j + F, in the reference's order
__device__ __forceinline__ double rhs_at(const double* x, int e, double F) {
    const double a = __dmul_rn(-x[e - 2], x[e - 1]);
    const double b = __dmul_rn(x[e - 1], x[e + 1]);
    return __dadd_rn(__dsub_rn(__dadd_rn(a, b), x[e]), F);
}

// x_next = step(x) (+ p), and optionally the step's stages [x1|x2|x3|x4] (4n, stride n)
__global__ void __launch_bounds__(kThreads) l96_step_kernel(int64_t n, double F, double dt,
                                                            const double* __restrict__ x,
                                                            double* __restrict__ xn,
                                                            const double* __restrict__ padd,
                                                            double* __restrict__ stages,
                                                            unsigned* status) {
    __shared__ double xs[kR], ts[kR], k1[kR], k2[kR], k3[kR];
    const int64_t j0 = (int64_t)blockIdx.x * kT;
    // region element e <-> grid point (j0 - kHL + e) mod n
    for (int e = threadIdx.x; e < kR; e += kThreads) {
        int64_t g = (j0 - kHL + e) % n;
        if (g < 0) g += n;
        xs[e] = x[g];
    }
    __syncthreads();
    const double hdt = 0.5 * dt;
    // k1 = rhs(x) and x2 = x + (0.5 dt) k1 on [2, kR - 1)
    for (int e = 2 + threadIdx.x; e < kR - 1; e += kThreads) {
        const double k = rhs_at(xs, e, F);
        k1[e] = k;
        ts[e] = __dadd_rn(xs[e], __dmul_rn(hdt, k));
    }
    __syncthreads();
    const int tl = kR - 1;
    // stage x2 out (tile centre) and k2 = rhs(x2) on [4, kR - 2)
    double x3v[(kR + kThreads - 1) / kThreads];
#pragma unroll
    for (int u = 0; u < (kR + kThreads - 1) / kThreads; ++u) {
        const int e = 4 + threadIdx.x + u * kThreads;
        if (e < tl - 1) {
            const double k = rhs_at(ts, e, F);
            k2[e] = k;
            x3v[u] = __dadd_rn(xs[e], __dmul_rn(hdt, k));
        }
    }
    if (stages) {
        for (int e = kHL + threadIdx.x; e < kHL + kT; e += kThreads) {
            const int64_t g = j0 + e - kHL;
            if (g < n) {
                stages[g] = xs[e];
                stages[n + g] = ts[e];
            }
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < (kR + kThreads - 1) / kThreads; ++u) {
        const int e = 4 + threadIdx.x + u * kThreads;
        if (e < tl - 1) ts[e] = x3v[u];
    }
    __syncthreads();
    // k3 = rhs(x3) and x4 = x + dt k3 on [6, kR - 3)
    double x4v[(kR + kThreads - 1) / kThreads];
#pragma unroll
    for (int u = 0; u < (kR + kThreads - 1) / kThreads; ++u) {
        const int e = 6 + threadIdx.x + u * kThreads;
        if (e < kR - 3) {
            const double k = rhs_at(ts, e, F);
            k3[e] = k;
            x4v[u] = __dadd_rn(xs[e], __dmul_rn(dt, k));
        }
    }
    if (stages) {
        for (int e = kHL + threadIdx.x; e < kHL + kT; e += kThreads) {
            const int64_t g = j0 + e - kHL;
            if (g < n) stages[2 * n + g] = ts[e];
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < (kR + kThreads - 1) / kThreads; ++u) {
        const int e = 6 + threadIdx.x + u * kThreads;
        if (e < kR - 3) ts[e] = x4v[u];
    }
    __syncthreads();
    // k4 = rhs(x4) on the tile; x_next = x + (dt / 6) (((k1 + 2 k2) + 2 k3) + k4) (+ p)
    const double dt6 = dt / 6.0;
    bool bad = false;
    for (int e = kHL + threadIdx.x; e < kHL + kT; e += kThreads) {
        const int64_t g = j0 + e - kHL;
        if (g >= n) continue;
        if (stages) stages[3 * n + g] = ts[e];
        if (xn) {
            const double k4 = rhs_at(ts, e, F);
            const double s = __dadd_rn(__dadd_rn(__dadd_rn(k1[e], __dmul_rn(2.0, k2[e])), __dmul_rn(2.0, k3[e])), k4);
            double y = __dadd_rn(xs[e], __dmul_rn(dt6, s));
            if (padd) y = __dadd_rn(y, padd[g]);
            bad |= !isfinite(y);
            xn[g] = y;
        }
    }
    if (status && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(status, 1u);
}

unsigned grid_of(int64_t n) { return (unsigned)cdiv(n, kT); }

}  // namespace

void l96_step_dev(int64_t n, double F, double dt, const double* x, double* xn, const double* padd,
                  double* stages, unsigned* status, cudaStream_t st) {
    l96_step_kernel<<<grid_of(n), kThreads, 0, st>>>(n, F, dt, x, xn, padd, stages, status);
    W4_LAUNCH();
}

void l96_trajectory_dev(int64_t n, double F, double dt, const double* x0, int64_t spinup, int64_t steps,
                        double* traj, int64_t ldt, double* work, cudaStream_t st) {
    // spin-up ping-pongs between traj column 0 and work; the recorded states go to traj
    const double* cur = x0;
    double* bufs[2] = {traj, work};
    for (int64_t i = 0; i < spinup; ++i) {
        double* dst = bufs[(spinup - 1 - i) & 1];  // the last spin-up step lands in traj[:, 0]
        l96_step_dev(n, F, dt, cur, dst, nullptr, nullptr, nullptr, st);
        cur = dst;
    }
    if (spinup == 0) W4_CUDA(cudaMemcpyAsync(traj, x0, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    for (int64_t c = 0; c < steps; ++c)
        l96_step_dev(n, F, dt, traj + c * ldt, traj + (c + 1) * ldt, nullptr, nullptr, nullptr, st);
}

void l96_integrate_p_dev(int64_t n, int N, int substeps, double F, double dt, const double* p,
                         double* traj, int64_t ldt, unsigned* status, cudaStream_t st) {
    W4_CUDA(cudaMemcpyAsync(traj, p, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    for (int i = 0; i < N; ++i)
        for (int r = 0; r < substeps; ++r) {
            const int64_t c = (int64_t)i * substeps + r;
            const bool last = r + 1 == substeps;
            // status[i] != 0: the end state of interval i + 1 is non-finite
            l96_step_dev(n, F, dt, traj + c * ldt, traj + (c + 1) * ldt, last ? p + (int64_t)(i + 1) * n : nullptr,
                         nullptr, last ? status + i : nullptr, st);
        }
}

void l96_stages_dev(int64_t n, double F, double dt, const double* traj, int64_t ldt, int64_t nsteps,
                    double* stages, cudaStream_t st) {
    for (int64_t c = 0; c < nsteps; ++c)
        l96_step_dev(n, F, dt, traj + c * ldt, nullptr, nullptr, stages + c * 4 * n, nullptr, st);
}

}  // namespace w4
