// Lorenz-96 nonlinear model on the device (see l96.cu).
#pragma once

#include "common.cuh"

namespace w4 {

// one RK4 step: xn = lorenz96_step(x) (+ padd) and / or the step's stages (4n)
void l96_step_dev(int64_t n, double F, double dt, const double* x, double* xn, const double* padd,
                  double* stages, unsigned* status, cudaStream_t st);
// `spinup` steps from x0, then traj[:, 0..steps] (ldt >= n); work: n doubles
void l96_trajectory_dev(int64_t n, double F, double dt, const double* x0, int64_t spinup, int64_t steps,
                        double* traj, int64_t ldt, double* work, cudaStream_t st);
// integrate_p with `substeps` RK4 steps per interval: traj[:, 0..N s]; status[i] != 0 when the
// end state of interval i is non-finite
void l96_integrate_p_dev(int64_t n, int N, int substeps, double F, double dt, const double* p,
                         double* traj, int64_t ldt, unsigned* status, cudaStream_t st);
// stages of traj columns 0..nsteps-1 -> stages (nsteps x 4n)
void l96_stages_dev(int64_t n, double F, double dt, const double* traj, int64_t ldt, int64_t nsteps,
                    double* stages, cudaStream_t st);

}  // namespace w4
