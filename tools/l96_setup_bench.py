"""Time the Lorenz-96 linearisation set-up on the device: spin-up +
trajectory (lorenz96_step) and the stage precompute of Lorenz96Linearized, at the C3
(n = 1e5, N s = 50) and C5 (n = 2e6, N s = 100) sizes with the 1000-step spin-up, against the
oracle's C restatement of lorenz96_step / Lorenz96Stages::at on one host core over a bounded
sample of steps (extrapolated per step).  Prints one JSON line per size."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_07249_b200 as W  # noqa: E402
from oracle import oracle as O  # noqa: E402


def run(name, n, nsteps, spinup=1000, F=8.0, dt=0.025):
    x0 = W.gaussian_matrix(n, 1, 3)[:, 0]
    W.lorenz96_trajectory_device(x0, F, dt, 2, 2)  # warm-up (module load, first launches)
    torch.cuda.synchronize()
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record()
    traj = W.lorenz96_trajectory_device(x0, F, dt, spinup, nsteps)
    e1.record()
    torch.cuda.synchronize()
    t_traj = e0.elapsed_time(e1)
    t0 = time.perf_counter()
    model = W.Lorenz96Linearized(traj, F, dt, 1)
    eye_n = min(n, 4)
    net = W.ObservationNetwork.build(n, nsteps, 2, 1)
    col = np.zeros(n)
    col[0] = 1.0
    f = W.CovarianceFactor(col, col, kind="circulant")
    op = W.HessianOperator(model, net, f, f, 0.2)
    torch.cuda.synchronize()
    t_stage = (time.perf_counter() - t0) * 1e3
    # oracle: bounded sample of steps / stage sets on one host core
    k = 20 if n <= 200_000 else 3
    x = np.array(x0)
    t0 = time.perf_counter()
    for _ in range(k):
        x = O.lorenz96_step(x, F, dt)
    t_cpu_step = (time.perf_counter() - t0) / k * 1e3
    t0 = time.perf_counter()
    for _ in range(k):
        O.lorenz96_stages(x, F, dt)
    t_cpu_stage = (time.perf_counter() - t0) / k * 1e3
    steps_total = spinup + nsteps
    res = {"workload": name, "n": n, "spinup": spinup, "trajectory_steps": nsteps,
           "device_trajectory_ms": t_traj, "device_trajectory_us_per_step": t_traj * 1e3 / steps_total,
           "device_operator_create_ms (incl. stages)": t_stage,
           "cpu_oracle_ms_per_step": t_cpu_step, "cpu_oracle_ms_per_stage_set": t_cpu_stage,
           "cpu_oracle_total_ms (extrapolated, 1 core)": t_cpu_step * steps_total + t_cpu_stage * nsteps,
           "cpu_sample": f"{k} steps + {k} stage sets", "hbm_gbs_per_step": 2 * 8 * n / (t_traj * 1e-3 / steps_total) / 1e9}
    print(json.dumps(res), flush=True)
    del traj, model, op
    torch.cuda.empty_cache()


if __name__ == "__main__":
    run("C3", 100_000, 50)
    run("C5", 2_000_000, 100)
