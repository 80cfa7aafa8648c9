"""Time the Hessian block apply A*Omega on the larger BASELINE configs (C3 Lorenz-96,
C4 advection-diffusion with circulant factors) on one GPU.  Omega is N(0,1) drawn on the
device (torch) for these sizes -- the bit-exact reference stream is used for parity at
small sizes -- so the numbers are throughput only.  Prints one JSON line per config."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2101_07249_b200 import configs  # noqa: E402


def run(wl, m, reps=3, warm=1):
    t0 = time.perf_counter()
    op = wl.hessian(0)
    setup = time.perf_counter() - t0
    n = op.dim()
    g = torch.Generator(device="cuda").manual_seed(1)
    V = torch.randn(m, n, dtype=torch.float64, device="cuda", generator=g)
    out = torch.empty_like(V)
    sp = torch.cuda.current_stream().cuda_stream
    for _ in range(warm):
        op.apply_block_dev(V, out, sp)
    op.profile(True)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    for _ in range(reps):
        op.apply_block_dev(V, out, sp)
    ev[1].record()
    torch.cuda.synchronize()
    ms = ev[0].elapsed_time(ev[1]) / reps
    st, calls = op.profile_read()
    nq = wl.net.q
    bytes_col = 8.0 * (3 * n + 2 * nq)
    res = {"workload": wl.name, "m": m, "n_A": n, "ms_per_apply": ms, "columns_per_s": m / (ms / 1e3),
           "stage_ms": [x / max(calls, 1) for x in st], "setup_s": setup,
           "hbm_frac_compulsory": bytes_col * m / (ms * 1e-3) / 6542.7e9}
    print(json.dumps(res), flush=True)
    del V, out, op
    torch.cuda.empty_cache()


if __name__ == "__main__":
    which = sys.argv[1:] or ["c3", "c4"]
    if "c3" in which:
        run(configs.config3(), 64)
    if "c4" in which:
        wl = configs.config4(16)
        for m in (16, 64):
            wl.m = m
            run(wl, m)
