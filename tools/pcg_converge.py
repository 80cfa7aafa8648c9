"""Iterations / time-to-solution of LMP-PCG to relative residual 1e-6 at a large cap:
python tools/pcg_converge.py {C3,C4,C5} max_iter [methods...]."""
import sys
import time

import torch

import paper_2101_07249_b200 as W
from paper_2101_07249_b200 import configs

name, cap = sys.argv[1], int(sys.argv[2])
methods = sys.argv[3:] or ["none", "nystrom"]
wl = {"C3": configs.config3, "C4": lambda: configs.config4(256), "C5": lambda: configs.config5(64),
      "C2": configs.config2}[name]()
op = wl.hessian(0)
nA, m, k = op.dim(), wl.m, wl.k
b = torch.empty((1, nA), dtype=torch.float64, device="cuda")
W.gaussian_block_dev(b, nA, 2)
bh = b[0].cpu().numpy()
for method in methods:
    f = None
    if method != "none":
        Om = torch.empty((m, nA), dtype=torch.float64, device="cuda")
        W.gaussian_block_dev(Om, nA, 1)
        U = torch.empty((k, nA), dtype=torch.float64, device="cuda")
        th = torch.empty(k, dtype=torch.float64, device="cuda")
        kk = W.sketch_eigenpairs_dev(op, W.SketchConfig(k, m - k, 1, method, 1), Om, U, th)
        del Om
        op.release_workspaces()
        torch.cuda.empty_cache()
        f = W.build_spectral_lmp_dev(U, th, kk, 0)
        del U, th
    t0 = time.perf_counter()
    r = W.pcg_split(op, bh, f, opts=W.PcgOptions(max_iter=cap, rel_tol=1e-6))
    s = time.perf_counter() - t0
    h = r.history
    mid = [f"{h.residual_norms[j] / h.residual_norms[0]:.2e}@{j}" for j in (10, 100, 1000, 3000) if j < len(h.residual_norms)]
    print(f"{name} {method}: converged {h.converged} in {h.iterations} iterations, {s:.2f} s "
          f"({1e3 * s / max(h.iterations, 1):.3f} ms/it); rel residual {' '.join(mid)} final "
          f"{h.residual_norms[-1] / h.residual_norms[0]:.2e}", flush=True)
    del f
    op.release_workspaces()
    torch.cuda.empty_cache()
