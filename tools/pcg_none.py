"""Per-iteration time of the unpreconditioned PCG at C4 / C3 / C2 (WC4DVAR_PCG_VECPASS=0: ring kernel)."""
import os, sys, time, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2101_07249_b200 as W
from paper_2101_07249_b200 import configs
from oracle import oracle as O
import numpy as np
only = sys.argv[1] if len(sys.argv) > 1 else None      # e.g. C4
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 300
for name, mk in (("C4", lambda: configs.config4(16)), ("C3", configs.config3), ("C2", configs.config2)):
    if only and name != only:
        continue
    wl = mk(); op = wl.hessian(0)
    b = np.asarray(W.gaussian_matrix(op.dim(), 1, 2))[:, 0].copy()
    for it in range(2):
        t0 = time.perf_counter()
        r = W.pcg_split(op, b, None, opts=W.PcgOptions(rel_tol=0.0, max_iter=iters))
        dt = time.perf_counter() - t0
    print(f"{name} none: {dt*1e3/ r.history.iterations:.3f} ms/iteration ({r.history.iterations} iterations)", flush=True)
