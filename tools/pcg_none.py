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
    # two run lengths: the slope is the per-iteration cost without the fixed part (H2D of b,
    # D2H of x through pageable numpy buffers, the first un-graphed iteration, graph build)
    ts = {}
    for its in (iters, iters, 2 * iters):
        t0 = time.perf_counter()
        r = W.pcg_split(op, b, None, opts=W.PcgOptions(rel_tol=0.0, max_iter=its))
        ts[r.history.iterations] = time.perf_counter() - t0
    (i1, t1), (i2, t2) = sorted(ts.items())
    print(f"{name} none: {(t2 - t1) * 1e3 / (i2 - i1):.3f} ms/iteration (slope {i1} -> {i2} iterations; "
          f"fixed part {(t1 - i1 * (t2 - t1) / (i2 - i1)) * 1e3:.1f} ms)", flush=True)
