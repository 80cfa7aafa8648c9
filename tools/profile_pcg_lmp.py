"""ncu driver: a few PCG iterations WITH a Nystrom LMP (C2, k = 50, by default; argv[2] = C3 for
the k = 32 Lorenz-96 configuration), per-iteration wall time."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2101_07249_b200 as W  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 20
wl = configs.config3() if (len(sys.argv) > 2 and sys.argv[2] == "C3") else configs.config2()
op = wl.hessian(0)
nA = op.dim()
p = W.sketch_eigenpairs(op, W.SketchConfig(wl.k, wl.m - wl.k, configs.OMEGA_SEED, "nystrom"))
f = W.build_spectral_lmp(p)
b = W.gaussian_matrix(nA, 1, configs.RHS_SEED)[:, 0]
W.pcg_split(op, b, f, opts=W.PcgOptions(max_iter=3, rel_tol=0.0))
t0 = time.perf_counter()
r = W.pcg_split(op, b, f, opts=W.PcgOptions(max_iter=iters, rel_tol=0.0))
print(json.dumps({"ms_per_iter": 1e3 * (time.perf_counter() - t0) / r.history.iterations}))
