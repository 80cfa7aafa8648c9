"""Per-iteration cost of the device PCG at C2: wall time per iteration, and the three
stage times of a single-column Hessian apply (D^1/2, sweeps, D^1/2 + identity).  Run under
ncu with a launch list to see every kernel of a few iterations."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2101_07249_b200 as W  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
wl = configs.config2()
op = wl.hessian(0)
nA = op.dim()
b = W.gaussian_matrix(nA, 1, configs.RHS_SEED)[:, 0]
W.pcg_split(op, b, None, opts=W.PcgOptions(max_iter=5, rel_tol=0.0))  # warm
t0 = time.perf_counter()
r = W.pcg_split(op, b, None, opts=W.PcgOptions(max_iter=iters, rel_tol=0.0))
wall = time.perf_counter() - t0
V = torch.randn(1, nA, dtype=torch.float64, device="cuda")
out = torch.empty_like(V)
sp = torch.cuda.current_stream().cuda_stream
op.apply_block_dev(V, out, sp)
op.profile(True)
torch.cuda.synchronize()
for _ in range(20):
    op.apply_block_dev(V, out, sp)
torch.cuda.synchronize()
st, calls = op.profile_read()
print(json.dumps({"ms_per_iter": 1e3 * wall / r.history.iterations, "iterations": r.history.iterations,
                  "apply_m1_stage_ms": [x / max(calls, 1) for x in st]}))
