"""Per-stage device times of one block apply: python tools/apply_stages.py {C3,C4,C5} m [reps]."""
import sys

import torch

import paper_2101_07249_b200 as W
from paper_2101_07249_b200 import configs

name, m = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
wl = {"C3": configs.config3, "C4": lambda: configs.config4(m), "C5": lambda: configs.config5(m)}[name]()
op = wl.hessian(0)
V = torch.empty((m, op.dim()), dtype=torch.float64, device="cuda")
W.gaussian_block_dev(V, op.dim(), 1)
Y = torch.empty_like(V)
sp = torch.cuda.current_stream().cuda_stream
op.apply_block_dev(V, Y, sp)
torch.cuda.synchronize()
ref = Y.clone()
op.profile(True)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    op.apply_block_dev(V, Y, sp)
e1.record()
torch.cuda.synchronize()
st, calls = op.profile_read()
print(f"{name} m={m}: {e0.elapsed_time(e1) / reps:.3f} ms/apply; d_half_in {st[0] / calls:.3f}, sweep {st[1] / calls:.3f}, "
      f"d_half_out {st[2] / calls:.3f} ms; rerun bitwise {bool(torch.equal(ref, Y))}", flush=True)
