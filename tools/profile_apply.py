"""Small driver for ncu: C2 operator, a few A*Omega block applies (device-resident)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_07249_b200 as W  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
wl = configs.config2()
op = wl.hessian(0)
Om = W.gaussian_matrix(op.dim(), wl.m, configs.OMEGA_SEED)
V = torch.from_numpy(np.ascontiguousarray(Om.T)).cuda()
out = torch.empty_like(V)
sp = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    op.apply_block_dev(V, out, sp)
torch.cuda.synchronize()
print("ok", float(out.abs().max()))
