"""ncu driver: one device-resident C4 sketch (n_A = 1.7e7, k + l = 256) of the given method."""
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2101_07249_b200 as W  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402

m = int(sys.argv[2]) if len(sys.argv) > 2 else 256
wl = configs.config4(m)
op = wl.hessian(0)
nA = op.dim()
Om = torch.empty((m, nA), dtype=torch.float64, device="cuda")
W.gaussian_block_dev(Om, nA, 1)
U = torch.empty((wl.k, nA), dtype=torch.float64, device="cuda")
th = torch.empty(wl.k, dtype=torch.float64, device="cuda")
method = sys.argv[1] if len(sys.argv) > 1 else "revd"
W.sketch_eigenpairs_dev(op, W.SketchConfig(wl.k, m - wl.k, 1, method), Om, U, th)
torch.cuda.synchronize()
print(method, W.last_sketch_timing())
