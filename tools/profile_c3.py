"""ncu driver: one C3 (Lorenz-96, n=1e5) block apply with m=16 columns."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2101_07249_b200 import configs  # noqa: E402

wl = configs.config3()
op = wl.hessian(0)
V = torch.randn(16, op.dim(), dtype=torch.float64, device="cuda")
out = torch.empty_like(V)
for _ in range(2):
    op.apply_block_dev(V, out, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok")
