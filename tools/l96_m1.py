"""Single-column (PCG / Lanczos) Hessian apply time at C3 (Lorenz-96 n = 1e5)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2101_07249_b200 import configs  # noqa: E402

op = configs.config3().hessian(0)
V = torch.randn(1, op.dim(), dtype=torch.float64, device="cuda")
Y = torch.empty_like(V)
sp = torch.cuda.current_stream().cuda_stream
op.apply_block_dev(V, Y, sp)
op.profile(True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    op.apply_block_dev(V, Y, sp)
e1.record()
torch.cuda.synchronize()
st, calls = op.profile_read()
print(json.dumps({"ms_per_apply_m1": e0.elapsed_time(e1) / 10, "stage_ms": [x / max(calls, 1) for x in st],
                  "y_sum": float(Y.sum())}))
