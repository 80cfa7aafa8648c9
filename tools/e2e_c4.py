"""C4 k = 256 end-to-end step through wc4dvar_gpu_op_apply_block with pinned HOST buffers (the
bench's e2e leg): python tools/e2e_c4.py [steps]; WC4DVAR_PIPELINE_STAGE_MB sets the chunk."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2101_07249_b200 as W  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
m = 256
op = configs.config4(m).hessian(0)
nA = op.dim()
Vh = torch.empty((m, nA), dtype=torch.float64, pin_memory=True)
V = torch.empty((m, nA), dtype=torch.float64, device="cuda")
W.gaussian_block_dev(V, nA, 1)
Vh.copy_(V)
del V
torch.cuda.empty_cache()
Oh = torch.empty((m, nA), dtype=torch.float64, pin_memory=True)
op.apply_block_host_ptr(Vh.data_ptr(), nA, m, Oh.data_ptr(), nA)
t0 = time.perf_counter()
for _ in range(steps):
    op.apply_block_host_ptr(Vh.data_ptr(), nA, m, Oh.data_ptr(), nA)
dt = (time.perf_counter() - t0) / steps
print(f"e2e C4 k=256 stage_mb={os.environ.get('WC4DVAR_PIPELINE_STAGE_MB', 'default')}: {dt * 1e3:.0f} ms per step, "
      f"{m / dt:.1f} columns/s; checksum {float(Oh[0, :4].sum()):.12e}")
