"""Small driver for ncu: one C4 (n = 1e6, Nsw = 16) block apply with m columns on the device,
i.e. two fused circulant D^{1/2} launches (fftconv_kernel) around the tiled sweeps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2101_07249_b200 import configs  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 16
wl = configs.config4(m)
op = wl.hessian(0)
g = torch.Generator(device="cuda").manual_seed(1)
V = torch.randn(m, op.dim(), dtype=torch.float64, device="cuda", generator=g)
out = torch.empty_like(V)
op.apply_block_dev(V, out, torch.cuda.current_stream().cuda_stream)
torch.cuda.synchronize()
print("ok", float(out.abs().max()))
