"""Time the circulant D^{1/2} (fused FFT convolution) alone: C4 (n = 1e6, Nsw = 16) or C3
(n = 1e5, Nsw = 10) block of m sketch columns through hessian_piece(D_HALF), CUDA events,
best of `reps`.  Prints ms, algorithmic TF/s (SURVEY §8(d) real-FFT convention) and the
fraction of the fp64 peak.  Knobs of the kernel are environment variables (WC4DVAR_FFT_*),
so run it once per setting:  python tools/fft_bench.py C4 64 [reps]"""
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_07249_b200 as W  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 64
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
wl = configs.config4(m) if cfg == "C4" else configs.config3() if cfg == "C3" else configs.config5(m)
op = wl.hessian(0)
nA, n, N = op.dim(), wl.model.n, wl.model.N
V = torch.empty((m, nA), dtype=torch.float64, device="cuda")
W.gaussian_block_dev(V, nA, 1)
out = torch.empty_like(V)
sp = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    op.piece_dev(2, V, out, sp)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    op.piece_dev(2, V, out, sp)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = min(ts)
flops = (N + 1) * m * (5.0 * n * math.log2(n) + n)
peak = W.probe_dmma_peak(0)
knobs = {k: v for k, v in os.environ.items() if k.startswith("WC4DVAR_FFT")}
print(f"{cfg} m={m} knobs={knobs}: {ms:.3f} ms (median {sorted(ts)[len(ts) // 2]:.3f}), "
      f"{flops / ms / 1e9:.2f} TF/s, frac {flops / ms / 1e9 / peak:.3f} of {peak:.1f}; "
      f"checksum {float(out[:, :1000].sum()):.12e}")
