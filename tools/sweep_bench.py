"""Time the fused sweeps piece L^{-T} H^T R^{-1} H L^{-1} (hessian_piece 4: forward TL sweep with
the observations, adjoint sweep with H^T y) on a BASELINE config block of m sketch columns,
CUDA events, best of `reps`, with the SURVEY §8(d) HBM bytes of the two sweeps:
    python tools/sweep_bench.py C4 64 [reps]"""
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
nA, n, N, q = op.dim(), wl.model.n, wl.model.N, wl.net.q
V = torch.empty((m, nA), dtype=torch.float64, device="cuda")
W.gaussian_block_dev(V, nA, 1)
out = torch.empty_like(V)
sp = torch.cuda.current_stream().cuda_stream
for _ in range(2):
    op.piece_dev(4, V, out, sp)
torch.cuda.synchronize()
ts = []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    op.piece_dev(4, V, out, sp)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = min(ts)
byt = 8.0 * m * (2 * n * N + 2 * q)  # forcing read + s written (+ y written / read)
knobs = {k: v for k, v in os.environ.items() if k.startswith("WC4DVAR_")}
print(f"sweeps {cfg} m={m} knobs={knobs}: {ms:.3f} ms (median {sorted(ts)[len(ts) // 2]:.3f}), "
      f"{byt / ms / 1e6:.0f} GB/s algorithmic; checksum {float(out[:, :1000].sum()):.12e}")
