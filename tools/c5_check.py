"""BASELINE configs[4] (C5: Lorenz-96 n = 2e6, Nsw = 20, s = 5) on one GPU at one rank's share
of the 8-GPU sketch (m = 32 columns): set-up time (device trajectory + stages), block-apply
time and stage split, and size-independent properties of A at this size -- symmetry
u.(A v) = v.(A u) and A >= I on random directions."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2101_07249_b200 import configs  # noqa: E402

m = int(sys.argv[1]) if len(sys.argv) > 1 else 32
t0 = time.perf_counter()
wl = configs.config5(m)
op = wl.hessian(0)
torch.cuda.synchronize()
setup = time.perf_counter() - t0
nA = op.dim()
g = torch.Generator(device="cuda").manual_seed(1)
V = torch.randn(m, nA, dtype=torch.float64, device="cuda", generator=g)
Y = torch.empty_like(V)
sp = torch.cuda.current_stream().cuda_stream
op.apply_block_dev(V, Y, sp)
op.profile(True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
op.apply_block_dev(V, Y, sp)
e1.record()
torch.cuda.synchronize()
st, calls = op.profile_read()
# symmetry and A >= I on the first columns (float64 dots on the device)
sym = []
for j in range(0, min(m, 8), 2):
    a = torch.dot(V[j], Y[j + 1]).item()
    b = torch.dot(V[j + 1], Y[j]).item()
    sym.append(abs(a - b) / max(abs(a), abs(b)))
ray = [(torch.dot(V[j], Y[j]) / torch.dot(V[j], V[j])).item() for j in range(min(m, 8))]
print(json.dumps({"workload": wl.name, "n_A": nA, "m": m, "setup_s": setup, "ms_per_apply": e0.elapsed_time(e1),
                  "stage_ms": [x / max(calls, 1) for x in st], "symmetry_relerr_max": max(sym),
                  "rayleigh_min": min(ray), "gpu_mem_GB": torch.cuda.max_memory_allocated() / 1e9}))
