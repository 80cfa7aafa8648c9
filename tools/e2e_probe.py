"""Where the C2 end-to-end time goes: device-only block apply for m = 100 and m = 50,
pinned H2D / D2H bandwidth for one step's bytes (alone and concurrently), and the
host-pointer apply (the e2e path) as configured by WC4DVAR_PIPELINE_CHUNKS."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_07249_b200 as W  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402

wl = configs.config2()
op = wl.hessian(0)
nA, m = op.dim(), wl.m
res = {}
V = torch.randn(m, nA, dtype=torch.float64, device="cuda")
out = torch.empty_like(V)
sp = torch.cuda.current_stream().cuda_stream
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for mm in (100, 50):
    op.apply_block_dev(V[:mm], out[:mm], sp)
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(10):
        op.apply_block_dev(V[:mm], out[:mm], sp)
    ev[1].record()
    torch.cuda.synchronize()
    res[f"dev_ms_m{mm}"] = ev[0].elapsed_time(ev[1]) / 10
Vh = torch.empty(m, nA, dtype=torch.float64).pin_memory()
Oh = torch.empty_like(Vh).pin_memory()
Vh.copy_(V.cpu())
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for name, fn in (("h2d", lambda: V.copy_(Vh, non_blocking=True)),
                 ("d2h", lambda: Oh.copy_(out, non_blocking=True))):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        fn()
    torch.cuda.synchronize()
    res[f"{name}_GBs"] = 10 * 8 * nA * m / (time.perf_counter() - t0) / 1e9
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    with torch.cuda.stream(s1):
        V.copy_(Vh, non_blocking=True)
    with torch.cuda.stream(s2):
        Oh.copy_(out, non_blocking=True)
torch.cuda.synchronize()
res["duplex_GBs_each"] = 10 * 8 * nA * m / (time.perf_counter() - t0) / 1e9
op.apply_block_host_ptr(Vh.data_ptr(), nA, m, Oh.data_ptr(), nA)
t0 = time.perf_counter()
for _ in range(10):
    op.apply_block_host_ptr(Vh.data_ptr(), nA, m, Oh.data_ptr(), nA)
res["e2e_ms"] = (time.perf_counter() - t0) * 100
res["chunks"] = os.environ.get("WC4DVAR_PIPELINE_CHUNKS", "2")
print(json.dumps(res))
