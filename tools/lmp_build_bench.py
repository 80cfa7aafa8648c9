"""LMP build ms on a BASELINE config with the sketch resident on the device (Omega -> U,
Theta), per method, warm call, with the sketch's stage split (apply / orth / small / gemm):
    python tools/lmp_build_bench.py C4 256 [revd,nystrom,ritzit]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_07249_b200 as W  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
m = int(sys.argv[2]) if len(sys.argv) > 2 else 256
methods = (sys.argv[3] if len(sys.argv) > 3 else "revd,nystrom,ritzit").split(",")
wl = {"C2": configs.config2, "C3": configs.config3}.get(cfg, lambda: configs.config4(m))() if cfg != "C5" \
    else configs.config5(m)
op = wl.hessian(0)
nA, k = op.dim(), wl.k
m = wl.m
Om = torch.empty((m, nA), dtype=torch.float64, device="cuda")
W.gaussian_block_dev(Om, nA, 1)
U = torch.empty((k, nA), dtype=torch.float64, device="cuda")
th = torch.empty(k, dtype=torch.float64, device="cuda")
for method in methods:
    cfgs = W.SketchConfig(k, m - k, 1, method, 1)
    W.sketch_eigenpairs_dev(op, cfgs, Om, U, th)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    W.sketch_eigenpairs_dev(op, cfgs, Om, U, th)
    torch.cuda.synchronize()
    wall = 1e3 * (time.perf_counter() - t0)
    t = W.last_sketch_timing()
    print(f"{cfg} m={m} k={k} {method}: {t['total_ms']:.1f} ms (wall {wall:.1f}) "
          + " ".join(f"{a}={b:.1f}" for a, b in t.items() if a != 'total_ms')
          + f" theta[0:2]={th[:2].tolist()}")
