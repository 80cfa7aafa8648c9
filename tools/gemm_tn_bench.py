"""Time the Gram kernel (wc4dvar_gpu_la_gram_dev) on an n x m block: python tools/gemm_tn_bench.py n m."""
import ctypes
import sys

import torch

import paper_2101_07249_b200 as W
from paper_2101_07249_b200 import wc4dvar as w

n, m = int(sys.argv[1]), int(sys.argv[2])
Y = torch.empty((m, n), dtype=torch.float64, device="cuda")
W.gaussian_block_dev(Y, n, 1)
G = torch.empty((m, m), dtype=torch.float64, device="cuda")
sp = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
for _ in range(2):
    w._check(w.lib.wc4dvar_gpu_la_gram_dev(0, n, m, m, Y.data_ptr(), n, Y.data_ptr(), n, G.data_ptr(), m, sp))
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    w._check(w.lib.wc4dvar_gpu_la_gram_dev(0, n, m, m, Y.data_ptr(), n, Y.data_ptr(), n, G.data_ptr(), m, sp))
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"gram n={n} m={m}: {ms:.2f} ms, {2.0 * n * m * m / ms / 1e9:.1f} TF/s", flush=True)
