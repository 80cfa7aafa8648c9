"""Time the device NormalStream (jump-ahead) on the C3 / C4 / C5 sketch shapes."""
import time

import torch

import paper_2101_07249_b200 as W

for name, nA, m in (("C3", 1_100_000, 64), ("C4", 17_000_000, 256), ("C5 rank share", 42_000_000, 32)):
    out = torch.empty((m, nA), dtype=torch.float64, device="cuda")
    t0 = time.perf_counter()
    W.gaussian_block_dev(out, nA, 1)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    W.gaussian_block_dev(out, nA, 1)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name}: n_A={nA} m={m}: first {1e3*(t1-t0):.1f} ms (incl. host jump polynomial), "
          f"warm {1e3*(t2-t1):.1f} ms, {nA*m/(t2-t1)/1e9:.2f} Gnormals/s", flush=True)
    del out
    torch.cuda.empty_cache()
