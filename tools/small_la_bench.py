"""Device timing of the one-CTA small dense kernels (C-ABI row-sharded building blocks) at the
sketch sizes: python tools/small_la_bench.py [m ...]."""
import sys

import numpy as np
import torch

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
from paper_2101_07249_b200 import distributed as D  # noqa: E402


def timed(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3  # us


def main():
    ms = [int(x) for x in sys.argv[1:]] or [64, 100, 128]
    ops = D.DeviceOps(0)
    for m in ms:
        rng = np.random.default_rng(m)
        Y = rng.standard_normal((4 * m, m))
        G = D.fcontig(torch.from_numpy(Y.T @ Y).cuda())
        R = ops.chol_upper(G)
        rows = {
            "chol_upper": timed(lambda: ops.chol_upper(G)),
            "tri_inv_upper": timed(lambda: ops.tri_inv_upper(R)),
            "chol_inv (fused)": timed(lambda: ops.chol_inv(G)),
            "pivoted_rank": timed(lambda: ops.pivoted_rank(G, 1e-13)),
            "sym_evd": timed(lambda: ops.eigh_desc(G), 5),
            "svd_left": timed(lambda: ops.svd_left(R), 5),
        }
        print(f"m={m}: " + ", ".join(f"{k} {v:.1f} us" for k, v in rows.items()), flush=True)


if __name__ == "__main__":
    main()
