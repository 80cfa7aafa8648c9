"""cond(Y) of the sketch sample Y = A Omega at the BASELINE configs (the regime of CholQR2 and
of the rank probe): Y on the device, Gram G = Y^T Y by the library's DMMA Gram, eigenvalues of
G in fp64 on the host; cond(Y) = sqrt(lambda_max / lambda_min) (trustworthy up to ~1e7, where
the Gram's own rounding takes over).  python tools/cond_y.py C2 C3 C4 C5"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2101_07249_b200 as W  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402
from paper_2101_07249_b200 import distributed as D  # noqa: E402

mk = {"C2": configs.config2, "C3": configs.config3, "C4": lambda: configs.config4(256),
      "C5": lambda: configs.config5(64)}
ops = D.DeviceOps(0)
for name in sys.argv[1:] or ["C2", "C3", "C4", "C5"]:
    wl = mk[name]()
    op = wl.hessian(0)
    nA, m = op.dim(), wl.m
    Om = torch.empty((m, nA), dtype=torch.float64, device="cuda")
    W.gaussian_block_dev(Om, nA, 1)
    Y = torch.empty_like(Om)
    op.apply_block_dev(Om, Y, torch.cuda.current_stream().cuda_stream)
    del Om
    Yc = Y.T  # n_A x m column-major view
    G = ops.gram(Yc, Yc).cpu().numpy()
    ev = np.linalg.eigvalsh(0.5 * (G + G.T))
    cond = float(np.sqrt(ev[-1] / max(ev[0], 1e-300)))
    print(f"{name} ({wl.name}, m = {m}): cond(Y) = {cond:.3e}; CholQR2 safe below ~1e8: {cond < 1e8}")
    del Y
    torch.cuda.empty_cache()
