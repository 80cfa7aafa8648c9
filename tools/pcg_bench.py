"""LMP-PCG per-iteration timing at C3 (k = 32) and C4 (k = 128): device Nystrom sketch ->
device LMP -> pcg_split for a fixed number of iterations (rel_tol 0)."""
import sys
import time

import torch

import paper_2101_07249_b200 as W
from paper_2101_07249_b200 import configs

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 40
for name, mk in (("C3", configs.config3), ("C4_k256", lambda: configs.config4(256))):
    wl = mk()
    op = wl.hessian(0)
    nA, m, k = op.dim(), wl.m, wl.k
    Om = torch.empty((m, nA), dtype=torch.float64, device="cuda")
    W.gaussian_block_dev(Om, nA, 1)
    U = torch.empty((k, nA), dtype=torch.float64, device="cuda")
    th = torch.empty(k, dtype=torch.float64, device="cuda")
    kk = W.sketch_eigenpairs_dev(op, W.SketchConfig(k, m - k, 1, "nystrom", 1), Om, U, th)
    del Om
    op.release_workspaces()
    torch.cuda.empty_cache()
    f = W.build_spectral_lmp_dev(U, th, kk, 0)
    b = torch.empty((1, nA), dtype=torch.float64, device="cuda")
    W.gaussian_block_dev(b, nA, 2)
    bh = b[0].cpu().numpy()
    for lmp in (None, f):
        W.pcg_split(op, bh, lmp, opts=W.PcgOptions(max_iter=3, rel_tol=0.0))
        t0 = time.perf_counter()
        r = W.pcg_split(op, bh, lmp, opts=W.PcgOptions(max_iter=iters, rel_tol=0.0))
        ms = 1e3 * (time.perf_counter() - t0)
        print(f"{name} {'nystrom k=%d' % kk if lmp else 'none'}: {r.history.iterations} iterations, "
              f"{ms / r.history.iterations:.3f} ms / iteration, rel res {r.history.residual_norms[-1] / r.history.residual_norms[0]:.3e}",
              flush=True)
    del f, U, th, op
    torch.cuda.empty_cache()
