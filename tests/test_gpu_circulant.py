"""Circulant covariance factors on the device (EXTENSION for BASELINE configs 3-5):
parity with the oracle's direct circulant convolution, and equivalence with the
reference's dense sym_sqrt representation on the same SOAR matrix."""
import math

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2101_07249_b200")
from gpu_helpers import pair, relerr  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402


def circ_factors(n, L, var_q=0.05):
    return (configs.circulant_sqrt(configs.soar_first_column(1.0, L, n)),
            configs.circulant_sqrt(configs.soar_first_column(math.sqrt(var_q), L, n)))


@pytest.mark.parametrize("n,N,s", [(64, 4, 3), (300, 6, 10), (1000, 3, 5)])
def test_circulant_hessian_vs_oracle(n, N, s):
    bh, qh = circ_factors(n, 5.0)
    g, o = pair(W.AdvDiffLinearized(n, N, 0.5, 0.2, s), W.ObservationNetwork.build(n, N, 4, 1), bh, qh, 0.1)
    V = O.gaussian_matrix(g.dim(), 6, 1)
    assert relerr(g.apply_block(V), o.apply_block(V)) <= 1e-12
    v = V[:, 0]
    assert relerr(g.apply_D_half(v), o.apply_D_half(v)) <= 1e-12
    assert relerr(g.apply_D_half_inv(v), o.apply_D_half_inv(v)) <= 1e-10


def test_circulant_equals_dense_representation():
    n, N = 256, 5
    bh, qh = circ_factors(n, 8.0)
    model, net = W.AdvDiffLinearized(n, N, 0.5, 0.2, 4), W.ObservationNetwork.build(n, N, 4, 1)
    gc, _ = pair(model, net, bh, qh, 0.1)
    bd = configs.sym_sqrt(configs.soar_matrix(1.0, 8.0, n))
    qd = configs.sym_sqrt(configs.soar_matrix(math.sqrt(0.05), 8.0, n))
    gd, _ = pair(model, net, bd, qd, 0.1)
    V = O.gaussian_matrix(gc.dim(), 8, 2)
    assert relerr(gc.apply_block(V), gd.apply_block(V)) <= 1e-11


def test_circulant_lorenz96_sketch_vs_oracle():
    wl = configs.lorenz96_workload("l96-small", 512, 4, 5, 16, 8, spinup=200)
    g, o = pair(wl.model, wl.net, wl.b_half, wl.q_half, wl.sigma_obs)
    for method in ("revd", "nystrom", "ritzit"):
        cfg = dict(target_rank=wl.k, oversample=wl.m - wl.k, seed=1, method=method)
        pg = W.sketch_eigenpairs(g, W.SketchConfig(**cfg))
        po = O.sketch_eigenpairs(o, O.SketchConfig(**cfg))
        assert relerr(pg.values, po.values) <= 1e-10, method


def _np_dhalf(bh, qh, v, n, N):
    """numpy FFT convolution of each window column (validated against the oracle's direct
    circulant convolution at n = 1e4 below)."""
    fb, fq = np.fft.rfft(bh.half), np.fft.rfft(qh.half)
    out = np.empty_like(v)
    for i in range(N + 1):
        out[i * n:(i + 1) * n] = np.fft.irfft(np.fft.rfft(v[i * n:(i + 1) * n]) * (fb if i == 0 else fq), n)
    return out


def test_fused_four_step_fft_vs_oracle():
    """n = 1e4 runs the fused four-step plan (fft4.cu, N1 = 400 x N2 = 25): block apply (the
    identity / add epilogue, paired and unpaired window columns) and both D^{1/2} factors
    against the oracle's direct circulant convolution; the numpy FFT reference used at the
    large sizes is pinned to the oracle here too."""
    n, N, m = 10000, 3, 5
    bh, qh = circ_factors(n, 5.0)
    g, o = pair(W.AdvDiffLinearized(n, N, 0.5, 0.2, 3), W.ObservationNetwork.build(n, N, 4, 1), bh, qh, 0.1)
    V = O.gaussian_matrix(g.dim(), m, 1)
    assert relerr(g.apply_block(V), o.apply_block(V)) <= 1e-12
    od = o.apply_D_half(V[:, 0])
    assert relerr(g.apply_D_half(V[:, 0]), od) <= 1e-12
    assert relerr(_np_dhalf(bh, qh, V[:, 0], n, N), od) <= 1e-12
    assert relerr(g.apply_D_half_inv(V[:, 1]), o.apply_D_half_inv(V[:, 1])) <= 1e-10


@pytest.mark.parametrize("n,N,L", [(100000, 2, 4.0), (1000000, 2, 50.0), (2000000, 1, 4.0)])
def test_fused_four_step_fft_large(n, N, L):
    """The C3 / C4 / C5 plans (n = 1e5, 1e6, 2e6) against the numpy FFT convolution."""
    bh, qh = circ_factors(n, L)
    g = W.HessianOperator(W.AdvDiffLinearized(n, N, 0.5, 0.2, 2), W.ObservationNetwork.build(n, N, 10, 1),
                          bh, qh, 0.1)
    v = np.random.default_rng(3).standard_normal(n * (N + 1))
    assert relerr(g.apply_D_half(v), _np_dhalf(bh, qh, v, n, N)) <= 1e-12


def test_cufft_fallback_vs_oracle():
    """WC4DVAR_FFT4=0 forces batched cuFFT (the path for n without a compiled split) on a
    fused-plan size; run in a fresh process because the knob is read once."""
    import os
    import subprocess
    import sys
    code = r"""
import math, sys, json
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
from oracle import oracle as O
import paper_2101_07249_b200 as W
from paper_2101_07249_b200 import configs
from gpu_helpers import pair, relerr
n, N, m = 10000, 3, 4
bh = configs.circulant_sqrt(configs.soar_first_column(1.0, 5.0, n))
qh = configs.circulant_sqrt(configs.soar_first_column(math.sqrt(0.05), 5.0, n))
g, o = pair(W.AdvDiffLinearized(n, N, 0.5, 0.2, 3), W.ObservationNetwork.build(n, N, 4, 1), bh, qh, 0.1)
V = O.gaussian_matrix(g.dim(), m, 1)
print(json.dumps([relerr(g.apply_block(V), o.apply_block(V)),
                  relerr(g.apply_D_half_inv(V[:, 0]), o.apply_D_half_inv(V[:, 0]))]))
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    p = subprocess.run([sys.executable, "-c", code], cwd=root, env=dict(os.environ, WC4DVAR_FFT4="0"),
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    import json
    e_apply, e_inv = json.loads(p.stdout.strip().splitlines()[-1])
    assert e_apply <= 1e-12 and e_inv <= 1e-10, (e_apply, e_inv)


def test_pcg_with_fused_fft_operator_vs_oracle():
    """Split PCG (iterations 2.. as one conditional-graph launch) on an operator whose
    D^{1/2} is the fused four-step FFT (n = 1e4): same step sizes and iterate as the oracle,
    with and without a Nystrom LMP."""
    n, N = 10000, 2
    bh, qh = circ_factors(n, 5.0)
    g, o = pair(W.AdvDiffLinearized(n, N, 0.5, 0.2, 3), W.ObservationNetwork.build(n, N, 4, 1), bh, qh, 0.1)
    b = O.NormalStream(2).draw(g.dim())
    pg = W.sketch_eigenpairs(g, W.SketchConfig(8, 4, 1, "nystrom"))
    po = O.sketch_eigenpairs(o, O.SketchConfig(8, 4, 1, "nystrom"))
    for fg, fo in ((None, None), (W.build_spectral_lmp(pg), O.build_spectral_lmp(po))):
        # a fixed 20 iterations (the oracle's direct O(n^2) convolution bounds the budget)
        rg = W.pcg_split(g, b, fg, opts=W.PcgOptions(max_iter=20, rel_tol=0.0))
        ro = O.pcg_split(o, b, fo, opts=O.PcgOptions(max_iter=20, rel_tol=0.0))
        assert rg.history.iterations == ro.history.iterations == 20
        assert np.allclose(rg.history.alphas, ro.history.alphas, rtol=1e-9, atol=0.0)
        assert relerr(rg.x, ro.x) <= 1e-9
