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


def test_fused_four_step_fft_vs_oracle():
    """The fused four-step FFT path (fft4.cu, opt-in via WC4DVAR_FFT4=1) against the oracle's
    direct circulant convolution, on splits that exercise radices 8, 5, 4, 3 and 2 and both
    paired and unpaired window columns (run in a fresh process: the knob is read once)."""
    import os
    import subprocess
    import sys
    code = r"""
import math, sys, json
sys.path.insert(0, 'tests'); sys.path.insert(0, '.')
import numpy as np
from oracle import oracle as O
import paper_2101_07249_b200 as W
from paper_2101_07249_b200 import configs
from gpu_helpers import pair, relerr
out = {}
for n, N, m in ((1000, 3, 5), (300, 4, 3), (2000, 2, 4), (64, 5, 2)):
    bh = configs.circulant_sqrt(configs.soar_first_column(1.0, 5.0, n))
    qh = configs.circulant_sqrt(configs.soar_first_column(math.sqrt(0.05), 5.0, n))
    g, o = pair(W.AdvDiffLinearized(n, N, 0.5, 0.2, 3), W.ObservationNetwork.build(n, N, 4, 1), bh, qh, 0.1)
    V = O.gaussian_matrix(g.dim(), m, 1)
    out[str(n)] = [relerr(g.apply_block(V), o.apply_block(V)),
                   relerr(g.apply_D_half_inv(V[:, 0]), o.apply_D_half_inv(V[:, 0]))]
print(json.dumps(out))
"""
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, WC4DVAR_FFT4="1")
    p = subprocess.run([sys.executable, "-c", code], cwd=root, env=env, capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    import json
    res = json.loads(p.stdout.strip().splitlines()[-1])
    for n, (e_apply, e_inv) in res.items():
        assert e_apply <= 1e-12, (n, e_apply)
        assert e_inv <= 1e-10, (n, e_inv)
