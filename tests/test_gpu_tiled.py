"""Parity of the tiled window sweeps (halo recompute, multi-launch chunking) and of the
Lorenz-96 TL/adjoint device path against the oracle.

The tiled path normally engages only for n > 14 500 (advection-diffusion) or always for
Lorenz-96; WC4DVAR_SWEEP_TILE forces it with a small tile so the same code runs at sizes
the oracle checks in seconds.  Each setting runs in a fresh process (the knob is read once)."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2101_07249_b200")
from gpu_helpers import factor, oracle_model, pair, relerr  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tile", ["0", "64", "37", "l96cb1", "l96cb4", "l96cb8", "l96cb16"])
def test_tiled_sweeps_vs_oracle(tile):
    """l96cbX: the register-blocked Lorenz-96 kernels (X columns per CTA) forced on every
    domain at least one region wide."""
    env = dict(os.environ)
    if tile.startswith("l96cb"):
        env["WC4DVAR_L96_BLK"] = "1"
        env["WC4DVAR_L96_CB"] = tile[5:]
    elif tile != "0":
        env["WC4DVAR_SWEEP_TILE"] = tile
    p = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "tiled_check.py")], env=env,
                       capture_output=True, text=True, timeout=600)
    assert p.returncode == 0, p.stderr[-2000:]
    res = json.loads(p.stdout.strip().splitlines()[-1])
    for name, errs in res.items():
        for piece, e in errs.items():
            assert e <= 1e-12, (tile, name, piece, e)


@pytest.mark.parametrize("s", [1, 5])
def test_lorenz96_reference_fixture(s):
    """test_operators.cpp:91-120 Lorenz-96 block: adjoint identity of the device sweeps
    on an 8-variable trajectory, plus parity with the oracle."""
    n, N, dt = 8, 5, 0.05
    st = O.NormalStream(7)
    traj = np.empty((n, N * s + 1))
    traj[:, 0] = 8.0 + 0.4 * st.draw(n)
    for c in range(N * s):
        traj[:, c + 1] = O.lorenz96_step(traj[:, c], 8.0, dt)
    model = W.Lorenz96Linearized(traj, 8.0, dt, s)
    om = O.Lorenz96Linearized(traj, 8.0, dt, s)
    assert model.stages is None and om.stages is not None  # stages are computed on the device
    eye = W.CovarianceFactor(np.eye(n, order="F"), np.eye(n, order="F"))
    g, o = pair(model, W.ObservationNetwork.build(n, N, 2, 2), eye, eye, 1.0)
    for _ in range(10):
        p, v = st.draw(n * (N + 1)), st.draw(n * (N + 1))
        a, b = g.apply_Linv(p) @ v, p @ g.apply_LinvT(v)
        assert abs(a - b) <= 1e-12 * (1 + abs(a))
        assert relerr(g.apply_Linv(p), o.apply_Linv(p)) <= 1e-13
        assert relerr(g.apply_LinvT(v), o.apply_LinvT(v)) <= 1e-13
    V = O.gaussian_matrix(g.dim(), 4, 1)
    assert relerr(g.apply_block(V), o.apply_block(V)) <= 1e-13
