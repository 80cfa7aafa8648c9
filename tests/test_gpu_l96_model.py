"""Lorenz-96 nonlinear model on the device: lorenz96_step trajectories
(models.cpp:72-78), integrate_p (assimilation.cpp:21-33) and the device-computed stages of
Lorenz96Linearized (operators.cpp:44-51), against the oracle's restatement of the same
reference code.  The trajectory kernel rounds every operation explicitly in the
reference's order, so trajectories are compared bitwise."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2101_07249_b200")
from gpu_helpers import pair, relerr  # noqa: E402


def oracle_trajectory(x0, F, dt, spinup, steps):
    x = np.array(x0, dtype=np.float64)
    for _ in range(spinup):
        x = O.lorenz96_step(x, F, dt)
    out = [x]
    for _ in range(steps):
        x = O.lorenz96_step(x, F, dt)
        out.append(x)
    return np.stack(out, axis=1)


@pytest.mark.parametrize("n,spinup,steps", [(4, 3, 5), (8, 0, 4), (37, 20, 6), (1500, 25, 5), (5000, 12, 3)])
def test_trajectory_bitwise(n, spinup, steps):
    x0 = O.NormalStream(3).draw(n)
    ref = oracle_trajectory(x0, 8.0, 0.025, spinup, steps)
    got = W.lorenz96_trajectory(x0, 8.0, 0.025, spinup, steps)
    assert np.array_equal(got, ref)
    dev = W.lorenz96_trajectory_device(x0, 8.0, 0.025, spinup, steps)
    assert np.array_equal(dev.cpu().numpy().T, ref)


@pytest.mark.parametrize("s", [1, 3])
def test_integrate_p_bitwise(s):
    n, N, F, dt = 1100, 4, 8.0, 0.05
    p = O.NormalStream(5).draw(n * (N + 1))
    p[:n] += 8.0
    ref = np.empty((n, N * s + 1))
    ref[:, 0] = p[:n]
    for i in range(N):
        x = ref[:, i * s]
        for r in range(s):
            x = O.lorenz96_step(x, F, dt)
            if r + 1 < s:
                ref[:, i * s + r + 1] = x
        ref[:, (i + 1) * s] = x + p[(i + 1) * n:(i + 2) * n]
    assert np.array_equal(W.integrate_p(p, n, N, F, dt, s), ref)


def test_integrate_p_errors():
    n, N = 16, 3
    with pytest.raises(ValueError, match="length mismatch"):
        W.integrate_p(np.zeros(n * N), n, N, 8.0, 0.05)
    p = np.zeros(n * (N + 1))
    p[2 * n + 3] = np.inf
    with pytest.raises(W.NumericalError, match="integrate_p: non-finite trajectory at step 2"):
        W.integrate_p(p, n, N, 8.0, 0.05)
    with pytest.raises(ValueError, match="n must be >= 4"):
        W.lorenz96_trajectory(np.zeros(3), 8.0, 0.05, 1, 1)


@pytest.mark.parametrize("n,N,s", [(64, 3, 2), (3000, 2, 5)])
def test_device_stages_operator_parity(n, N, s):
    """Stages computed on the device from a host or a device trajectory give the operator
    of the oracle's host-computed stages."""
    x0 = O.NormalStream(9).draw(n)
    traj = W.lorenz96_trajectory(x0, 8.0, 0.025, 50, N * s)
    net = W.ObservationNetwork.build(n, N, 2, 1)
    eye = W.CovarianceFactor(np.eye(n, order="F"), np.eye(n, order="F"))
    V = O.gaussian_matrix(n * (N + 1), 3, 1)
    outs = []
    for tr in (traj, W.lorenz96_trajectory_device(x0, 8.0, 0.025, 50, N * s)):
        g, o = pair(W.Lorenz96Linearized(tr, 8.0, 0.025, s), net, eye, eye, 0.2)
        ref = o.apply_block(V)
        got = g.apply_block(V)
        assert relerr(got, ref) <= 1e-13
        outs.append(got)
    assert np.array_equal(outs[0], outs[1])
