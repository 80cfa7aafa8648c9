"""Known-answer tests of the reference's own suites, ported onto the oracle
(proj/tests/test_models.cpp, test_covariance.cpp, test_operators.cpp)."""
import math

import numpy as np
import pytest

from oracle import oracle as O


# ---- test_models.cpp -------------------------------------------------------
def test_advection_constant_invariance():  # :11-17
    u = np.full(12, 3.0)
    for c in (0.2, 0.8, 1.0):
        assert np.array_equal(O.advection_step(u, c), u)


def test_advection_spike_shift_c1():  # :19-25
    u = np.zeros(10)
    u[5] = 1.0
    out = O.advection_step(u, 1.0)
    assert out[6] == 1.0 and out.sum() == 1.0


def test_advection_hand_values():  # :27-35
    out = O.advection_step([1.0, 0.0, 0.0, 0.0], 0.8)
    assert out[0] == pytest.approx(0.2, rel=1e-15)
    assert out[1] == pytest.approx(0.8, rel=1e-15)
    assert out[2] == 0.0 and out[3] == 0.0


def test_advection_linear_and_adjoint():  # :37-54
    s = O.NormalStream(41)
    u, v = s.draw(16), s.draw(16)
    lhs = O.advection_step(1.7 * u - 0.3 * v, 0.8)
    rhs = 1.7 * O.advection_step(u, 0.8) - 0.3 * O.advection_step(v, 0.8)
    assert np.abs(lhs - rhs).max() <= 1e-14
    s = O.NormalStream(7)
    for _ in range(20):
        d, lam = s.draw(24), s.draw(24)
        a = O.advection_step(d, 0.8) @ lam
        b = d @ O.advection_adjoint_step(lam, 0.8)
        assert abs(a - b) <= 1e-12 * (1 + abs(a))


def test_advection_adjoint_reverse_shift():  # :56-62
    lam = np.zeros(8)
    lam[3] = 1.0
    out = O.advection_adjoint_step(lam, 1.0)
    assert out[2] == 1.0 and out.sum() == 1.0


def test_advdiff_extension_stencil_and_adjoint():
    # EXTENSION (BASELINE configs): C=0.5, D=0.2 -> 0.1 x_j + 0.7 x_{j-1} + 0.2 x_{j+1}
    e = np.zeros(6)
    e[2] = 1.0
    out = O.advdiff_step(e, 0.5, 0.2)
    assert out[2] == pytest.approx(0.1, abs=1e-15)
    assert out[3] == pytest.approx(0.7, abs=1e-15)
    assert out[1] == pytest.approx(0.2, abs=1e-15)
    assert np.array_equal(O.advdiff_step(np.ones(5) * 2.5, 0.5, 0.2), np.ones(5) * 2.5)
    assert np.array_equal(O.advdiff_step(e, 0.8, 0.0), O.advection_step(e, 0.8))
    s = O.NormalStream(3)
    for _ in range(10):
        d, lam = s.draw(17), s.draw(17)
        a = O.advdiff_step(d, 0.5, 0.2) @ lam
        b = d @ O.advdiff_adjoint_step(lam, 0.5, 0.2)
        assert abs(a - b) <= 1e-13 * (1 + abs(a))


def test_l96_rhs_known_answers():  # :64-95
    assert np.abs(O.lorenz96_rhs(np.full(8, 8.0), 8.0)).max() <= 1e-14
    d = O.lorenz96_rhs([1.0, 2.0, 3.0, 4.0], 8.0)
    np.testing.assert_allclose(d, [3.0, 5.0, 11.0, 1.0], rtol=1e-15)
    assert np.array_equal(O.lorenz96_rhs(np.zeros(6), 8.0), np.full(6, 8.0))
    x = O.NormalStream(5).draw(10)
    d = O.lorenz96_rhs(x, 8.0)
    xr = np.roll(x, -3)
    assert np.abs(O.lorenz96_rhs(xr, 8.0) - np.roll(d, -3)).max() <= 1e-13


def test_l96_rk4_fixed_point_and_order():  # :97-124
    x = np.full(8, 8.0)
    assert np.abs(O.lorenz96_step(x, 8.0, 0.05) - x).max() <= 1e-13
    y = O.NormalStream(11).draw(8)
    assert np.array_equal(O.lorenz96_step(y, 8.0, 0.0), y)
    x0 = np.full(8, 8.0) + 0.5 * O.NormalStream(3).draw(8)

    def integrate(dt, steps):
        x = x0
        for _ in range(steps):
            x = O.lorenz96_step(x, 8.0, dt)
        return x

    ref = integrate(0.4 / 512, 512)
    errs = [np.linalg.norm(integrate(0.4 / s, s) - ref) for s in (8, 16, 32)]
    assert math.log2(errs[0] / errs[1]) == pytest.approx(4.0, rel=0.05)
    assert math.log2(errs[1] / errs[2]) == pytest.approx(4.0, rel=0.05)


def test_l96_tlm_linear_taylor_adjoint():  # :126-165
    s = O.NormalStream(17)
    x = s.draw(8)
    st = O.lorenz96_stages(x, 8.0, 0.05)
    d1, d2 = s.draw(8), s.draw(8)
    assert np.abs(O.lorenz96_tlm_step(st, np.zeros(8), 0.05)).max() == 0.0
    lhs = O.lorenz96_tlm_step(st, 2 * d1 - 0.5 * d2, 0.05)
    rhs = 2 * O.lorenz96_tlm_step(st, d1, 0.05) - 0.5 * O.lorenz96_tlm_step(st, d2, 0.05)
    assert np.abs(lhs - rhs).max() <= 1e-12
    s = O.NormalStream(23)
    x = np.full(8, 8.0) + 0.5 * s.draw(8)
    d = s.draw(8)
    d /= np.linalg.norm(d)
    base = O.lorenz96_step(x, 8.0, 0.05)
    tl = O.lorenz96_tlm_step(O.lorenz96_stages(x, 8.0, 0.05), d, 0.05)
    errs = [np.linalg.norm(O.lorenz96_step(x + e * d, 8.0, 0.05) - base - e * tl)
            for e in (1e-2, 1e-3, 1e-4, 1e-5)]
    for i in range(3):
        assert math.log10(errs[i] / errs[i + 1]) == pytest.approx(2.0, rel=0.05)
    s = O.NormalStream(29)
    x = np.full(12, 8.0) + 0.5 * s.draw(12)
    st = O.lorenz96_stages(x, 8.0, 0.05)
    for _ in range(20):
        d, lam = s.draw(12), s.draw(12)
        a = O.lorenz96_tlm_step(st, d, 0.05) @ lam
        b = d @ O.lorenz96_adjoint_step(st, lam, 0.05)
        assert abs(a - b) <= 1e-12 * (1 + abs(a))


def test_observation_network():  # :167-200
    assert O.ObservationNetwork.build(40, 50, 4, 5).q == 100
    assert O.ObservationNetwork.build(80, 150, 10, 10).q == 120
    assert O.ObservationNetwork.build(80, 150, 5, 5).q == 480
    assert O.ObservationNetwork.build(80, 150, 2, 2).q == 3000
    net = O.ObservationNetwork.build(8, 7, 2, 3)
    assert net.times == [1, 4, 7] and net.q_at(0) == 0 and net.q_at(7) == 4
    net = O.ObservationNetwork.build(6, 4, 2, 2)
    s = O.NormalStream(31)
    traj = s.draw(30)
    y = O.observe(traj, net)
    back = O.observe_adjoint(y, net)
    nz = back != 0
    assert nz.sum() == net.q and np.array_equal(back[nz], traj[nz])
    lam = s.draw(net.q)
    assert abs(O.observe(traj, net) @ lam - traj @ O.observe_adjoint(lam, net)) <= 1e-13
    for args in ((8, 7, 0, 2), (8, 7, 9, 2), (8, 7, 2, 8)):
        with pytest.raises(ValueError):
            O.ObservationNetwork.build(*args)


# ---- test_covariance.cpp ---------------------------------------------------
def test_soar_properties():  # :23-43
    C = O.build_soar(0.5, 1e-8, 12)
    assert np.abs(C - 0.25 * np.eye(12)).max() <= 1e-6
    C = O.build_soar(0.3, 4.0, 17)
    assert np.array_equal(C, C.T)
    np.testing.assert_allclose(np.diag(C), 0.09, rtol=1e-15)
    C = O.build_soar(1.0, 3.0, 15)
    for i in range(1, 15):
        for j in range(15):
            assert C[i, j] == pytest.approx(C[0, (j - i) % 15], rel=1e-13)


def test_sym_sqrt():  # :60-90
    f = O.sym_sqrt(np.eye(5))
    assert np.abs(f.half - np.eye(5)).max() <= 1e-14
    f = O.sym_sqrt(np.diag([4.0, 9.0]))
    assert f.half[0, 0] == pytest.approx(2.0, rel=1e-14)
    assert f.half[1, 1] == pytest.approx(3.0, rel=1e-14)
    C = O.random_spd(0.1 + 0.35 * np.arange(20), 77)
    f = O.sym_sqrt(C)
    assert np.linalg.norm(f.half @ f.half - C) <= 1e-10 * np.linalg.norm(C)
    assert np.linalg.norm(f.half @ f.half_inv - np.eye(20)) <= 1e-10
    with pytest.raises(O.NumericalError, match="-0.5"):
        O.sym_sqrt(np.diag([1.0, 1.0, -0.5]))


def test_circulant_sqrt_matches_dense_sym_sqrt():
    # EXTENSION pin: the circulant factor equals the reference's dense sym_sqrt(SOAR)
    for n, L in ((64, 5.0), (100, 4.0), (257, 20.0)):
        dense = O.sym_sqrt(O.build_soar(1.0, L, n))
        col = O.soar_first_column(1.0, L, n)
        assert np.abs(col - O.build_soar(1.0, L, n)[:, 0]).max() <= 1e-15
        circ = O.circulant_sqrt(col)
        assert np.abs(circ.dense_half() - dense.half).max() <= 1e-12
        v = O.NormalStream(n).draw(n)
        assert np.abs(circ.apply(v) - dense.half @ v).max() <= 1e-12 * np.abs(v).max() * n ** 0.5
        # both inverses carry an O(eps * cond^2) error of their own construction
        ref = dense.half_inv @ v
        cond = np.linalg.cond(dense.half)
        assert np.abs(circ.apply_inv(v) - ref).max() <= 1e-14 * cond ** 2 * np.abs(ref).max()
