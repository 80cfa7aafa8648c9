"""Host-side logic of the Python mirror that needs no GPU: the CG-Lanczos tridiagonal
(krylov.cpp:122-134), ClusteredSpectrum's accessors (spectrum.cpp:9-29), the assimilation
system's initial condition (assimilation.cpp:54-63) and the oracle's twin generator
(assimilation.cpp:75-110; "regeneration with equal seeds is bitwise stable",
assimilation.hpp:45-46)."""
import math

import numpy as np
import pytest

from oracle import oracle as O

W = pytest.importorskip("paper_2101_07249_b200")
from paper_2101_07249_b200 import assimilation as A  # noqa: E402


def test_tridiagonal_from_cg_known_values():
    T = W.tridiagonal_from_cg(W.CgHistory([0.5], [0.1]))  # test_krylov.cpp:153-161
    assert T.dim() == 1 and abs(T.gammas[0] - 2.0) <= 2e-15 and len(T.taus) == 0
    with pytest.raises(ValueError, match="history is empty"):
        W.tridiagonal_from_cg(W.CgHistory())
    al, be = [0.5, 0.25, 0.2], [0.3, 0.2, 0.1]
    T = W.tridiagonal_from_cg(W.CgHistory(al, be))
    assert np.allclose(T.gammas, [2.0, 4.0 + 0.3 / 0.5, 5.0 + 0.2 / 0.25], rtol=1e-15)
    assert np.allclose(T.taus, [math.sqrt(0.3) / 0.5, math.sqrt(0.2) / 0.25], rtol=1e-15)
    D = T.dense()
    assert np.array_equal(D, D.T) and np.array_equal(np.diag(D), T.gammas)


def test_clustered_spectrum_accessors():
    cs = W.ClusteredSpectrum(np.array([3.0, 1.5, 0.25]), 4)
    assert cs.min_eigenvalue() == 0.25 and cs.max_eigenvalue() == 3.0
    assert cs.full().tolist() == [3.0, 1.5, 1.0, 1.0, 1.0, 1.0, 0.25]
    only_unit = W.ClusteredSpectrum(np.zeros(0), 3)
    assert only_unit.min_eigenvalue() == 1.0 == only_unit.max_eigenvalue()
    no_unit = W.ClusteredSpectrum(np.array([2.0, 0.5]), 0)
    assert no_unit.min_eigenvalue() == 0.5 and no_unit.max_eigenvalue() == 2.0


def test_advection_initial_condition():
    g = A.ModelGrid(40, 50, 0.0, 1.0 / 40)
    u = A._advection_initial_condition(g)
    assert u.shape == (40,) and abs(u[20] - 6.0) <= 1e-15 and u.argmax() == 20
    assert np.allclose(u, 6.0 * np.exp(-0.5 * ((np.arange(40) / 40 - 0.5) / 0.1) ** 2), rtol=1e-14)
    assert g.window_dim() == 40 * 51


@pytest.mark.parametrize("kind", ["advection", "lorenz96"])
def test_oracle_twin_bitwise_stable_and_consistent(kind):
    n, N = (40, 20) if kind == "advection" else (16, 6)
    bh = O.sym_sqrt(O.build_soar(0.1 if kind == "advection" else 1.0, 3.0, n))
    qh = O.sym_sqrt(O.build_soar(0.05, 3.0, n))
    sysd = O.AssimSystem(kind, n, N, 0.05, 1.0 / n, O.ObservationNetwork.build(n, N, 4, 2), bh, qh, 0.1,
                         courant=0.5, spinup_steps=50)
    a = O.generate_twin(sysd, (1, 2, 3), 1.0, True)
    b = O.generate_twin(sysd, (1, 2, 3), 1.0, True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    truth, bg, y = O.generate_twin(sysd, (1, 2, 3), 0.0)
    assert np.array_equal(bg, truth[:, 0])  # noise_scale 0: exact background and data
    assert np.array_equal(y, O.observe(truth.reshape(-1, order="F"), sysd.net))
    p = np.zeros(n * (N + 1))
    p[:n] = truth[:, 0]
    assert np.array_equal(sysd.integrate_p(p), truth)  # unforced truth = integrate_p(x0)
    bb, dd = O.compute_innovations(sysd, p, truth, bg, y)
    assert np.array_equal(bb, np.zeros_like(bb)) and np.array_equal(dd, np.zeros_like(dd))
