"""The inner loop on the device path (run_inner_loop, assimilation.cpp:192-253) and the
QuadraticCost identities of proj/tests/test_assimilation.cpp:136-276, with seeded
innovations standing in for the twin experiment (generate_twin is out of scope)."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2101_07249_b200")
from gpu_helpers import factor, pair, relerr  # noqa: E402


def tiny_advection(n=4, N=2, sx=2, st=1):  # test_assimilation.cpp:15-27
    bh = factor(O.build_soar(0.1, 2.0, n))
    qh = factor(O.build_laplacian_corr(0.05, 1.5, n))
    return pair(W.AdvectionLinearized(n, N, 0.8), W.ObservationNetwork.build(n, N, sx, st), bh, qh, 0.05)


def innovations(g, seed):
    s = O.NormalStream(seed)
    return 0.1 * s.draw(g.dim()), 0.1 * s.draw(g.network().q)


def test_cost_second_order_expansion():  # :175-189
    g, o = tiny_advection()
    b, d = innovations(g, 41)
    cost = W.QuadraticCost(g, b, d)
    x = O.NormalStream(17).draw(g.dim())
    direct = cost(x)
    expansion = 0.5 * x @ g.apply(x) - x @ cost.rhs() + cost(np.zeros(g.dim()))
    assert direct == pytest.approx(expansion, rel=1e-10)
    assert cost(x) == pytest.approx(O.QuadraticCost(o, b, d)(x), rel=1e-13)
    # gradient vs central differences (:153-173)
    grad = cost.gradient(x)
    s = O.NormalStream(13)
    for _ in range(5):
        dr = s.draw(g.dim())
        dr /= np.linalg.norm(dr)
        fd = (cost(x + 1e-6 * dr) - cost(x - 1e-6 * dr)) / 2e-6
        assert abs(fd - grad @ dr) <= 1e-6 * (1 + abs(grad @ dr))


def test_inner_loop_matches_dense_solve():  # :191-219
    g, o = tiny_advection(4, 2, 2, 1)
    b, d = innovations(g, 51)
    rep = W.run_inner_loop(g, b, d, W.PrecondSpec(), W.SolverSpec(max_iter=200, rel_tol=1e-12))
    A = W.assemble_dense(g)
    cost = W.QuadraticCost(g, b, d)
    direct = np.linalg.solve(A, cost.rhs())
    assert np.linalg.norm(rep.delta_p_tilde - direct) <= 1e-8 * np.linalg.norm(direct)
    assert np.linalg.norm(rep.delta_p - g.apply_D_half(direct)) <= 1e-8 * np.linalg.norm(direct)
    assert np.linalg.norm(cost.gradient(rep.delta_p_tilde)) <= 1e-6 * np.linalg.norm(cost.rhs())


def test_control_variable_transform_invariance():  # :221-249
    n, N = 4, 3
    g, o = tiny_advection(n, N, 2, 1)
    b, d = innovations(g, 141)
    L = np.column_stack([o.apply_Linv(e) for e in np.eye(n * (N + 1))])
    net = g.network()
    H = np.zeros((net.q, n * (N + 1)))
    r = 0
    for t in net.times:
        for j in net.points:
            H[r, t * n + j] = 1.0
            r += 1
    Dh = np.column_stack([o.apply_D_half(e) for e in np.eye(n * (N + 1))])
    Dinv = np.linalg.inv(Dh) @ np.linalg.inv(Dh)
    r_inv = 1.0 / 0.05 ** 2
    HL = H @ L
    Au = Dinv + r_inv * HL.T @ HL
    dp_direct = np.linalg.solve(Au, Dinv @ b + r_inv * L.T @ H.T @ d)
    rep = W.run_inner_loop(g, b, d, W.PrecondSpec(), W.SolverSpec(max_iter=300, rel_tol=1e-13))
    assert np.linalg.norm(rep.delta_p - dp_direct) <= 1e-8 * np.linalg.norm(dp_direct)


def test_no_preconditioner_equals_identity_lmp_bitwise():  # :251-276
    g, _ = tiny_advection()
    b, d = innovations(g, 61)
    a = W.run_inner_loop(g, b, d, W.PrecondSpec(), W.SolverSpec(max_iter=30))
    cost = W.QuadraticCost(g, b, d)
    r = W.pcg_split(g, cost.rhs(), W.LmpFactor.identity(g.dim()), None,
                    W.PcgOptions(max_iter=30, rel_tol=1e-6, cost=cost))
    assert np.array_equal(a.delta_p_tilde, r.x)
    assert a.quadratic_costs == r.history.quadratic_costs


@pytest.mark.parametrize("kind", ["revd", "nystrom", "ritzit"])
def test_randomized_inner_loop_vs_oracle(kind):
    g, o = tiny_advection(40, 50, 4, 5)  # the advection study shape (n_A = 2040)
    b, d = innovations(g, 2024)
    rep = W.run_inner_loop(g, b, d, W.PrecondSpec(kind, 25, 5, 3), W.SolverSpec(max_iter=10))
    cost = O.QuadraticCost(o, b, d)
    pairs = O.sketch_eigenpairs(o, O.SketchConfig(25, 5, 3, kind))
    ref = O.pcg_split(o, cost.rhs(), O.build_spectral_lmp(pairs), opts=O.PcgOptions(10, 1e-6, cost_eval=cost))
    assert relerr(rep.ritz_values, pairs.values) <= 1e-10
    assert rep.iterations == ref.history.iterations  # capped at the ten plotted iterations
    assert relerr(rep.quadratic_costs, ref.history.quadratic_costs) <= 1e-9
    assert relerr(rep.residual_norms, ref.history.residual_norms) <= 1e-8
