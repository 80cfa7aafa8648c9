"""Deterministic LMP eigenpairs on the device: matrix-free Lanczos with full
re-orthogonalisation (krylov.cpp:178-278), the CG-Lanczos tridiagonal and Ritz recovery
(krylov.cpp:122-176) and exact_top_pairs / the deterministic inner loop
(assimilation.cpp:173-211) -- the reference's test_krylov.cpp:153-309 and
test_assimilation.cpp:361-373 cases on the GPU path."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2101_07249_b200")
from gpu_helpers import factor, pair  # noqa: E402


def linspace_eigs(n, lo, hi):  # test_krylov.cpp:15-19
    return np.array([lo + (hi - lo) * i / (n - 1) for i in range(n)])


def dense_op(A):
    return W.DenseOperator(np.asfortranarray(A))


def test_tridiagonal_from_single_iteration():  # test_krylov.cpp:153-161
    T = W.tridiagonal_from_cg(W.CgHistory([0.5], [0.1]))
    assert T.dim() == 1 and abs(T.gammas[0] - 2.0) <= 2e-15
    with pytest.raises(ValueError):
        W.tridiagonal_from_cg(W.CgHistory())


def lanczos_tridiagonal(A, b, j):
    """Explicit Lanczos with full re-orthogonalisation (test_support.hpp's oracle)."""
    n = len(b)
    V = np.zeros((n, j + 1))
    V[:, 0] = b / np.linalg.norm(b)
    a, bb = np.zeros(j), np.zeros(j)
    for i in range(j):
        w = A @ V[:, i] - (bb[i - 1] * V[:, i - 1] if i else 0)
        a[i] = V[:, i] @ w
        w -= a[i] * V[:, i]
        for _ in range(2):
            w -= V[:, :i + 1] @ (V[:, :i + 1].T @ w)
        bb[i] = np.linalg.norm(w)
        V[:, i + 1] = w / bb[i]
    return np.diag(a) + np.diag(bb[:-1], 1) + np.diag(bb[:-1], -1)


def test_cg_tridiagonal_matches_explicit_lanczos():  # test_krylov.cpp:163-184
    A = O.random_spd(linspace_eigs(100, 0.8, 120.0), 61)
    b = O.NormalStream(9).draw(100)
    r = W.pcg_split(dense_op(A), b, opts=W.PcgOptions(max_iter=40, rel_tol=1e-16, reorthogonalize=True))
    assert r.history.iterations == 40
    T = W.tridiagonal_from_cg(r.history)
    e1 = np.linalg.eigvalsh(T.dense())
    e2 = np.linalg.eigvalsh(lanczos_tridiagonal(A, b, 40))
    assert np.abs(e1 - e2).max() <= 1e-8 * np.abs(e2).max()


def test_extreme_ritz_values_inside_spectrum():  # test_krylov.cpp:186-199
    A = O.random_spd(linspace_eigs(80, 2.0, 55.0), 71)
    r = W.pcg_split(dense_op(A), O.NormalStream(10).draw(80),
                    opts=W.PcgOptions(max_iter=25, rel_tol=1e-16, reorthogonalize=True))
    ev = np.linalg.eigvalsh(W.tridiagonal_from_cg(r.history).dense())
    assert ev.min() >= 2.0 - 1e-9 and ev.max() <= 55.0 + 1e-9


def test_ritz_from_one_dimensional_tridiagonal():  # test_krylov.cpp:201-209
    p = W.ritz_from_tridiagonal(W.TridiagonalMatrix(np.array([2.0]), np.zeros(0)), [np.eye(6)[:, 0]], 1)
    assert abs(p.values[0] - 2.0) <= 2e-14
    assert np.abs(p.vectors[:, 0] - np.eye(6)[:, 0]).max() <= 1e-14


def test_fully_converged_cg_recovers_spectrum():  # test_krylov.cpp:211-233
    eigs = linspace_eigs(12, 1.0, 30.0)
    A = O.random_spd(eigs, 81)
    r = W.pcg_split(dense_op(A), O.NormalStream(11).draw(12),
                    opts=W.PcgOptions(max_iter=12, rel_tol=1e-16, reorthogonalize=True))
    assert r.history.iterations == 12 and len(r.history.normalized_residuals) >= 12
    p = W.ritz_from_tridiagonal(W.tridiagonal_from_cg(r.history), r.history.normalized_residuals, 12)
    expect = eigs[::-1]
    assert np.abs(p.values - expect).max() <= 1e-8 * expect.max()
    p.validate(1e-8)
    for i in range(12):
        u = p.vectors[:, i]
        assert np.linalg.norm(A @ u - p.values[i] * u) <= 1e-7 * expect.max()


def test_store_residual_vectors_without_reorthogonalization():
    """krylov.cpp:30: store_residual_vectors keeps f_j without changing the iteration."""
    A = O.random_spd(linspace_eigs(30, 1.0, 10.0), 5)
    b = O.NormalStream(4).draw(30)
    r0 = W.pcg_split(dense_op(A), b, opts=W.PcgOptions(max_iter=8, rel_tol=1e-16))
    r1 = W.pcg_split(dense_op(A), b, opts=W.PcgOptions(max_iter=8, rel_tol=1e-16, store_residual_vectors=True))
    assert r0.history.alphas == r1.history.alphas and np.array_equal(r0.x, r1.x)
    assert len(r0.history.normalized_residuals) == 0 and len(r1.history.normalized_residuals) == 9
    for j, f in enumerate(r1.history.normalized_residuals):
        assert abs(np.linalg.norm(f) - 1.0) <= 1e-13, j


def test_ghost_ritz_values_collapse():  # test_krylov.cpp:266-275
    T = W.TridiagonalMatrix(np.full(2, 3.0), np.zeros(1))
    basis = [np.eye(5)[:, 0], np.eye(5)[:, 1]]
    assert abs(W.ritz_from_tridiagonal(T, basis, 1).values[0] - 3.0) <= 1e-12
    with pytest.raises(W.NumericalError, match="fewer distinct Ritz values"):
        W.ritz_from_tridiagonal(T, basis, 2)


def test_ritz_rejects_degenerate_basis():  # test_krylov.cpp:277-283
    T = W.TridiagonalMatrix(np.full(2, 2.0), np.full(1, 0.5))
    with pytest.raises(W.NumericalError, match="lost orthogonality"):
        W.ritz_from_tridiagonal(T, [np.eye(5)[:, 0], np.eye(5)[:, 0]], 1)


def test_lanczos_matches_dense_decomposition():  # test_krylov.cpp:285-297
    eigs = linspace_eigs(150, 0.5, 90.0)
    A = O.random_spd(eigs, 101)
    op = dense_op(A)
    p = W.lanczos_eigenpairs(op, 6, W.LanczosOptions(tol=1e-12))
    p.validate(1e-9)
    for i in range(6):
        assert abs(p.values[i] - eigs[149 - i]) <= 1e-9 * eigs[149 - i]
        u = p.vectors[:, i]
        assert np.linalg.norm(A @ u - p.values[i] * u) <= 1e-8 * p.values[i]
    assert op.apply_count() <= 8 * 6 + 120


def test_lanczos_clustered_plus_spikes():  # test_krylov.cpp:299-309
    eigs = np.ones(120)
    eigs[-5:] = [4.0, 9.0, 17.0, 33.0, 70.0]
    p = W.lanczos_eigenpairs(dense_op(O.random_spd(eigs, 111)), 5)
    assert np.abs(p.values - np.array([70.0, 33.0, 17.0, 9.0, 4.0])).max() <= 1e-8 * 70.0


def lorenz_pair(n=12, N=4):
    x0 = 8.0 + O.NormalStream(121).draw(n)
    traj = W.lorenz96_trajectory(x0, 8.0, 0.05, 0, N)
    bh = factor(O.build_soar(1.0, 2.0, n))
    qh = factor(O.build_soar(0.3, 2.0, n))
    return pair(W.Lorenz96Linearized(traj, 8.0, 0.05), W.ObservationNetwork.build(n, N, 2, 1), bh, qh, 0.5)


def test_exact_top_pairs_vs_dense_hessian():
    """test_assimilation.cpp:361-373: the exact top pairs of a Lorenz-96 Hessian agree with
    the dense eigendecomposition (values 1e-8, vectors aligned to 1e-6)."""
    g, o = lorenz_pair()
    ev, V = np.linalg.eigh(O.assemble_dense(o))
    p = W.exact_top_pairs(g, 4)
    assert np.abs(p.values - ev[::-1][:4]).max() <= 1e-8 * ev.max()
    for i in range(4):
        assert abs(abs(p.vectors[:, i] @ V[:, ::-1][:, i]) - 1.0) <= 1e-6
    q = W.exact_top_pairs(g, 4, dense_cap=8)  # the matrix-free route
    assert np.abs(p.values - q.values).max() <= 1e-8 * ev.max()


def test_deterministic_inner_loop_end_to_end():
    """test_assimilation.cpp:375-: the second inner loop preconditioned by the previous
    loop's exact top pairs; the reference's error for a missing previous Hessian."""
    g1, _ = lorenz_pair()
    g2, o2 = lorenz_pair()
    b = O.NormalStream(5).draw(g2.dim())
    d = O.NormalStream(6).draw(g2.network().q)
    rep = W.run_inner_loop(g2, b, d, W.PrecondSpec("deterministic", 4), W.SolverSpec(max_iter=200, rel_tol=1e-10),
                           previous_hessian=g1)
    assert rep.converged and len(rep.ritz_values) == 4
    base = W.run_inner_loop(g2, b, d, W.PrecondSpec("none"), W.SolverSpec(max_iter=200, rel_tol=1e-10))
    assert rep.iterations <= base.iterations
    assert np.abs(rep.delta_p - base.delta_p).max() <= 1e-7 * np.abs(base.delta_p).max()
    with pytest.raises(ValueError, match="needs a previous inner loop"):
        W.run_inner_loop(g2, b, d, W.PrecondSpec("deterministic", 4), W.SolverSpec())
