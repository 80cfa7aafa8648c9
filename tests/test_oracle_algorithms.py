"""proj/tests/test_randevd.cpp, test_lmp.cpp, test_krylov.cpp (PCG part) ported onto
the oracle."""
import numpy as np
import pytest

from oracle import oracle as O


def head_tail():  # test_randevd.cpp:15-20
    d = np.ones(100)
    d[:10] = 10.0 - np.arange(10)
    return np.diag(d)


def test_rayleigh_ritz_invariant_subspace_and_bracket():  # :40-80
    eigs = np.linspace(1, 30, 30)
    V = O.random_orthogonal(30, 3)
    A = V @ np.diag(eigs) @ V.T
    op = O.DenseOperator(0.5 * (A + A.T))
    pr = O.rayleigh_ritz(op, V[:, [29, 25, 20]])
    np.testing.assert_allclose(pr.values, [30, 26, 21], rtol=1e-10)
    A = O.random_spd(np.linspace(2, 9, 50), 7)
    pr = O.rayleigh_ritz(O.DenseOperator(A), O.random_orthogonal(50, 11)[:, :8])
    assert pr.values.min() >= 2 - 1e-10 and pr.values.max() <= 9 + 1e-10
    Z = np.zeros((10, 2))
    Z[0, :] = 1.0
    with pytest.raises(O.NumericalError):
        O.rayleigh_ritz(O.DenseOperator(np.eye(10)), Z)


def test_sketches_identity_units():  # :82-95
    op = O.DenseOperator(np.eye(60))
    for m in ("revd", "nystrom", "ritzit"):
        pr = O.sketch_eigenpairs(op, O.SketchConfig(4, 3, 12345, m))
        assert pr.k() == 4
        assert np.abs(pr.values - 1).max() <= 1e-12
        pr.validate(1e-10)


def test_head_tail_accuracy_ordering():  # :100-151
    A = head_tail()
    op = O.DenseOperator(A)
    target = np.array([10.0, 9, 8, 7, 6])
    mr, mn, mz = np.zeros(5), np.zeros(5), np.zeros(5)
    er = en = 0.0
    for seed in range(1, 21):
        cfg = O.SketchConfig(5, 5, seed)
        r, n, z = O.revd(op, cfg), O.nystrom(op, cfg), O.revd_ritzit(op, cfg)
        assert (r.values <= target + 1e-10).all() and (n.values <= target + 1e-10).all()
        assert (z.values <= target + 1e-10).all() and (r.values / target >= 0.5).all()
        mr += r.values / target / 20
        mn += n.values / target / 20
        mz += z.values / target / 20
        er += np.linalg.norm(A - r.vectors @ np.diag(r.values) @ r.vectors.T)
        en += np.linalg.norm(A - n.vectors @ np.diag(n.values) @ n.vectors.T)
    assert (mr >= 0.65).all() and (mn >= mr).all() and (mz <= mn).all() and (mz <= mr).all()
    assert en <= er


def test_nystrom_low_rank_and_rank_collapse():  # :153-168, :229-241
    B = O.NormalStream(17).fill(40, 3)
    A = B @ B.T
    A = 0.5 * (A + A.T)
    pr = O.nystrom(O.DenseOperator(A), O.SketchConfig(5, 2, 4))
    assert pr.k() == 3
    assert np.linalg.norm(A - pr.vectors @ np.diag(pr.values) @ pr.vectors.T) <= 1e-10 * np.linalg.norm(A)
    B = O.NormalStream(29).fill(30, 1)
    A = B @ B.T
    with pytest.raises(O.NumericalError):
        O.revd(O.DenseOperator(0.5 * (A + A.T)), O.SketchConfig(3, 2, 3))


def test_determinism_counts_bracket_validation():  # :170-251
    op = O.DenseOperator(head_tail())
    for m in ("revd", "nystrom", "ritzit"):
        a = O.sketch_eigenpairs(op, O.SketchConfig(6, 4, 31, m))
        b = O.sketch_eigenpairs(op, O.SketchConfig(6, 4, 31, m))
        assert np.array_equal(a.values, b.values) and np.array_equal(a.vectors, b.vectors)
    cfg = O.SketchConfig(7, 3, 5)
    for m, k in (("revd", 20), ("nystrom", 20), ("ritzit", 10)):
        op.reset_apply_count()
        cfg.method = m
        O.sketch_eigenpairs(op, cfg)
        assert op.apply_count() == k
    A = O.random_spd(np.linspace(0.5, 17, 64), 23)
    for seed in range(1, 11):
        for m in ("revd", "nystrom", "ritzit"):
            pr = O.sketch_eigenpairs(O.DenseOperator(A), O.SketchConfig(6, 4, seed, m))
            pr.validate(1e-10)
            assert pr.values.min() >= 0.5 - 1e-8 and pr.values.max() <= 17 + 1e-8
    with pytest.raises(ValueError):
        O.revd(O.DenseOperator(np.eye(6)), O.SketchConfig(5, 5, 0))
    with pytest.raises(ValueError):
        O.revd(O.DenseOperator(np.eye(6)), O.SketchConfig(0, 5, 0))


def test_lmp_algebra():  # test_lmp.cpp:34-110, :209-224
    idf = O.LmpFactor.identity(12)
    v = O.NormalStream(1).draw(12)
    assert np.array_equal(idf.apply(v), v) and np.array_equal(idf.apply_transpose(v), v)
    f = O.build_spectral_lmp(O.RitzPairs(O.random_orthogonal(8, 5)[:, :3], np.ones(3)))
    v = O.NormalStream(7).draw(8)
    assert np.abs(f.apply(v) - v).max() <= 1e-15
    A = O.random_spd(np.linspace(0.5, 20, 10), 11)
    w, V = np.linalg.eigh(A)
    f = O.build_spectral_lmp(O.RitzPairs(V[:, ::-1].copy(), w[::-1].copy()))
    P = np.column_stack([f.apply(f.apply_transpose(e)) for e in np.eye(10)])
    Ai = np.linalg.inv(A)
    assert np.linalg.norm(P - Ai) <= 1e-9 * np.linalg.norm(Ai)
    Q = O.random_orthogonal(9, 13)
    f = O.build_spectral_lmp(O.RitzPairs(Q[:, :2], np.array([16.0, 4.0])))
    assert np.abs(f.apply(Q[:, 5]) - Q[:, 5]).max() <= 1e-14
    f1 = O.build_spectral_lmp(O.RitzPairs(Q[:, :1], np.array([16.0])))
    assert np.abs(f1.apply(Q[:, 0]) - 0.25 * Q[:, 0]).max() <= 1e-14
    Q = O.random_orthogonal(14, 17)
    th = np.array([30.0, 11, 5, 2, 1.3])
    f = O.build_spectral_lmp(O.RitzPairs(Q[:, :5], th))
    P = O.dense_spectral_lmp(Q[:, :5], th)
    s = O.NormalStream(19)
    for _ in range(10):
        v = s.draw(14)
        assert np.abs(f.apply(f.apply_transpose(v)) - P @ v).max() <= 1e-10 * (1 + np.abs(v).max())
    v = s.draw(14)
    assert np.abs(f.apply(v) - f.apply_transpose(v)).max() <= 1e-13
    with pytest.raises(O.NumericalError):
        O.build_spectral_lmp(O.RitzPairs(O.random_orthogonal(6, 83)[:, :2], np.array([2.0, -0.1])))
    assert O.build_spectral_lmp(O.RitzPairs(O.random_orthogonal(6, 89)[:, :2], np.array([2.0, 0.7]))).k() == 2


def test_pcg_known_answers():  # test_krylov.cpp:31-151
    s = O.NormalStream(1)
    b = s.draw(9)
    r = O.pcg_split(O.DenseOperator(np.eye(9)), b, opts=O.PcgOptions(rel_tol=1e-12))
    assert r.history.iterations == 1 and r.history.converged and np.abs(r.x - b).max() <= 1e-13
    A = np.diag(np.arange(1.0, 11.0))
    w, V = np.linalg.eigh(A)
    f = O.LmpFactor(V[:, ::-1].copy(), w[::-1].copy())
    r = O.pcg_split(O.DenseOperator(A), O.NormalStream(2).draw(10), f, opts=O.PcgOptions(rel_tol=1e-10))
    assert r.history.iterations == 1 and r.history.converged
    A = O.random_spd(np.linspace(0.5, 60, 200), 11)
    b = O.NormalStream(3).draw(200)
    r = O.pcg_split(O.DenseOperator(A), b, opts=O.PcgOptions(max_iter=2000, rel_tol=1e-10))
    direct = np.linalg.solve(A, b)
    assert r.history.converged and np.linalg.norm(r.x - direct) <= 1e-8 * np.linalg.norm(direct)
    with pytest.raises(O.NumericalError):
        O.pcg_split(O.DenseOperator(-np.eye(5)), O.NormalStream(4).draw(5))
    A = O.random_spd(np.linspace(1, 9, 30), 51)
    op = O.DenseOperator(A)
    b = O.NormalStream(8).draw(30)
    op.reset_apply_count()
    r = O.pcg_split(op, b, opts=O.PcgOptions(max_iter=12, rel_tol=1e-15))
    assert op.apply_count() == r.history.iterations
    A = O.random_spd(np.linspace(1, 80, 60), 31)
    b = O.NormalStream(6).draw(60)
    r = O.pcg_split(O.DenseOperator(A), b, opts=O.PcgOptions(
        max_iter=60, rel_tol=1e-14, cost_eval=lambda x: 0.5 * x @ A @ x - b @ x))
    c = r.history.quadratic_costs
    assert len(c) == r.history.iterations + 1
    assert all(c[i + 1] <= c[i] + 1e-10 * abs(c[i]) for i in range(len(c) - 1))
