"""Rank rule of the sketches (ColPivHouseholderQR::rank, randevd.cpp:67-73 / 89-92): Eigen
counts pivots |R_ii| > m eps max|R_kk|.  An ill-conditioned but full-rank sample (cond(Y)
~1e8, beyond what a double Gram can resolve) must pass REVD and keep every Nystrom column,
exactly as the oracle's LAPACK dgeqp3 rule does; a sample whose last singular value is
below Eigen's threshold collapses in both."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu
W = pytest.importorskip("paper_2101_07249_b200")
from gpu_helpers import relerr  # noqa: E402


def _operator(top, tail, n=200, k=12, seed=5):
    V = O.random_orthogonal(n, seed)
    lam = np.concatenate([top, np.full(n - len(top), tail)])
    A = (V * lam) @ V.T
    return 0.5 * (A + A.T)


@pytest.mark.parametrize("method", ["revd", "nystrom"])
def test_ill_conditioned_full_rank_sample(method):
    A = _operator(np.logspace(8, 0, 12), 1e-7)
    k, l = 9, 3
    Om = O.gaussian_matrix(200, k + l, 3)
    r_or, _ = O.colpiv_rank(A @ Om)
    assert r_or == k + l  # Eigen's rule: full rank
    s = np.linalg.svd(A @ Om, compute_uv=False)
    assert s[-1] / s[0] < 1e-7  # far beyond the double Gram's resolution
    cfg = dict(target_rank=k, oversample=l, seed=3, method=method)
    pg = W.sketch_eigenpairs(W.DenseOperator(A), W.SketchConfig(**cfg), Om)
    po = O.sketch_eigenpairs(O.DenseOperator(A), O.SketchConfig(**cfg), Om)
    assert pg.k() == po.k() == k
    assert relerr(pg.values, po.values) <= 1e-10
    assert pg.orthonormality_defect() <= 1e-10


def test_rank_below_eigen_threshold_collapses():
    # the 12th direction of Y sits below 12 eps of the largest: Eigen's rank is 11
    A = _operator(np.concatenate([np.logspace(2, 0, 11), [0.0]]), 0.0)
    k, l = 8, 4
    Om = O.gaussian_matrix(200, k + l, 4)
    r_or, _ = O.colpiv_rank(A @ Om)
    assert r_or == 11
    with pytest.raises(W.NumericalError, match="rank collapsed to 11 of 12"):
        W.sketch_eigenpairs(W.DenseOperator(A), W.SketchConfig(k, l, 4, "revd"), Om)
    pg = W.sketch_eigenpairs(W.DenseOperator(A), W.SketchConfig(k, l, 4, "nystrom"), Om)
    po = O.sketch_eigenpairs(O.DenseOperator(A), O.SketchConfig(k, l, 4, "nystrom"), Om)
    assert pg.k() == po.k() == 8
    assert relerr(pg.values, po.values) <= 1e-10
