"""GPU parity of the Hessian block apply and its pieces against the oracle, plus the
reference's operator known-answer tests (proj/tests/test_operators.cpp) on the device path."""
import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2101_07249_b200")
from gpu_helpers import factor, identity_factor, pair, relerr, workload_pair  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402


def adv_factors(n):
    return factor(O.build_soar(0.1, 3.0, n)), factor(O.build_laplacian_corr(0.05, 2.0, n))


def advection_pair(n, N, courant, sx, st):  # test_operators.cpp:30-34
    bh, qh = adv_factors(n)
    return pair(W.AdvectionLinearized(n, N, courant), W.ObservationNetwork.build(n, N, sx, st), bh, qh,
                0.05)


@pytest.mark.parametrize("m", [1, 3, 8])
def test_advection_reference_model_block(m):
    g, o = advection_pair(40, 50, 0.8, 4, 5)  # the advection study operator shape
    V = O.gaussian_matrix(g.dim(), m, 7)
    assert relerr(g.apply_block(V), o.apply_block(V)) <= 1e-13


@pytest.mark.parametrize("wl", [configs.small_advdiff(), configs.small_advdiff(n=37, N=3, s=1, sx=3),
                                configs.config1()], ids=lambda w: w.name)
def test_advdiff_substeps_block(wl):
    g, o = workload_pair(wl)
    V = O.gaussian_matrix(g.dim(), wl.m, 1)
    assert relerr(g.apply_block(V), o.apply_block(V)) <= 1e-13
    for name in ("apply_Linv", "apply_LinvT", "apply_D_half", "apply_D_half_inv"):
        v = V[:, 0]
        assert relerr(getattr(g, name)(v), getattr(o, name)(v)) <= 1e-12, name


def test_identity_model_cumulative_sums():  # :38-63
    g, _ = pair(W.IdentityLinearized(3, 3), W.ObservationNetwork.build(3, 3, 1, 1), identity_factor(3),
                identity_factor(3), 1.0)
    s = O.NormalStream(2)
    p = s.draw(12)
    assert np.abs(g.apply_Linv(p) - np.cumsum(p.reshape(4, 3), axis=0).ravel()).max() <= 1e-14
    v = s.draw(12)
    exp = np.cumsum(v.reshape(4, 3)[::-1], axis=0)[::-1].ravel()
    assert np.abs(g.apply_LinvT(v) - exp).max() <= 1e-14


def test_zero_step_window_and_no_observations():  # :65-76, :122-133
    g, _ = pair(W.IdentityLinearized(4, 0), W.ObservationNetwork.empty(4, 0), identity_factor(4),
                identity_factor(4), 1.0)
    p = O.NormalStream(3).draw(4)
    assert np.array_equal(g.apply_Linv(p), p) and np.array_equal(g.apply_LinvT(p), p)
    g, _ = pair(W.IdentityLinearized(5, 3), W.ObservationNetwork.empty(5, 3), identity_factor(5),
                identity_factor(5), 1.0)
    v = O.NormalStream(9).draw(20)
    assert np.abs(g.apply(v) - v).max() <= 1e-14
    assert np.abs(g.apply(np.zeros(20))).max() == 0.0


def test_first_principles_dense_and_spd():  # :135-169
    n, N = 4, 3
    bh, qh = factor(O.build_soar(0.1, 2.0, n)), factor(O.build_laplacian_corr(0.05, 1.5, n))
    g, o = pair(W.AdvectionLinearized(n, N, 0.8), W.ObservationNetwork.build(n, N, 2, 1), bh, qh, 0.05)
    L = np.column_stack([o.apply_Linv(e) for e in np.eye(16)])
    H = np.zeros((o.network().q, 16))
    r = 0
    for t in o.network().times:
        for j in o.network().points:
            H[r, t * n + j] = 1.0
            r += 1
    D = np.zeros((16, 16))
    D[:4, :4] = bh.half
    for i in range(1, N + 1):
        D[i * 4:(i + 1) * 4, i * 4:(i + 1) * 4] = qh.half
    dense = np.eye(16) + D @ L.T @ H.T @ H @ L @ D / 0.05 ** 2
    assert np.abs(W.assemble_dense(g) - dense).max() <= 1e-11
    g, _ = advection_pair(6, 4, 0.8, 2, 2)
    s = O.NormalStream(11)
    for _ in range(20):
        a, b = s.draw(30), s.draw(30)
        Aa, Ab = g.apply(a), g.apply(b)
        assert abs(Aa @ b - a @ Ab) <= 1e-10 * (1 + abs(Aa @ b))
        assert Aa @ a >= (a @ a) * (1 - 1e-10)


def test_unit_cluster():  # :171-186
    g, _ = advection_pair(8, 5, 0.8, 2, 1)
    eigs = np.linalg.eigvalsh(W.assemble_dense(g))
    q = g.network().q
    assert (np.abs(eigs - 1) <= 1e-8).sum() == g.dim() - q and (eigs > 1 + 1e-8).sum() == q


def test_block_equals_columns_bitwise_and_counts():  # :188-221
    g, _ = advection_pair(5, 3, 0.8, 2, 1)
    V = O.NormalStream(13).fill(g.dim(), 7)
    serial = np.column_stack([g.apply(V[:, j]) for j in range(7)])
    assert np.array_equal(g.apply_block(V), serial)
    g.reset_apply_count()
    s = O.NormalStream(17)
    g.apply(s.draw(g.dim()))
    assert g.apply_count() == 1
    g.apply_block(s.fill(g.dim(), 4))
    assert g.apply_count() == 5
    wl = configs.small_advdiff()
    g2, _ = workload_pair(wl)
    V = O.gaussian_matrix(g2.dim(), 40, 3)  # enough columns to switch GEMM tile shapes
    B = g2.apply_block(V)
    for j in (0, 17, 39):
        assert np.array_equal(B[:, j], g2.apply(V[:, j]))


def test_stream_k_block_equals_columns_bitwise():
    """At C2 size the D^1/2 GEMM runs stream-K (272 tiles on 148 SMs, tiles split across
    CTAs); the split resumes the published DMMA accumulators, so the block apply still equals
    the column-wise apply (one-CTA-per-tile kernels) bit for bit (test_operators.cpp:188-211)."""
    g = configs.config2().hessian(0)
    V = O.gaussian_matrix(g.dim(), 100, 5)
    B = g.apply_block(V)
    for j in (0, 37, 63, 99):
        assert np.array_equal(B[:, j], g.apply(V[:, j])), j
    assert np.array_equal(g.apply_block(V), B)  # run-to-run deterministic


def test_errors():  # :263-277
    g, _ = pair(W.IdentityLinearized(4, 2), W.ObservationNetwork.build(4, 2, 2, 1), identity_factor(4),
                identity_factor(4), 1.0)
    bad = np.zeros(12)
    bad[0] = np.nan
    with pytest.raises(W.NumericalError, match="forward sweep"):
        g.apply(bad)
    g, _ = advection_pair(5, 3, 0.8, 2, 1)
    with pytest.raises(ValueError):
        g.apply(np.zeros(7))
    with pytest.raises(ValueError):
        g.apply_Linv(np.zeros(7))
    with pytest.raises(W.DenseCapError):
        W.assemble_dense(g, g.dim() - 1)


def test_dense_operator_apply():
    A = O.random_spd(np.linspace(1, 9, 33), 3)
    g = W.DenseOperator(A)
    V = O.gaussian_matrix(33, 5, 2)
    assert relerr(g.apply_block(V), A @ V) <= 1e-14
    assert g.apply_count() == 5


def test_config2_columns_vs_oracle():
    # BASELINE configs[1] operator: a few columns against the oracle at full size.
    wl = configs.config2()
    g, o = workload_pair(wl)
    V = O.gaussian_matrix(g.dim(), 4, 1)
    assert relerr(g.apply_block(V), o.apply_block(V)) <= 1e-12
