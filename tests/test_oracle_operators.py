"""proj/tests/test_operators.cpp ported onto the oracle's HessianOperator."""
import numpy as np
import pytest

from oracle import oracle as O


def identity_factor(n):
    return O.sym_sqrt(np.eye(n))


def soar_factor(n, sigma, length):
    return O.sym_sqrt(O.build_soar(sigma, length, n))


def laplacian_factor(n, sigma, length):
    return O.sym_sqrt(O.build_laplacian_corr(sigma, length, n))


def advection_hessian(n, N, courant, sx, st):  # test_operators.cpp:30-34
    return O.HessianOperator(O.AdvectionLinearized(n, N, courant),
                             O.ObservationNetwork.build(n, N, sx, st),
                             soar_factor(n, 0.1, 3.0), laplacian_factor(n, 0.05, 2.0), 0.05)


def dense_Linv(op):  # test_support.hpp:31-49 (first principles, column by column)
    n, N = op.model.n, op.model.N
    return np.column_stack([op.apply_Linv(e) for e in np.eye(n * (N + 1))])


def dense_H(net):  # test_support.hpp:52-58
    H = np.zeros((net.q, net.n * (net.N + 1)))
    r = 0
    for t in net.times:
        for j in net.points:
            H[r, t * net.n + j] = 1.0
            r += 1
    return H


def test_identity_model_cumulative_sums():  # :38-63
    op = O.HessianOperator(O.IdentityLinearized(3, 3), O.ObservationNetwork.build(3, 3, 1, 1),
                           identity_factor(3), identity_factor(3), 1.0)
    s = O.NormalStream(2)
    p = s.draw(12)
    expect = np.cumsum(p.reshape(4, 3), axis=0).ravel()
    assert np.abs(op.apply_Linv(p) - expect).max() <= 1e-14
    v = s.draw(12)
    expect_t = np.cumsum(v.reshape(4, 3)[::-1], axis=0)[::-1].ravel()
    assert np.abs(op.apply_LinvT(v) - expect_t).max() <= 1e-14


def test_zero_step_window_identity():  # :65-76
    op = O.HessianOperator(O.IdentityLinearized(4, 0), O.ObservationNetwork.empty(4, 0),
                           identity_factor(4), identity_factor(4), 1.0)
    p = O.NormalStream(3).draw(4)
    assert np.array_equal(op.apply_Linv(p), p)
    assert np.array_equal(op.apply_LinvT(p), p)


def test_Linv_vs_dense_and_adjoint_identity():  # :78-120
    model = O.AdvectionLinearized(4, 2, 0.8)
    op = O.HessianOperator(model, O.ObservationNetwork.build(4, 2, 2, 1), identity_factor(4),
                           identity_factor(4), 1.0)
    # first-principles L^{-1} from tlm steps
    n, N = 4, 2
    L = np.zeros((12, 12))
    for col in range(12):
        blk = col // n
        x = np.zeros(n)
        x[col % n] = 1.0
        L[blk * n:(blk + 1) * n, col] = x
        for i in range(blk, N):
            x = O.advection_step(x, 0.8)
            L[(i + 1) * n:(i + 2) * n, col] = x
    s = O.NormalStream(5)
    for _ in range(5):
        p = s.draw(12)
        assert np.abs(op.apply_Linv(p) - L @ p).max() <= 1e-12
        assert np.abs(op.apply_LinvT(p) - L.T @ p).max() <= 1e-12
    s = O.NormalStream(7)
    op = O.HessianOperator(O.AdvectionLinearized(6, 4, 0.8), O.ObservationNetwork.build(6, 4, 2, 2),
                           identity_factor(6), identity_factor(6), 1.0)
    for _ in range(10):
        p, v = s.draw(30), s.draw(30)
        a, b = op.apply_Linv(p) @ v, p @ op.apply_LinvT(v)
        assert abs(a - b) <= 1e-12 * (1 + abs(a))
    traj = np.empty((8, 6))
    traj[:, 0] = 8.0 + 0.4 * s.draw(8)
    for i in range(5):
        traj[:, i + 1] = O.lorenz96_step(traj[:, i], 8.0, 0.05)
    op = O.HessianOperator(O.Lorenz96Linearized(traj, 8.0, 0.05), O.ObservationNetwork.build(8, 5, 2, 2),
                           identity_factor(8), identity_factor(8), 1.0)
    for _ in range(10):
        p, v = s.draw(48), s.draw(48)
        a, b = op.apply_Linv(p) @ v, p @ op.apply_LinvT(v)
        assert abs(a - b) <= 1e-12 * (1 + abs(a))


def test_no_observations_is_identity():  # :122-133
    op = O.HessianOperator(O.IdentityLinearized(5, 3), O.ObservationNetwork.empty(5, 3),
                           identity_factor(5), identity_factor(5), 1.0)
    v = O.NormalStream(9).draw(20)
    assert np.abs(op.apply(v) - v).max() <= 1e-14
    assert np.abs(op.apply(np.zeros(20))).max() == 0.0


def test_hessian_vs_first_principles():  # :135-153
    n, N = 4, 3
    model = O.AdvectionLinearized(n, N, 0.8)
    net = O.ObservationNetwork.build(n, N, 2, 1)
    bh, qh = soar_factor(n, 0.1, 2.0), laplacian_factor(n, 0.05, 1.5)
    op = O.HessianOperator(model, net, bh, qh, 0.05)
    L = dense_Linv(op)
    H = dense_H(net)
    D = np.zeros((16, 16))
    D[:4, :4] = bh.half
    for i in range(1, N + 1):
        D[i * 4:(i + 1) * 4, i * 4:(i + 1) * 4] = qh.half
    dense = np.eye(16) + D @ L.T @ H.T @ H @ L @ D / 0.05 ** 2
    assert np.abs(O.assemble_dense(op) - dense).max() <= 1e-11


def test_linear_symmetric_pd():  # :155-169
    op = advection_hessian(6, 4, 0.8, 2, 2)
    s = O.NormalStream(11)
    u, v = s.draw(30), s.draw(30)
    lhs = op.apply(1.3 * u - 0.7 * v)
    rhs = 1.3 * op.apply(u) - 0.7 * op.apply(v)
    assert np.abs(lhs - rhs).max() <= 1e-12 * (1 + np.abs(lhs).max())
    for _ in range(50):
        a, b = s.draw(30), s.draw(30)
        sym = op.apply(a) @ b - a @ op.apply(b)
        assert abs(sym) <= 1e-10 * (1 + abs(op.apply(a) @ b))
        assert op.apply(a) @ a >= (a @ a) * (1 - 1e-10)


def test_unit_cluster():  # :171-186
    op = advection_hessian(8, 5, 0.8, 2, 1)
    eigs = np.linalg.eigvalsh(O.assemble_dense(op))
    q = op.network().q
    assert (np.abs(eigs - 1.0) <= 1e-8).sum() == op.dim() - q
    assert (eigs > 1 + 1e-8).sum() == q
    assert eigs.min() >= 1 - 1e-8


def test_block_equals_columns_thread_invariant():  # :188-209
    op = advection_hessian(5, 3, 0.8, 2, 1)
    V = O.NormalStream(13).fill(op.dim(), 7)
    serial = np.column_stack([op.apply(V[:, j]) for j in range(7)])
    assert np.array_equal(op.apply_block(V, threads=3), serial)
    assert np.array_equal(op.apply_block(V, threads=1), serial)
    assert np.array_equal(op.apply_block(V[:, :1])[:, 0], op.apply(V[:, 0]))


def test_apply_counting():  # :211-221
    op = advection_hessian(5, 3, 0.8, 2, 1)
    op.reset_apply_count()
    s = O.NormalStream(17)
    op.apply(s.draw(op.dim()))
    assert op.apply_count() == 1
    op.apply_block(s.fill(op.dim(), 4))
    assert op.apply_count() == 5


def test_dense_cap_and_errors():  # :223-227, :263-277
    op = advection_hessian(8, 5, 0.8, 2, 1)
    with pytest.raises(O.DenseCapError):
        O.assemble_dense(op, op.dim() - 1)
    op = O.HessianOperator(O.IdentityLinearized(4, 2), O.ObservationNetwork.build(4, 2, 2, 1),
                           identity_factor(4), identity_factor(4), 1.0)
    bad = np.zeros(12)
    bad[0] = np.nan
    with pytest.raises(O.NumericalError):
        op.apply(bad)
    op = advection_hessian(5, 3, 0.8, 2, 1)
    with pytest.raises(ValueError):
        op.apply(np.zeros(7))
    with pytest.raises(ValueError):
        op.apply_Linv(np.zeros(7))


def test_clustered_spectrum_vs_dense():  # :228-261
    op = advection_hessian(6, 5, 0.8, 2, 2)
    A = O.assemble_dense(op)
    full = O.clustered_spectrum(op).full()
    assert np.abs(full - np.linalg.eigvalsh(A)[::-1]).max() <= 1e-9
    w, V = np.linalg.eigh(A)
    f = O.LmpFactor(V[:, ::-1][:, :4].copy(), w[::-1][:4].copy())
    cs = O.clustered_spectrum(op, f)
    C = np.eye(op.dim())
    for i in range(4):
        C -= (1 - 1 / np.sqrt(f.values[i])) * np.outer(f.vectors[:, i], f.vectors[:, i])
    dense = np.linalg.eigvalsh(C.T @ A @ C)[::-1]
    assert np.abs(cs.full() - dense).max() <= 1e-9


def test_substeps_compose_interval_steps():
    # EXTENSION: s sub-steps per subwindow == reference window with N*s intervals, observed
    # only at subwindow ends (D^{1/2} = identity, so L^{-1} is pure propagation).
    n, N, s = 7, 3, 4
    sub = O.HessianOperator(O.AdvDiffLinearized(n, N, 0.5, 0.2, s), O.ObservationNetwork.build(n, N, 1, 1),
                            identity_factor(n), identity_factor(n), 1.0)
    p = O.NormalStream(1).draw(n * (N + 1))
    x = sub.apply_Linv(p)
    cur = p[:n]
    for i in range(N):
        for _ in range(s):
            cur = O.advdiff_step(cur, 0.5, 0.2)
        cur = cur + p[(i + 1) * n:(i + 2) * n]
        assert np.abs(x[(i + 1) * n:(i + 2) * n] - cur).max() <= 1e-13
    v = O.NormalStream(2).draw(n * (N + 1))
    assert abs(sub.apply_Linv(p) @ v - p @ sub.apply_LinvT(v)) <= 1e-12 * (1 + abs(p @ v))
