"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: column-sharded A*Omega,
the all-to-all column<->row transposes, row-sharded CholQR2 / REVD / Nystrom / ritzit with
all-reduced Gram matrices and row-sharded PCG with all-reduced dots -- each against the
single-process oracle on the same inputs (TorchOps backend; the device backend is
tests/test_gpu_distributed.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn_name):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        globals()[fn_name](rank, world)
    finally:
        dist.destroy_process_group()


def _run(fn_name, world=2):
    mp.spawn(_worker, args=(world, _free_port(), fn_name), nprocs=world, join=True)


# ----------------------------------------------------------------------------- bodies
def _body_sharded_apply(rank, world):
    from oracle import oracle as O
    from paper_2101_07249_b200.distributed import all_gather_cat, column_range
    n, N, m = 40, 5, 7
    op = O.HessianOperator(O.AdvDiffLinearized(n, N, 0.5, 0.2, 3), O.ObservationNetwork.build(n, N, 4, 1),
                           O.sym_sqrt(O.build_soar(1.0, 4.0, n)), O.sym_sqrt(O.build_soar(0.3, 4.0, n)), 0.1)
    Om = O.gaussian_matrix(op.dim(), m, 1)
    a, b = column_range(m, world, rank)
    local = torch.from_numpy(op.apply_block(Om[:, a:b]))
    sizes = [column_range(m, world, r)[1] - column_range(m, world, r)[0] for r in range(world)]
    full = all_gather_cat(local, sizes, dim=1).numpy()
    assert np.array_equal(full, op.apply_block(Om))  # column sharding is bitwise invariant


def _body_transposes(rank, world):
    from paper_2101_07249_b200.distributed import cols_to_rows, column_range, row_range, rows_to_cols
    n, m = 23, 9
    full = torch.arange(n * m, dtype=torch.float64).reshape(m, n).T.contiguous()  # n x m
    a, b = column_range(m, world, rank)
    rows = cols_to_rows(full[:, a:b].contiguous(), n, m)
    ra, rb = row_range(n, world, rank)
    assert torch.equal(rows, full[ra:rb, :])
    back = rows_to_cols(rows, n, m)
    assert torch.equal(back, full[:, a:b])


def _spd_case():
    from oracle import oracle as O
    n_ = 80
    A = O.random_spd(np.concatenate([np.linspace(40, 5, 10), np.linspace(2, 1, n_ - 10)]), 3)
    return n_, A


def _body_revd_pcg(rank, world):
    from oracle import oracle as O
    from paper_2101_07249_b200.distributed import (all_gather_cat, column_range, dist_cholqr2, dist_pcg,
                                                   dist_revd, row_range)
    n_, A = _spd_case()
    k, l = 6, 4
    m = k + l
    Om = O.gaussian_matrix(n_, m, 5)
    a, b = column_range(m, world, rank)
    At = torch.from_numpy(A)
    apply_cols = lambda X: At @ X  # noqa: E731
    U_rows, theta = dist_revd(apply_cols, torch.from_numpy(Om[:, a:b].copy()), n_, m, k)
    ref = O.revd(O.DenseOperator(A), O.SketchConfig(k, l, 5), Om)
    assert np.abs(theta.numpy() - ref.values).max() <= 1e-10 * ref.values.max()
    # U is row-sharded; gather and compare the projector
    ra, rb = row_range(n_, world, rank)
    rsz = [row_range(n_, world, r)[1] - row_range(n_, world, r)[0] for r in range(world)]
    U = all_gather_cat(U_rows.contiguous(), rsz).numpy()
    assert np.abs(U @ U.T - ref.vectors @ ref.vectors.T).max() <= 1e-8
    # CholQR2 orthonormality and Y = Q R on row shards
    Y = torch.from_numpy(Om[ra:rb, :].copy())
    Q, R = dist_cholqr2(Y, want_r=True)
    G = (Q.T @ Q).contiguous()
    dist.all_reduce(G)
    assert (G - torch.eye(m, dtype=torch.float64)).abs().max() <= 1e-13
    assert (Q @ R - Y).abs().max() <= 1e-13 * Y.abs().max()
    # row-sharded PCG with the LMP vs the oracle
    b = O.NormalStream(2).draw(n_)

    def apply_rows(p_rows):  # replicated apply: gather p, apply, keep the own rows
        return (At @ all_gather_cat(p_rows, rsz))[ra:rb]

    res = dist_pcg(apply_rows, torch.from_numpy(b[ra:rb].copy()), U_rows, theta, 200, 1e-10)
    oref = O.pcg_split(O.DenseOperator(A), b, O.build_spectral_lmp(ref), opts=O.PcgOptions(200, 1e-10))
    assert res.converged and abs(res.iterations - oref.history.iterations) <= 1
    x = all_gather_cat(res.x_rows, rsz).numpy()
    assert np.abs(x - oref.x).max() <= 1e-9 * np.abs(oref.x).max()
    # the device-side stop test (host check every 8 / 5 iterations, later iterations masked)
    # reproduces the per-iteration loop exactly: same iterations, residuals and x bits
    for ce in (5, 8):
        r1 = dist_pcg(apply_rows, torch.from_numpy(b[ra:rb].copy()), U_rows, theta, 200, 1e-10, check_every=1)
        r2 = dist_pcg(apply_rows, torch.from_numpy(b[ra:rb].copy()), U_rows, theta, 200, 1e-10, check_every=ce)
        assert r1.iterations == r2.iterations == res.iterations and r1.converged and r2.converged
        assert r1.residual_norms == r2.residual_norms
        assert torch.equal(r1.x_rows, r2.x_rows)
    # max_iter reached without convergence: every issued iteration is live
    r3 = dist_pcg(apply_rows, torch.from_numpy(b[ra:rb].copy()), U_rows, theta, 3, 1e-14, check_every=8)
    assert not r3.converged and r3.iterations == 3 and len(r3.residual_norms) == 4


def _gather_rows(U_rows, n_, world):
    from paper_2101_07249_b200.distributed import all_gather_cat, row_range
    rsz = [row_range(n_, world, r)[1] - row_range(n_, world, r)[0] for r in range(world)]
    return all_gather_cat(U_rows.contiguous(), rsz).numpy()


def _body_nystrom_ritzit(rank, world):
    from oracle import oracle as O
    from paper_2101_07249_b200.distributed import column_range, dist_nystrom, dist_ritzit, row_range
    n_, A = _spd_case()
    At = torch.from_numpy(A)
    apply_cols = lambda X: At @ X  # noqa: E731
    k, l = 6, 4
    m = k + l
    a, b = column_range(m, world, rank)
    ra, rb = row_range(n_, world, rank)
    for seed in (5, 6):
        Om = O.gaussian_matrix(n_, m, seed)
        U_rows, theta = dist_nystrom(apply_cols, torch.from_numpy(Om[:, a:b].copy()), n_, m, k)
        ref = O.nystrom(O.DenseOperator(A), O.SketchConfig(k, l, seed, "nystrom"), Om)
        assert np.abs(theta.numpy() - ref.values).max() <= 1e-10 * ref.values.max()
        U = _gather_rows(U_rows, n_, world)
        assert np.abs(U @ U.T - ref.vectors @ ref.vectors.T).max() <= 1e-8
        for p_iter in (1, 3):
            U_rows, theta = dist_ritzit(apply_cols, torch.from_numpy(Om[ra:rb, :].copy()), n_, m, k,
                                        p_iter=p_iter)
            ref = O.revd_ritzit(O.DenseOperator(A), O.SketchConfig(k, l, seed, "ritzit", p_iter), Om)
            assert np.abs(theta.numpy() - ref.values).max() <= 1e-10 * ref.values.max()
            U = _gather_rows(U_rows, n_, world)
            assert np.abs(U @ U.T - ref.vectors @ ref.vectors.T).max() <= 1e-8


def _body_nystrom_rank_cap(rank, world):
    # test_randevd.cpp:153-168: a rank-3 operator; Nystrom caps k at the detected rank
    from oracle import oracle as O
    from paper_2101_07249_b200.distributed import column_range, dist_nystrom
    n_ = 50
    V = O.random_orthogonal(n_, 7)[:, :3]
    A = V @ np.diag([5.0, 3.0, 2.0]) @ V.T
    At = torch.from_numpy(A)
    m = 8
    a, b = column_range(m, world, rank)
    Om = O.gaussian_matrix(n_, m, 11)
    U_rows, theta = dist_nystrom(lambda X: At @ X, torch.from_numpy(Om[:, a:b].copy()), n_, m, 6)
    assert theta.numel() == 3
    assert np.abs(np.sort(theta.numpy())[::-1] - [5.0, 3.0, 2.0]).max() <= 1e-10 * 5.0


@pytest.mark.parametrize("body", ["_body_sharded_apply", "_body_transposes", "_body_revd_pcg",
                                  "_body_nystrom_ritzit", "_body_nystrom_rank_cap"])
def test_world_size_2_gloo(body):
    _run(body, 2)


def test_column_range_partition():
    from paper_2101_07249_b200.distributed import column_range
    for m in (1, 7, 100, 256):
        for world in (1, 2, 3, 8):
            cols = []
            for r in range(world):
                a, b = column_range(m, world, r)
                cols.extend(range(a, b))
            assert cols == list(range(m))


# ----------------------------------------------------------------------------- row-sharded apply
class OracleSlabOps:
    """CPU local steps of the row-sharded apply from the oracle (test infrastructure): the
    n-point covariance factors, and the window sweeps on the extended slab (oracle model of
    n_ext points, observed points inside the slab) -- orc_hessian_sweeps."""

    def __init__(self, o, geom, net):
        from oracle import oracle as O
        from paper_2101_07249_b200.distributed import slab_network
        self.O, self.o, self.geom = O, o, geom
        m = o.model
        ne = geom.n_ext
        idx = geom.ext_points().numpy()
        st = None
        if m.kind == "l96":
            st = m.stages.reshape(-1, 4, m.n)[:, :, idx].reshape(-1, 4 * ne)
        smodel = O.LinearizedModel(m.kind, ne, m.N, m.substeps, m.courant, m.diffusion, m.dt, st)
        pts, times = slab_network(net.points, net.times, m.n, geom)
        snet = O.ObservationNetwork(ne, m.N, 1, 1, list(times), list(pts), len(times) * len(pts))
        e0 = np.zeros(ne)
        e0[0] = 1.0
        eye = O.CovarianceFactor(e0, e0, "circulant")
        self.sop = O.HessianOperator(smodel, snet, eye, eye, o.sigma_obs())

    def factor(self, X, which):
        f = self.o.b_half if which == 0 else self.o.q_half
        return torch.from_numpy(np.stack([f.apply(x) for x in X.numpy()]))

    def sweeps(self, T):
        import ctypes
        t = np.ascontiguousarray(T.numpy().reshape(-1))
        assert self.O._lib.orc_hessian_sweeps(ctypes.byref(self.sop._h), self.O._ptr(t)) == 0
        return torch.from_numpy(t.reshape(T.shape))


def _row_sharded_cases():
    from oracle import oracle as O
    from oracle import workloads as OW
    adv = OW._advdiff("advdiff", 64, 4, 3, 4.0, 4, 6, 3)
    circ = OW._advdiff("advdiff-circ", 90, 5, 4, 5.0, 3, 6, 3, circulant=True)
    l96 = OW._l96("l96", 120, 3, 2, 6, 3, spinup=40)
    return [adv, circ, l96]


def _body_row_sharded_apply(rank, world):
    """RowShardedHessian (spatial slabs, block-sharded D^{1/2} by all-to-all, one halo
    exchange per apply) vs the oracle's full HessianOperator::apply, and row-sharded PCG
    on it vs the oracle's pcg_split."""
    from oracle import oracle as O
    from paper_2101_07249_b200.distributed import (RowShardedHessian, SlabGeometry, dist_pcg,
                                                   window_halo)
    for wl in _row_sharded_cases():
        o = wl.op
        geom = SlabGeometry(wl.n, wl.N, world, rank, window_halo(wl.kind, wl.N, wl.substeps))
        rsh = RowShardedHessian(geom, OracleSlabOps(o, geom, o.network()))
        idx = geom.window_indices().numpy()
        V = O.gaussian_matrix(wl.dim, 3, 17)
        ref = o.apply_block(V)
        for c in range(3):
            v = torch.from_numpy(np.ascontiguousarray(V[idx, c]).reshape(wl.N + 1, geom.n_loc))
            out = rsh.apply(v).reshape(-1).numpy()
            err = np.abs(out - ref[idx, c]).max() / np.abs(ref).max()
            assert err <= 1e-13, (wl.name, c, err)
        # PCG with an LMP, row-sharded on the slabs
        cfg = O.SketchConfig(wl.k, wl.m - wl.k, 1, "nystrom")
        pairs = O.sketch_eigenpairs(o, cfg)
        b = O.NormalStream(2).draw(wl.dim)
        res = dist_pcg(rsh.apply_rows, torch.from_numpy(b[idx].copy()),
                       torch.from_numpy(np.ascontiguousarray(pairs.vectors[idx, :])),
                       torch.from_numpy(pairs.values.copy()), 200, 1e-10)
        oref = O.pcg_split(o, b, O.build_spectral_lmp(pairs), opts=O.PcgOptions(200, 1e-10))
        # iteration counts within one where the run is insensitive to the summation order
        # of the dots (2 ranks); with 3 ranks the 1e-10 stop of the Lorenz-96 case moves by a
        # few iterations under reordering alone, so the bound there is 5 % of the count
        allow = 1 if world == 2 else max(1, oref.history.iterations // 20)
        assert res.converged and abs(res.iterations - oref.history.iterations) <= allow, (
            wl.name, res.iterations, oref.history.iterations)
        err = np.abs(res.x_rows.numpy() - oref.x[idx]).max() / np.abs(oref.x).max()
        assert err <= 1e-9, (wl.name, err)


def test_row_sharded_apply_gloo():
    _run("_body_row_sharded_apply", 2)


def test_row_sharded_apply_three_ranks():
    _run("_body_row_sharded_apply", 3)


def test_window_halo_reach():
    from paper_2101_07249_b200.distributed import window_halo
    assert window_halo("advdiff", 16, 10) == 320 and window_halo("l96", 20, 5) == 1208
    assert window_halo("advection", 50, 1) == 50
    assert window_halo("identity", 4, 3) == 0
