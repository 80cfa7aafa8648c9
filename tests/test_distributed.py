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
