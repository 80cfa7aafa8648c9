"""Device backend of the multi-GPU sketches (paper_2101_07249_b200/distributed.py DeviceOps
over the C-ABI row-sharded building blocks), on one rank: the distributed REVD / Nystrom /
ritzit run the same kernel sequence as wc4dvar_gpu_sketch, so their Ritz pairs must be
bitwise identical to it; row-sharded PCG must match pcg_split (iterations within one,
solution 1e-9 relative).  The N>1 exchange logic is covered by the gloo tests
(tests/test_distributed.py)."""
import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2101_07249_b200")
from gpu_helpers import workload_pair  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402
from paper_2101_07249_b200 import distributed as D  # noqa: E402


def _dev(a):
    return D.fcontig(torch.from_numpy(np.asfortranarray(a)).cuda())


def _ops_case():
    wl = configs.config1()
    g, _ = workload_pair(wl)
    return wl, g


@pytest.mark.parametrize("method", ["revd", "nystrom", "ritzit"])
def test_device_ops_match_single_gpu_sketch_bitwise(method):
    wl, g = _ops_case()
    n, k, m = g.dim(), wl.k, wl.m
    Om = W.gaussian_matrix(n, m, configs.OMEGA_SEED)
    ops = D.DeviceOps(0)
    apply_cols = D.hessian_apply_cols(g)
    if method == "revd":
        U, th = D.dist_revd(apply_cols, _dev(Om), n, m, k, ops)
    elif method == "nystrom":
        U, th = D.dist_nystrom(apply_cols, _dev(Om), n, m, k, ops)
    else:
        U, th = D.dist_ritzit(apply_cols, _dev(Om), n, m, k, ops, p_iter=1)
    torch.cuda.synchronize()
    ref = W.sketch_eigenpairs(g, W.SketchConfig(k, m - k, configs.OMEGA_SEED, method), Om)
    assert np.array_equal(th.cpu().numpy(), ref.values)
    assert np.array_equal(U.cpu().numpy(), ref.vectors)


def test_device_ops_building_blocks_vs_torch():
    rng = np.random.default_rng(3)
    Y = rng.standard_normal((1001, 37))
    Yd = _dev(Y)
    dev, cpu = D.DeviceOps(0), D.TorchOps
    Yc = D.fcontig(torch.from_numpy(Y))
    G = dev.gram(Yd, Yd)
    assert np.abs(G.cpu().numpy() - Y.T @ Y).max() <= 1e-12 * np.abs(Y.T @ Y).max()
    R = dev.chol_upper(G)
    Rc = cpu.chol_upper(D.fcontig(G.cpu()))
    assert np.abs(R.cpu().numpy() - Rc.numpy()).max() <= 1e-12 * np.abs(Rc.numpy()).max()
    Ri = dev.tri_inv_upper(R)
    Q = dev.tall_times_small(Yd, Ri)
    Qc = Yc @ cpu.tri_inv_upper(Rc)
    assert np.abs(Q.cpu().numpy() - Qc.numpy()).max() <= 1e-11
    K = dev.small_mm(R, R, tb=True)
    assert np.abs(K.cpu().numpy() - (Rc @ Rc.T).numpy()).max() <= 1e-12 * float((Rc @ Rc.T).abs().max())
    vals, V = dev.eigh_desc(K)
    vc, _ = cpu.eigh_desc(D.fcontig(K.cpu()))
    assert np.abs(vals.cpu().numpy() - vc.numpy()).max() <= 1e-10 * float(vc.abs().max())
    s, U = dev.svd_left(R)
    sc, _ = cpu.svd_left(D.fcontig(R.cpu()))
    assert np.abs(s.cpu().numpy() - sc.numpy()).max() <= 1e-10 * float(sc.max())
    # pivoted rank probe on a rank-5 Gram: same rank and pivot order as the torch rule
    Z = rng.standard_normal((300, 5)) @ rng.standard_normal((5, 12))
    Gz = _dev(Z.T @ Z)
    r, perm = dev.pivoted_rank(Gz, 32 * np.sqrt(300) * 2.2e-16)
    rc, permc = cpu.pivoted_rank(D.fcontig(Gz.cpu()), 32 * np.sqrt(300) * 2.2e-16)
    assert r == rc == 5
    assert perm.cpu().tolist()[:5] == permc.tolist()[:5]
    Sel = dev.gather_cols(_dev(Z), perm, r)
    assert np.array_equal(Sel.cpu().numpy(), Z[:, perm.cpu().numpy()[:5]])


def test_device_ops_errors_are_typed():
    ops = D.DeviceOps(0)
    bad = _dev(-np.eye(4))
    with pytest.raises(W.NumericalError):
        ops.chol_upper(bad)


def test_row_sharded_pcg_device_ops_vs_pcg_split():
    wl, g = _ops_case()
    n, k, m = g.dim(), wl.k, wl.m
    pr = W.sketch_eigenpairs(g, W.SketchConfig(k, m - k, configs.OMEGA_SEED, "nystrom"))
    b = O.NormalStream(configs.RHS_SEED).draw(n)
    ref = W.pcg_split(g, b, W.build_spectral_lmp(pr), None, W.PcgOptions(200, 1e-8))
    apply_cols = D.hessian_apply_cols(g)
    res = D.dist_pcg(lambda p: apply_cols(p.reshape(-1, 1)).reshape(-1), _dev(b).reshape(-1),
                     _dev(pr.vectors), torch.from_numpy(pr.values).cuda(), 200, 1e-8, ops=D.DeviceOps(0))
    assert res.converged and abs(res.iterations - ref.history.iterations) <= 1
    x = res.x_rows.cpu().numpy()
    assert np.abs(x - ref.x).max() <= 1e-9 * np.abs(ref.x).max()


@pytest.mark.parametrize("m", [1, 2, 20, 37, 64, 100, 128, 129])
def test_chol_inv_fused_vs_torch(m):
    rng = np.random.default_rng(m)
    Y = rng.standard_normal((4 * m + 8, m))
    G = Y.T @ Y
    R, Ri = D.DeviceOps(0).chol_inv(_dev(G))
    R, Ri = R.cpu().numpy(), Ri.cpu().numpy()
    Rc = np.linalg.cholesky(G).T
    assert np.array_equal(np.tril(R, -1), np.zeros((m, m))) and np.array_equal(np.tril(Ri, -1), np.zeros((m, m)))
    assert np.abs(R - Rc).max() <= 1e-12 * np.abs(Rc).max()
    assert np.abs(Ri @ R - np.eye(m)).max() <= 1e-12
    with pytest.raises(W.NumericalError):
        D.DeviceOps(0).chol_inv(_dev(G - 2 * np.abs(G).max() * np.eye(m)))


@pytest.mark.parametrize("m", [1, 2, 7, 20, 64, 100, 128, 129, 200, 255, 256])
def test_small_evd_svd_vs_lapack(m):
    """sym_evd_desc (Cholesky + one-sided Jacobi for SPD -- register kernel for m <= 128, the
    4-CTA cluster kernel for 128 < m <= 256 -- with the two-sided Jacobi fallback for
    indefinite input) and svd_left_desc against LAPACK: values 1e-12 relative to the
    largest, vectors through the projector of well-separated leading pairs."""
    rng = np.random.default_rng(100 + m)
    ops = D.DeviceOps(0)
    Q, _ = np.linalg.qr(rng.standard_normal((m, m)))
    for spd in (True, False):
        lam = np.linspace(1.0, 50.0, m) if spd else np.linspace(-20.0, 30.0, m)
        K = (Q * lam) @ Q.T
        vals, V = ops.eigh_desc(_dev(K))
        vals, V = vals.cpu().numpy(), V.cpu().numpy()
        ref = np.sort(lam)[::-1]
        assert np.abs(vals - ref).max() <= 1e-12 * np.abs(ref).max(), (spd, np.abs(vals - ref).max())
        assert np.abs(V.T @ V - np.eye(m)).max() <= 1e-12
        assert np.abs(K @ V - V * vals).max() <= 1e-11 * np.abs(ref).max()
    X = rng.standard_normal((m, m))
    s, U = ops.svd_left(_dev(X))
    s, U = s.cpu().numpy(), U.cpu().numpy()
    sref = np.linalg.svd(X, compute_uv=False)
    assert np.abs(s - sref).max() <= 1e-12 * sref.max()
    assert np.abs(U.T @ U - np.eye(m)).max() <= 1e-12
    # U diag(s) is X's column space image: X X^T U = U diag(s^2)
    assert np.abs(X @ X.T @ U - U * s * s).max() <= 1e-11 * sref.max() ** 2



@pytest.mark.parametrize("case", ["advdiff-dense", "advdiff-circulant", "lorenz96"])
@pytest.mark.parametrize("world", [2, 3])
def test_row_sharded_apply_device(case, world):
    """The row-sharded Hessian apply (spatial slabs, block-sharded D^{1/2}, one halo exchange,
    distributed.RowShardedHessian) on the DEVICE backend: `world` ranks as host threads on
    one GPU (ThreadComm; every exchange completes on the host between launches), each with
    its own C-ABI handles (factor apply + the WC4DVAR_SWEEPS piece on its extended slab),
    against the single-handle block apply."""
    import threading

    from paper_2101_07249_b200.distributed import (DeviceSlabOps, RowShardedHessian, SlabGeometry, ThreadComm,
                                                   window_halo)
    if case == "advdiff-dense":
        wl = configs.small_advdiff(n=96, N=5, s=3)
    elif case == "advdiff-circulant":
        wl = configs.Workload("c", W.AdvDiffLinearized(400, 6, 0.5, 0.2, 4), W.ObservationNetwork.build(400, 6, 3, 1),
                              configs.circulant_sqrt(configs.soar_first_column(1.0, 6.0, 400)),
                              configs.circulant_sqrt(configs.soar_first_column(0.3, 6.0, 400)), 0.1, 6, 3)
    else:
        wl = configs.lorenz96_workload("l96", 300, 3, 2, 6, 3, spinup=50)
    g = wl.hessian(0)
    nA, n, N = g.dim(), wl.model.n, wl.model.N
    V = torch.from_numpy(O.gaussian_matrix(nA, 2, 23).T.copy()).cuda()
    ref = torch.empty_like(V)
    g.apply_block_dev(V, ref)
    torch.cuda.synchronize()
    hub = ThreadComm(world)
    errs, outs = [], {}

    def run(rank):
        try:
            geom = SlabGeometry(n, N, world, rank, window_halo(wl.model.kind, N, wl.model.substeps))
            ops = DeviceSlabOps(wl.model, wl.net, wl.b_half, wl.q_half, wl.sigma_obs, geom, 0)
            rsh = RowShardedHessian(geom, ops, hub.bind(rank))
            idx = geom.window_indices().cuda()
            for c in range(2):
                outs[(rank, c)] = (rsh.apply(V[c][idx].reshape(N + 1, geom.n_loc)).reshape(-1), idx)
        except Exception as e:  # surfaced below
            errs.append(e)

    th = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    scale = ref.abs().max()
    for (rank, c), (out, idx) in outs.items():
        err = float((out - ref[c][idx]).abs().max() / scale)
        assert err <= 1e-13, (case, rank, c, err)
