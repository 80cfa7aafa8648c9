"""Fourier-space form of the Hessian block apply (csrc/spectral.cu, the forward-only /
inverse-only modes of csrc/fft4.cu): parity with the oracle's grid-space apply
(operators.cpp:127-144 restated), agreement with the product's own grid-space path on the same
operator, eligibility rules and the reference's stage errors."""
import math

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2101_07249_b200")
from gpu_helpers import pair, relerr  # noqa: E402
from paper_2101_07249_b200 import configs  # noqa: E402


def circ_factors(n, L, var_q=0.05):
    return (configs.circulant_sqrt(configs.soar_first_column(1.0, L, n)),
            configs.circulant_sqrt(configs.soar_first_column(math.sqrt(var_q), L, n)))


def _net(n, N, sx, st=1, times=None):
    net = W.ObservationNetwork.build(n, N, sx, st)
    if times is not None:  # an irregular subset of observation times (time 0 included)
        net = W.ObservationNetwork(n, N, sx, st, list(times), list(net.points), len(times) * len(net.points))
    return net


# n = 1e4 runs the fused plan 400 x 25 (last row radix 20): strides 1, 2, 4, 5, 10, 20 divide it
@pytest.mark.parametrize("sx,m,kind", [(4, 5, "advdiff"), (10, 4, "advdiff"), (1, 2, "advdiff"), (20, 3, "advdiff"),
                                       (5, 1, "advdiff"), (2, 6, "advection"), (10, 3, "identity")])
def test_spectral_apply_vs_oracle(sx, m, kind):
    n, N, s = 10000, 3, 3
    bh, qh = circ_factors(n, 5.0)
    model = {"advdiff": W.AdvDiffLinearized(n, N, 0.5, 0.2, s),
             "advection": W.LinearizedModel("advection", n, N, s, 0.4),
             "identity": W.LinearizedModel("identity", n, N)}[kind]
    g, o = pair(model, _net(n, N, sx), bh, qh, 0.1)
    assert g.spectral(), "operator should be eligible for the Fourier-space apply"
    V = O.gaussian_matrix(g.dim(), m, 1)
    ref = o.apply_block(V)
    spec = g.apply_block(V)
    assert relerr(spec, ref) <= 1e-12
    assert g.spectral(0) is False
    grid = g.apply_block(V)
    assert relerr(grid, ref) <= 1e-12
    err = relerr(spec, grid)
    print(f"sx={sx} m={m} {kind}: spectral vs oracle {relerr(spec, ref):.2e}, vs grid-space path {err:.2e}")
    assert err <= 1e-12
    assert g.spectral(1) is True
    v = V[:, 0].copy()
    assert relerr(g.apply(v), o.apply(v)) <= 1e-12  # single vector: window blocks packed in pairs


def test_spectral_single_column_block_packing():
    """One column packs its window blocks in pairs and separates the spectra by Hermitian
    symmetry (spectral_window1): odd and even block counts, the self-mirrored row k2 = 0 of the
    digit-reversed order, against the oracle and against the generic (half-empty) packing."""
    for n, N, sx in ((10000, 3, 10), (10000, 4, 4), (100000, 6, 10), (1000000, 16, 10)):  # the last: C4's grid and window
        bh, qh = circ_factors(n, 7.0)
        model, net = W.AdvDiffLinearized(n, N, 0.5, 0.2, 3), _net(n, N, sx)
        g, o = pair(model, net, bh, qh, 0.1)
        assert g.spectral()
        v = O.gaussian_matrix(g.dim(), 1, 5)[:, 0].copy()
        ref = o.apply(v) if n <= 10000 else None
        packed = g.apply(v)
        # the same column as one of two sketch columns runs the generic column-packed form
        generic = g.apply_block(np.asfortranarray(np.stack([v, 0.5 * v], axis=1)))[:, 0]
        if ref is not None:
            assert relerr(packed, ref) <= 1e-12
        err = relerr(packed, generic)
        print(f"n={n} N={N}: block-packed single column vs column-packed {err:.2e}")
        assert err <= 1e-12


def test_spectral_time_subsets_and_long_window():
    """Observation times that skip intervals and include time 0 (slot table), and a window longer
    than the kernel's load ring."""
    n, N, s = 10000, 9, 2
    bh, qh = circ_factors(n, 8.0)
    for net in (_net(n, N, 10, 2), _net(n, N, 10, 1, times=[0, 3, 4, 9]), _net(n, N, 4, 3)):
        g, o = pair(W.AdvDiffLinearized(n, N, 0.5, 0.2, s), net, bh, qh, 0.2)
        assert g.spectral()
        V = O.gaussian_matrix(g.dim(), 3, 2)
        assert relerr(g.apply_block(V), o.apply_block(V)) <= 1e-12


def test_spectral_eligibility():
    n, N = 10000, 2
    bh, qh = circ_factors(n, 5.0)
    model = W.AdvDiffLinearized(n, N, 0.5, 0.2, 2)
    # stride 8 divides n but not the last row radix (20); stride 3 does not divide n
    for sx in (8, 3):
        g, o = pair(model, _net(n, N, sx), bh, qh, 0.1)
        assert not g.spectral()
        with pytest.raises(ValueError):
            g.spectral(1)
        V = O.gaussian_matrix(g.dim(), 2, 1)
        assert relerr(g.apply_block(V), o.apply_block(V)) <= 1e-12
    # irregular points
    net = _net(n, N, 10)
    pts = list(net.points)
    pts[5] += 1
    irr = W.ObservationNetwork(n, N, 10, 1, list(net.times), pts, net.q)
    assert not pair(model, irr, bh, qh, 0.1)[0].spectral()
    # dense factors (C1 / C2 representation) and a grid without a fused plan
    wl = configs.small_advdiff()
    assert not wl.hessian(0).spectral()
    b2, q2 = circ_factors(300, 5.0)
    assert not pair(W.AdvDiffLinearized(300, 2, 0.5, 0.2, 2), _net(300, 2, 10), b2, q2, 0.1)[0].spectral()
    # Lorenz-96 is not a constant-coefficient stencil
    wl = configs.lorenz96_workload("l96-1e4", 10000, 2, 2, 4, 2, spinup=50)
    assert not wl.hessian(0).spectral()


def test_spectral_stage_errors():
    """operators.cpp:133-143: a non-finite input surfaces as the forward-sweep error."""
    n, N = 10000, 2
    bh, qh = circ_factors(n, 5.0)
    g, _ = pair(W.AdvDiffLinearized(n, N, 0.5, 0.2, 2), _net(n, N, 10), bh, qh, 0.1)
    assert g.spectral()
    V = O.gaussian_matrix(g.dim(), 2, 1)
    V[17, 1] = np.nan
    with pytest.raises(W.NumericalError, match="forward sweep"):
        g.apply_block(V)
    V[17, 1] = 0.0
    assert np.isfinite(g.apply_block(V)).all()


def test_spectral_sketch_and_pcg_vs_oracle():
    """The LMP build and LMP-PCG on top of the Fourier-space apply (randevd.cpp:62-136,
    krylov.cpp:22-99) against the oracle on its grid-space apply."""
    n, N, s = 10000, 2, 3
    bh, qh = circ_factors(n, 5.0)
    g, o = pair(W.AdvDiffLinearized(n, N, 0.5, 0.2, s), _net(n, N, 10), bh, qh, 0.1)
    assert g.spectral()
    pairs = {}
    for method in ("revd", "nystrom", "ritzit"):
        cfg = dict(target_rank=8, oversample=8, seed=1, method=method)
        pg = W.sketch_eigenpairs(g, W.SketchConfig(**cfg))
        po = O.sketch_eigenpairs(o, O.SketchConfig(**cfg))
        assert relerr(pg.values, po.values) <= 1e-10, method
        pairs[method] = (pg, po)
    b = O.NormalStream(7).draw(g.dim())
    pg, po = pairs["nystrom"]
    rg = W.pcg_split(g, b, W.build_spectral_lmp(pg), opts=W.PcgOptions(rel_tol=1e-8, max_iter=400))
    ro = O.pcg_split(o, b, O.build_spectral_lmp(po), opts=O.PcgOptions(rel_tol=1e-8, max_iter=400))
    assert abs(rg.history.iterations - ro.history.iterations) <= 1
    assert relerr(rg.x, ro.x) <= 1e-9


@pytest.mark.parametrize("n,N,s,sx,m", [(100000, 6, 10, 10, 4), (1000000, 16, 10, 10, 3)])
def test_spectral_vs_grid_space_large(n, N, s, sx, m):
    """The n = 1e5 (400 x 250) and n = 1e6 (4000 x 250, the C4 grid and window) plans: the
    Fourier-space apply against the grid-space path (two fused convolutions + tiled sweeps,
    itself checked against the oracle at these sizes in test_gpu_configs_parity.py), plus the
    adjoint identity <A u, v> = <u, A v> on the spectral path."""
    bh, qh = circ_factors(n, 50.0)
    g = W.HessianOperator(W.AdvDiffLinearized(n, N, 0.5, 0.2, s), _net(n, N, sx), bh, qh, 0.1)
    assert g.spectral()
    V = W.gaussian_matrix(g.dim(), m, 3)
    spec = g.apply_block(V)
    g.spectral(0)
    grid = g.apply_block(V)
    err = relerr(spec, grid)
    print(f"n={n}: spectral vs grid-space path {err:.2e}")
    assert err <= 1e-12
    g.spectral(1)
    lhs, rhs = float(spec[:, 0] @ V[:, 1]), float(V[:, 0] @ spec[:, 1])
    assert abs(lhs - rhs) <= 1e-11 * max(abs(lhs), abs(rhs))
