"""Outer loop and twin data on the device path: generate_twin,
initial_state, compute_innovations, outer_update and the outer-loop driver
(assimilation.cpp:11-128, 255-263) against the oracle's restatement, for the advection and
Lorenz-96 systems of the reference's test suite shapes."""

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

W = pytest.importorskip("paper_2101_07249_b200")
from paper_2101_07249_b200 import assimilation as A  # noqa: E402
from gpu_helpers import factor, relerr  # noqa: E402


def systems(kind):
    if kind == "advection":  # the advection study shape (n = 40, N = 50, strides 4 / 5)
        n, N, dt = 40, 50, 0.0
        bc, qc = O.build_covariance("soar", 0.1, 10.0, n), O.build_covariance("laplacian", 0.05, 10.0, n)
        net = (4, 5)
        kw = dict(courant=0.02 * n)
        sig = 0.05
    else:  # a small Lorenz-96 system (tiny_lorenz-like)
        n, N, dt = 24, 8, 0.05
        bc, qc = O.build_soar(1.0, 2.0, n), O.build_soar(0.3, 2.0, n)
        net = (2, 1)
        kw = dict(forcing=8.0, spinup_steps=100)
        sig = 0.5
    bo, qo = O.sym_sqrt(bc), O.sym_sqrt(qc)
    gsys = A.AssimilationSystem(kind, A.ModelGrid(n, N, dt, 1.0 / n), W.ObservationNetwork.build(n, N, *net),
                                factor(bc), factor(qc), sig, **kw)
    osys = O.AssimSystem(kind, n, N, dt, 1.0 / n, O.ObservationNetwork.build(n, N, *net), bo, qo, sig, **kw)
    return gsys, osys


@pytest.mark.parametrize("kind", ["advection", "lorenz96"])
@pytest.mark.parametrize("model_error", [False, True])
def test_generate_twin_vs_oracle(kind, model_error):
    g, o = systems(kind)
    tw = A.generate_twin(g, A.TwinSeeds(11, 12, 13), 1.0, model_error)
    truth, bg, y = O.generate_twin(o, (11, 12, 13), 1.0, model_error)
    assert relerr(tw.truth, truth) <= 1e-12
    assert relerr(tw.background, bg) <= 1e-12
    assert relerr(tw.y, y) <= 1e-12
    exact = A.generate_twin(g, A.TwinSeeds(11, 12, 13), 0.0)
    assert np.array_equal(exact.y, g.observe(exact.truth))  # noise_scale 0: exact data


@pytest.mark.parametrize("kind", ["advection", "lorenz96"])
def test_initial_state_innovations_update(kind):
    g, o = systems(kind)
    tw = A.generate_twin(g, A.TwinSeeds(), 1.0, True)
    st = A.initial_state(g, tw)
    p = np.zeros(g.window_dim())
    p[:g.grid.n] = tw.background
    assert relerr(st.traj, o.integrate_p(p)) <= 1e-12
    inn = A.compute_innovations(g, st, tw)
    b, d = O.compute_innovations(o, st.p, st.traj, tw.background, tw.y)
    assert np.array_equal(inn.b, b) and relerr(inn.d, d) <= 1e-14
    dp = 1e-2 * O.NormalStream(4).draw(g.window_dim())
    nxt = A.outer_update(g, st, dp)
    assert nxt.loop_index == 1
    assert relerr(nxt.traj, o.integrate_p(st.p + dp)) <= 1e-12
    with pytest.raises(ValueError, match="increment length mismatch"):
        A.outer_update(g, st, dp[:-1])


@pytest.mark.parametrize("kind,precond", [("advection", "nystrom"), ("lorenz96", "revd"),
                                          ("lorenz96", "deterministic")])
def test_outer_loops_vs_oracle(kind, precond):
    """Two outer loops; every inner loop's solution and the final control vector agree with
    the oracle driving its own operators on the same data."""
    g, o = systems(kind)
    tw = A.generate_twin(g, A.TwinSeeds(21, 22, 23), 1.0, True)
    spec = W.PrecondSpec(precond, 8, 4, 5)
    solver = W.SolverSpec(max_iter=300, rel_tol=1e-10, record_cost=False)
    rep = A.run_outer_loops(g, tw, spec, solver, 2)
    # oracle twin of the same loop
    p = np.zeros(g.window_dim())
    p[:g.grid.n] = tw.background
    traj = o.integrate_p(p)
    prev = None
    for loop in range(2):
        h = o.hessian(traj)
        b, d = O.compute_innovations(o, p, traj, tw.background, tw.y)
        cost = O.QuadraticCost(h, b, d)
        f = None
        if precond == "deterministic" and prev is not None:
            ev, V = np.linalg.eigh(O.assemble_dense(prev))
            f = O.build_spectral_lmp(O.RitzPairs(np.asfortranarray(V[:, ::-1][:, :8]), ev[::-1][:8].copy()))
        elif precond != "deterministic":
            f = O.build_spectral_lmp(O.sketch_eigenpairs(h, O.SketchConfig(8, 4, 5, precond)))
        sol = O.pcg_split(h, cost.rhs(), f, opts=O.PcgOptions(max_iter=300, rel_tol=1e-10))
        dp = h.apply_D_half(sol.x)
        if loop == 0:
            scale = np.abs(dp).max()
        # relative to the first increment: for the linear advection model the second
        # increment is rounding-level (the first loop already solved the problem)
        assert np.abs(rep.inner[loop].delta_p - dp).max() <= 1e-7 * scale, loop
        p = p + dp
        traj = o.integrate_p(p)
        prev = h
    assert relerr(rep.final.p, p) <= 1e-8
    assert rep.final.loop_index == 2
