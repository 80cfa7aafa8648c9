"""Outer loop and twin data over the device path: the reference's
AssimilationSystem (assimilation.hpp:19-37, assimilation.cpp:11-50), generate_twin
(:75-110), initial_state (:112-118), compute_innovations (:120-128) and outer_update
(:255-263), so that a whole incremental weak-constraint 4D-Var study -- truth, background
and observations, then outer loops of sketch -> LMP -> PCG -> update -- runs on the GPU.

The n(N+1)-long work goes through the C-ABI: the nonlinear trajectory (integrate_p: the
advection forward sweep L^{-1}p, which IS the nonlinear model for the linear advection
equation, or the Lorenz-96 device integrator), the covariance square roots of the noise
draws (D^{1/2} of a window vector), observe() and every inner loop.  What stays on the host
is what the reference's drivers do on scalars and short vectors: seeds, the initial
condition formula, and vector additions of the innovations.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import wc4dvar as W


@dataclass
class ModelGrid:
    """models.hpp:11-21"""

    n: int
    N: int
    dt: float = 0.0
    dx: float = 0.0

    def window_dim(self) -> int:
        return self.n * (self.N + 1)


@dataclass
class TwinSeeds:
    """assimilation.hpp:39-43"""

    background: int = 1
    observations: int = 2
    model_error: int = 3


@dataclass
class TwinData:
    """assimilation.hpp:45-51"""

    truth: np.ndarray       # n x (N+1)
    background: np.ndarray  # n
    y: np.ndarray           # q, network order
    seeds: TwinSeeds


@dataclass
class OuterState:
    """assimilation.hpp:58-63"""

    p: np.ndarray
    traj: np.ndarray  # n x (N+1)
    loop_index: int = 0


@dataclass
class Innovations:
    """assimilation.hpp:67-71"""

    b: np.ndarray
    d: np.ndarray


class AssimilationSystem:
    """assimilation.hpp:19-37: model ("advection" | "lorenz96"), grid, observation network
    and error statistics, fixed across outer loops."""

    def __init__(self, kind: str, grid: ModelGrid, net: W.ObservationNetwork,
                 background_half: W.CovarianceFactor, model_error_half: W.CovarianceFactor,
                 sigma_obs: float, courant: float = 0.0, forcing: float = 8.0, spinup_steps: int = 500,
                 device: int = 0):
        W.require(kind in ("advection", "lorenz96"), "AssimilationSystem: unknown model kind")
        self.kind, self.grid, self.net = kind, grid, net
        self.background_half, self.model_error_half = background_half, model_error_half
        self.sigma_obs, self.courant, self.forcing, self.spinup_steps = sigma_obs, courant, forcing, spinup_steps
        self.device = device
        n, N = grid.n, grid.N
        # device helpers: D^{1/2} and observe() do not depend on the linearisation; the
        # advection operator's forward sweep is the nonlinear model itself
        self._aux = W.HessianOperator(W.IdentityLinearized(n, N), net, background_half, model_error_half,
                                      sigma_obs, device)
        self._adv = (W.HessianOperator(W.AdvectionLinearized(n, N, courant), net, background_half,
                                       model_error_half, sigma_obs, device) if kind == "advection" else None)

    def window_dim(self) -> int:
        return self.grid.window_dim()

    def integrate_p(self, p) -> np.ndarray:
        """assimilation.cpp:21-33: x_0 = p_0, x_{i+1} = M(x_i) + p_{i+1}, on the device."""
        p = np.ascontiguousarray(p, dtype=np.float64)
        W.require(len(p) == self.window_dim(), "integrate_p: control vector length mismatch")
        n, N = self.grid.n, self.grid.N
        if self.kind == "lorenz96":
            return W.integrate_p(p, n, N, self.forcing, self.grid.dt, 1, self.device)
        traj = self._adv.apply_Linv(p).reshape(n, N + 1, order="F")
        if not np.all(np.isfinite(traj)):
            bad = int(np.argmax(~np.all(np.isfinite(traj), axis=0)))
            raise W.NumericalError(f"integrate_p: non-finite trajectory at step {bad}")
        return traj

    def linearize(self, trajectory) -> W.LinearizedModel:
        """assimilation.cpp:35-44"""
        if self.kind == "advection":
            return W.AdvectionLinearized(self.grid.n, self.grid.N, self.courant)
        return W.Lorenz96Linearized(trajectory, self.forcing, self.grid.dt)

    def hessian(self, trajectory) -> W.HessianOperator:
        """assimilation.cpp:46-50"""
        return W.HessianOperator(self.linearize(trajectory), self.net, self.background_half,
                                 self.model_error_half, self.sigma_obs, self.device)

    def observe(self, traj) -> np.ndarray:
        return self._aux.observe(traj)

    def d_half(self, v) -> np.ndarray:
        return self._aux.apply_D_half(v)


def _advection_initial_condition(grid: ModelGrid) -> np.ndarray:
    """assimilation.cpp:54-63: Gaussian bump 6 exp(-(z - 0.5)^2 / (2 0.1^2)), z = j dx."""
    u = np.empty(grid.n)
    for j in range(grid.n):
        arg = (j * grid.dx - 0.5) / 0.1
        u[j] = 6.0 * math.exp(-0.5 * arg * arg)
    return u


def _lorenz96_initial_condition(sys: AssimilationSystem) -> np.ndarray:
    """assimilation.cpp:65-71: perturbed equilibrium spun up on the device."""
    x = np.full(sys.grid.n, sys.forcing)
    x[0] += 0.01
    return W.lorenz96_trajectory(x, sys.forcing, sys.grid.dt, sys.spinup_steps, 0, sys.device)[:, 0]


def generate_twin(sys: AssimilationSystem, seeds: TwinSeeds, noise_scale: float = 1.0,
                  truth_model_error: bool = False) -> TwinData:
    """assimilation.cpp:75-110: truth by the nonlinear model (optionally forced by
    noise_scale Q^{1/2} xi_i), background x_0 + noise_scale B^{1/2} xi_b, observations
    H(truth) + noise_scale sigma_o xi_o -- the truth integration, both square roots and
    observe() on the device."""
    W.require(noise_scale >= 0.0, "generate_twin: noise scale must be nonnegative")
    n, N = sys.grid.n, sys.grid.N
    x0 = _advection_initial_condition(sys.grid) if sys.kind == "advection" else _lorenz96_initial_condition(sys)
    p = np.zeros(sys.window_dim())
    p[:n] = x0
    if truth_model_error and noise_scale > 0.0:
        xi = np.zeros(sys.window_dim())
        xi[n:] = W.gaussian_matrix(n * N, 1, seeds.model_error)[:, 0]  # model_noise.draw(n) per step
        p[n:] = noise_scale * sys.d_half(xi)[n:]                       # Q^{1/2} xi_{i+1}
    try:
        truth = sys.integrate_p(p)
    except W.NumericalError:
        raise W.NumericalError("generate_twin: truth integration became non-finite") from None
    background = truth[:, 0].copy()
    if noise_scale > 0.0:
        xb = np.zeros(sys.window_dim())
        xb[:n] = W.gaussian_matrix(n, 1, seeds.background)[:, 0]
        background = background + noise_scale * sys.d_half(xb)[:n]
    y = sys.observe(truth)
    if noise_scale > 0.0:
        y = y + noise_scale * sys.sigma_obs * W.gaussian_matrix(len(y), 1, seeds.observations)[:, 0]
    return TwinData(truth, background, y, seeds)


def initial_state(sys: AssimilationSystem, twin: TwinData) -> OuterState:
    """assimilation.cpp:112-118"""
    p = np.zeros(sys.window_dim())
    p[:sys.grid.n] = twin.background
    return OuterState(p, sys.integrate_p(p), 0)


def compute_innovations(sys: AssimilationSystem, state: OuterState, twin: TwinData) -> Innovations:
    """assimilation.cpp:120-128: b = (x^b - x_0, -eta_1, ..., -eta_N), d = y - H(x)."""
    n = sys.grid.n
    b = -state.p
    b[:n] = twin.background - state.traj[:, 0]
    return Innovations(b, twin.y - sys.observe(state.traj))


def outer_update(sys: AssimilationSystem, state: OuterState, delta_p) -> OuterState:
    """assimilation.cpp:255-263"""
    delta_p = np.asarray(delta_p, dtype=np.float64)
    W.require(len(delta_p) == len(state.p), "outer_update: increment length mismatch")
    p = state.p + delta_p
    return OuterState(p, sys.integrate_p(p), state.loop_index + 1)


@dataclass
class OuterLoopReport:
    """One inner loop per outer iteration plus the final state."""

    inner: List[W.InnerLoopReport] = field(default_factory=list)
    final: Optional[OuterState] = None


def run_outer_loops(sys: AssimilationSystem, twin: TwinData, precond: W.PrecondSpec, solver: W.SolverSpec,
                    n_outer: int, dense_cap: int = 4096) -> OuterLoopReport:
    """The incremental loop of the reference's runner: linearise at the current trajectory,
    run the inner loop on the innovations, update the control vector.  A deterministic
    preconditioner takes the previous loop's Hessian (assimilation.cpp:204-211)."""
    state = initial_state(sys, twin)
    rep = OuterLoopReport()
    prev = None
    for _ in range(n_outer):
        h = sys.hessian(state.traj)
        inn = compute_innovations(sys, state, twin)
        spec = precond if (precond.kind != "deterministic" or prev is not None) else W.PrecondSpec("none")
        r = W.run_inner_loop(h, inn.b, inn.d, spec, solver, dense_cap=dense_cap, previous_hessian=prev)
        rep.inner.append(r)
        state = outer_update(sys, state, r.delta_p)
        prev = h
    rep.final = state
    return rep
