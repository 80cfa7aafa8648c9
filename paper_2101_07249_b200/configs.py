"""BASELINE.json workload builders (host-side setup, like the reference's covariance.cpp
builders and ExperimentConfig::build_system, config.cpp:313-327).

The covariance factors are INPUTS of the operator API (HessianOperator takes
CovarianceFactor objects, operators.hpp:119-123); building them is one-time host setup
(an O(n^3) symmetric EVD for dense factors, exactly as sym_sqrt does in the reference).

Seeds are not given by BASELINE.json; we use Omega seed 1 (the reference's own
``sketch_base = 1``, proj/configs/advection.cfg:39), right-hand side seed 2 and
Lorenz-96 initial-state seed 3.
"""
from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .wc4dvar import (AdvDiffLinearized, CovarianceFactor, HessianOperator, LinearizedModel,
                      ObservationNetwork)

OMEGA_SEED = 1
RHS_SEED = 2
L96_X0_SEED = 3


def soar_matrix(sigma: float, length: float, n: int) -> np.ndarray:
    """build_soar, covariance.cpp:25-48 (chordal distance), vectorised."""
    i = np.arange(n)
    d = np.abs(i[:, None] - i[None, :])
    d = np.minimum(d, n - d).astype(np.float64)
    r = (n / math.pi) * np.sin(math.pi * d / n)
    return np.asfortranarray(sigma * sigma * (1.0 + r / length) * np.exp(-r / length))


def sym_sqrt(C: np.ndarray) -> CovarianceFactor:
    """sym_sqrt, covariance.cpp:86-105."""
    w, V = np.linalg.eigh(C)
    if w.min() <= 0.0:
        raise ValueError(f"sym_sqrt: matrix is not positive definite (eigenvalue {w.min()})")
    root = np.sqrt(w)
    half = (V * root) @ V.T
    half_inv = (V / root) @ V.T
    return CovarianceFactor(np.asfortranarray(0.5 * (half + half.T)),
                            np.asfortranarray(0.5 * (half_inv + half_inv.T)))


def soar_first_column(sigma: float, length: float, n: int) -> np.ndarray:
    """First column of build_soar (covariance.cpp:31-44) without forming n x n."""
    d = np.minimum(np.arange(n), n - np.arange(n)).astype(np.float64)
    r = (n / math.pi) * np.sin(math.pi * d / n)
    return sigma * sigma * (1.0 + r / length) * np.exp(-r / length)


def circulant_sqrt(first_col: np.ndarray) -> CovarianceFactor:
    """EXTENSION: symmetric square root of a symmetric circulant SPD matrix
    from its first column (eigenvalues = DFT of the column); equals sym_sqrt of the dense
    matrix to rounding (pinned in tests/test_oracle_models.py)."""
    lam = np.real(np.fft.fft(first_col))
    if lam.min() <= 0.0:
        raise ValueError(f"circulant_sqrt: matrix is not positive definite (eigenvalue {lam.min()})")
    half = np.real(np.fft.ifft(np.sqrt(lam)))
    half_inv = np.real(np.fft.ifft(1.0 / np.sqrt(lam)))
    return CovarianceFactor(np.ascontiguousarray(half), np.ascontiguousarray(half_inv), kind="circulant")


@dataclass
class Workload:
    name: str
    model: LinearizedModel
    net: ObservationNetwork
    b_half: CovarianceFactor
    q_half: CovarianceFactor
    sigma_obs: float
    m: int                  # sketch columns k + l
    k: int                  # LMP rank
    p_iter: int = 1

    @property
    def dim(self) -> int:
        return self.model.n * (self.model.N + 1)

    def hessian(self, device: int = 0) -> HessianOperator:
        return HessianOperator(self.model, self.net, self.b_half, self.q_half, self.sigma_obs, device)


def advdiff_workload(name, n, N, s, L, sx, m, k, sigma_b=1.0, var_q=0.05, sigma_o=0.1,
                     courant=0.5, diffusion=0.2, p_iter=1) -> Workload:
    model = AdvDiffLinearized(n, N, courant, diffusion, s)
    net = ObservationNetwork.build(n, N, sx, 1)
    b = sym_sqrt(soar_matrix(sigma_b, L, n))
    q = sym_sqrt(soar_matrix(math.sqrt(var_q), L, n))
    return Workload(name, model, net, b, q, sigma_o, m, k, p_iter)


def config1() -> Workload:
    """BASELINE configs[0]: n=100, Nsw=4, s=10, SOAR L=5, obs every 5th point, m=20, k=10."""
    return advdiff_workload("C1-advdiff-n100-N4-s10", 100, 4, 10, 5.0, 5, 20, 10, p_iter=3)


def config2() -> Workload:
    """BASELINE configs[1]: n=2000, Nsw=20, s=10, SOAR L=20, obs every 4th point, m=100, k=50."""
    return advdiff_workload("C2-advdiff-n2000-N20-s10", 2000, 20, 10, 20.0, 4, 100, 50)


def small_advdiff(n=64, N=5, s=3, L=4.0, sx=4, m=12, k=6) -> Workload:
    """A fast parity case with the C1/C2 structure."""
    return advdiff_workload(f"advdiff-n{n}-N{N}-s{s}", n, N, s, L, sx, m, k)


def config4(m: int = 64) -> Workload:
    """BASELINE configs[3]: advection-diffusion n=1e6, Nsw=16, s=10, circulant SOAR L=50
    (sigma_b = 1, Q variance 0.05 -- BASELINE gives no values; chosen as in C1/C2),
    R = 0.01 I, every 10th point observed; sketch width m in {16, 64, 256}."""
    n, N = 1_000_000, 16
    model = AdvDiffLinearized(n, N, 0.5, 0.2, 10)
    net = ObservationNetwork.build(n, N, 10, 1)
    b = circulant_sqrt(soar_first_column(1.0, 50.0, n))
    q = circulant_sqrt(soar_first_column(math.sqrt(0.05), 50.0, n))
    return Workload(f"C4-advdiff-n1e6-N16-s10-m{m}", model, net, b, q, 0.1, m, m // 2)


def lorenz96_workload(name, n, N, s, m, k, forcing=8.0, dt=0.025, spinup=1000, L=4.0,
                      var_q_ratio=0.1, sigma_o=0.2) -> Workload:
    """BASELINE configs[2] / [4]: Lorenz-96 TL/adjoint, RK4 dt=0.025, F=8, s sub-steps per
    subwindow; linearisation trajectory from a seeded N(0,1) state spun up `spinup` steps
    (composed from the reference primitives NormalStream::draw and lorenz96_step, SURVEY
    §0.2-4); B = SOAR(L) circulant, Q = 0.1 B, R = 0.04 I, every other variable observed."""
    from .wc4dvar import Lorenz96Linearized, gaussian_matrix, lorenz96_trajectory_device
    x0 = gaussian_matrix(n, 1, L96_X0_SEED)[:, 0]
    # spin-up, trajectory and stages stay on the device
    traj = lorenz96_trajectory_device(x0, forcing, dt, spinup, N * s)
    model = Lorenz96Linearized(traj, forcing, dt, s)
    net = ObservationNetwork.build(n, N, 2, 1)
    col = soar_first_column(1.0, L, n)
    b = circulant_sqrt(col)
    q = circulant_sqrt(var_q_ratio * col)
    return Workload(name, model, net, b, q, sigma_o, m, k)


def config3() -> Workload:
    """BASELINE configs[2]: Lorenz-96 n=1e5, Nsw=10, s=5, m=64, k=32."""
    return lorenz96_workload("C3-l96-n1e5-N10-s5", 100_000, 10, 5, 64, 32)


def config5(m: int = 256) -> Workload:
    """BASELINE configs[4]: Lorenz-96 n=2e6, Nsw=20, s=5; Nystrom sketch of width 256
    ("k=256" read as the sketch width; LMP rank 240 with oversampling 16)."""
    return lorenz96_workload("C5-l96-n2e6-N20-s5", 2_000_000, 20, 5, m, m - 16)
