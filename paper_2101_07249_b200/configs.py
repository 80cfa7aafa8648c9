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
