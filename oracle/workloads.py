"""BASELINE.json configs restated for the CPU oracle -- TEST INFRASTRUCTURE ONLY.

The same five workloads as the product's ``paper_2101_07249_b200/configs.py``, built
from the oracle's own primitives (``oracle.py`` / ``wc4dvar_oracle.c``) so that
``bench.py --impl reference`` and the ``cpu_baseline`` leg never import the product
package (importing it would dlopen ``libwc4dvar_gpu.so`` into the reference process).
``tests/test_host_logic.py::test_oracle_workloads_match_product_configs`` checks the two
descriptions agree field by field.

Seeds (BASELINE.json gives none): Omega seed 1 (the reference's ``sketch_base = 1``,
proj/configs/advection.cfg:39), right-hand side seed 2, Lorenz-96 initial state seed 3.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import oracle as O

OMEGA_SEED = 1
RHS_SEED = 2
L96_X0_SEED = 3


@dataclass
class OracleWorkload:
    name: str
    op: "O.HessianOperator"
    m: int    # sketch columns k + l
    k: int    # LMP rank
    n: int
    N: int
    substeps: int
    q: int
    kind: str
    covariance: str

    @property
    def dim(self) -> int:
        return self.n * (self.N + 1)


def _advdiff(name, n, N, s, L, sx, m, k, sigma_b=1.0, var_q=0.05, sigma_o=0.1, circulant=False,
             threads=1):
    model = O.AdvDiffLinearized(n, N, 0.5, 0.2, s)
    net = O.ObservationNetwork.build(n, N, sx, 1)
    if circulant:
        b = O.circulant_sqrt(O.soar_first_column(sigma_b, L, n))
        qf = O.circulant_sqrt(O.soar_first_column(math.sqrt(var_q), L, n))
    else:
        b = O.sym_sqrt(O.build_soar(sigma_b, L, n))
        qf = O.sym_sqrt(O.build_soar(math.sqrt(var_q), L, n))
    op = O.HessianOperator(model, net, b, qf, sigma_o, threads=threads)
    return OracleWorkload(name, op, m, k, n, N, s, net.q, "advdiff", "circulant SOAR" if circulant else "dense SOAR")


def config1(threads=1):
    """BASELINE configs[0]."""
    return _advdiff("C1-advdiff-n100-N4-s10", 100, 4, 10, 5.0, 5, 20, 10, threads=threads)


def config2(threads=1):
    """BASELINE configs[1]."""
    return _advdiff("C2-advdiff-n2000-N20-s10", 2000, 20, 10, 20.0, 4, 100, 50, threads=threads)


def config4(m=64, threads=1):
    """BASELINE configs[3] (circulant SOAR L = 50; sigma_b = 1, Q variance 0.05)."""
    return _advdiff(f"C4-advdiff-n1e6-N16-s10-m{m}", 1_000_000, 16, 10, 50.0, 10, m, m // 2,
                    circulant=True, threads=threads)


def l96_trajectory(n, forcing, dt, spinup, steps, seed=L96_X0_SEED):
    """Seeded N(0,1) state (NormalStream::draw, random.hpp:33-37) spun up with
    lorenz96_step (models.cpp:72-78), then `steps` more states (n x (steps+1))."""
    x = O.NormalStream(seed).draw(n)
    for _ in range(spinup):
        x = O.lorenz96_step(x, forcing, dt)
    traj = np.empty((n, steps + 1), order="F")
    traj[:, 0] = x
    for c in range(steps):
        x = O.lorenz96_step(x, forcing, dt)
        traj[:, c + 1] = x
    return traj


def _l96(name, n, N, s, m, k, forcing=8.0, dt=0.025, spinup=1000, L=4.0, var_q_ratio=0.1,
         sigma_o=0.2, threads=1):
    traj = l96_trajectory(n, forcing, dt, spinup, N * s)
    model = O.Lorenz96Linearized(traj, forcing, dt, s)
    net = O.ObservationNetwork.build(n, N, 2, 1)
    col = O.soar_first_column(1.0, L, n)
    op = O.HessianOperator(model, net, O.circulant_sqrt(col), O.circulant_sqrt(var_q_ratio * col), sigma_o,
                           threads=threads)
    return OracleWorkload(name, op, m, k, n, N, s, net.q, "l96", "circulant SOAR")


def config3(threads=1):
    """BASELINE configs[2]."""
    return _l96("C3-l96-n1e5-N10-s5", 100_000, 10, 5, 64, 32, threads=threads)


def config5(m=256, threads=1):
    """BASELINE configs[4] ("k = 256" read as the sketch width; LMP rank m - 16)."""
    return _l96("C5-l96-n2e6-N20-s5", 2_000_000, 20, 5, m, m - 16, threads=threads)
