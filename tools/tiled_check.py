"""Parity driver for the tiled window sweeps (run as a subprocess by tests/test_gpu_tiled.py
with WC4DVAR_SWEEP_TILE set, so the halo / multi-launch path runs on sizes the oracle
checks quickly).  Prints one JSON line of max relative errors vs the oracle."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
import paper_2101_07249_b200 as W  # noqa: E402
from gpu_helpers import factor, pair, relerr  # noqa: E402


def case(model, net, n, sigma_o=0.1, m=5):
    bh = factor(O.build_soar(1.0, 3.0, n))
    qh = factor(O.build_soar(0.3, 3.0, n))
    g, o = pair(model, net, bh, qh, sigma_o)
    V = O.gaussian_matrix(g.dim(), m, 3)
    out = {"apply": relerr(g.apply_block(V), o.apply_block(V))}
    for name in ("apply_Linv", "apply_LinvT"):
        out[name] = relerr(getattr(g, name)(V), np.column_stack([getattr(o, name)(V[:, j]) for j in range(m)]))
    return out


def main():
    res = {}
    n = 300
    res["advdiff_s3"] = case(W.AdvDiffLinearized(n, 6, 0.5, 0.2, 3), W.ObservationNetwork.build(n, 6, 4, 1), n)
    res["advection_s1"] = case(W.AdvectionLinearized(n, 9, 0.8), W.ObservationNetwork.build(n, 9, 5, 3), n)
    res["identity"] = case(W.IdentityLinearized(n, 4), W.ObservationNetwork.build(n, 4, 7, 2), n)
    # Lorenz-96: the reference's own single-step linearisation and the s = 5 extension
    for s in (1, 5):
        N, dt = 6, 0.025
        x0 = 8.0 + O.NormalStream(3).draw(n)
        traj = W.lorenz96_trajectory(x0, 8.0, dt, 50, N * s)
        res[f"l96_s{s}"] = case(W.Lorenz96Linearized(traj, 8.0, dt, s), W.ObservationNetwork.build(n, N, 2, 1), n,
                                sigma_o=0.2)
    # a domain wider than one register-blocked region (WC4DVAR_L96_BLK=1 engages it)
    nb, N, s, dt = 1500, 4, 5, 0.025
    traj = W.lorenz96_trajectory(8.0 + O.NormalStream(5).draw(nb), 8.0, dt, 20, N * s)
    res["l96_n1500"] = case(W.Lorenz96Linearized(traj, 8.0, dt, s), W.ObservationNetwork.build(nb, N, 3, 2), nb,
                            sigma_o=0.2, m=6)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
