"""Shared helpers for the GPU parity tests: build the oracle twin of a product operator."""
import numpy as np

from oracle import oracle as O
import paper_2101_07249_b200 as W


def oracle_model(m: W.LinearizedModel) -> O.LinearizedModel:
    if m.kind == "l96" and m.stages is None:  # stages built on the device from the trajectory
        tr = m.trajectory
        tr = tr if isinstance(tr, np.ndarray) else tr.cpu().numpy().T
        return O.Lorenz96Linearized(tr, m.forcing, m.dt, m.substeps)
    return O.LinearizedModel(m.kind, m.n, m.N, m.substeps, m.courant, m.diffusion, m.dt, m.stages)


def oracle_net(net: W.ObservationNetwork) -> O.ObservationNetwork:
    return O.ObservationNetwork(net.n, net.N, net.space_stride, net.time_stride, list(net.times),
                                list(net.points), net.q)


def oracle_factor(f: W.CovarianceFactor) -> O.CovarianceFactor:
    return O.CovarianceFactor(np.asarray(f.half), np.asarray(f.half_inv), f.kind)


def pair(model, net, bh, qh, sigma_o, threads=8):
    """(gpu_op, oracle_op) for the same operator description (product-side descriptors)."""
    g = W.HessianOperator(model, net, bh, qh, sigma_o)
    o = O.HessianOperator(oracle_model(model), oracle_net(net), oracle_factor(bh), oracle_factor(qh),
                          sigma_o, threads=threads)
    return g, o


def workload_pair(wl, threads=8):
    return pair(wl.model, wl.net, wl.b_half, wl.q_half, wl.sigma_obs, threads)


def factor(C):
    f = O.sym_sqrt(C)
    return W.CovarianceFactor(f.half, f.half_inv)


def identity_factor(n):
    return W.CovarianceFactor(np.eye(n, order="F"), np.eye(n, order="F"))


def relerr(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / max(np.abs(np.asarray(b)).max(), 1e-300))
