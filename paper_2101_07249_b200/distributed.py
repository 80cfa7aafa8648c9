"""Multi-GPU orchestration of the randomized-LMP path.

One process per GPU, torch.distributed for the plumbing (NCCL on GPU ranks, gloo on the
CPU test ranks).  The data layout follows the path's natural sharding:

* A*Omega shards by sketch COLUMNS with no communication (`column_range`): each rank
  applies the Hessian to its own columns (bench.py, weak scaling);
* the tall-skinny algebra (CholQR2, Rayleigh-Ritz, Nystrom) works on ROW shards: an
  all-to-all transposes column shards into row shards (`cols_to_rows` / `rows_to_cols`),
  Gram matrices are summed with one all-reduce of m x m, the small factorizations are
  replicated on every rank;
* PCG shards by rows with all-reduced dot products (`dist_pcg`).

Local dense work goes through a `LocalOps` backend: `TorchOps` (torch tensors; used by the
gloo CPU tests and as a reference) or the device library on GPU ranks.  The operator
apply is a callback so each rank can use its own `HessianOperator` handle.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import torch
import torch.distributed as dist


def column_range(m: int, world: int, rank: int):
    """Balanced contiguous column shard [start, stop) of m sketch columns."""
    base, extra = divmod(m, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def row_range(n: int, world: int, rank: int):
    return column_range(n, world, rank)


class TorchOps:
    """Local dense kernels on torch tensors (float64)."""

    @staticmethod
    def gram(A, B):
        return A.T @ B

    @staticmethod
    def tall_times_small(A, W):
        return A @ W

    @staticmethod
    def chol_upper(G):
        G = 0.5 * (G + G.T)
        L, info = torch.linalg.cholesky_ex(G)
        if int(info) != 0:
            raise RuntimeError(f"cholqr: Gram matrix not positive definite (pivot {int(info)})")
        return L.T

    @staticmethod
    def eigh_desc(K):
        w, V = torch.linalg.eigh(0.5 * (K + K.T))
        return torch.flip(w, [0]), torch.flip(V, [1])


def allreduce_sum(t: torch.Tensor) -> torch.Tensor:
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return t


def all_gather_cat(t: torch.Tensor, sizes: List[int], dim: int = 0) -> torch.Tensor:
    """All-gather shards of unequal length along `dim` (padded to the largest, then trimmed;
    gloo requires equal sizes) and concatenate them in rank order."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return t
    mx = max(sizes)
    pad_shape = list(t.shape)
    pad_shape[dim] = mx
    padded = torch.zeros(pad_shape, dtype=t.dtype, device=t.device)
    padded.narrow(dim, 0, t.shape[dim]).copy_(t)
    outs = [torch.empty_like(padded) for _ in sizes]
    dist.all_gather(outs, padded)
    return torch.cat([o.narrow(dim, 0, s) for o, s in zip(outs, sizes)], dim=dim)


def _alltoall(recv: List[torch.Tensor], send: List[torch.Tensor]) -> None:
    """Grouped point-to-point all-to-all (ncclSend/ncclRecv under NCCL; gloo has no
    alltoall collective, so the same grouped P2P form serves the CPU tests)."""
    rank = dist.get_rank()
    ops = []
    for r, (rv, sd) in enumerate(zip(recv, send)):
        if r == rank:
            rv.copy_(sd)
            continue
        ops.append(dist.P2POp(dist.isend, sd, r))
        ops.append(dist.P2POp(dist.irecv, rv, r))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def cols_to_rows(Y_cols: torch.Tensor, n: int, m: int) -> torch.Tensor:
    """All-to-all transpose: this rank holds all n rows of its column shard; return all m
    columns of its row shard.  Y_cols: (n, m_local) -> (n_local, m)."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    if world == 1:
        return Y_cols
    send = []
    for r in range(world):
        a, b = row_range(n, world, r)
        send.append(Y_cols[a:b, :].contiguous())
    recv = []
    ra, rb = row_range(n, world, rank)
    for r in range(world):
        ca, cb = column_range(m, world, r)
        recv.append(torch.empty((rb - ra, cb - ca), dtype=Y_cols.dtype, device=Y_cols.device))
    _alltoall(recv, send)
    return torch.cat(recv, dim=1)


def rows_to_cols(Y_rows: torch.Tensor, n: int, m: int) -> torch.Tensor:
    """Inverse of cols_to_rows: (n_local, m) -> (n, m_local)."""
    world = dist.get_world_size() if dist.is_initialized() else 1
    rank = dist.get_rank() if dist.is_initialized() else 0
    if world == 1:
        return Y_rows
    send = []
    for r in range(world):
        a, b = column_range(m, world, r)
        send.append(Y_rows[:, a:b].contiguous())
    ca, cb = column_range(m, world, rank)
    recv = []
    for r in range(world):
        a, b = row_range(n, world, r)
        recv.append(torch.empty((b - a, cb - ca), dtype=Y_rows.dtype, device=Y_rows.device))
    _alltoall(recv, send)
    return torch.cat(recv, dim=0)


def dist_cholqr2(Y_rows: torch.Tensor, ops=TorchOps):
    """Row-partitioned CholQR2: Gram all-reduce (m x m), replicated Cholesky, local Y R^{-1}.
    Returns (Q_rows, R) with Y = Q R."""
    G = allreduce_sum(ops.gram(Y_rows, Y_rows).contiguous())
    R1 = ops.chol_upper(G)
    Q1 = torch.linalg.solve_triangular(R1, Y_rows, upper=True, left=False)
    G2 = allreduce_sum(ops.gram(Q1, Q1).contiguous())
    R2 = ops.chol_upper(G2)
    Q = torch.linalg.solve_triangular(R2, Q1, upper=True, left=False)
    return Q, R2 @ R1


def dist_revd(apply_cols: Callable[[torch.Tensor], torch.Tensor], omega_cols: torch.Tensor, n: int,
              m: int, k: int, ops=TorchOps):
    """Distributed REVD (randevd.cpp:62-80): column-sharded applies, row-sharded CholQR2 and
    Rayleigh-Ritz (randevd.cpp:47-60).  Returns (U_rows, theta) with U row-sharded."""
    Y_rows = cols_to_rows(apply_cols(omega_cols), n, m)
    Z_rows, _ = dist_cholqr2(Y_rows, ops)
    AZ_rows = cols_to_rows(apply_cols(rows_to_cols(Z_rows, n, m)), n, m)
    K = allreduce_sum(ops.gram(Z_rows, AZ_rows).contiguous())
    vals, W = ops.eigh_desc(K)
    return ops.tall_times_small(Z_rows, W[:, :k]), vals[:k]


@dataclass
class DistPcgResult:
    x_rows: torch.Tensor
    residual_norms: List[float] = field(default_factory=list)
    iterations: int = 0
    converged: bool = False


def dist_pcg(apply_rows: Callable[[torch.Tensor], torch.Tensor], b_rows: torch.Tensor,
             U_rows: Optional[torch.Tensor], theta: Optional[torch.Tensor], max_iter: int = 100,
             rel_tol: float = 1e-6) -> DistPcgResult:
    """Row-sharded split PCG (krylov.cpp:22-99) with the compact-WY spectral LMP: every dot
    product and every U^T v is one all-reduce of (k + 1) doubles."""
    k = 0 if U_rows is None else U_rows.shape[1]
    if k:
        c = 1.0 - 1.0 / torch.sqrt(theta)
        S = allreduce_sum((U_rows.T @ U_rows).contiguous())
        T = torch.zeros((k, k), dtype=b_rows.dtype, device=b_rows.device)
        for i in range(k):  # compact-WY recurrence (lmp_pcg.cuh)
            T[i, i] = c[i]
            if i:
                T[:i, i] = -c[i] * (T[:i, :i] @ S[:i, i])

    def utv_dot(v, a=None):
        parts = [U_rows.T @ v] if k else []
        parts.append((a @ v).reshape(1) if a is not None else torch.zeros(1, dtype=v.dtype, device=v.device))
        red = allreduce_sum(torch.cat(parts).contiguous())
        return red[:k], red[k]

    def C(v, g):      # C v = v - U T (U^T v)
        return v - U_rows @ (T @ g) if k else v.clone()

    def Ct(v, g):     # C^T v = v - U T^T (U^T v)
        return v - U_rows @ (T.T @ g) if k else v.clone()

    x = torch.zeros_like(b_rows)
    g, _ = utv_dot(b_rows)
    r = Ct(b_rows, g)
    h, rho = utv_dot(r, r)
    p = C(r, h)
    r0 = math.sqrt(float(rho))
    res = DistPcgResult(x, [r0])
    if r0 == 0.0:
        res.converged = True
        return res
    rho = float(rho)
    for j in range(1, max_iter + 1):
        w = apply_rows(p)
        g, curv = utv_dot(w, p)
        curv = float(curv)
        if not math.isfinite(curv) or curv <= 0.0:
            raise RuntimeError(f"pcg_split: p^T A p = {curv} at iteration {j}")
        alpha = rho / curv
        x = x + alpha * p
        r = r - alpha * Ct(w, g)
        h, rn = utv_dot(r, r)
        rn = float(rn)
        beta = rn / rho
        res.residual_norms.append(math.sqrt(rn))
        res.iterations = j
        if math.sqrt(rn) / r0 <= rel_tol:
            res.converged = True
            break
        p = C(r, h) + beta * p
        rho = rn
    res.x_rows = x
    return res
