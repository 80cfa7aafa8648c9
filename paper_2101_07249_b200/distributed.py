"""Multi-GPU orchestration of the randomized-LMP path.

One process per GPU, torch.distributed for the plumbing (NCCL on GPU ranks, gloo on the
CPU test ranks).  The data layout follows the path's natural sharding:

* A*Omega shards by sketch COLUMNS with no communication (`column_range`): each rank
  applies the Hessian to its own columns (bench.py, weak scaling);
* the tall-skinny algebra of REVD, Nystrom and ritzit (randevd.cpp:47-136) works on ROW
  shards: an all-to-all transposes column shards into row shards (`cols_to_rows` /
  `rows_to_cols`), every Gram-type product is a local partial plus one all-reduce of an
  m x m matrix, and the small factorizations (Cholesky, pivoted rank probe, EVD, SVD) are
  replicated on every rank;
* PCG shards by rows with all-reduced dot products (`dist_pcg`).

Local dense work goes through an ops backend:

* `DeviceOps` -- the library's own kernels (C-ABI "row-sharded building blocks",
  include/wc4dvar_gpu.h) on the rank's GPU, on torch's current stream.  With one rank the
  distributed methods run exactly the kernel sequence of `wc4dvar_gpu_sketch`.
* `TorchOps` -- the same steps on torch tensors (float64), used by the gloo CPU tests.

Tall matrices are torch tensors of shape (rows, cols) in COLUMN-major storage (strides
(1, rows)), the layout of the C-ABI and of Eigen.  The operator apply is a callback so
each rank can use its own `HessianOperator` handle (`hessian_apply_cols`).
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import Callable, List, Optional

import torch
import torch.distributed as dist

from .wc4dvar import NumericalError

_EPS = 2.220446049250313e-16


# ----------------------------------------------------------------------------- layout
def fmat(rows: int, cols: int, like: torch.Tensor) -> torch.Tensor:
    """Uninitialised column-major (rows x cols) tensor on like's device."""
    return torch.empty((cols, rows), dtype=torch.float64, device=like.device).T


def fcontig(t: torch.Tensor) -> torch.Tensor:
    """Column-major contiguous copy of a 2-D tensor (no copy when it already is)."""
    if t.dim() == 1:
        t = t.reshape(-1, 1)
    rows, cols = t.shape
    if t.stride(0) == 1 and t.stride(1) == rows:
        return t
    if t.stride(0) == 1 and cols == 1:  # one dense column: restate its leading dimension
        return t.as_strided((rows, 1), (1, max(rows, 1)))
    return t.T.contiguous().T


def column_range(m: int, world: int, rank: int):
    """Balanced contiguous column shard [start, stop) of m sketch columns."""
    base, extra = divmod(m, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def row_range(n: int, world: int, rank: int):
    return column_range(n, world, rank)


def _world_rank():
    if dist.is_available() and dist.is_initialized():
        return dist.get_world_size(), dist.get_rank()
    return 1, 0


# ----------------------------------------------------------------------------- backends
class TorchOps:
    """Local dense steps on torch tensors (float64); same contracts as DeviceOps."""

    @staticmethod
    def gram(A, B):
        return fcontig(A.T @ B)

    @staticmethod
    def tall_times_small(A, W):
        return fcontig(A @ W)

    @staticmethod
    def chol_upper(G, what="cholqr"):
        G = 0.5 * (G + G.T)
        L, info = torch.linalg.cholesky_ex(G)
        if int(info) != 0:
            raise NumericalError(f"{what}: matrix is not positive definite (pivot {int(info) - 1})")
        return fcontig(L.T)

    @staticmethod
    def tri_inv_upper(R):
        eye = torch.eye(R.shape[0], dtype=R.dtype, device=R.device)
        return fcontig(torch.linalg.solve_triangular(R, eye, upper=True))

    @staticmethod
    def chol_inv(G, what="cholqr"):
        R = TorchOps.chol_upper(G, what)
        return R, TorchOps.tri_inv_upper(R)

    @staticmethod
    def small_mm(A, B, ta=False, tb=False):
        return fcontig((A.T if ta else A) @ (B.T if tb else B))

    @staticmethod
    def pivoted_rank(G, tol_rel):
        """Diagonally pivoted Cholesky rank probe (the device rule of smallla.cu)."""
        A = (0.5 * (G + G.T)).clone()
        m = A.shape[0]
        perm = list(range(m))
        tol = tol_rel * float(torch.diagonal(A).max()) if m else 0.0
        for j in range(m):
            d = torch.diagonal(A)[j:]
            p = j + int(torch.argmax(d))
            best = float(A[p, p])
            if not (best > tol) or not math.isfinite(best):
                return j, torch.tensor(perm, dtype=torch.int32, device=G.device)
            if p != j:
                perm[j], perm[p] = perm[p], perm[j]
                A[[j, p], :] = A[[p, j], :]
                A[:, [j, p]] = A[:, [p, j]]
            A[j, j] = math.sqrt(A[j, j])
            A[j, j + 1:] /= A[j, j]
            A[j + 1:, j + 1:] -= torch.outer(A[j, j + 1:], A[j, j + 1:])
        return m, torch.tensor(perm, dtype=torch.int32, device=G.device)

    @staticmethod
    def eigh_desc(K):
        w, V = torch.linalg.eigh(0.5 * (K + K.T))
        return torch.flip(w, [0]).contiguous(), fcontig(torch.flip(V, [1]))

    @staticmethod
    def svd_left(X):
        U, s, _ = torch.linalg.svd(X)
        return s.contiguous(), fcontig(U)

    @staticmethod
    def gather_cols(Y, perm, r):
        return fcontig(Y[:, perm[:r].long()])


class DeviceOps:
    """The library's kernels on this rank's GPU (include/wc4dvar_gpu.h, row-sharded
    building blocks), issued on torch's current stream."""

    def __init__(self, device: Optional[int] = None):
        from . import wc4dvar as _w
        self._w = _w
        self.device = torch.cuda.current_device() if device is None else int(device)

    def _st(self):
        return ctypes.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def _call(self, name, *args):
        self._w._check(getattr(self._w.lib, name)(self.device, *args, self._st()))

    def gram(self, A, B):
        A, B = fcontig(A), fcontig(B)
        G = fmat(A.shape[1], B.shape[1], A)
        self._call("wc4dvar_gpu_la_gram_dev", A.shape[0], A.shape[1], B.shape[1], A.data_ptr(),
                   max(A.stride(1), A.shape[0], 1), B.data_ptr(), max(B.stride(1), B.shape[0], 1),
                   G.data_ptr(), max(A.shape[1], 1))
        return G

    def tall_times_small(self, A, W):
        A, W = fcontig(A), fcontig(W)
        C = fmat(A.shape[0], W.shape[1], A)
        self._call("wc4dvar_gpu_la_tall_times_small_dev", A.shape[0], A.shape[1], W.shape[1],
                   A.data_ptr(), max(A.shape[0], 1), W.data_ptr(), W.shape[0], C.data_ptr(),
                   max(A.shape[0], 1))
        return C

    def chol_upper(self, G, what="cholqr"):
        G = fcontig(G)
        R = fmat(G.shape[0], G.shape[0], G)
        try:
            self._call("wc4dvar_gpu_la_chol_upper_dev", G.shape[0], G.data_ptr(), R.data_ptr())
        except NumericalError as e:
            raise NumericalError(f"{what}: {e}") from None
        return R

    def chol_inv(self, G, what="cholqr"):
        G = fcontig(G)
        R, Ri = fmat(G.shape[0], G.shape[0], G), fmat(G.shape[0], G.shape[0], G)
        try:
            self._call("wc4dvar_gpu_la_chol_inv_upper_dev", G.shape[0], G.data_ptr(), R.data_ptr(),
                       Ri.data_ptr())
        except NumericalError as e:
            raise NumericalError(f"{what}: {e}") from None
        return R, Ri

    def tri_inv_upper(self, R):
        R = fcontig(R)
        Ri = fmat(R.shape[0], R.shape[0], R)
        self._call("wc4dvar_gpu_la_tri_inv_upper_dev", R.shape[0], R.data_ptr(), Ri.data_ptr())
        return Ri

    def small_mm(self, A, B, ta=False, tb=False):
        A, B = fcontig(A), fcontig(B)
        M = A.shape[1] if ta else A.shape[0]
        K = A.shape[0] if ta else A.shape[1]
        N = B.shape[0] if tb else B.shape[1]
        C = fmat(M, N, A)
        self._call("wc4dvar_gpu_la_small_gemm_dev", int(ta), int(tb), M, N, K, 1.0, A.data_ptr(),
                   A.shape[0], B.data_ptr(), B.shape[0], 0.0, C.data_ptr(), M)
        return C

    def pivoted_rank(self, G, tol_rel):
        G = fcontig(G)
        m = G.shape[0]
        perm = torch.empty(m, dtype=torch.int32, device=G.device)
        r = ctypes.c_int64(0)
        self._call("wc4dvar_gpu_la_pivoted_rank_dev", m, G.data_ptr(), float(tol_rel), ctypes.byref(r),
                   perm.data_ptr())
        return int(r.value), perm

    def eigh_desc(self, K):
        K = fcontig(K)
        m = K.shape[0]
        vals = torch.empty(m, dtype=torch.float64, device=K.device)
        W = fmat(m, m, K)
        self._call("wc4dvar_gpu_la_sym_evd_dev", m, K.data_ptr(), vals.data_ptr(), W.data_ptr())
        return vals, W

    def svd_left(self, X):
        X = fcontig(X)
        m = X.shape[0]
        s = torch.empty(m, dtype=torch.float64, device=X.device)
        U = fmat(m, m, X)
        self._call("wc4dvar_gpu_la_svd_left_dev", m, X.data_ptr(), s.data_ptr(), U.data_ptr())
        return s, U

    def gather_cols(self, Y, perm, r):
        Y = fcontig(Y)
        out = fmat(Y.shape[0], r, Y)
        self._call("wc4dvar_gpu_la_gather_cols_dev", Y.shape[0], r, Y.data_ptr(), max(Y.shape[0], 1),
                   perm.data_ptr(), out.data_ptr(), max(Y.shape[0], 1))
        return out


def hessian_apply_cols(op) -> Callable[[torch.Tensor], torch.Tensor]:
    """Column-block apply of a device operator handle on column-major CUDA tensors
    (wc4dvar_gpu_op_apply_block_dev on torch's current stream; counts m applies)."""

    def apply(X: torch.Tensor) -> torch.Tensor:
        X = fcontig(X)
        out = fmat(X.shape[0], X.shape[1], X)
        if X.shape[1]:
            op.apply_block_dev(X.T, out.T, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        return out

    return apply


# ----------------------------------------------------------------------------- collectives
def allreduce_sum(t: torch.Tensor) -> torch.Tensor:
    world, _ = _world_rank()
    if world > 1:
        t = t.contiguous() if t.dim() == 1 else fcontig(t)
        flat = t.T if t.dim() == 2 else t  # row-major view of the same bytes
        dist.all_reduce(flat, op=dist.ReduceOp.SUM)
    return t


def all_gather_cat(t: torch.Tensor, sizes: List[int], dim: int = 0) -> torch.Tensor:
    """All-gather shards of unequal length along `dim` (padded to the largest, then trimmed;
    gloo requires equal sizes) and concatenate them in rank order."""
    world, _ = _world_rank()
    if world == 1:
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
        if sd.numel():
            ops.append(dist.P2POp(dist.isend, sd, r))
        if rv.numel():
            ops.append(dist.P2POp(dist.irecv, rv, r))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()


def cols_to_rows(Y_cols: torch.Tensor, n: int, m: int) -> torch.Tensor:
    """All-to-all transpose: this rank holds all n rows of its column shard; return all m
    columns of its row shard.  Y_cols: (n, m_local) -> (n_local, m), column-major.
    Messages travel as the row-major (cols, rows) image of each column-major block."""
    world, rank = _world_rank()
    if world == 1:
        return fcontig(Y_cols)
    send = []
    for r in range(world):
        a, b = row_range(n, world, r)
        send.append(Y_cols[a:b, :].T.contiguous())
    ra, rb = row_range(n, world, rank)
    recv = []
    for r in range(world):
        ca, cb = column_range(m, world, r)
        recv.append(torch.empty((cb - ca, rb - ra), dtype=Y_cols.dtype, device=Y_cols.device))
    _alltoall(recv, send)
    return torch.cat(recv, dim=0).T


def rows_to_cols(Y_rows: torch.Tensor, n: int, m: int) -> torch.Tensor:
    """Inverse of cols_to_rows: (n_local, m) -> (n, m_local), column-major."""
    world, rank = _world_rank()
    if world == 1:
        return fcontig(Y_rows)
    send = []
    for r in range(world):
        a, b = column_range(m, world, r)
        send.append(Y_rows[:, a:b].T.contiguous())
    ca, cb = column_range(m, world, rank)
    recv = []
    for r in range(world):
        a, b = row_range(n, world, r)
        recv.append(torch.empty((cb - ca, b - a), dtype=Y_rows.dtype, device=Y_rows.device))
    _alltoall(recv, send)
    return torch.cat(recv, dim=1).T


# ----------------------------------------------------------------------------- sketches
def dist_cholqr2(Y_rows: torch.Tensor, ops=TorchOps, G0: Optional[torch.Tensor] = None,
                 want_r: bool = False, what: str = "cholqr"):
    """Row-partitioned CholQR2 (replaces householder_q, randevd.cpp:27-30): Gram all-reduce
    (m x m), replicated Cholesky and triangular inverse, local Y R^{-1}; twice.  G0 is an
    already all-reduced Y^T Y.  Returns Q_rows, and R with Y = Q R when want_r."""
    G = G0 if G0 is not None else allreduce_sum(ops.gram(Y_rows, Y_rows))
    R1, R1i = ops.chol_inv(G, what)
    Q1 = ops.tall_times_small(Y_rows, R1i)
    # sketch.cu cholqr2: when a pass is expensive (2 n m^2 >= 1e11 over all ranks) and cond(Y) <= 4
    # (singular values of the replicated R1), the first pass is as orthonormal as Householder QR
    m = Y_rows.shape[1]
    if os.environ.get("WC4DVAR_CHOLQR_ADAPT", "1") != "0":
        n_glob = allreduce_sum(torch.tensor([float(Y_rows.shape[0])], dtype=torch.float64,
                                            device=Y_rows.device))
        if 2.0 * float(n_glob.item()) * m * m >= 1e11:
            sig, _ = ops.svd_left(R1)
            if float(sig[-1]) > 0.0 and float(sig[0]) <= 4.0 * float(sig[-1]):
                return (Q1, R1) if want_r else Q1
    G2 = allreduce_sum(ops.gram(Q1, Q1))
    R2, R2i = ops.chol_inv(G2, what)
    Q = ops.tall_times_small(Q1, R2i)
    return (Q, ops.small_mm(R2, R1)) if want_r else Q


def _rank_tol(n: int) -> float:
    return 32.0 * math.sqrt(n) * _EPS  # sketch.cu rank_probe


def _apply_rows(apply_cols, Z_rows, n, m):
    """A Z for row-sharded Z: rows -> cols, column-sharded apply, cols -> rows."""
    return cols_to_rows(apply_cols(rows_to_cols(Z_rows, n, m)), n, m)


def dist_rayleigh_ritz(apply_cols, Z_rows, n: int, keep: int, ops=TorchOps):
    """rayleigh_ritz (randevd.cpp:47-60) on a row-sharded orthonormal Z."""
    m = Z_rows.shape[1]
    G = allreduce_sum(ops.gram(Z_rows, Z_rows))
    eye = torch.eye(m, dtype=G.dtype, device=G.device)
    if float((G - eye).abs().max()) > 1e-8:
        raise NumericalError("rayleigh_ritz: Z is not orthonormal")
    AZ_rows = _apply_rows(apply_cols, Z_rows, n, m)
    K = allreduce_sum(ops.gram(Z_rows, AZ_rows))
    vals, W = ops.eigh_desc(K)
    return ops.tall_times_small(Z_rows, W[:, :keep]), vals[:keep].clone()


def dist_revd(apply_cols: Callable[[torch.Tensor], torch.Tensor], omega_cols: torch.Tensor, n: int,
              m: int, k: int, ops=TorchOps):
    """Distributed REVD (randevd.cpp:62-80): column-sharded applies, row-sharded rank probe,
    CholQR2 and Rayleigh-Ritz.  Transposes: 3.  Returns (U_rows, theta), U row-sharded."""
    Y_rows = cols_to_rows(apply_cols(omega_cols), n, m)
    G = allreduce_sum(ops.gram(Y_rows, Y_rows))
    r, _ = ops.pivoted_rank(G, _rank_tol(n))
    if r < m:
        raise NumericalError(f"revd: sample matrix rank collapsed to {r} of {m} columns")
    Z_rows = dist_cholqr2(Y_rows, ops, G0=G,
                          what="revd: sample matrix is numerically rank deficient (CholQR breakdown)")
    return dist_rayleigh_ritz(apply_cols, Z_rows, n, k, ops)


def dist_nystrom(apply_cols, omega_cols: torch.Tensor, n: int, m: int, k: int, ops=TorchOps):
    """Distributed Nystrom (randevd.cpp:82-114): pivoted rank probe on the all-reduced Gram,
    CholQR2 of the kept columns, E1 = A Z, E2 = Z^T E1 (all-reduced), Cholesky,
    F = E1 U^{-1}, CholQR2(F) and the replicated SVD of R_F.  Transposes: 3."""
    Y_rows = cols_to_rows(apply_cols(omega_cols), n, m)
    G = allreduce_sum(ops.gram(Y_rows, Y_rows))
    r, perm = ops.pivoted_rank(G, _rank_tol(n))
    if r == 0:
        raise NumericalError("nystrom: sample matrix is zero")
    what = "nystrom: sample matrix is numerically rank deficient (CholQR breakdown)"
    if r < m:
        Z_rows = dist_cholqr2(ops.gather_cols(Y_rows, perm, r), ops, what=what)
    else:
        Z_rows = dist_cholqr2(Y_rows, ops, G0=G, what=what)
    E1_rows = _apply_rows(apply_cols, Z_rows, n, r)
    E2 = allreduce_sum(ops.gram(Z_rows, E1_rows))
    _, Rui = ops.chol_inv(E2, "nystrom: Cholesky of Z^T A Z failed; the projected operator is "
                              "numerically indefinite. Increase the oversampling parameter or use "
                              "revd for indefinite spectra.")
    F_rows = ops.tall_times_small(E1_rows, Rui)
    QF_rows, RF = dist_cholqr2(F_rows, ops, want_r=True,
                               what="nystrom: factor F is numerically rank deficient (CholQR breakdown)")
    sig, W = ops.svd_left(RF)
    keep = min(k, r)
    return ops.tall_times_small(QF_rows, W[:, :keep]), (sig[:keep] * sig[:keep]).clone()


def dist_ritzit(apply_cols, omega_rows: torch.Tensor, n: int, m: int, k: int, ops=TorchOps,
                p_iter: int = 1):
    """Distributed ritzit (randevd.cpp:116-136; p_iter > 1 is the BASELINE extension): the
    sample is ROW-sharded from the start (QR(Omega) needs rows), so only 2 transposes per
    apply.  Returns (U_rows, theta)."""
    G3 = dist_cholqr2(omega_rows, ops, what="revd_ritzit: Gaussian sample is numerically rank deficient")
    Y3 = _apply_rows(apply_cols, G3, n, m)
    for _ in range(max(p_iter, 1) - 1):
        G3 = dist_cholqr2(Y3, ops, what="revd_ritzit: QR of the sample matrix is rank deficient")
        Y3 = _apply_rows(apply_cols, G3, n, m)
    Z3, R3 = dist_cholqr2(Y3, ops, want_r=True, what="revd_ritzit: QR of the sample matrix is rank deficient")
    d = torch.diagonal(R3).abs()
    if float(d.min()) <= 1e-14 * float(d.max()):
        raise NumericalError("revd_ritzit: QR of the sample matrix is rank deficient")
    vals, W = ops.eigh_desc(ops.small_mm(R3, R3, tb=True))
    if float(vals[min(k, m) - 1]) <= 0.0:
        raise NumericalError("revd_ritzit: nonpositive squared Ritz value")
    return ops.tall_times_small(Z3, W[:, :k]), torch.sqrt(vals[:k])


# ----------------------------------------------------------------------------- PCG
@dataclass
class DistPcgResult:
    x_rows: torch.Tensor
    residual_norms: List[float] = field(default_factory=list)
    iterations: int = 0
    converged: bool = False


def dist_pcg(apply_rows: Callable[[torch.Tensor], torch.Tensor], b_rows: torch.Tensor,
             U_rows: Optional[torch.Tensor], theta: Optional[torch.Tensor], max_iter: int = 100,
             rel_tol: float = 1e-6, ops=TorchOps, comm=None, check_every: int = 8) -> DistPcgResult:
    """Row-sharded split PCG (krylov.cpp:22-99) with the compact-WY spectral LMP: every dot
    product and every U^T v of an iteration is one all-reduce of (k + 1) doubles.  Any row
    partition works (contiguous rows, or the spatial slabs of RowShardedHessian) as long as
    b, U and apply_rows use the same one.

    The loop keeps alpha / beta / rho, the stop test and the curvature check on the device
    (no host round trip per iteration): the host looks at the device flags every
    `check_every` iterations.  Iterations issued after the one that converged (or failed)
    run masked -- alpha is zeroed, r and rho are frozen -- so x, the residual history and the
    iteration count are exactly those of the per-iteration loop (krylov.cpp:92-95)."""
    allreduce_sum = comm.allreduce_sum if comm is not None else globals()["allreduce_sum"]
    k = 0 if U_rows is None else U_rows.shape[1]
    if k:
        c = 1.0 - 1.0 / torch.sqrt(theta)
        S = allreduce_sum(ops.gram(U_rows, U_rows))
        T = torch.zeros((k, k), dtype=b_rows.dtype, device=b_rows.device)
        for i in range(k):  # compact-WY recurrence (lmp_pcg.cuh)
            T[i, i] = c[i]
            if i:
                T[:i, i] = -c[i] * (T[:i, :i] @ S[:i, i])

    def utv_dot(v, a=None):
        parts = [ops.gram(U_rows, v.reshape(-1, 1)).reshape(-1)] if k else []
        parts.append((a @ v).reshape(1) if a is not None else torch.zeros(1, dtype=v.dtype, device=v.device))
        red = allreduce_sum(torch.cat(parts).contiguous())
        return red[:k], red[k]

    def C(v, g):      # C v = v - U T (U^T v)
        return v - ops.tall_times_small(U_rows, (T @ g).reshape(-1, 1)).reshape(-1) if k else v.clone()

    def Ct(v, g):     # C^T v = v - U T^T (U^T v)
        return v - ops.tall_times_small(U_rows, (T.T @ g).reshape(-1, 1)).reshape(-1) if k else v.clone()

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
    dev, dt = b_rows.device, b_rows.dtype
    zero = torch.zeros((), dtype=dt, device=dev)
    done = torch.zeros((), dtype=torch.bool, device=dev)      # converged or failed
    conv = torch.zeros((), dtype=torch.bool, device=dev)
    fail_at = torch.zeros((), dtype=torch.int64, device=dev)  # first iteration with curv <= 0
    curv_bad = torch.zeros((), dtype=dt, device=dev)
    hist = []
    check_every = max(1, int(check_every))
    j_issued = 0
    for j in range(1, max_iter + 1):
        w = apply_rows(p)
        g, curv = utv_dot(w, p)
        active = ~done
        bad = active & (~torch.isfinite(curv) | (curv <= 0.0))
        fail_at = torch.where(bad, torch.full_like(fail_at, j), fail_at)
        curv_bad = torch.where(bad, curv, curv_bad)
        done = done | bad
        live = ~done
        alpha = torch.where(live, rho / curv, zero)
        x = x + alpha * p
        r = r - alpha * Ct(w, g)
        h, rn = utv_dot(r, r)
        rn = torch.where(live, rn, rho)
        beta = rn / rho
        hist.append(torch.where(live, torch.sqrt(rn), zero))
        now = live & (torch.sqrt(rn) / r0 <= rel_tol)
        conv = conv | now
        done = done | now
        p = C(r, h) + beta * p
        rho = rn
        j_issued = j
        if j % check_every == 0 or j == max_iter:
            if bool(done):  # the one host sync per `check_every` iterations
                break
    fj = int(fail_at)
    if fj:
        cv = float(curv_bad)
        raise NumericalError(f"pcg_split: p^T A p = {cv} at iteration {fj}")
    hv = torch.stack(hist).cpu().tolist() if hist else []
    nlive = j_issued
    if bool(conv):
        nlive = next(i for i, v in enumerate(hv, 1) if v / r0 <= rel_tol)
    res.residual_norms += hv[:nlive]
    res.iterations = nlive
    res.converged = bool(conv)
    res.x_rows = x
    return res


# ----------------------------------------------------------------------------- row-sharded apply
class TorchComm:
    """torch.distributed (NCCL on GPU ranks, gloo on CPU ranks) for the row-sharded apply."""

    def world_rank(self):
        return _world_rank()

    def alltoall(self, recv: List[torch.Tensor], send: List[torch.Tensor]) -> None:
        world, rank = _world_rank()
        if world == 1:
            recv[0].copy_(send[0])
            return
        _alltoall(recv, send)

    def allreduce_sum(self, t: torch.Tensor) -> torch.Tensor:
        return allreduce_sum(t)


class ThreadComm:
    """In-process ranks (one host thread each) sharing one device: the same collectives as
    TorchComm through a barrier and a mailbox, deterministic rank order.  Used to run the
    multi-rank device path on a single GPU (no kernel waits on another rank's kernel: each
    exchange completes on the host between launches)."""

    def __init__(self, world: int):
        import threading
        self.world = world
        self._bar = threading.Barrier(world)
        self._box = {}

    def bind(self, rank: int) -> "ThreadComm._Rank":
        return ThreadComm._Rank(self, rank)

    class _Rank:
        def __init__(self, hub, rank):
            self.hub, self.rank = hub, rank

        def world_rank(self):
            return self.hub.world, self.rank

        def alltoall(self, recv, send):
            h = self.hub
            for q, sd in enumerate(send):
                h._box[(self.rank, q)] = sd.clone() if sd.numel() else sd
            if any(sd.is_cuda for sd in send):
                torch.cuda.synchronize()
            h._bar.wait()
            for q, rv in enumerate(recv):
                if rv.numel():
                    rv.copy_(h._box[(q, self.rank)])
            if recv and recv[0].is_cuda:
                torch.cuda.synchronize()
            h._bar.wait()

        def allreduce_sum(self, t):
            h = self.hub
            h._box[("ar", self.rank)] = t.clone()
            if t.is_cuda:
                torch.cuda.synchronize()
            h._bar.wait()
            acc = h._box[("ar", 0)].clone()
            for q in range(1, h.world):
                acc += h._box[("ar", q)]
            h._bar.wait()
            t.copy_(acc)
            return t


def window_halo(kind: str, N: int, s: int) -> int:
    """Stencil reach (grid points) of one forward + adjoint window sweep (N intervals of s
    TL sub-steps): a slab extended by this many points on each side computes its own points
    of L^{-T} H^T R^{-1} H L^{-1} exactly with no further exchange.  s_0 on the slab needs
    s_i (and so H^T y_i, i.e. the forward state x_i) within i r_adj of it, while the forward
    state x_i is exact within H - i r_fwd of the slab: per side H >= N (r_fwd + r_adj), with
    (r_fwd, r_adj) per interval = the TL step's reach on that side and the adjoint's.
    Upwind advection (models.cpp:27-45): (s, 0) left, (0, s) right -> N s; advection-
    diffusion: (s, s) -> 2 N s; the RK4 Lorenz-96 Jacobian (models.cpp:92-116, radius 2
    left / 1 right per stage, 4 stages per step): (8 s, 4 s) left, (4 s, 8 s) right -> 12 N s,
    plus 8 points for the RK4 stages recomputed on the slab from its trajectory rows (three
    dependent right-hand sides, models.cpp:80-87)."""
    if kind == "identity":
        return 0
    if kind == "advection":
        return N * s
    if kind == "advdiff":
        return 2 * N * s
    if kind == "l96":
        return 12 * N * s + 8
    raise ValueError(f"window_halo: unknown model {kind}")


@dataclass
class SlabGeometry:
    """Spatial decomposition for the row-sharded Hessian apply: rank r owns
    grid points [a, b) of EVERY window block (N + 1 blocks of n points); a local vector is
    the (N + 1) x n_loc block-major array.  The sweeps run on the slab extended by `halo`
    points per side as a periodic domain of n_ext = n_loc + 2 halo points."""
    n: int
    N: int
    world: int
    rank: int
    halo: int

    @property
    def a(self) -> int:
        return row_range(self.n, self.world, self.rank)[0]

    @property
    def b(self) -> int:
        return row_range(self.n, self.world, self.rank)[1]

    @property
    def n_loc(self) -> int:
        return self.b - self.a

    @property
    def n_ext(self) -> int:
        return self.n_loc + 2 * self.halo

    def ext_points(self, rank: Optional[int] = None) -> torch.Tensor:
        """Global grid index of every extended-slab point of `rank` (periodic)."""
        r = self.rank if rank is None else rank
        a, b = row_range(self.n, self.world, r)
        return (torch.arange(a - self.halo, b + self.halo, dtype=torch.int64) % self.n)

    def owner(self, g: torch.Tensor) -> torch.Tensor:
        bounds = torch.tensor([row_range(self.n, self.world, r)[1] for r in range(self.world)], dtype=torch.int64)
        return torch.bucketize(g, bounds, right=True)

    def window_indices(self) -> torch.Tensor:
        """Indices into a full window vector (n (N+1)) of this rank's local vector."""
        j = torch.arange(self.a, self.b, dtype=torch.int64)
        return (torch.arange(self.N + 1, dtype=torch.int64)[:, None] * self.n + j[None, :]).reshape(-1)


def slab_network(points, times, n: int, geom: SlabGeometry):
    """The observation network restricted to the extended slab, in local (extended) indices:
    (local points, times).  Observation times are unchanged."""
    pts = set(int(p) for p in points)
    g = geom.ext_points().tolist()
    return [j for j, gj in enumerate(g) if gj in pts], list(times)


class RowShardedHessian:
    """HessianOperator::apply (operators.cpp:127-144) on spatial slabs, one rank per GPU:

      t = D^{1/2} v   -- block-sharded: an all-to-all turns slabs into whole window blocks,
                         each rank applies B^{1/2} / Q^{1/2} to its blocks, and a second
                         all-to-all returns slabs;
      s = L^{-T} H^T R^{-1} H L^{-1} t
                      -- ONE halo exchange of t (window_halo points per side, every block),
                         then the whole forward + adjoint window sweep on the extended slab
                         with no further communication (the halo is the stencil reach);
      out = v + D^{1/2} s.

    `ops` supplies the local steps: factor(X (c, n), which) and sweeps(T_ext (N+1, n_ext)).
    The DEVICE backend is `DeviceSlabOps` (library kernels through the C-ABI); tests inject a
    CPU backend built on the oracle."""

    def __init__(self, geom: SlabGeometry, ops, comm=None):
        self.geom, self.ops = geom, ops
        self.comm = comm if comm is not None else TorchComm()
        g = geom
        self.blocks = [column_range(g.N + 1, g.world, r) for r in range(g.world)]
        self.slabs = [row_range(g.n, g.world, r) for r in range(g.world)]
        # halo exchange plan: for every rank q, the positions of its extended slab owned by
        # each rank (the same plan on every rank, so sender and receiver agree on the order)
        self._ext_src = []   # per q: list over r of (ext positions j, global indices)
        for q in range(g.world):
            gq = g.ext_points(q)
            own = g.owner(gq)
            self._ext_src.append([(torch.nonzero(own == r).reshape(-1), gq[own == r]) for r in range(g.world)])

    # -- D^{1/2}: slabs -> whole blocks -> factor -> slabs
    def d_half(self, x: torch.Tensor) -> torch.Tensor:
        g = self.geom
        n_loc = g.n_loc
        send = [x[i0:i1].reshape(-1) for (i0, i1) in self.blocks]
        my0, my1 = self.blocks[g.rank]
        nb = my1 - my0
        recv = [torch.empty(nb * (b - a), dtype=x.dtype, device=x.device) for (a, b) in self.slabs]
        self.comm.alltoall(recv, send)
        full = torch.empty((nb, g.n), dtype=x.dtype, device=x.device)
        for (a, b), rv in zip(self.slabs, recv):
            full[:, a:b] = rv.reshape(nb, b - a)
        out = torch.empty_like(full)
        if nb:
            if my0 == 0:  # block 0 takes B^{1/2} (operators.cpp:106), the rest Q^{1/2} (:110)
                out[:1] = self.ops.factor(full[:1], 0)
                if nb > 1:
                    out[1:] = self.ops.factor(full[1:], 1)
            else:
                out[:] = self.ops.factor(full, 1)
        send2 = [out[:, a:b].reshape(-1).contiguous() for (a, b) in self.slabs]
        recv2 = [torch.empty((i1 - i0) * n_loc, dtype=x.dtype, device=x.device) for (i0, i1) in self.blocks]
        self.comm.alltoall(recv2, send2)
        return torch.cat([rv.reshape(-1, n_loc) for rv in recv2], dim=0)

    # -- halo exchange: the extended slab of every block
    def extend(self, t: torch.Tensor) -> torch.Tensor:
        g = self.geom
        a = g.a
        send = []
        for q in range(g.world):  # what q's extended slab needs from this rank
            _, gidx = self._ext_src[q][g.rank]
            send.append(t[:, (gidx - a).to(t.device)].reshape(-1).contiguous())
        recv = [torch.empty(g.N + 1, len(self._ext_src[g.rank][r][0]), dtype=t.dtype, device=t.device).reshape(-1)
                for r in range(g.world)]
        self.comm.alltoall(recv, send)
        ext = torch.empty((g.N + 1, g.n_ext), dtype=t.dtype, device=t.device)
        for r in range(g.world):
            pos, _ = self._ext_src[g.rank][r]
            ext[:, pos.to(t.device)] = recv[r].reshape(g.N + 1, -1)
        return ext

    def apply(self, v: torch.Tensor) -> torch.Tensor:
        """v: (N+1, n_loc) local slab of one window vector -> A v on the same slab."""
        g = self.geom
        t = self.d_half(v)
        s_ext = self.ops.sweeps(self.extend(t))
        s = s_ext[:, g.halo:g.halo + g.n_loc].contiguous()
        return v + self.d_half(s)

    def apply_rows(self, v_flat: torch.Tensor) -> torch.Tensor:
        """dist_pcg's callback: the flattened slab (block-major) in, the same out."""
        g = self.geom
        return self.apply(v_flat.reshape(g.N + 1, g.n_loc)).reshape(-1)


class DeviceSlabOps:
    """The row-sharded apply's local steps on this rank's GPU, through the C-ABI: the factor
    applies on an operator holding the n-point covariance factors, and the sweeps
    (WC4DVAR_SWEEPS piece) on an operator built for the extended slab: the same model on
    n_ext points (for Lorenz-96 the linearisation trajectory's extended-slab rows), the
    network's observed points inside the slab and R^{-1}."""

    def __init__(self, model, net, b_half, q_half, sigma_obs: float, geom: SlabGeometry, device: int = 0):
        from . import wc4dvar as w
        self.w = w
        self.geom = geom
        n, N = model.n, model.N
        # D^{1/2}: the full-size factors on a minimal operator (identity model, no network)
        self.fop = w.HessianOperator(w.IdentityLinearized(n, 1), w.ObservationNetwork.empty(n, 1), b_half, q_half,
                                     sigma_obs, device)
        ne = geom.n_ext
        pts, times = slab_network(net.points, net.times, n, geom)
        snet = w.ObservationNetwork(ne, N, 1, 1, list(times), list(pts), len(times) * len(pts))
        if model.kind == "l96" and model.stages is not None:  # host stages (N s, 4 n)
            idx = geom.ext_points().numpy()
            st = model.stages.reshape(-1, 4, n)[:, :, idx].reshape(-1, 4 * ne)
            smodel = w.LinearizedModel("l96", ne, N, model.substeps, dt=model.dt, stages=st)
        elif model.kind == "l96":
            tr = model.trajectory
            idx = geom.ext_points()
            if isinstance(tr, torch.Tensor):     # device (steps + 1, n) row-major
                tslab = tr[:, idx.to(tr.device)].contiguous()
            else:                                # host n x (steps + 1)
                tslab = tr[idx.numpy(), :]
            smodel = w.Lorenz96Linearized(tslab, model.forcing, model.dt, model.substeps)
        else:
            smodel = w.LinearizedModel(model.kind, ne, N, model.substeps, model.courant, model.diffusion)
        unit = torch.zeros(ne, dtype=torch.float64)
        unit[0] = 1.0
        eye = w.CovarianceFactor(unit.numpy(), unit.numpy(), kind="circulant")  # unused by the sweeps
        self.sop = w.HessianOperator(smodel, snet, eye, eye, sigma_obs, device)

    def factor(self, X: torch.Tensor, which: int) -> torch.Tensor:
        X = X.contiguous()
        out = torch.empty_like(X)
        self.fop.factor_apply_dev(which, False, X, out, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        return out

    def sweeps(self, T: torch.Tensor) -> torch.Tensor:
        g = self.geom
        V = T.reshape(1, -1).contiguous()  # one window column of the extended slab
        out = torch.empty_like(V)
        self.sop.piece_dev(4, V, out, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        return out.reshape(g.N + 1, g.n_ext)
