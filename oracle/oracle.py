"""CPU oracle for the randomized-LMP hot path -- TEST INFRASTRUCTURE ONLY.

This module is the parity checker for the CUDA library.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` / ``--impl
reference`` legs may import it; the product package never does.

It restates the reference (``/root/reference/proj``, C++20 + Eigen 3) as:

* ``oracle/wc4dvar_oracle.c`` (loaded here through ctypes): the bit-exact
  ``NormalStream`` RNG, the model steps, the observation operator and the
  matrix-free ``HessianOperator`` apply with its threaded ``apply_block``;
* numpy / scipy LAPACK below, standing in for the Eigen dense decompositions
  the reference calls (HouseholderQR, ColPivHouseholderQR, SelfAdjointEigenSolver,
  LLT, BDCSVD).  Results agree with Eigen to rounding, not bitwise.

Pinning: the RNG is checked bit-for-bit against
libstdc++'s ``std::mt19937_64`` (tests/golden/normal_stream.json), every
known-answer test of the reference's own suites for this path is ported in
tests/test_oracle_*.py, and the reference's recorded acceptance_5 ensemble
result (proj/test_output.txt:29: mean minimum eigenvalues 0.173 / 0.684 /
0.797) is reproduced.  The BASELINE-only extensions (advection-diffusion,
sub-steps, ritzit p_iter > 1, circulant factors) are *parity unpinned*.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np
import scipy.linalg

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")


def _load():
    if not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(
        os.path.join(_HERE, "wc4dvar_oracle.c")
    ):
        subprocess.check_call(["make", "-s", "-C", _HERE, "all"])
    return ctypes.CDLL(_LIB_PATH)


_lib = _load()
_dp = ctypes.POINTER(ctypes.c_double)
_ip = ctypes.POINTER(ctypes.c_int)
_i64 = ctypes.c_int64


def _ptr(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(_dp)


# ---------------------------------------------------------------------------
# Error contract (proj/include/wc4dvar/types.hpp:14-30)
# ---------------------------------------------------------------------------
class NumericalError(RuntimeError):
    """types.hpp:19-21"""


class DenseCapError(RuntimeError):
    """types.hpp:24-26"""


def require(cond: bool, what: str) -> None:
    """types.hpp:28-30 -- std::invalid_argument maps to ValueError."""
    if not cond:
        raise ValueError(what)


# ---------------------------------------------------------------------------
# NormalStream (random.hpp:14-42)
# ---------------------------------------------------------------------------
_lib.orc_stream_new.restype = ctypes.c_void_p
_lib.orc_stream_new.argtypes = [ctypes.c_uint64]
_lib.orc_stream_free.argtypes = [ctypes.c_void_p]
_lib.orc_stream_fill.argtypes = [ctypes.c_void_p, _i64, _dp]
_lib.orc_stream_raw.restype = ctypes.c_uint64
_lib.orc_stream_raw.argtypes = [ctypes.c_void_p]
_lib.orc_gaussian_matrix.argtypes = [_i64, _i64, ctypes.c_uint64, _dp]


class NormalStream:
    """random.hpp:14-42: mt19937_64 + Box-Muller, two raw draws per normal."""

    def __init__(self, seed: int):
        self._h = _lib.orc_stream_new(ctypes.c_uint64(seed & 0xFFFFFFFFFFFFFFFF))

    def __del__(self):
        if getattr(self, "_h", None):
            _lib.orc_stream_free(self._h)
            self._h = None

    def raw(self) -> int:
        return int(_lib.orc_stream_raw(self._h))

    def next(self) -> float:
        return float(self.draw(1)[0])

    def draw(self, n: int) -> np.ndarray:
        out = np.empty(int(n), dtype=np.float64)
        if n:
            _lib.orc_stream_fill(self._h, int(n), _ptr(out))
        return out

    def fill(self, rows: int, cols: int) -> np.ndarray:
        """Column-major fill (random.hpp:28-31); returns an (rows, cols) array."""
        flat = self.draw(rows * cols)
        return flat.reshape(cols, rows).T.copy(order="F")


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """randevd.cpp:16-21."""
    out = np.empty(rows * cols, dtype=np.float64)
    if rows * cols:
        _lib.orc_gaussian_matrix(int(rows), int(cols), ctypes.c_uint64(seed), _ptr(out))
    return out.reshape(cols, rows).T.copy(order="F")


def random_orthogonal(n: int, seed: int) -> np.ndarray:
    """proj/tests/test_support.hpp:14-20 (Householder Q of a seeded Gaussian)."""
    G = NormalStream(seed).fill(n, n)
    Q, _ = np.linalg.qr(G)
    return Q


def random_spd(eigenvalues: np.ndarray, seed: int) -> np.ndarray:
    """test_support.hpp:23-27."""
    V = random_orthogonal(len(eigenvalues), seed)
    A = V @ np.diag(eigenvalues) @ V.T
    return 0.5 * (A + A.T)


# ---------------------------------------------------------------------------
# Models (proj/src/models.cpp)
# ---------------------------------------------------------------------------
for _name in ("orc_advection_step", "orc_advection_adjoint_step"):
    getattr(_lib, _name).argtypes = [_i64, _dp, ctypes.c_double, _dp]
for _name in ("orc_advdiff_step", "orc_advdiff_adjoint_step"):
    getattr(_lib, _name).argtypes = [_i64, _dp, ctypes.c_double, ctypes.c_double, _dp]
_lib.orc_l96_rhs.argtypes = [_i64, _dp, ctypes.c_double, _dp]
_lib.orc_l96_step.argtypes = [_i64, _dp, ctypes.c_double, ctypes.c_double, _dp]
_lib.orc_l96_stages.argtypes = [_i64, _dp, ctypes.c_double, ctypes.c_double, _dp]
_lib.orc_l96_tlm_step.argtypes = [_i64, _dp, _dp, ctypes.c_double, _dp]
_lib.orc_l96_adjoint_step.argtypes = [_i64, _dp, _dp, ctypes.c_double, _dp]


def _vec(v) -> np.ndarray:
    return np.ascontiguousarray(v, dtype=np.float64)


def advection_step(u, courant: float) -> np.ndarray:
    """models.cpp:27-35."""
    u = _vec(u)
    out = np.empty_like(u)
    _lib.orc_advection_step(len(u), _ptr(u), courant, _ptr(out))
    return out


def advection_adjoint_step(lam, courant: float) -> np.ndarray:
    """models.cpp:37-45."""
    lam = _vec(lam)
    out = np.empty_like(lam)
    _lib.orc_advection_adjoint_step(len(lam), _ptr(lam), courant, _ptr(out))
    return out


def advdiff_step(u, courant: float, diffusion: float) -> np.ndarray:
    """EXTENSION: upwind advection + centred diffusion (BASELINE configs 1, 2, 4)."""
    u = _vec(u)
    out = np.empty_like(u)
    _lib.orc_advdiff_step(len(u), _ptr(u), courant, diffusion, _ptr(out))
    return out


def advdiff_adjoint_step(lam, courant: float, diffusion: float) -> np.ndarray:
    lam = _vec(lam)
    out = np.empty_like(lam)
    _lib.orc_advdiff_adjoint_step(len(lam), _ptr(lam), courant, diffusion, _ptr(out))
    return out


def lorenz96_rhs(x, forcing: float) -> np.ndarray:
    """models.cpp:59-70."""
    x = _vec(x)
    require(len(x) >= 4, "lorenz96_rhs: n must be >= 4")
    out = np.empty_like(x)
    _lib.orc_l96_rhs(len(x), _ptr(x), forcing, _ptr(out))
    return out


def lorenz96_step(x, forcing: float, dt: float) -> np.ndarray:
    """models.cpp:72-78."""
    x = _vec(x)
    out = np.empty_like(x)
    _lib.orc_l96_step(len(x), _ptr(x), forcing, dt, _ptr(out))
    return out


def lorenz96_stages(x, forcing: float, dt: float) -> np.ndarray:
    """models.cpp:80-87; returns [x1 | x2 | x3 | x4] (4n)."""
    x = _vec(x)
    out = np.empty(4 * len(x))
    _lib.orc_l96_stages(len(x), _ptr(x), forcing, dt, _ptr(out))
    return out


def lorenz96_tlm_step(stages, dx, dt: float) -> np.ndarray:
    """models.cpp:120-128."""
    stages, dx = _vec(stages), _vec(dx)
    out = np.empty_like(dx)
    _lib.orc_l96_tlm_step(len(dx), _ptr(stages), _ptr(dx), dt, _ptr(out))
    return out


def lorenz96_adjoint_step(stages, lam, dt: float) -> np.ndarray:
    """models.cpp:130-148."""
    stages, lam = _vec(stages), _vec(lam)
    out = np.empty_like(lam)
    _lib.orc_l96_adjoint_step(len(lam), _ptr(stages), _ptr(lam), dt, _ptr(out))
    return out


@dataclass
class ObservationNetwork:
    """models.hpp:45-56 / models.cpp:159-182."""

    n: int = 0
    N: int = 0
    space_stride: int = 1
    time_stride: int = 1
    times: List[int] = field(default_factory=list)
    points: List[int] = field(default_factory=list)
    q: int = 0

    @staticmethod
    def build(n: int, N: int, space_stride: int, time_stride: int) -> "ObservationNetwork":
        require(n >= 1 and N >= 1, "ObservationNetwork: grid must be nonempty")
        require(1 <= space_stride <= n, "ObservationNetwork: space stride inconsistent with grid")
        require(1 <= time_stride <= N, "ObservationNetwork: time stride inconsistent with window")
        times = list(range(N, 0, -time_stride))[::-1]
        points = list(range(0, n, space_stride))
        return ObservationNetwork(n, N, space_stride, time_stride, times, points,
                                  len(times) * len(points))

    @staticmethod
    def empty(n: int, N: int) -> "ObservationNetwork":
        """The hand-built q = 0 network of test_operators.cpp:65-76,122-133."""
        return ObservationNetwork(n, N, 1, 1, [], [], 0)

    def q_at(self, t: int) -> int:
        return len(self.points) if t in self.times else 0


def observe(traj: np.ndarray, net: ObservationNetwork) -> np.ndarray:
    """models.cpp:184-192."""
    require(len(traj) == net.n * (net.N + 1), "observe: trajectory length mismatch")
    idx = [t * net.n + j for t in net.times for j in net.points]
    return np.asarray(traj)[idx].copy()


def observe_adjoint(y: np.ndarray, net: ObservationNetwork) -> np.ndarray:
    """models.cpp:194-201."""
    require(len(y) == net.q, "observe_adjoint: observation length mismatch")
    out = np.zeros(net.n * (net.N + 1))
    idx = [t * net.n + j for t in net.times for j in net.points]
    out[idx] = y
    return out


# ---------------------------------------------------------------------------
# Covariances (proj/src/covariance.cpp)
# ---------------------------------------------------------------------------
_lib.orc_build_soar.argtypes = [ctypes.c_int, ctypes.c_double, ctypes.c_double, _dp]


def build_soar(sigma: float, length_scale: float, n: int) -> np.ndarray:
    """covariance.cpp:25-48 (chordal distance SOAR, SPD-checked)."""
    require(n >= 1, "build_soar: dimension must be positive")
    require(sigma > 0.0, "build_soar: sigma must be positive")
    require(length_scale > 0.0, "build_soar: length scale must be positive")
    C = np.empty((n, n), order="F")
    _lib.orc_build_soar(n, sigma, length_scale, _ptr(C))
    mn = np.linalg.eigvalsh(C).min()
    if mn <= 0.0:
        raise NumericalError(f"build_soar: matrix is not positive definite (smallest eigenvalue {mn})")
    return C


def build_laplacian_corr(sigma: float, length_scale: float, n: int) -> np.ndarray:
    """covariance.cpp:50-71."""
    require(n >= 2, "build_laplacian_corr: dimension must be >= 2")
    require(sigma > 0.0, "build_laplacian_corr: sigma must be positive")
    require(length_scale > 0.0, "build_laplacian_corr: length scale must be positive")
    l2 = length_scale * length_scale
    M = np.eye(n)
    for i in range(n):
        M[i, i] += 2.0 * l2
        M[i, (i + 1) % n] -= l2
        M[i, (i + n - 1) % n] -= l2
    w, V = np.linalg.eigh(M)
    if w.min() <= 0.0:
        raise NumericalError("build_laplacian_corr: shifted Laplacian not positive definite")
    C0 = V @ np.diag((1.0 / w) ** 2) @ V.T
    C0 = 0.5 * (C0 + C0.T)
    gamma = 1.0 / np.diag(C0).max()
    return np.asfortranarray(sigma * sigma * gamma * C0)


def build_covariance(kind: str, sigma: float, length_scale: float, n: int) -> np.ndarray:
    """covariance.cpp:73-84."""
    if kind == "diagonal":
        require(n >= 1 and sigma > 0.0, "build_covariance: bad diagonal spec")
        return sigma * sigma * np.eye(n, order="F")
    if kind == "soar":
        return build_soar(sigma, length_scale, n)
    if kind == "laplacian":
        return build_laplacian_corr(sigma, length_scale, n)
    raise ValueError("build_covariance: unknown kind")


@dataclass
class CovarianceFactor:
    """covariance.hpp:31-38 (dense), plus the EXTENSION circulant representation:
    ``kind == 'circulant'`` stores the first columns of C^{1/2} and C^{-1/2}."""

    half: np.ndarray
    half_inv: np.ndarray
    kind: str = "dense"

    def dim(self) -> int:
        return self.half.shape[0]

    def apply(self, v):
        if self.kind == "dense":
            return self.half @ v
        return _circ_apply(self.half, v)

    def apply_inv(self, v):
        if self.kind == "dense":
            return self.half_inv @ v
        return _circ_apply(self.half_inv, v)

    def dense_half(self) -> np.ndarray:
        if self.kind == "dense":
            return self.half
        return scipy.linalg.circulant(self.half)


def _circ_apply(c: np.ndarray, v: np.ndarray) -> np.ndarray:
    return np.real(np.fft.ifft(np.fft.fft(c) * np.fft.fft(v, axis=0).T).T) if v.ndim == 2 else \
        np.real(np.fft.ifft(np.fft.fft(c) * np.fft.fft(v)))


def sym_sqrt(C: np.ndarray) -> CovarianceFactor:
    """covariance.cpp:86-105."""
    C = np.asarray(C, dtype=np.float64)
    require(C.shape[0] == C.shape[1], "sym_sqrt: matrix must be square")
    require(np.abs(C - C.T).max(initial=0.0) <= 1e-12 * (1.0 + np.abs(C).max(initial=0.0)),
            "sym_sqrt: matrix must be symmetric")
    w, V = np.linalg.eigh(C)
    if w.min() <= 0.0:
        raise NumericalError(f"sym_sqrt: matrix is not positive definite (eigenvalue {w.min()})")
    root = np.sqrt(w)
    half = V @ np.diag(root) @ V.T
    half_inv = V @ np.diag(1.0 / root) @ V.T
    return CovarianceFactor(np.asfortranarray(0.5 * (half + half.T)),
                            np.asfortranarray(0.5 * (half_inv + half_inv.T)))


def circulant_sqrt(first_col: np.ndarray) -> CovarianceFactor:
    """EXTENSION: symmetric square root of a symmetric circulant SPD
    matrix from its first column, via the DFT eigenbasis.  For SOAR on the periodic
    grid (circulant by covariance.cpp:36-41, pinned by test_covariance.cpp:41-43) this
    equals sym_sqrt(build_soar(...)) to rounding."""
    lam = np.real(np.fft.fft(first_col))
    if lam.min() <= 0.0:
        raise NumericalError(f"circulant_sqrt: matrix is not positive definite (eigenvalue {lam.min()})")
    half = np.real(np.fft.ifft(np.sqrt(lam)))
    half_inv = np.real(np.fft.ifft(1.0 / np.sqrt(lam)))
    return CovarianceFactor(half, half_inv, kind="circulant")


def soar_first_column(sigma: float, length_scale: float, n: int) -> np.ndarray:
    """First column of build_soar (covariance.cpp:31-44) without forming n x n."""
    d = np.minimum(np.arange(n), n - np.arange(n)).astype(np.float64)
    r = (n / math.pi) * np.sin(math.pi * d / n)
    return sigma * sigma * (1.0 + r / length_scale) * np.exp(-r / length_scale)


def sample_noise(factor: CovarianceFactor, seed: int) -> np.ndarray:
    """covariance.cpp:107-111."""
    if factor.dim() == 0:
        return np.zeros(0)
    return factor.apply(NormalStream(seed).draw(factor.dim()))


# ---------------------------------------------------------------------------
# Operators (proj/src/operators.cpp)
# ---------------------------------------------------------------------------
class LinearOperator:
    """operators.hpp:15-40: apply counting; apply_block is column-wise."""

    def __init__(self):
        self._applies = 0

    def dim(self) -> int:
        raise NotImplementedError

    def _apply(self, v: np.ndarray) -> np.ndarray:
        raise NotImplementedError

    def apply(self, v) -> np.ndarray:
        v = _vec(v)
        require(len(v) == self.dim(), f"{type(self).__name__}::apply: dimension mismatch")
        self._applies += 1
        return self._apply(v)

    def apply_block(self, V, threads: int = 1) -> np.ndarray:
        """operators.cpp:9-19."""
        V = np.asarray(V, dtype=np.float64)
        require(V.shape[0] == self.dim(), "LinearOperator::apply_block: dimension mismatch")
        out = np.empty_like(V, order="F")
        for j in range(V.shape[1]):
            out[:, j] = self.apply(V[:, j])
        return out

    def apply_count(self) -> int:
        return self._applies

    def reset_apply_count(self) -> None:
        self._applies = 0

    def count(self, k: int) -> None:
        self._applies += k


class DenseOperator(LinearOperator):
    """operators.hpp:42-53 / operators.cpp:21-29."""

    def __init__(self, A):
        super().__init__()
        A = np.asarray(A, dtype=np.float64)
        require(A.shape[0] == A.shape[1], "DenseOperator: matrix must be square")
        self.A = np.asfortranarray(A)

    def dim(self):
        return self.A.shape[0]

    def _apply(self, v):
        return self.A @ v

    def apply_block(self, V, threads: int = 1):
        V = np.asarray(V, dtype=np.float64)
        require(V.shape[0] == self.dim(), "LinearOperator::apply_block: dimension mismatch")
        self._applies += V.shape[1]
        return np.asfortranarray(self.A @ V)


@dataclass
class LinearizedModel:
    """operators.hpp:57-111: identity / advection (reference) plus the EXTENSION kinds
    advdiff (upwind + diffusion) and sub-steps s > 1; lorenz96 carries RK4 stages for
    each of the N*s sub-steps (operators.cpp:44-51 generalised)."""

    kind: str
    n: int
    N: int
    substeps: int = 1
    courant: float = 0.0
    diffusion: float = 0.0
    dt: float = 0.0
    stages: Optional[np.ndarray] = None  # (N*s, 4n) flattened

    def state_dim(self):
        return self.n

    def steps(self):
        return self.N


def IdentityLinearized(n: int, N: int) -> LinearizedModel:
    return LinearizedModel("identity", n, N)


def AdvectionLinearized(n: int, N: int, courant: float) -> LinearizedModel:
    """operators.cpp:31-42."""
    require(n >= 1 and N >= 0, "AdvectionLinearized: bad window")
    return LinearizedModel("advection", n, N, 1, courant)


def AdvDiffLinearized(n: int, N: int, courant: float, diffusion: float, substeps: int = 1):
    """EXTENSION (BASELINE configs 1, 2, 4)."""
    require(n >= 1 and N >= 0 and substeps >= 1, "AdvDiffLinearized: bad window")
    return LinearizedModel("advdiff", n, N, substeps, courant, diffusion)


def Lorenz96Linearized(trajectory: np.ndarray, forcing: float, dt: float, substeps: int = 1):
    """operators.cpp:44-51.  ``trajectory`` has N*s + 1 columns (n each); sub-step k of
    subwindow i is linearised at column i*s + k.  s = 1 is the reference exactly."""
    trajectory = np.asarray(trajectory, dtype=np.float64)
    require(trajectory.shape[1] >= 2, "Lorenz96Linearized: trajectory too short")
    n = trajectory.shape[0]
    total = trajectory.shape[1] - 1
    require(total % substeps == 0, "Lorenz96Linearized: trajectory/sub-step mismatch")
    stages = np.stack([lorenz96_stages(trajectory[:, c], forcing, dt) for c in range(total)])
    return LinearizedModel("l96", n, total // substeps, substeps, dt=dt, stages=stages)


class _OrcHessian(ctypes.Structure):
    _fields_ = [
        ("model", ctypes.c_int), ("n", _i64), ("N", ctypes.c_int), ("substeps", ctypes.c_int),
        ("courant", ctypes.c_double), ("diffusion", ctypes.c_double), ("dt", ctypes.c_double),
        ("stages", _dp), ("n_times", ctypes.c_int), ("times", _ip), ("n_points", ctypes.c_int),
        ("points", _ip), ("cov_kind", ctypes.c_int), ("b_half", _dp), ("b_half_inv", _dp),
        ("q_half", _dp), ("q_half_inv", _dp), ("sigma_obs", ctypes.c_double),
    ]


_HP = ctypes.POINTER(_OrcHessian)
for _name in ("orc_apply_Linv", "orc_apply_LinvT", "orc_apply_D_half", "orc_apply_D_half_inv"):
    getattr(_lib, _name).argtypes = [_HP, _dp, _dp]
_lib.orc_hessian_apply.argtypes = [_HP, _dp, _dp]
_lib.orc_hessian_apply.restype = ctypes.c_int
_lib.orc_hessian_apply_block.argtypes = [_HP, _i64, _dp, _dp, ctypes.c_int]
_lib.orc_hessian_apply_block.restype = ctypes.c_int
_lib.orc_hessian_sweeps_block.argtypes = [_HP, _i64, _dp, ctypes.c_int]
_lib.orc_hessian_sweeps_block.restype = ctypes.c_int
_MODEL_CODES = {"identity": 0, "advection": 1, "advdiff": 2, "l96": 3}
_STAGE_MSG = {
    1: "hessian apply: non-finite value after forward sweep",
    2: "hessian apply: non-finite value after adjoint sweep",
    3: "hessian apply: non-finite result",
}


class HessianOperator(LinearOperator):
    """operators.hpp:116-152 / operators.cpp:127-144 (Eq. 12 of the paper):
    A = I + D^{1/2} L^{-T} H^T R^{-1} H L^{-1} D^{1/2}."""

    def __init__(self, model: LinearizedModel, net: ObservationNetwork,
                 background_half: CovarianceFactor, model_error_half: CovarianceFactor,
                 sigma_obs: float, threads: int = 1):
        super().__init__()
        require(sigma_obs > 0.0, "HessianOperator: sigma_obs must be positive")
        require(background_half is not None and background_half.dim() == model.n,
                "HessianOperator: background factor mismatch")
        require(model_error_half is not None and model_error_half.dim() == model.n,
                "HessianOperator: model-error factor mismatch")
        require(net.n == model.n and net.N == model.N, "HessianOperator: network/window mismatch")
        require(background_half.kind == model_error_half.kind,
                "HessianOperator: factors must share a representation")
        self.model, self.net = model, net
        self.b_half, self.q_half = background_half, model_error_half
        self.sigma_obs_ = sigma_obs
        self.threads = threads
        self._keep = []
        self._fft = {}
        # fast = True routes apply / apply_block through apply_block_fast (batched D^{1/2}:
        # BLAS GEMM or real FFT); the default per-column C path is the reference's loop order.
        self.fast = False

        def keep(a, dtype=np.float64):
            a = np.ascontiguousarray(a, dtype=dtype)
            self._keep.append(a)
            return a

        h = _OrcHessian()
        h.model = _MODEL_CODES[model.kind]
        h.n, h.N, h.substeps = model.n, model.N, model.substeps
        h.courant, h.diffusion, h.dt = model.courant, model.diffusion, model.dt
        h.stages = _ptr(keep(model.stages)) if model.stages is not None else None
        times, points = keep(net.times, np.int32), keep(net.points, np.int32)
        h.n_times, h.times = len(net.times), times.ctypes.data_as(_ip)
        h.n_points, h.points = len(net.points), points.ctypes.data_as(_ip)
        h.cov_kind = 0 if background_half.kind == "dense" else 1
        # dense factors are symmetric, so C order == F order
        h.b_half = _ptr(keep(np.asfortranarray(background_half.half).ravel(order="F")))
        h.b_half_inv = _ptr(keep(np.asfortranarray(background_half.half_inv).ravel(order="F")))
        h.q_half = _ptr(keep(np.asfortranarray(model_error_half.half).ravel(order="F")))
        h.q_half_inv = _ptr(keep(np.asfortranarray(model_error_half.half_inv).ravel(order="F")))
        h.sigma_obs = sigma_obs
        self._h = h

    def dim(self):
        return self.model.n * (self.model.N + 1)

    def network(self):
        return self.net

    def sigma_obs(self):
        return self.sigma_obs_

    def _call(self, name, v):
        v = _vec(v)
        require(len(v) == self.dim(), f"{name}: window length mismatch")
        out = np.empty_like(v)
        getattr(_lib, "orc_" + name)(ctypes.byref(self._h), _ptr(v), _ptr(out))
        return out

    def apply_Linv(self, p):
        return self._call("apply_Linv", p)

    def apply_LinvT(self, v):
        return self._call("apply_LinvT", v)

    def apply_D_half(self, v):
        return self._call("apply_D_half", v)

    def apply_D_half_inv(self, v):
        return self._call("apply_D_half_inv", v)

    def _apply(self, v):
        if self.fast:
            return self.apply_block_fast(v.reshape(-1, 1), self.threads, count=False)[:, 0]
        out = np.empty_like(v)
        st = _lib.orc_hessian_apply(ctypes.byref(self._h), _ptr(v), _ptr(out))
        if st:
            raise NumericalError(_STAGE_MSG[st])
        return out

    def apply_block(self, V, threads: Optional[int] = None):
        if self.fast:
            return self.apply_block_fast(V, threads)
        V = np.asfortranarray(V, dtype=np.float64)
        require(V.shape[0] == self.dim(), "LinearOperator::apply_block: dimension mismatch")
        out = np.empty_like(V, order="F")
        m = V.shape[1]
        self._applies += m
        if m:
            st = _lib.orc_hessian_apply_block(ctypes.byref(self._h), m, _ptr(V), _ptr(out),
                                              threads or self.threads)
            if st:
                raise NumericalError(_STAGE_MSG[st])
        return out

    def apply_D_half_block(self, V, inv: bool = False, threads: Optional[int] = None) -> np.ndarray:
        """apply_D_half / _inv (operators.cpp:103-125) on a whole block.  The window block
        V (dim x m) is viewed as the n x (N+1)m matrix of its n-blocks; the dense factor is
        then ONE GEMM over that view (what operators.cpp:107-111 does per column, as
        Q^{1/2} [v_1 .. v_N]), multithreaded BLAS.  The circulant EXTENSION is one batched
        real FFT convolution (scipy.fft, `threads` workers): C^{1/2} = F^{-1} diag(lambda) F
        with lambda = DFT of the factor's first column (real: the column is symmetric)."""
        import scipy.fft
        V = np.asfortranarray(V, dtype=np.float64)
        n, N = self.model.n, self.model.N
        m = V.shape[1]
        X = V.reshape((n, (N + 1) * m), order="F")
        b = self.b_half.half_inv if inv else self.b_half.half
        qf = self.q_half.half_inv if inv else self.q_half.half
        first = np.arange(m) * (N + 1)
        if self.b_half.kind == "dense":
            out = np.asfortranarray(qf @ X) if N > 0 else np.empty_like(X, order="F")
            out[:, first] = b @ X[:, first]
        else:
            key = ("lam", inv)
            if key not in self._fft:
                self._fft[key] = (np.real(scipy.fft.rfft(b)), np.real(scipy.fft.rfft(qf)))
            lb, lq = self._fft[key]
            w = threads or self.threads or 1
            # X^T is the C-contiguous ((N+1)m, n) matrix of the n-blocks: row i + (N+1) j is
            # block i of column j
            F = scipy.fft.rfft(X.T, axis=1, workers=w)
            F3 = F.reshape((m, N + 1, F.shape[1]))
            F3[:, 0, :] *= lb
            F3[:, 1:, :] *= lq
            out = scipy.fft.irfft(F, n=n, axis=1, workers=w).T
        return out.reshape((n * (N + 1), m), order="F")

    def apply_block_fast(self, V, threads: Optional[int] = None, count: bool = True) -> np.ndarray:
        """HessianOperator::apply (operators.cpp:127-144) on a block, batched for the CPU
        baseline: D^{1/2} of the whole block (apply_D_half_block), then the per-column
        sweeps L^{-T} H^T R^{-1} H L^{-1} in C with the apply_block column fan-out
        (threads.cpp:25-44), then out = V + D^{1/2} S.  Same arithmetic as apply_block up
        to the summation order of the factor products."""
        V = np.asfortranarray(V, dtype=np.float64)
        require(V.shape[0] == self.dim(), "LinearOperator::apply_block: dimension mismatch")
        m = V.shape[1]
        if count:
            self._applies += m
        if m == 0:
            return np.empty_like(V, order="F")
        w = threads or self.threads or 1
        T = np.asfortranarray(self.apply_D_half_block(V, False, w))
        st = _lib.orc_hessian_sweeps_block(ctypes.byref(self._h), m, _ptr(T), w)
        if st:
            raise NumericalError(_STAGE_MSG[st])
        out = self.apply_D_half_block(T, False, w)
        out += V
        if not np.isfinite(out).all():
            raise NumericalError(_STAGE_MSG[3])
        return out

    def observation_range(self) -> np.ndarray:
        """operators.cpp:146-154: columns D^{1/2} L^{-T} H^T e_r."""
        W = np.empty((self.dim(), self.net.q), order="F")
        for r in range(self.net.q):
            e = np.zeros(self.net.q)
            e[r] = 1.0
            W[:, r] = self.apply_D_half(self.apply_LinvT(observe_adjoint(e, self.net)))
        return W


def assemble_dense(op: LinearOperator, cap: int = 4096) -> np.ndarray:
    """operators.cpp:156-164."""
    if op.dim() > cap:
        raise DenseCapError(f"assemble_dense: dimension {op.dim()} exceeds cap {cap}")
    A = op.apply_block(np.eye(op.dim(), order="F"))
    return 0.5 * (A + A.T)


# ---------------------------------------------------------------------------
# Ritz pairs / randomized EVD (proj/src/ritz.cpp, randevd.cpp)
# ---------------------------------------------------------------------------
@dataclass
class RitzPairs:
    """ritz.hpp:9-27."""

    vectors: np.ndarray
    values: np.ndarray
    source: str = "exact"

    def k(self):
        return len(self.values)

    def dim(self):
        return self.vectors.shape[0]

    def orthonormality_defect(self) -> float:
        if self.k() == 0:
            return 0.0
        G = self.vectors.T @ self.vectors
        return float(np.abs(G - np.eye(self.k())).max())

    def validate(self, tol: float = 1e-10) -> None:
        """ritz.cpp:7-20."""
        require(self.vectors.shape[1] == len(self.values), "RitzPairs: U/Theta size mismatch")
        for i in range(len(self.values) - 1):
            if self.values[i] < self.values[i + 1]:
                raise NumericalError("RitzPairs: values are not decreasing")
        if self.k() > 0 and self.values.min() <= 0.0:
            raise NumericalError("RitzPairs: nonpositive Ritz value")
        d = self.orthonormality_defect()
        if d > tol:
            raise NumericalError(f"RitzPairs: vectors not orthonormal (defect {d})")


@dataclass
class SketchConfig:
    """randevd.hpp:13-21; ``p_iter`` is the EXTENSION ritzit iteration count
    (1 = the reference's single-pass ritzit)."""

    target_rank: int = 1
    oversample: int = 5
    seed: int = 0
    method: str = "revd"
    p_iter: int = 1

    def sample_size(self):
        return self.target_rank + self.oversample

    def validate(self, n: int):
        """randevd.cpp:10-14."""
        require(self.target_rank >= 1, "SketchConfig: target rank must be >= 1")
        require(self.oversample >= 0, "SketchConfig: oversampling must be >= 0")
        require(self.sample_size() <= n, "SketchConfig: k + l exceeds operator dimension")


def householder_q(Y: np.ndarray) -> np.ndarray:
    """randevd.cpp:27-30."""
    Q, _ = np.linalg.qr(Y, mode="reduced")
    return Q


def colpiv_rank(Y: np.ndarray):
    """Eigen ColPivHouseholderQR::rank(): #{|R_ii| > min(r,c) * eps * max|R_kk|}
    (randevd.cpp:67,89).  Returns (rank, Q_thin) from LAPACK dgeqp3."""
    Q, R, _ = scipy.linalg.qr(Y, mode="economic", pivoting=True)
    d = np.abs(np.diag(R))
    if d.size == 0 or d.max() == 0.0:
        return 0, Q
    thr = min(Y.shape) * np.finfo(np.float64).eps * d.max()
    return int((d > thr).sum()), Q


def sorted_symmetric_evd(K: np.ndarray):
    """randevd.cpp:37-43: EVD of sym(K), decreasing order."""
    w, V = np.linalg.eigh(0.5 * (K + K.T))
    return w[::-1].copy(), V[:, ::-1].copy()


def rayleigh_ritz(op: LinearOperator, Z: np.ndarray) -> RitzPairs:
    """randevd.cpp:47-60."""
    require(Z.shape[0] == op.dim(), "rayleigh_ritz: dimension mismatch")
    m = Z.shape[1]
    if np.abs(Z.T @ Z - np.eye(m)).max(initial=0.0) > 1e-8:
        raise NumericalError("rayleigh_ritz: Z is not orthonormal")
    AZ = op.apply_block(Z)
    vals, W = sorted_symmetric_evd(Z.T @ AZ)
    return RitzPairs(Z @ W, vals, "revd")


def revd(op: LinearOperator, cfg: SketchConfig, G: Optional[np.ndarray] = None) -> RitzPairs:
    """randevd.cpp:62-80 (two block applies)."""
    cfg.validate(op.dim())
    m = cfg.sample_size()
    if G is None:
        G = gaussian_matrix(op.dim(), m, cfg.seed)
    Y = op.apply_block(G)
    rank, _ = colpiv_rank(Y)
    if rank < m:
        raise NumericalError(f"revd: sample matrix rank collapsed to {rank} of {m} columns")
    Z = householder_q(Y)
    pairs = rayleigh_ritz(op, Z)
    return RitzPairs(pairs.vectors[:, :cfg.target_rank].copy(),
                     pairs.values[:cfg.target_rank].copy(), "revd")


def nystrom(op: LinearOperator, cfg: SketchConfig, G: Optional[np.ndarray] = None) -> RitzPairs:
    """randevd.cpp:82-114 (two block applies)."""
    cfg.validate(op.dim())
    m = cfg.sample_size()
    if G is None:
        G = gaussian_matrix(op.dim(), m, cfg.seed)
    Y = op.apply_block(G)
    rank, Q = colpiv_rank(Y)
    if rank == 0:
        raise NumericalError("nystrom: sample matrix is zero")
    Z = Q[:, :rank]
    E1 = op.apply_block(Z)
    E2 = Z.T @ E1
    E2 = 0.5 * (E2 + E2.T)
    try:
        L = np.linalg.cholesky(E2)
    except np.linalg.LinAlgError:
        raise NumericalError(
            "nystrom: Cholesky of Z^T A Z failed; the projected operator is numerically "
            "indefinite. Increase the oversampling parameter or use revd for indefinite spectra.")
    # F = E1 U^{-1} with U = L^T  (randevd.cpp:103-105)
    F = scipy.linalg.solve_triangular(L, E1.T, lower=True).T
    U, s, _ = np.linalg.svd(F, full_matrices=False)
    keep = min(cfg.target_rank, rank)
    return RitzPairs(U[:, :keep].copy(), (s[:keep] ** 2).copy(), "nystrom")


def revd_ritzit(op: LinearOperator, cfg: SketchConfig, G: Optional[np.ndarray] = None) -> RitzPairs:
    """randevd.cpp:116-136 (one block apply).  EXTENSION: ``cfg.p_iter`` > 1 runs
    p_iter - 1 extra subspace-iteration passes Y <- A Q(Y) before the final R-factor
    step (BASELINE config 1's "ritzit (3 iterations)"; parity unpinned)."""
    cfg.validate(op.dim())
    m = cfg.sample_size()
    if G is None:
        G = gaussian_matrix(op.dim(), m, cfg.seed)
    G3 = householder_q(G)
    Y3 = op.apply_block(G3)
    for _ in range(max(cfg.p_iter, 1) - 1):
        Y3 = op.apply_block(householder_q(Y3))
    Z3, R3 = np.linalg.qr(Y3, mode="reduced")
    d = np.abs(np.diag(R3))
    if d.min() <= 1e-14 * d.max():
        raise NumericalError("revd_ritzit: QR of the sample matrix is rank deficient")
    vals, W = sorted_symmetric_evd(R3 @ R3.T)
    k = cfg.target_rank
    if vals[min(k, m) - 1] <= 0.0:
        raise NumericalError("revd_ritzit: nonpositive squared Ritz value")
    return RitzPairs(Z3 @ W[:, :k], np.sqrt(vals[:k]), "ritzit")


def sketch_eigenpairs(op: LinearOperator, cfg: SketchConfig, G=None) -> RitzPairs:
    """randevd.cpp:138-148."""
    if cfg.method == "revd":
        return revd(op, cfg, G)
    if cfg.method == "nystrom":
        return nystrom(op, cfg, G)
    if cfg.method == "ritzit":
        return revd_ritzit(op, cfg, G)
    raise ValueError("sketch_eigenpairs: unknown method")


# ---------------------------------------------------------------------------
# LMP (proj/src/lmp.cpp)
# ---------------------------------------------------------------------------
_lib.orc_lmp_apply.argtypes = [_i64, _i64, _dp, _dp, _dp, _dp]
_lib.orc_lmp_apply_transpose.argtypes = [_i64, _i64, _dp, _dp, _dp, _dp]


@dataclass
class LmpFactor:
    """lmp.hpp:12-26: C = prod_i (I - (1 - theta_i^{-1/2}) u_i u_i^T)."""

    vectors: np.ndarray
    values: np.ndarray

    def k(self):
        return len(self.values)

    def dim(self):
        return self.vectors.shape[0]

    def is_identity(self):
        return self.k() == 0

    def _run(self, fn, v):
        v = _vec(v)
        require(self.is_identity() or len(v) == self.dim(), "LmpFactor::apply: dimension mismatch")
        if self.is_identity():
            return v.copy()
        U = np.asfortranarray(self.vectors)
        th = _vec(self.values)
        out = np.empty_like(v)
        fn(len(v), self.k(), _ptr(U), _ptr(th), _ptr(v), _ptr(out))
        return out

    def apply(self, v):
        """lmp.cpp:8-16 (i = k..1)."""
        return self._run(_lib.orc_lmp_apply, v)

    def apply_transpose(self, v):
        """lmp.cpp:18-26 (i = 1..k)."""
        return self._run(_lib.orc_lmp_apply_transpose, v)

    @staticmethod
    def identity(n: int) -> "LmpFactor":
        return LmpFactor(np.zeros((n, 0), order="F"), np.zeros(0))


def build_spectral_lmp(pairs: RitzPairs) -> LmpFactor:
    """lmp.cpp:35-52."""
    if pairs.k() == 0:
        return LmpFactor.identity(pairs.dim())
    if pairs.values.min() <= 0.0:
        raise NumericalError(f"build_spectral_lmp: nonpositive Ritz value {pairs.values.min()}")
    d = pairs.orthonormality_defect()
    if d > 1e-8:
        raise NumericalError(f"build_spectral_lmp: Ritz vectors not orthonormal (defect {d})")
    return LmpFactor(np.asfortranarray(pairs.vectors), pairs.values.copy())


def dense_spectral_lmp(U, theta) -> np.ndarray:
    """lmp.cpp:81-88."""
    P = np.eye(U.shape[0])
    for i in range(len(theta)):
        P -= (1.0 - 1.0 / theta[i]) * np.outer(U[:, i], U[:, i])
    return P


# ---------------------------------------------------------------------------
# PCG (proj/src/krylov.cpp:22-108)
# ---------------------------------------------------------------------------
@dataclass
class PcgOptions:
    """krylov.hpp:32-38."""

    max_iter: int = 100
    rel_tol: float = 1e-6
    reorthogonalize: bool = False
    store_residual_vectors: bool = False
    cost_eval: Optional[Callable[[np.ndarray], float]] = None


@dataclass
class CgHistory:
    """krylov.hpp:17-30."""

    alphas: List[float] = field(default_factory=list)
    betas: List[float] = field(default_factory=list)
    residual_norms: List[float] = field(default_factory=list)
    quadratic_costs: List[float] = field(default_factory=list)
    normalized_residuals: List[np.ndarray] = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    stop_reason: str = ""


@dataclass
class PcgResult:
    x: np.ndarray
    history: CgHistory


def _check_finite(v, what, j):
    if not math.isfinite(v):
        raise NumericalError(f"pcg_split: non-finite {what} at iteration {j}")


def pcg_split(op: LinearOperator, b, precond: Optional[LmpFactor] = None,
              x0=None, opts: Optional[PcgOptions] = None) -> PcgResult:
    """krylov.cpp:22-99 (Algorithm 1, split preconditioned CG)."""
    opts = opts or PcgOptions()
    n = op.dim()
    b = _vec(b)
    precond = precond if precond is not None else LmpFactor.identity(n)
    require(len(b) == n, "pcg_split: right-hand side dimension mismatch")
    require(x0 is None or len(x0) == 0 or len(x0) == n, "pcg_split: initial guess dimension mismatch")
    hist = CgHistory()
    keep_f = opts.reorthogonalize or opts.store_residual_vectors
    x = np.zeros(n) if x0 is None or len(x0) == 0 else _vec(x0).copy()
    if x0 is None or len(x0) == 0 or not np.any(x0):
        r = precond.apply_transpose(b)
    else:
        r = precond.apply_transpose(b - op.apply(x))
    p = precond.apply(r)
    rho = float(r @ r)
    r0 = math.sqrt(rho)
    hist.residual_norms.append(r0)
    if opts.cost_eval:
        hist.quadratic_costs.append(opts.cost_eval(x))
    if keep_f and r0 > 0.0:
        hist.normalized_residuals.append(r / r0)
    if r0 == 0.0:
        hist.converged = True
        hist.stop_reason = "zero initial residual"
        return PcgResult(x, hist)
    for j in range(1, opts.max_iter + 1):
        w = op.apply(p)
        curv = float(p @ w)
        _check_finite(curv, "curvature", j)
        if curv <= 0.0:
            raise NumericalError(f"pcg_split: p^T A p = {curv} at iteration {j}; operator lost positive definiteness")
        alpha = rho / curv
        _check_finite(alpha, "alpha", j)
        x = x + alpha * p
        ct_w = precond.apply_transpose(w)
        r = r - alpha * ct_w
        if opts.reorthogonalize:
            for f in hist.normalized_residuals:
                r = r - float(f @ r) * f
        rho_next = float(r @ r)
        beta = rho_next / rho
        _check_finite(beta, "beta", j)
        hist.alphas.append(alpha)
        hist.betas.append(beta)
        hist.residual_norms.append(math.sqrt(rho_next))
        if opts.cost_eval:
            hist.quadratic_costs.append(opts.cost_eval(x))
        if keep_f and rho_next > 0.0:
            hist.normalized_residuals.append(r / math.sqrt(rho_next))
        hist.iterations = j
        if math.sqrt(rho_next) / r0 <= opts.rel_tol:
            hist.converged = True
            hist.stop_reason = "relative residual tolerance reached"
            break
        p = precond.apply(r) + beta * p
        rho = rho_next
    if not hist.converged:
        hist.stop_reason = "maximum iterations reached"
    return PcgResult(x, hist)


# ---------------------------------------------------------------------------
# Spectrum / cost (proj/src/spectrum.cpp, assimilation.cpp:130-150)
# ---------------------------------------------------------------------------
@dataclass
class ClusteredSpectrum:
    """spectrum.hpp:10-18."""

    nonunit: np.ndarray
    unit_multiplicity: int

    def min_eigenvalue(self):
        m = 1.0 if self.unit_multiplicity > 0 else math.inf
        return min(m, self.nonunit.min()) if self.nonunit.size else m

    def max_eigenvalue(self):
        m = 1.0 if self.unit_multiplicity > 0 else -math.inf
        return max(m, self.nonunit.max()) if self.nonunit.size else m

    def full(self):
        return np.sort(np.concatenate([self.nonunit, np.ones(self.unit_multiplicity)]))[::-1]


def clustered_spectrum(op: HessianOperator, precond: Optional[LmpFactor] = None,
                       obs_range: Optional[np.ndarray] = None) -> ClusteredSpectrum:
    """spectrum.cpp:31-64."""
    n = op.dim()
    W = obs_range if obs_range is not None else op.observation_range()
    k = precond.k() if (precond is not None and not precond.is_identity()) else 0
    B = np.hstack([W, precond.vectors]) if k > 0 else W
    Q = householder_q(B)
    AQ = Q
    if precond is not None:
        AQ = np.column_stack([precond.apply(Q[:, j]) for j in range(Q.shape[1])])
    AQ = op.apply_block(AQ)
    if precond is not None:
        AQ = np.column_stack([precond.apply_transpose(AQ[:, j]) for j in range(Q.shape[1])])
    K = Q.T @ AQ
    K = 0.5 * (K + K.T)
    return ClusteredSpectrum(np.linalg.eigvalsh(K)[::-1].copy(), n - Q.shape[1])


class QuadraticCost:
    """assimilation.cpp:130-150 (first-level preconditioned inner-loop cost)."""

    def __init__(self, op: HessianOperator, b, d):
        self.op = op
        self.b_tilde = op.apply_D_half_inv(b)
        self.d = _vec(d)
        require(len(self.d) == op.network().q, "QuadraticCost: innovation length mismatch")

    def __call__(self, x):
        r_inv = 1.0 / (self.op.sigma_obs() ** 2)
        traj = self.op.apply_Linv(self.op.apply_D_half(x))
        mis = observe(traj, self.op.network()) - self.d
        return 0.5 * float((x - self.b_tilde) @ (x - self.b_tilde)) + 0.5 * r_inv * float(mis @ mis)

    def rhs(self):
        r_inv = 1.0 / (self.op.sigma_obs() ** 2)
        sc = observe_adjoint(self.d, self.op.network())
        return self.b_tilde + r_inv * self.op.apply_D_half(self.op.apply_LinvT(sc))

    def gradient(self, x):
        return self.op.apply(x) - self.rhs()


# ---------------------------------------------------------------------------
# Outer loop and twin data (proj/src/assimilation.cpp:11-128, 255-263), SURVEY §8(f)-4.
# Test infrastructure: the checker for paper_2101_07249_b200/assimilation.py.
# ---------------------------------------------------------------------------
@dataclass
class AssimSystem:
    """assimilation.hpp:19-37 (plain fields; factors are oracle CovarianceFactors)."""

    kind: str          # "advection" | "lorenz96"
    n: int
    N: int
    dt: float
    dx: float
    net: ObservationNetwork
    bh: CovarianceFactor
    qh: CovarianceFactor
    sigma_obs: float
    courant: float = 0.0
    forcing: float = 8.0
    spinup_steps: int = 500

    def model_step(self, x):
        """assimilation.cpp:11-19"""
        if self.kind == "advection":
            return advection_step(x, self.courant)
        return lorenz96_step(x, self.forcing, self.dt)

    def integrate_p(self, p) -> np.ndarray:
        """assimilation.cpp:21-33"""
        n = self.n
        traj = np.empty((n, self.N + 1))
        traj[:, 0] = p[:n]
        for i in range(self.N):
            traj[:, i + 1] = self.model_step(traj[:, i]) + p[(i + 1) * n:(i + 2) * n]
            if not np.all(np.isfinite(traj[:, i + 1])):
                raise NumericalError(f"integrate_p: non-finite trajectory at step {i + 1}")
        return traj

    def hessian(self, traj, threads: int = 8) -> "HessianOperator":
        """assimilation.cpp:35-50"""
        model = (AdvectionLinearized(self.n, self.N, self.courant) if self.kind == "advection"
                 else Lorenz96Linearized(traj, self.forcing, self.dt))
        return HessianOperator(model, self.net, self.bh, self.qh, self.sigma_obs, threads=threads)


def generate_twin(sys: AssimSystem, seeds=(1, 2, 3), noise_scale: float = 1.0, truth_model_error: bool = False):
    """assimilation.cpp:75-110 (seeds = background, observations, model_error).
    Returns (truth, background, y)."""
    n = sys.n
    if sys.kind == "advection":
        x0 = np.array([6.0 * math.exp(-0.5 * ((j * sys.dx - 0.5) / 0.1) ** 2) for j in range(n)])
    else:
        x0 = np.full(n, sys.forcing)
        x0[0] += 0.01
        for _ in range(sys.spinup_steps):
            x0 = lorenz96_step(x0, sys.forcing, sys.dt)
    truth = np.empty((n, sys.N + 1))
    truth[:, 0] = x0
    mn = NormalStream(seeds[2])
    for i in range(sys.N):
        nxt = sys.model_step(truth[:, i])
        if truth_model_error and noise_scale > 0.0:
            nxt = nxt + noise_scale * sys.qh.apply(mn.draw(n))
        if not np.all(np.isfinite(nxt)):
            raise NumericalError("generate_twin: truth integration became non-finite")
        truth[:, i + 1] = nxt
    bg = truth[:, 0].copy()
    if noise_scale > 0.0:
        bg = bg + noise_scale * sys.bh.apply(NormalStream(seeds[0]).draw(n))
    y = observe(truth.reshape(-1, order="F"), sys.net)
    if noise_scale > 0.0:
        y = y + noise_scale * sys.sigma_obs * NormalStream(seeds[1]).draw(len(y))
    return truth, bg, y


def compute_innovations(sys: AssimSystem, p, traj, background, y):
    """assimilation.cpp:120-128 -> (b, d)."""
    b = -np.asarray(p, dtype=np.float64)
    b[:sys.n] = background - traj[:, 0]
    return b, y - observe(traj.reshape(-1, order="F"), sys.net)
