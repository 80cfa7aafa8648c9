"""Python mirror of the reference's operator / sketch / LMP / PCG API over the C-ABI.

Every call goes through ``libwc4dvar_gpu.so`` (include/wc4dvar_gpu.h); there is no CPU
fallback: if the library or a GPU is missing the call raises ``DeviceError``.  Names,
argument meaning and exception types follow the reference (proj/include/wc4dvar/*.hpp):
``std::invalid_argument`` -> ``ValueError``, ``NumericalError``, ``DenseCapError``.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libwc4dvar_gpu.so")


class NumericalError(RuntimeError):
    """types.hpp:19-21"""


class DenseCapError(RuntimeError):
    """types.hpp:24-26"""


class DeviceError(RuntimeError):
    """CUDA failure or missing device/library (no reference equivalent)."""


def _load():
    if not os.path.exists(LIB_PATH):
        raise DeviceError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
    return ctypes.CDLL(LIB_PATH)


lib = _load()

_dp = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p


class ModelDesc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("N", ctypes.c_int32), ("n", _i64),
                ("substeps", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("courant", ctypes.c_double), ("diffusion", ctypes.c_double),
                ("dt", ctypes.c_double), ("stages", _dp), ("trajectory", _dp), ("ld_trajectory", _i64),
                ("forcing", ctypes.c_double), ("trajectory_on_device", ctypes.c_int32),
                ("reserved2", ctypes.c_int32)]


class NetworkDesc(ctypes.Structure):
    _fields_ = [("n", _i64), ("N", ctypes.c_int32), ("n_times", ctypes.c_int32),
                ("times", _i32p), ("n_points", ctypes.c_int32), ("reserved", ctypes.c_int32),
                ("points", _i32p)]


class CovDesc(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("reserved", ctypes.c_int32), ("half", _dp),
                ("half_inv", _dp)]


class SketchDesc(ctypes.Structure):
    _fields_ = [("target_rank", ctypes.c_int32), ("oversample", ctypes.c_int32),
                ("seed", ctypes.c_uint64), ("method", ctypes.c_int32), ("p_iter", ctypes.c_int32)]


class PcgOpts(ctypes.Structure):
    _fields_ = [("max_iter", ctypes.c_int32), ("reorthogonalize", ctypes.c_int32), ("rel_tol", ctypes.c_double),
                ("store_residual_vectors", ctypes.c_int32), ("reserved", ctypes.c_int32)]


class PcgHist(ctypes.Structure):
    _fields_ = [("alphas", _dp), ("betas", _dp), ("residual_norms", _dp),
                ("quadratic_costs", _dp), ("iterations", ctypes.c_int32),
                ("converged", ctypes.c_int32), ("stop_reason", ctypes.c_int32),
                ("reserved", ctypes.c_int32), ("normalized_residuals", _dp), ("ld_residuals", _i64),
                ("n_residuals", ctypes.c_int32), ("reserved2", ctypes.c_int32)]


class LanczosOpts(ctypes.Structure):
    _fields_ = [("max_iter", ctypes.c_int32), ("reserved", ctypes.c_int32), ("tol", ctypes.c_double),
                ("seed", ctypes.c_uint64)]


# Every entry point of include/wc4dvar_gpu.h with its ctypes signature.
SIGNATURES = {
    "wc4dvar_gpu_last_error": (ctypes.c_char_p, []),
    "wc4dvar_gpu_version": (ctypes.c_char_p, []),
    "wc4dvar_gpu_hessian_create": (ctypes.c_int, [ctypes.POINTER(ModelDesc), ctypes.POINTER(NetworkDesc),
                                                  ctypes.POINTER(CovDesc), ctypes.POINTER(CovDesc),
                                                  ctypes.c_double, ctypes.c_int, ctypes.POINTER(_vp)]),
    "wc4dvar_gpu_dense_create": (ctypes.c_int, [_i64, _dp, _i64, ctypes.c_int, ctypes.POINTER(_vp)]),
    "wc4dvar_gpu_op_destroy": (ctypes.c_int, [_vp]),
    "wc4dvar_gpu_op_dim": (_i64, [_vp]),
    "wc4dvar_gpu_op_apply_count": (_i64, [_vp]),
    "wc4dvar_gpu_op_reset_apply_count": (None, [_vp]),
    "wc4dvar_gpu_op_device": (ctypes.c_int, [_vp]),
    "wc4dvar_gpu_op_apply": (ctypes.c_int, [_vp, _dp, _dp]),
    "wc4dvar_gpu_op_apply_block": (ctypes.c_int, [_vp, _dp, _i64, _i64, _dp, _i64]),
    "wc4dvar_gpu_op_apply_block_dev": (ctypes.c_int, [_vp, _vp, _i64, _i64, _vp, _i64, _vp]),
    "wc4dvar_gpu_hessian_piece": (ctypes.c_int, [_vp, ctypes.c_int, _dp, _i64, _i64, _dp, _i64]),
    "wc4dvar_gpu_hessian_piece_dev": (ctypes.c_int, [_vp, ctypes.c_int, _vp, _i64, _i64, _vp, _i64, _vp]),
    "wc4dvar_gpu_observe": (ctypes.c_int, [_vp, _dp, _dp]),
    "wc4dvar_gpu_observe_dev": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "wc4dvar_gpu_observation_range": (ctypes.c_int, [_vp, _dp, _i64]),
    "wc4dvar_gpu_observation_range_dev": (ctypes.c_int, [_vp, _vp, _i64, _vp]),
    "wc4dvar_gpu_clustered_spectrum": (ctypes.c_int, [_vp, _vp, _dp, _i64, _dp, ctypes.POINTER(_i64),
                                                      ctypes.POINTER(_i64)]),
    "wc4dvar_gpu_op_spectral": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.POINTER(ctypes.c_int)]),
    "wc4dvar_gpu_op_profile": (ctypes.c_int, [_vp, ctypes.c_int]),
    "wc4dvar_gpu_op_profile_read": (ctypes.c_int, [_vp, _dp, ctypes.POINTER(_i64)]),
    "wc4dvar_gpu_probe_dmma_peak": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(ctypes.c_double)]),
    "wc4dvar_gpu_gaussian_matrix": (ctypes.c_int, [_i64, _i64, ctypes.c_uint64, _dp]),
    "wc4dvar_gpu_l96_trajectory": (ctypes.c_int, [_i64, ctypes.c_double, ctypes.c_double, _dp, _i64, _i64, _dp,
                                                  _i64, ctypes.c_int]),
    "wc4dvar_gpu_l96_trajectory_dev": (ctypes.c_int, [_i64, ctypes.c_double, ctypes.c_double, _vp, _i64, _i64,
                                                      _vp, _i64, ctypes.c_int, _vp]),
    "wc4dvar_gpu_l96_integrate_p": (ctypes.c_int, [_i64, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                                   ctypes.c_double, _dp, _dp, _i64, ctypes.c_int]),
    "wc4dvar_gpu_sketch": (ctypes.c_int, [_vp, ctypes.POINTER(SketchDesc), _dp, _dp, _i64, _dp,
                                          ctypes.POINTER(_i64)]),
    "wc4dvar_gpu_launch_count": (ctypes.c_int64, []),
    "wc4dvar_gpu_factor_apply_dev": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, _i64, _i64, _vp, _i64, _vp]),
    "wc4dvar_gpu_op_release_workspaces": (ctypes.c_int, [_vp]),
    "wc4dvar_gpu_gaussian_block_dev": (ctypes.c_int, [_i64, _i64, _i64, _i64, _i64, ctypes.c_uint64, _vp, _i64,
                                                      ctypes.c_int, _vp]),
    "wc4dvar_gpu_mt19937_raw_dev": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, _i64, _vp, ctypes.c_int, _vp]),
    "wc4dvar_gpu_mt19937_raw_host": (ctypes.c_int, [ctypes.c_uint64, ctypes.c_uint64, _i64, _vp]),
    "wc4dvar_gpu_sketch_dev": (ctypes.c_int, [_vp, ctypes.POINTER(SketchDesc), _vp, _vp, _i64, _vp,
                                              ctypes.POINTER(_i64), _vp]),
    "wc4dvar_gpu_rayleigh_ritz": (ctypes.c_int, [_vp, _dp, _i64, _i64, _dp, _i64, _dp]),
    "wc4dvar_gpu_last_sketch_timing": (ctypes.c_int, [_dp]),
    "wc4dvar_gpu_la_gram_dev": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i64, _vp, _i64, _vp, _i64,
                                               _vp, _i64, _vp]),
    "wc4dvar_gpu_la_tall_times_small_dev": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _i64, _vp, _i64,
                                                           _vp, _i64, _vp, _i64, _vp]),
    "wc4dvar_gpu_la_chol_upper_dev": (ctypes.c_int, [ctypes.c_int, _i64, _vp, _vp, _vp]),
    "wc4dvar_gpu_la_chol_inv_upper_dev": (ctypes.c_int, [ctypes.c_int, _i64, _vp, _vp, _vp, _vp]),
    "wc4dvar_gpu_la_tri_inv_upper_dev": (ctypes.c_int, [ctypes.c_int, _i64, _vp, _vp, _vp]),
    "wc4dvar_gpu_la_pivoted_rank_dev": (ctypes.c_int, [ctypes.c_int, _i64, _vp, ctypes.c_double,
                                                       ctypes.POINTER(_i64), _vp, _vp]),
    "wc4dvar_gpu_la_sym_evd_dev": (ctypes.c_int, [ctypes.c_int, _i64, _vp, _vp, _vp, _vp]),
    "wc4dvar_gpu_la_svd_left_dev": (ctypes.c_int, [ctypes.c_int, _i64, _vp, _vp, _vp, _vp]),
    "wc4dvar_gpu_la_small_gemm_dev": (ctypes.c_int, [ctypes.c_int, ctypes.c_int32, ctypes.c_int32, _i64,
                                                     _i64, _i64, ctypes.c_double, _vp, _i64, _vp, _i64,
                                                     ctypes.c_double, _vp, _i64, _vp]),
    "wc4dvar_gpu_la_gather_cols_dev": (ctypes.c_int, [ctypes.c_int, _i64, _i64, _vp, _i64, _vp, _vp,
                                                      _i64, _vp]),
    "wc4dvar_gpu_lmp_build": (ctypes.c_int, [_i64, _i64, _dp, _i64, _dp, ctypes.c_int, ctypes.POINTER(_vp)]),
    "wc4dvar_gpu_lmp_build_dev": (ctypes.c_int, [_i64, _i64, _vp, _i64, _vp, ctypes.c_int, ctypes.POINTER(_vp)]),
    "wc4dvar_gpu_lmp_destroy": (ctypes.c_int, [_vp]),
    "wc4dvar_gpu_lmp_apply": (ctypes.c_int, [_vp, ctypes.c_int, _dp, _dp]),
    "wc4dvar_gpu_cost_create": (ctypes.c_int, [_vp, _dp, _dp, ctypes.POINTER(_vp)]),
    "wc4dvar_gpu_cost_destroy": (ctypes.c_int, [_vp]),
    "wc4dvar_gpu_cost_eval": (ctypes.c_int, [_vp, _dp, _dp]),
    "wc4dvar_gpu_cost_rhs": (ctypes.c_int, [_vp, _dp]),
    "wc4dvar_gpu_pcg": (ctypes.c_int, [_vp, _dp, _vp, _dp, ctypes.POINTER(PcgOpts), _vp, _dp,
                                       ctypes.POINTER(PcgHist)]),
    "wc4dvar_gpu_comm_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "wc4dvar_gpu_comm_create": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                               ctypes.POINTER(_vp)]),
    "wc4dvar_gpu_comm_destroy": (ctypes.c_int, [_vp]),
    "wc4dvar_gpu_comm_allreduce_sum": (ctypes.c_int, [_vp, _vp, _i64, _vp]),
    "wc4dvar_gpu_comm_allgather": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp]),
    "wc4dvar_gpu_comm_cols_to_rows": (ctypes.c_int, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "wc4dvar_gpu_comm_rows_to_cols": (ctypes.c_int, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "wc4dvar_gpu_lanczos_eigenpairs": (ctypes.c_int, [_vp, _i64, ctypes.POINTER(LanczosOpts), _dp, _i64, _dp,
                                                      ctypes.POINTER(_i64)]),
    "wc4dvar_gpu_ritz_from_tridiagonal": (ctypes.c_int, [_i64, _i64, _dp, _dp, _dp, _i64, _i64, _dp, _i64, _dp,
                                                         ctypes.c_int]),
}
for _name, (_res, _args) in SIGNATURES.items():
    _f = getattr(lib, _name)
    _f.restype = _res
    _f.argtypes = _args


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = (lib.wc4dvar_gpu_last_error() or b"").decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise NumericalError(msg)
    if rc == 4:
        raise DenseCapError(msg)
    raise DeviceError(msg)


def require(cond: bool, what: str) -> None:
    if not cond:
        raise ValueError(what)


def _fcol(a) -> np.ndarray:
    a = np.asarray(a, dtype=np.float64)
    if a.ndim == 1:
        return np.ascontiguousarray(a)
    return np.asfortranarray(a)


def _p(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(_dp)


def version() -> str:
    return lib.wc4dvar_gpu_version().decode()


def probe_dmma_peak(device: int = 0) -> float:
    """Sustained fp64 DMMA TFLOP/s of this device (all-SM mma.sync.f64 loop)."""
    v = ctypes.c_double(0)
    _check(lib.wc4dvar_gpu_probe_dmma_peak(device, ctypes.byref(v)))
    return v.value


def gaussian_matrix(rows: int, cols: int, seed: int) -> np.ndarray:
    """randevd.cpp:16-21 (bit-exact NormalStream, column-major fill)."""
    out = np.empty((rows, cols), dtype=np.float64, order="F")
    _check(lib.wc4dvar_gpu_gaussian_matrix(rows, cols, ctypes.c_uint64(seed & (2 ** 64 - 1)), _p(out)))
    return out


# ---------------------------------------------------------------------------
# Descriptors (models.hpp, covariance.hpp, operators.hpp)
# ---------------------------------------------------------------------------
def launch_count() -> int:
    """Kernel launches issued by the library so far (wc4dvar_gpu_launch_count)."""
    return int(lib.wc4dvar_gpu_launch_count())


def gaussian_block_dev(out, n_total: int, seed: int, row0: int = 0, col0: int = 0, stream=None) -> None:
    """Device NormalStream with jump-ahead (wc4dvar_gpu_gaussian_block_dev): fills the torch
    CUDA tensor ``out`` (shape (cols, rows), row j = column col0 + j of the column-major
    sketch) with rows [row0, row0 + rows) of columns [col0, col0 + cols) of
    gaussian_matrix(n_total, *, seed) (randevd.cpp:16-21)."""
    cols, rows = out.shape
    require(out.stride(1) == 1, "gaussian_block_dev: rows must be contiguous")
    _check(lib.wc4dvar_gpu_gaussian_block_dev(n_total, row0, rows, col0, cols, seed, out.data_ptr(),
                                              out.stride(0) if cols > 1 else rows, out.device.index,
                                              None if stream is None else stream))


def mt19937_raw_host(seed: int, offset: int, count: int) -> np.ndarray:
    """Raw std::mt19937_64(seed) outputs from draw `offset` via the library's host jump-ahead."""
    out = np.empty(count, dtype=np.uint64)
    _check(lib.wc4dvar_gpu_mt19937_raw_host(seed, offset, count, out.ctypes.data_as(_vp)))
    return out


def mt19937_raw_dev(seed: int, offset: int, count: int, device: int = 0) -> np.ndarray:
    """Raw outputs generated on the device from a jump-ahead state (test hook)."""
    import torch
    t = torch.empty(count, dtype=torch.int64, device=f"cuda:{device}")
    _check(lib.wc4dvar_gpu_mt19937_raw_dev(seed, offset, count, t.data_ptr(), device, None))
    torch.cuda.synchronize(device)
    return t.cpu().numpy().view(np.uint64)


@dataclass
class ObservationNetwork:
    """models.hpp:45-56; build rule of models.cpp:159-176."""

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
        return ObservationNetwork(n, N, 1, 1, [], [], 0)


@dataclass
class CovarianceFactor:
    """covariance.hpp:31-38: dense symmetric square root and its inverse.  kind='circulant'
    (EXTENSION) stores first columns instead of n x n matrices."""

    half: np.ndarray
    half_inv: Optional[np.ndarray] = None
    kind: str = "dense"

    def dim(self) -> int:
        return self.half.shape[0]


@dataclass
class LinearizedModel:
    """operators.hpp:57-111 plus the EXTENSION kinds (advdiff, sub-steps)."""

    kind: str
    n: int
    N: int
    substeps: int = 1
    courant: float = 0.0
    diffusion: float = 0.0
    dt: float = 0.0
    stages: Optional[np.ndarray] = None
    trajectory: Optional[object] = None  # L96: n x (N s + 1) numpy array or device tensor (steps+1, n)
    forcing: float = 0.0


def IdentityLinearized(n: int, N: int) -> LinearizedModel:
    return LinearizedModel("identity", n, N)


def AdvectionLinearized(n: int, N: int, courant: float) -> LinearizedModel:
    require(n >= 1 and N >= 0, "AdvectionLinearized: bad window")
    return LinearizedModel("advection", n, N, 1, courant)


def AdvDiffLinearized(n: int, N: int, courant: float, diffusion: float, substeps: int = 1):
    require(n >= 1 and N >= 0 and substeps >= 1, "AdvDiffLinearized: bad window")
    return LinearizedModel("advdiff", n, N, substeps, courant, diffusion)


def Lorenz96Linearized(trajectory, forcing: float, dt: float, substeps: int = 1):
    """operators.cpp:44-51: the operator stores the RK4 stages of every trajectory column;
    the library computes them on the device at construction (wc4dvar_model_desc.trajectory).
    ``trajectory`` is an n x (N*s+1) host array, or a device tensor of shape (N*s+1, n)
    (each row one state, i.e. the same column-major block) from lorenz96_trajectory_device;
    s = 1 is the reference."""
    if isinstance(trajectory, np.ndarray) or not hasattr(trajectory, "data_ptr"):
        trajectory = np.asfortranarray(trajectory, dtype=np.float64)
        require(trajectory.ndim == 2 and trajectory.shape[1] >= 2, "Lorenz96Linearized: trajectory too short")
        n, total = trajectory.shape[0], trajectory.shape[1] - 1
    else:
        require(trajectory.dim() == 2 and trajectory.shape[0] >= 2, "Lorenz96Linearized: trajectory too short")
        require(trajectory.is_contiguous(), "Lorenz96Linearized: device trajectory must be contiguous")
        n, total = trajectory.shape[1], trajectory.shape[0] - 1
    require(total % substeps == 0, "Lorenz96Linearized: trajectory/sub-step mismatch")
    return LinearizedModel("l96", n, total // substeps, substeps, dt=dt, trajectory=trajectory, forcing=forcing)


def lorenz96_trajectory(x0, forcing: float, dt: float, spinup: int, steps: int, device: int = 0) -> np.ndarray:
    """Spin x0 up for `spinup` RK4 steps (lorenz96_step, models.cpp:72-78), then return the
    next `steps` + 1 states as an n x (steps+1) host array; integrated on the device
    (wc4dvar_gpu_l96_trajectory), bitwise equal to the reference arithmetic."""
    x0 = np.ascontiguousarray(x0, dtype=np.float64)
    n = len(x0)
    traj = np.empty((n, steps + 1), order="F")
    _check(lib.wc4dvar_gpu_l96_trajectory(n, forcing, dt, _p(x0), spinup, steps, _p(traj), n, device))
    return traj


def lorenz96_trajectory_device(x0, forcing: float, dt: float, spinup: int, steps: int, device: int = 0):
    """lorenz96_trajectory kept on the device: a (steps+1, n) float64 tensor (row c = state c),
    ready for Lorenz96Linearized without a host round trip."""
    import torch
    x0 = torch.as_tensor(np.ascontiguousarray(x0, dtype=np.float64)).to(f"cuda:{device}")
    n = x0.numel()
    traj = torch.empty((steps + 1, n), dtype=torch.float64, device=x0.device)
    stream = torch.cuda.current_stream(x0.device)
    _check(lib.wc4dvar_gpu_l96_trajectory_dev(n, forcing, dt, ctypes.c_void_p(x0.data_ptr()), spinup, steps,
                                              ctypes.c_void_p(traj.data_ptr()), n, device,
                                              ctypes.c_void_p(stream.cuda_stream)))
    return traj


def integrate_p(p, n: int, N: int, forcing: float, dt: float, substeps: int = 1, device: int = 0) -> np.ndarray:
    """AssimilationSystem::integrate_p (assimilation.cpp:21-33) for Lorenz-96, on the device:
    x_0 = p_0, x_{i+1} = M^s(x_i) + p_{i+1}; returns every sub-step state, n x (N s + 1)
    (s = 1: the reference's n x (N+1)).  NumericalError on a non-finite interval end."""
    p = np.ascontiguousarray(p, dtype=np.float64)
    require(p.size == n * (N + 1), "integrate_p: control vector length mismatch")
    traj = np.empty((n, N * substeps + 1), order="F")
    _check(lib.wc4dvar_gpu_l96_integrate_p(n, N, substeps, forcing, dt, _p(p), _p(traj), n, device))
    return traj


_MODEL_KIND = {"identity": 0, "advection": 1, "advdiff": 2, "l96": 3}


class LinearOperator:
    """operators.hpp:15-40 over a C-ABI handle."""

    def __init__(self, handle, keep=()):
        self._h = handle
        self._keep = list(keep)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # the module global is gone at interpreter shutdown
            lib.wc4dvar_gpu_op_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def dim(self) -> int:
        return int(lib.wc4dvar_gpu_op_dim(self._h))

    def device(self) -> int:
        return int(lib.wc4dvar_gpu_op_device(self._h))

    def apply_count(self) -> int:
        return int(lib.wc4dvar_gpu_op_apply_count(self._h))

    def reset_apply_count(self) -> None:
        lib.wc4dvar_gpu_op_reset_apply_count(self._h)

    def apply(self, v) -> np.ndarray:
        v = np.ascontiguousarray(v, dtype=np.float64)
        require(v.ndim == 1 and len(v) == self.dim(), f"{type(self).__name__}::apply: dimension mismatch")
        out = np.empty_like(v)
        _check(lib.wc4dvar_gpu_op_apply(self._h, _p(v), _p(out)))
        return out

    def apply_block(self, V) -> np.ndarray:
        """operators.cpp:9-19 (counts m applies)."""
        V = _fcol(V)
        require(V.ndim == 2 and V.shape[0] == self.dim(), "LinearOperator::apply_block: dimension mismatch")
        out = np.empty_like(V, order="F")
        _check(lib.wc4dvar_gpu_op_apply_block(self._h, _p(V), V.shape[0], V.shape[1], _p(out),
                                              out.shape[0]))
        return out

    def release_workspaces(self) -> None:
        """Free the operator's grow-only device workspaces (wc4dvar_gpu_op_release_workspaces)."""
        _check(lib.wc4dvar_gpu_op_release_workspaces(self._h))

    def spectral(self, mode: int = -1) -> bool:
        """Fourier-space apply (wc4dvar_gpu_op_spectral): mode 1 / 0 switches it on / off,
        -1 queries; returns whether it is active."""
        active = ctypes.c_int(0)
        _check(lib.wc4dvar_gpu_op_spectral(self._h, int(mode), ctypes.byref(active)))
        return bool(active.value)

    def profile(self, enable: bool = True) -> None:
        _check(lib.wc4dvar_gpu_op_profile(self._h, int(enable)))

    def profile_read(self):
        """(ms per stage summed over calls [D^1/2 GEMM, sweep, D^1/2 GEMM + I], calls)."""
        ms = np.zeros(3)
        calls = _i64(0)
        _check(lib.wc4dvar_gpu_op_profile_read(self._h, _p(ms), ctypes.byref(calls)))
        return ms, calls.value

    def apply_block_host_ptr(self, V_ptr: int, ldv: int, m: int, out_ptr: int, ldo: int) -> None:
        """apply_block on raw HOST pointers (e.g. pinned torch tensors): the e2e path."""
        _check(lib.wc4dvar_gpu_op_apply_block(self._h, ctypes.cast(V_ptr, _dp), ldv, m,
                                              ctypes.cast(out_ptr, _dp), ldo))

    def apply_block_dev(self, V, out, stream=None) -> None:
        """Device-resident block apply on torch CUDA tensors (column-major views:
        pass ``V.T`` of a row-major (m, dim) tensor, i.e. column j = V[j])."""
        m, dim = V.shape
        require(dim == self.dim() and tuple(out.shape) == (m, dim), "apply_block_dev: shape mismatch")
        _check(lib.wc4dvar_gpu_op_apply_block_dev(self._h, V.data_ptr(), V.stride(0), m,
                                                  out.data_ptr(), out.stride(0),
                                                  None if stream is None else stream))


class DenseOperator(LinearOperator):
    """operators.hpp:42-53."""

    def __init__(self, A, device: int = 0):
        A = np.asfortranarray(A, dtype=np.float64)
        require(A.ndim == 2 and A.shape[0] == A.shape[1], "DenseOperator: matrix must be square")
        h = _vp()
        _check(lib.wc4dvar_gpu_dense_create(A.shape[0], _p(A), A.shape[0], device, ctypes.byref(h)))
        super().__init__(h)
        self.A = A

    def matrix(self):
        return self.A


class HessianOperator(LinearOperator):
    """operators.hpp:116-152: A = I + D^{1/2} L^{-T} H^T R^{-1} H L^{-1} D^{1/2}."""

    def __init__(self, model: LinearizedModel, net: ObservationNetwork,
                 background_half: CovarianceFactor, model_error_half: CovarianceFactor,
                 sigma_obs: float, device: int = 0):
        require(sigma_obs > 0.0, "HessianOperator: sigma_obs must be positive")
        require(background_half is not None and background_half.dim() == model.n,
                "HessianOperator: background factor mismatch")
        require(model_error_half is not None and model_error_half.dim() == model.n,
                "HessianOperator: model-error factor mismatch")
        require(net.n == model.n and net.N == model.N, "HessianOperator: network/window mismatch")
        keep = []

        def arr(a, dtype=np.float64):
            if a is None:
                return None
            a = np.asfortranarray(a, dtype=dtype)
            keep.append(a)
            return a

        md = ModelDesc()
        md.kind = _MODEL_KIND[model.kind]
        md.N, md.n, md.substeps = model.N, model.n, model.substeps
        md.courant, md.diffusion, md.dt = model.courant, model.diffusion, model.dt
        st = arr(model.stages)
        md.stages = _p(st)
        tr = model.trajectory
        if tr is not None and st is None:
            if isinstance(tr, np.ndarray):
                tr = arr(tr)
                md.trajectory, md.ld_trajectory, md.trajectory_on_device = _p(tr), tr.shape[0], 0
            else:
                require(tr.device.index == device, "HessianOperator: trajectory on another device")
                keep.append(tr)
                md.trajectory = ctypes.cast(ctypes.c_void_p(tr.data_ptr()), _dp)
                md.ld_trajectory, md.trajectory_on_device = tr.shape[1], 1
                import torch
                torch.cuda.current_stream(tr.device).synchronize()  # the library uses its own stream
            md.forcing = model.forcing
        nd = NetworkDesc()
        times = arr(np.asarray(net.times, dtype=np.int32), np.int32)
        points = arr(np.asarray(net.points, dtype=np.int32), np.int32)
        nd.n, nd.N = net.n, net.N
        nd.n_times, nd.times = len(net.times), times.ctypes.data_as(_i32p)
        nd.n_points, nd.points = len(net.points), points.ctypes.data_as(_i32p)
        covs = []
        for f in (background_half, model_error_half):
            c = CovDesc()
            c.kind = 0 if f.kind == "dense" else 1
            c.half = _p(arr(f.half))
            c.half_inv = _p(arr(f.half_inv))
            covs.append(c)
        h = _vp()
        _check(lib.wc4dvar_gpu_hessian_create(ctypes.byref(md), ctypes.byref(nd), ctypes.byref(covs[0]),
                                              ctypes.byref(covs[1]), sigma_obs, device, ctypes.byref(h)))
        super().__init__(h)
        self.model, self.net = model, net
        self.sigma_obs_ = sigma_obs

    def network(self) -> ObservationNetwork:
        return self.net

    def sigma_obs(self) -> float:
        return self.sigma_obs_

    def state_size(self) -> int:
        return self.model.n

    def window_steps(self) -> int:
        return self.model.N

    def _piece(self, which: int, name: str, v):
        v = _fcol(v)
        require(v.shape[0] == self.dim(), f"{name}: window length mismatch")
        m = 1 if v.ndim == 1 else v.shape[1]
        out = np.empty_like(v)
        _check(lib.wc4dvar_gpu_hessian_piece(self._h, which, _p(v), v.shape[0], m, _p(out), v.shape[0]))
        return out

    def sweeps(self, v):
        """L^{-T} H^T R^{-1} H L^{-1} v: the middle of apply (operators.cpp:132-141), no D^{1/2}."""
        return self._piece(4, "sweeps", v)

    def piece_dev(self, which: int, V, out, stream=None) -> None:
        """Device-resident hessian piece (0 Linv, 1 LinvT, 2 D^{1/2}, 3 D^{-1/2}, 4 sweeps) on
        torch CUDA tensors in the (columns, rows) layout."""
        m, dim = V.shape
        require(dim == self.dim() and tuple(out.shape) == (m, dim), "hessian piece: shape mismatch")
        _check(lib.wc4dvar_gpu_hessian_piece_dev(self._h, which, V.data_ptr(), V.stride(0) if m > 1 else dim, m,
                                                 out.data_ptr(), out.stride(0) if m > 1 else dim,
                                                 None if stream is None else stream))

    def factor_apply_dev(self, which: int, inv: bool, X, out, stream=None) -> None:
        """B^{1/2} (which 0) or Q^{1/2} (which 1), or their inverses, on the rows of the torch
        CUDA tensor X (c, n) -> out (c, n) (wc4dvar_gpu_factor_apply_dev)."""
        c, n = X.shape
        require(n == self.state_size() and tuple(out.shape) == (c, n), "factor apply: shape mismatch")
        _check(lib.wc4dvar_gpu_factor_apply_dev(self._h, which, int(inv), X.data_ptr(), X.stride(0) if c > 1 else n,
                                                c, out.data_ptr(), out.stride(0) if c > 1 else n,
                                                None if stream is None else stream))

    def observe(self, traj) -> np.ndarray:
        """observe (models.cpp:184-192) with this operator's network, on the device."""
        traj = np.ascontiguousarray(np.asarray(traj, dtype=np.float64).reshape(-1, order="F"))
        require(len(traj) == self.dim(), "observe: trajectory length mismatch")
        y = np.empty(self.net.q)
        if self.net.q:
            _check(lib.wc4dvar_gpu_observe(self.handle, _p(traj), _p(y)))
        return y

    def observation_range(self) -> np.ndarray:
        """operators.cpp:146-154: D^{1/2} L^{-T} H^T [e_1..e_q] (dim x q), one block
        adjoint sweep on the device."""
        q = self.net.q
        W = np.empty((self.dim(), q), order="F")
        if q:
            _check(lib.wc4dvar_gpu_observation_range(self.handle, _p(W), self.dim()))
        return W

    def apply_Linv(self, p):
        """operators.cpp:79-89 (vector or block)."""
        return self._piece(0, "apply_Linv", p)

    def apply_LinvT(self, v):
        """operators.cpp:91-101."""
        return self._piece(1, "apply_LinvT", v)

    def apply_D_half(self, v):
        """operators.cpp:103-113."""
        return self._piece(2, "apply_D_half", v)

    def apply_D_half_inv(self, v):
        """operators.cpp:115-125."""
        return self._piece(3, "apply_D_half_inv", v)


def assemble_dense(op: LinearOperator, cap: int = 4096) -> np.ndarray:
    """operators.cpp:156-164."""
    if op.dim() > cap:
        raise DenseCapError(f"assemble_dense: dimension {op.dim()} exceeds cap {cap}")
    A = op.apply_block(np.eye(op.dim(), order="F"))
    return 0.5 * (A + A.T)


# ---------------------------------------------------------------------------
# Sketches (randevd.hpp / ritz.hpp)
# ---------------------------------------------------------------------------
_METHOD = {"revd": 0, "nystrom": 1, "ritzit": 2}


@dataclass
class SketchConfig:
    """randevd.hpp:13-21 (+ p_iter EXTENSION)."""

    target_rank: int = 1
    oversample: int = 5
    seed: int = 0
    method: str = "revd"
    p_iter: int = 1

    def sample_size(self) -> int:
        return self.target_rank + self.oversample

    def _desc(self) -> SketchDesc:
        d = SketchDesc()
        d.target_rank, d.oversample = self.target_rank, self.oversample
        d.seed = self.seed & (2 ** 64 - 1)
        require(self.method in _METHOD, "sketch_eigenpairs: unknown method")
        d.method = _METHOD[self.method]
        d.p_iter = self.p_iter
        return d


@dataclass
class RitzPairs:
    """ritz.hpp:9-27."""

    vectors: np.ndarray
    values: np.ndarray
    source: str = "exact"

    def k(self) -> int:
        return len(self.values)

    def dim(self) -> int:
        return self.vectors.shape[0]

    def orthonormality_defect(self) -> float:
        if self.k() == 0:
            return 0.0
        return float(np.abs(self.vectors.T @ self.vectors - np.eye(self.k())).max())

    def validate(self, tol: float = 1e-10) -> None:
        """ritz.cpp:7-20."""
        require(self.vectors.shape[1] == len(self.values), "RitzPairs: U/Theta size mismatch")
        if np.any(self.values[:-1] < self.values[1:]):
            raise NumericalError("RitzPairs: values are not decreasing")
        if self.k() > 0 and self.values.min() <= 0.0:
            raise NumericalError("RitzPairs: nonpositive Ritz value")
        d = self.orthonormality_defect()
        if d > tol:
            raise NumericalError(f"RitzPairs: vectors not orthonormal (defect {d})")


def sketch_eigenpairs(op: LinearOperator, cfg: SketchConfig, omega: Optional[np.ndarray] = None) -> RitzPairs:
    """randevd.cpp:138-148; ``omega`` defaults to gaussian_matrix(dim, k+l, cfg.seed)."""
    n = op.dim()
    d = cfg._desc()
    U = np.empty((n, max(cfg.target_rank, 0)), order="F")
    th = np.empty(max(cfg.target_rank, 0))
    kout = _i64(0)
    om = None if omega is None else _fcol(omega)
    if om is not None:
        require(om.shape == (n, cfg.sample_size()), "sketch: omega shape mismatch")
    _check(lib.wc4dvar_gpu_sketch(op.handle, ctypes.byref(d), _p(om), _p(U), n, _p(th), ctypes.byref(kout)))
    k = kout.value
    return RitzPairs(U[:, :k].copy(order="F"), th[:k].copy(), cfg.method if cfg.method != "ritzit" else "ritzit")


def sketch_eigenpairs_dev(op: LinearOperator, cfg: SketchConfig, omega, U, theta, stream=None) -> int:
    """Device-resident sketch_eigenpairs (wc4dvar_gpu_sketch_dev) on torch CUDA tensors in the
    (columns, rows) layout: omega (k+l, dim), U (>= k, dim), theta (>= k).  Returns the number
    of pairs written (Nystrom caps it at the detected rank)."""
    d = cfg._desc()
    n = op.dim()
    require(tuple(omega.shape) == (cfg.sample_size(), n) and omega.stride(1) == 1, "sketch: omega shape mismatch")
    require(U.shape[1] == n and U.shape[0] >= cfg.target_rank and U.stride(1) == 1, "sketch: U shape mismatch")
    kout = _i64(0)
    _check(lib.wc4dvar_gpu_sketch_dev(op.handle, ctypes.byref(d), omega.data_ptr(), U.data_ptr(), U.stride(0),
                                      theta.data_ptr(), ctypes.byref(kout), None if stream is None else stream))
    return kout.value


def revd(op, cfg, omega=None):
    """randevd.cpp:62-80."""
    return sketch_eigenpairs(op, SketchConfig(cfg.target_rank, cfg.oversample, cfg.seed, "revd", cfg.p_iter), omega)


def nystrom(op, cfg, omega=None):
    """randevd.cpp:82-114."""
    return sketch_eigenpairs(op, SketchConfig(cfg.target_rank, cfg.oversample, cfg.seed, "nystrom", cfg.p_iter), omega)


def revd_ritzit(op, cfg, omega=None):
    """randevd.cpp:116-136."""
    return sketch_eigenpairs(op, SketchConfig(cfg.target_rank, cfg.oversample, cfg.seed, "ritzit", cfg.p_iter), omega)


def rayleigh_ritz(op: LinearOperator, Z) -> RitzPairs:
    """randevd.cpp:47-60."""
    Z = _fcol(Z)
    require(Z.shape[0] == op.dim(), "rayleigh_ritz: dimension mismatch")
    m = Z.shape[1]
    U = np.empty_like(Z, order="F")
    th = np.empty(m)
    _check(lib.wc4dvar_gpu_rayleigh_ritz(op.handle, _p(Z), Z.shape[0], m, _p(U), U.shape[0], _p(th)))
    return RitzPairs(U, th, "revd")


def last_sketch_timing() -> dict:
    t = np.zeros(5)
    _check(lib.wc4dvar_gpu_last_sketch_timing(_p(t)))
    return dict(zip(("apply_ms", "orth_ms", "small_ms", "gemm_ms", "total_ms"), t.tolist()))


# ---------------------------------------------------------------------------
# LMP (lmp.hpp)
# ---------------------------------------------------------------------------
class LmpFactor:
    """lmp.hpp:12-26, held on device in compact-WY form."""

    def __init__(self, handle, n: int, vectors: np.ndarray, values: np.ndarray):
        self._h = handle
        self.n = n
        self.vectors = vectors
        self.values = values

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # the module global is gone at interpreter shutdown
            lib.wc4dvar_gpu_lmp_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def k(self) -> int:
        return len(self.values)

    def dim(self) -> int:
        return self.n

    def is_identity(self) -> bool:
        return self.k() == 0

    def _run(self, transpose: int, v):
        v = np.ascontiguousarray(v, dtype=np.float64)
        require(self.is_identity() or len(v) == self.dim(), "LmpFactor::apply: dimension mismatch")
        out = np.empty_like(v)
        _check(lib.wc4dvar_gpu_lmp_apply(self._h, transpose, _p(v), _p(out)) if not self.is_identity()
               else 0)
        if self.is_identity():
            out[:] = v
        return out

    def apply(self, v):
        """C v (lmp.cpp:8-16)."""
        return self._run(0, v)

    def apply_transpose(self, v):
        """C^T v (lmp.cpp:18-26)."""
        return self._run(1, v)

    @staticmethod
    def identity(n: int, device: int = 0) -> "LmpFactor":
        h = _vp()
        _check(lib.wc4dvar_gpu_lmp_build(n, 0, None, n, None, device, ctypes.byref(h)))
        return LmpFactor(h, n, np.zeros((n, 0), order="F"), np.zeros(0))


def build_spectral_lmp(pairs: RitzPairs, device: int = 0) -> LmpFactor:
    """lmp.cpp:35-52."""
    U = _fcol(pairs.vectors)
    th = np.ascontiguousarray(pairs.values, dtype=np.float64)
    h = _vp()
    _check(lib.wc4dvar_gpu_lmp_build(U.shape[0], len(th), _p(U) if len(th) else None, U.shape[0],
                                     _p(th) if len(th) else None, device, ctypes.byref(h)))
    return LmpFactor(h, U.shape[0], U, th)


def build_spectral_lmp_dev(U, theta, k: int, device: int = 0) -> LmpFactor:
    """build_spectral_lmp (lmp.cpp:35-52) from device-resident Ritz pairs: torch CUDA tensors
    U (>= k, dim) (row j = vector j) and theta (>= k); the factor copies them."""
    n = U.shape[1]
    require(U.stride(1) == 1, "build_spectral_lmp: U rows must be contiguous")
    h = _vp()
    _check(lib.wc4dvar_gpu_lmp_build_dev(n, k, U.data_ptr() if k else None, U.stride(0),
                                         theta.data_ptr() if k else None, device, ctypes.byref(h)))
    return LmpFactor(h, n, None, np.zeros(k))


# ---------------------------------------------------------------------------
# Cost and PCG (assimilation.hpp:82-97, krylov.hpp)
# ---------------------------------------------------------------------------
class QuadraticCost:
    """assimilation.cpp:130-150."""

    def __init__(self, op: HessianOperator, b, d):
        b = np.ascontiguousarray(b, dtype=np.float64)
        d = np.ascontiguousarray(d, dtype=np.float64)
        require(len(d) == op.network().q, "QuadraticCost: innovation length mismatch")
        h = _vp()
        _check(lib.wc4dvar_gpu_cost_create(op.handle, _p(b), _p(d) if len(d) else None, ctypes.byref(h)))
        self._h = h
        self.op = op

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:  # the module global is gone at interpreter shutdown
            lib.wc4dvar_gpu_cost_destroy(h)
            self._h = None

    @property
    def handle(self):
        return self._h

    def __call__(self, x) -> float:
        x = np.ascontiguousarray(x, dtype=np.float64)
        v = ctypes.c_double(0)
        _check(lib.wc4dvar_gpu_cost_eval(self._h, _p(x), ctypes.byref(v)))
        return v.value

    def rhs(self) -> np.ndarray:
        out = np.empty(self.op.dim())
        _check(lib.wc4dvar_gpu_cost_rhs(self._h, _p(out)))
        return out

    def gradient(self, x) -> np.ndarray:
        return self.op.apply(x) - self.rhs()


@dataclass
class PcgOptions:
    """krylov.hpp:32-38 (cost_eval is a QuadraticCost handle on this side)."""

    max_iter: int = 100
    rel_tol: float = 1e-6
    reorthogonalize: bool = False
    cost: Optional[QuadraticCost] = None
    store_residual_vectors: bool = False


@dataclass
class CgHistory:
    alphas: List[float] = field(default_factory=list)
    betas: List[float] = field(default_factory=list)
    residual_norms: List[float] = field(default_factory=list)
    quadratic_costs: List[float] = field(default_factory=list)
    iterations: int = 0
    converged: bool = False
    stop_reason: str = ""
    normalized_residuals: List[np.ndarray] = field(default_factory=list)  # f_j = r_j / ||r_j||

    def relative_residual(self, j: int) -> float:
        return self.residual_norms[j] / self.residual_norms[0]


@dataclass
class PcgResult:
    x: np.ndarray
    history: CgHistory


_STOP = {0: "zero initial residual", 1: "relative residual tolerance reached", 2: "maximum iterations reached"}


@dataclass
class PrecondSpec:
    """assimilation.hpp:66-77."""

    kind: str = "none"   # none | deterministic | revd | nystrom | ritzit
    k: int = 0
    l: int = 5
    seed: int = 0
    p_iter: int = 1


@dataclass
class SolverSpec:
    """assimilation.hpp:79-84."""

    max_iter: int = 100
    rel_tol: float = 1e-6
    reorthogonalize: bool = False
    record_cost: bool = True


@dataclass
class ClusteredSpectrum:
    """spectrum.hpp:13-24: the eigenvalues of the (preconditioned) Hessian that can differ
    from 1 (decreasing) and the multiplicity of the unit cluster."""

    nonunit: np.ndarray
    unit_multiplicity: int

    def min_eigenvalue(self) -> float:
        """spectrum.cpp:9-13"""
        m = 1.0 if self.unit_multiplicity > 0 else math.inf
        return min(m, float(self.nonunit.min())) if len(self.nonunit) else m

    def max_eigenvalue(self) -> float:
        """spectrum.cpp:15-19"""
        m = 1.0 if self.unit_multiplicity > 0 else -math.inf
        return max(m, float(self.nonunit.max())) if len(self.nonunit) else m

    def full(self) -> np.ndarray:
        """spectrum.cpp:21-29: every eigenvalue, decreasing."""
        return np.sort(np.concatenate([self.nonunit, np.ones(self.unit_multiplicity)]))[::-1]


def clustered_spectrum(op: "HessianOperator", precond: Optional["LmpFactor"] = None,
                       obs_range: Optional[np.ndarray] = None) -> ClusteredSpectrum:
    """spectrum.cpp:31-64 on the device: orthonormal basis of [W | U], C^T A C on it (q + k
    block applies), symmetric EVD of the projected matrix."""
    require(isinstance(op, HessianOperator), "clustered_spectrum: operator is not a HessianOperator")
    k = precond.k() if (precond is not None and not precond.is_identity()) else 0
    q = op.net.q
    W = None
    if obs_range is not None:
        W = np.asfortranarray(obs_range, dtype=np.float64)
        require(W.shape[0] == op.dim(), "clustered_spectrum: observation range mismatch")
        q = W.shape[1]
    vals = np.empty(max(q + k, 1))
    nn, unit = _i64(0), _i64(0)
    _check(lib.wc4dvar_gpu_clustered_spectrum(op.handle, precond.handle if k else None, _p(W),
                                              W.shape[0] if W is not None else op.dim(), _p(vals),
                                              ctypes.byref(nn), ctypes.byref(unit)))
    return ClusteredSpectrum(vals[:nn.value].copy(), int(unit.value))


@dataclass
class InnerLoopReport:
    """assimilation.hpp:86-97."""

    delta_p: np.ndarray
    delta_p_tilde: np.ndarray
    quadratic_costs: List[float]
    residual_norms: List[float]
    iterations: int
    converged: bool
    precond: PrecondSpec
    ritz_values: np.ndarray
    preconditioned_extremes: Optional[tuple] = None  # (min, max) when dim <= dense_cap


def run_inner_loop(hessian: HessianOperator, b, d, precond: PrecondSpec, solver: SolverSpec,
                   omega: Optional[np.ndarray] = None, dense_cap: int = 4096,
                   previous_hessian: Optional[HessianOperator] = None) -> InnerLoopReport:
    """run_inner_loop, assimilation.cpp:192-253, from the innovations b (control space) and
    d (observation space) of compute_innovations (assimilation.cpp:119-128): QuadraticCost
    -> randomized LMP -> split PCG on the cost's RHS -> delta_p = D^{1/2} x."""
    cost = QuadraticCost(hessian, b, d)
    factor, ritz = None, np.zeros(0)
    if precond.kind == "deterministic":  # previous-loop Lanczos LMP (assimilation.cpp:204-211)
        require(previous_hessian is not None, "run_inner_loop: deterministic LMP needs a previous inner loop")
        pairs = exact_top_pairs(previous_hessian, precond.k, dense_cap)
        factor = build_spectral_lmp(pairs, hessian.device())
        ritz = pairs.values
    elif precond.kind != "none":
        cfg = SketchConfig(precond.k, precond.l, precond.seed, precond.kind, precond.p_iter)
        pairs = sketch_eigenpairs(hessian, cfg, omega)
        factor = build_spectral_lmp(pairs, hessian.device())
        ritz = pairs.values
    opts = PcgOptions(solver.max_iter, solver.rel_tol, solver.reorthogonalize,
                      cost if solver.record_cost else None)
    sol = pcg_split(hessian, cost.rhs(), factor, None, opts)
    extremes = None
    if hessian.dim() <= dense_cap:  # desk-scale diagnostic (assimilation.cpp:248-251)
        cs = clustered_spectrum(hessian, factor)
        extremes = (cs.min_eigenvalue(), cs.max_eigenvalue())
    return InnerLoopReport(hessian.apply_D_half(sol.x), sol.x, sol.history.quadratic_costs,
                           sol.history.residual_norms, sol.history.iterations, sol.history.converged,
                           precond, ritz, extremes)


def pcg_split(op: LinearOperator, b, precond: Optional[LmpFactor] = None, x0=None,
              opts: Optional[PcgOptions] = None) -> PcgResult:
    """krylov.cpp:22-108."""
    opts = opts or PcgOptions()
    n = op.dim()
    b = np.ascontiguousarray(b, dtype=np.float64)
    require(len(b) == n, "pcg_split: right-hand side dimension mismatch")
    x0a = None if x0 is None or len(x0) == 0 else np.ascontiguousarray(x0, dtype=np.float64)
    require(x0a is None or len(x0a) == n, "pcg_split: initial guess dimension mismatch")
    o = PcgOpts()
    o.max_iter, o.reorthogonalize, o.rel_tol = opts.max_iter, int(opts.reorthogonalize), opts.rel_tol
    o.store_residual_vectors = int(opts.store_residual_vectors)
    mi = max(opts.max_iter, 0)
    al, be = np.zeros(mi + 1), np.zeros(mi + 1)
    rn, qc = np.zeros(mi + 2), np.zeros(mi + 2)
    hst = PcgHist()
    hst.alphas, hst.betas, hst.residual_norms, hst.quadratic_costs = _p(al), _p(be), _p(rn), _p(qc)
    F = None
    if opts.reorthogonalize or opts.store_residual_vectors:
        F = np.empty((n, mi + 1), order="F")
        hst.normalized_residuals, hst.ld_residuals = _p(F), n
    x = np.empty(n)
    _check(lib.wc4dvar_gpu_pcg(op.handle, _p(b), precond.handle if precond is not None else None,
                               _p(x0a), ctypes.byref(o), opts.cost.handle if opts.cost else None,
                               _p(x), ctypes.byref(hst)))
    it = hst.iterations
    h = CgHistory(al[:it].tolist(), be[:it].tolist(), rn[:it + 1].tolist(),
                  qc[:it + 1].tolist() if opts.cost else [], it, bool(hst.converged),
                  _STOP.get(hst.stop_reason, ""),
                  [F[:, j].copy() for j in range(hst.n_residuals)] if F is not None else [])
    return PcgResult(x, h)


# ---------------------------------------------------------------------------------------------
# Deterministic LMP eigenpairs (krylov.hpp:56-91, assimilation.cpp:173-190), SURVEY §8(f)-3
@dataclass
class TridiagonalMatrix:
    """krylov.hpp:56-63: gamma (diagonal) / tau (off-diagonal) parameterisation."""

    gammas: np.ndarray
    taus: np.ndarray

    def dim(self) -> int:
        return len(self.gammas)

    def dense(self) -> np.ndarray:
        """krylov.cpp:110-120"""
        return np.diag(self.gammas) + np.diag(self.taus, 1) + np.diag(self.taus, -1)


def tridiagonal_from_cg(history: CgHistory) -> TridiagonalMatrix:
    """krylov.cpp:122-134: gamma_1 = 1/alpha_1, gamma_j = 1/alpha_j + beta_{j-1}/alpha_{j-1},
    tau_j = sqrt(beta_j)/alpha_j (scalar recurrences on the CG history)."""
    j = len(history.alphas)
    require(j >= 1, "tridiagonal_from_cg: history is empty")
    g = np.empty(j)
    t = np.empty(max(j - 1, 0))
    for i in range(j):
        g[i] = 1.0 / history.alphas[i]
        if i > 0:
            g[i] += history.betas[i - 1] / history.alphas[i - 1]
        if i + 1 < j:
            t[i] = math.sqrt(history.betas[i]) / history.alphas[i]
    return TridiagonalMatrix(g, t)


def ritz_from_tridiagonal(T: TridiagonalMatrix, residual_basis, k: int, device: int = 0) -> RitzPairs:
    """krylov.cpp:136-176 on the device: top-k Ritz pairs from T_j and the stored normalised
    CG residuals (sign-alternated into the Lanczos basis), ghosts collapsed."""
    j = T.dim()
    require(1 <= k <= j, "ritz_from_tridiagonal: k out of range")
    require(len(residual_basis) >= j, "ritz_from_tridiagonal: residual basis shorter than T")
    F = np.asfortranarray(np.column_stack([np.asarray(residual_basis[i], dtype=np.float64) for i in range(j)]))
    n = F.shape[0]
    U = np.empty((n, k), order="F")
    vals = np.empty(k)
    g = np.ascontiguousarray(T.gammas, dtype=np.float64)
    t = np.ascontiguousarray(T.taus, dtype=np.float64) if j > 1 else np.zeros(1)
    _check(lib.wc4dvar_gpu_ritz_from_tridiagonal(n, j, _p(g), _p(t), _p(F), n, k, _p(U), n, _p(vals), device))
    return RitzPairs(U, vals, "lanczos")


@dataclass
class LanczosOptions:
    """krylov.hpp:81-85."""

    max_iter: int = 0
    tol: float = 1e-10
    seed: int = 0x5EED0F4D


def lanczos_eigenpairs(op: LinearOperator, k: int, opts: Optional[LanczosOptions] = None) -> RitzPairs:
    """krylov.cpp:178-278 on the device: Lanczos with full re-orthogonalisation until the
    top-k pairs converge (residual b |W(m-1, i)| <= tol |theta_0|)."""
    opts = opts or LanczosOptions()
    n = op.dim()
    require(1 <= k <= n, "lanczos_eigenpairs: k out of range")
    o = LanczosOpts()
    o.max_iter, o.tol, o.seed = opts.max_iter, opts.tol, opts.seed
    U = np.empty((n, k), order="F")
    vals = np.empty(k)
    steps = _i64(0)
    _check(lib.wc4dvar_gpu_lanczos_eigenpairs(op.handle, k, ctypes.byref(o), _p(U), n, _p(vals), ctypes.byref(steps)))
    return RitzPairs(U, vals, "exact")


def exact_top_pairs(op: LinearOperator, k: int, dense_cap: int = 4096, lanczos_seed: int = 0x5EED0F4D,
                    tol: float = 1e-12) -> RitzPairs:
    """assimilation.cpp:173-190.  The reference takes a dense EVD when dim <= dense_cap and
    Lanczos otherwise; on the device both routes are Lanczos with full re-orthogonalisation,
    with the tolerance tightened to 1e-12 on the desk-scale route (the reference's own
    dense-vs-Lanczos agreement test is 1e-8, test_assimilation.cpp:361-373)."""
    require(1 <= k <= op.dim(), "exact_top_pairs: k out of range")
    return lanczos_eigenpairs(op, k, LanczosOptions(0, tol if op.dim() <= dense_cap else 1e-10, lanczos_seed))
