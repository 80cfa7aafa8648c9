"""B200-native (sm_100a) randomized-LMP hot path of arxiv 2101.07249 (weak-constraint 4D-Var).

The product is ``libwc4dvar_gpu.so`` (C-ABI in include/wc4dvar_gpu.h); this package is
the Python mirror of the reference's C++ operator / sketch / LMP / PCG interface over it.
"""
from .wc4dvar import (  # noqa: F401
    AdvDiffLinearized, AdvectionLinearized, CgHistory, CovarianceFactor, DenseCapError,
    DenseOperator, DeviceError, HessianOperator, IdentityLinearized, LinearizedModel,
    LinearOperator, LmpFactor, NumericalError, ObservationNetwork, PcgOptions, PcgResult,
    QuadraticCost, RitzPairs, SketchConfig, assemble_dense, build_spectral_lmp, gaussian_matrix,
    last_sketch_timing, nystrom, pcg_split, probe_dmma_peak, rayleigh_ritz, revd, revd_ritzit,
    sketch_eigenpairs, version, LIB_PATH, SIGNATURES, Lorenz96Linearized,
    lorenz96_trajectory, lorenz96_trajectory_device, integrate_p, InnerLoopReport, PrecondSpec, SolverSpec,
    run_inner_loop, ClusteredSpectrum, clustered_spectrum, TridiagonalMatrix, tridiagonal_from_cg,
    ritz_from_tridiagonal, LanczosOptions, lanczos_eigenpairs, exact_top_pairs,
    gaussian_block_dev, mt19937_raw_host, mt19937_raw_dev, sketch_eigenpairs_dev, launch_count, build_spectral_lmp_dev,
)
