"""B200-native quantization-tree transition estimator (arXiv 1101.3228).

Drop-in for the reference's hot path (qtree::tree::estimate*, the Voronoi
projection and the backward-DP pricer) on hand-written sm_100a kernels behind
the C ABI in include/qtree_cuda.h. See DESIGN.md / INTEGRATION.md.
"""
from .qtree import (  # noqa: F401
    BrownianChain1d, BuildPhases, ConfigError, CountMatrixSet, EngineKind, EstimateOptions,
    EstimatorKind, GbmChain3d, IoError, NnBackend, NumericError, OuChain1d, QuantGrid, QuantTree,
    StoppingResult, SwingResult, TwoFactorChain, TwoFactorParams, accumulate_paths,
    ar1_coefficients, base_grid, build_brownian_grids, build_gbm_grids, build_ou_grids,
    build_two_factor_grids, estimate, estimate_alg1, estimate_alg2, estimate_alg3,
    DeviceTree, estimate_device,
    cond_expectation, estimate_with_normals, layout, nearest, path_normals, solve_stopping,
    solve_swing,
    swing_window, tabulate, uniforms)

__all__ = [n for n in dir() if not n.startswith("_")]
