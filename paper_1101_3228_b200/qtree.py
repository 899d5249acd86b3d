"""Python mirror of the reference's public API for the hot path, on the C ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/qtree, cited file:line):

  tree::estimate / estimate_alg1 / estimate_alg2 / estimate_alg3   estimate.hpp:133-309
  tree::detail::accumulate_paths                                  estimate.hpp:88-126
  tree::QuantTree (counts, pi, row_count, row_visited, pi_row)    quant_tree.hpp:46-84
  quant::QuantGrid, quant::nearest                                 grid.hpp:20-61, nn.hpp:150-176
  model::TwoFactorParams, ar1_coefficients, TwoFactorChain,
        BrownianChain1d (+ the config-3/5 chains OuChain1d, GbmChain3d)
  pricer::solve_stopping / solve_swing                             bdp.hpp:58-96, swing.hpp:47-129

Every count, projection and price is computed by libqtree_cuda.so on the GPU;
this module only marshals host arrays. Reference exceptions map to:
std::invalid_argument -> ValueError, ConfigError / IoError / NumericError ->
the classes below (errors.hpp:9-21); device failures -> NumericError("cuda: ...").
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import functools
import math
import os
from dataclasses import dataclass, field
from typing import Callable, Sequence

import numpy as np

from . import _lib as L


# ---------------------------------------------------------------------------
# errors (errors.hpp:9-21)
# ---------------------------------------------------------------------------
class ConfigError(RuntimeError):
    """Bad or inconsistent run parameters (CLI exit code 1)."""


class IoError(RuntimeError):
    """File-format or filesystem failures (CLI exit code 2)."""


class NumericError(RuntimeError):
    """Numerical breakdown or device failure (CLI exit code 3)."""


def _check(rc: int, where: str) -> None:
    if rc == L.QT_OK:
        return
    msg = f"{where}: {L.last_error()}"
    if rc == L.QT_ERR_INVALID_ARGUMENT:
        raise ValueError(msg)
    if rc == L.QT_ERR_CONFIG:
        raise ConfigError(msg)
    if rc == L.QT_ERR_IO:
        raise IoError(msg)
    raise NumericError(msg)


# ---------------------------------------------------------------------------
# enums / options (stream.hpp:16, estimate.hpp:18-36, nn.hpp:16)
# ---------------------------------------------------------------------------
class EngineKind(enum.IntEnum):
    Lcg48 = 0
    Mrg32k3a = 1
    Xorwow = 2


class EstimatorKind(enum.IntEnum):
    AlgI = 0
    AlgII = 1
    AlgIII = 2


class NnBackend(enum.IntEnum):
    BruteForce = 0
    KdTree = 1  # accepted; the device projection is exact, so results are identical


@dataclass
class BuildPhases:
    simulate_ms: float = 0.0
    nn_ms: float = 0.0
    merge_ms: float = 0.0
    normalize_ms: float = 0.0
    total_ms: float = 0.0


@dataclass
class EstimateOptions:
    engine: EngineKind = EngineKind.Mrg32k3a
    seed: int = 12345
    workers: int = 1          # accepted and ignored (the device decides the parallelism)
    nn: NnBackend = NnBackend.BruteForce
    phases: BuildPhases | None = None
    devices: int = 1          # GPUs of this process to shard over (one NCCL all-reduce)


# ---------------------------------------------------------------------------
# model (two_factor.hpp, chains.hpp)
# ---------------------------------------------------------------------------
@dataclass
class TwoFactorParams:
    s0: float = 100.0
    sigma1: float = 0.5
    sigma2: float = 0.3
    alpha1: float = 1.0
    alpha2: float = 4.0
    rho: float = 0.0
    r: float = 0.0
    strike: float = 100.0
    horizon: float = 1.0
    steps: int = 365

    def c(self, gbm_rho=(0.0, 0.0, 0.0)) -> L.QtModelParams:
        return L.QtModelParams(self.s0, self.sigma1, self.sigma2, self.alpha1, self.alpha2,
                               self.rho, self.r, self.strike, self.horizon, int(self.steps),
                               (C.c_double * 3)(*gbm_rho))


CHAIN_BROWNIAN_1D, CHAIN_TWO_FACTOR, CHAIN_OU_1D, CHAIN_GBM_3D = 0, 1, 2, 3


class _Chain:
    kind: int
    _dim: int

    def __init__(self, params: TwoFactorParams, gbm_rho=(0.0, 0.0, 0.0)):
        self.params = params
        self.gbm_rho = tuple(gbm_rho)
        n = int(params.steps)
        self.step_coef = np.zeros(max(n, 0) * 6, np.float64)
        self.marg_coef = np.zeros((max(n, 0) + 1) * 6, np.float64)
        p = params.c(self.gbm_rho)
        _check(L.lib().qt_chain_coefficients(self.kind, C.byref(p), _f(self.step_coef),
                                              _f(self.marg_coef)), type(self).__name__)

    def dim(self) -> int:
        return self._dim

    def layers(self) -> int:
        return int(self.params.steps)

    def normals_per_step(self) -> int:
        return self._dim

    def dt(self) -> float:
        return self.params.horizon / self.params.steps

    def time(self, k: int) -> float:
        return k * self.dt()

    def c(self) -> L.QtChain:
        return L.QtChain(self.kind, self.layers(), _f(self.step_coef), _f(self.marg_coef))


class BrownianChain1d(_Chain):
    """X_{k+1} = X_k + sqrt(dt) eps (chains.hpp:68-95)."""
    kind, _dim = CHAIN_BROWNIAN_1D, 1

    def __init__(self, steps: int, horizon: float = 1.0):
        super().__init__(TwoFactorParams(steps=steps, horizon=horizon))


class TwoFactorChain(_Chain):
    """Exact AR(1) form of the 2-factor OU pair (chains.hpp:30-64)."""
    kind, _dim = CHAIN_TWO_FACTOR, 2

    def __init__(self, params: TwoFactorParams):
        super().__init__(params)


class OuChain1d(_Chain):
    """Config 3: factor 1 of TwoFactorChain (a = e^{-alpha1 dt}, l11)."""
    kind, _dim = CHAIN_OU_1D, 1

    def __init__(self, params: TwoFactorParams):
        super().__init__(params)


class GbmChain3d(_Chain):
    """Config 5: 3-D correlated Brownian log-state, X' = X + sqrt(dt) L eps."""
    kind, _dim = CHAIN_GBM_3D, 3

    def __init__(self, steps: int, horizon: float = 1.0, rho=(0.0, 0.0, 0.0)):
        super().__init__(TwoFactorParams(steps=steps, horizon=horizon), gbm_rho=rho)


def ar1_coefficients(p: TwoFactorParams) -> TwoFactorParams:
    """Ar1Spec::from_params validation (two_factor.hpp:90-101); the chain keeps the params."""
    TwoFactorChain(p)
    return p


# ---------------------------------------------------------------------------
# grids (grid.hpp)
# ---------------------------------------------------------------------------
class QuantGrid:
    """N points in R^d, row-major FP64 (grid.hpp:20-61). Validity (finite,
    distinct) is enforced by the library when a grid is used."""

    def __init__(self, dim: int, points):
        self._dim = int(dim)
        self.points = np.ascontiguousarray(points, dtype=np.float64).reshape(-1)
        if self._dim < 1:
            raise NumericError("grid: dimension must be >= 1")
        if self.points.size == 0 or self.points.size % self._dim:
            raise NumericError("grid: point data size is not a positive multiple of dim")
        if not np.all(np.isfinite(self.points)):
            raise NumericError("grid: non-finite point coordinate")

    def dim(self) -> int:
        return self._dim

    def size(self) -> int:
        return self.points.size // self._dim

    def point(self, i: int) -> np.ndarray:
        return self.points[i * self._dim:(i + 1) * self._dim]

    def data(self) -> np.ndarray:
        return self.points

    def __eq__(self, o) -> bool:
        return isinstance(o, QuantGrid) and self._dim == o._dim and np.array_equal(
            self.points, o.points)


def _f(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _u(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_uint64))


class _GridPack:
    """Flattened layers 1..n for qt_grids (keeps the arrays alive)."""

    def __init__(self, chain: _Chain, grids: Sequence[QuantGrid]):
        if len(grids) != chain.layers():
            raise ValueError("estimate: need one grid per layer 1..n")
        for g in grids:
            if g.dim() != chain.dim():
                raise ValueError("estimate: grid dimension mismatch")
        self.sizes = np.array([1] + [g.size() for g in grids], np.uint64)
        self.points = np.ascontiguousarray(np.concatenate([g.data() for g in grids]))
        self.s = L.QtGrids(chain.dim(), chain.layers(), _u(self.sizes), _f(self.points))


def layout(sizes) -> tuple[int, int]:
    sizes = [int(s) for s in sizes]
    return sum(sizes), sum(sizes[k - 1] * sizes[k] for k in range(1, len(sizes)))


# ---------------------------------------------------------------------------
# tree (quant_tree.hpp)
# ---------------------------------------------------------------------------
@dataclass
class CountMatrixSet:
    visits: list = field(default_factory=list)  # layer 0..n, u64 arrays
    joint: list = field(default_factory=list)   # transition 1..n, row-major N_{k-1} x N_k


class QuantTree:
    """Grids 0..n, counts, dense FP64 pi and M (quant_tree.hpp:46-84)."""

    def __init__(self, grids, sizes, visits, joint, pi, samples):
        self.grids = grids
        self.sizes = np.asarray(sizes, np.uint64)
        self.flat_visits, self.flat_joint, self.flat_pi = visits, joint, pi
        self.samples = int(samples)
        self.counts = CountMatrixSet()
        self.pi = []
        vo = jo = 0
        for k, s in enumerate(self.sizes):
            self.counts.visits.append(visits[vo:vo + int(s)])
            vo += int(s)
            if k:
                r = int(self.sizes[k - 1])
                self.counts.joint.append(joint[jo:jo + r * int(s)])
                self.pi.append(pi[jo:jo + r * int(s)])
                jo += r * int(s)

    def layers(self) -> int:
        return len(self.pi)

    def layer_size(self, k: int) -> int:
        return int(self.sizes[k])

    def row_count(self, k: int, i: int) -> int:
        return int(self.counts.visits[k - 1][i])

    def row_visited(self, k: int, i: int) -> bool:
        return self.row_count(k, i) > 0

    def pi_row(self, k: int, i: int) -> np.ndarray:
        c = self.layer_size(k)
        return self.pi[k - 1][i * c:(i + 1) * c]


def _estimate(kind: int, chain: _Chain, grids: Sequence[QuantGrid], paths: int,
              opt: EstimateOptions | None, normals=None) -> QuantTree:
    opt = opt or EstimateOptions()
    if kind in (EstimatorKind.AlgII, EstimatorKind.AlgIII) and opt.workers < 1:
        raise ValueError(f"estimate_alg{int(kind) + 1}: workers must be >= 1")
    if paths <= 0:
        raise ValueError("estimate: need at least one path")
    gp = _GridPack(chain, grids)
    nvis, njoint = layout(gp.sizes)
    visits = np.zeros(nvis, np.uint64)
    joint = np.zeros(njoint, np.uint64)
    pi = np.zeros(njoint, np.float64)
    ph = np.zeros(5, np.float64)
    ch = chain.c()
    if normals is None:
        rc = L.lib().qt_estimate(int(kind), C.byref(ch), C.byref(gp.s), int(paths),
                                 int(opt.engine), int(opt.seed), int(opt.devices), _u(visits),
                                 _u(joint), _f(pi), _f(ph))
    else:
        nrm = np.ascontiguousarray(normals, dtype=np.float64)
        rc = L.lib().qt_estimate_normals(int(kind), C.byref(ch), C.byref(gp.s), int(paths),
                                         _f(nrm), _u(visits), _u(joint), _f(pi))
    _check(rc, "estimate")
    if opt.phases is not None:
        opt.phases.simulate_ms, opt.phases.nn_ms, opt.phases.merge_ms, \
            opt.phases.normalize_ms, opt.phases.total_ms = (float(x) for x in ph)
    x0 = QuantGrid(chain.dim(), np.zeros(chain.dim()))
    return QuantTree([x0] + list(grids), gp.sizes, visits, joint, pi, paths)


class DeviceTree:
    """An estimated tree kept in device memory (qt_estimate_device): the
    counts, visits and pi stay on the GPU and solve_stopping / solve_swing read
    them in place, the way the reference's pricers hold a non-owning tree
    pointer (bdp.hpp:20-23, run_pipeline pipeline.hpp:190-215). No pi round
    trip: at config 4 that is 2.9 GB each way. download() gives the host
    QuantTree; close() (or the context manager) frees the device memory."""

    def __init__(self, handle: int, grids: list, sizes: np.ndarray, samples: int):
        self._h = C.c_void_p(handle)
        self.grids, self.sizes, self.samples = grids, sizes, samples

    def layers(self) -> int:
        return len(self.sizes) - 1

    def layer_size(self, k: int) -> int:
        return int(self.sizes[k])

    def handle(self) -> C.c_void_p:
        if not self._h:
            raise ValueError("DeviceTree: already closed")
        return self._h

    def device_arrays(self) -> tuple[int, int, int]:
        """Raw device pointers (visits, joint, pi), owned by this tree."""
        v, j, p = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _check(L.lib().qt_dtree_device_arrays(self.handle(), C.byref(v), C.byref(j), C.byref(p)),
               "dtree")
        return v.value, j.value, p.value

    def download(self) -> QuantTree:
        nvis, njoint = layout(self.sizes)
        visits = np.zeros(nvis, np.uint64)
        joint = np.zeros(njoint, np.uint64)
        pi = np.zeros(njoint, np.float64)
        _check(L.lib().qt_dtree_download(self.handle(), _u(visits), _u(joint), _f(pi)), "dtree")
        return QuantTree(self.grids, self.sizes, visits, joint, pi, self.samples)

    def close(self) -> None:
        if self._h:
            L.lib().qt_dtree_destroy(self._h)
            self._h = C.c_void_p()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass


def estimate_device(kind, chain, grids, paths, opt=None) -> DeviceTree:
    """estimate() with the result kept on the GPU (see DeviceTree)."""
    opt = opt or EstimateOptions()
    if int(kind) not in (0, 1, 2):
        raise ValueError("estimate: unknown estimator kind")
    if int(kind) in (1, 2) and opt.workers < 1:
        raise ValueError(f"estimate_alg{int(kind) + 1}: workers must be >= 1")
    if paths <= 0:
        raise ValueError("estimate: need at least one path")
    gp = _GridPack(chain, grids)
    ph = np.zeros(5, np.float64)
    ch = chain.c()
    h = C.c_void_p()
    _check(L.lib().qt_estimate_device(int(kind), C.byref(ch), C.byref(gp.s), int(paths),
                                      int(opt.engine), int(opt.seed), int(opt.devices),
                                      C.byref(h), _f(ph)), "estimate")
    if opt.phases is not None:
        opt.phases.simulate_ms, opt.phases.nn_ms, opt.phases.merge_ms, \
            opt.phases.normalize_ms, opt.phases.total_ms = (float(x) for x in ph)
    x0 = QuantGrid(chain.dim(), np.zeros(chain.dim()))
    return DeviceTree(h.value, [x0] + list(grids), gp.sizes, int(paths))


def estimate_alg1(chain, grids, paths, opt=None) -> QuantTree:
    """Algorithm I (estimate.hpp:133-157): pathwise estimation."""
    return _estimate(EstimatorKind.AlgI, chain, grids, paths, opt)


def estimate_alg2(chain, grids, paths, opt=None) -> QuantTree:
    """Algorithm II (estimate.hpp:163-207): path-parallel; identical counts to Alg I."""
    return _estimate(EstimatorKind.AlgII, chain, grids, paths, opt)


def estimate_alg3(chain, grids, samples_per_layer, opt=None) -> QuantTree:
    """Algorithm III (estimate.hpp:213-296): layer-parallel pair sampling."""
    return _estimate(EstimatorKind.AlgIII, chain, grids, samples_per_layer, opt)


def estimate(kind, chain, grids, paths, opt=None) -> QuantTree:
    """Dispatch by estimator kind (estimate.hpp:299-309)."""
    if int(kind) not in (0, 1, 2):
        raise ValueError("estimate: unknown estimator kind")
    return _estimate(EstimatorKind(int(kind)), chain, grids, paths, opt)


def estimate_with_normals(kind, chain, grids, paths, normals) -> QuantTree:
    """Parity mode: the estimator consumes caller-supplied normals."""
    return _estimate(EstimatorKind(int(kind)), chain, grids, paths, None, normals=normals)


def accumulate_paths(chain, grids, engine, seed, first, count, total):
    """detail::accumulate_paths over paths [first, first+count) of `total`
    (estimate.hpp:88-126). Returns flat (visits, joint)."""
    gp = _GridPack(chain, grids)
    nvis, njoint = layout(gp.sizes)
    visits = np.zeros(nvis, np.uint64)
    joint = np.zeros(njoint, np.uint64)
    ch = chain.c()
    _check(L.lib().qt_accumulate_paths(C.byref(ch), C.byref(gp.s), int(engine), int(seed),
                                       int(first), int(count), int(total), _u(visits),
                                       _u(joint)), "accumulate_paths")
    return visits, joint


def nearest(grid: QuantGrid, queries) -> np.ndarray:
    """Batch NnIndex::nearest (nn.hpp:18-46): exact, smallest index on ties."""
    q = np.ascontiguousarray(queries, dtype=np.float64).reshape(-1)
    if q.size % grid.dim():
        raise ValueError("nearest: query dimension mismatch")
    out = np.zeros(q.size // grid.dim(), np.uint64)
    _check(L.lib().qt_nearest(grid.dim(), grid.size(), _f(grid.points), out.size, _f(q),
                              _u(out)), "nearest")
    return out


def path_normals(engine, seed, normals_per_path, first, count) -> np.ndarray:
    out = np.zeros(int(count) * int(normals_per_path), np.float64)
    _check(L.lib().qt_path_normals(int(engine), int(seed), int(normals_per_path), int(first),
                                   int(count), _f(out)), "path_normals")
    return out


# ---------------------------------------------------------------------------
# files (quant_tree.hpp:138-207 save_tree / load_tree, grid.hpp:84-117)
# ---------------------------------------------------------------------------
def save_tree(tree: QuantTree, path) -> None:
    """QTRE v1, byte-identical to the reference's save_tree."""
    dim = tree.grids[0].dim()
    pts = np.ascontiguousarray(np.concatenate([np.asarray(g.data(), np.float64) for g in tree.grids]))
    sizes = np.ascontiguousarray(tree.sizes, np.uint64)
    v = np.ascontiguousarray(tree.flat_visits, np.uint64)
    j = np.ascontiguousarray(tree.flat_joint, np.uint64)
    p = np.ascontiguousarray(tree.flat_pi, np.float64)
    _check(L.lib().qt_save_tree(str(path).encode(), tree.layers(), dim, _u(sizes), _f(pts),
                                tree.samples, v.ctypes.data, j.ctypes.data, p.ctypes.data, 0),
           "save_tree")


def load_tree(path) -> QuantTree:
    n, d, m = C.c_int32(0), C.c_int32(0), C.c_uint64(0)
    _check(L.lib().qt_tree_file_info(str(path).encode(), C.byref(n), C.byref(d), C.byref(m),
                                     None, 0), "load_tree")
    sizes = np.zeros(n.value + 1, np.uint64)
    _check(L.lib().qt_tree_file_info(str(path).encode(), C.byref(n), C.byref(d), C.byref(m),
                                     _u(sizes), sizes.size), "load_tree")
    nvis, njoint = layout(sizes)
    pts = np.zeros(nvis * d.value, np.float64)
    v = np.zeros(nvis, np.uint64)
    j = np.zeros(njoint, np.uint64)
    p = np.zeros(njoint, np.float64)
    _check(L.lib().qt_load_tree(str(path).encode(), n.value, d.value, _u(sizes), _f(pts), _u(v),
                                nvis, _u(j), _f(p), njoint), "load_tree")
    grids, o = [], 0
    for s in sizes:
        grids.append(QuantGrid(d.value, pts[o:o + int(s) * d.value]))
        o += int(s) * d.value
    return QuantTree(grids, sizes, v, j, p, m.value)


def save_grid(grid: QuantGrid, path) -> None:
    pts = np.ascontiguousarray(grid.data(), np.float64)
    _check(L.lib().qt_save_grid(str(path).encode(), grid.dim(), grid.size(), _f(pts)), "save_grid")


def load_grid(path) -> QuantGrid:
    d, n = C.c_int32(0), C.c_uint64(0)
    _check(L.lib().qt_load_grid(str(path).encode(), C.byref(d), C.byref(n), None, 0), "load_grid")
    pts = np.zeros(n.value * d.value, np.float64)
    _check(L.lib().qt_load_grid(str(path).encode(), C.byref(d), C.byref(n), _f(pts), pts.size),
           "load_grid")
    return QuantGrid(d.value, pts)


# ---------------------------------------------------------------------------
# micro-benchmarks (qtree_main.cpp bench-rng / bench-nn)
# ---------------------------------------------------------------------------
@dataclass
class PiEstimate:
    estimate: float
    std_error: float
    points: int
    inside: int
    ms: float


def bench_pi(engine: int, seed: int, samples: int, streams: int = 1,
             skip_ahead: bool = False) -> PiEstimate:
    """estimate_pi_partitioned (monte_carlo.hpp:51-77) on the GPU."""
    inside, est, se, ms = C.c_uint64(0), C.c_double(0), C.c_double(0), C.c_double(0)
    _check(L.lib().qt_bench_pi(int(engine), int(seed), int(samples), int(streams),
                               1 if skip_ahead else 0, C.byref(inside), C.byref(est),
                               C.byref(se), C.byref(ms)), "bench_pi")
    return PiEstimate(est.value, se.value, int(samples) // 2, inside.value, ms.value)


def bench_nn(n: int, queries: int, seed: int = 12345) -> tuple[int, float]:
    """(sum of nearest indices, device ms of the searches), qtree_main.cpp:162-191."""
    sink, ms = C.c_uint64(0), C.c_double(0)
    _check(L.lib().qt_bench_nn(int(n), int(queries), int(seed), C.byref(sink), C.byref(ms)),
           "bench_nn")
    return sink.value, ms.value


def plan_cache_clear() -> None:
    """Free the device plans qt_estimate keeps for repeated calls on the same
    inputs (tables, scratch and result buffers)."""
    _check(L.lib().qt_plan_cache_clear(), "plan_cache_clear")


CERTIFIED_1D, FAST_FP32_1D, EXACT_1D = 2, 1, 0


def set_fast_path(mode) -> None:
    """1-D MRG32k3a kernel (identical counts in every mode): 2 = certified with
    approximate FP64 normals (the default), True / 1 = certified with FP32
    normals (k_paths_fast), False / 0 = the exact kernel for every path."""
    m = int(mode) if not isinstance(mode, bool) else (1 if mode else 0)
    _check(L.lib().qt_set_fast_path(m), "set_fast_path")


def apx_bounds_check() -> np.ndarray:
    """Measured maxima of the certified kernel's approximate Box-Muller vs the
    glibc-exact one over all MRG32k3a uniforms, and the bounds it assumes."""
    out = np.zeros(7, np.float64)
    _check(L.lib().qt_apx_bounds_check(_f(out)), "apx_bounds_check")
    return out


def fast_stats() -> dict:
    out = (C.c_uint64 * 3)()
    _check(L.lib().qt_fast_stats(out), "fast_stats")
    return {"fast_paths": int(out[0]), "replayed": int(out[1]), "inline_replayed": int(out[2])}


def fast_bounds_check() -> np.ndarray:
    """Exhaustive device check of the FP32 Box-Muller error bounds."""
    out = np.zeros(4, np.float64)
    _check(L.lib().qt_fast_bounds_check(_f(out)), "fast_bounds_check")
    return out


def math_checksum(domain: int) -> np.ndarray:
    """Device checksums of log / sin / cos over a whole engine domain
    (0: MRG32k3a, 1: XORWOW); equal to glibc's iff every value is."""
    out = np.zeros(3, np.uint64)
    _check(L.lib().qt_math_checksum(int(domain), _u(out)), "math_checksum")
    return out


def uniforms(engine, seed, offset, count) -> np.ndarray:
    out = np.zeros(int(count), np.float64)
    _check(L.lib().qt_uniforms(int(engine), int(seed), int(offset), int(count), _f(out)),
           "uniforms")
    return out


# ---------------------------------------------------------------------------
# pricer (bdp.hpp, swing.hpp)
# ---------------------------------------------------------------------------
NodePayoff = Callable[[int, np.ndarray], float]


PAYOFF_PUT, PAYOFF_CALL, PAYOFF_SWING, PAYOFF_MAX_CALL = 0, 1, 2, 3


def _rmax(a: float, b: float) -> float:
    return b if a < b else a  # std::max


class Payoff:
    """A discounted obstacle from the factories below: callable per node like
    the reference's NodePayoff (bdp.hpp:17), and tabulated for a whole tree in
    one C-ABI call (qt_payoff_table) by tabulate(). Both evaluate the
    reference's expressions in its order with the same libm, so the values
    are bit-identical to the reference factories (pipeline.hpp:120-170)."""

    def __init__(self, kind: int, chain_kind: int, params: TwoFactorParams,
                 gbm_sigma=(0.2, 0.2, 0.2)):
        self.kind, self.chain_kind, self.params = kind, chain_kind, params
        self.gbm_sigma = tuple(float(v) for v in gbm_sigma)

    @staticmethod
    def _spot(p: TwoFactorParams, t: float, x1: float, x2: float) -> float:
        # model::spot / spot_compensator / ou_covariance (two_factor.hpp:57-63,144-152)
        c11 = -math.expm1(-2.0 * p.alpha1 * t) / (2.0 * p.alpha1)
        c22 = -math.expm1(-2.0 * p.alpha2 * t) / (2.0 * p.alpha2)
        c12 = -p.rho * math.expm1(-(p.alpha1 + p.alpha2) * t) / (p.alpha1 + p.alpha2)
        comp = (p.sigma1 * p.sigma1 * c11 + 2.0 * p.sigma1 * p.sigma2 * c12 +
                p.sigma2 * p.sigma2 * c22)
        return p.s0 * math.exp(p.sigma1 * x1 + p.sigma2 * x2 - 0.5 * comp)

    def __call__(self, k: int, x) -> float:
        p = self.params
        t = k * (p.horizon / p.steps)
        disc = math.exp(-p.r * t)
        if self.chain_kind == CHAIN_GBM_3D or self.kind == PAYOFF_MAX_CALL:
            best = -math.inf
            for a in range(3):
                sg = self.gbm_sigma[a]
                best = _rmax(best, p.s0 * math.exp((p.r - 0.5 * sg * sg) * t + sg * float(x[a])))
            return disc * _rmax(best - p.strike, 0.0)
        if self.chain_kind == CHAIN_OU_1D:
            q = dataclasses.replace(p, sigma2=0.0)
            sp = self._spot(q, t, float(x[0]), 0.0)
        elif self.chain_kind == CHAIN_BROWNIAN_1D:
            sp = p.s0 * math.exp((p.r - 0.5 * p.sigma1 * p.sigma1) * t + p.sigma1 * float(x[0]))
        else:
            sp = self._spot(p, t, float(x[0]), float(x[1]))
        if self.kind == PAYOFF_PUT:
            return disc * _rmax(p.strike - sp, 0.0)
        if self.kind == PAYOFF_CALL:
            return disc * _rmax(sp - p.strike, 0.0)
        return disc * (sp - p.strike)

    def table(self, tree: "QuantTree") -> np.ndarray:
        phi = np.zeros(int(tree.sizes.sum()), np.float64)
        pts = np.ascontiguousarray(np.concatenate([g.data() for g in tree.grids]), np.float64)
        sig = (C.c_double * 3)(*self.gbm_sigma)
        _check(L.lib().qt_payoff_table(self.kind, self.chain_kind, C.byref(self.params.c()), sig,
                                       tree.layers(), _u(tree.sizes), _f(pts), _f(phi)),
               "payoff_table")
        return phi


def _chain_kind_for_dim(dim: int) -> int:
    if dim not in (1, 2):
        raise ValueError("payoff: the reference factories take dim 1 or 2")
    return CHAIN_BROWNIAN_1D if dim == 1 else CHAIN_TWO_FACTOR


def make_put_payoff(params: TwoFactorParams, dim: int) -> Payoff:
    """pipeline.hpp:123-136: dim 1 = lognormal benchmark put, dim 2 = 2-factor spot put."""
    return Payoff(PAYOFF_PUT, _chain_kind_for_dim(dim), params)


def make_call_payoff(params: TwoFactorParams, dim: int) -> Payoff:
    """pipeline.hpp:138-151."""
    return Payoff(PAYOFF_CALL, _chain_kind_for_dim(dim), params)


def make_swing_payoff(params: TwoFactorParams, dim: int) -> Payoff:
    """pipeline.hpp:153-170: discounted signed spread v_k."""
    return Payoff(PAYOFF_SWING, _chain_kind_for_dim(dim), params)


def make_ou_swing_payoff(params: TwoFactorParams) -> Payoff:
    """Config 3 (new): v_k = e^{-rt} (spot(p, t, x, 0) - K) with sigma2 = 0 on the
    OuChain1d state (two_factor.hpp:150-152,172-176)."""
    return Payoff(PAYOFF_SWING, CHAIN_OU_1D, params)


def make_max_call_payoff(params: TwoFactorParams, sigma=(0.2, 0.2, 0.2)) -> Payoff:
    """Config 5 (new): e^{-rt} max(max_a s0 e^{(r - sigma_a^2/2) t + sigma_a x_a} - K, 0)
    on the GbmChain3d state."""
    return Payoff(PAYOFF_MAX_CALL, CHAIN_GBM_3D, params, sigma)


def tabulate(tree: QuantTree, payoff) -> np.ndarray:
    """NodePayoff -> phi laid out like visits. Accepts a Payoff from the
    factories above (one C-ABI call), a callable f(layer, node_coords)
    (bdp.hpp:17) or an already flat table."""
    if isinstance(payoff, Payoff):
        return payoff.table(tree)
    if not callable(payoff):
        phi = np.ascontiguousarray(payoff, dtype=np.float64)
        if phi.size != int(tree.sizes.sum()):
            raise ValueError("payoff table length mismatch")
        return phi
    out = []
    for k in range(tree.layers() + 1):
        g = tree.grids[k]
        out.extend(float(payoff(k, g.point(i))) for i in range(g.size()))
    return np.array(out, np.float64)


@dataclass
class StoppingResult:
    value: list
    exercise: list
    price: float


@dataclass
class SwingResult:
    q_min: int
    q_max: int
    m_lo: list
    m_count: list
    value: list
    take: list
    price: float


def solve_stopping(tree: QuantTree, payoff) -> StoppingResult:
    """V_k = max(phi_k, E(V_{k+1}|node)), absorbing unvisited nodes (bdp.hpp:58-96)."""
    if tree is None or payoff is None:
        raise ValueError("solve_stopping: incomplete problem")
    phi = tabulate(tree, payoff)
    n = tree.layers()
    value = np.zeros(phi.size, np.float64)
    ex = np.zeros(phi.size, np.uint8)
    price = C.c_double()
    exp = ex.ctypes.data_as(C.POINTER(C.c_uint8))
    if isinstance(tree, DeviceTree):  # in place on the device
        rc = L.lib().qt_dtree_stopping(tree.handle(), _f(phi), _f(value), exp, C.byref(price))
    else:
        rc = L.lib().qt_bdp_stopping(n, _u(tree.sizes), _u(tree.flat_visits), _f(tree.flat_pi),
                                     _f(phi), _f(value), exp, C.byref(price))
    _check(rc, "solve_stopping")
    vs, es, o = [], [], 0
    for k in range(n + 1):
        s = tree.layer_size(k)
        vs.append(value[o:o + s])
        es.append(ex[o:o + s])
        o += s
    return StoppingResult(vs, es, price.value)


def swing_window(n: int, qmin: int, qmax: int):
    lo = [max(0, qmin - (n - k)) for k in range(n + 1)]
    cnt = [min(k, qmax) - lo[k] + 1 for k in range(n + 1)]
    return lo, cnt


def solve_swing(tree: QuantTree, payoff, q_min: int, q_max: int) -> SwingResult:
    """Bang-bang swing recursion over (layer, node, consumption) (swing.hpp:47-129)."""
    if tree is None or payoff is None:
        raise ValueError("solve_swing: incomplete problem")
    phi = tabulate(tree, payoff)
    n = tree.layers()
    lo, cnt = swing_window(n, q_min, q_max)
    total = sum(max(c, 0) * tree.layer_size(k) for k, c in enumerate(cnt))
    vals = np.zeros(max(total, 1), np.float64)
    takes = np.zeros(max(total, 1), np.uint8)
    price = C.c_double()
    tkp = takes.ctypes.data_as(C.POINTER(C.c_uint8))
    if isinstance(tree, DeviceTree):  # in place on the device
        rc = L.lib().qt_dtree_swing(tree.handle(), _f(phi), int(q_min), int(q_max),
                                    C.byref(price), _f(vals), tkp)
    else:
        rc = L.lib().qt_bdp_swing(n, _u(tree.sizes), _u(tree.flat_visits), _f(tree.flat_pi),
                                  _f(phi), int(q_min), int(q_max), C.byref(price), _f(vals), tkp)
    _check(rc, "solve_swing")
    value, take, o = [], [], 0
    for k in range(n + 1):
        s = cnt[k] * tree.layer_size(k)
        value.append(vals[o:o + s])
        if k < n:
            take.append(takes[o:o + s])
        o += s
    return SwingResult(q_min, q_max, lo, cnt, value, take, price.value)


def cond_expectation(tree: QuantTree, k: int, f) -> np.ndarray:
    """E(f(X_{k+1}) | X_k = x_i) = pi^{k+1} f, NaN on unvisited rows (bdp.hpp:36-54)."""
    if k < 0 or k >= tree.layers():
        raise ValueError("cond_expectation: layer out of range")
    rows, cols = tree.layer_size(k), tree.layer_size(k + 1)
    f = np.ascontiguousarray(f, dtype=np.float64)
    if f.size != cols:
        raise ValueError("cond_expectation: value vector length mismatch")
    vo = int(tree.sizes[:k].sum())
    po = int(sum(int(tree.sizes[t]) * int(tree.sizes[t + 1]) for t in range(k)))
    vis = np.ascontiguousarray(tree.flat_visits[vo:vo + rows])
    pi = np.ascontiguousarray(tree.flat_pi[po:po + rows * cols])
    out = np.zeros(rows, np.float64)
    _check(L.lib().qt_bdp_cond_expectation(rows, cols, _u(vis), _f(pi), _f(f), _f(out)),
           "cond_expectation")
    return out


# ---------------------------------------------------------------------------
# grid inputs: the reference's per-layer mappings (pipeline.hpp:27-77) of the
# standard-normal Lloyd base quantizers, built on the GPU
# ---------------------------------------------------------------------------


@dataclass
class LloydResult:
    grid: "QuantGrid"
    distortion: np.ndarray


def lloyd_build(dim: int, n_points: int, iterations: int = 40, samples_per_iter: int = 0,
                seed: int = 12345, normals=None) -> LloydResult:
    """Randomized Lloyd on the GPU (lloyd.hpp:59-107) with the standard-normal
    sampler, on the serial MRG32k3a stream the reference's grid builders use
    (seed ^ 0x9E3779B9, pipeline.hpp:35,63). samples_per_iter 0 -> max(20000,
    200 N) (pipeline.hpp:18-20). normals: the stream's normals supplied (parity
    mode, bit-identical to the reference)."""
    spi = samples_per_iter or max(20000, 200 * n_points)
    out = np.zeros(n_points * dim, np.float64)
    dist = np.zeros(max(iterations, 1), np.float64)
    nrm = None if normals is None else np.ascontiguousarray(normals, np.float64)
    _check(L.lib().qt_lloyd_build(int(dim), int(n_points), int(iterations), int(spi),
                                  (int(seed) ^ 0x9E3779B9) & 0xFFFFFFFFFFFFFFFF,
                                  None if nrm is None else _f(nrm),
                                  0 if nrm is None else nrm.size, _f(out), _f(dist)),
           "lloyd_build")
    return LloydResult(QuantGrid(dim, out), dist[:iterations])


@functools.lru_cache(maxsize=16)
def _base_grid(grid_size: int, dim: int, seed: int) -> np.ndarray:
    g = np.asarray(lloyd_build(dim, grid_size, seed=seed).grid.data(), np.float64)
    g.setflags(write=False)
    return g


def base_grid(grid_size: int, dim: int, seed: int = 12345) -> np.ndarray:
    """The standard-normal base quantizer of the grid builders
    (lloyd_build(GaussianSampler{dim}, N, dim, 40, max(20000, 200 N), g),
    pipeline.hpp:27-77), built on the GPU. Bit-identical to the reference's:
    the device Box-Muller restates glibc's log/sincos, the projection is exact
    and every cell mean is summed in sample order (tests/test_lloyd.py against
    the reference's own grids, tests/golden/base_grids.npz). Cached per process."""
    return np.array(_base_grid(int(grid_size), int(dim), int(seed)))


def _cholesky2_marginal(p: TwoFactorParams, t: float):
    c11 = -math.expm1(-2.0 * p.alpha1 * t) / (2.0 * p.alpha1)
    c22 = -math.expm1(-2.0 * p.alpha2 * t) / (2.0 * p.alpha2)
    c12 = -p.rho * math.expm1(-(p.alpha1 + p.alpha2) * t) / (p.alpha1 + p.alpha2)
    l11 = math.sqrt(c11)
    l21 = c12 / l11 if l11 > 0.0 else 0.0
    rem = c22 - l21 * l21
    return l11, l21, math.sqrt(max(0.0, rem))


def build_brownian_grids(chain: BrownianChain1d, grid_size: int):
    """sqrt(t_k) times the N(0,1) base grid (pipeline.hpp:57-77)."""
    base = base_grid(grid_size, 1)
    return [QuantGrid(1, base * math.sqrt(chain.time(k))) for k in range(1, chain.layers() + 1)]


def build_two_factor_grids(chain: TwoFactorChain, grid_size: int):
    """Base grid mapped by the marginal Cholesky factor per layer (pipeline.hpp:27-53)."""
    base = base_grid(grid_size, 2).reshape(-1, 2)
    p = chain.params
    out = []
    for k in range(1, chain.layers() + 1):
        l11, l21, l22 = _cholesky2_marginal(p, k * (p.horizon / p.steps))
        z1, z2 = base[:, 0], base[:, 1]
        pts = np.stack([l11 * z1, l21 * z1 + l22 * z2], axis=1)
        out.append(QuantGrid(2, pts))
    return out


def build_ou_grids(chain: OuChain1d, grid_size: int):
    """Config 3: base grid times the factor-1 marginal sd of each layer."""
    base = base_grid(grid_size, 1)
    p = chain.params
    return [QuantGrid(1, base * _cholesky2_marginal(p, k * (p.horizon / p.steps))[0])
            for k in range(1, chain.layers() + 1)]


def build_gbm_grids(chain: GbmChain3d, grid_size: int):
    """Config 5: base grid mapped by sqrt(t_k) L per layer."""
    base = base_grid(grid_size, 3).reshape(-1, 3)
    m = chain.marg_coef.reshape(-1, 6)
    out = []
    for k in range(1, chain.layers() + 1):
        c = m[k]
        z0, z1, z2 = base[:, 0], base[:, 1], base[:, 2]
        pts = np.stack([c[0] * z0, c[1] * z0 + c[2] * z1, (c[3] * z0 + c[4] * z1) + c[5] * z2],
                       axis=1)
        out.append(QuantGrid(3, pts))
    return out
