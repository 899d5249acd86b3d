"""TEST INFRASTRUCTURE ONLY: numpy/ctypes front end of the CPU checkers.

Loads either checker behind oracle/oracle_api.h:
  * ``Oracle("restatement")`` -> oracle/build/libqtree_oracle.so (C restatement)
  * ``Oracle("reference")``   -> oracle/_ref/libqtree_ref.so (the unmodified
    reference headers compiled in place by oracle/Makefile)

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline leg may
import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "restatement": os.path.join(HERE, "build", "libqtree_oracle.so"),
    "reference": os.path.join(HERE, "_ref", "libqtree_ref.so"),
}

CHAIN_BROWNIAN1D, CHAIN_TWO_FACTOR, CHAIN_OU1D, CHAIN_GBM3D = 0, 1, 2, 3
ENGINE_LCG48, ENGINE_MRG32K3A, ENGINE_XORWOW = 0, 1, 2
ALG_I, ALG_II, ALG_III = 0, 1, 2
PAYOFF_PUT, PAYOFF_CALL, PAYOFF_SWING, PAYOFF_MAXCALL = 0, 1, 2, 3

ERRORS = {1: "invalid_argument", 2: "ConfigError", 3: "IoError", 4: "NumericError", 9: "other"}


class OracleError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {ERRORS.get(code, code)}")
        self.code = code
        self.kind = ERRORS.get(code, str(code))


class _Chain(C.Structure):
    _fields_ = [
        ("kind", C.c_int), ("steps", C.c_int), ("horizon", C.c_double),
        ("s0", C.c_double), ("sigma1", C.c_double), ("sigma2", C.c_double),
        ("alpha1", C.c_double), ("alpha2", C.c_double), ("rho", C.c_double),
        ("r", C.c_double), ("strike", C.c_double),
        ("gbm_sigma", C.c_double * 3), ("gbm_rho", C.c_double * 3),
    ]


@dataclass
class ChainSpec:
    """Model by parameters (TwoFactorParams defaults, two_factor.hpp:16-26)."""
    kind: int
    steps: int
    horizon: float = 1.0
    s0: float = 100.0
    sigma1: float = 0.5
    sigma2: float = 0.3
    alpha1: float = 1.0
    alpha2: float = 4.0
    rho: float = 0.0
    r: float = 0.0
    strike: float = 100.0
    gbm_sigma: tuple = (0.2, 0.2, 0.2)
    gbm_rho: tuple = (0.0, 0.0, 0.0)

    def c(self) -> _Chain:
        return _Chain(self.kind, self.steps, self.horizon, self.s0, self.sigma1, self.sigma2,
                      self.alpha1, self.alpha2, self.rho, self.r, self.strike,
                      (C.c_double * 3)(*self.gbm_sigma), (C.c_double * 3)(*self.gbm_rho))

    @property
    def dim(self) -> int:
        return {0: 1, 1: 2, 2: 1, 3: 3}[self.kind]

    @property
    def nps(self) -> int:
        return self.dim


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def ensure_built(which: str) -> str:
    path = LIBS[which]
    if not os.path.exists(path):
        target = "restatement" if which == "restatement" else "ref"
        subprocess.run(["make", "-s", "-C", HERE, target], check=True)
    if not os.path.exists(path):
        raise FileNotFoundError(path)
    return path


@dataclass
class Counts:
    visits: np.ndarray
    joint: np.ndarray
    pi: np.ndarray
    phases: np.ndarray = field(default_factory=lambda: np.zeros(5))


def layout(sizes):
    sizes = [int(s) for s in sizes]
    nvis = sum(sizes)
    njoint = sum(sizes[k - 1] * sizes[k] for k in range(1, len(sizes)))
    return nvis, njoint


class Oracle:
    def __init__(self, which: str = "restatement"):
        self.which = which
        self.lib = C.CDLL(ensure_built(which))
        u64p, f64p = C.POINTER(C.c_uint64), C.POINTER(C.c_double)
        L = self.lib
        L.oq_estimate.argtypes = [C.c_int, C.POINTER(_Chain), u64p, f64p, C.c_uint64, C.c_int,
                                  C.c_uint64, C.c_int, u64p, u64p, f64p, f64p]
        L.oq_accumulate_paths.argtypes = [C.POINTER(_Chain), u64p, f64p, C.c_int, C.c_uint64,
                                          C.c_uint64, C.c_uint64, C.c_uint64, u64p, u64p]
        L.oq_path_normals.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64,
                                      C.c_uint64, f64p]
        L.oq_uniforms.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_uint64, C.c_uint64,
                                  C.c_uint64, C.c_uint64, f64p]
        L.oq_nearest_brute.argtypes = [C.c_int, C.c_uint64, f64p, C.c_uint64, f64p, u64p]
        L.oq_normalize.argtypes = [C.c_int, u64p, u64p, u64p, f64p]
        L.oq_payoff_table.argtypes = [C.POINTER(_Chain), C.c_int, u64p, f64p, f64p]
        L.oq_solve_stopping.argtypes = [C.c_int, u64p, u64p, f64p, f64p, f64p,
                                        C.POINTER(C.c_uint8), f64p]
        L.oq_solve_swing.argtypes = [C.c_int, u64p, u64p, f64p, f64p, C.c_int, C.c_int, f64p,
                                     f64p]
        L.oq_lloyd_base.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, f64p]
        L.oq_build_grids.argtypes = [C.POINTER(_Chain), C.c_uint64, C.c_uint64, C.c_uint64,
                                     C.c_int, f64p]

    def _check(self, rc, where):
        if rc:
            raise OracleError(rc, f"{self.which}.{where}")

    def estimate(self, alg, chain: ChainSpec, sizes, pts, paths, engine=ENGINE_MRG32K3A,
                 seed=12345, workers=1) -> Counts:
        sizes = np.ascontiguousarray(sizes, dtype=np.uint64)
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        nvis, njoint = layout(sizes)
        v = np.zeros(nvis, np.uint64)
        j = np.zeros(njoint, np.uint64)
        pi = np.zeros(njoint, np.float64)
        ph = np.zeros(5, np.float64)
        c = chain.c()
        rc = self.lib.oq_estimate(alg, C.byref(c), _p(sizes, C.c_uint64), _p(pts, C.c_double),
                                  paths, engine, seed, workers, _p(v, C.c_uint64),
                                  _p(j, C.c_uint64), _p(pi, C.c_double), _p(ph, C.c_double))
        self._check(rc, "estimate")
        return Counts(v, j, pi, ph)

    def accumulate_paths(self, chain, sizes, pts, engine, seed, first, count, total):
        sizes = np.ascontiguousarray(sizes, dtype=np.uint64)
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        nvis, njoint = layout(sizes)
        v = np.zeros(nvis, np.uint64)
        j = np.zeros(njoint, np.uint64)
        c = chain.c()
        rc = self.lib.oq_accumulate_paths(C.byref(c), _p(sizes, C.c_uint64), _p(pts, C.c_double),
                                          engine, seed, first, count, total, _p(v, C.c_uint64),
                                          _p(j, C.c_uint64))
        self._check(rc, "accumulate_paths")
        return v, j

    def path_normals(self, engine, seed, normals_per_path, first, count, total):
        out = np.zeros(int(count) * int(normals_per_path), np.float64)
        rc = self.lib.oq_path_normals(engine, seed, normals_per_path, first, count, total,
                                      _p(out, C.c_double))
        self._check(rc, "path_normals")
        return out

    def uniforms(self, engine, seed, n, skip_ahead=False, streams=1, index=0, block=1):
        out = np.zeros(int(n), np.float64)
        rc = self.lib.oq_uniforms(engine, seed, int(skip_ahead), streams, index, block, n,
                                  _p(out, C.c_double))
        self._check(rc, "uniforms")
        return out

    def nearest(self, dim, pts, queries):
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        q = np.ascontiguousarray(queries, dtype=np.float64)
        nq = q.size // dim
        out = np.zeros(nq, np.uint64)
        rc = self.lib.oq_nearest_brute(dim, pts.size // dim, _p(pts, C.c_double), nq,
                                       _p(q, C.c_double), _p(out, C.c_uint64))
        self._check(rc, "nearest")
        return out

    def normalize(self, sizes, visits, joint):
        sizes = np.ascontiguousarray(sizes, dtype=np.uint64)
        visits = np.ascontiguousarray(visits, dtype=np.uint64)
        joint = np.ascontiguousarray(joint, dtype=np.uint64)
        pi = np.zeros(joint.size, np.float64)
        self._check(self.lib.oq_normalize(len(sizes) - 1, _p(sizes, C.c_uint64),
                                          _p(visits, C.c_uint64), _p(joint, C.c_uint64),
                                          _p(pi, C.c_double)), "normalize")
        return pi

    def payoff_table(self, chain, payoff, sizes, pts_all):
        sizes = np.ascontiguousarray(sizes, dtype=np.uint64)
        pts_all = np.ascontiguousarray(pts_all, dtype=np.float64)
        phi = np.zeros(int(sizes.sum()), np.float64)
        c = chain.c()
        self._check(self.lib.oq_payoff_table(C.byref(c), payoff, _p(sizes, C.c_uint64),
                                             _p(pts_all, C.c_double), _p(phi, C.c_double)),
                    "payoff_table")
        return phi

    def solve_stopping(self, sizes, visits, pi, phi):
        sizes = np.ascontiguousarray(sizes, dtype=np.uint64)
        visits = np.ascontiguousarray(visits, dtype=np.uint64)
        pi = np.ascontiguousarray(pi, dtype=np.float64)
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        value = np.zeros(int(sizes.sum()), np.float64)
        ex = np.zeros(int(sizes.sum()), np.uint8)
        price = C.c_double(0.0)
        self._check(self.lib.oq_solve_stopping(len(sizes) - 1, _p(sizes, C.c_uint64),
                                               _p(visits, C.c_uint64), _p(pi, C.c_double),
                                               _p(phi, C.c_double), _p(value, C.c_double),
                                               _p(ex, C.c_uint8), C.byref(price)),
                    "solve_stopping")
        return price.value, value, ex

    def solve_swing(self, sizes, visits, pi, phi, qmin, qmax, want_values=False):
        sizes = np.ascontiguousarray(sizes, dtype=np.uint64)
        visits = np.ascontiguousarray(visits, dtype=np.uint64)
        pi = np.ascontiguousarray(pi, dtype=np.float64)
        phi = np.ascontiguousarray(phi, dtype=np.float64)
        n = len(sizes) - 1
        total = sum((min(k, qmax) - max(0, qmin - (n - k)) + 1) * int(sizes[k])
                    for k in range(n + 1))
        vals = np.zeros(max(total, 1), np.float64) if want_values else None
        price = C.c_double(0.0)
        self._check(self.lib.oq_solve_swing(n, _p(sizes, C.c_uint64), _p(visits, C.c_uint64),
                                            _p(pi, C.c_double), _p(phi, C.c_double), qmin,
                                            qmax, C.byref(price),
                                            _p(vals, C.c_double) if want_values else None),
                    "solve_swing")
        return (price.value, vals) if want_values else price.value

    def build_grids(self, chain: ChainSpec, grid_size, seed=12345, per_iter=0, iterations=40):
        out = np.zeros(chain.steps * grid_size * chain.dim, np.float64)
        c = chain.c()
        self._check(self.lib.oq_build_grids(C.byref(c), grid_size, seed, per_iter, iterations,
                                            _p(out, C.c_double)), "build_grids")
        return out

    # --- files (reference harness only: the reference's own save_tree etc.) ---
    def save_tree(self, path, dim, sizes, pts_all, samples, visits, joint, pi):
        sizes = np.ascontiguousarray(sizes, dtype=np.uint64)
        L = self.lib
        L.oq_save_tree.argtypes = [C.c_char_p, C.c_int, C.c_int, C.POINTER(C.c_uint64),
                                   C.POINTER(C.c_double), C.c_uint64, C.POINTER(C.c_uint64),
                                   C.POINTER(C.c_uint64), C.POINTER(C.c_double)]
        pa = np.ascontiguousarray(pts_all, dtype=np.float64)
        v = np.ascontiguousarray(visits, dtype=np.uint64)
        j = np.ascontiguousarray(joint, dtype=np.uint64)
        pi_ = np.ascontiguousarray(pi, dtype=np.float64)
        self._check(L.oq_save_tree(str(path).encode(), len(sizes) - 1, dim, _p(sizes, C.c_uint64),
                                   _p(pa, C.c_double), samples, _p(v, C.c_uint64),
                                   _p(j, C.c_uint64), _p(pi_, C.c_double)), "save_tree")

    def load_tree(self, path, max_layers, max_points, max_joint):
        L = self.lib
        u64p, f64p, ip = C.POINTER(C.c_uint64), C.POINTER(C.c_double), C.POINTER(C.c_int)
        L.oq_load_tree.argtypes = [C.c_char_p, ip, ip, u64p, u64p, f64p, u64p, u64p, f64p]
        n, d, m = C.c_int(0), C.c_int(0), C.c_uint64(0)
        sizes = np.zeros(max_layers + 1, np.uint64)
        pts = np.zeros(max_points, np.float64)
        v = np.zeros(max_points, np.uint64)
        j = np.zeros(max_joint, np.uint64)
        pi = np.zeros(max_joint, np.float64)
        self._check(L.oq_load_tree(str(path).encode(), C.byref(n), C.byref(d), C.byref(m),
                                   _p(sizes, C.c_uint64), _p(pts, C.c_double), _p(v, C.c_uint64),
                                   _p(j, C.c_uint64), _p(pi, C.c_double)), "load_tree")
        sizes = sizes[:n.value + 1]
        nvis, njoint = layout(sizes)
        return (n.value, d.value, m.value, sizes, pts[:nvis * d.value], v[:nvis], j[:njoint],
                pi[:njoint])

    def save_grid(self, path, dim, pts):
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        L = self.lib
        L.oq_save_grid.argtypes = [C.c_char_p, C.c_int, C.c_uint64, C.POINTER(C.c_double)]
        self._check(L.oq_save_grid(str(path).encode(), dim, pts.size // dim, _p(pts, C.c_double)),
                    "save_grid")

    def bench_pi(self, engine, seed, samples, streams, skip):
        L = self.lib
        L.oq_bench_pi.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_int,
                                  C.POINTER(C.c_double), C.POINTER(C.c_double)]
        e, se = C.c_double(0), C.c_double(0)
        self._check(L.oq_bench_pi(engine, seed, samples, streams, int(skip), C.byref(e),
                                  C.byref(se)), "bench_pi")
        return e.value, se.value

    def bench_nn(self, n, queries, seed):
        L = self.lib
        L.oq_bench_nn.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]
        s = C.c_uint64(0)
        self._check(L.oq_bench_nn(n, queries, seed, C.byref(s)), "bench_nn")
        return s.value

    def lloyd_base(self, dim, grid_size, seed=12345, per_iter=0, iterations=40):
        out = np.zeros(grid_size * dim, np.float64)
        self._check(self.lib.oq_lloyd_base(dim, grid_size, seed, per_iter, iterations,
                                           _p(out, C.c_double)), "lloyd_base")
        return out
