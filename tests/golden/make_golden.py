"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Runs oracle/_ref/libqtree_ref.so (the unmodified reference headers compiled in
place by oracle/Makefile) in THIS container, where /root/reference exists, and
writes small .npz fixtures that travel with the repo:

  rng.npz          uniforms / skip-ahead / block substreams / path normals (3 engines)
  small_trees.npz  full counts+pi of small Alg I/II/III runs on all four chains
  configs.npz      BASELINE.json config grids' hashes, C1 counts hashes + put price,
                   C2-shape path-window hashes at M = 1e9
  pricing.npz      stopping / swing value tables on random row-stochastic trees

It also writes tests/golden/base_grids.npz: the standard-normal Lloyd base
quantizers the reference's grid builders map per layer (pipeline.hpp:27-77),
produced by the reference's own lloyd_build with its default seed convention.
The product builds them on the GPU (qt_lloyd_build); tests/test_lloyd.py
requires the two to be bit-identical.

Usage: python tests/golden/make_golden.py [--skip-c5]
"""
from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
from pyoracle import (  # noqa: E402
    ALG_I, ALG_II, ALG_III, CHAIN_BROWNIAN1D, CHAIN_GBM3D, CHAIN_OU1D, CHAIN_TWO_FACTOR,
    ChainSpec, Oracle, PAYOFF_PUT, PAYOFF_SWING)

OUT = os.path.join(ROOT, "tests", "golden")
DATA = os.path.join(ROOT, "tests", "golden")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def small_chain_spec(kind: int, steps: int) -> ChainSpec:
    # test_tree.cpp:18-27 small_chain parameters
    return ChainSpec(kind, steps, sigma1=0.4, sigma2=0.7, alpha1=0.8, alpha2=3.5, rho=0.3,
                     gbm_rho=(0.3, 0.1, -0.2))


def main() -> None:
    R = Oracle("reference")
    os.makedirs(DATA, exist_ok=True)
    t0 = time.time()

    # ---- RNG ----------------------------------------------------------------
    rng = {}
    for e, name in enumerate(("lcg48", "mrg32k3a", "xorwow")):
        rng[f"{name}_serial"] = R.uniforms(e, 12345, 64)
        rng[f"{name}_block"] = R.uniforms(e, 12345, 64, False, 5, 2, 1001)
        if e != 2:
            rng[f"{name}_skip"] = R.uniforms(e, 12345, 64, True, 7, 3)
        rng[f"{name}_paths"] = R.path_normals(e, 99, 11, 5, 4, 1000)
    np.savez_compressed(os.path.join(OUT, "rng.npz"), **rng)

    # ---- small trees ---------------------------------------------------------
    g = np.random.default_rng(20261017)
    st = {}
    for kind, tag in ((CHAIN_BROWNIAN1D, "bm"), (CHAIN_TWO_FACTOR, "tf"), (CHAIN_OU1D, "ou"),
                      (CHAIN_GBM3D, "gbm")):
        spec = small_chain_spec(kind, 5)
        n, N = 5, 24
        sizes = np.array([1] + [N] * n, np.uint64)
        pts = g.standard_normal(n * N * spec.dim)
        st[f"{tag}_sizes"] = sizes
        st[f"{tag}_pts"] = pts
        for alg, an in ((ALG_I, "alg1"), (ALG_III, "alg3")):
            for e, en in enumerate(("lcg48", "mrg32k3a", "xorwow")):
                c = R.estimate(alg, spec, sizes, pts, 4000, engine=e, seed=99, workers=3)
                st[f"{tag}_{an}_{en}_visits"] = c.visits
                st[f"{tag}_{an}_{en}_joint"] = c.joint
                st[f"{tag}_{an}_{en}_pi"] = c.pi
        # one window of a large run: paths [777, 777+300) of 10^6
        v, j = R.accumulate_paths(spec, sizes, pts, 1, 12345, 777, 300, 10**6)
        st[f"{tag}_window_visits"] = v
        st[f"{tag}_window_joint"] = j
    np.savez_compressed(os.path.join(OUT, "small_trees.npz"), **st)

    # ---- base grids (fixture: the GPU Lloyd must reproduce them bit for bit) ----
    bases = {}
    for tag, dim, N in (("n100_d1", 1, 100), ("n500_d1", 1, 500), ("n200_d1", 1, 200),
                        ("n1000_d2", 2, 1000)):
        bases[tag] = R.lloyd_base(dim, N)
        print(f"base {tag} done {time.time() - t0:.1f}s", flush=True)
    if "--skip-c5" not in sys.argv:
        bases["n4000_d3"] = R.lloyd_base(3, 4000)
        print(f"base n4000_d3 done {time.time() - t0:.1f}s", flush=True)
    else:
        old = os.path.join(DATA, "base_grids.npz")
        if os.path.exists(old):
            with np.load(old) as z:
                if "n4000_d3" in z:
                    bases["n4000_d3"] = z["n4000_d3"]
    np.savez_compressed(os.path.join(DATA, "base_grids.npz"), **bases)

    # ---- configs -------------------------------------------------------------
    cf = {}
    c1 = ChainSpec(CHAIN_BROWNIAN1D, 10, sigma1=0.2, r=0.05)
    g1 = R.build_grids(c1, 100)
    cf["c1_grid_sha"] = np.array(sha(g1))
    s1 = np.array([1] + [100] * 10, np.uint64)
    cnt = R.estimate(ALG_II, c1, s1, g1, 10**6, workers=8)
    cf["c1_visits"] = cnt.visits
    cf["c1_joint_sha"] = np.array(sha(cnt.joint))
    cf["c1_pi_sha"] = np.array(sha(cnt.pi))
    pts_all = np.concatenate([[0.0], g1])
    phi = R.payoff_table(c1, PAYOFF_PUT, s1, pts_all)
    cf["c1_put_price"] = np.array(R.solve_stopping(s1, cnt.visits, cnt.pi, phi)[0])
    print(f"c1 done {time.time() - t0:.1f}s", flush=True)

    c2 = ChainSpec(CHAIN_BROWNIAN1D, 50, sigma1=0.2, r=0.05)
    g2 = R.build_grids(c2, 500)
    cf["c2_grid_sha"] = np.array(sha(g2))
    s2 = np.array([1] + [500] * 50, np.uint64)
    for first in (0, 123456789, 999980000):
        v, j = R.accumulate_paths(c2, s2, g2, 1, 12345, first, 20000, 10**9)
        cf[f"c2_win{first}_visits"] = v
        cf[f"c2_win{first}_joint_sha"] = np.array(sha(j))
    print(f"c2 windows done {time.time() - t0:.1f}s", flush=True)

    c3 = ChainSpec(CHAIN_OU1D, 365, sigma1=0.5, alpha1=1.0, sigma2=0.0)
    cf["c3_grid_sha"] = np.array(sha(R.build_grids(c3, 200)))
    c4 = ChainSpec(CHAIN_TWO_FACTOR, 365)
    cf["c4_grid_sha"] = np.array(sha(R.build_grids(c4, 1000)))
    np.savez_compressed(os.path.join(OUT, "configs.npz"), **cf)

    # ---- pricing ---------------------------------------------------------------
    pr = {}
    for case, (n, N, qmin, qmax) in enumerate(((4, 3, 0, 4), (6, 5, 2, 4), (8, 3, 3, 3),
                                               (12, 7, 0, 12))):
        sizes = np.array([1] + [N] * n, np.uint64)
        joint = g.integers(1, 41, size=sum(int(sizes[k - 1] * sizes[k]) for k in range(1, n + 1)),
                           dtype=np.uint64)
        # a few unvisited rows (absorbing nodes)
        off = int(sizes[0] * sizes[1])
        joint[off:off + N] = 0
        visits = np.zeros(int(sizes.sum()), np.uint64)
        vo, jo = 0, 0
        for k in range(1, n + 1):
            r, c = int(sizes[k - 1]), int(sizes[k])
            blk = joint[jo:jo + r * c].reshape(r, c)
            visits[vo:vo + r] = blk.sum(axis=1)
            vo += r
            jo += r * c
        visits[vo:] = joint[jo - int(sizes[n - 1] * sizes[n]):jo].reshape(
            int(sizes[n - 1]), int(sizes[n])).sum(axis=0)
        pi = R.normalize(sizes, visits, joint)
        phi = g.uniform(-1.0, 1.0, size=int(sizes.sum()))
        price, value, ex = R.solve_stopping(sizes, visits, pi, phi)
        sprice, svals = R.solve_swing(sizes, visits, pi, phi, qmin, qmax, True)
        for key, val in (("sizes", sizes), ("visits", visits), ("joint", joint), ("pi", pi),
                         ("phi", phi), ("stop_price", np.array(price)), ("stop_value", value),
                         ("stop_exercise", ex), ("swing_q", np.array([qmin, qmax])),
                         ("swing_price", np.array(sprice)), ("swing_values", svals)):
            pr[f"case{case}_{key}"] = val
    np.savez_compressed(os.path.join(OUT, "pricing.npz"), **pr)
    print(f"all done {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
