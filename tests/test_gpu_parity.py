"""Parity of the CUDA path against the CPU checker, through the C ABI.

Bar: bit-exact cell indices, counts, visits and pi (integer / index work and
a correctly rounded division), bit-exact BDP values (sequential row sums in
the reference's order). The in-kernel normals are bit-identical to the
reference's by construction (csrc/qt_math.h restates the glibc log/sincos the
reference calls; exhaustive over the MRG32k3a and XORWOW domains), so the
in-kernel counts are the reference's; the seeded configs below check that."""
from __future__ import annotations

import hashlib

import numpy as np
import pytest

from pyoracle import (ALG_I, ALG_II, ALG_III, CHAIN_BROWNIAN1D, CHAIN_GBM3D, CHAIN_OU1D,
                      CHAIN_TWO_FACTOR, ChainSpec, PAYOFF_PUT, PAYOFF_SWING)

pytestmark = pytest.mark.gpu

ENGINES = ("lcg48", "mrg32k3a", "xorwow")
TAGS = {"bm": CHAIN_BROWNIAN1D, "tf": CHAIN_TWO_FACTOR, "ou": CHAIN_OU1D, "gbm": CHAIN_GBM3D}


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def Q():
    from paper_1101_3228_b200 import qtree
    return qtree


def product_chain(spec: ChainSpec):
    q = Q()
    p = q.TwoFactorParams(s0=spec.s0, sigma1=spec.sigma1, sigma2=spec.sigma2, alpha1=spec.alpha1,
                          alpha2=spec.alpha2, rho=spec.rho, r=spec.r, strike=spec.strike,
                          horizon=spec.horizon, steps=spec.steps)
    if spec.kind == CHAIN_BROWNIAN1D:
        return q.BrownianChain1d(spec.steps, spec.horizon)
    if spec.kind == CHAIN_TWO_FACTOR:
        return q.TwoFactorChain(p)
    if spec.kind == CHAIN_OU1D:
        return q.OuChain1d(p)
    return q.GbmChain3d(spec.steps, spec.horizon, spec.gbm_rho)


def product_grids(spec, sizes, pts):
    q = Q()
    out, o = [], 0
    for s in sizes[1:]:
        s = int(s)
        out.append(q.QuantGrid(spec.dim, pts[o:o + s * spec.dim]))
        o += s * spec.dim
    return out


def small_spec(kind, steps=5):
    return ChainSpec(kind, steps, sigma1=0.4, sigma2=0.7, alpha1=0.8, alpha2=3.5, rho=0.3,
                     gbm_rho=(0.3, 0.1, -0.2))


def assert_tree_equal(t, visits, joint, pi):
    assert np.array_equal(t.flat_joint, joint)
    assert np.array_equal(t.flat_visits, visits)
    assert np.array_equal(t.flat_pi, pi)


# --- RNG ----------------------------------------------------------------------
def test_uniforms_bit_exact(gpu, oracle):
    q = Q()
    for e in (0, 1):
        for off in (0, 1, 12345, 10**9 + 7, 2**40 + 3):
            # block substream `off` of size 1 starts at serial draw `off` (stream.hpp:156-158)
            ref = oracle.uniforms(e, 12345, 257, False, off + 1, off, 1)
            got = q.uniforms(e, 12345, off, 257)
            assert np.array_equal(got, ref), (e, off)


def test_normals_bit_identical_to_glibc(gpu, oracle):
    """In-kernel Box-Muller vs the oracle's (glibc log + sincos): 0 ulp on
    1e8 normals per engine (2e6 paths x 50 normals, in chunks)."""
    q = Q()
    for e in range(3):
        for c in range(10):
            first = 10**9 // 3 * e + c * 200000 + 17
            ref = oracle.path_normals(e, 12345, 50, first, 200000, 10**9)
            got = q.path_normals(e, 12345, 50, first, 200000)
            bad = np.flatnonzero(got.view(np.int64) != ref.view(np.int64))
            assert bad.size == 0, (e, c, int(bad.size), bad[:5].tolist())


def test_math_checksum_exhaustive(gpu):
    """The device log / sin / cos over EVERY MRG32k3a and XORWOW uniform equal
    glibc's (order-independent checksums, tests/golden/glibc_checksums.json)."""
    import json
    import os
    here = os.path.dirname(os.path.abspath(__file__))
    with open(os.path.join(here, "golden", "glibc_checksums.json")) as f:
        g = json.load(f)
    for dom, name in ((0, "mrg32k3a"), (1, "xorwow")):
        got = [str(int(v)) for v in Q().math_checksum(dom)]
        assert got == g[name], (name, got, g[name])


# --- estimator, parity mode (reference normals in) -------------------------------
@pytest.mark.parametrize("tag", list(TAGS))
@pytest.mark.parametrize("alg", [ALG_I, ALG_II, ALG_III])
def test_normals_in_bit_exact(gpu, oracle, golden, tag, alg):
    st = golden["small_trees"]
    spec = small_spec(TAGS[tag])
    sizes, pts = st[f"{tag}_sizes"], st[f"{tag}_pts"]
    n, d = spec.steps, spec.dim
    M = 3000
    if alg == ALG_III:
        normals = oracle.path_normals(1, 42, 2 * d, 0, n * M, n * M)
    else:
        normals = oracle.path_normals(1, 42, n * d, 0, M, M)
    ref = oracle.estimate(alg, spec, sizes, pts, M, engine=1, seed=42, workers=2)
    t = Q().estimate_with_normals(alg, product_chain(spec), product_grids(spec, sizes, pts), M,
                                  normals)
    assert_tree_equal(t, ref.visits, ref.joint, ref.pi)


# --- estimator, in-kernel stream ---------------------------------------------------
@pytest.mark.parametrize("tag", list(TAGS))
def test_small_trees_all_engines(gpu, golden, tag):
    st = golden["small_trees"]
    spec = small_spec(TAGS[tag])
    sizes, pts = st[f"{tag}_sizes"], st[f"{tag}_pts"]
    q = Q()
    ch, grids = product_chain(spec), product_grids(spec, sizes, pts)
    for alg, an in ((ALG_I, "alg1"), (ALG_III, "alg3")):
        for e, en in enumerate(ENGINES):
            t = q.estimate(alg, ch, grids, 4000, q.EstimateOptions(engine=e, seed=99))
            assert_tree_equal(t, st[f"{tag}_{an}_{en}_visits"], st[f"{tag}_{an}_{en}_joint"],
                              st[f"{tag}_{an}_{en}_pi"])
    v, j = q.accumulate_paths(ch, grids, 1, 12345, 777, 300, 10**6)
    assert np.array_equal(v, st[f"{tag}_window_visits"])
    assert np.array_equal(j, st[f"{tag}_window_joint"])


def test_alg2_equals_alg1_and_device_sharding(gpu, golden):
    # worker-count invariance (test_tree.cpp:128-152) -> shard invariance
    st = golden["small_trees"]
    spec = small_spec(CHAIN_TWO_FACTOR)
    q = Q()
    ch, grids = product_chain(spec), product_grids(spec, st["tf_sizes"], st["tf_pts"])
    base = q.estimate_alg1(ch, grids, 4000, q.EstimateOptions(seed=99))
    t = q.estimate_alg2(ch, grids, 4000, q.EstimateOptions(seed=99, workers=8))
    assert_tree_equal(t, base.flat_visits, base.flat_joint, base.flat_pi)
    import torch
    from paper_1101_3228_b200.device import Plan
    plan = Plan(ch, grids, 0)
    for shards in (1, 2, 3, 8):
        joint = plan.zeros_joint()
        for s in range(shards):
            b, e = 4000 * s // shards, 4000 * (s + 1) // shards
            plan.count(1, 1, 99, b, e - b, 4000, joint)
        torch.cuda.synchronize()
        assert np.array_equal(joint.cpu().numpy().view(np.uint64), base.flat_joint)


def test_1d_sorted_cell_counts_accumulate_over_windows(gpu):
    """k_paths_x / k_alg3_x count in sorted-cell space into a plan scratch and
    permute-add into the caller's joint: windowed plan.count calls must add up
    to the one-call tree (Alg II, Brownian and OU; Alg III, OU), twice over
    the same joint doubling it."""
    import torch
    from paper_1101_3228_b200.device import Plan
    q = Q()
    ou = q.OuChain1d(q.TwoFactorParams(sigma1=0.5, alpha1=1.0, sigma2=0.0, steps=6))
    cases = [(1, q.BrownianChain1d(6), 20000), (1, ou, 20000), (2, ou, 3000)]
    for alg, ch, M in cases:
        grids = (q.build_ou_grids(ch, 40) if isinstance(ch, q.OuChain1d)
                 else q.build_brownian_grids(ch, 40))
        ref = q.estimate(alg, ch, grids, M)
        units = M * 6 if alg == 2 else M
        plan = Plan(ch, grids, 0)
        for shards in (1, 3, 8):
            joint = plan.zeros_joint()
            for s in range(shards):
                b, e = units * s // shards, units * (s + 1) // shards
                plan.count(alg, 1, 12345, b, e - b, units, joint)
            torch.cuda.synchronize()
            assert np.array_equal(joint.cpu().numpy().view(np.uint64), ref.flat_joint), (alg, shards)
        plan.count(alg, 1, 12345, 0, units, units, joint)
        torch.cuda.synchronize()
        assert np.array_equal(joint.cpu().numpy().view(np.uint64), 2 * ref.flat_joint)


def test_one_call_plan_cache_is_keyed_by_inputs(gpu, oracle):
    """qt_estimate caches plans by every input byte: a repeat on the same grids
    reuses it, a grid with one point moved or other coefficients must not,
    and every result equals the oracle (the reference's restatement)."""
    q = Q()
    spec = ChainSpec(CHAIN_BROWNIAN1D, 5, sigma1=0.2, r=0.05)
    ch = q.BrownianChain1d(5)
    grids = q.build_brownian_grids(ch, 30)
    moved = [q.QuantGrid(1, g.data().copy()) for g in grids]
    moved[2].points[7] += 1e-9  # one bit of one point: a different grid
    ch2 = q.BrownianChain1d(5, 2.0)  # same grids, other step coefficients
    for chain, gr, sp in ((ch, grids, spec), (ch, grids, spec), (ch, moved, spec),
                          (ch2, grids, ChainSpec(CHAIN_BROWNIAN1D, 5, sigma1=0.2, r=0.05,
                                                 horizon=2.0)),
                          (ch, grids, spec)):
        t = q.estimate_alg2(chain, gr, 5000)
        pts = np.concatenate([g.data() for g in gr])
        ref = oracle.estimate(ALG_II, sp, t.sizes, pts, 5000, workers=2)
        assert np.array_equal(t.flat_joint, ref.joint)
        assert np.array_equal(t.flat_visits, ref.visits)


def test_plan_cache_clear_and_disable(gpu, monkeypatch):
    """qt_plan_cache_clear() drops the cached plans (their device memory is
    freed: the next call rebuilds), QT_PLAN_CACHE=0 keeps none; results equal
    the cached call's either way."""
    import torch
    q = Q()
    ch = q.BrownianChain1d(10)
    grids = q.build_brownian_grids(ch, 100)
    a = q.estimate_alg2(ch, grids, 200000)
    torch.cuda.synchronize()
    q.plan_cache_clear()
    free0 = torch.cuda.mem_get_info()[0]
    b = q.estimate_alg2(ch, grids, 200000)  # rebuilt and cached again
    torch.cuda.synchronize()
    free1 = torch.cuda.mem_get_info()[0]
    assert free1 < free0  # the new plan holds device memory
    q.plan_cache_clear()
    assert torch.cuda.mem_get_info()[0] > free1  # and clearing returns it
    monkeypatch.setenv("QT_PLAN_CACHE", "0")
    c = q.estimate_alg2(ch, grids, 200000)
    for t in (b, c):
        assert np.array_equal(t.flat_joint, a.flat_joint)
        assert np.array_equal(t.flat_pi, a.flat_pi)


def test_c1_config_bit_exact(gpu, oracle, golden):
    """BASELINE config 1: 1-D BS put, n=10, N=100, M=1e6, MRG32k3a seed 12345."""
    q = Q()
    cf = golden["configs"]
    ch = q.BrownianChain1d(10)
    grids = q.build_brownian_grids(ch, 100)
    t = q.estimate_alg2(ch, grids, 10**6)
    assert np.array_equal(t.flat_visits, cf["c1_visits"])
    assert sha(t.flat_joint) == str(cf["c1_joint_sha"])
    assert sha(t.flat_pi) == str(cf["c1_pi_sha"])
    spec = ChainSpec(CHAIN_BROWNIAN1D, 10, sigma1=0.2, r=0.05)
    pts_all = np.concatenate([[0.0]] + [g.data() for g in grids])
    phi = oracle.payoff_table(spec, PAYOFF_PUT, t.sizes, pts_all)
    res = q.solve_stopping(t, phi)
    assert res.price == float(cf["c1_put_price"])


def test_c2_windows_bit_exact(gpu, golden):
    """BASELINE config 2 (n=50, N=500, M=1e9): three 20000-path windows."""
    q = Q()
    cf = golden["configs"]
    ch = q.BrownianChain1d(50)
    grids = q.build_brownian_grids(ch, 500)
    for first in (0, 123456789, 999980000):
        v, j = q.accumulate_paths(ch, grids, 1, 12345, first, 20000, 10**9)
        assert np.array_equal(v, cf[f"c2_win{first}_visits"]), first
        assert sha(j) == str(cf[f"c2_win{first}_joint_sha"]), first


def test_c2_random_window_vs_oracle(gpu, oracle):
    q = Q()
    ch = q.BrownianChain1d(50)
    grids = q.build_brownian_grids(ch, 500)
    spec = ChainSpec(CHAIN_BROWNIAN1D, 50)
    sizes = np.array([1] + [500] * 50, np.uint64)
    pts = np.concatenate([g.data() for g in grids])
    rng = np.random.default_rng(2026)
    for first in rng.integers(0, 10**9 - 50000, size=2):
        v, j = q.accumulate_paths(ch, grids, 1, 12345, int(first), 50000, 10**9)
        rv, rj = oracle.accumulate_paths(spec, sizes, pts, 1, 12345, int(first), 50000, 10**9)
        assert np.array_equal(v, rv) and np.array_equal(j, rj), int(first)


def test_c3_c4_shapes_vs_oracle(gpu, oracle):
    q = Q()
    # C3: OU 1-D, Alg III, n = 365, N = 200 (reduced M)
    p = q.TwoFactorParams(sigma1=0.5, alpha1=1.0, sigma2=0.0, steps=365)
    ch = q.OuChain1d(p)
    grids = q.build_ou_grids(ch, 200)
    spec = ChainSpec(CHAIN_OU1D, 365, sigma1=0.5, alpha1=1.0, sigma2=0.0)
    sizes = np.array([1] + [200] * 365, np.uint64)
    pts = np.concatenate([g.data() for g in grids])
    t = q.estimate_alg3(ch, grids, 2000)
    r = oracle.estimate(ALG_III, spec, sizes, pts, 2000, workers=8)
    assert_tree_equal(t, r.visits, r.joint, r.pi)
    # C4: 2-factor, n = 365, N = 1000 (reduced M)
    tf = q.TwoFactorChain(q.TwoFactorParams())
    g4 = q.build_two_factor_grids(tf, 1000)
    spec4 = ChainSpec(CHAIN_TWO_FACTOR, 365)
    s4 = np.array([1] + [1000] * 365, np.uint64)
    p4 = np.concatenate([g.data() for g in g4])
    v, j = q.accumulate_paths(tf, g4, 1, 12345, 5000, 600, 10**8)
    rv, rj = oracle.accumulate_paths(spec4, s4, p4, 1, 12345, 5000, 600, 10**8)
    assert np.array_equal(v, rv) and np.array_equal(j, rj)


def test_conservation_at_scale(gpu):
    """Sum of counts per transition = M at a size the oracle cannot run."""
    import torch
    q = Q()
    from paper_1101_3228_b200.device import Plan
    ch = q.BrownianChain1d(50)
    plan = Plan(ch, q.build_brownian_grids(ch, 500), 0)
    M = 10**8
    joint = plan.zeros_joint()
    plan.count(1, 1, 12345, 0, M, M, joint)
    visits = torch.zeros(plan.n_visits, dtype=torch.int64, device="cuda")
    pi = torch.zeros(plan.n_joint, dtype=torch.float64, device="cuda")
    plan.finalize(1, M, joint, visits, pi)
    torch.cuda.synchronize()
    j = joint.cpu().numpy().view(np.uint64)
    assert int(j[:500].sum()) == M
    rest = j[500:].reshape(49, 500, 500)
    assert np.all(rest.sum(axis=(1, 2)) == M)
    v = visits.cpu().numpy().view(np.uint64)
    assert v[0] == M and np.all(v[1:].reshape(50, 500).sum(1) == M)


# --- projection -----------------------------------------------------------------------
def test_nearest_matches_reference_including_edges(gpu, oracle):
    q = Q()
    rng = np.random.default_rng(11)
    for d, N in ((1, 1), (1, 2), (1, 500), (1, 4000), (2, 1000), (3, 400)):
        pts = rng.standard_normal(N * d)
        qs = [rng.standard_normal(20000 * d) * 1.5]
        if d == 1:
            s = np.sort(pts)
            mids = (s[:-1] + s[1:]) / 2 if N > 1 else np.array([])
            qs += [pts, mids, np.nextafter(mids, np.inf), np.nextafter(mids, -np.inf),
                   np.array([-1e300, 1e300, 1e200, -1e-300, 0.0, -0.0, np.inf, -np.inf, np.nan])]
        else:
            qs += [pts]
        qq = np.concatenate([x.reshape(-1) for x in qs])
        got = q.nearest(q.QuantGrid(d, pts), qq)
        ref = oracle.nearest(d, pts, qq)
        assert np.array_equal(got, ref), (d, N)
    # symmetric tie -> smallest index (test_quant.cpp:42-45)
    assert q.nearest(q.QuantGrid(2, [0.0, 0.0, 1.0, 0.0]), [0.5, 0.0]).tolist() == [0]
    assert q.nearest(q.QuantGrid(1, [1.0, -1.0]), [0.0]).tolist() == [0]
    assert q.nearest(q.QuantGrid(1, [-1.0, 1.0]), [0.0]).tolist() == [0]


# --- pricer ---------------------------------------------------------------------------
def test_bdp_matches_golden_exactly(gpu, golden):
    q = Q()
    pr = golden["pricing"]
    for case in range(4):
        g = {k.split("_", 1)[1]: v for k, v in pr.items() if k.startswith(f"case{case}_")}
        sizes = g["sizes"]
        t = q.QuantTree([q.QuantGrid(1, np.arange(int(s), dtype=np.float64)) for s in sizes],
                        sizes, g["visits"], g["joint"], g["pi"], 1)
        res = q.solve_stopping(t, g["phi"])
        assert res.price == float(g["stop_price"])
        assert np.array_equal(np.concatenate(res.value), g["stop_value"])
        assert np.array_equal(np.concatenate(res.exercise), g["stop_exercise"])
        qmin, qmax = (int(x) for x in g["swing_q"])
        sw = q.solve_swing(t, g["phi"], qmin, qmax)
        assert sw.price == float(g["swing_price"])
        assert np.array_equal(np.concatenate(sw.value), g["swing_values"])
    with pytest.raises(q.ConfigError):
        q.solve_swing(t, g["phi"], 3, 2)


def test_swing_on_estimated_tree(gpu, oracle):
    q = Q()
    ch = q.BrownianChain1d(10)
    grids = q.build_brownian_grids(ch, 100)
    t = q.estimate_alg1(ch, grids, 200000)
    spec = ChainSpec(CHAIN_BROWNIAN1D, 10, sigma1=0.2, r=0.05)
    pts_all = np.concatenate([[0.0]] + [g.data() for g in grids])
    phi = oracle.payoff_table(spec, PAYOFF_SWING, t.sizes, pts_all)
    sp = q.solve_swing(t, phi, 2, 6)
    rp = oracle.solve_swing(t.sizes, t.flat_visits, t.flat_pi, phi, 2, 6)
    assert sp.price == rp


def test_cond_expectation_non_finite_f(gpu):
    """cond_expectation (bdp.hpp:36-54) with inf / NaN in f: the reference's
    dense loop multiplies every pi entry, so 0 * inf = NaN reaches rows whose
    non-zero entries avoid the non-finite columns; the device must agree bit
    for bit (a sequential Python-float loop is the reference's arithmetic)."""
    q = Q()
    rng = np.random.default_rng(7)
    rows, cols = 9, 7
    pi = rng.random((rows, cols)) * (rng.random((rows, cols)) < 0.5)
    pi[2] = 0.0
    pi[3, 4] = 0.3
    vis = np.array([5, 3, 0, 7, 1, 2, 9, 4, 6], np.uint64)
    flat_vis = np.concatenate([[1], vis, np.zeros(cols)]).astype(np.uint64)
    flat_pi = np.concatenate([np.full(rows, 1.0 / rows), pi.reshape(-1)])
    tree = q.QuantTree([q.QuantGrid(1, [0.0]), q.QuantGrid(1, np.arange(rows, dtype=float)),
                        q.QuantGrid(1, np.arange(cols, dtype=float))],
                       np.array([1, rows, cols], np.uint64), flat_vis,
                       np.zeros(rows + rows * cols, np.uint64), flat_pi, 1)
    for f in ([1.0, np.inf, 2.0, 3.0, 4.0, 5.0, 6.0], [1.0, 2.0, np.nan, 3.0, -np.inf, 5.0, 6.0],
              [np.inf, -np.inf, 1.0, 1.0, 1.0, 1.0, 1.0], list(rng.standard_normal(cols))):
        f = np.array(f)
        got = q.cond_expectation(tree, 1, f)
        want = []
        for i in range(rows):
            if vis[i] == 0:
                want.append(float("nan"))
                continue
            acc = 0.0
            for j in range(cols):
                acc += float(pi[i, j]) * float(f[j])
            want.append(acc)
        want = np.array(want)
        assert np.array_equal(np.isnan(got), np.isnan(want)), (f, got, want)
        ok = ~np.isnan(want)
        assert np.array_equal(got[ok].view(np.uint64), want[ok].view(np.uint64)), (f, got, want)
