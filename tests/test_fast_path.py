"""The fast 1-D path (FP32 Box-Muller + certified cells + exact FP64 replay).

Its contract is that the counts are IDENTICAL to the exact kernel's (k_paths)
for every input: a transition is counted only when the bounded state interval
lies inside one cell, and every path with an uncertified transition is
recomputed exactly from that layer on. These tests check (1) the FP32 error
bounds exhaustively over all 2^32 MRG32k3a outputs, (2) fast == exact on the
configs and on adversarial grids, including the replay-list overflow path, and
(3) fast == the CPU oracle on fresh windows (the other parity tests in
test_gpu_parity.py also run through the fast path, which is the default)."""
from __future__ import annotations

import os

import numpy as np
import pytest

from pyoracle import CHAIN_BROWNIAN1D, CHAIN_OU1D, ChainSpec

pytestmark = pytest.mark.gpu

# qt_device.cuh: kRadA, kRadB, kAng
K_RAD_A, K_ANG = 2.2e-7, 5.5e-7


def Q():
    from paper_1101_3228_b200 import qtree
    return qtree


@pytest.fixture(autouse=True)
def fast_on():
    """These tests select the FP32 certified kernel (set_fast_path(True)); each
    ends by restoring the default (the certified FP64 kernel, mode 2)."""
    Q().set_fast_path(True)
    yield
    Q().set_fast_path(2)


def _counts(plan, M, first=0, total=None, fast=True):
    import torch
    q = Q()
    q.set_fast_path(fast)
    try:
        joint = plan.zeros_joint()
        plan.count(1, 1, 12345, first, M, total or M, joint)
        torch.cuda.synchronize()
        return joint.cpu().numpy().view(np.uint64).copy()
    finally:
        q.set_fast_path(True)


def test_fp32_box_muller_bounds_exhaustive(gpu):
    out = Q().fast_bounds_check()
    assert out[0] <= K_RAD_A, out
    assert out[1] <= K_ANG and out[2] <= K_ANG, out
    assert out[3] <= 1.0, out


def test_fast_equals_exact_c2(gpu):
    from paper_1101_3228_b200.device import Plan
    q = Q()
    ch = q.BrownianChain1d(50)
    plan = Plan(ch, q.build_brownian_grids(ch, 500), 0)
    for first in (0, 987654321):
        fast = _counts(plan, 2 * 10**6, first, 10**9, True)
        exact = _counts(plan, 2 * 10**6, first, 10**9, False)
        assert np.array_equal(fast, exact), first
    st = plan.fast_stats()
    assert st["fast_paths"] == 4 * 10**6
    # the replay path is exercised (a few % of paths are not certified)
    assert 0 < st["replayed"] < 4 * 10**5, st
    assert st["inline_replayed"] == 0, st


def test_fast_equals_exact_ou(gpu):
    from paper_1101_3228_b200.device import Plan
    q = Q()
    p = q.TwoFactorParams(sigma1=0.5, alpha1=1.0, sigma2=0.0, steps=365)
    ch = q.OuChain1d(p)
    plan = Plan(ch, q.build_ou_grids(ch, 200), 0)
    assert np.array_equal(_counts(plan, 200000, 0, 10**6, True),
                          _counts(plan, 200000, 0, 10**6, False))


def test_fast_replay_list_overflow(gpu, monkeypatch):
    """A replay list of 3 entries: every further ambiguous path is replayed
    inline by the path kernel; the counts do not change."""
    from paper_1101_3228_b200.device import Plan
    q = Q()
    ch = q.BrownianChain1d(50)
    grids = q.build_brownian_grids(ch, 500)
    exact = _counts(Plan(ch, grids, 0), 300000, 5, 10**9, False)
    monkeypatch.setenv("QT_FAST_REPLAY_CAP", "3")
    plan = Plan(ch, grids, 0)
    fast = _counts(plan, 300000, 5, 10**9, True)
    st = plan.fast_stats()
    assert np.array_equal(fast, exact)
    assert st["replayed"] == 3 and st["inline_replayed"] > 0, st


@pytest.mark.parametrize("case", ["dense", "single", "tiny_gap", "huge_spread"])
def test_fast_equals_exact_adversarial_grids(gpu, case):
    """Grids that make certification hard or impossible (very dense cells,
    one-point layers, near-duplicate points -> x_safe tiny or 0, points far
    apart) must still give the exact kernel's counts."""
    from paper_1101_3228_b200.device import Plan
    q = Q()
    n = 12
    ch = q.BrownianChain1d(n)
    rng = np.random.default_rng(7)
    grids = []
    for k in range(1, n + 1):
        if case == "dense":
            pts = np.sort(rng.standard_normal(2000)) * np.sqrt(k / n)
        elif case == "single":
            pts = np.array([0.1 * k]) if k % 2 else np.array([-1.0, 1.0])
        elif case == "tiny_gap":
            base = rng.standard_normal(64)
            pts = np.concatenate([base, base + 1e-13])
        else:
            pts = rng.standard_normal(100) * 1e6
        grids.append(q.QuantGrid(1, pts))
    plan = Plan(ch, grids, 0)
    assert np.array_equal(_counts(plan, 100000, 0, 10**7, True),
                          _counts(plan, 100000, 0, 10**7, False)), case


def test_fast_window_vs_oracle(gpu, oracle):
    q = Q()
    ch = q.BrownianChain1d(50)
    grids = q.build_brownian_grids(ch, 500)
    spec = ChainSpec(CHAIN_BROWNIAN1D, 50)
    sizes = np.array([1] + [500] * 50, np.uint64)
    pts = np.concatenate([g.data() for g in grids])
    first = 314159265
    v, j = q.accumulate_paths(ch, grids, 1, 12345, first, 40000, 10**9)
    rv, rj = oracle.accumulate_paths(spec, sizes, pts, 1, 12345, first, 40000, 10**9)
    assert np.array_equal(v, rv) and np.array_equal(j, rj)
    st = q.fast_stats()
    assert st["fast_paths"] >= 40000


@pytest.mark.parametrize("case", ["dense", "single", "tiny_gap", "huge_spread"])
def test_xtables_equal_thr_kernels_adversarial_grids(gpu, case, monkeypatch):
    """k_paths_x / k_alg3_x (threshold-pair x-tables, sorted-cell counts +
    permute-add) against k_paths / k_alg3 (Thr records, original-index counts)
    on the adversarial grids above: identical Alg II and Alg III trees."""
    q = Q()
    n = 12
    ch = q.BrownianChain1d(n)
    rng = np.random.default_rng(11)
    grids = []
    for k in range(1, n + 1):
        if case == "dense":
            pts = rng.standard_normal(2000) * np.sqrt(k / n)
        elif case == "single":
            pts = np.array([0.1 * k]) if k % 2 else np.array([1.0, -1.0])
        elif case == "tiny_gap":
            base = rng.standard_normal(64)
            pts = np.concatenate([base + 1e-13, base])
        else:
            pts = rng.standard_normal(100) * 1e6
        grids.append(q.QuantGrid(1, pts))
    for alg, M in ((1, 60000), (2, 8000)):
        monkeypatch.setenv("QT_XKERNEL", "1")
        x = q.estimate(alg, ch, grids, M)
        monkeypatch.setenv("QT_XKERNEL", "0")
        ref = q.estimate(alg, ch, grids, M)
        assert np.array_equal(x.flat_joint, ref.flat_joint), (case, alg)
        assert np.array_equal(x.flat_visits, ref.flat_visits), (case, alg)


# --- the certified FP64 kernel (the default, k_paths_x<CERT>) ----------------------

def test_apx_box_muller_bounds_exhaustive(gpu):
    """qt_math_fast.h vs the glibc-exact pair over every MRG32k3a output: the
    measured maxima must sit inside the bounds the certified kernel assumes."""
    out = Q().apx_bounds_check()
    rad, ang_c, ang_s, mag, k_rad, k_ang, k_z = (float(v) for v in out)
    assert rad <= k_rad, (rad, k_rad)
    assert ang_c <= k_ang and ang_s <= k_ang, (ang_c, ang_s, k_ang)
    assert mag <= 1.0, mag
    assert k_z >= (k_rad + k_ang + 2.0**-52) * (1 + 2.0**-40)


@pytest.mark.parametrize("kind", ["bm", "ou"])
def test_certified_fp64_equals_exact(gpu, kind):
    """Mode 2 (the default) equals the exact kernel on C2- and C3-shaped chains,
    at path windows deep in a 1e9-path stream."""
    from paper_1101_3228_b200.device import Plan
    q = Q()
    if kind == "bm":
        ch = q.BrownianChain1d(50)
        grids = q.build_brownian_grids(ch, 500)
    else:
        p = q.TwoFactorParams(sigma1=0.5, alpha1=1.0, sigma2=0.0, steps=60)
        ch = q.OuChain1d(p)
        grids = q.build_ou_grids(ch, 200)
    plan = Plan(ch, grids, 0)
    for first in (0, 555555555):
        cert = _counts(plan, 10**6, first, 10**9, 2)
        exact = _counts(plan, 10**6, first, 10**9, False)
        assert np.array_equal(cert, exact), (kind, first)


def test_certified_fp64_replays_adversarial(gpu):
    """A grid with cells narrower than the state bound (1e-14 wide pairs) makes
    most paths uncertified: the replay must still give the exact counts,
    including the inline replay when the list overflows."""
    from paper_1101_3228_b200.device import Plan
    q = Q()
    ch = q.BrownianChain1d(8)
    rng = np.random.default_rng(4)
    grids = []
    for k in range(1, 9):
        base = np.sort(rng.standard_normal(40)) * np.sqrt(k / 8)
        pts = np.concatenate([base, base + 3e-14 * (1 + np.abs(base))])
        grids.append(q.QuantGrid(1, pts))
    plan = Plan(ch, grids, 0)
    cert = _counts(plan, 200000, 0, None, 2)
    exact = _counts(plan, 200000, 0, None, False)
    assert np.array_equal(cert, exact)


def _counts3(plan, M, n, mode):
    import torch
    q = Q()
    q.set_fast_path(mode)
    try:
        joint = plan.zeros_joint()
        plan.count(2, 1, 4242, 0, M * n, M * n, joint)
        torch.cuda.synchronize()
        return joint.cpu().numpy().view(np.uint64).copy()
    finally:
        q.set_fast_path(True)


@pytest.mark.parametrize("case", ["c3", "adversarial"])
def test_certified_alg3_equals_exact(gpu, case):
    """Alg III (k_alg3_x) certified with the approximate FP64 pair equals the
    exact kernel: on the C3 OU chain (no sample needs the replay) and on grids
    of 3e-14-wide cell pairs (most samples replayed by k_replay3)."""
    from paper_1101_3228_b200.device import Plan
    q = Q()
    n = 40 if case == "c3" else 6
    p = q.TwoFactorParams(sigma1=0.5, alpha1=1.0, sigma2=0.0, steps=n)
    ch = q.OuChain1d(p)
    if case == "c3":
        grids = q.build_ou_grids(ch, 200)
    else:
        rng = np.random.default_rng(9)
        grids = []
        for k in range(1, n + 1):
            base = np.sort(rng.standard_normal(30)) * 0.4
            grids.append(q.QuantGrid(1, np.concatenate([base, base + 3e-14 * (1 + np.abs(base))])))
    plan = Plan(ch, grids, 0)
    M = 200000 if case == "c3" else 30000
    cert = _counts3(plan, M, n, 2)
    exact = _counts3(plan, M, n, False)
    assert np.array_equal(cert, exact), case


@pytest.mark.parametrize("mode", [2, 0])
def test_alg3_count_tile_equals_l2_reds(gpu, monkeypatch, mode):
    """The default Alg III kernel counts into a per-CTA shared-memory tile and
    flushes it once; QT_A3_PRIV=0 issues one L2 RED per sample. Same counts,
    certified (mode 2) and exact (mode 0), with several slices per layer."""
    from paper_1101_3228_b200.device import Plan
    q = Q()
    n = 12
    ch = q.OuChain1d(q.TwoFactorParams(sigma1=0.5, alpha1=1.0, sigma2=0.0, steps=n))
    plan = Plan(ch, q.build_ou_grids(ch, 200), 0)
    M = 300000
    monkeypatch.setenv("QT_A3_SLICES", "3")
    tile = _counts3(plan, M, n, mode)
    monkeypatch.setenv("QT_A3_PRIV", "0")
    reds = _counts3(plan, M, n, mode)
    assert tile.sum() == M * n
    assert np.array_equal(tile, reds)


@pytest.mark.parametrize("mode", [2, 0])
def test_first_transition_histogram_equals_reds(gpu, monkeypatch, mode):
    """k_paths_x counts the first transition (x0 -> layer 1, a single row every
    path hits) in a per-CTA shared-memory histogram; QT_X_HIST1=0 issues one RED
    per path instead. Same counts, certified (mode 2) and exact (mode 0)."""
    import torch
    from paper_1101_3228_b200.device import Plan
    q = Q()
    ch = q.BrownianChain1d(10)
    plan = Plan(ch, q.build_brownian_grids(ch, 100), 0)
    q.set_fast_path(mode)
    try:
        out = []
        for h in ("1", "0"):
            monkeypatch.setenv("QT_X_HIST1", h)
            joint = plan.zeros_joint()
            plan.count(1, 1, 12345, 777, 300001, 10**6, joint)
            torch.cuda.synchronize()
            out.append(joint.cpu().numpy().view(np.uint64).copy())
    finally:
        q.set_fast_path(True)
    assert out[0][:100].sum() == 300001
    assert np.array_equal(out[0], out[1])


def test_alg3_count_tile_ragged_layers(gpu, monkeypatch):
    """The Alg III count tile with layer sizes that differ from layer to layer
    (the tile is sized for the largest N_{k-1} x N_k, each layer uses its own
    N_{k-1} x N_k block) equals the one-RED-per-sample kernel."""
    from paper_1101_3228_b200.device import Plan
    q = Q()
    n = 9
    ch = q.OuChain1d(q.TwoFactorParams(sigma1=0.5, alpha1=1.0, sigma2=0.0, steps=n))
    rng = np.random.default_rng(21)
    sizes = [37, 250, 3, 120, 199, 64, 1, 90, 180]
    grids = [q.QuantGrid(1, np.sort(rng.standard_normal(s)) * 0.5 + 0.01 * k)
             for k, s in enumerate(sizes)]
    plan = Plan(ch, grids, 0)
    M = 120001
    monkeypatch.setenv("QT_A3_SLICES", "2")
    tile = _counts3(plan, M, n, 2)
    monkeypatch.setenv("QT_A3_PRIV", "0")
    reds = _counts3(plan, M, n, 2)
    assert tile.sum() == M * n
    assert np.array_equal(tile, reds)


@pytest.mark.parametrize("mode", [2, 0])
def test_paths_per_thread_variants_agree(gpu, monkeypatch, mode):
    """k_paths_x runs one path per thread for small path counts and two for
    large ones (a heuristic on the count); both variants, forced through
    QT_X_P, give the same counts on the same window."""
    from paper_1101_3228_b200.device import Plan
    q = Q()
    ch = q.BrownianChain1d(50)
    plan = Plan(ch, q.build_brownian_grids(ch, 500), 0)
    q.set_fast_path(mode)
    try:
        out = []
        for pp in ("1", "2"):
            monkeypatch.setenv("QT_X_P", pp)
            out.append(_counts(plan, 400003, 123456789, 10**9, fast=mode))
    finally:
        q.set_fast_path(True)
    assert out[0][:500].sum() == 400003
    assert np.array_equal(out[0], out[1])
