"""K2 for d >= 2: both fast projections must give exactly the reference's cells
-- the default exact cell-list search (k_paths_cell / k_alg3_cell, qt_cell.cu)
and the FP32 brute-force scan with an exact FP64 decision (k_paths_scan /
k_alg3_scan, qt_scan.cu; QT_NN=scan).

Both are checked against the exact FP64 brute-force kernel (QT_NN=scan +
QT_SCAN=0) on the config-4 and config-5 chains and grids, on adversarial grids
(exact ties, near-ties closer than the FP32 error bound, coordinates too large
for FP32, far-away queries, degenerate and tiny grids), and against the CPU
oracle on windows of the config chains."""
from __future__ import annotations

import numpy as np
import pytest

from pyoracle import CHAIN_GBM3D, CHAIN_TWO_FACTOR, ChainSpec

pytestmark = pytest.mark.gpu


def Q():
    from paper_1101_3228_b200 import qtree
    return qtree


MODES = ("cell", "scan", "exact")


def _mode(monkeypatch, mode):
    if mode == "cell":
        monkeypatch.delenv("QT_NN", raising=False)
        monkeypatch.setenv("QT_SCAN", "1")
    else:
        monkeypatch.setenv("QT_NN", "scan")
        monkeypatch.setenv("QT_SCAN", "1" if mode == "scan" else "0")


def _counts(monkeypatch, chain, grids, M, first=0, total=None, mode="cell", engine=1):
    import torch
    from paper_1101_3228_b200.device import Plan
    _mode(monkeypatch, mode)
    plan = Plan(chain, grids, 0)
    joint = plan.zeros_joint()
    plan.count(1, engine, 12345, first, M, total or M, joint)
    torch.cuda.synchronize()
    plan.close()
    return joint.cpu().numpy().view(np.uint64).copy()


def test_scan_equals_exact_c4(gpu, monkeypatch):
    q = Q()
    tf = q.TwoFactorChain(q.TwoFactorParams())
    g4 = q.build_two_factor_grids(tf, 1000)
    for first in (0, 31415926):
        a, b, c = (_counts(monkeypatch, tf, g4, 20000, first, 10**8, m) for m in MODES)
        assert np.array_equal(a, c) and np.array_equal(b, c), first
        assert int(a[:1000].sum()) == 20000


def test_scan_equals_exact_c5(gpu, monkeypatch):
    q = Q()
    ch = q.GbmChain3d(20, 1.0, (0.0, 0.0, 0.0))
    g5 = q.build_gbm_grids(ch, 4000)
    a, b, c = (_counts(monkeypatch, ch, g5, 20000, 777, 4 * 10**9, m) for m in MODES)
    assert np.array_equal(a, c) and np.array_equal(b, c)


@pytest.mark.parametrize("engine", [0, 2])
def test_scan_other_engines(gpu, monkeypatch, engine):
    q = Q()
    tf = q.TwoFactorChain(q.TwoFactorParams(steps=30))
    g = q.build_two_factor_grids(tf, 1000)
    a, b, c = (_counts(monkeypatch, tf, g, 30000, 0, None, m, engine) for m in MODES)
    assert np.array_equal(a, c) and np.array_equal(b, c)


@pytest.mark.parametrize("case", ["ties", "near_ties", "huge", "far", "tiny_grid", "two_points",
                                  "collinear", "near_duplicates", "cluster_and_outlier"])
def test_scan_adversarial_grids(gpu, monkeypatch, case):
    q = Q()
    n = 8
    tf = q.TwoFactorChain(q.TwoFactorParams(steps=n))
    rng = np.random.default_rng(3)
    grids = []
    for k in range(1, n + 1):
        if case == "ties":  # lattice: many exactly equidistant pairs -> smallest index
            xs = np.linspace(-1, 1, 9)
            pts = np.array([(a, b) for a in xs for b in xs]).reshape(-1)
        elif case == "near_ties":  # pairs mirrored to ~1e-9: below the FP32 bound
            base = rng.standard_normal((150, 2)) * 0.5
            pts = np.concatenate([base, -base + 1e-9]).reshape(-1)
        elif case == "huge":  # FP32 cannot hold these: every query takes the FP64 scan
            pts = rng.standard_normal(400) * 1e13
        elif case == "far":  # queries far outside a small cluster
            pts = rng.standard_normal(400) * 1e-3 + 5.0
        elif case == "tiny_grid":  # fewer points than one chunk
            pts = rng.standard_normal(6)
        elif case == "two_points":
            pts = np.array([0.1, -0.2, -0.3, 0.4])
        elif case == "collinear":  # zero span on one axis: one bucket across it
            pts = np.stack([np.linspace(-1, 1, 50), np.full(50, 0.25)], axis=1).reshape(-1)
        elif case == "near_duplicates":  # copies 1 ulp apart (exact copies are invalid grids)
            base = rng.standard_normal((60, 2)) * 0.4
            pts = np.concatenate([base, np.nextafter(base, np.inf)[::-1]]).reshape(-1)
        else:  # a dense cluster and one far point: most buckets empty
            pts = np.concatenate([rng.standard_normal((200, 2)) * 1e-2, [[3.0, -2.0]]]).reshape(-1)
        grids.append(q.QuantGrid(2, pts))
    a, b, c = (_counts(monkeypatch, tf, grids, 50000, 0, None, m) for m in MODES)
    assert np.array_equal(a, c), ("cell", case)
    assert np.array_equal(b, c), ("scan", case)


def test_scan_c4_window_vs_oracle(gpu, oracle):
    q = Q()
    tf = q.TwoFactorChain(q.TwoFactorParams())
    g4 = q.build_two_factor_grids(tf, 1000)
    spec4 = ChainSpec(CHAIN_TWO_FACTOR, 365)
    s4 = np.array([1] + [1000] * 365, np.uint64)
    p4 = np.concatenate([g.data() for g in g4])
    v, j = q.accumulate_paths(tf, g4, 1, 12345, 98765, 1000, 10**8)
    rv, rj = oracle.accumulate_paths(spec4, s4, p4, 1, 12345, 98765, 1000, 10**8)
    assert np.array_equal(v, rv) and np.array_equal(j, rj)


def test_scan_c5_window_vs_oracle(gpu, oracle):
    q = Q()
    ch = q.GbmChain3d(20, 1.0, (0.0, 0.0, 0.0))
    g5 = q.build_gbm_grids(ch, 4000)
    spec5 = ChainSpec(CHAIN_GBM3D, 20, gbm_rho=(0.0, 0.0, 0.0))
    s5 = np.array([1] + [4000] * 20, np.uint64)
    p5 = np.concatenate([g.data() for g in g5])
    v, j = q.accumulate_paths(ch, g5, 1, 12345, 2 * 10**9, 800, 4 * 10**9)
    rv, rj = oracle.accumulate_paths(spec5, s5, p5, 1, 12345, 2 * 10**9, 800, 4 * 10**9)
    assert np.array_equal(v, rv) and np.array_equal(j, rj)


@pytest.mark.parametrize("kind,engine", [("tf", 1), ("tf", 2), ("gbm", 1), ("gbm", 0)])
def test_alg3_scan_equals_exact(gpu, monkeypatch, kind, engine):
    """Alg III (layer-parallel pairs) through k_alg3_cell and k_alg3_scan vs
    the FP64 k_alg3."""
    import torch
    from paper_1101_3228_b200.device import Plan
    q = Q()
    if kind == "tf":
        ch = q.TwoFactorChain(q.TwoFactorParams(steps=20))
        grids = q.build_two_factor_grids(ch, 1000)
    else:
        ch = q.GbmChain3d(6, 1.0, (0.2, 0.1, -0.3))
        grids = q.build_gbm_grids(ch, 4000)
    M = 20000
    units = M * ch.layers()
    out = []
    for mode in MODES:
        _mode(monkeypatch, mode)
        plan = Plan(ch, grids, 0)
        joint = plan.zeros_joint()
        plan.count(2, engine, 4242, 0, units, units, joint)
        torch.cuda.synchronize()
        out.append(joint.cpu().numpy().copy())
        plan.close()
    assert np.array_equal(out[0], out[2]) and np.array_equal(out[1], out[2])
