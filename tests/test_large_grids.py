"""Grids larger than the shared-memory staging limit (the reference has no
size limit): tables are read from global memory by k_paths_gmem / k_alg3_gmem
with the same exact arithmetic; counts must equal the CPU oracle's."""
from __future__ import annotations

import numpy as np
import pytest

from pyoracle import ALG_II, ALG_III, CHAIN_BROWNIAN1D, CHAIN_TWO_FACTOR, ChainSpec

pytestmark = pytest.mark.gpu


def Q():
    from paper_1101_3228_b200 import qtree
    return qtree


@pytest.mark.parametrize("alg", [ALG_II, ALG_III])
def test_large_1d_grid_equals_oracle(gpu, oracle, alg):
    q = Q()
    rng = np.random.default_rng(9)
    n = 4
    sizes = np.array([1] + [20000, 15000, 20000, 9000], np.uint64)
    pts = np.concatenate([np.sort(rng.standard_normal(int(s))) * np.sqrt((k + 1) / n)
                          for k, s in enumerate(sizes[1:])])
    spec = ChainSpec(CHAIN_BROWNIAN1D, n)
    ch = q.BrownianChain1d(n)
    grids, o = [], 0
    for s in sizes[1:]:
        grids.append(q.QuantGrid(1, pts[o:o + int(s)]))
        o += int(s)
    M = 3000
    t = q.estimate(alg, ch, grids, M)
    ref = oracle.estimate(alg, spec, sizes, pts, M, workers=4)
    assert np.array_equal(t.flat_joint, ref.joint)
    assert np.array_equal(t.flat_pi, ref.pi)


def test_large_2d_grid_equals_oracle(gpu, oracle):
    q = Q()
    rng = np.random.default_rng(10)
    n = 2
    sizes = np.array([1, 12000, 10000], np.uint64)
    pts = rng.standard_normal(int(sizes[1:].sum()) * 2) * 0.5
    spec = ChainSpec(CHAIN_TWO_FACTOR, n)
    ch = q.TwoFactorChain(q.TwoFactorParams(steps=n))
    grids = [q.QuantGrid(2, pts[:24000]), q.QuantGrid(2, pts[24000:])]
    M = 400
    t = q.estimate(ALG_II, ch, grids, M)
    ref = oracle.estimate(ALG_II, spec, sizes, pts, M, workers=4)
    assert np.array_equal(t.flat_joint, ref.joint)
