"""Grid construction on the GPU (lloyd.hpp:59-107).

Parity mode: fed the reference stream's own normals, the GPU Lloyd must
return the reference's base grid bit for bit (same distinct-center
initialisation, exact projection, per-cell sums in sample order). With the
in-kernel stream (device Box-Muller, <= 1 ulp from glibc per normal) the grid
and its distortion must agree with the reference's to a tight tolerance."""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def Q():
    from paper_1101_3228_b200 import qtree
    return qtree


@pytest.mark.parametrize("dim,N,iters,spi", [(1, 100, 40, 20000), (2, 200, 8, 40000),
                                             (3, 150, 5, 30000), (1, 1, 3, 1000)])
def test_lloyd_normals_in_bit_exact(gpu, reference, dim, N, iters, spi):
    q = Q()
    seed = 12345
    stream_seed = seed ^ 0x9E3779B9
    # enough normals for the initialisation and every batch
    K = (N + 64) * dim + iters * spi * dim + 2
    normals = reference.path_normals(1, stream_seed, K, 0, 1, 1)
    got = q.lloyd_build(dim, N, iters, spi, seed, normals=normals)
    ref = reference.lloyd_base(dim, N, seed, spi, iters)
    assert np.array_equal(np.asarray(got.grid.data()).view(np.uint64), ref.view(np.uint64))


def test_lloyd_stream_matches_shipped_base_grid(gpu):
    """The shipped base quantizer (the reference's lloyd_build, N = 100, d = 1)
    vs the GPU build on the in-kernel stream."""
    q = Q()
    with np.load(q._DATA) as z:
        ref = np.array(z["n100_d1"])
    got = np.asarray(q.lloyd_build(1, 100).grid.data())
    assert np.max(np.abs(got - ref)) < 1e-9, np.max(np.abs(got - ref))


def test_lloyd_any_grid_size(gpu):
    """Grid sizes that are not shipped are built on the GPU: a 2-D grid of 300
    points drives a full estimate (was: ValueError, no base quantizer)."""
    q = Q()
    tf = q.TwoFactorChain(q.TwoFactorParams(steps=5))
    grids = q.build_two_factor_grids(tf, 300)
    assert len(grids) == 5 and grids[0].size() == 300
    t = q.estimate_alg2(tf, grids, 10000)
    assert int(t.flat_visits[:1][0]) == 10000
