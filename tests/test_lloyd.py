"""Grid construction on the GPU (lloyd.hpp:59-107).

Parity mode: fed the reference stream's own normals, the GPU Lloyd must
return the reference's base grid bit for bit (same distinct-center
initialisation, exact projection, per-cell sums in sample order). On its own
in-kernel stream (the device Box-Muller restates glibc's log / sincos) it must
too: that is the product's grid path at every BASELINE size."""
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


@pytest.mark.parametrize("key", ["n100_d1", "n200_d1", "n500_d1", "n1000_d2", "n4000_d3"])
def test_lloyd_stream_bit_identical_to_reference(gpu, key):
    """The product's grid path: the GPU Lloyd on its own in-kernel stream
    returns the reference's base quantizer (its own lloyd_build, committed in
    tests/golden/base_grids.npz by make_golden.py) bit for bit, at every
    BASELINE grid size: C1 N=100, C3 N=200, C2 N=500 (d=1), C4 N=1000 (d=2),
    C5 N=4000 (d=3; 40 iterations x 800000 samples)."""
    import os
    q = Q()
    here = os.path.dirname(os.path.abspath(__file__))
    with np.load(os.path.join(here, "golden", "base_grids.npz")) as z:
        ref = np.array(z[key])
    N, dim = (int(v) for v in key[1:].split("_d"))
    got = np.asarray(q.base_grid(N, dim))
    assert got.shape == ref.shape
    bad = np.flatnonzero(got.view(np.uint64) != ref.view(np.uint64))
    assert bad.size == 0, (key, bad.size, float(np.max(np.abs(got - ref))))


def test_lloyd_any_grid_size(gpu):
    """Grid sizes that are not shipped are built on the GPU: a 2-D grid of 300
    points drives a full estimate (was: ValueError, no base quantizer)."""
    q = Q()
    tf = q.TwoFactorChain(q.TwoFactorParams(steps=5))
    grids = q.build_two_factor_grids(tf, 300)
    assert len(grids) == 5 and grids[0].size() == 300
    t = q.estimate_alg2(tf, grids, 10000)
    assert int(t.flat_visits[:1][0]) == 10000
