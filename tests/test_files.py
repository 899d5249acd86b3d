"""Tree and grid files: QTRE v1 (quant_tree.hpp:138-207) and
the grid text format (grid.hpp:84-117). Our writers must produce the same bytes
as the reference's own save_tree / save_grid (compiled from the reference
headers in oracle/_ref), files written by either side must load in the other,
and the loaders must raise the reference's IoError messages."""
from __future__ import annotations

import numpy as np
import pytest


def Q():
    from paper_1101_3228_b200 import qtree
    return qtree


def _tree(dim=1, sizes=(1, 7, 5, 9), seed=0):
    q = Q()
    rng = np.random.default_rng(seed)
    sizes = np.array(sizes, np.uint64)
    grids = [q.QuantGrid(dim, np.zeros(dim))]
    for s in sizes[1:]:
        grids.append(q.QuantGrid(dim, rng.standard_normal(int(s) * dim) * 1.7 + 1e-9))
    nvis = int(sizes.sum())
    njoint = int(sum(sizes[k - 1] * sizes[k] for k in range(1, len(sizes))))
    visits = rng.integers(0, 2**40, nvis).astype(np.uint64)
    joint = rng.integers(0, 2**62, njoint).astype(np.uint64)
    pi = rng.random(njoint) * (rng.random(njoint) < 0.7)
    return q.QuantTree(grids, sizes, visits, joint, pi, 123456789012)


def _flat(tree):
    return np.concatenate([np.asarray(g.data(), np.float64) for g in tree.grids])


@pytest.mark.parametrize("dim", [1, 2, 3])
def test_save_tree_bytes_equal_reference(tmp_path, reference, dim):
    t = _tree(dim, seed=dim)
    ours, ref = tmp_path / "ours.qtre", tmp_path / "ref.qtre"
    Q().save_tree(t, ours)
    reference.save_tree(ref, dim, t.sizes, _flat(t), t.samples, t.flat_visits, t.flat_joint,
                        t.flat_pi)
    assert ours.read_bytes() == ref.read_bytes()


def test_load_reference_tree_and_round_trip(tmp_path, reference):
    q = Q()
    t = _tree(2, sizes=(1, 4, 6), seed=5)
    ref = tmp_path / "ref.qtre"
    reference.save_tree(ref, 2, t.sizes, _flat(t), t.samples, t.flat_visits, t.flat_joint,
                        t.flat_pi)
    u = q.load_tree(ref)
    assert u.samples == t.samples and np.array_equal(u.sizes, t.sizes)
    assert np.array_equal(u.flat_visits, t.flat_visits)
    assert np.array_equal(u.flat_joint, t.flat_joint)
    assert np.array_equal(u.flat_pi.view(np.uint64), t.flat_pi.view(np.uint64))
    assert np.array_equal(_flat(u).view(np.uint64), _flat(t).view(np.uint64))
    # ours -> reference loader
    ours = tmp_path / "ours.qtre"
    q.save_tree(u, ours)
    n, d, m, sizes, pts, v, j, pi = reference.load_tree(ours, 8, 64, 256)
    assert (n, d, m) == (2, 2, t.samples)
    assert np.array_equal(j, t.flat_joint) and np.array_equal(pi, t.flat_pi)


def test_tree_load_errors(tmp_path):
    q = Q()
    t = _tree()
    good = tmp_path / "t.qtre"
    q.save_tree(t, good)
    raw = good.read_bytes()
    cases = {
        "missing": (None, "load_tree: cannot open"),
        "magic": (b"QTRX" + raw[4:], "load_tree: bad magic in"),
        "version": (raw[:4] + (2).to_bytes(4, "little") + raw[8:], "load_tree: unsupported version 2"),
        "empty": (raw[:8] + (0).to_bytes(4, "little") + raw[12:], "load_tree: empty tree"),
        "truncated": (raw[:-5], "tree file: truncated"),
    }
    for name, (data, msg) in cases.items():
        p = tmp_path / f"{name}.qtre"
        if data is not None:
            p.write_bytes(data)
        with pytest.raises(q.IoError, match=msg):
            q.load_tree(p)


def test_grid_files_match_reference(tmp_path, reference):
    q = Q()
    rng = np.random.default_rng(1)
    for dim in (1, 2, 3):
        pts = rng.standard_normal(11 * dim) * 10.0 ** rng.integers(-30, 30, 11 * dim)
        g = q.QuantGrid(dim, pts)
        ours, ref = tmp_path / f"o{dim}.txt", tmp_path / f"r{dim}.txt"
        q.save_grid(g, ours)
        reference.save_grid(ref, dim, pts)
        assert ours.read_bytes() == ref.read_bytes()
        h = q.load_grid(ref)
        assert h.dim() == dim and np.array_equal(np.asarray(h.data()).view(np.uint64),
                                                 pts.view(np.uint64))
    bad = tmp_path / "bad.txt"
    for text, msg in (("x 1\n", "malformed header"), ("2 1\n1.0\n", "expected 2 rows of 1"),
                      ("1 1\n1.0\n2.0\n", "trailing data"), ("2 1\n1.0\n1.0\n", "duplicate")):
        bad.write_text(text)
        with pytest.raises(q.IoError, match=msg):
            q.load_grid(bad)


@pytest.mark.gpu
def test_device_tree_writer_equals_host_writer(gpu, tmp_path, reference):
    """Estimate C1 on the GPU, write the tree straight from HBM, compare with the
    reference's save_tree of the same (host) tree, byte for byte."""
    import torch
    q = Q()
    from paper_1101_3228_b200.device import Plan
    ch = q.BrownianChain1d(10)
    grids = q.build_brownian_grids(ch, 100)
    plan = Plan(ch, grids, 0)
    M = 10**6
    joint = plan.zeros_joint()
    plan.count(1, 1, 12345, 0, M, M, joint)
    visits = torch.zeros(plan.n_visits, dtype=torch.int64, device="cuda")
    pi = torch.zeros(plan.n_joint, dtype=torch.float64, device="cuda")
    plan.finalize(1, M, joint, visits, pi)
    dev = tmp_path / "dev.qtre"
    plan.save_tree(dev, M, joint, visits, pi)
    t = q.estimate_alg2(ch, grids, M)
    ref = tmp_path / "ref.qtre"
    reference.save_tree(ref, 1, t.sizes, _flat(t), M, t.flat_visits, t.flat_joint, t.flat_pi)
    assert dev.read_bytes() == ref.read_bytes()


def _qtre(samples, grids_text, visits, mats):
    """Raw QTRE v1 bytes (quant_tree.hpp:138-163) from explicit parts, to build
    files the reference's own writer cannot produce."""
    import struct
    b = b"QTRE" + struct.pack("<IIQ", 1, len(grids_text) - 1, samples)
    for t in grids_text:
        b += struct.pack("<Q", len(t)) + t.encode()
    b += np.asarray(visits, np.uint64).tobytes()
    for r, c, j, p in mats:
        b += struct.pack("<QQ", r, c) + np.asarray(j, np.uint64).tobytes() + \
            np.asarray(p, np.float64).tobytes()
    return b


def test_tree_load_rejects_mixed_dims_and_overflow(tmp_path):
    """A malformed file whose grids differ in dim (grid 0 of dim 8, grid 1 of
    dim 1) used to size the caller's buffers from the last grid and overflow
    them; it is an IoError now, and the loader never writes past what the
    caller says it allocated."""
    q = Q()
    g0 = "1 8\n" + " ".join(["0"] * 8) + "\n"
    g1 = "2 1\n0.5\n1.5\n"
    p = tmp_path / "mixed.qtre"
    p.write_bytes(_qtre(7, [g0, g1], [7, 3, 4], [(1, 2, [3, 4], [3 / 7, 4 / 7])]))
    with pytest.raises(q.IoError, match="differing dimension"):
        q.load_tree(p)
    # consistent file, but the caller's capacities are too small
    good = tmp_path / "good.qtre"
    good.write_bytes(_qtre(7, ["1 1\n0\n", g1], [7, 3, 4], [(1, 2, [3, 4], [3 / 7, 4 / 7])]))
    import ctypes as C
    from paper_1101_3228_b200 import _lib
    lib = _lib.lib()
    sizes = np.zeros(2, np.uint64)
    pts = np.full(3, -1.0)
    v = np.zeros(3, np.uint64)
    j = np.zeros(2, np.uint64)
    pi = np.zeros(2)

    def load(layers, vcap, jcap):
        return lib.qt_load_tree(str(good).encode(), layers, 1, sizes.ctypes.data_as(C.POINTER(C.c_uint64)),
                                pts.ctypes.data_as(C.POINTER(C.c_double)),
                                v.ctypes.data_as(C.POINTER(C.c_uint64)), vcap,
                                j.ctypes.data_as(C.POINTER(C.c_uint64)),
                                pi.ctypes.data_as(C.POINTER(C.c_double)), jcap)
    assert load(1, 3, 2) == 0 and list(v) == [7, 3, 4] and list(j) == [3, 4]
    assert load(2, 3, 2) == 3            # layer count disagrees with the caller's
    pts[:] = -1.0
    assert load(1, 2, 2) == 3 and pts[2] == -1.0   # visits capacity: nothing past it
    assert load(1, 3, 1) == 3
    q.load_tree(good)
