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
