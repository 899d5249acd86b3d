"""Multi-process sharding on CPU (gloo, world size 2): the host logic of the
N>1 path. Each rank counts its shard of paths (the reference's worker formula,
estimate.hpp:180-181) with the CPU checker standing in for the device kernel,
the int64 partial counts are summed with one collective, and the result must
equal the single-process run bit for bit (test_tree.cpp:128-152 analogue)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    import sys
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from paper_1101_3228_b200.dist import shard
    from pyoracle import ChainSpec, Oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    orc = Oracle("restatement")
    spec = ChainSpec(1, 4, sigma1=0.4, sigma2=0.7, alpha1=0.8, alpha2=3.5, rho=0.3)
    rng = np.random.default_rng(5)
    sizes = np.array([1, 9, 11, 7, 13], np.uint64)
    pts = rng.standard_normal(int(sizes[1:].sum()) * 2)
    M = 5001
    first, count = shard(M, rank, world)
    v, j = orc.accumulate_paths(spec, sizes, pts, 1, 12345, first, count, M)
    joint = torch.from_numpy(j.view(np.int64).copy())
    dist.all_reduce(joint, op=dist.ReduceOp.SUM)
    if rank == 0:
        np.save(out_path, joint.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_counts_equal_single_process(tmp_path, world):
    import sys
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import ChainSpec, Oracle
    out = str(tmp_path / "joint.npy")
    mp.start_processes(_worker, args=(world, _free_port(), out), nprocs=world, join=True,
                       start_method="spawn")
    got = np.load(out).view(np.uint64)
    orc = Oracle("restatement")
    spec = ChainSpec(1, 4, sigma1=0.4, sigma2=0.7, alpha1=0.8, alpha2=3.5, rho=0.3)
    rng = np.random.default_rng(5)
    sizes = np.array([1, 9, 11, 7, 13], np.uint64)
    pts = rng.standard_normal(int(sizes[1:].sum()) * 2)
    ref = orc.estimate(1, spec, sizes, pts, 5001, workers=3)
    assert np.array_equal(got, ref.joint)


def test_shard_partition_covers_units_exactly():
    from paper_1101_3228_b200.dist import shard
    for units in (1, 7, 1000, 10**9, 10**9 * 365):
        for world in (1, 2, 3, 4, 8):
            spans = [shard(units, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (b0, c0), (b1, _) in zip(spans, spans[1:]):
                assert b0 + c0 == b1
            assert spans[-1][0] + spans[-1][1] == units
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
