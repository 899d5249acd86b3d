"""The N > 1 path on real device kernels: two ranks (torch.distributed, gloo,
both on cuda:0 — the gpurun box has one GPU) shard the paths with the
reference's worker formula (estimate.hpp:180-181), count with the path kernel,
and all-reduce the int64 counts. The tree on rank 0 must equal the
single-process estimate bit for bit (the G-GPU analogue of test_tree.cpp:128-152)."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out, kind):
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1101_3228_b200 import qtree as q
    from paper_1101_3228_b200.dist import estimate_distributed
    if kind == "bm":
        ch = q.BrownianChain1d(10)
        grids = q.build_brownian_grids(ch, 100)
        alg, M = 1, 300001
    else:
        ch = q.TwoFactorChain(q.TwoFactorParams(steps=6))
        grids = q.build_two_factor_grids(ch, 1000)
        alg, M = 2, 20001  # Alg III
    t = estimate_distributed(alg, ch, grids, M)
    if rank == 0:
        np.savez(out, visits=t.flat_visits, joint=t.flat_joint, pi=t.flat_pi)
    dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["bm", "tf3"])
def test_two_rank_estimate_equals_single_process(gpu, tmp_path, kind):
    from paper_1101_3228_b200 import qtree as q
    out = str(tmp_path / "tree.npz")
    mp.start_processes(_worker, args=(2, _free_port(), out, kind), nprocs=2, join=True,
                       start_method="spawn")
    got = np.load(out)
    if kind == "bm":
        ch = q.BrownianChain1d(10)
        t = q.estimate_alg2(ch, q.build_brownian_grids(ch, 100), 300001)
    else:
        ch = q.TwoFactorChain(q.TwoFactorParams(steps=6))
        t = q.estimate_alg3(ch, q.build_two_factor_grids(ch, 1000), 20001)
    assert np.array_equal(got["joint"], t.flat_joint)
    assert np.array_equal(got["visits"], t.flat_visits)
    assert np.array_equal(got["pi"], t.flat_pi)
