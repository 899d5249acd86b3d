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


def test_multi_device_one_call_equals_single_device(gpu):
    """qt_estimate(devices=G) (estimate.hpp:163-207's worker merge across the
    GPUs of one process: shards [M g/G, M (g+1)/G), one grouped NCCL
    all-reduce) equals devices=1 bit for bit, and the caller's current
    device is left as it was. Needs two visible GPUs (the gpurun box has
    one: then only the single-device half and the error path run)."""
    import torch
    from paper_1101_3228_b200 import qtree as q
    ch = q.BrownianChain1d(12)
    grids = q.build_brownian_grids(ch, 120)
    one = q.estimate_alg2(ch, grids, 200001)
    visible = torch.cuda.device_count()
    if visible < 2:
        with pytest.raises(ValueError, match="devices"):
            q.estimate_alg2(ch, grids, 1000, q.EstimateOptions(devices=2))
        assert torch.cuda.current_device() == 0
        pytest.skip(f"devices=2 needs two GPUs; this box has {visible} (error path checked)")
    for G in sorted({2, min(visible, 4), visible}):
        many = q.estimate_alg2(ch, grids, 200001, q.EstimateOptions(devices=G))
        assert np.array_equal(many.flat_joint, one.flat_joint), G
        assert np.array_equal(many.flat_visits, one.flat_visits), G
        assert np.array_equal(many.flat_pi.view(np.uint64), one.flat_pi.view(np.uint64)), G
        assert torch.cuda.current_device() == 0
    # from another base device: devices [1, 2) of the process
    torch.cuda.set_device(1)
    try:
        t = q.estimate_alg2(ch, grids, 200001)
        assert np.array_equal(t.flat_joint, one.flat_joint)
        assert torch.cuda.current_device() == 1
    finally:
        torch.cuda.set_device(0)
