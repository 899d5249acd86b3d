"""Multi-process estimation: one process per GPU under torch.distributed.

Paths are sharded exactly like the reference's Algorithm II workers,
[M g / G, M (g+1) / G) (estimate.hpp:180-181); each rank counts its shard with
the fused path kernel into a private int64 joint matrix, and a single NCCL
all-reduce (sum) replaces CountMatrixSet::add (quant_tree.hpp:35-40).
Counts are bit-identical for any world size because every path's stream is
positioned by its global index (stream.hpp:190-199) and integer sums are
associative.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .device import Plan
from .qtree import EstimatorKind, QuantGrid, QuantTree


def shard(units: int, rank: int, world: int) -> tuple[int, int]:
    """[first, first+count) of rank's share of `units` (estimate.hpp:180-181)."""
    b = units * rank // world
    e = units * (rank + 1) // world
    return b, e - b


def estimate_distributed(kind, chain, grids, samples: int, engine=1, seed=12345,
                         plan: Plan | None = None, group=None) -> QuantTree | None:
    """tree::estimate over all ranks of `group`; rank 0 returns the QuantTree
    (host), the other ranks return None."""
    kind = EstimatorKind(int(kind))
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    dev = torch.cuda.current_device()
    plan = plan or Plan(chain, grids, dev)
    units = samples * chain.layers() if kind == EstimatorKind.AlgIII else samples
    first, count = shard(units, rank, world)
    joint = plan.zeros_joint()
    plan.count(kind, engine, seed, first, count, units, joint)
    if world > 1:
        dist.all_reduce(joint, op=dist.ReduceOp.SUM, group=group)
    if rank != 0:
        return None
    visits = torch.empty(plan.n_visits, dtype=torch.int64, device=joint.device)
    pi = torch.empty(plan.n_joint, dtype=torch.float64, device=joint.device)
    plan.finalize(kind, samples, joint, visits, pi)
    # device -> pinned host (a pageable .cpu() of the 2 x 98 MB at C2 runs at a few GB/s)
    hv = torch.empty(visits.shape, dtype=visits.dtype, pin_memory=True)
    hj = torch.empty(joint.shape, dtype=joint.dtype, pin_memory=True)
    hp = torch.empty(pi.shape, dtype=pi.dtype, pin_memory=True)
    hv.copy_(visits, non_blocking=True)
    hj.copy_(joint, non_blocking=True)
    hp.copy_(pi, non_blocking=True)
    torch.cuda.current_stream(joint.device).synchronize()
    v = hv.numpy().view(np.uint64)
    j = hj.numpy().view(np.uint64)
    p = hp.numpy()
    x0 = QuantGrid(chain.dim(), np.zeros(chain.dim()))
    return QuantTree([x0] + list(grids), plan.sizes, v, j, p, samples)
