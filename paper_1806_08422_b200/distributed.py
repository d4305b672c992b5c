"""Replica sharding across GPUs (one process per GPU, torch.distributed).

The reference runs replicas on a thread pool (solver.py:277-280) and its
results do not depend on the thread count.  Here replicas are split into
contiguous global ranges, one per rank; replica r always draws its noise
from key seed + r (common.cuh), so every global replica produces the same
configuration whatever the world size (tests/test_distributed.py).  The data
path has no collective: the only communication is one all-gather of each
rank's (best energy, global index) pair for the best-of-reads result.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def shard_range(n_total, world, rank):
    """(r0, count) of the contiguous replica shard owned by `rank`."""
    n_total, world, rank = int(n_total), int(world), int(rank)
    if n_total < 1 or world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad shard request n={n_total} world={world} rank={rank}")
    r0 = n_total * rank // world
    r1 = n_total * (rank + 1) // world
    return r0, r1 - r0


def pick_best(pairs):
    """Global best from rows of (energy, global index): min energy, lowest index."""
    pairs = np.asarray(pairs, dtype=np.float64).reshape(-1, 2)
    k = np.lexsort((pairs[:, 1], pairs[:, 0]))[0]
    return float(pairs[k, 0]), int(pairs[k, 1])


def gather_best(best_energy, best_index, group=None):
    """All-gather every rank's (best energy, global index) and reduce on all ranks.

    Works with NCCL (device tensors) and gloo (CPU tensors); with no
    initialised process group it is the identity.
    """
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()):
        return float(best_energy), int(best_index)
    dev = torch.device("cpu")
    if dist.get_backend(group) == "nccl":
        dev = torch.device("cuda", torch.cuda.current_device())
    mine = torch.tensor([float(best_energy), float(best_index)], dtype=torch.float64, device=dev)
    world = dist.get_world_size(group)
    allp = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(allp, mine, group=group)
    return pick_best(torch.stack(allp).cpu().numpy())


@dataclass
class ShardedSample:
    sample: object          # the local SampleSet (device tensors)
    r0: int                 # first global replica of this shard
    n_total: int
    best_energy: float      # global best-of-reads
    best_index: int         # global replica index attaining it


def sample_sharded(problem, params, n_total, rank=None, world=None, device=None, sampler=None):
    """Run this rank's shard of n_total replicas and reduce the global best.

    `sampler(problem, params, count, r0=..., device=...)` defaults to
    `solver.sample`; tests substitute a CPU stand-in to exercise the
    host-side logic under gloo.
    """
    import torch.distributed as dist

    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    if sampler is None:
        from .solver import sample as sampler
    r0, count = shard_range(n_total, world, rank)
    dev = rank if device is None else device
    ss = sampler(problem, params, count, r0=r0, device=dev)
    e = ss.energies.double().cpu().numpy()
    k = int(np.lexsort((np.arange(e.size), e))[0])
    best_e, best_i = gather_best(e[k], r0 + k)
    return ShardedSample(ss, r0, int(n_total), best_e, best_i)
