"""Multi-process host logic of replica sharding (gloo, world size 2, CPU).

The GPU kernels are not exercised here; a CPU stand-in sampler returns an
energy that is a fixed function of the GLOBAL replica index, which is exactly
the property the device path guarantees (noise keyed by seed + r).  The test
checks that shards tile [0, n) and that the gathered best-of-reads equals the
single-process answer for every world size.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1806_08422_b200.distributed import gather_best, pick_best, sample_sharded, shard_range


class _FakeSample:
    def __init__(self, energies):
        self.energies = torch.as_tensor(energies, dtype=torch.float64)


def fake_energy(r):
    r = np.asarray(r, dtype=np.int64)
    return -((r * 2654435761) % 1009).astype(np.float64)   # many ties at the minimum


def fake_sampler(problem, params, count, r0=0, device=None):
    return _FakeSample(fake_energy(np.arange(r0, r0 + count)))


def test_shard_range_tiles_replicas():
    for n in (1, 7, 100, 8192, 65536):
        for world in (1, 2, 3, 8):
            if world > n:
                continue
            spans = [shard_range(n, world, k) for k in range(world)]
            assert spans[0][0] == 0
            assert all(spans[k][0] + spans[k][1] == spans[k + 1][0] for k in range(world - 1))
            assert spans[-1][0] + spans[-1][1] == n
            assert max(c for _, c in spans) - min(c for _, c in spans) <= 1
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


def test_pick_best_breaks_ties_by_index():
    assert pick_best([(-3.0, 9), (-3.0, 4), (-1.0, 0)]) == (-3.0, 4)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_total, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = sample_sharded(None, None, n_total, rank=rank, world=world, sampler=fake_sampler)
        # every rank sees the same global best
        t = torch.tensor([res.best_energy, res.best_index], dtype=torch.float64)
        allt = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        out[rank] = (res.r0, len(res.sample.energies), [tuple(x.tolist()) for x in allt])
        # gather_best with ties across ranks -> lowest global index
        be, bi = gather_best(-5.0, 100 + rank)
        assert (be, bi) == (-5.0, 100)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_best_of_matches_single_process(world):
    n_total = 1000
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), n_total, out), nprocs=world, join=True)
    e = fake_energy(np.arange(n_total))
    want = (float(e.min()), int(np.flatnonzero(e == e.min())[0]))
    spans = sorted((out[k][0], out[k][1]) for k in range(world))
    assert spans[0][0] == 0 and sum(c for _, c in spans) == n_total
    for k in range(world):
        assert all(tuple(p) == want for p in out[k][2])


def test_single_process_identity():
    res = sample_sharded(None, None, 37, rank=0, world=1, sampler=fake_sampler)
    e = fake_energy(np.arange(37))
    assert res.best_energy == e.min() and res.best_index == int(np.argmin(e))
