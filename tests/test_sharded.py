"""Row-sharded J (config 5) host logic on CPU: shard geometry, the Philox
twin of the on-device SK generator (pinned to the published Random123
known-answer vectors), and the in-place slice all-gather under gloo world 2."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import nmfa_oracle as O
from paper_1806_08422_b200.sharded import exchange_slices, row_shard


def test_row_shard_tiles_rows():
    n, world = 65536, 8
    spans = [row_shard(n, world, g) for g in range(world)]
    assert spans[0][0] == 0 and spans[-1][1] == n
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
    assert all(lo % 128 == 0 for lo, _ in spans)
    with pytest.raises(ValueError):
        row_shard(1000, 2, 0)


# Random123 philox4x32_10 known-answer vectors (kat_vectors: ctr, key -> out)
PHILOX_KAT = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, (0xFFFFFFFF,) * 2, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", PHILOX_KAT)
def test_philox_twin_known_answers(ctr, key, want):
    got = O.philox4x32_10(*[np.array([c], np.uint32) for c in ctr], *key)
    assert tuple(int(w[0]) for w in got) == want


def test_sk_device_couplings_shape_and_balance():
    J = O.sk_device_couplings(256, 5)
    assert np.array_equal(J, J.T) and np.all(np.diag(J) == 0)
    off = J[~np.eye(256, dtype=bool)]
    assert set(np.unique(off)) == {-1.0, 1.0}
    # fair coin: mean of 32,640 independent +-1 within 5 sigma
    assert abs(off.mean()) < 5 / np.sqrt(off.size / 2)
    assert not np.array_equal(J, O.sk_device_couplings(256, 6))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_slices_per, sb, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        img = torch.full((world * n_slices_per * sb + 7,), 255, dtype=torch.uint8)
        lo, hi = rank * n_slices_per, (rank + 1) * n_slices_per
        mine = torch.arange(lo * sb, hi * sb, dtype=torch.int64) % 251
        img[lo * sb: hi * sb] = mine.to(torch.uint8)
        exchange_slices(img, lo, hi, sb)
        out[rank] = img.numpy().copy()
    finally:
        dist.destroy_process_group()


def test_exchange_slices_gathers_every_shard():
    world, per, sb = 2, 3, 64
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), per, sb, out), nprocs=world, join=True)
    want = (np.arange(world * per * sb) % 251).astype(np.uint8)
    for g in range(world):
        assert np.array_equal(out[g][: world * per * sb], want)
        assert np.all(out[g][world * per * sb:] == 255)   # bytes past the slabs untouched


def test_device_normals_spec_moments():
    """The oracle twin of the in-kernel noise (tests/test_gpu_noise.py pins the
    kernels to it): N(0, sigma^2) moments, the 20-bit radius tail bound, and
    replica / step streams that differ."""
    z = O.device_normals(7, np.arange(0, 2000), 0, 64, 1.0)
    assert abs(z.mean()) < 0.01 and abs(z.var() - 1.0) < 0.02
    assert abs(np.mean(z ** 4) - 3.0) < 0.1          # Gaussian kurtosis
    assert np.abs(z).max() <= np.sqrt(-2 * np.log(0.5 * 2.0 ** -20)) + 1e-12
    z1 = O.device_normals(7, np.arange(0, 4), 1, 64, 1.0)
    assert not np.allclose(z[:4], z1) and not np.allclose(z[0], z[1])


# ---------------------------------------------------------------------------
# The full RowShardedSK.run host protocol (ShardProtocol.run) under gloo world 2,
# with a CPU stand-in for the CUDA shard: same image geometry (k-slice-major
# flat bytes, one contiguous chunk per rank), same sweep / exchange / energy
# pass / all-reduce order.  Compared with the unsharded (world 1) run.
# ---------------------------------------------------------------------------
from paper_1806_08422_b200.sharded import ShardProtocol  # noqa: E402
from paper_1806_08422_b200.solver import NmfaParams  # noqa: E402


class CpuShard(ShardProtocol):
    SLICE = 128

    def __init__(self, J, R, params, world, rank, group=None):
        self.J, self.n, self.R, self.params = J, J.shape[0], R, params
        self.world, self.rank, self.group = world, rank, group
        self.n_slices = self.n // self.SLICE
        per = self.n_slices // world
        self.slice_lo, self.slice_hi = rank * per, (rank + 1) * per
        self.slice_bytes = R * self.SLICE * 8                  # float64 state, [slice][r][128]
        self.images = [torch.zeros(self.n_slices * self.slice_bytes, dtype=torch.uint8)
                       for _ in range(2)]
        self.norm = np.sqrt((J ** 2).sum(axis=1))
        self.temps = params.schedule.temperatures(params.t_f)

    def state(self, parity):
        v = self.images[parity].numpy().view(np.float64).reshape(self.n_slices, self.R, self.SLICE)
        return v.transpose(1, 0, 2).reshape(self.R, self.n)       # (R, n) copy

    def noise(self, seed, r0, t):
        # keyed by (global replica, step): the same values whatever the sharding
        return np.stack([np.random.default_rng([seed, r0 + r, t]).standard_normal(self.n)
                         for r in range(self.R)]) * self.params.sigma

    def sweeps(self, seed, t_begin, t_end, r0=0, energy=None, stream=None):
        a, lo, hi = self.params.alpha, self.slice_lo * self.SLICE, self.slice_hi * self.SLICE
        for t in range(t_begin, t_end):
            S = self.state(t & 1)
            phi = S @ self.J[lo:hi].T / self.norm[lo:hi] + self.noise(seed, r0, t)[:, lo:hi]
            new = a * -np.tanh(phi / self.temps[t]) + (1 - a) * S[:, lo:hi]
            if t == self.params.t_f - 1:
                new = np.where(new < 0, -1.0, 1.0)      # the last sweep writes the +-1 config
            dst = self.images[(t + 1) & 1].numpy().view(np.float64).reshape(
                self.n_slices, self.R, self.SLICE)
            dst[self.slice_lo:self.slice_hi] = new.reshape(self.R, -1, self.SLICE).transpose(1, 0, 2)
        if energy is not None:
            c = self.state(self.params.t_f & 1)
            part = 0.5 * np.einsum("ri,ri->r", c[:, lo:hi], c @ self.J[lo:hi].T)
            energy.copy_(torch.from_numpy(part))

    def new_energy(self):
        return torch.zeros(self.R, dtype=torch.float64)

    def read_config(self, stream=None):
        return torch.from_numpy(self.state(self.params.t_f & 1).astype(np.int8))


def _protocol_J(n=256):
    J = O.sk_device_couplings(n, 3)
    return J


def _protocol_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        shard = CpuShard(_protocol_J(), 8, NmfaParams(t_f=40, seed=5), world, rank)
        res = shard.run(5, r0=16)
        out[rank] = (res.configs.numpy().copy(), res.energies.numpy().copy(), res.sweeps)
    finally:
        dist.destroy_process_group()


def test_row_sharded_protocol_world2_equals_unsharded():
    J = _protocol_J()
    solo = CpuShard(J, 8, NmfaParams(t_f=40, seed=5), 1, 0).run(5, r0=16)
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_protocol_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    want_e = 0.5 * np.einsum("ri,ri->r", solo.configs.numpy().astype(np.float64),
                             solo.configs.numpy().astype(np.float64) @ J)
    assert np.allclose(solo.energies.numpy(), want_e)
    for g in range(2):
        cfg, en, sweeps = out[g]
        assert sweeps == 40
        assert np.array_equal(cfg, solo.configs.numpy()), g      # every rank sees all spins
        assert np.array_equal(en, solo.energies.numpy()), g      # integers: exact all-reduce
