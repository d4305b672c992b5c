"""Row-sharded J over GPUs (BASELINE config 5: synthetic SK N = 65,536).

Each rank holds rows [g*N/G, (g+1)*N/G) of J (its spins) and computes the
mean fields of its spins for ALL replicas over the full K = N, so the
contraction needs every spin's state: after each sweep the ranks all-gather
the k-slices of the next operand image they wrote (one contiguous chunk per
rank, NCCL over NVLink).  Energies are per-shard partials of
1/2 sum_i c_i (J c)_i, all-reduced (exact: integers in f64).

The reference has no counterpart (its dense J is an n x n float64 matrix,
problem.py:100-104, infeasible at N = 65,536); this is the §8(e) scaling mode.
On one GPU the problem is unsharded and the whole anneal is one persistent
launch.  With G > 1 a sweep is one launch followed by the exchange:
  exchange="nccl"  one in-place NCCL all-gather of the sweep's image;
  exchange="p2p"   fused: the operand images live in symmetric (peer-mapped)
                   memory and each sweep's epilogue stores every new state
                   line into all G images itself (nmfa_plan_set_exchange), so
                   the transfer overlaps the GEMM; a device-side barrier
                   separates sweeps.
Noise is keyed by the global replica and spin index and the K order is fixed,
so results do not depend on G or on the exchange.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _native
from .solver import MASK64, NmfaParams


def row_shard(n, world, rank, align=128):
    """Spin rows [lo, hi) of rank `rank`; every shard but the last is `align`-aligned."""
    n, world, rank = int(n), int(world), int(rank)
    if n % (align * world) != 0:
        raise ValueError(f"row sharding needs n divisible by {align} x world ({align * world}), "
                         f"got n = {n}")
    per = n // world
    return rank * per, (rank + 1) * per


def _default_group():
    import torch.distributed as dist
    return dist.group.WORLD


def link_images(shard, ptrs, world, rank, nbytes):
    """Point `shard`'s plan at every shard's operand images: ptrs[p][g] is shard
    g's image of sweep parity p.  Entry [rank] becomes the shard's own image."""
    P = ctypes.c_void_p * world
    _native.check(_native.load().nmfa_plan_set_exchange(
        shard.plan, ctypes.cast(P(*ptrs[0]), ctypes.c_void_p),
        ctypes.cast(P(*ptrs[1]), ctypes.c_void_p), int(world), int(rank), int(nbytes)))


def link_local_shards(shards):
    """Single-process emulation of the fused exchange: shards that live on one
    device store straight into each other's images (tests; one GPU)."""
    G = len(shards)
    ptrs = [[s.images[p].data_ptr() for s in shards] for p in range(2)]
    for g, s in enumerate(shards):
        link_images(s, ptrs, G, g, s.images[0].numel())


class _CudaBytes:
    """__cuda_array_interface__ view of raw device bytes (zero copy)."""

    def __init__(self, ptr, nbytes):
        self.__cuda_array_interface__ = {"shape": (int(nbytes),), "typestr": "|u1",
                                         "data": (int(ptr), False), "version": 3}


def exchange_slices(image, slice_lo, slice_hi, slice_bytes, group=None):
    """In-place all-gather of every rank's contiguous k-slice chunk of `image`.

    `image` is a flat uint8 tensor (CUDA with NCCL, CPU with gloo); rank g owns
    bytes [slice_lo*slice_bytes, slice_hi*slice_bytes) and all ranks own equally
    many slices in rank order.
    """
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return
    world = dist.get_world_size(group)
    chunk = (slice_hi - slice_lo) * slice_bytes
    out = image[: world * chunk]
    mine = image[slice_lo * slice_bytes: slice_hi * slice_bytes]
    dist.all_gather_into_tensor(out, mine, group=group)


def allreduce_sum(t, group=None):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class ShardProtocol:
    """The per-anneal host protocol of a row-sharded plan, independent of where
    the shard computes (CUDA plan here; a CPU stand-in in tests/test_sharded.py).

    A shard provides: world, rank, R, params, images[2] (flat uint8 tensors),
    slice_lo/slice_hi/slice_bytes, group, sweeps(seed, t_begin, t_end, r0,
    energy, stream), new_energy(), read_config(stream), exchange_after(t,
    stream)."""

    def exchange_after(self, t, stream=None):
        """Make sweep t's new image (parity (t + 1) & 1) complete on every shard."""
        exchange_slices(self.images[(t + 1) & 1], self.slice_lo, self.slice_hi, self.slice_bytes,
                        self.group)

    def run(self, seed, r0=0, stream=None):
        """One anneal of all t_f sweeps; returns configs and exact total energies.

        G = 1: one persistent launch (all sweeps + the energy pass).  G > 1: per
        sweep t one launch on the shard, then the exchange of image (t+1) & 1;
        after the last sweep the energy pass gives per-shard partials of
        1/2 sum_i c_i (J c)_i + h.c (integers in f64), summed over the ranks."""
        t_f = self.params.t_f
        en = self.new_energy()
        if self.world == 1:
            self.sweeps(seed, 0, t_f, r0, energy=en, stream=stream)
        else:
            for t in range(t_f):
                self.sweeps(seed, t, t + 1, r0, stream=stream)
                self.exchange_after(t, stream)
            self.sweeps(seed, t_f, t_f, r0, energy=en, stream=stream)
            self.reduce_energy(en, stream)
        return ShardedResult(self.read_config(stream), en, t_f)

    def reduce_energy(self, en, stream=None):
        allreduce_sum(en, self.group)


@dataclass
class ShardedResult:
    configs: object        # torch.int8 (R, n) on this rank's device (all spins)
    energies: object       # torch.float64 (R,) total energies (all-reduced)
    sweeps: int


class RowShardedSK(ShardProtocol):
    """SK instance with J row-sharded over the ranks of `group`: the synthetic
    on-device generator (`seed`), or a user's complete +-1 instance given as
    packed sign bits (`bits`, the bit-packed device format of
    problem.PackedSignProblem; each rank expands only its rows)."""

    def __init__(self, n, seed, n_reads, params=None, group=None, device=None, shard=None,
                 exchange="nccl", bits=None, h=None):
        import torch
        import torch.distributed as dist

        self.params = params or NmfaParams()
        self.group = group
        if shard is not None:            # explicit (world, rank): single-process emulation
            self.world, self.rank = int(shard[0]), int(shard[1])
        else:
            init = dist.is_available() and dist.is_initialized()
            self.world = dist.get_world_size(group) if init else 1
            self.rank = dist.get_rank(group) if init else 0
        self.device = torch.cuda.current_device() if device is None else int(device)
        self.n, self.R = int(n), int(n_reads)
        self.row_lo, self.row_hi = row_shard(n, self.world, self.rank) if self.world > 1 else (0, n)
        lib = _native.load()
        out = ctypes.c_void_p()
        if bits is None:
            _native.check(lib.nmfa_problem_create_sk_device(self.n, int(seed) & MASK64,
                                                            self.row_lo, self.row_hi, self.device,
                                                            ctypes.byref(out)))
        else:
            self._bits = np.ascontiguousarray(bits, dtype=np.uint32)
            self._h = None if h is None else np.ascontiguousarray(h, dtype=np.float64)
            if self._bits.size < (self.n * self.n + 31) // 32:
                raise ValueError("bitmap too short for n")
            _native.check(lib.nmfa_problem_create_bits_device(
                self.n, _native.ptr(self._bits), _native.ptr(self._h), self.row_lo, self.row_hi,
                self.device, ctypes.byref(out)))
        self.problem = out
        self.temps = np.ascontiguousarray(self.params.schedule.temperatures(self.params.t_f))
        plan = ctypes.c_void_p()
        _native.check(lib.nmfa_plan_create(self.problem, self.R, self.params.t_f,
                                           _native.ptr(self.temps), self.params.alpha,
                                           self.params.sigma, ctypes.byref(plan)))
        self.plan = plan
        i0, i1 = ctypes.c_void_p(), ctypes.c_void_p()
        sb = ctypes.c_int64()
        ns, slo, shi = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        _native.check(lib.nmfa_plan_image_info(self.plan, ctypes.byref(i0), ctypes.byref(i1),
                                               ctypes.byref(sb), ctypes.byref(ns),
                                               ctypes.byref(slo), ctypes.byref(shi)))
        self.slice_bytes, self.n_slices = sb.value, ns.value
        self.slice_lo, self.slice_hi = slo.value, shi.value
        dev = torch.device("cuda", self.device)
        nbytes = self.slice_bytes * self.n_slices
        self.images = [torch.as_tensor(_CudaBytes(p.value, nbytes), device=dev) for p in (i0, i1)]
        if exchange not in ("nccl", "p2p"):
            raise ValueError(f"exchange must be 'nccl' or 'p2p', got {exchange!r}")
        self.exchange = exchange
        self._symm = None
        if exchange == "p2p" and self.world > 1 and shard is None:
            try:
                self._setup_p2p(nbytes, dev)
            except Exception as exc:  # no symmetric memory / multicast here: NCCL exchange
                import warnings
                warnings.warn(f"fused p2p exchange unavailable ({exc}); using the NCCL all-gather")
                self.exchange = "nccl"

    def _setup_p2p(self, nbytes, dev):
        """Symmetric-memory images + pointer exchange (nmfa_plan_set_exchange)."""
        import torch
        from torch.distributed import _symmetric_memory as symm_mem

        bufs = [symm_mem.empty(nbytes, dtype=torch.uint8, device=dev) for _ in range(2)]
        hdls = [symm_mem.rendezvous(b, self.group or _default_group()) for b in bufs]
        link_images(self, [h.buffer_ptrs for h in hdls], self.world, self.rank, nbytes)
        self.images = bufs
        self._symm = (bufs, hdls)

    def _barrier(self):
        """Every shard's stores of this sweep are visible before the next one reads."""
        self._symm[1][0].barrier(channel=0)

    # -- the protocol, one piece at a time (run() strings them together) --
    def _stream(self, stream):
        import torch
        return stream or torch.cuda.current_stream(torch.device("cuda", self.device))

    def sweeps(self, seed, t_begin, t_end, r0=0, energy=None, stream=None):
        """Sweeps [t_begin, t_end) on this shard (+ the energy pass if `energy`)."""
        sp = ctypes.c_void_p(self._stream(stream).cuda_stream)
        _native.check(_native.load().nmfa_plan_run_sweeps(
            self.plan, int(seed) & MASK64, int(r0), int(t_begin), int(t_end),
            1 if energy is not None else 0, None, _native.ptr(energy), sp))

    def image_chunk(self, parity):
        """This shard's k-slices of operand image `parity` (what it contributes)."""
        sb = self.slice_bytes
        return self.images[parity][self.slice_lo * sb: self.slice_hi * sb]

    def read_config(self, stream=None):
        import torch
        cfg = torch.empty((self.R, self.n), dtype=torch.int8,
                          device=torch.device("cuda", self.device))
        sp = ctypes.c_void_p(self._stream(stream).cuda_stream)
        _native.check(_native.load().nmfa_plan_read_config(self.plan, _native.ptr(cfg), sp))
        return cfg

    def new_energy(self):
        import torch
        return torch.empty(self.R, dtype=torch.float64, device=torch.device("cuda", self.device))

    def exchange_after(self, t, stream=None):
        import torch
        with torch.cuda.stream(self._stream(stream)):
            if self._symm is not None:
                self._barrier()          # the epilogue already stored into every image
            else:
                super().exchange_after(t, stream)

    def reduce_energy(self, en, stream=None):
        import torch
        with torch.cuda.stream(self._stream(stream)):
            allreduce_sum(en, self.group)

    def __del__(self):
        try:
            lib = _native.load()
            if getattr(self, "plan", None):
                lib.nmfa_plan_destroy(self.plan)
            if getattr(self, "problem", None):
                lib.nmfa_problem_destroy(self.problem)
        except Exception:
            pass
