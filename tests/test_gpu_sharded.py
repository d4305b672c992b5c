"""GPU: the on-device SK generator and the row-sharded-J protocol (config 5).

* the device-generated instance equals the host-built problem with the
  oracle's twin couplings (same configs, bit-exact energies);
* G-way row sharding is invariant: G shards run one sweep each, exchange
  their k-slices, sum their energy partials -- bit-identical to G = 1.  The
  shards run one after another in one process (no kernel waits on another).
"""

import ctypes

import numpy as np
import pytest

import nmfa_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1806_08422_b200 as nb  # noqa: E402
from paper_1806_08422_b200 import _native  # noqa: E402
from paper_1806_08422_b200.sharded import RowShardedSK  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1806_08422_b200 import build
    build.build()
    _native.load()


def host_problem(n, sk_seed):
    J = O.sk_device_couplings(n, sk_seed)
    ei, ej = np.triu_indices(n, 1)
    return nb.IsingProblem.from_arrays(n, ei, ej, J[ei, ej]), J


@pytest.mark.parametrize("n", [512, 600])
def test_device_sk_equals_host_built_problem(n):
    sk_seed, params, R = 9, nb.NmfaParams(t_f=120, seed=3), 256
    p, J = host_problem(n, sk_seed)
    want = nb.sample(p, params, R)
    got = RowShardedSK(n, sk_seed, R, params).run(params.seed)
    assert torch.equal(got.configs, want.configs)
    assert torch.equal(got.energies, want.energies)
    cfg = got.configs.cpu().numpy().astype(np.float64)
    e_ref = 0.5 * np.einsum("ri,ij,rj->r", cfg, J, cfg)   # H = 1/2 c^T J c (h = 0)
    assert np.array_equal(got.energies.cpu().numpy(), e_ref)


def run_emulated(n, sk_seed, R, params, G):
    shards = [RowShardedSK(n, sk_seed, R, params, shard=(G, g)) for g in range(G)]
    for t in range(params.t_f):
        for s in shards:
            s.sweeps(params.seed, t, t + 1)
        full = torch.cat([s.image_chunk((t + 1) & 1) for s in shards])
        for s in shards:
            s.images[(t + 1) & 1][: full.numel()].copy_(full)
    parts = []
    for s in shards:
        e = torch.empty(R, dtype=torch.float64, device="cuda")
        s.sweeps(params.seed, params.t_f, params.t_f, energy=e)
        parts.append(e)
    cfgs = [s.read_config() for s in shards]
    for c in cfgs[1:]:
        assert torch.equal(c, cfgs[0])
    return cfgs[0], torch.stack(parts).sum(0)


@pytest.mark.parametrize("G", [2, 4])
def test_row_sharding_is_invariant(G):
    n, sk_seed, R, params = 512, 4, 256, nb.NmfaParams(t_f=60, seed=21)
    ref = RowShardedSK(n, sk_seed, R, params).run(params.seed)
    cfg, e = run_emulated(n, sk_seed, R, params, G)
    assert torch.equal(cfg, ref.configs)
    assert torch.equal(e, ref.energies)


def test_sharded_problem_guards():
    lib = _native.load()
    s = RowShardedSK(512, 1, 256, nb.NmfaParams(t_f=10, seed=0), shard=(2, 1))
    assert (s.slice_lo, s.slice_hi, s.n_slices) == (2, 4, 4)
    with pytest.raises(ValueError):
        s.sweeps(0, 0, 2)                       # one sweep per call when sharded
    with pytest.raises(ValueError):
        s.sweeps(0, 0, 1, energy=torch.empty(256, dtype=torch.float64, device="cuda"))
    cfg = torch.empty((256, 512), dtype=torch.int8, device="cuda")
    e = torch.empty(256, dtype=torch.float64, device="cuda")
    assert lib.nmfa_energy(s.problem, _native.ptr(cfg), 256, _native.ptr(e), None) != 0
    assert lib.nmfa_problem_set_path(s.problem, _native.PATH_SPARSE) != 0
    with pytest.raises(ValueError):
        RowShardedSK(1000, 1, 256, nb.NmfaParams(t_f=10), shard=(2, 0))


@pytest.mark.parametrize("G", [2, 4])
def test_fused_exchange_equals_unsharded(G):
    """Fused exchange (nmfa_plan_set_exchange): each shard's epilogue stores its
    new state lines into every shard's image, no separate all-gather.  Shards
    run one after another on one device; results must equal G = 1 bit for bit."""
    from paper_1806_08422_b200.sharded import link_local_shards
    n, sk_seed, R, params = 512, 4, 256, nb.NmfaParams(t_f=60, seed=21)
    ref = RowShardedSK(n, sk_seed, R, params).run(params.seed)
    shards = [RowShardedSK(n, sk_seed, R, params, shard=(G, g)) for g in range(G)]
    link_local_shards(shards)
    for t in range(params.t_f):
        for s in shards:
            s.sweeps(params.seed, t, t + 1)
    parts = []
    for s in shards:
        e = torch.empty(R, dtype=torch.float64, device="cuda")
        s.sweeps(params.seed, params.t_f, params.t_f, energy=e)
        parts.append(e)
    for s in shards:
        assert torch.equal(s.read_config(), ref.configs)
    assert torch.equal(torch.stack(parts).sum(0), ref.energies)


def test_fused_exchange_argument_checks():
    lib = _native.load()
    s = RowShardedSK(512, 1, 256, nb.NmfaParams(t_f=10, seed=0), shard=(2, 0))
    P = ctypes.c_void_p * 2
    ptr = ctypes.c_void_p(s.images[0].data_ptr())
    good = P(ptr, ptr)
    assert lib.nmfa_plan_set_exchange(s.plan, ctypes.cast(good, ctypes.c_void_p),
                                      ctypes.cast(good, ctypes.c_void_p), 9, 0, 1 << 30) != 0
    assert lib.nmfa_plan_set_exchange(s.plan, ctypes.cast(good, ctypes.c_void_p),
                                      ctypes.cast(good, ctypes.c_void_p), 2, 0, 16) != 0
