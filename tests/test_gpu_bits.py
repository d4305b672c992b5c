"""GPU: the bit-packed +-1 device format.

* A complete +-1 instance given as packed sign bits and expanded on the
  device (nmfa_problem_create_bits_device) anneals bit-identically to the
  same instance built from a host edge list (same configurations, same
  exact energies), with and without integer fields.
* nmfa_energy on a device-built problem (tensor-core energy pass) is exact:
  equal to the float64 oracle's energy of random configurations.
* Above 4096 spins nmfa_problem_create_dense_bits takes the device route.
* Row shards of a bit-packed instance run the row-sharded protocol
  bit-identically to one GPU (G = 2, emulated in one process).
"""

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


def random_pm1(n, seed):
    rng = np.random.default_rng(seed)
    J = np.where(rng.random((n, n)) < 0.5, -1.0, 1.0)
    J = np.triu(J, 1)
    return J + J.T


@pytest.mark.parametrize("n,fields", [(600, False), (777, True)])
def test_device_expanded_bits_equal_host_problem(n, fields):
    J = random_pm1(n, n)
    h = np.random.default_rng(1).integers(-3, 4, n).astype(np.float64) if fields else None
    ei, ej = np.triu_indices(n, 1)
    host = nb.IsingProblem.from_arrays(n, ei, ej, J[ei, ej], h)
    host.device_handle().set_path("dense")
    dev = nb.PackedSignProblem.from_dense(J, h)
    assert dev.device_info()["path"] == "dense"
    params = nb.NmfaParams(t_f=150, seed=5)
    a = nb.sample(host, params, 300)
    b = nb.sample(dev, params, 300)
    assert torch.equal(a.configs, b.configs)
    assert torch.equal(a.energies, b.energies)
    op = O.problem_from_edges(n, ei, ej, J[ei, ej], h)
    assert np.array_equal(b.energies.cpu().numpy(), O.energies(op, b.configs.cpu().numpy().astype(float)))
    assert dev.w_total == J[ei, ej].sum()


def test_energy_of_device_problem_is_exact():
    n = 1000
    J = random_pm1(n, 3)
    dev = nb.PackedSignProblem.from_dense(J)
    cfg = np.where(np.random.default_rng(4).random((70, n)) < 0.5, -1.0, 1.0)
    e = nb.energies(dev, cfg)
    ei, ej = np.triu_indices(n, 1)
    assert np.array_equal(e, O.energies(O.problem_from_edges(n, ei, ej, J[ei, ej]), cfg))
    # the on-device SK generator's problems get exact energies the same way
    sk = RowShardedSK(512, 9, 64, nb.NmfaParams(t_f=5))   # keep it alive: it owns the handle
    out = torch.empty(3, dtype=torch.float64, device="cuda")
    c = torch.ones((3, 512), dtype=torch.int8, device="cuda")
    _native.check(_native.load().nmfa_energy(sk.problem, _native.ptr(c), 3, _native.ptr(out), None))
    Jsk = O.sk_device_couplings(512, 9)
    assert out[0].item() == 0.5 * Jsk.sum()


def test_large_bitmap_takes_the_device_route():
    n = 4500   # > 4096: no host edge list
    J = random_pm1(n, 7)
    bits = nb.pack_sign_bits(J)
    import ctypes
    out = ctypes.c_void_p()
    lib = _native.load()
    _native.check(lib.nmfa_problem_create_dense_bits(n, _native.ptr(bits), None, 0, ctypes.byref(out)))
    info = _native.ProblemInfo()
    _native.check(lib.nmfa_problem_get_info(out, ctypes.byref(info)))
    assert info.path == _native.PATH_DENSE and info.n == n
    lib.nmfa_problem_destroy(out)
    p = nb.PackedSignProblem(n, bits)
    r = nb.sample(p, nb.NmfaParams(t_f=40, seed=2), 256)
    cfg = r.configs.cpu().numpy().astype(np.float64)
    e_ref = 0.5 * np.einsum("ri,ij,rj->r", cfg, J, cfg)
    assert np.array_equal(r.energies.cpu().numpy(), e_ref)


def test_bit_packed_row_shards_equal_one_gpu():
    n, R, params, G = 768, 256, nb.NmfaParams(t_f=50, seed=13), 2
    J = random_pm1(n, 11)
    bits = nb.pack_sign_bits(J)
    ref = RowShardedSK(n, None, R, params, bits=bits).run(params.seed)
    want = nb.sample(nb.PackedSignProblem(n, bits), params, R)
    assert torch.equal(ref.configs, want.configs) and torch.equal(ref.energies, want.energies)
    shards = [RowShardedSK(n, None, R, params, shard=(G, g), bits=bits) for g in range(G)]
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
    assert torch.equal(shards[0].read_config(), ref.configs)
    assert torch.equal(torch.stack(parts).sum(0), ref.energies)


def test_gset_text_straight_to_device_problem():
    """nmfa_problem_create_gset: instance text -> device problem in one C call,
    the same problem as parse_gset + IsingProblem (and the same errors)."""
    import ctypes
    p = nb.gen_dense_maxcut(700, 0.02, 3)
    text = nb.write_gset(p).encode()
    lib = _native.load()
    out = ctypes.c_void_p()
    _native.check(lib.nmfa_problem_create_gset(text, len(text), 0, ctypes.byref(out)))
    info = _native.ProblemInfo()
    _native.check(lib.nmfa_problem_get_info(out, ctypes.byref(info)))
    ref = nb.parse_gset(text.decode())
    assert info.n == ref.n and info.n_edges == ref.num_edges
    assert nb.IsingProblem is type(ref)
    temps = np.ascontiguousarray(nb.DEFAULT_SCHEDULE.temperatures(50))
    cfg = torch.empty((64, ref.n), dtype=torch.int8, device="cuda")
    e = torch.empty(64, dtype=torch.float64, device="cuda")
    _native.check(lib.nmfa_anneal(out, 64, 50, _native.ptr(temps), 0.15, 0.15, 4, 0, None, None,
                                  _native.ptr(cfg), _native.ptr(e), None, None, None, None))
    torch.cuda.synchronize()
    want = nb.sample(ref, nb.NmfaParams(t_f=50, seed=4), 64)
    assert torch.equal(cfg, want.configs) and torch.equal(e, want.energies)
    lib.nmfa_problem_destroy(out)
    bad = b"3 2\n1 2 1\n1 9 1\n"
    assert lib.nmfa_problem_create_gset(bad, len(bad), 0, ctypes.byref(out)) == _native.NMFA_ERR_ARG
    assert lib.nmfa_last_error().decode().startswith("line 3")
