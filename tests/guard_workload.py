"""Workload for tests/test_gpu_guarded.py (not collected by pytest): one
short run of every kernel path with fixed seeds, outputs saved to an .npz.

Run once against the product library and once with NMFA_LIB=guard (the
checked build, csrc/guard.cu: redzones around every library allocation,
poisoned fresh memory, randomised sleeps at the persistent kernels' protocol
points).  The test asserts the two .npz files are bitwise identical and that
the checked build saw no redzone write.  Caller-owned outputs of the direct
C-ABI calls below carry their own redzones, checked here.

    python tests/guard_workload.py OUT.npz
"""

import ctypes
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1806_08422_b200 as nb  # noqa: E402
from paper_1806_08422_b200 import _native  # noqa: E402

MARGIN = 4096
out = {}
lib = _native.load()
dev = torch.device("cuda:0")


def guarded(shape, dtype):
    """A caller buffer with MARGIN bytes of 0x5A on each side."""
    nbytes = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
    raw = torch.full((nbytes + 2 * MARGIN,), 0x5A, dtype=torch.uint8, device=dev)
    view = raw[MARGIN:MARGIN + nbytes].view(dtype).view(shape)
    return raw, view


def margins_ok(raw):
    r = raw.cpu().numpy()
    return bool(np.all(r[:MARGIN] == 0x5A) and np.all(r[-MARGIN:] == 0x5A))


def c_anneal(name, prob, R, t_f, seed, r0=0, path=None, hist=False, noise=None, field=None):
    """Direct nmfa_anneal with redzoned caller buffers."""
    if path:
        prob.device_handle().set_path(path)
    if field:
        prob.device_handle().set_field_precision(field)
    n = prob.n
    temps = np.ascontiguousarray(nb.DEFAULT_SCHEDULE.temperatures(t_f))
    bufs = {"cfg": guarded((R, n), torch.int8), "e": guarded((R,), torch.float64),
            "s": guarded((R, n), torch.float32)}
    if hist:
        bufs["sh"] = guarded((R, t_f, n), torch.float32)
        bufs["eh"] = guarded((R, t_f), torch.float64)
    nz = None
    if noise is not None:
        nz = torch.as_tensor(noise, dtype=torch.float32, device=dev).contiguous()
    v = {k: b[1] for k, b in bufs.items()}
    _native.check(lib.nmfa_anneal(
        prob.device_handle().handle, R, t_f, _native.ptr(temps), 0.15, 0.15, seed, r0,
        _native.ptr(nz), None, _native.ptr(v["cfg"]), _native.ptr(v["e"]), _native.ptr(v["s"]),
        _native.ptr(v.get("sh")), _native.ptr(v.get("eh")),
        ctypes.c_void_p(torch.cuda.current_stream(dev).cuda_stream)))
    torch.cuda.synchronize()
    for k, (raw, view) in bufs.items():
        assert margins_ok(raw), f"{name}: caller buffer {k} written out of bounds"
        out[f"{name}_{k}"] = view.cpu().numpy()


T = int(os.environ.get("GUARD_TF", "40"))
c_anneal("small", nb.gen_sk(100, 0), 300, T, 3, hist=True)                    # 3 replica blocks, ragged
c_anneal("small_r0", nb.gen_sk(100, 0), 37, T, 3, r0=1000)
c_anneal("dense", nb.gen_sk(600, 1), 300, T, 5, path="dense")                  # ragged spin tiles, 2 blocks
c_anneal("dense_big", nb.gen_sk(2000, 7), 1024, T, 5, path="dense")            # the K2000 tiling
c_anneal("dense_hist", nb.gen_sk(300, 2), 64, T, 5, path="dense", hist=True)
rng = np.random.default_rng(4)
c_anneal("dense_inj", nb.gen_sk(520, 5), 33, T, 0, path="dense",
         noise=rng.standard_normal((33, T, 520)) * 0.15)
# HILO field: the second lo image (ping-pong) and two MMAs per k-slice / K step
c_anneal("dense_hilo", nb.gen_sk(600, 1), 300, T, 5, path="dense", field="hilo", hist=True)
c_anneal("dense_hilo_inj", nb.gen_sk(520, 5), 33, T, 0, path="dense", field="hilo",
         noise=rng.standard_normal((33, T, 520)) * 0.15)
c_anneal("small_hilo", nb.gen_sk(100, 0), 300, T, 3, field="hilo", hist=True)
c_anneal("ell", nb.moebius_ladder(1000), 100, T, 7)                             # degree-3 ELL kernel
c_anneal("ell_hist", nb.moebius_ladder(600), 37, T, 7, hist=True)
c_anneal("csr", nb.gen_dense_maxcut(1200, 0.01, 2), 70, T, 9, path="sparse")   # CSR kernel
c_anneal("csr_inj", nb.gen_dense_maxcut(700, 0.02, 3), 40, T, 0, path="sparse",
         noise=rng.standard_normal((40, T, 700)) * 0.15)
# energies, best-of, enumeration, grouped launch through the Python API
p = nb.gen_dense_maxcut(300, 0.2, 4)
cfg = np.where(np.random.default_rng(2).random((33, 300)) < 0.5, -1.0, 1.0)
out["energy"] = np.asarray(nb.energies(p, cfg))
g = nb.brute_force_ground(nb.gen_sk(16, 2))
out["ground"] = np.array([g.energy, g.degeneracy])
cfgm, enm, _ = nb.sample_many([nb.gen_sk(40, k) for k in range(3)], nb.NmfaParams(t_f=T, seed=3), 64)
out["many_cfg"], out["many_e"] = cfgm.cpu().numpy(), enm.cpu().numpy()
torch.cuda.synchronize()
bad = int(lib.nmfa_debug_guard_check())
out["guard_bad"] = np.array(bad)
if bad > 0:
    print("guard:", lib.nmfa_last_error().decode())
np.savez(sys.argv[1], **out)
print(f"ok: {len(out)} arrays, guard check = {bad}")
