"""Where does a seeded success-probability difference come from?  (CPU only)

Runs the replica-batched float64 NMFA loop on one instance with the noise and
arithmetic swapped one factor at a time, and prints p(E <= E_ref) with its
Wilson interval for each variant:

  ref64     float64, the reference's numpy streams          (= nmfa_batch)
  dev64     float64, the device's Philox4x32 + Box-Muller noise (exact math)
  dev_f16   device noise, fp32 state, fp16-rounded GEMM operand (the GPU's
            small-kernel arithmetic up to MUFU approximations)

    python tools/stat_bisect.py --inst sk100 --reads 65536 --variants dev64,dev_f16
"""

import argparse
import os
import sys
import time
from multiprocessing import Pool

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))

import numpy as np  # noqa: E402

import nmfa_oracle as O  # noqa: E402

ALPHA = SIGMA = 0.15
TAG = 0x4E4D4641
M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)


def philox_keys(c0, c1, c2, c3, k0, k1):
    """Philox4x32-10 with per-element keys (all uint32 arrays, broadcast)."""
    c0, c1, c2, c3, k0, k1 = np.broadcast_arrays(*(np.asarray(x, dtype=np.uint32)
                                                   for x in (c0, c1, c2, c3, k0, k1)))
    c0, c1, c2, c3, k0, k1 = (x.copy() for x in (c0, c1, c2, c3, k0, k1))
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = c0.astype(np.uint64) * M0
            p1 = c2.astype(np.uint64) * M1
            n0 = (p1 >> np.uint64(32)).astype(np.uint32) ^ c1 ^ k0
            n2 = (p0 >> np.uint64(32)).astype(np.uint32) ^ c3 ^ k1
            c0, c1, c2, c3 = n0, p1.astype(np.uint32), n2, p0.astype(np.uint32)
            k0 = k0 + W0
            k1 = k1 + W1
    return c0, c1, c2, c3


def device_noise_step(keys, t, n, sigma, scheme="bm12"):
    """(n, R) noise of step t for 64-bit keys (R,): the in-kernel spec
    (oracle.device_normals), vectorised over replicas."""
    q = np.arange((n + 7) // 8, dtype=np.uint32)[:, None]
    k0 = (keys & 0xFFFFFFFF).astype(np.uint32)[None, :]
    k1 = (keys >> 32).astype(np.uint32)[None, :]
    words = philox_keys(q, np.uint32(t), np.uint32(TAG), np.uint32(0), k0, k1)
    z = np.empty((q.size, 8, keys.size))
    for w in range(4):
        x = words[w].astype(np.int64)
        u1 = ((x >> 12) + 0.5) * 2.0 ** -20
        rad = sigma * np.sqrt(-2.0 * np.log(u1))
        ang = (x & 0xFFF) * (2.0 * np.pi / 4096.0)
        z[:, 2 * w] = rad * np.cos(ang)
        z[:, 2 * w + 1] = rad * np.sin(ang)
    return z.reshape(-1, keys.size)[:n]


def instance(name):
    if name == "sk100":
        return O.problem_from_edges(100, *O.gen_sk_edges(100, 0)), -730.0
    if name == "moebius100":
        return O.problem_from_edges(100, *O.moebius_edges(100)), -146.0
    raise ValueError(name)


def chunk(args):
    name, variant, r0, r1, t_f = args
    p, _ = instance(name)
    temps = O.temperatures(t_f)
    R = r1 - r0
    keys = np.arange(r0, r1, dtype=np.uint64)
    J, h, nrm = p.dense, p.h[:, None], p.normalizers_safe[:, None]
    if variant == "ref64":
        gens = [O.noise_stream(r) for r in range(r0, r1)]
    S = np.zeros((p.n, R))
    for t in range(t_f):
        if variant == "ref64":
            Z = np.stack([g.standard_normal(p.n) for g in gens], axis=1) * SIGMA
        else:
            Z = device_noise_step(keys, t, p.n, SIGMA)
        if variant == "dev_f16":
            A = S.astype(np.float16).astype(np.float32)
            mv = (J.astype(np.float32) @ A).astype(np.float32)
            phi = mv * (1.0 / nrm).astype(np.float32) + (h / nrm).astype(np.float32) + Z.astype(np.float32)
            sh = -np.tanh(phi * np.float32(1.0 / temps[t]))
            S = (np.float32(ALPHA) * sh + np.float32(1.0 - ALPHA) * S.astype(np.float32)).astype(np.float32)
        else:
            phi = (h + J @ S) / nrm + Z
            S = ALPHA * (-np.tanh(phi / temps[t])) + (1.0 - ALPHA) * S
    C = np.where(S < 0.0, -1.0, 1.0).T
    return r0, O.energies(p, C)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--inst", default="sk100")
    ap.add_argument("--reads", type=int, default=65536)
    ap.add_argument("--t_f", type=int, default=1000)
    ap.add_argument("--chunk", type=int, default=1024)
    ap.add_argument("--variants", default="dev64,dev_f16")
    a = ap.parse_args()
    _, eref = instance(a.inst)
    for v in a.variants.split(","):
        t0 = time.time()
        jobs = [(a.inst, v, s, min(s + a.chunk, a.reads), a.t_f) for s in range(0, a.reads, a.chunk)]
        E = np.empty(a.reads)
        with Pool(os.cpu_count()) as pool:
            for r0, e in pool.imap_unordered(chunk, jobs):
                E[r0:r0 + e.size] = e
        k = int(np.count_nonzero(E <= eref + 1e-9))
        lo, hi = O.wilson_interval(k, a.reads)
        print(f"{a.inst} {v}: p = {k}/{a.reads} = {k / a.reads:.4f}  95% [{lo:.4f}, {hi:.4f}]  "
              f"mean E {E.mean():.3f}  ({time.time() - t0:.0f} s)", flush=True)


if __name__ == "__main__":
    main()
