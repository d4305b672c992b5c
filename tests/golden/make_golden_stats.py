"""Large reference success-statistics samples, produced from the REFERENCE's
own streams and problem arithmetic.  Build container only (imports
/root/reference); outputs tests/golden/stats_large.npz, committed.

    OPENBLAS_NUM_THREADS=1 python tests/golden/make_golden_stats.py [--quick]

Why batched: the reference loop `nmfa_batch` (solver.py:262-280) costs ~0.17 s
per K2000 run, so thousands of reads are hours.  This script runs the SAME
algorithm replica-batched: run k draws `noise_stream(seed+k)
.standard_normal((t_f, n)) * sigma` exactly as `_run` does (solver.py:236-241),
then steps `s = a * -tanh(((h + J s) / norm) + z_t) / T_t) + (1 - a) * s`
(_kernels_numba.py:71-75) with S held as (n, R) so one dgemm serves all
replicas.  Final configs go through `sign_round` and energies through the
canonical edge list (problem.py:150-183).  The only difference from the
per-run loop is dgemm vs dgemv summation order (ulp-level), so the first
reads are checked for identical energies against `stats.npz`, which
`nmfa_batch` itself produced (make_golden.py).  The check result is stored.
"""

import argparse
import os
import sys
import time
from multiprocessing import Pool

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import nmfa  # noqa: E402
from nmfa.solver import DEFAULT_SCHEDULE, noise_stream  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
ALPHA = SIGMA = 0.15

_P = {}


def _instance(name):
    if name not in _P:
        _P[name] = {
            "sk100": lambda: nmfa.gen_sk(100, 0),
            "moebius100": lambda: nmfa.moebius_ladder(100),
            "g2000": lambda: nmfa.gen_dense_maxcut(2000, 0.01, 7),
            "sk2000": lambda: nmfa.gen_sk(2000, 7),
        }[name]()
    return _P[name]


def _chunk(args):
    """Energies of runs seed+r0 .. seed+r1-1 of instance `name` (t_f steps)."""
    name, r0, r1, t_f = args
    p = _instance(name)
    n = p.n
    J = p.dense_couplings() if hasattr(p, "dense_couplings") else None
    if J is None:
        J = np.zeros((n, n))
        J[p.edges_i, p.edges_j] = p.edge_weights
        J[p.edges_j, p.edges_i] = p.edge_weights
    temps = DEFAULT_SCHEDULE.temperatures(t_f)
    R = r1 - r0
    # (R, t_f, n) drawn per run in one call, as _run does (solver.py:238-241)
    noise = np.empty((t_f, n, R))
    for k in range(R):
        z = noise_stream(r0 + k).standard_normal((t_f, n))
        z *= SIGMA
        noise[:, :, k] = z
    if name == "g2000":  # 1% density: CSR product, same per-row sums up to order (ulp-level)
        import scipy.sparse as sp
        J = sp.csr_matrix(J)
    h = p.h[:, None]
    norm = p.normalizers_safe[:, None]
    S = np.zeros((n, R))
    for t in range(t_f):
        phi = (h + J @ S) / norm + noise[t]
        S = ALPHA * (-np.tanh(phi / temps[t])) + (1.0 - ALPHA) * S
    C = np.where(S < 0.0, -1.0, 1.0).T                     # sign_round (problem.py:181-183)
    E = (C[:, p.edges_i] * C[:, p.edges_j]) @ p.edge_weights + C @ p.h
    return r0, E


def sample(name, R, t_f, workers, chunk):
    jobs = [(name, a, min(a + chunk, R), t_f) for a in range(0, R, chunk)]
    out = np.empty(R)
    with Pool(workers) as pool:
        for r0, E in pool.imap_unordered(_chunk, jobs):
            out[r0:r0 + E.size] = E
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--only", default="")
    ap.add_argument("--extend", type=int, default=0,
                    help="grow the --only samples to this many reads (appends seeds past the stored ones)")
    a = ap.parse_args()
    workers = os.cpu_count() or 8
    ref = np.load(os.path.join(OUT, "stats.npz"))
    plan = [  # (name, reads, chunk, t_f)
        ("sk100", 65536, 512, 1000),
        ("moebius100", 32768, 512, 1000),
        ("g2000", 4096, 16, 1000),
        ("sk2000", 4096, 16, 1000),
    ]
    if a.quick:
        plan = [(n, min(R, 256), c, t) for n, R, c, t in plan]
    if a.only:
        plan = [x for x in plan if x[0] in a.only.split(",")]
    path = os.path.join(OUT, "stats_large.npz")
    st = dict(np.load(path)) if os.path.exists(path) else {}
    for name, R, chunk, t_f in plan:
        t0 = time.time()
        if a.extend and name + "_E" in st:
            old = st[name + "_E"].astype(np.float64)
            jobs = [(name, r, min(r + chunk, a.extend), t_f) for r in range(old.size, a.extend, chunk)]
            E = np.concatenate([old, np.empty(a.extend - old.size)])
            with Pool(workers) as pool:
                for r0, e in pool.imap_unordered(_chunk, jobs):
                    E[r0:r0 + e.size] = e
        else:
            E = sample(name, R, t_f, workers, chunk)
        wall = time.time() - t0
        base = ref[name + "_E"]
        m = min(base.size, E.size)
        same = int(np.count_nonzero(E[:m] == base[:m]))
        print(f"{name}: R={R} wall={wall:.0f}s min={E.min()} mean={E.mean():.2f}; "
              f"identical to nmfa_batch on {same}/{m} shared seeds", flush=True)
        st[name + "_E"] = E.astype(np.int32) if np.all(E == np.round(E)) else E
        st[name + "_t_f"] = np.array(t_f)
        st[name + "_same_as_nmfa_batch"] = np.array([same, m])
    np.savez_compressed(path, **st)
    print("wrote", path, sorted(st))


if __name__ == "__main__":
    main()
