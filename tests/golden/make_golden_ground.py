"""Golden fixtures for the exact enumerator, produced by the REFERENCE itself:
nmfa.brute_force_ground (metrics.py:53-67) on the numba backend
(gray_ground, _kernels_numba.py:83-114), cross-checked against the numpy
backend (_kernels_numpy.py:64-87).  Build container only (needs /root/reference).

    NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden_ground.py
"""
import os
import sys

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import nmfa  # noqa: E402
from nmfa import kernels  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def specs():
    rng = np.random.default_rng(20261018)
    out = {
        "pair": nmfa.IsingProblem(2, [(0, 1, 1.0)]),
        "single_h": nmfa.IsingProblem(1, [], h=[0.5]),
        "triangle": nmfa.IsingProblem(3, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 1.0)]),
        "moebius16": nmfa.moebius_ladder(16),
        "cubic24_s5": nmfa.gen_cubic_maxcut(24, 5),
        "sk20_s3": nmfa.gen_sk(20, 3),
        "sk26_s1": nmfa.gen_sk(26, 1),
        "dense18_p05": nmfa.gen_dense_maxcut(18, 0.5, 2),
    }
    # integer h with +-1 couplings (exact integer path)
    sk = nmfa.gen_sk(22, 4)
    h = rng.integers(-2, 3, size=22).astype(np.float64)
    out["sk22_inth"] = nmfa.IsingProblem(22, list(zip(sk.edges_i, sk.edges_j, sk.edge_weights)), h=h)
    # integer weights outside {-1,0,1} (float64 path, exact integers)
    e = [(i, j, float(rng.choice([-2, -1, 1, 2]))) for i in range(18) for j in range(i + 1, 18)
         if rng.random() < 0.4]
    out["w2_18"] = nmfa.IsingProblem(18, e)
    # real weights and fields
    e = [(i, j, float(rng.normal())) for i in range(16) for j in range(i + 1, 16) if rng.random() < 0.5]
    out["real16_h"] = nmfa.IsingProblem(16, e, h=rng.normal(size=16) * 0.3)
    return out


def main():
    print("reference backend:", kernels.BACKEND)
    fx = {}
    for name, p in specs().items():
        gt = nmfa.brute_force_ground(p)
        if p.n <= 22:  # the numpy backend materialises chunks of 2^20 configurations
            args = (p.csr_indptr, p.csr_indices, p.csr_weights, p.h)
            assert kernels.numpy_impl.gray_ground(*args) == (gt.energy, gt.degeneracy) or \
                abs(kernels.numpy_impl.gray_ground(*args)[0] - gt.energy) < 1e-9, name
        fx[name + "_n"] = np.array(p.n)
        fx[name + "_ei"] = p.edges_i.astype(np.int64)
        fx[name + "_ej"] = p.edges_j.astype(np.int64)
        fx[name + "_w"] = p.edge_weights.copy()
        fx[name + "_h"] = p.h.copy()
        fx[name + "_E"] = np.array(gt.energy)
        fx[name + "_deg"] = np.array(gt.degeneracy)
        print(f"  {name}: n={p.n} E={gt.energy} degeneracy={gt.degeneracy}")
    try:
        nmfa.brute_force_ground(nmfa.IsingProblem(nmfa.metrics.MAX_EXACT_N + 1))
    except ValueError as err:
        fx["too_big_msg"] = np.array(str(err))
    np.savez_compressed(os.path.join(OUT, "ground.npz"), **fx)
    print("wrote ground.npz")


if __name__ == "__main__":
    main()
