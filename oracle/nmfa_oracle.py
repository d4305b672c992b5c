"""CPU oracle for the NMFA hot path -- TEST INFRASTRUCTURE ONLY.

This module is a float64 numpy restatement of the reference package `nmfa`
(King et al., arXiv 1806.08422, Algorithm 1).  It exists to check the CUDA
path, never to replace it: only `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` may import it.  The
product package `paper_1806_08422_b200` never imports anything from here and
fails loudly when its CUDA library is missing.

Parity pinning: every function below is checked in `tests/test_oracle.py`
against golden vectors produced by running the reference itself in the
build container (`tests/golden/make_golden.py`, committed with its outputs).

Third-party arithmetic restated (the reference leaves versions unpinned,
pyproject.toml:10-14): numpy's Philox4x64-10 bit generator + ziggurat
`standard_normal` (solver.py:182-185, 238-241) -- used here through numpy
itself, since the stream identity *is* numpy's; BLAS dgemv/dgemm via `@`.
"""

from __future__ import annotations

import math
from concurrent.futures import ThreadPoolExecutor

import numpy as np

MASK64 = (1 << 64) - 1
RUN_STREAM_TAG = 2          # solver.py:33
GEN_STREAM_TAG = 1          # generators.py:13
DEFAULT_BREAKPOINTS = ((0.0, 2.0), (0.25, 0.8), (0.75, 0.2), (1.0, 0.02))  # solver.py:133
DENSE_THRESHOLD = 0.5       # problem.py:13
TIE_TOL = 1e-9              # metrics.py:21


# --------------------------------------------------------------------------
# schedule (solver.py:70-84)
# --------------------------------------------------------------------------
def temperatures(t_f, breakpoints=DEFAULT_BREAKPOINTS):
    """Piecewise-geometric T for iterations 1..t_f (solver.py:70-84): iteration
    t sits at f = (t-1)/(t_f-1); inside segment [f_k, f_k+1) the temperature
    is T_k (T_k+1 / T_k)^((f - f_k)/(f_k+1 - f_k)); f at or past the last
    breakpoint takes the last temperature exactly."""
    knots = [(float(f), float(T)) for f, T in breakpoints]
    t_f = int(t_f)
    f = np.arange(t_f) / (t_f - 1) if t_f > 1 else np.zeros(1)
    out = np.empty_like(f)
    for (f0, T0), (f1, T1) in zip(knots[:-1], knots[1:]):
        inside = (f >= f0) & (f < f1)
        out[inside] = T0 * (T1 / T0) ** ((f[inside] - f0) / (f1 - f0))
    out[f >= knots[-1][0]] = knots[-1][1]
    return out


# --------------------------------------------------------------------------
# randomness (solver.py:182-185, 236-241)
# --------------------------------------------------------------------------
def noise_stream(seed):
    """numpy Philox4x64-10 keyed (2 << 64) | seed (solver.py:182-185)."""
    key = (RUN_STREAM_TAG << 64) | (int(seed) & MASK64)
    return np.random.Generator(np.random.Philox(key=key))


def run_noise(seed, t_f, n, sigma):
    """Pre-scaled additive noise of one run, shape (t_f, n) (solver.py:238-241)."""
    z = noise_stream(seed).standard_normal((int(t_f), int(n)))
    if sigma != 1.0:
        z *= sigma
    return z


# --------------------------------------------------------------------------
# problem arithmetic (problem.py:25-116, 150-183)
# --------------------------------------------------------------------------
class Problem:
    """Canonical edge list + symmetric CSR + normalizers (problem.py:25-116)."""

    def __init__(self, n, couplers=(), h=None):
        self.n = n = int(n)
        self.h = np.zeros(n) if h is None else np.asarray(h, dtype=np.float64).copy()
        arr = np.asarray(couplers, dtype=np.float64).reshape(-1, 3)
        ii = arr[:, 0].astype(np.int64)
        jj = arr[:, 1].astype(np.int64)
        ww = arr[:, 2].copy()
        lo, hi = np.minimum(ii, jj), np.maximum(ii, jj)
        order = np.lexsort((hi, lo))                       # problem.py:63-66
        self.edges_i, self.edges_j, self.edge_weights = lo[order], hi[order], ww[order]
        rows = np.concatenate([self.edges_i, self.edges_j])  # problem.py:78-88
        cols = np.concatenate([self.edges_j, self.edges_i])
        vals = np.concatenate([self.edge_weights, self.edge_weights])
        perm = np.lexsort((cols, rows))
        self.csr_indptr = np.zeros(n + 1, dtype=np.int64)
        np.cumsum(np.bincount(rows, minlength=n), out=self.csr_indptr[1:])
        self.csr_indices = cols[perm]
        self.csr_weights = vals[perm]
        norm = np.sqrt(self.h ** 2 + np.bincount(rows, weights=vals ** 2, minlength=n))
        self.normalizers_safe = np.where(norm == 0.0, 1.0, norm)   # problem.py:90-95
        pairs = n * (n - 1) // 2
        self.density = 0.0 if pairs == 0 else self.edges_i.size / pairs
        self.is_dense = self.density > DENSE_THRESHOLD              # problem.py:97-99
        J = np.zeros((n, n))
        J[self.edges_i, self.edges_j] = self.edge_weights
        J[self.edges_j, self.edges_i] = self.edge_weights
        self.dense = J


def sign_round(s):
    """s < 0 -> -1, else +1 (0 and -0 -> +1) (problem.py:181-183)."""
    return np.where(np.asarray(s, dtype=np.float64) < 0.0, -1.0, 1.0)


def energy(p, config):
    """sum_(i<j) w c_i c_j + h.c over the canonical edge list (problem.py:150-154)."""
    c = np.asarray(config, dtype=np.float64)
    pair = float(np.dot(p.edge_weights, c[p.edges_i] * c[p.edges_j]))
    return pair + float(np.dot(p.h, c))


def energies(p, configs):
    """Row-wise `energy` for a (R, n) batch of +-1 configurations."""
    C = np.asarray(configs, dtype=np.float64)
    return (C[:, p.edges_i] * C[:, p.edges_j]) @ p.edge_weights + C @ p.h


def cut_value(p, config):
    """sum w (1 - c_i c_j) / 2 (problem.py:157-163)."""
    c = np.asarray(config, dtype=np.float64)
    return float(np.dot(p.edge_weights, 1.0 - c[p.edges_i] * c[p.edges_j])) * 0.5


# --------------------------------------------------------------------------
# the anneal loop (_kernels_numpy.py:17-53 / _kernels_numba.py:39-80)
# --------------------------------------------------------------------------
def anneal(p, s, temps, noise, alpha, record=False):
    """One run: s <- a*(-tanh(((h + J s)/norm + noise_t)/T_t)) + (1-a)*s per step.

    Dense problems use the BLAS matvec (_kernels_numba.py:72-75); sparse ones
    the CSR row sum in column order (_kernels_numba.py:48-56).  Returns
    (s, s_hist, e_hist) like the reference kernels.
    """
    s = np.array(s, dtype=np.float64)
    t_f = len(temps)
    s_hist = np.empty((t_f if record else 0, p.n))
    e_hist = np.empty(t_f if record else 0)
    if p.is_dense:
        mv_of = lambda v: np.dot(p.dense, v)
    else:
        import scipy.sparse as sp
        csr = sp.csr_matrix((p.csr_weights, p.csr_indices, p.csr_indptr), shape=(p.n, p.n))
        mv_of = lambda v: csr @ v
    for t in range(t_f):
        phi = (p.h + mv_of(s)) / p.normalizers_safe + noise[t]
        s = alpha * (-np.tanh(phi / temps[t])) + (1.0 - alpha) * s
        if record:
            s_hist[t] = s
            e_hist[t] = energy(p, sign_round(s))
    return s, s_hist, e_hist


# Compiled restatement of the same loop for the CPU-baseline timing: the
# reference's default backend is numba (kernels.py:16-27), so the port times
# a jitted loop too.  dgemv via np.dot and libm tanh, as _kernels_numba.py:71-75
# and 48-56 do; results agree with `anneal` to ~1e-12 (tests/test_oracle.py).
try:
    from numba import njit

    @njit(nogil=True, cache=False)
    def _loop_dense(J, h, norm, s, temps, noise, alpha):
        for t in range(temps.shape[0]):
            phi = (h + np.dot(J, s)) / norm + noise[t]
            s = alpha * (-np.tanh(phi / temps[t])) + (1.0 - alpha) * s
        return s

    @njit(nogil=True, cache=False)
    def _loop_sparse(row_start, col, val, h, norm, s, temps, noise, alpha):
        # synchronous update: all fields from the incoming state, then all spins
        # (_kernels_numba.py:48-56); arithmetic order kept for bit-exact energies
        n = s.shape[0]
        field = np.empty(n)
        for step in range(temps.shape[0]):
            T = temps[step]
            for a in range(n):
                total = 0.0
                for q in range(row_start[a], row_start[a + 1]):
                    total += val[q] * s[col[q]]
                field[a] = (h[a] + total) / norm[a] + noise[step, a]
            for a in range(n):
                s[a] = alpha * (-np.tanh(field[a] / T)) + (1.0 - alpha) * s[a]
        return s

    HAVE_JIT = True
except ImportError:  # pragma: no cover
    HAVE_JIT = False


def anneal_fast(p, s, temps, noise, alpha):
    """Final state of `anneal` through the jitted loop (falls back to numpy)."""
    if not HAVE_JIT:
        return anneal(p, s, temps, noise, alpha)[0]
    s = np.array(s, dtype=np.float64)
    temps = np.asarray(temps, dtype=np.float64)
    if p.is_dense:
        return _loop_dense(p.dense, p.h, p.normalizers_safe, s, temps, noise, float(alpha))
    return _loop_sparse(p.csr_indptr, p.csr_indices, p.csr_weights, p.h, p.normalizers_safe, s,
                        temps, noise, float(alpha))


def run(p, seed, t_f=1000, alpha=0.15, sigma=0.15, temps=None, jit=True):
    """One seeded run (solver.py:236-253): returns (config, energy)."""
    temps = temperatures(t_f) if temps is None else temps
    noise = run_noise(seed, t_f, p.n, sigma)
    if jit:
        s = anneal_fast(p, np.zeros(p.n), temps, noise, alpha)
    else:
        s, _, _ = anneal(p, np.zeros(p.n), temps, noise, alpha)
    cfg = sign_round(s)
    return cfg, energy(p, cfg)


def batch(p, seed, n_runs, t_f=1000, alpha=0.15, sigma=0.15, threads=1, jit=True):
    """n_runs independent runs, run k seeded seed+k (solver.py:262-280)."""
    temps = temperatures(t_f)
    seeds = [(int(seed) + k) & MASK64 for k in range(int(n_runs))]
    one = lambda sd: run(p, sd, t_f, alpha, sigma, temps, jit)
    if threads <= 1:
        out = [one(sd) for sd in seeds]
    else:
        with ThreadPoolExecutor(max_workers=int(threads)) as pool:
            out = list(pool.map(one, seeds))
    return np.array([c for c, _ in out]), np.array([e for _, e in out])


def batched_anneal(p, seeds, t_f=1000, alpha=0.15, sigma=0.15, temps=None, noise=None):
    """Replica-batched float64 restatement: S is (n, R), one GEMM per step.

    Replica r draws its per-step noise from noise_stream(seeds[r]) in the same
    order as the reference's (t_f, n) matrix (test_solver.py:181-190 pins
    that per-step draws equal the one-shot draw).  When `noise` (R, t_f, n) is
    given it is used instead.  Returns final analog S as (R, n).
    """
    temps = temperatures(t_f) if temps is None else np.asarray(temps, dtype=np.float64)
    R = len(seeds) if noise is None else noise.shape[0]
    S = np.zeros((p.n, R))
    gens = None if noise is not None else [noise_stream(sd) for sd in seeds]
    J = p.dense
    hn = p.h[:, None]
    nrm = p.normalizers_safe[:, None]
    for t in range(len(temps)):
        if noise is None:
            Z = np.stack([g.standard_normal(p.n) for g in gens], axis=1)
            if sigma != 1.0:
                Z *= sigma
        else:
            Z = noise[:, t, :].T
        phi = (hn + J @ S) / nrm + Z
        S = alpha * (-np.tanh(phi / temps[t])) + (1.0 - alpha) * S
    return S.T.copy()


# --------------------------------------------------------------------------
# benchmark statistics (metrics.py:70-94)
# --------------------------------------------------------------------------
def success_probability(final_energies, e_ref):
    e = np.asarray(final_energies, dtype=np.float64)
    return float(np.count_nonzero(e <= e_ref + TIE_TOL)) / e.size


def time_to_solution(p, tau, confidence=0.99):
    if p == 0.0:
        return math.inf
    if p >= confidence:
        return tau
    return tau * math.log(1.0 - confidence) / math.log(1.0 - p)


def wilson_interval(k, n, z=1.96):
    """Wilson score interval for a binomial proportion."""
    if n == 0:
        return (0.0, 1.0)
    ph = k / n
    den = 1.0 + z * z / n
    c = (ph + z * z / (2 * n)) / den
    half = z * math.sqrt(ph * (1 - ph) / n + z * z / (4 * n * n)) / den
    return (c - half, c + half)


# --------------------------------------------------------------------------
# instance generators (generators.py:16-86) -- used to pin the package's
# own generators against golden fixtures
# --------------------------------------------------------------------------
def _gen_rng(seed):
    return np.random.Generator(np.random.Philox(key=(GEN_STREAM_TAG << 64) | (int(seed) & MASK64)))


def gen_sk_edges(n, seed):
    ii, jj = np.triu_indices(int(n), 1)
    w = np.where(_gen_rng(seed).random(ii.size) < 0.5, 1.0, -1.0)
    return ii.astype(np.int64), jj.astype(np.int64), w


def moebius_edges(n):
    """Ring 0-1-...-(n-1)-0 plus rungs (k, k + n/2), unit weights (generators.py:76-86)."""
    v = np.arange(n, dtype=np.int64)
    ring = np.stack([v, np.roll(v, -1)])
    rungs = np.stack([v[: n // 2], v[: n // 2] + n // 2])
    ends = np.concatenate([ring, rungs], axis=1)
    return ends.min(axis=0), ends.max(axis=0), np.ones(ends.shape[1])


def problem_from_edges(n, ii, jj, w, h=None):
    return Problem(n, np.column_stack([ii, jj, w]), h)


# --------------------------------------------------------------------------
# Twin of the on-device SK generator (nmfa_problem_create_sk_device,
# include/nmfa_b200.h) -- test infrastructure for config 5 (SK N = 65,536),
# which the reference itself cannot build (problem.py:41-104).
# --------------------------------------------------------------------------
def philox4x32_10(c0, c1, c2, c3, k0, k1):
    """Vectorised Philox4x32-10 (Salmon et al. 2011) on uint32 numpy arrays."""
    M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
    W0, W1 = np.uint32(0x9E3779B9), np.uint32(0xBB67AE85)
    c0, c1, c2, c3 = (np.asarray(x, dtype=np.uint32).copy() for x in (c0, c1, c2, c3))
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    with np.errstate(over="ignore"):
        for _ in range(10):
            p0 = c0.astype(np.uint64) * M0
            p1 = c2.astype(np.uint64) * M1
            n0 = (p1 >> np.uint64(32)).astype(np.uint32) ^ c1 ^ k0
            n2 = (p0 >> np.uint64(32)).astype(np.uint32) ^ c3 ^ k1
            c0, c1, c2, c3 = n0, p1.astype(np.uint32), n2, p0.astype(np.uint32)
            k0 = np.uint32((int(k0) + int(W0)) & 0xFFFFFFFF)
            k1 = np.uint32((int(k1) + int(W1)) & 0xFFFFFFFF)
    return c0, c1, c2, c3


def sk_device_couplings(n, seed):
    """Dense +-1 J of the device-generated SK instance (zero diagonal)."""
    i, j = np.triu_indices(int(n), 1)
    a = i.astype(np.uint32)
    b = j.astype(np.uint32)
    words = philox4x32_10(b >> np.uint32(7), a, np.uint32(0x534B4A31), np.uint32(0),
                          int(seed) & 0xFFFFFFFF, (int(seed) >> 32) & 0xFFFFFFFF)
    sel = (b & np.uint32(127)) >> np.uint32(5)
    w = np.choose(sel.astype(np.int64), words)
    bit = (w >> (b & np.uint32(31))) & np.uint32(1)
    J = np.zeros((n, n))
    J[i, j] = np.where(bit == 1, 1.0, -1.0)
    return J + J.T


# --------------------------------------------------------------------------
# Exact ground state (brute_force_ground, metrics.py:53-67).  Restates the
# reference's chunked numpy enumerator (_kernels_numpy.py:64-87): energies of
# every configuration k (bit i of k set -> s_i = -1, as 1 - 2*bits), minimum
# and the count within TIE_TOL.  Test infrastructure; the product enumerates
# on the GPU (csrc/ground.cu).
# --------------------------------------------------------------------------
TIE_TOL = 1e-9


def gray_ground(problem, chunk_bits=16):
    """Minimum energy over all 2^n configurations and its multiplicity within
    TIE_TOL (the semantics of _kernels_numpy.py:64-87), enumerated chunk by
    chunk in configuration-index order: configuration k sets s_i = -1 where bit
    i of k is set, and its energy is summed over the canonical edge list."""
    n = problem.n
    ei, ej = np.asarray(problem.edges_i), np.asarray(problem.edges_j)
    w = np.asarray(problem.edge_weights, dtype=np.float64)
    h = np.asarray(problem.h, dtype=np.float64)
    bit = np.uint64(1) << np.arange(n, dtype=np.uint64)
    best, ties = np.inf, 0
    step = 1 << min(n, chunk_bits)
    for first in range(0, 1 << n, step):
        k = np.arange(first, min(first + step, 1 << n), dtype=np.uint64)
        spins = np.where((k[:, None] & bit[None, :]) != 0, -1.0, 1.0)
        e = (spins[:, ei] * spins[:, ej]) @ w + spins @ h
        low = float(e.min())
        if low < best - TIE_TOL:  # a new minimum resets the count
            best = low
            ties = int(np.count_nonzero(e <= best + TIE_TOL))
        else:
            ties += int(np.count_nonzero(e <= best + TIE_TOL))
    return best, ties


def gray_ground_fast(problem):
    """CPU baseline for the enumerator: the reference's sequential Gray-code walk
    (_kernels_numba.py:83-114) jitted with numba -- one spin flip per step, the
    flipped spin's field summed over its CSR row, ties within 1e-9."""
    from numba import njit

    global _gray_jit
    if "_gray_jit" not in globals():
        @njit(cache=False, nogil=True)
        def _walk(ptr, col, val, field):
            n = field.shape[0]
            spin = -np.ones(n)
            # E(all -1) = sum_{i<j} w + sum_i -h_i
            energy = 0.0
            for a in range(n):
                for q in range(ptr[a], ptr[a + 1]):
                    if col[q] > a:
                        energy += val[q]
                energy -= field[a]
            best, ties = energy, 1
            for code in range(1, np.int64(1) << n):
                flip = 0  # index of the lowest set bit of `code`
                c = code
                while (c & 1) == 0:
                    c >>= 1
                    flip += 1
                spin[flip] = -spin[flip]
                local = field[flip]
                for q in range(ptr[flip], ptr[flip + 1]):
                    local += val[q] * spin[col[q]]
                energy += 2.0 * spin[flip] * local
                if energy < best - 1e-9:
                    best, ties = energy, 1
                elif energy <= best + 1e-9:
                    ties += 1
            return best, ties
        _gray_jit = _walk
    return _gray_jit(problem.csr_indptr, problem.csr_indices, problem.csr_weights,
                     np.asarray(problem.h, dtype=np.float64))


def device_normals(seed, replicas, t, n, sigma):
    """The in-kernel noise spec (common.cuh normal8; DESIGN §2 "Noise stream"):
    N(0, sigma^2) for global replicas `replicas`, 0-based step t, spins 0..n-1.
    key = (lo32, hi32)(seed + r); counter = (i >> 3, t, 0x4E4D4641, 0); word
    w = (i & 7) >> 1 is one Box-Muller pair: u1 = ((w >> 12) + 1/2) 2^-20,
    angle = 2 pi (w & 0xFFF) / 4096, spin 8q + 2w -> r cos, 8q + 2w + 1 -> r sin.
    float64 here; the device uses MUFU approximations (agree to ~1e-6)."""
    replicas = np.asarray(replicas, dtype=np.int64)
    q = np.arange((n + 7) // 8, dtype=np.uint32)
    out = np.zeros((replicas.size, n))
    for a, r in enumerate(replicas):
        key = (int(seed) + int(r)) & 0xFFFFFFFFFFFFFFFF
        words = philox4x32_10(q, np.uint32(t), np.uint32(0x4E4D4641), np.uint32(0),
                              key & 0xFFFFFFFF, key >> 32)
        z = np.zeros((q.size, 8))
        for w in range(4):
            x = words[w].astype(np.int64)
            u1 = ((x >> 12) + 0.5) * 2.0 ** -20
            rad = sigma * np.sqrt(-2.0 * np.log(u1))
            ang = (x & 0xFFF) * (2.0 * np.pi / 4096.0)
            z[:, 2 * w] = rad * np.cos(ang)
            z[:, 2 * w + 1] = rad * np.sin(ang)
        out[a] = z.reshape(-1)[:n]
    return out
