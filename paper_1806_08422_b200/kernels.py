"""B200 backend behind the reference's own operator API (kernels.py:13-32).

The reference selects its hot kernels at import time and calls them through
module attributes -- ``kernels.anneal_dense`` / ``kernels.anneal_sparse``
from run_with_noise (solver.py:206-216) and ``kernels.gray_ground`` from
brute_force_ground (metrics.py:64).  This module provides the same three
functions with the same contract (_kernels_numba.py:3-13), so installing it is
three assignments (``install(nmfa.kernels)``) and every reference entry point
-- nmfa_run, nmfa_batch, run_with_noise, brute_force_ground, the CLI -- then
runs on the GPU:

* ``anneal_dense(J, h, norm, s, temps, noise, alpha, record)`` and
  ``anneal_sparse(indptr, indices, weights, h, norm, s, temps, noise, alpha,
  record)`` advance ``s`` in place through one noisy mean-field sweep per
  temperature with the caller's pre-scaled noise and return
  ``(s, s_hist, e_hist)`` (histories empty unless ``record``).
* ``gray_ground(indptr, indices, weights, h)`` returns ``(emin, count)``.

The device problem for a coupling matrix is built once and cached on the
identity of the caller's arrays (a batch passes the same arrays for every
run), so repeated calls only move s, noise and the results.  ``norm`` must be
the problem's own normalizers (the reference always passes
``problem.normalizers_safe``); it is checked.  The tensor-core paths run the
HILO field here (the full state as the GEMM operand, include/nmfa_b200.h
NMFA_FIELD_HILO): the contract is the reference's float64 kernel.
"""

from __future__ import annotations

import threading
from collections import OrderedDict

import numpy as np

from .problem import IsingProblem

BACKEND = "b200"      # kernels.py:13-32: the reference reports its backend here
FORCE_NUMPY = False   # no CPU backend exists in this package

_CACHE_SIZE = 8
_cache: "OrderedDict[tuple, tuple]" = OrderedDict()
_lock = threading.Lock()


def _key(*arrays):
    return tuple((id(a), a.__array_interface__["data"][0], a.shape, a.strides) for a in arrays)


def _cached(key, arrays, build):
    with _lock:
        hit = _cache.get(key)
        if hit is not None:
            _cache.move_to_end(key)
            return hit[0]
    prob = build()
    with _lock:
        _cache[key] = (prob, arrays)  # keep the arrays alive so their ids stay unique
        while len(_cache) > _CACHE_SIZE:
            _cache.popitem(last=False)
    return prob


def _problem_dense(J, h):
    J = np.asarray(J, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)

    def build():
        i, j = np.nonzero(np.triu(J, 1))
        return IsingProblem.from_arrays(J.shape[0], i, j, J[i, j], h)

    return _cached(_key(J, h), (J, h), build)


def _problem_csr(indptr, indices, weights, h):
    indptr = np.asarray(indptr)
    indices = np.asarray(indices)
    weights = np.asarray(weights, dtype=np.float64)
    h = np.asarray(h, dtype=np.float64)

    def build():
        n = indptr.shape[0] - 1
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(indptr))
        keep = indices > rows
        return IsingProblem.from_arrays(n, rows[keep], indices[keep].astype(np.int64),
                                        weights[keep], h)

    return _cached(_key(indptr, indices, weights, h), (indptr, indices, weights, h), build)


def _anneal(problem, norm, s, temps, noise, alpha, record):
    from .solver import _replay_field, run_with_noise

    if not np.allclose(np.asarray(norm, dtype=np.float64), problem.normalizers_safe, rtol=1e-12,
                       atol=0.0):
        raise ValueError("norm must be the problem's normalizers_safe (problem.py:90-95)")
    s0 = np.asarray(s, dtype=np.float64)
    s_new, traj = run_with_noise(problem, np.asarray(temps, dtype=np.float64),
                                 np.asarray(noise, dtype=np.float64), float(alpha), s0=s0,
                                 record_trajectory=bool(record),
                                 field=_replay_field(problem, 0, None))
    if isinstance(s, np.ndarray) and s.dtype == np.float64 and s.flags.writeable:
        s[...] = s_new  # the contract advances s in place (_kernels_numba.py:3-13)
        s_new = s
    n = s0.shape[0]
    if record:
        return s_new, np.asarray(traj.spins, dtype=np.float64), np.asarray(traj.energies)
    return s_new, np.empty((0, n)), np.empty(0)


def anneal_dense(J, h, norm, s, temps, noise, alpha, record):
    """_kernels_numba.py:64-80 on the GPU (dense J)."""
    return _anneal(_problem_dense(J, h), norm, s, temps, noise, alpha, record)


def anneal_sparse(indptr, indices, weights, h, norm, s, temps, noise, alpha, record):
    """_kernels_numba.py:39-61 on the GPU (symmetric CSR)."""
    return _anneal(_problem_csr(indptr, indices, weights, h), norm, s, temps, noise, alpha, record)


def gray_ground(indptr, indices, weights, h):
    """_kernels_numba.py:83-114 on the GPU: (emin, count) over all 2^n configurations."""
    from .metrics import brute_force_ground

    p = _problem_csr(indptr, indices, weights, h)
    gt = brute_force_ground(p, max_n=40)
    return gt.energy, gt.degeneracy


def install(kernels_module):
    """Point a reference ``nmfa.kernels`` module at this backend (kernels.py:30-32)."""
    kernels_module.anneal_dense = anneal_dense
    kernels_module.anneal_sparse = anneal_sparse
    kernels_module.gray_ground = gray_ground
    kernels_module.BACKEND = "b200"
    return kernels_module
