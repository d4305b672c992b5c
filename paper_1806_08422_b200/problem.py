"""Ising problem: the host-side mirror of the reference `nmfa.problem` API.

`IsingProblem(n, couplers, h)` validates and canonicalises exactly like the
reference (problem.py:25-116) and owns a device-resident handle per CUDA
device (`nmfa_problem_create`, include/nmfa_b200.h).  The arithmetic helpers
`energy` / `cut_value` evaluate on the GPU through the C-ABI (bit-exact for
integer weights); `mean_field` / `normalizers` / `sign_round` are the same
small host-side utilities the reference exposes.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native

DENSE_THRESHOLD = 0.5  # problem.py:13


def _spin_count(n):
    n = int(n)
    if n < 1:
        raise ValueError(f"spin count must be positive, got {n}")
    return n


def _fields(n, h):
    if h is None:
        return np.zeros(n)
    out = np.array(h, dtype=np.float64)  # private copy
    if out.shape != (n,):
        raise ValueError(f"h must have length {n}, got shape {out.shape}")
    if not np.isfinite(out).all():
        raise ValueError("h contains non-finite entries")
    return out


class IsingProblem:
    """Immutable coupling structure: n spins, fields h, couplers (i, j, w).

    Validation order and messages are the reference's (problem.py:25-76):
    indices in range, no self-couplings, finite nonzero weights, no duplicate
    unordered pair.  Couplers are stored canonically, as i < j in lexicographic order.
    """

    def __init__(self, n, couplers=(), h=None):
        n = _spin_count(n)
        h = _fields(n, h)
        table = np.asarray(couplers, dtype=np.float64)
        if table.size == 0:
            table = table.reshape(0, 3)
        if table.ndim != 2 or table.shape[1] != 3:
            raise ValueError("couplers must be a sequence of (i, j, w) triples")
        ends = table[:, :2]
        if np.any(ends != np.floor(ends)):
            raise ValueError("coupler indices must be integers")
        self._setup(n, h, ends[:, 0].astype(np.int64), ends[:, 1].astype(np.int64),
                    table[:, 2].copy())

    @classmethod
    def from_arrays(cls, n, edges_i, edges_j, weights, h=None):
        """Build from integer edge arrays without the (E, 3) float triple table."""
        self = cls.__new__(cls)
        n = _spin_count(n)
        self._setup(n, _fields(n, h), np.asarray(edges_i, dtype=np.int64),
                    np.asarray(edges_j, dtype=np.int64), np.array(weights, dtype=np.float64))
        return self

    def _setup(self, n, h, a, b, w):
        rules = (
            (lambda: ((a < 0) | (a >= n) | (b < 0) | (b >= n)).any(),
             f"coupler index out of range [0, {n})"),
            (lambda: (a == b).any(), "self-couplings are not allowed"),
            (lambda: not np.isfinite(w).all(), "coupler weights must be finite"),
            (lambda: (w == 0.0).any(), "coupler weights must be nonzero"),
        )
        for broken, message in rules:
            if broken():
                raise ValueError(message)
        first, second = np.minimum(a, b), np.maximum(a, b)
        rank = first * n + second  # lexicographic rank of the unordered pair
        if rank.size > 1 and not (rank[1:] > rank[:-1]).all():
            order = np.argsort(rank, kind="stable")
            first, second, w, rank = first[order], second[order], w[order], rank[order]
            repeated = np.flatnonzero(rank[1:] == rank[:-1])
            if repeated.size:
                k = int(repeated[0])
                raise ValueError(f"duplicate coupler ({first[k]}, {second[k]})")
        self.n, self.h = n, h
        self.edges_i, self.edges_j, self.edge_weights = first, second, w
        pairs = n * (n - 1) // 2
        density = first.size / pairs if pairs else 0.0
        self.density, self.is_dense = density, density > DENSE_THRESHOLD
        for arr in (self.h, self.edges_i, self.edges_j, self.edge_weights):
            arr.flags.writeable = False
        self._handles = {}
        self._hlock = threading.Lock()
        self._csr = None

    # ---- reference-compatible views (problem.py:78-138), built on demand ----
    def _build_csr(self):
        if self._csr is None:
            lo, hi, ww = self.edges_i, self.edges_j, self.edge_weights
            rows = np.concatenate([lo, hi])
            cols = np.concatenate([hi, lo])
            vals = np.concatenate([ww, ww])
            perm = np.lexsort((cols, rows))
            indptr = np.zeros(self.n + 1, dtype=np.int64)
            np.cumsum(np.bincount(rows, minlength=self.n), out=indptr[1:])
            norm = np.sqrt(self.h ** 2 + np.bincount(rows, weights=vals ** 2, minlength=self.n))
            self._csr = (indptr, cols[perm], vals[perm], norm)
        return self._csr

    @property
    def csr_indptr(self):
        return self._build_csr()[0]

    @property
    def csr_indices(self):
        return self._build_csr()[1]

    @property
    def csr_weights(self):
        return self._build_csr()[2]

    @property
    def normalizers_safe(self):
        norm = self._build_csr()[3]
        return np.where(norm == 0.0, 1.0, norm)

    @property
    def dense_weights(self):
        if not self.is_dense:
            return None
        J = np.zeros((self.n, self.n))
        J[self.edges_i, self.edges_j] = self.edge_weights
        J[self.edges_j, self.edges_i] = self.edge_weights
        return J

    @property
    def num_edges(self):
        return int(self.edges_i.size)

    @property
    def w_total(self):
        return float(self.edge_weights.sum())

    def neighbors(self, i):
        indptr, idx, w, _ = self._build_csr()
        a, b = indptr[i], indptr[i + 1]
        return idx[a:b], w[a:b]

    def matvec(self, s):
        indptr, idx, w, _ = self._build_csr()
        s = np.asarray(s, dtype=np.float64)
        out = np.zeros(self.n)
        np.add.at(out, np.repeat(np.arange(self.n), np.diff(indptr)), w * s[idx])
        return out

    def __repr__(self):
        return f"IsingProblem(n={self.n}, edges={self.num_edges})"

    # ---- device handle ----
    def device_handle(self, device=0):
        """The immutable device-resident problem on `device` (created once)."""
        device = int(device)
        with self._hlock:
            h = self._handles.get(device)
            if h is None:
                lib = _native.load()
                out = ctypes.c_void_p()
                ei = np.ascontiguousarray(self.edges_i, dtype=np.int64)
                ej = np.ascontiguousarray(self.edges_j, dtype=np.int64)
                w = np.ascontiguousarray(self.edge_weights, dtype=np.float64)
                hv = np.ascontiguousarray(self.h, dtype=np.float64)
                _native.check(lib.nmfa_problem_create(
                    self.n, int(ei.size), _native.ptr(ei), _native.ptr(ej), _native.ptr(w),
                    _native.ptr(hv), device, ctypes.byref(out)))
                h = _DeviceProblem(out, device)
                self._handles[device] = h
            return h

    def device_info(self, device=0):
        return self.device_handle(device).info()


class _DeviceProblem:
    def __init__(self, handle, device):
        self.handle = handle
        self.device = device

    def info(self):
        info = _native.ProblemInfo()
        _native.check(_native.load().nmfa_problem_get_info(self.handle, ctypes.byref(info)))
        return {"n": info.n, "n_edges": info.n_edges, "density": info.density,
                "is_dense": bool(info.is_dense), "path": _native.PATH_NAMES[info.path],
                "j_exact": bool(info.j_exact), "int_weights": bool(info.int_weights),
                "j_scale": info.j_scale, "ell_slots": info.ell_slots,
                "field": _native.FIELD_NAMES[info.field]}

    def set_path(self, path):
        code = {v: k for k, v in _native.PATH_NAMES.items()}[path]
        _native.check(_native.load().nmfa_problem_set_path(self.handle, code))

    def set_field_precision(self, field):
        """Dense-path GEMM operand: "fp16" (hi only, the throughput mode) or
        "hilo" (hi + lo, the fidelity mode); see NMFA_FIELD_* in the header."""
        codes = {v: k for k, v in _native.FIELD_NAMES.items()}
        if field not in codes:
            raise ValueError(f"field precision must be one of {sorted(codes)}, got {field!r}")
        _native.check(_native.load().nmfa_problem_set_field_precision(self.handle, codes[field]))

    def __del__(self):
        try:
            if self.handle:
                _native.load().nmfa_problem_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


def pack_sign_bits(J):
    """Pack the signs of a symmetric +-1 matrix into the bitmap of the
    bit-packed device format: bit i * n + j (i < j, row-major, 32 per uint32,
    LSB first) set iff J_ij > 0.  1/64 of the float64 matrix."""
    J = np.asarray(J)
    n = J.shape[0]
    if J.ndim != 2 or J.shape != (n, n):
        raise ValueError("J must be a square matrix")
    iu, ju = np.triu_indices(n, 1)
    if np.any(np.abs(J[iu, ju]) != 1.0) or not np.array_equal(J[iu, ju], J[ju, iu]):
        raise ValueError("J must be symmetric with +-1 off-diagonal entries")
    flat = np.zeros(n * n, dtype=np.uint8)
    flat[iu * n + ju] = J[iu, ju] > 0
    pad = (-flat.size) % 32
    bits = np.packbits(np.concatenate([flat, np.zeros(pad, np.uint8)]), bitorder="little")
    return bits.view(np.uint32).copy()


class PackedSignProblem:
    """A complete +-1 instance (SK, K2000-style MAX-CUT) held as packed sign
    bits: the bit-packed device format.  The bitmap is
    expanded on the GPU into the dense path's J image
    (nmfa_problem_create_bits_device); no n(n-1)/2 host edge list exists, so
    n may reach the row-sharded sizes (65,536: a 512 MiB bitmap).  Accepted by
    sample / nmfa_batch / nmfa_run / energies like an IsingProblem; energies
    come from the exact tensor-core energy pass."""

    def __init__(self, n, bits, h=None):
        n = _spin_count(n)
        if n < 2:
            raise ValueError("a complete +-1 graph needs n >= 2")
        bits = np.ascontiguousarray(bits, dtype=np.uint32)
        if bits.ndim != 1 or bits.size < (n * n + 31) // 32:
            raise ValueError(f"bitmap needs {(n * n + 31) // 32} uint32 words for n = {n}")
        self.n, self.bits, self.h = n, bits, _fields(n, h)
        self._handles = {}
        self._hlock = threading.Lock()

    @classmethod
    def from_dense(cls, J, h=None):
        return cls(np.asarray(J).shape[0], pack_sign_bits(J), h)

    @property
    def num_edges(self):
        return self.n * (self.n - 1) // 2

    @property
    def w_total(self):
        """Sum of the couplings (cut_value's W_total): #(+1) - #(-1) over i < j."""
        words = (self.n * self.n + 31) // 32
        plus = int(np.unpackbits(self.bits[:words].view(np.uint8)).sum())
        return float(2 * plus - self.num_edges)

    @property
    def normalizers_safe(self):
        """sqrt(h_i^2 + n - 1): every spin has n - 1 unit couplers (problem.py:90-95)."""
        return np.sqrt(self.h * self.h + float(self.n - 1))

    def _rows(self, i0, i1):
        """Dense +-1 rows [i0, i1) of J from the bitmap (0 on the diagonal)."""
        n = self.n
        ii = np.arange(i0, i1)[:, None]
        jj = np.arange(n)[None, :]
        a, b = np.minimum(ii, jj), np.maximum(ii, jj)
        k = a * n + b
        bit = (self.bits[k >> 5] >> (k & 31).astype(np.uint32)) & 1
        J = np.where(bit == 1, 1.0, -1.0)
        J[ii == jj] = 0.0
        return J

    def matvec(self, s):
        """J @ s, unpacking the bitmap in row blocks (mean_field's sum_j J_ij s_j)."""
        s = np.asarray(s, dtype=np.float64)
        out = np.empty(self.n)
        step = max(1, (1 << 22) // self.n)
        for i0 in range(0, self.n, step):
            out[i0:i0 + step] = self._rows(i0, min(self.n, i0 + step)) @ s
        return out

    def _build_csr(self):  # normalizers(); the bitmap has no CSR, only its norms
        return None, None, None, np.sqrt(self.h * self.h + float(self.n - 1))

    def coupling(self, i, j):
        """J_ij from the bitmap (i != j)."""
        a, b = (i, j) if i < j else (j, i)
        k = a * self.n + b
        return 1.0 if (int(self.bits[k >> 5]) >> (k & 31)) & 1 else -1.0

    def device_handle(self, device=0):
        device = int(device)
        with self._hlock:
            h = self._handles.get(device)
            if h is None:
                out = ctypes.c_void_p()
                hv = np.ascontiguousarray(self.h, dtype=np.float64)
                _native.check(_native.load().nmfa_problem_create_bits_device(
                    self.n, _native.ptr(self.bits), _native.ptr(hv), 0, self.n, device,
                    ctypes.byref(out)))
                h = _DeviceProblem(out, device)
                self._handles[device] = h
            return h

    def device_info(self, device=0):
        return self.device_handle(device).info()


def as_problem(obj):
    """Accept our IsingProblem or any object with the reference's fields."""
    if isinstance(obj, (IsingProblem, PackedSignProblem)):
        return obj
    cached = getattr(obj, "_nmfa_b200_problem", None)
    if cached is not None:
        return cached
    p = IsingProblem.from_arrays(obj.n, obj.edges_i, obj.edges_j, obj.edge_weights, obj.h)
    try:
        object.__setattr__(obj, "_nmfa_b200_problem", p)
    except Exception:
        pass
    return p


def _check_length(problem, v, what):
    """Configurations / spins must end in a length-n axis (problem.py:150-183 messages)."""
    arr = np.asarray(v, dtype=np.float64)
    if arr.shape[-1:] == (problem.n,):
        return arr
    raise ValueError(f"{what} length {arr.shape} does not match problem size {problem.n}")


def energies(problem, configs, device=0):
    """GPU energies of a (R, n) batch of +-1 configurations (float64)."""
    import torch

    problem = as_problem(problem)
    c = _check_length(problem, configs, "configuration")
    c2 = np.atleast_2d(c)
    cfg = torch.from_numpy(np.where(c2 < 0.0, -1, 1).astype(np.int8)).to(f"cuda:{device}")
    out = torch.empty(cfg.shape[0], dtype=torch.float64, device=cfg.device)
    stream = torch.cuda.current_stream(cfg.device).cuda_stream
    _native.check(_native.load().nmfa_energy(problem.device_handle(device).handle,
                                             _native.ptr(cfg), cfg.shape[0], _native.ptr(out),
                                             ctypes.c_void_p(stream)))
    return out.cpu().numpy()


def energy(problem, config, device=0):
    """Ising energy sum_(i<j) w s_i s_j + sum_i h_i s_i of a +-1 config (problem.py:150)."""
    c = np.asarray(config, dtype=np.float64)
    problem = as_problem(problem)
    if c.shape != (problem.n,):
        raise ValueError(
            f"configuration length {c.shape} does not match problem size {problem.n}")
    return float(energies(problem, c[None, :], device)[0])


def cut_value(problem, config, device=0):
    """Total weight of cut edges; requires h = 0 (problem.py:157-163)."""
    problem = as_problem(problem)
    if np.any(problem.h != 0.0):
        raise ValueError("cut value is only defined for problems with zero fields")
    return (problem.w_total - energy(problem, config, device)) * 0.5


def mean_field(problem, s):
    """Raw mean field phi_i = h_i + sum_j J_ij s_j (problem.py:166-169)."""
    problem = as_problem(problem)
    v = _check_length(problem, s, "spin vector")
    return problem.h + problem.matvec(v)


def normalizers(problem):
    """sqrt(h_i^2 + sum_j J_ij^2); zero for isolated field-free spins (problem.py:172)."""
    return as_problem(problem)._build_csr()[3].copy()


def sign_round(s):
    """Round analog spins to +-1; exact zeros map to +1 (problem.py:181-183)."""
    return np.where(np.asarray(s, dtype=np.float64) < 0.0, -1.0, 1.0)
