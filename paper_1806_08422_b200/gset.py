"""Instance text I/O (reference gset.py): parse / load / write the edge-list
("G-set") format.  Parsing runs in the native library (nmfa_gset_parse, a
single pass over the bytes: tens of milliseconds for a K2000-size file the
reference needs ~6.5 s for); the messages and line numbers of
GsetParseError are the reference's (gset.py:18-89).
"""

from __future__ import annotations

import ctypes
import re

import numpy as np

from . import _native
from .problem import IsingProblem, cut_value  # noqa: F401  (cut_value: the reference's gset namespace)

# non-ASCII characters str.splitlines() / str.split() treat as breaks / spaces
_NON_ASCII_BREAKS = "\x85\u2028\u2029"
_NON_ASCII_SPACE = "".join(chr(c) for c in range(0x80, 0x3001) if chr(c).isspace()
                           and chr(c) not in _NON_ASCII_BREAKS)
_TRANSLATE = {ord(c): "\n" for c in _NON_ASCII_BREAKS} | {ord(c): " " for c in _NON_ASCII_SPACE}
_LINE_RE = re.compile(r"^line (-?\d+): (.*)$", re.S)


class GsetParseError(ValueError):
    """Malformed instance text; carries the 1-based offending line number (gset.py:18-23)."""

    def __init__(self, line_no, message):
        super().__init__(f"line {line_no}: {message}")
        self.line_no = line_no


def _parse_bytes(data):
    lib = _native.load()
    n, m = ctypes.c_int64(), ctypes.c_int64()

    def check(code):
        if code == _native.NMFA_OK:
            return
        msg = lib.nmfa_last_error().decode(errors="replace")
        hit = _LINE_RE.match(msg)
        if code == _native.NMFA_ERR_ARG and hit:
            raise GsetParseError(int(hit.group(1)), hit.group(2))
        _native.check(code)

    check(lib.nmfa_gset_parse(data, len(data), ctypes.byref(n), ctypes.byref(m), None, None, None, 0))
    ei = np.empty(m.value, dtype=np.int64)
    ej = np.empty(m.value, dtype=np.int64)
    w = np.empty(m.value, dtype=np.float64)
    check(lib.nmfa_gset_parse(data, len(data), ctypes.byref(n), ctypes.byref(m), _native.ptr(ei),
                              _native.ptr(ej), _native.ptr(w), m.value))
    return IsingProblem.from_arrays(n.value, ei, ej, w)


def parse_gset(text):
    """Parse instance text into a zero-field problem (gset.py:35-89)."""
    if not text.isascii():
        text = text.translate(_TRANSLATE)
    return _parse_bytes(text.encode("utf-8", errors="replace"))


def load_gset(path):
    """Read and parse an instance file; undecodable bytes become parse errors (gset.py:92-96)."""
    with open(path, "rb") as fh:
        raw = fh.read()
    if raw.isascii():
        return _parse_bytes(raw)
    return parse_gset(raw.decode("utf-8", errors="replace"))


def write_gset(problem):
    """Canonical instance text (gset.py:99-109): header, then one "u v w" line
    per coupler in canonical order with 1-based vertices and integer weights;
    instances with fields or fractional weights cannot be written."""
    weights = np.asarray(problem.edge_weights)
    if (np.asarray(problem.h) != 0.0).any():
        raise ValueError("instance format has no field column; h must be zero")
    if (weights != np.round(weights)).any():
        raise ValueError("instance format requires integer weights")
    body = "".join(f"{a + 1} {b + 1} {int(x)}\n"
                   for a, b, x in zip(problem.edges_i, problem.edges_j, weights))
    return f"{problem.n} {problem.num_edges}\n" + body


# one row per run, fixed column order (reference gset.py:107-130: the results
# file of the CLI's solve/bench commands)
RESULT_COLUMNS = ("instance_id", "seed", "final_energy", "cut_value", "wall_clock_us")


def write_results_csv(results, metadata):
    """CSV text of RunResults: instance_id on every row; cut_value when
    metadata["problem"] has zero fields; wall_clock_us = round(wall_clock * 1e6)
    when metadata["timings"] is true, else 0 (reruns of the same seeds then give
    byte-identical files).  Floats are written with repr, like the reference.
    The cut is (W_total - E) / 2 from each run's exact final energy, the
    identity the reference's own tests pin (test_problem.py:138-145): equal to
    its edge sum for integer weights, within an ulp for real ones, and O(1)
    per row instead of a pass over the edges."""
    import csv
    import io

    from .problem import as_problem

    meta = dict(metadata)
    problem = meta.get("problem")
    if problem is not None:
        problem = as_problem(problem)
    with_cut = problem is not None and not np.any(np.asarray(problem.h) != 0.0)
    timed = bool(meta.get("timings", False))
    out = io.StringIO()
    rows = csv.writer(out, lineterminator="\n")
    rows.writerow(RESULT_COLUMNS)
    for run in results:
        rows.writerow([meta.get("instance_id", ""), run.seed, repr(run.final_energy),
                       repr((problem.w_total - float(run.final_energy)) * 0.5) if with_cut else "",
                       int(round(run.wall_clock * 1e6)) if timed else 0])
    return out.getvalue()

