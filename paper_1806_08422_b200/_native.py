"""ctypes binding of the C-ABI library `libnmfa_b200.so` (include/nmfa_b200.h).

There is no fallback: if the shared library is missing or no CUDA device is
present, every entry point raises.  Build it with `__graft_entry__.build()`
(or `python -m paper_1806_08422_b200.build`).
"""

from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# NMFA_LIB=guard selects the checked build (redzones + protocol jitter,
# csrc/guard.cu) for the guard tests; the default is the product library.
LIB_PATH = os.path.join(_HERE, "libnmfa_b200_guard.so" if os.environ.get("NMFA_LIB") == "guard"
                        else "libnmfa_b200.so")

NMFA_OK, NMFA_ERR_ARG, NMFA_ERR_CUDA, NMFA_ERR_STATE = 0, 1, 2, 3
PATH_SMALL, PATH_DENSE, PATH_SPARSE = 0, 1, 2
PATH_NAMES = {PATH_SMALL: "small", PATH_DENSE: "dense", PATH_SPARSE: "sparse"}
# dense-path GEMM operand precision (NMFA_FIELD_*, include/nmfa_b200.h)
FIELD_NAMES = {0: "fp16", 1: "hilo"}

# Every symbol include/nmfa_b200.h declares: name -> (restype, argtypes)
_p, _i32, _i64, _u64, _f64 = (ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64,
                              ctypes.c_uint64, ctypes.c_double)
SIGNATURES = {
    "nmfa_problem_create": (_i32, [_i64, _i64, _p, _p, _p, _p, _i32, ctypes.POINTER(_p)]),
    "nmfa_problem_destroy": (_i32, [_p]),
    "nmfa_problem_create_dense": (_i32, [_i64, _p, _p, _i32, ctypes.POINTER(_p)]),
    "nmfa_problem_create_dense_bits": (_i32, [_i64, _p, _p, _i32, ctypes.POINTER(_p)]),
    "nmfa_problem_create_bits_device": (_i32, [_i64, _p, _p, _i64, _i64, _i32, ctypes.POINTER(_p)]),
    "nmfa_problem_create_csr": (_i32, [_i64, _p, _p, _p, _p, _i32, ctypes.POINTER(_p)]),
    "nmfa_problem_get_info": (_i32, [_p, _p]),
    "nmfa_problem_set_path": (_i32, [_p, _i32]),
    "nmfa_problem_set_field_precision": (_i32, [_p, _i32]),
    "nmfa_plan_create": (_i32, [_p, _i64, _i32, _p, _f64, _f64, ctypes.POINTER(_p)]),
    "nmfa_plan_destroy": (_i32, [_p]),
    "nmfa_plan_run": (_i32, [_p, _u64, _i64, _p, _p, _p, _p, _p, _p, _p, _p]),
    "nmfa_anneal": (_i32, [_p, _i64, _i32, _p, _f64, _f64, _u64, _i64,
                           _p, _p, _p, _p, _p, _p, _p, _p]),
    "nmfa_anneal_host": (_i32, [_p, _i64, _i32, _p, _f64, _f64, _u64, _i64, _p, _p]),
    "nmfa_energy": (_i32, [_p, _p, _i64, _p, _p]),
    "nmfa_best_of": (_i32, [_p, _i64, _p, _p, _p]),
    "nmfa_last_error": (ctypes.c_char_p, []),
    "nmfa_version": (ctypes.c_char_p, []),
    "nmfa_last_launch_count": (_i64, []),
    "nmfa_debug_guard_check": (_i64, []),
    "nmfa_reference_noise": (_i32, [_u64, _i64, _i64, _i64, _f64, _p, _p, _p]),
    "nmfa_problem_create_sk_device": (_i32, [_i64, _u64, _i64, _i64, _i32, ctypes.POINTER(_p)]),
    "nmfa_plan_run_sweeps": (_i32, [_p, _u64, _i64, _i32, _i32, _i32, _p, _p, _p]),
    "nmfa_plan_image_info": (_i32, [_p, ctypes.POINTER(_p), ctypes.POINTER(_p),
                                    ctypes.POINTER(_i64), ctypes.POINTER(_i32),
                                    ctypes.POINTER(_i32), ctypes.POINTER(_i32)]),
    "nmfa_plan_read_config": (_i32, [_p, _p, _p]),
    "nmfa_anneal_many": (_i32, [_p, _i32, _i64, _i32, _p, _f64, _f64, _p, _p, _p, _p]),
    "nmfa_plan_set_exchange": (_i32, [_p, _p, _p, _i32, _i32, _i64]),
    "nmfa_gset_parse": (_i32, [ctypes.c_char_p, _i64, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                               _p, _p, _p, _i64]),
    "nmfa_problem_create_gset": (_i32, [ctypes.c_char_p, _i64, _i32, ctypes.POINTER(_p)]),
    "nmfa_ground_state": (_i32, [_p, _i32, ctypes.POINTER(_f64), ctypes.POINTER(_i64), _p]),
}


class ProblemInfo(ctypes.Structure):
    _fields_ = [("n", _i64), ("n_edges", _i64), ("density", _f64), ("is_dense", _i32),
                ("path", _i32), ("j_exact", _i32), ("int_weights", _i32), ("j_scale", _f64),
                ("ell_slots", _i32), ("field", _i32)]


_lib = None
_lock = threading.Lock()


def load():
    """Load the library once; raise ImportError with a build hint if absent."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"NMFA CUDA library not built ({LIB_PATH} missing); "
                "run __graft_entry__.build() -- there is no CPU fallback")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def check(code):
    """Map a status code to the reference's exception types."""
    if code == NMFA_OK:
        return
    msg = load().nmfa_last_error().decode(errors="replace")
    if code == NMFA_ERR_ARG:
        raise ValueError(msg)
    raise RuntimeError(msg)


def ptr(t):
    """Raw pointer of a torch tensor / numpy array (None -> NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return ctypes.c_void_p(t.data_ptr())
    return t.ctypes.data_as(ctypes.c_void_p)
