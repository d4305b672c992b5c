"""The C-ABI library loads and exports every symbol include/nmfa_b200.h declares."""

import os
import re
import subprocess

import pytest

from paper_1806_08422_b200 import _native
from paper_1806_08422_b200 import build as nbuild

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include",
                      "nmfa_b200.h")


def declared():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(nmfa_\w+)\s*\(", txt, re.M)))


@pytest.fixture(scope="module")
def lib():
    nbuild.build()
    return _native.load()


def test_header_declares_expected_surface():
    names = declared()
    assert "nmfa_plan_run" in names and "nmfa_best_of" in names and len(names) >= 12
    assert set(names) == set(_native.SIGNATURES), "binding table out of sync with header"


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", _native.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\bT (nmfa_\w+)", out))
    missing = [n for n in declared() if n not in exported]
    assert not missing, missing


def test_version_and_error_without_gpu(lib):
    assert lib.nmfa_version().startswith(b"nmfa_b200")
    with pytest.raises(ValueError):
        _native.check(lib.nmfa_best_of(None, 0, None, None, None))
    assert b"NULL" in lib.nmfa_last_error()


def test_problem_create_rejects_bad_arguments(lib):
    import ctypes
    import numpy as np
    out = ctypes.c_void_p()
    ei = np.array([0], dtype=np.int64)
    ej = np.array([0], dtype=np.int64)
    w = np.array([1.0])
    with pytest.raises(ValueError, match="self-couplings"):
        _native.check(lib.nmfa_problem_create(2, 1, _native.ptr(ei), _native.ptr(ej),
                                              _native.ptr(w), None, 0, ctypes.byref(out)))
    with pytest.raises(ValueError, match="positive"):
        _native.check(lib.nmfa_problem_create(0, 0, None, None, None, None, 0, ctypes.byref(out)))


def test_backend_matches_reference_operator_signatures():
    """paper_1806_08422_b200.kernels has the reference backend's call signatures
    (kernels.py:30-32) -- checked against the installed reference when present."""
    import inspect
    import os
    import sys

    from paper_1806_08422_b200 import kernels as b200
    ref = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "nmfa")):
        pytest.skip("reference package not installed in baseline/_ref")
    sys.path.insert(0, ref)
    from nmfa import _kernels_numpy as refk
    for name in ("anneal_dense", "anneal_sparse", "gray_ground"):
        assert list(inspect.signature(getattr(b200, name)).parameters) == \
            list(inspect.signature(getattr(refk, name)).parameters), name


def test_problem_info_struct_matches_header(tmp_path):
    """The ctypes mirror of nmfa_problem_info_t has the C layout (size and every
    field offset, compiled from the header with gcc)."""
    import ctypes
    fields = [f for f, _ in _native.ProblemInfo._fields_]
    src = tmp_path / "layout.c"
    src.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"nmfa_b200.h\"\nint main(void){\n"
                   "printf(\"%zu\\n\", sizeof(nmfa_problem_info_t));\n" +
                   "".join(f"printf(\"%zu\\n\", offsetof(nmfa_problem_info_t, {f}));\n" for f in fields) +
                   "return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)], check=True)
    got = [int(x) for x in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [ctypes.sizeof(_native.ProblemInfo)] + [getattr(_native.ProblemInfo, f).offset
                                                   for f in fields]
    assert got == want, (got, want)


def test_missing_library_fails_loudly():
    """No CPU fallback: without the CUDA library every entry point raises
    (a fresh interpreter pointed at a missing library file)."""
    import subprocess
    import sys
    prog = (
        "import sys; sys.path.insert(0, %r)\n"
        "import paper_1806_08422_b200._native as N\n"
        "N.LIB_PATH = '/nonexistent/libnmfa_b200.so'; N._lib = None\n"
        "import paper_1806_08422_b200 as nb\n"
        "try:\n"
        "    nb.nmfa_batch(nb.gen_sk(20, 1), nb.NmfaParams(t_f=10), 4)\n"
        "except ImportError as e:\n"
        "    print('RAISED', 'no CPU fallback' in str(e))\n"
    ) % os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", prog], capture_output=True, text=True, timeout=300)
    assert "RAISED True" in out.stdout, out.stdout + out.stderr[-1500:]
