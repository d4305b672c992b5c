"""Checked-build run of every kernel path (the memcheck / racecheck substitute:
compute-sanitizer is closed on this GPU pool).

tests/guard_workload.py runs the same seeded workload against the product
library and against libnmfa_b200_guard.so (csrc/guard.cu: 4 KB redzones
around every device allocation the library makes, fresh memory poisoned with
NaN bytes, randomised sleeps inside the persistent kernels' TMA / MMA /
epilogue protocol).  Required: no redzone byte written (library and caller
buffers), and every output bitwise identical to the product library's -- a
read of unwritten memory, an out-of-bounds read feeding a result, or a
readiness/fence hole exposed by the jitter would change them.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(tmp_path, lib):
    out = tmp_path / f"{lib}.npz"
    env = dict(os.environ, NMFA_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(REPO, "tests", "guard_workload.py"), str(out)],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    print(lib, r.stdout.strip().splitlines()[-1])
    return dict(np.load(out))


def test_checked_build_matches_and_keeps_redzones(tmp_path):
    from paper_1806_08422_b200 import build
    build.build()
    build.build(guard=True)
    plain = run(tmp_path, "product")
    checked = run(tmp_path, "guard")
    assert int(plain["guard_bad"]) == -1      # the product library has no guard allocator
    assert int(checked["guard_bad"]) == 0     # no redzone byte of any library allocation written
    keys = sorted(k for k in plain if k != "guard_bad")
    assert keys == sorted(k for k in checked if k != "guard_bad")
    diff = [k for k in keys if not np.array_equal(plain[k], checked[k], equal_nan=True)]
    assert not diff, diff
