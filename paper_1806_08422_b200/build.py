"""Build the in-tree C-ABI library libnmfa_b200.so for sm_100a with nvcc.

    python -m paper_1806_08422_b200.build
"""

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
OUT = os.path.join(HERE, "libnmfa_b200.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def up_to_date():
    if not os.path.exists(OUT):
        return False
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.h*")) + \
        glob.glob(os.path.join(REPO, "include", "*.h"))
    return os.path.getmtime(OUT) >= max(os.path.getmtime(d) for d in deps)


def build(force=False, verbose=False):
    if not force and up_to_date():
        return OUT
    nvcc = os.environ.get("NVCC", "nvcc")
    extra = os.environ.get("NMFA_NVCC_DEFS", "").split()   # experiment builds only
    tmp = f"{OUT}.{os.getpid()}.tmp"  # per process: concurrent ranks may build at once
    cmd = [nvcc, *NVCC_FLAGS, *extra, "-I", os.path.join(REPO, "include"), "-o", tmp, *sources()]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libnmfa_b200.so")
    if verbose:
        sys.stderr.write(res.stderr)
    os.replace(tmp, OUT)  # atomic: a loader sees the old or the new library, never a partial one
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
