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
# checked build: redzone allocator + protocol jitter (csrc/guard.cu), tests only
GUARD_OUT = os.path.join(HERE, "libnmfa_b200_guard.so")
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-shared", "-Xcompiler", "-fPIC", "-Xptxas", "-v"]


def sources():
    return sorted(glob.glob(os.path.join(HERE, "csrc", "*.cu")))


def up_to_date(out=OUT):
    if not os.path.exists(out):
        return False
    deps = sources() + glob.glob(os.path.join(HERE, "csrc", "*.h*")) + \
        glob.glob(os.path.join(REPO, "include", "*.h"))
    return os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps)


def build(force=False, verbose=False, guard=False):
    out = GUARD_OUT if guard else OUT
    if not force and up_to_date(out):
        return out
    nvcc = os.environ.get("NVCC", "nvcc")
    extra = os.environ.get("NMFA_NVCC_DEFS", "").split()   # experiment builds only
    if guard:
        extra = ["-DNMFA_GUARD"]
    tmp = f"{out}.{os.getpid()}.tmp"  # per process: concurrent ranks may build at once
    # one nvcc per source in parallel (each .cu is self-contained), then one link
    from concurrent.futures import ThreadPoolExecutor
    objs = [f"{tmp}.{os.path.basename(src)}.o" for src in sources()]
    flags = [f for f in NVCC_FLAGS if f != "-shared"]

    def compile_one(src_obj):
        src, obj = src_obj
        return subprocess.run([nvcc, *flags, *extra, "-I", os.path.join(REPO, "include"), "-c",
                               "-o", obj, src], capture_output=True, text=True)

    try:
        with ThreadPoolExecutor(max_workers=min(len(objs), os.cpu_count() or 4)) as ex:
            results = list(ex.map(compile_one, zip(sources(), objs)))
        if all(r.returncode == 0 for r in results):
            results.append(subprocess.run([nvcc, "-shared", "-o", tmp, *objs],
                                          capture_output=True, text=True))
        bad = [r for r in results if r.returncode != 0]
        if bad:
            sys.stderr.write(bad[0].stdout + bad[0].stderr)
            raise RuntimeError(f"nvcc failed building {os.path.basename(out)}")
        if verbose:
            sys.stderr.write("".join(r.stderr for r in results))
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    os.replace(tmp, out)  # atomic: a loader sees the old or the new library, never a partial one
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, guard="--guard" in sys.argv))
