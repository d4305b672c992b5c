"""Extract numpy's ziggurat tables (ki_double / wi_double / fi_double of
numpy/random/src/distributions/ziggurat_constants.h) from the installed
numpy's libnpyrandom.a and write them as a CUDA header, then verify a
pure-Python restatement of Generator(Philox(key)).standard_normal against
numpy itself, bit for bit.  Build container only; the header is committed.

    python tools/gen_numpy_normal_tables.py

numpy is a third-party dependency of the reference (numpy
2.3.5 here; pyproject.toml:10-14 gives only numpy>=1.24).  The reference
draws each run's noise as noise_stream(seed).standard_normal((t_f, n))
(solver.py:182-185, 236-241): Philox4x64-10 keyed [seed, RUN_STREAM_TAG=2],
counter from 0, four-word output buffer, and numpy's 256-layer ziggurat.
"""

import os
import struct
import subprocess
import sys
import tempfile

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(REPO, "paper_1806_08422_b200", "csrc", "numpy_normal_tables.h")
MASK = (1 << 64) - 1
M0, M1 = 0xD2E7470EE14C6C93, 0xCA5A826395121157
W0, W1 = 0x9E3779B97F4A7C15, 0xBB67AE8584CAA73B
ZIG_R = 3.6541528853610087963519472518
ZIG_INV_R = 0.27366123732975827203338247596


def extract():
    lib = os.path.join(os.path.dirname(np.__file__), "random", "lib", "libnpyrandom.a")
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["ar", "x", lib], cwd=d, check=True)
        obj = [f for f in os.listdir(d) if f.endswith("distributions.c.o")][0]
        path = os.path.join(d, obj)
        sec = subprocess.run(["readelf", "-S", "-W", path], capture_output=True, text=True).stdout
        syms = subprocess.run(["readelf", "-s", "-W", path], capture_output=True, text=True).stdout
        blob = open(path, "rb").read()
    shdr = {}
    for line in sec.splitlines():
        parts = line.replace("[ ", "[").split()
        if len(parts) > 5 and parts[0].startswith("[") and parts[1].startswith("."):
            shdr[int(parts[0].strip("[]"))] = (parts[1], int(parts[4], 16))
    tabs = {}
    for line in syms.splitlines():
        p = line.split()
        if len(p) == 8 and p[7] in ("ki_double", "wi_double", "fi_double"):
            off = shdr[int(p[6])][1] + int(p[1], 16)
            raw = blob[off:off + int(p[2])]
            tabs[p[7]] = struct.unpack("<256Q" if p[7] == "ki_double" else "<256d", raw)
    return tabs


def philox4x64(ctr, key):
    c, k = list(ctr), list(key)
    for _ in range(10):
        p0, p1 = M0 * c[0], M1 * c[2]
        c = [(p1 >> 64) ^ c[1] ^ k[0], p1 & MASK, (p0 >> 64) ^ c[3] ^ k[1], p0 & MASK]
        k = [(k[0] + W0) & MASK, (k[1] + W1) & MASK]
    return c


class Stream:
    """numpy Generator(Philox(key=(2 << 64) | seed)) restated."""

    def __init__(self, seed, tabs):
        self.ctr, self.key, self.buf, self.pos = [0, 0, 0, 0], [seed & MASK, 2], [0] * 4, 4
        self.ki, self.wi, self.fi = tabs["ki_double"], tabs["wi_double"], tabs["fi_double"]

    def u64(self):
        if self.pos < 4:
            self.pos += 1
            return self.buf[self.pos - 1]
        for i in range(4):  # 256-bit counter increment with carry
            self.ctr[i] = (self.ctr[i] + 1) & MASK
            if self.ctr[i]:
                break
        self.buf, self.pos = philox4x64(self.ctr, self.key), 1
        return self.buf[0]

    def double(self):
        return (self.u64() >> 11) * (1.0 / 9007199254740992.0)

    def normal(self):
        while True:
            r = self.u64()
            idx = r & 0xFF
            r >>= 8
            sign = r & 1
            rabs = (r >> 1) & 0x000FFFFFFFFFFFFF
            x = rabs * self.wi[idx]
            if sign:
                x = -x
            if rabs < self.ki[idx]:
                return x
            if idx == 0:
                while True:
                    xx = -ZIG_INV_R * np.log1p(-self.double())
                    yy = -np.log1p(-self.double())
                    if yy + yy > xx * xx:
                        return -(ZIG_R + xx) if (rabs >> 8) & 1 else ZIG_R + xx
            elif (self.fi[idx - 1] - self.fi[idx]) * self.double() + self.fi[idx] < np.exp(-0.5 * x * x):
                return x


def verify(tabs, seeds=(0, 1, 12345, MASK), count=20000):
    for s in seeds:
        want = np.random.Generator(np.random.Philox(key=(2 << 64) | s)).standard_normal(count)
        st = Stream(s, tabs)
        got = np.array([st.normal() for _ in range(count)])
        if not np.array_equal(got.view(np.uint64), want.view(np.uint64)):
            bad = int(np.argmax(got != want))
            sys.exit(f"seed {s}: mismatch at draw {bad}: {got[bad]!r} vs {want[bad]!r}")
    print(f"restatement == numpy {np.__version__} bit for bit on {len(seeds)} streams x {count} normals")


def main():
    tabs = extract()
    verify(tabs)
    with open(OUT, "w") as f:
        f.write("// numpy's ziggurat tables for Generator.standard_normal (numpy/random/src/\n"
                f"// distributions/ziggurat_constants.h), extracted from numpy {np.__version__}'s\n"
                "// libnpyrandom.a by tools/gen_numpy_normal_tables.py, which also checks a\n"
                "// restatement against numpy bit for bit.  Used by refnoise.cu.  Generated.\n#pragma once\n"
                "#include <cstdint>\nnamespace nmfa {\n")
        f.write(f"constexpr double kZigR = {ZIG_R!r};\nconstexpr double kZigInvR = {ZIG_INV_R!r};\n")
        f.write("__device__ const uint64_t kZigKi[256] = {\n")
        f.write(",\n".join("  " + ", ".join(f"0x{v:016X}ull" for v in tabs["ki_double"][i:i + 4])
                           for i in range(0, 256, 4)))
        for name, key in (("kZigWi", "wi_double"), ("kZigFi", "fi_double")):
            f.write(f"}};\n__device__ const double {name}[256] = {{\n")
            f.write(",\n".join("  " + ", ".join(f"{v!r}" for v in tabs[key][i:i + 4])
                               for i in range(0, 256, 4)))
        f.write("};\n}  // namespace nmfa\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
