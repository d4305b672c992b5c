"""GPU: the small kernel's shared-memory sincos table (anneal_small.cu kTab,
common.cuh sincos_table_fill) reproduces the inline MUFU.SIN/COS noise bit
for bit: same configurations and energies with the table on and off
(NMFA_SMALL_TABLE, read once per process), on SK100, a Moebius ladder, a
grouped multi-instance launch and the largest small size (n = 256)."""

import os
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_PROG = r"""
import hashlib, sys, torch
sys.path.insert(0, sys.argv[1])
import paper_1806_08422_b200 as nb
h = hashlib.sha1()
for p in [nb.gen_sk(100, 0), nb.moebius_ladder(100), nb.gen_sk(256, 3)]:
    p.device_handle().set_path("small")
    r = nb.sample(p, nb.NmfaParams(t_f=200, seed=9), 1000)
    h.update(r.configs.cpu().numpy().tobytes() + r.energies.cpu().numpy().tobytes())
cfg, en, _ = nb.sample_many([nb.gen_sk(40, k) for k in range(4)], nb.NmfaParams(t_f=100, seed=2), 300)
h.update(cfg.cpu().numpy().tobytes() + en.cpu().numpy().tobytes())
print("HASH", h.hexdigest())
"""


def _run(table):
    env = dict(os.environ, NMFA_SMALL_TABLE=table)
    r = subprocess.run([sys.executable, "-c", _PROG, ROOT], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return [ln for ln in r.stdout.splitlines() if ln.startswith("HASH")][-1]


def test_sincos_table_is_bitwise_the_inline_noise():
    assert _run("1") == _run("0")
