"""GPU: the CSR kernel's instances (anneal_sparse.cu sparse_step_kernel<2, k96,
kRL>, chosen per problem from the segment-size histogram, capi.cu
csr_variant) give bit-identical results: each instance sums every row in CSR
order from +0.  The instance is read once per process (NMFA_CSR_VARIANT), so
each runs in its own interpreter, on graphs of mean degree 5, 10 and 18 (the
three shapes the selection separates), with injected noise and seeded noise."""

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
import hashlib, sys, numpy as np, torch
sys.path.insert(0, sys.argv[1])
import paper_1806_08422_b200 as nb
out = []
for n, d in [(3000, 5), (3000, 10), (2048, 18)]:
    p = nb.gen_dense_maxcut(n, d / (n - 1), 2)
    p.device_handle().set_path("sparse")
    res = nb.sample(p, nb.NmfaParams(t_f=60, seed=4), 640)
    noise = np.random.default_rng(n).standard_normal((64, 30, n)) * 0.15
    S, _ = nb.run_with_noise(p, nb.DEFAULT_SCHEDULE.temperatures(30), noise, 0.15)
    out.append(hashlib.sha1(res.configs.cpu().numpy().tobytes() + res.energies.cpu().numpy().tobytes()
                            + np.ascontiguousarray(S).tobytes()).hexdigest())
print("HASH", " ".join(out))
"""


def _run(variant):
    env = dict(os.environ)
    env.pop("NMFA_CSR_VARIANT", None)
    if variant is not None:
        env["NMFA_CSR_VARIANT"] = str(variant)
    r = subprocess.run([sys.executable, "-c", _PROG, ROOT], env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    return [ln for ln in r.stdout.splitlines() if ln.startswith("HASH")][-1]


def test_csr_instances_bitwise_identical():
    auto = _run(None)
    for v in (0, 1, 2):
        assert _run(v) == auto, f"CSR instance {v} changed the results"
