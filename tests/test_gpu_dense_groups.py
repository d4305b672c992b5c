"""GPU: the dense path's L2-aware replica groups (anneal_dense.cu
dense_plan_alloc) do not change results.

Replica blocks never interact, so annealing them as k groups one after
another (one persistent launch each) must give bit-identical configurations
and energies to one launch over all blocks: the K order is natural and the
noise is keyed by the global replica index in every group.  The group count
is read once per process (NMFA_DENSE_GROUPS), so each variant runs in its own
interpreter.  Uneven groups (5 replica blocks in 2 and 3 groups) and the
energy pass are covered; the automatic split itself is exercised by the
size sweep (profiles/r02/dense_groups.log).
"""

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
p = nb.gen_sk(640, 11)
p.device_handle().set_path("dense")
R, t_f = 1200, 40
params = nb.NmfaParams(t_f=t_f, seed=5)
plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
cfg = torch.empty((R, 640), dtype=torch.int8, device="cuda")
en = torch.empty(R, dtype=torch.float64, device="cuda")
plan.run(0, 0, config=cfg, energy=en)
torch.cuda.synchronize()
h = hashlib.sha1(cfg.cpu().numpy().tobytes() + en.cpu().numpy().tobytes()).hexdigest()
print("HASH", h, float(en.min()))
"""


def _run(groups):
    env = dict(os.environ)
    env.pop("NMFA_DENSE_GROUPS", None)
    if groups is not None:
        env["NMFA_DENSE_GROUPS"] = str(groups)
    env["NMFA_DENSE_VERBOSE"] = "1"
    out = subprocess.run([sys.executable, "-c", _PROG, ROOT], env=env, capture_output=True,
                         text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    line = [ln for ln in out.stdout.splitlines() if ln.startswith("HASH")][-1]
    plan_line = [ln for ln in out.stderr.splitlines() if ln.startswith("dense plan:")][-1]
    return line.split()[1], plan_line


def test_groups_bitwise_identical():
    base, plan1 = _run(1)
    assert "groups=1" in plan1
    for g in (2, 3, 5):
        h, plan_g = _run(g)
        assert f"groups={g}" in plan_g, plan_g
        assert h == base, f"{g} groups changed the results ({plan_g})"
