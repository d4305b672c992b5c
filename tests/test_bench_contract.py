"""bench.py's JSON contract on CPU: the reference arm (which times the
reference's nmfa_batch from baseline/_ref, or the oracle's port of its
per-run loop when that is not installed, on host cores) prints one JSON
line with the keys the driver reads."""

import json
import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(*args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], cwd=REPO,
                         capture_output=True, text=True, timeout=timeout,
                         env=dict(os.environ, OMP_NUM_THREADS="2"))
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_k2000_line():
    d = run("--impl", "reference", "--steps", "1", "--warmup", "0", "--ref-runs", "2")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "impl",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["metric"].endswith("on K2000")
    assert d["unit"] == "spin-updates/s" and d["value"] > 0 and d["higher_is_better"] is True
    # "reference" when baseline/_ref holds the installed reference, else the oracle "port"
    assert d["cpu_baseline"]["kind"] in ("reference", "port")
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_unavailable_workload():
    d = run("--workload", "sk65536", "--impl", "reference")
    assert d["impl"] == "reference" and "unavailable" in d


@pytest.mark.parametrize("wl", ["sk100", "moebius100", "g2000", "moebius131072"])
def test_workloads_are_declared(wl):
    sys.path.insert(0, REPO)
    import bench
    assert wl in bench.WORKLOADS and bench.metric_name(wl).endswith(wl)


def test_reference_arm_nonzero_rank_exits_quietly():
    """Under torchrun the reference arm runs on rank 0 only; other ranks exit 0
    with no output and no process group."""
    out = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--impl", "reference"],
                         cwd=REPO, capture_output=True, text=True, timeout=120,
                         env=dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1"))
    assert out.returncode == 0 and not out.stdout.strip(), out.stdout + out.stderr
