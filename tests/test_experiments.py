"""Multi-instance sweeps (cli.py:280-347) and their aggregation
(metrics.py:109-142): host logic on CPU, batched anneals on the GPU."""

import math

import numpy as np
import pytest

import paper_1806_08422_b200 as nb
from paper_1806_08422_b200.metrics import RunStats


def test_median_iqr_examples():  # test_metrics.py:123-129
    assert nb.median_iqr([1.0, 2.0, 3.0]) == (2.0, 1.5, 2.5)
    assert nb.median_iqr([7.0]) == (7.0, 7.0, 7.0)
    with pytest.raises(ValueError):
        nb.median_iqr([])


def test_median_iqr_matches_numpy_percentiles():  # test_metrics.py:131-141
    rng = np.random.Generator(np.random.Philox(key=41))
    for _ in range(300):
        v = rng.standard_normal(int(rng.integers(1, 30)))
        med, q1, q3 = nb.median_iqr(v)
        lq1, lmed, lq3 = np.percentile(v, [25.0, 50.0, 75.0])
        assert (med, q1, q3) == pytest.approx((lmed, lq1, lq3), rel=1e-12)


def test_aggregate_over_instances():  # test_metrics.py:143-153
    stats = [RunStats(p_success=p, tts_seconds=t, mean_energy=0.0, best_energy=0.0)
             for p, t in [(0.2, 10.0), (0.5, 4.0), (0.8, 1.0)]]
    agg = nb.aggregate(stats)
    assert agg.p_success_median == 0.5
    assert (agg.p_success_q1, agg.p_success_q3) == (0.35, 0.65)
    assert agg.tts_median == 4.0


def test_aggregate_with_infinite_tts():
    stats = [RunStats(p_success=p, tts_seconds=t, mean_energy=0.0, best_energy=0.0)
             for p, t in [(0.0, math.inf), (0.5, 4.0), (0.9, 2.0), (0.0, math.inf)]]
    agg = nb.aggregate(stats)
    assert agg.tts_q3 == math.inf and not math.isnan(agg.tts_median)


def test_bench_argument_checks():
    from paper_1806_08422_b200.experiments import bench, make_instance
    with pytest.raises(ValueError, match="at least 1"):
        bench("sk", [10], 0, 10)
    with pytest.raises(ValueError, match="enumeration bound"):
        bench("sk", [30], 2, 10)
    with pytest.raises(ValueError, match="unknown instance class"):
        make_instance("torus", 10, 0.5, 0)


torch = pytest.importorskip("torch")


@pytest.mark.gpu
@pytest.mark.parametrize("n,cls", [(40, "sk"), (100, "cubic"), (300, "sk")])
def test_sample_many_equals_per_instance_runs(n, cls):
    """Grouped launch (n <= 256) and the per-instance fallback give the same
    replicas, bit for bit, as separate sample() calls with the bench seeds."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from dataclasses import replace

    from paper_1806_08422_b200.experiments import make_instance
    params = nb.NmfaParams(t_f=150, seed=5)
    probs = [make_instance(cls, n, 0.5, 100 + k) for k in range(5)]
    cfg, en, _ = nb.sample_many(probs, params, 200)
    for k, p in enumerate(probs):
        one = nb.sample(p, replace(params, seed=params.seed + k * 200), 200)
        assert torch.equal(cfg[k], one.configs)
        assert torch.equal(en[k], one.energies)


@pytest.mark.gpu
def test_bench_rows():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_1806_08422_b200.experiments import BENCH_COLUMNS, bench
    rows, text, per = bench("moebius", [16], 3, 512, nb.NmfaParams(t_f=100, seed=0))
    assert text.splitlines()[0] == ",".join(BENCH_COLUMNS)
    assert rows[0][:4] == ["moebius", 16, 3, 512]
    # Moebius-16 at t_f = 100 reaches the ground state essentially always (stats.npz: p = 1.0)
    assert float(rows[0][5]) >= 0.95
    rows, _, per = bench("sk", [12, 16], 4, 256, nb.NmfaParams(t_f=200, seed=1))
    for n in (12, 16):
        assert all(0.0 <= s.p_success <= 1.0 for s in per[n])
        assert all(s.best_energy <= s.mean_energy for s in per[n])
