"""GPU: the reference's acceptance criteria 4 and 5 (test_acceptance.py:
169-235) on these kernels.

* Criterion 5 (scaling-curve shape): the `nmfa bench` sweep over SK and
  dense MAX-CUT instances of 10..26 spins (10 instances, 1000 runs, t_f = 30,
  seed 0, exact ground truth from the GPU enumerator) has strictly decreasing
  success-probability medians with ordered IQRs.
* Criterion 4 (published 2000-spin quality, calibrated protocol t_f = 2000,
  100 runs): the K2000 file is not shipped (instances/README.md), so the
  reference's own stand-in gen_sk(2000, 7) (calibrate.py:44) carries its
  declared floor: best cut >= 32500.  G22 / G39 files are absent as in the
  reference's own run (its criterion 4 is skipped here).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1806_08422_b200 as nb  # noqa: E402
from paper_1806_08422_b200.experiments import BENCH_COLUMNS, bench  # noqa: E402


@pytest.mark.parametrize("cls", ["sk", "dense"])
def test_criterion_5_scaling_curve_shape(cls):
    rows, _, _ = bench(cls, [10, 14, 18, 22, 26], 10, 1000, nb.NmfaParams(t_f=30, seed=0))
    med = BENCH_COLUMNS.index("p_success_median")
    q1, q3 = BENCH_COLUMNS.index("p_success_q1"), BENCH_COLUMNS.index("p_success_q3")
    medians = [float(r[med]) for r in rows]
    print(f"\n{cls} medians: {np.round(medians, 3).tolist()}")
    for r in rows:
        assert float(r[q1]) <= float(r[med]) <= float(r[q3])
    assert all(a > b for a, b in zip(medians, medians[1:])), medians


def test_criterion_4_k2000_stand_in_quality():
    p = nb.gen_sk(2000, 7)
    runs = nb.nmfa_batch(p, nb.NmfaParams(t_f=2000, seed=1), 100)
    cuts = [nb.cut_value(p, r.final_config) for r in runs]
    print(f"\nK2000 stand-in: best cut {max(cuts)}, mean {np.mean(cuts):.1f}")
    assert max(cuts) >= 32500.0
