"""GPU: the reference's solver property tests (test_solver.py:181-253,
SURVEY 4), run through the C ABI on every kernel path.

* run == iterated steps (test_solver.py:181-190): with the replay mode the
  run draws the reference's own stream noise_stream(seed), so nmfa_run and t_f
  calls of nmfa_step sharing one generator see the same noise; the state
  crosses the step boundary at the kernels' own precision, so the two agree
  bit for bit.
* relabelling equivariance (test_solver.py:231-253): permuting the spins and
  the injected noise permutes the trajectory.  The reference asserts exact
  equality; here the permutation changes the summation order (tensor-core K
  order; CSR column order), so it holds within a stated tolerance (2e-3 on
  the fp16-operand paths, 1e-4 on the fp32 sparse path, whose two summation
  orders measure 1.6e-5 apart here) with identical signs wherever the spin is
  clear of zero.
* trajectory shape and boundedness (test_solver.py:192-201).
"""

import numpy as np
import pytest

import nmfa_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1806_08422_b200 as nb  # noqa: E402

PATHS = ["small", "sparse", "dense"]
# permuted vs unpermuted run (two fp32-sum orders, not GPU vs float64): the
# sparse bound is 1e-4 here (measured 1.6e-5 on this degree-20 graph after 120 steps)
TOL = {"small": 2e-3, "dense": 2e-3, "sparse": 1e-4}


@pytest.mark.parametrize("path", PATHS)
def test_run_equals_iterated_steps(path):
    p = nb.moebius_ladder(16)
    p.device_handle().set_path(path)
    params = nb.NmfaParams(t_f=20, seed=5)
    r = nb.nmfa_run(p, params, record_trajectory=True, noise="reference")
    temps = params.schedule.temperatures(params.t_f)
    rng = nb.noise_stream(params.seed)
    s = np.zeros(p.n)
    for t in range(params.t_f):
        s = nb.nmfa_step(p, s, float(temps[t]), params, rng)
    assert np.array_equal(s, r.trajectory.spins[-1]), np.abs(s - r.trajectory.spins[-1]).max()


@pytest.mark.parametrize("path", PATHS)
def test_relabeling_equivariance(path):
    rng = np.random.Generator(np.random.Philox(key=21))
    n = 40
    couplers = [(i, j, float(rng.integers(1, 4))) for i in range(n) for j in range(i + 1, n)
                if rng.random() < 0.5]
    p = nb.IsingProblem(n, couplers)
    perm = rng.permutation(n)
    q = nb.IsingProblem(n, [(min(perm[i], perm[j]), max(perm[i], perm[j]), w)
                            for i, j, w in couplers])
    p.device_handle().set_path(path)
    q.device_handle().set_path(path)
    temps = nb.DEFAULT_SCHEDULE.temperatures(120)
    noise = O.run_noise(8, 120, n, 0.15)
    s_base, _ = nb.run_with_noise(p, temps, noise, 0.15)
    inv = np.argsort(perm)             # spin k of the permuted problem is spin inv[k]
    s_perm, _ = nb.run_with_noise(q, temps, noise[:, inv], 0.15)
    err = np.abs(s_perm - s_base[inv])
    assert err.max() <= TOL[path], err.max()
    firm = np.abs(s_base[inv]) > TOL[path]
    assert np.array_equal(np.sign(s_perm[firm]), np.sign(s_base[inv][firm]))


@pytest.mark.parametrize("path", PATHS)
def test_trajectory_shapes_and_boundedness(path):
    p = nb.moebius_ladder(16)
    p.device_handle().set_path(path)
    r = nb.nmfa_run(p, nb.NmfaParams(t_f=100, seed=1), record_trajectory=True)
    assert r.trajectory.spins.shape == (100, 16) and r.trajectory.energies.shape == (100,)
    assert np.all(np.abs(r.trajectory.spins) < 1.0)
    assert np.abs(r.trajectory.spins[0]).max() < 0.3          # grow from 0 toward +-1
    assert np.abs(r.trajectory.spins[-1]).mean() > 0.8
    for t in (0, 10, 99):
        assert r.trajectory.energies[t] == nb.energy(p, nb.sign_round(r.trajectory.spins[t]))
