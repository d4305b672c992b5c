"""GPU: the reference's solver edge cases (test_solver.py), on every kernel path.

The reference runs these on its CPU kernels; here each one is forced onto the
small, sparse and dense paths in turn (the dense path pads a 1- or 2-spin
instance to a 128-spin k-slice and a 256-replica block, the ragged extreme):

* single spin in a field aligns against it, in every run
  (test_solver.py:167-172, 274-277);
* alpha = 0 keeps the initial state exactly (test_solver.py:292-297) and
  alpha = 0, sigma = 0 is the identity step (106-113);
* results stay strictly inside the unit box (123-130);
* the same seed gives bit-identical results and final energies are
  recomputable with energy() (157-165, 174-179);
* nmfa_batch seeds are seed + k in order, and `threads` changes nothing
  (257-272); zero runs and bad shapes are rejected (279-290).
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1806_08422_b200 as nb  # noqa: E402

PATHS = ["small", "sparse", "dense"]


def on(path, p):
    p.device_handle().set_path(path)
    return p


def two_spin():
    return nb.IsingProblem(2, [(0, 1, 1.0)])


@pytest.mark.parametrize("path", PATHS)
def test_single_spin_field_alignment(path):
    p = on(path, nb.IsingProblem(1, [], h=[1.0]))
    r = nb.nmfa_run(p, nb.NmfaParams(sigma=0.0, t_f=50, seed=0))
    assert np.array_equal(r.final_config, [-1.0])
    assert r.final_energy == -1.0
    res = nb.nmfa_batch(p, nb.NmfaParams(sigma=0.0, t_f=20, seed=0), 300)
    assert all(np.array_equal(x.final_config, [-1.0]) for x in res)


@pytest.mark.parametrize("path", PATHS)
def test_zero_alpha_keeps_initial_state(path):
    p = on(path, two_spin())
    s0 = np.array([0.25, -0.5])
    temps = np.full(10, 0.5)
    s, _ = nb.run_with_noise(p, temps, np.zeros((10, 2)), 0.0, s0=s0)
    assert np.array_equal(s, s0)
    # with noise too: alpha = 0 ignores the field entirely
    noise = np.random.default_rng(1).standard_normal((10, 2))
    s, _ = nb.run_with_noise(p, temps, noise, 0.0, s0=s0)
    assert np.array_equal(s, s0)


@pytest.mark.parametrize("path", PATHS)
def test_result_strictly_inside_unit_box(path):
    p = on(path, nb.gen_sk(12, 3))
    temps = np.full(40, 1e-3)           # saturating: tanh of a huge argument
    noise = np.random.default_rng(2).standard_normal((64, 40, 12)) * 5.0
    S, _ = nb.run_with_noise(p, temps, noise, 1.0)
    assert np.all(np.abs(S) < 1.0)
    assert np.all(np.abs(S) > 0.5)


@pytest.mark.parametrize("path", PATHS)
def test_same_seed_bit_identical_and_energy_recomputable(path):
    p = on(path, nb.moebius_ladder(16))
    params = nb.NmfaParams(t_f=50, seed=9)
    a = nb.nmfa_batch(p, params, 40)
    b = nb.nmfa_batch(p, params, 40)
    for x, y in zip(a, b):
        assert np.array_equal(x.final_config, y.final_config)
        assert x.final_energy == y.final_energy
        assert x.final_energy == nb.energy(p, x.final_config)


@pytest.mark.parametrize("path", PATHS)
def test_seeds_offset_order_and_threads(path):
    p = on(path, nb.moebius_ladder(16))
    params = nb.NmfaParams(t_f=30, seed=100)
    res = nb.nmfa_batch(p, params, 5)
    assert [r.seed for r in res] == [100, 101, 102, 103, 104]
    # run k of the batch is nmfa_run with seed + k
    for k in (0, 3):
        one = nb.nmfa_run(p, nb.NmfaParams(t_f=30, seed=100 + k))
        assert np.array_equal(one.final_config, res[k].final_config)
    threaded = nb.nmfa_batch(p, params, 5, threads=4)
    for x, y in zip(res, threaded):
        assert np.array_equal(x.final_config, y.final_config)


@pytest.mark.parametrize("path", PATHS)
def test_rejections(path):
    p = on(path, two_spin())
    with pytest.raises(ValueError):
        nb.nmfa_batch(p, nb.NmfaParams(), 0)
    with pytest.raises(ValueError, match="noise shape"):
        nb.run_with_noise(p, np.array([1.0]), np.zeros((2, 2)), 0.15)
    with pytest.raises(ValueError, match="s0 length"):
        nb.run_with_noise(p, np.array([1.0]), np.zeros((1, 2)), 0.15, s0=np.zeros(3))
