"""GPU regression tests for the round-1 advisor findings:
a plan cached for one path reused after set_path, the tensor-core energy
exactness gate with a power-of-two J scale, and trajectory energies for more
than 65535 * 32 recorded configurations."""

import numpy as np
import pytest

import nmfa_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1806_08422_b200 as nb  # noqa: E402
from paper_1806_08422_b200 import _native  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1806_08422_b200 import build
    build.build()
    _native.load()


@pytest.mark.parametrize("first,second", [("dense", "sparse"), ("sparse", "dense"),
                                          ("small", "sparse"), ("sparse", "small")])
def test_set_path_drops_the_cached_plan(first, second):
    p = nb.gen_cubic_maxcut(200, 3)
    h = p.device_handle()
    params = nb.NmfaParams(t_f=60, seed=9)
    h.set_path(first)
    nb.sample(p, params, 40)                 # caches a plan for `first`
    h.set_path(second)
    got = nb.sample(p, params, 40)           # same params: must not reuse it
    q = nb.gen_cubic_maxcut(200, 3)
    q.device_handle().set_path(second)
    want = nb.sample(q, params, 40)
    assert torch.equal(got.configs, want.configs)
    assert torch.equal(got.energies, want.energies)


def test_explicit_plan_rejects_a_changed_path():
    p = nb.gen_cubic_maxcut(200, 3)
    h = p.device_handle()
    h.set_path("sparse")
    plan = nb.Plan(p, 16, nb.Schedule([(0.0, 2.0), (1.0, 0.02)]).temperatures(20), 0.15, 0.15)
    h.set_path("dense")
    cfg = torch.empty((16, p.n), dtype=torch.int8, device="cuda")
    with pytest.raises(RuntimeError, match="another path"):
        plan.run(1, config=cfg)
    with pytest.raises(ValueError, match="unknown path"):
        _native.check(_native.load().nmfa_problem_set_path(h.handle, 7))


def test_scaled_integer_energies_stay_exact_past_2_24():
    """Weights in {+-1, +-2^15}: J is stored as J / 2^15, so a row sum is exact
    in fp32 only while sum |J_ij| < 2^24 in integer units.  Here the bound is
    exceeded, so energies must come from the edge-list kernel, bit-exact."""
    rng = np.random.default_rng(5)
    n = 1200
    ii, jj = np.triu_indices(n, 1)
    big = rng.random(ii.size) < 0.7
    w = np.where(big, 32768.0, 1.0) * np.where(rng.random(ii.size) < 0.5, 1.0, -1.0)
    p = nb.IsingProblem.from_arrays(n, ii, jj, w)
    info = p.device_info()
    assert info["path"] == "dense" and info["j_scale"] == 32768.0
    res = nb.sample(p, nb.NmfaParams(t_f=40, seed=3), 64)
    op = O.problem_from_edges(n, ii, jj, w)
    cfg = res.configs.cpu().numpy().astype(np.float64)
    assert np.array_equal(res.energies.cpu().numpy(), O.energies(op, cfg))


def test_trajectory_energies_beyond_the_old_grid_limit():
    """R * t_f = 4096 * 520 > 65535 * 32 recorded configurations."""
    p = nb.gen_sk(8, 2)
    R, t_f = 4096, 520
    res = nb.sample(p, nb.NmfaParams(t_f=t_f, seed=1), R, record_trajectory=True)
    s_hist = res.s_hist.cpu().numpy()
    e_hist = res.e_hist.cpu().numpy()
    op = O.problem_from_edges(p.n, p.edges_i, p.edges_j, p.edge_weights)
    for r in (0, 1777, R - 1):
        cfg = O.sign_round(s_hist[r])
        assert np.array_equal(e_hist[r], O.energies(op, cfg)), r
