"""Host-side mirror of the reference API (no GPU needed)."""

import hashlib

import numpy as np
import pytest

import paper_1806_08422_b200 as nb
from paper_1806_08422_b200 import solver


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("t_f", [1, 2, 37, 101, 1000])
def test_schedule_golden(G, t_f):
    assert np.array_equal(nb.DEFAULT_SCHEDULE.temperatures(t_f), G["schedule"][f"default_{t_f}"])


def test_schedule_semantics():
    assert nb.schedule_eval(nb.DEFAULT_SCHEDULE, 26, 101) == 0.8
    assert nb.schedule_eval(nb.DEFAULT_SCHEDULE, 76, 101) == 0.2
    assert nb.schedule_eval(nb.Schedule([(0.0, 1.0), (1.0, 0.01)]), 2, 3) == pytest.approx(0.1)
    temps = nb.DEFAULT_SCHEDULE.temperatures(37)
    assert all(temps[t - 1] == nb.DEFAULT_SCHEDULE.temperature(t, 37) for t in range(1, 38))
    s = nb.Schedule.parse("0:2,0.25:0.8,0.75:0.2,1:0.02")
    assert s == nb.DEFAULT_SCHEDULE and nb.Schedule.parse(s.format()) == s
    for bad in ([(0.0, 1.0)], [(0.1, 1.0), (1.0, 0.1)], [(0.0, 1.0), (0.5, 0.5), (0.5, 0.2), (1.0, 0.1)],
                [(0.0, 1.0), (1.0, 0.0)]):
        with pytest.raises(ValueError):
            nb.Schedule(bad)
    with pytest.raises(ValueError):
        nb.Schedule.parse("0:2,half:1,1:0.1")
    with pytest.raises(ValueError):
        nb.schedule_eval(nb.DEFAULT_SCHEDULE, 0, 10)


@pytest.mark.parametrize("kw", [{"alpha": -0.1}, {"alpha": 1.5}, {"sigma": -1.0}, {"t_f": 0},
                                {"seed": -1}, {"seed": 1 << 64}])
def test_params_validation(kw):
    with pytest.raises(ValueError):
        nb.NmfaParams(**kw)


def test_params_defaults():
    p = nb.NmfaParams()
    assert (p.alpha, p.sigma, p.t_f, p.seed) == (0.15, 0.15, 1000, 0)


def test_problem_validation_messages():
    with pytest.raises(ValueError, match="spin count must be positive"):
        nb.IsingProblem(0)
    with pytest.raises(ValueError, match="self-couplings"):
        nb.IsingProblem(3, [(1, 1, 1.0)])
    with pytest.raises(ValueError, match="out of range"):
        nb.IsingProblem(3, [(0, 3, 1.0)])
    with pytest.raises(ValueError, match="duplicate coupler"):
        nb.IsingProblem(3, [(0, 1, 1.0), (1, 0, 2.0)])
    with pytest.raises(ValueError, match="nonzero"):
        nb.IsingProblem(3, [(0, 1, 0.0)])
    with pytest.raises(ValueError, match="finite"):
        nb.IsingProblem(3, [(0, 1, np.inf)])
    with pytest.raises(ValueError, match="h must have length"):
        nb.IsingProblem(3, [], h=[1.0])
    with pytest.raises(ValueError, match="integers"):
        nb.IsingProblem(3, [(0.5, 1, 1.0)])


def test_problem_canonicalisation_and_csr():
    p = nb.IsingProblem(4, [(3, 1, 2.0), (0, 2, -1.0), (2, 1, 5.0)], h=[1, 0, 0, 0])
    assert p.edges_i.tolist() == [0, 1, 1] and p.edges_j.tolist() == [2, 2, 3]
    idx, w = p.neighbors(1)
    assert idx.tolist() == [2, 3] and w.tolist() == [5.0, 2.0]
    assert np.allclose(p.normalizers_safe, np.sqrt([1 + 1, 29, 26, 4]))
    assert np.array_equal(nb.mean_field(p, np.ones(4)), [0.0, 7.0, 4.0, 2.0])
    iso = nb.IsingProblem(2)
    assert np.array_equal(iso.normalizers_safe, [1.0, 1.0])
    assert np.array_equal(nb.normalizers(iso), [0.0, 0.0])


def test_sign_round():
    assert np.array_equal(nb.sign_round([-0.0, 0.0, -1e-300, 3.0]), [1.0, 1.0, -1.0, 1.0])


@pytest.mark.parametrize("name,builder", [
    ("sk100_s0", lambda: nb.gen_sk(100, 0)), ("sk30_s2", lambda: nb.gen_sk(30, 2)),
    ("moebius16", lambda: nb.moebius_ladder(16)), ("moebius100", lambda: nb.moebius_ladder(100)),
    ("cubic40_s1", lambda: nb.gen_cubic_maxcut(40, 1)),
    ("dense60_p03_s3", lambda: nb.gen_dense_maxcut(60, 0.3, 3))])
def test_generators_match_reference(G, name, builder):
    I = G["instances"]
    p = builder()
    assert np.array_equal(p.edges_i, I[name + "_ei"])
    assert np.array_equal(p.edges_j, I[name + "_ej"])
    assert np.array_equal(p.edge_weights, I[name + "_w"])
    assert np.array_equal(p.normalizers_safe, I[name + "_norm"])
    assert p.is_dense == bool(I[name + "_is_dense"])


def test_large_standins_match_reference(G):
    I = G["instances"]
    for name, p in (("sk2000_s7", nb.gen_sk(2000, 7)),
                    ("g2000_p001_s7", nb.gen_dense_maxcut(2000, 0.01, 7))):
        assert p.num_edges == int(I[name + "_nedges"])
        assert sha(p.edges_i) == str(I[name + "_sha_ei"])
        assert sha(p.edges_j) == str(I[name + "_sha_ej"])
        assert sha(p.edge_weights) == str(I[name + "_sha_w"])
        assert p.is_dense == bool(I[name + "_is_dense"])


def test_metrics():
    assert nb.time_to_solution(0.5, 12.3e-6) == pytest.approx(81.72e-6, abs=1e-8)
    assert nb.time_to_solution(0.0, 1.0) == float("inf")
    assert nb.time_to_solution(0.99, 1.0) == 1.0
    ps = np.linspace(1e-9, 1.0, 1000)
    tts = [nb.time_to_solution(float(p), 1.0) for p in ps]
    assert all(a >= b for a, b in zip(tts, tts[1:]))
    with pytest.raises(ValueError):
        nb.time_to_solution(1.5, 1.0)
    gt = nb.GroundTruth(-2.0, 1, "EXACT")
    rs = [solver.RunResult(np.ones(2), e, 0, 1.0) for e in (-2.0, -1.0, -2.0 + 1e-12, 0.0)]
    assert nb.success_probability(rs, gt) == 0.5
    st = nb.instance_stats(rs, gt, 1e-3)
    assert st.best_energy == -2.0 and st.p_success == 0.5


def test_accepts_reference_like_objects():
    class Ref:
        n = 3
        edges_i = np.array([0, 1])
        edges_j = np.array([1, 2])
        edge_weights = np.array([1.0, -1.0])
        h = np.zeros(3)
    p = nb.as_problem(Ref())
    assert isinstance(p, nb.IsingProblem) and p.num_edges == 2


def test_toroidal_grid_generator():
    """toroidal_grid: every spin has degree 4, 2*rows*cols couplers of +-1,
    deterministic in the seed (the torus bench workload)."""
    import paper_1806_08422_b200 as nb
    p = nb.toroidal_grid(7, 5, 3)
    deg = np.bincount(np.concatenate([p.edges_i, p.edges_j]), minlength=p.n)
    assert p.n == 35 and p.num_edges == 70 and np.all(deg == 4)
    assert set(np.unique(p.edge_weights)) <= {-1.0, 1.0}
    q = nb.toroidal_grid(7, 5, 3)
    assert np.array_equal(p.edge_weights, q.edge_weights)
    with pytest.raises(ValueError):
        nb.toroidal_grid(2, 5, 0)


def test_noise_mode_is_validated_before_any_device_work():
    import paper_1806_08422_b200 as nb
    p = nb.moebius_ladder(8)
    with pytest.raises(ValueError, match="noise must be one of"):
        nb.nmfa_batch(p, nb.NmfaParams(t_f=10), 4, noise="numpy")
    with pytest.raises(ValueError, match="noise must be one of"):
        nb.nmfa_run(p, nb.NmfaParams(t_f=10), noise=None)


def test_pack_sign_bits_layout_and_validation():
    rng = np.random.default_rng(0)
    n = 37
    J = np.triu(np.where(rng.random((n, n)) < 0.5, -1.0, 1.0), 1)
    J = J + J.T
    bits = nb.pack_sign_bits(J)
    assert bits.dtype == np.uint32 and bits.size == (n * n + 31) // 32
    p = nb.PackedSignProblem(n, bits)
    for i, j in [(0, 1), (3, 30), (36, 2), (10, 11)]:
        assert p.coupling(i, j) == J[i, j]
        b = min(i, j) * n + max(i, j)
        assert ((int(bits[b >> 5]) >> (b & 31)) & 1) == (J[i, j] > 0)
    iu = np.triu_indices(n, 1)
    assert p.w_total == J[iu].sum() and p.num_edges == n * (n - 1) // 2
    with pytest.raises(ValueError, match="symmetric"):
        nb.pack_sign_bits(np.triu(J))
    with pytest.raises(ValueError, match="uint32 words"):
        nb.PackedSignProblem(n, bits[:-1])


def test_packed_sign_problem_host_helpers():
    rng = np.random.default_rng(3)
    n = 50
    J = np.triu(np.where(rng.random((n, n)) < 0.5, -1.0, 1.0), 1)
    J = J + J.T
    h = rng.integers(-2, 3, n).astype(float)
    p = nb.PackedSignProblem.from_dense(J, h)
    s = rng.uniform(-1, 1, n)
    assert np.allclose(nb.mean_field(p, s), h + J @ s, atol=1e-12)
    assert np.allclose(nb.normalizers(p), np.sqrt(h * h + (J * J).sum(1)), atol=1e-12)
    assert np.allclose(p.normalizers_safe, np.sqrt(h * h + n - 1))
