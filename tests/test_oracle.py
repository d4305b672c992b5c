"""The CPU oracle is pinned to golden vectors produced by the reference itself."""

import hashlib

import numpy as np
import pytest

import nmfa_oracle as O
from conftest import golden


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def prob(E, name):
    h = E[name + "_h"] if name + "_h" in E else None
    return O.problem_from_edges(int(E[name + "_n"]) if name + "_n" in E else None,
                                E[name + "_ei"], E[name + "_ej"], E[name + "_w"], h)


@pytest.mark.parametrize("t_f", [1, 2, 37, 101, 1000])
def test_schedule_matches_reference(G, t_f):
    assert np.array_equal(O.temperatures(t_f), G["schedule"][f"default_{t_f}"])


def test_custom_schedules(G):
    assert np.array_equal(O.temperatures(3, ((0.0, 1.0), (1.0, 0.01))), G["schedule"]["custom_3"])
    assert np.array_equal(O.temperatures(50, ((0.0, 2.0), (0.3, 0.7), (1.0, 0.02))),
                          G["schedule"]["custom3pt_50"])


def test_noise_stream_identity(G):
    assert np.array_equal(O.noise_stream(5).standard_normal((3, 4)), G["noise"]["seed5"])
    assert np.array_equal(O.run_noise(0, 2, 100, 0.15), G["noise"]["seed0_sigma"])


def test_energy_golden(G):
    E = G["energies"]
    names = sorted({k[:-3] for k in E.files if k.endswith("_ei")})
    assert len(names) >= 8
    for name in names:
        p = O.problem_from_edges(int(E[name + "_n"]), E[name + "_ei"], E[name + "_ej"],
                                 E[name + "_w"], E[name + "_h"])
        cfg = E[name + "_cfg"].astype(np.float64)
        got = O.energies(p, cfg)
        want = E[name + "_E"]
        if np.all(p.edge_weights == np.round(p.edge_weights)) and np.all(p.h == np.round(p.h)):
            assert np.array_equal(got, want), name
        else:
            assert np.allclose(got, want, rtol=1e-12, atol=1e-12), name
        assert all(O.energy(p, c) == w for c, w in zip(cfg, want)), name
        if name + "_cut" in E:
            assert np.array_equal([O.cut_value(p, c) for c in cfg], E[name + "_cut"])


def test_instances_normalizers(G):
    I = G["instances"]
    for name in ("sk100_s0", "sk30_s2", "moebius16", "moebius100", "cubic40_s1", "dense60_p03_s3"):
        n = int(max(I[name + "_ei"].max(), I[name + "_ej"].max())) + 1
        p = O.problem_from_edges(n, I[name + "_ei"], I[name + "_ej"], I[name + "_w"])
        assert np.array_equal(p.normalizers_safe, I[name + "_norm"])
        assert bool(p.is_dense) == bool(I[name + "_is_dense"])


def test_oracle_generators_match_reference(G):
    I = G["instances"]
    ii, jj, w = O.gen_sk_edges(100, 0)
    assert np.array_equal(ii, I["sk100_s0_ei"]) and np.array_equal(w, I["sk100_s0_w"])
    ii, jj, w = O.gen_sk_edges(2000, 7)
    assert sha(w) == str(I["sk2000_s7_sha_w"])
    ii, jj, w = O.moebius_edges(100)
    p = O.problem_from_edges(100, ii, jj, w)
    assert np.array_equal(p.edges_i, I["moebius100_ei"])


def _traj_problem(G, name):
    src = G["energies"]
    return O.problem_from_edges(int(src[name + "_n"]), src[name + "_ei"], src[name + "_ej"],
                                src[name + "_w"], src[name + "_h"])


@pytest.mark.parametrize("name", ["moebius16", "cubic40_s1", "sk30_s2", "dense60_p03_s3",
                                  "int40_h", "real24_h"])
def test_run_with_noise_matches_reference(G, name):
    T = G["trajectories"]
    p = _traj_problem(G, name)
    t_f, seed = int(T[name + "_tf"]), int(T[name + "_seed"])
    noise = O.run_noise(seed, t_f, p.n, 0.15)
    s, sh, eh = O.anneal(p, np.zeros(p.n), O.temperatures(t_f), noise, 0.15, record=True)
    assert np.allclose(s, T[name + "_s"], rtol=0, atol=1e-10)
    assert np.allclose(sh[-10:], T[name + "_s_hist_last10"], rtol=0, atol=1e-10)
    if name == "real24_h":   # dense record path sums 0.5 r.(J r) + h.r (_kernels_numba.py:78)
        assert np.allclose(eh, T[name + "_e_hist"], rtol=1e-12, atol=1e-12)
    else:
        assert np.array_equal(eh, T[name + "_e_hist"])


def test_run_with_noise_sk100_long(G):
    T = G["trajectories"]
    p = _traj_problem(G, "sk100_s0")
    noise = O.run_noise(7, 1000, p.n, 0.15)
    s, _, _ = O.anneal(p, np.zeros(p.n), O.temperatures(1000), noise, 0.15)
    assert np.allclose(s, T["sk100_s0_s"], rtol=0, atol=1e-9)
    assert np.array_equal(O.sign_round(s), O.sign_round(T["sk100_s0_s"]))


@pytest.mark.parametrize("jit", [False, True])
def test_batch_matches_reference_seeded(G, jit):
    B = G["batches"]
    I = G["instances"]
    p = O.problem_from_edges(16, I["moebius16_ei"], I["moebius16_ej"], I["moebius16_w"])
    cfg, e = O.batch(p, 0, 100, t_f=100, threads=4, jit=jit)
    assert np.array_equal(e, B["moebius16_tf100_E"])
    assert np.array_equal(cfg.astype(np.int8), B["moebius16_tf100_cfg"])
    p = O.problem_from_edges(100, I["sk100_s0_ei"], I["sk100_s0_ej"], I["sk100_s0_w"])
    cfg, e = O.batch(p, 0, 8, t_f=1000, threads=4, jit=jit)
    assert np.array_equal(e, B["sk100_tf1000_E"][:8])


def test_jit_loop_matches_numpy_loop(G):
    I = G["instances"]
    for name, n in (("cubic40_s1", 40), ("sk30_s2", 30)):
        p = O.problem_from_edges(n, I[name + "_ei"], I[name + "_ej"], I[name + "_w"])
        noise = O.run_noise(4, 200, n, 0.15)
        a = O.anneal(p, np.zeros(n), O.temperatures(200), noise, 0.15)[0]
        b = O.anneal_fast(p, np.zeros(n), O.temperatures(200), noise, 0.15)
        assert np.allclose(a, b, rtol=0, atol=1e-10)


def test_batched_restatement_equals_reference_energies(G):
    B = G["batches"]
    I = G["instances"]
    p = O.problem_from_edges(100, I["sk100_s0_ei"], I["sk100_s0_ej"], I["sk100_s0_w"])
    S = O.batched_anneal(p, list(range(32)), t_f=1000)
    e = O.energies(p, O.sign_round(S))
    assert np.array_equal(e, B["sk100_tf1000_E"])


def test_tts_and_stats_kats(G):
    assert O.time_to_solution(0.5, 12.3e-6) == pytest.approx(81.72e-6, abs=1e-8)
    assert O.time_to_solution(0.5, 12.3e-6) == float(G["stats"]["tts_kat"])
    S = G["stats"]
    assert float(S["moebius16_ground"]) == -20.0
    assert S["sk100_E"].min() == -730.0
    p = O.success_probability(S["sk100_E"], -730.0)
    assert p == pytest.approx(0.2334, abs=1e-4)
    lo, hi = O.wilson_interval(int(round(p * 10000)), 10000)
    assert lo < p < hi and hi - lo < 0.02


def test_large_reference_samples_are_pinned_to_nmfa_batch():
    """stats_large.npz (make_golden_stats.py: the reference's streams and
    arithmetic, replica-batched) agrees with the reference's own nmfa_batch
    energies (stats.npz) on every seed the two share."""
    big, small = golden("stats_large.npz"), golden("stats.npz")
    sizes = {"sk100": 65536, "moebius100": 32768, "g2000": 32768, "sk2000": 16384}
    for name, size in sizes.items():
        same, m = big[name + "_same_as_nmfa_batch"]
        assert same == m and m >= 64, name
        assert big[name + "_E"].size == size and int(big[name + "_t_f"]) == 1000
        assert np.array_equal(big[name + "_E"][:m].astype(np.float64), small[name + "_E"][:m])
