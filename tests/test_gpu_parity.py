"""GPU parity: the CUDA path through the C ABI against the reference-pinned oracle.

Tolerances: the device state is fp32 with an fp16
tensor-core operand, the reference is float64, so trajectories under the
same injected noise agree to |dS| <= 2e-3 (fp16-operand paths) / 1e-5 (fp32
sparse path) with identical final signs wherever the reference spin is not
within that bound of zero; energies are bit-exact for
integer weights; seeded statistics agree within binomial confidence bounds.
"""

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


def eprob(G, name):
    E = G["energies"]
    return nb.IsingProblem.from_arrays(int(E[name + "_n"]), E[name + "_ei"], E[name + "_ej"],
                                       E[name + "_w"], E[name + "_h"])


def oprob(G, name):
    E = G["energies"]
    return O.problem_from_edges(int(E[name + "_n"]), E[name + "_ei"], E[name + "_ej"],
                                E[name + "_w"], E[name + "_h"])


TRAJ = ["moebius16", "cubic40_s1", "sk30_s2", "dense60_p03_s3", "int40_h", "real24_h", "sk100_s0"]


def assert_traj_close(s_gpu, s_ref, tol=2e-2):
    s_gpu, s_ref = np.asarray(s_gpu), np.asarray(s_ref)
    assert np.max(np.abs(s_gpu - s_ref)) <= tol, np.max(np.abs(s_gpu - s_ref))
    firm = np.abs(s_ref) > tol
    assert np.array_equal(np.sign(s_gpu[firm]), np.sign(s_ref[firm]))


PATHS = ["small", "sparse", "dense"]


@pytest.mark.parametrize("name", TRAJ)
@pytest.mark.parametrize("path", PATHS)
def test_injected_noise_trajectory_matches_reference(G, name, path):
    T = G["trajectories"]
    p = eprob(G, name)
    p.device_handle().set_path(path)
    t_f, seed = int(T[name + "_tf"]), int(T[name + "_seed"])
    noise = O.run_noise(seed, t_f, p.n, 0.15)
    s, tr = nb.run_with_noise(p, O.temperatures(t_f), noise, 0.15, record_trajectory=True)
    # SURVEY 8(c) proposes max|dS| <= 1e-2 for N <= 500; measured on these fixtures
    # (tools/traj_fixture_maxds.py): <= 9.6e-4 with the fp16 GEMM operand (small,
    # dense), <= 2.5e-6 on the fp32 sparse path, so the bounds are 2e-3 and 1e-5
    tol = 1e-5 if path == "sparse" else 2e-3
    assert_traj_close(s, T[name + "_s"], tol)
    assert_traj_close(tr.spins[-10:], T[name + "_s_hist_last10"], tol)
    # trajectory energies are exact energies of the GPU's own rounded spins
    op = oprob(G, name)
    want = O.energies(op, O.sign_round(tr.spins))
    if op.edge_weights.dtype.kind == "f" and np.all(op.edge_weights == np.round(op.edge_weights)) \
            and np.all(op.h == np.round(op.h)):
        assert np.array_equal(tr.energies, want)
    else:
        assert np.allclose(tr.energies, want, rtol=1e-12, atol=1e-12)
    # ... and agree with the reference's trajectory energies at almost every step
    agree = np.mean(tr.energies == T[name + "_e_hist"]) if name != "real24_h" else \
        np.mean(np.isclose(tr.energies, T[name + "_e_hist"], rtol=1e-9))
    assert agree >= 0.9, agree


@pytest.mark.parametrize("name", ["moebius16", "cubic40_s1", "sk30_s2", "sk100_s0"])
@pytest.mark.parametrize("path", PATHS)
def test_noise_negation_is_exact(G, name, path):
    p = eprob(G, name)
    p.device_handle().set_path(path)
    noise = O.run_noise(3, 80, p.n, 0.15)
    temps = O.temperatures(80)
    s_pos, tp = nb.run_with_noise(p, temps, noise, 0.15, record_trajectory=True)
    s_neg, tn = nb.run_with_noise(p, temps, -noise, 0.15, record_trajectory=True)
    assert np.array_equal(s_neg, -s_pos)
    assert np.array_equal(tn.spins, -tp.spins)


def test_batched_noise_equals_single_runs(G):
    p = eprob(G, "sk30_s2")
    temps = O.temperatures(50)
    noise = np.stack([O.run_noise(s, 50, p.n, 0.15) for s in range(5)])
    S, _ = nb.run_with_noise(p, temps, noise, 0.15)
    for r in range(5):
        s1, _ = nb.run_with_noise(p, temps, noise[r], 0.15)
        assert np.array_equal(S[r], s1)


def test_identity_step_and_validation():
    p = nb.IsingProblem(2, [(0, 1, 1.0)])
    s0 = np.array([0.25, -0.5])
    s, _ = nb.run_with_noise(p, np.full(10, 0.5), np.zeros((10, 2)), 0.0, s0=s0)
    assert np.array_equal(s, s0)
    with pytest.raises(ValueError, match="noise shape"):
        nb.run_with_noise(p, np.array([1.0]), np.zeros((2, 2)), 0.15)
    with pytest.raises(ValueError, match="s0 length"):
        nb.run_with_noise(p, np.array([1.0]), np.zeros((1, 2)), 0.15, s0=np.zeros(3))
    with pytest.raises(ValueError):
        nb.nmfa_step(p, np.zeros(2), 0.0, nb.NmfaParams(), nb.noise_stream(0))
    with pytest.raises(ValueError):
        nb.nmfa_batch(p, nb.NmfaParams(), 0)


def test_tanh_kat(G):
    p = nb.IsingProblem(2, [(0, 1, 1.0)])
    out = nb.nmfa_step(p, np.array([0.9, 0.9]), 0.5, nb.NmfaParams(alpha=1.0, sigma=0.0, t_f=1),
                       nb.noise_stream(0))
    # 0.9 is not exact in the fp16 tensor-core operand (0.89990234): the step
    # is within 2^-11 relative of the reference, so the KAT tolerance is 5e-5
    # instead of the reference's 1e-5 (test_solver.py:115-121).
    assert out == pytest.approx([-0.94681, -0.94681], abs=5e-5)
    assert np.allclose(out, G["trajectories"]["kat_tanh"], atol=5e-5)
    # with an fp16-exact state the step is fp32-accurate
    out = nb.nmfa_step(p, np.array([0.875, 0.875]), 0.5, nb.NmfaParams(alpha=1.0, sigma=0.0, t_f=1),
                       nb.noise_stream(0))
    assert out == pytest.approx([-np.tanh(1.75)] * 2, abs=2e-7)


def test_zero_temperature_limit_and_boundedness():
    rng = np.random.Generator(np.random.Philox(key=12))
    cold = nb.NmfaParams(alpha=1.0, sigma=0.0, t_f=1)
    for trial in range(5):
        n = 25
        cpl = [(i, j, 1.0 if rng.random() < 0.5 else -1.0) for i in range(n) for j in range(i + 1, n)
               if rng.random() < 0.5]
        p = nb.IsingProblem(n, cpl)
        cfg = np.where(rng.random(n) < 0.5, 1.0, -1.0)
        phi = nb.mean_field(p, cfg)
        out = nb.nmfa_step(p, cfg, 1e-6, cold, nb.noise_stream(trial))
        nz = phi != 0.0
        assert np.all(np.abs(out[nz] + np.sign(phi[nz])) < 1e-7)   # fp32 state: 1e-9 -> 1e-7
        assert np.all(np.abs(out) < 1.0)
    # 20 random-temperature steps keep |s| < 1 strictly (acceptance criterion 2a)
    p = nb.gen_sk(20, 3)
    s = np.zeros(p.n)
    for k in range(20):
        T = float(np.exp(rng.uniform(np.log(0.02), np.log(2.0))))
        s = nb.nmfa_step(p, s, T, nb.NmfaParams(alpha=0.9, sigma=0.15, t_f=1), nb.noise_stream(k))
        assert np.all(np.abs(s) < 1.0)


def test_energies_bit_exact_against_reference(G):
    E = G["energies"]
    names = sorted({k[:-3] for k in E.files if k.endswith("_ei")})
    for name in names:
        p = eprob(G, name)
        got = nb.energies(p, E[name + "_cfg"].astype(np.float64))
        if name == "real24_h":
            assert np.allclose(got, E[name + "_E"], rtol=1e-12, atol=1e-12)
        else:
            assert np.array_equal(got, E[name + "_E"]), name
        if name + "_cut" in E:
            assert [nb.cut_value(p, c) for c in E[name + "_cfg"][:3]] == list(E[name + "_cut"][:3])


@pytest.mark.parametrize("path", PATHS)
def test_replica_sharding_invariance(G, path):
    p = {"small": lambda: nb.gen_sk(60, 1), "sparse": lambda: nb.gen_cubic_maxcut(300, 2),
         "dense": lambda: nb.gen_sk(300, 2)}[path]()
    p.device_handle().set_path(path)
    params = nb.NmfaParams(t_f=200, seed=11)
    full = nb.sample(p, params, 64, return_s=True)
    tail = nb.sample(p, params, 32, r0=32, return_s=True)
    assert torch.equal(full.configs[32:], tail.configs)
    assert torch.equal(full.energies[32:], tail.energies)
    assert torch.equal(full.s_final[32:], tail.s_final)
    # seed + k semantics (solver.py:272): batch(seed=100)[2] == run(seed=102)
    res = nb.nmfa_batch(p, nb.NmfaParams(t_f=50, seed=100), 5)
    solo = nb.nmfa_run(p, nb.NmfaParams(t_f=50, seed=102))
    assert [r.seed for r in res] == [100, 101, 102, 103, 104]
    assert np.array_equal(res[2].final_config, solo.final_config)
    assert res[2].final_energy == solo.final_energy


def test_dense_results_do_not_depend_on_the_schedule():
    """Exact fields (2^-11 operand grid, integer J): a different replica count
    gives a different tile schedule and per-tile K order, yet the replicas the
    two runs share must agree bit for bit."""
    p = nb.gen_sk(600, 3)
    assert p.device_info()["path"] == "dense"
    params = nb.NmfaParams(t_f=150, seed=4)
    full = nb.sample(p, params, 1280, return_s=True)
    tail = nb.sample(p, params, 256, r0=1024, return_s=True)
    assert torch.equal(full.configs[1024:], tail.configs)
    assert torch.equal(full.energies[1024:], tail.energies)
    assert torch.equal(full.s_final[1024:], tail.s_final)


def test_returned_energies_match_oracle_energy(G):
    p = nb.gen_sk(100, 0)
    op = O.problem_from_edges(100, p.edges_i, p.edges_j, p.edge_weights)
    res = nb.sample(p, nb.NmfaParams(t_f=300, seed=5), 512)
    cfg = res.configs.cpu().numpy().astype(np.float64)
    assert np.array_equal(res.energies.cpu().numpy(), O.energies(op, cfg))


def test_best_of_matches_numpy():
    e = torch.tensor([3.0, -1.0, 2.0, -1.0, -1.0, 5.0], dtype=torch.float64, device="cuda")
    ss = nb.SampleSet(None, e, 0, 7, 0.0)
    assert ss.best() == (-1.0, 8)
    big = torch.randint(-50, 50, (100001,), device="cuda").double()
    ss = nb.SampleSet(None, big, 0, 0, 0.0)
    be, bi = ss.best()
    arr = big.cpu().numpy()
    assert be == arr.min() and bi == int(np.argmin(arr))


def test_moebius16_reaches_ground(G):
    p = nb.moebius_ladder(16)
    res = nb.nmfa_batch(p, nb.NmfaParams(t_f=100, seed=0), 100)
    hits = sum(r.final_energy <= -20.0 + 1e-9 for r in res)
    assert hits >= 95      # reference: 1000/1000 at t_f=100 (stats.npz)
    traj = nb.nmfa_run(p, nb.NmfaParams(t_f=100, seed=0), record_trajectory=True).trajectory
    mag = np.abs(traj.spins).mean(axis=1)
    assert mag[0] < 0.2 and mag[-1] > 0.8 and mag[-1] > mag[50] > mag[0]


def test_host_entry_point_matches_device_api():
    import ctypes
    p = nb.gen_sk(50, 4)
    temps = nb.DEFAULT_SCHEDULE.temperatures(100)
    cfg = np.empty((16, 50), dtype=np.int8)
    en = np.empty(16)
    lib = _native.load()
    _native.check(lib.nmfa_anneal_host(p.device_handle().handle, 16, 100, _native.ptr(temps),
                                       0.15, 0.15, 9, 0, _native.ptr(cfg), _native.ptr(en)))
    res = nb.sample(p, nb.NmfaParams(t_f=100, seed=9), 16)
    assert np.array_equal(cfg, res.configs.cpu().numpy())
    assert np.array_equal(en, res.energies.cpu().numpy())
    assert ctypes.c_int64(lib.nmfa_last_launch_count()).value >= 1


def test_dense_large_injected_noise_matches_oracle():
    """n = 520 (not a multiple of 16/64), several replica blocks, dense tcgen05 path."""
    p = nb.gen_sk(520, 5)
    assert p.device_info()["path"] == "dense"
    op = O.problem_from_edges(520, p.edges_i, p.edges_j, p.edge_weights)
    t_f, R = 120, 300
    temps = O.temperatures(t_f)
    rng = np.random.Generator(np.random.Philox(key=99))
    noise = rng.standard_normal((R, t_f, p.n)) * 0.15
    S, _ = nb.run_with_noise(p, temps, noise, 0.15)
    Sref = O.batched_anneal(op, None, t_f=t_f, temps=temps, noise=noise)
    err = np.abs(S - Sref)
    # SURVEY 8c parity criterion for large n: mean over replicas of <= 0.1% spins with a
    # different final sign (fp16 operand rounding occasionally flips a correlated cluster).
    flips = np.mean(np.sign(S) != np.sign(Sref))
    print(f"n=520 dense: mean|dS|={err.mean():.2e} frac(|dS|>2e-2)={np.mean(err > 2e-2):.2e} "
          f"sign flips={flips:.2e}")
    assert np.mean(err) < 1e-3 and np.mean(err > 2e-2) < 5e-3, (np.mean(err), err.max())
    assert flips <= 1e-3, flips


def test_host_entry_is_thread_safe():
    """Concurrent nmfa_anneal_host calls on one problem (different read counts,
    so the cached buffers are resized) give the same results as sequential ones."""
    import ctypes
    import threading

    from paper_1806_08422_b200 import _native
    p = nb.gen_sk(120, 4)
    params = nb.NmfaParams(t_f=100, seed=9)
    temps = np.ascontiguousarray(params.schedule.temperatures(params.t_f))
    lib = _native.load()
    h = p.device_handle().handle

    def call(R, seed):
        cfg = np.empty((R, p.n), np.int8)
        e = np.empty(R)
        _native.check(lib.nmfa_anneal_host(h, R, params.t_f, _native.ptr(temps), params.alpha,
                                           params.sigma, seed, 0, _native.ptr(cfg), _native.ptr(e)))
        return cfg, e

    jobs = [(256 + 128 * (k % 3), 100 + k) for k in range(8)]
    want = [call(R, s) for R, s in jobs]
    got = [None] * len(jobs)

    def worker(k):
        got[k] = call(*jobs[k])

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(len(jobs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for (wc, we), (gc, ge) in zip(want, got):
        assert np.array_equal(wc, gc) and np.array_equal(we, ge)


def test_dense_and_bit_constructors_equal_edge_list():
    """nmfa_problem_create_dense / _dense_bits build the same problem as the
    edge list: same info and bit-identical anneals (plan_run on each handle)."""
    import ctypes

    from paper_1806_08422_b200 import _native
    lib = _native.load()
    n = 300
    p = nb.gen_sk(n, 6)
    J = np.zeros((n, n))
    J[p.edges_i, p.edges_j] = p.edge_weights
    J = J + J.T
    bits = np.zeros((n * n + 31) // 32, np.uint32)
    for i, j, w in zip(p.edges_i, p.edges_j, p.edge_weights):
        if w > 0:
            b = int(i) * n + int(j)
            bits[b >> 5] |= np.uint32(1 << (b & 31))
    hd, hb = ctypes.c_void_p(), ctypes.c_void_p()
    _native.check(lib.nmfa_problem_create_dense(n, _native.ptr(np.ascontiguousarray(J)), None, 0,
                                                ctypes.byref(hd)))
    _native.check(lib.nmfa_problem_create_dense_bits(n, _native.ptr(bits), None, 0, ctypes.byref(hb)))
    hc = ctypes.c_void_p()
    ip, ix, wx = (np.ascontiguousarray(p.csr_indptr, np.int64), np.ascontiguousarray(p.csr_indices, np.int64),
                  np.ascontiguousarray(p.csr_weights, np.float64))
    _native.check(lib.nmfa_problem_create_csr(n, _native.ptr(ip), _native.ptr(ix), _native.ptr(wx), None,
                                              0, ctypes.byref(hc)))
    params = nb.NmfaParams(t_f=80, seed=2)
    temps = np.ascontiguousarray(params.schedule.temperatures(params.t_f))
    outs = []
    for h in (p.device_handle().handle, hd, hb, hc):
        cfg = torch.empty((256, n), dtype=torch.int8, device="cuda")
        e = torch.empty(256, dtype=torch.float64, device="cuda")
        _native.check(lib.nmfa_anneal(h, 256, params.t_f, _native.ptr(temps), params.alpha,
                                      params.sigma, params.seed, 0, None, None, _native.ptr(cfg),
                                      _native.ptr(e), None, None, None, None))
        outs.append((cfg, e))
    for cfg, e in outs[1:]:
        assert torch.equal(cfg, outs[0][0]) and torch.equal(e, outs[0][1])
    lib.nmfa_problem_destroy(hd)
    lib.nmfa_problem_destroy(hb)
    lib.nmfa_problem_destroy(hc)
    bad = np.eye(3)
    assert lib.nmfa_problem_create_dense(3, _native.ptr(bad), None, 0, ctypes.byref(hd)) == 1


RAGGED = [(17, 1), (100, 37), (129, 256), (255, 300), (256, 257), (257, 64), (383, 513), (640, 5)]


@pytest.mark.parametrize("path", PATHS)
@pytest.mark.parametrize("n,R", RAGGED)
def test_ragged_shapes_match_oracle(path, n, R):
    """Boundary sizes on every kernel path (n around the 16 / 128 / 256 tile
    edges, partial replica blocks, a single replica): injected-noise trajectories
    within the parity bound of the float64 oracle, energies exact."""
    if path == "small" and n > 256:
        pytest.skip("the small path holds n <= 256")
    rng = np.random.default_rng(n * 1000 + R)
    p = nb.gen_sk(n, n) if n <= 300 else nb.gen_dense_maxcut(n, 0.05, n)
    p.device_handle().set_path(path)
    t_f = 40
    temps = O.temperatures(t_f)
    noise = rng.standard_normal((R, t_f, n)) * 0.15
    S, _ = nb.run_with_noise(p, temps, noise, 0.15)
    S = np.atleast_2d(S)
    op = O.problem_from_edges(n, p.edges_i, p.edges_j, p.edge_weights)
    ref = np.stack([O.anneal(op, np.zeros(n), temps, noise[r], 0.15)[0] for r in range(R)])
    err = np.abs(S - ref)
    # SURVEY 8c for many replicas: fp16-operand rounding occasionally pushes a
    # single near-critical element off (n=129: 1 of 33k elements, replica 75 spin 74,
    # on both fp16 paths; tools/diag_ragged.py), so the bound is statistical
    assert err.mean() < 1e-3 and np.mean(err > 2e-2) <= 1e-3, (err.mean(), np.mean(err > 2e-2))
    firm = np.abs(ref) > 2e-2
    assert np.mean(np.sign(S[firm]) != np.sign(ref[firm])) <= 1e-3
    cfg = O.sign_round(S)
    assert np.array_equal(nb.energies(p, cfg), O.energies(op, cfg))


@pytest.mark.parametrize("path", PATHS)
def test_problem_without_couplers(path):
    """No couplers: norm_safe = 1 (problem.py:90-95), the field is the noise
    alone, every configuration has energy h . c."""
    n = 300 if path != "small" else 40
    h = np.linspace(-1.0, 1.0, n)
    p = nb.IsingProblem(n, [], h=h)
    p.device_handle().set_path(path)
    t_f, R = 30, 64
    temps = O.temperatures(t_f)
    noise = np.random.default_rng(5).standard_normal((R, t_f, n)) * 0.15
    S, _ = nb.run_with_noise(p, temps, noise, 0.15)
    op = O.problem_from_edges(n, [], [], [], h)
    ref = np.stack([O.anneal(op, np.zeros(n), temps, noise[r], 0.15)[0] for r in range(R)])
    assert np.abs(S - ref).max() <= 2e-2
    res = nb.sample(p, nb.NmfaParams(t_f=50, seed=1), 128)
    cfg = res.configs.cpu().numpy().astype(np.float64)
    assert np.allclose(res.energies.cpu().numpy(), cfg @ h, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("path,make", [("small", lambda: nb.gen_sk(60, 1)),
                                       ("dense", lambda: nb.gen_sk(300, 2)),
                                       ("sparse", lambda: nb.moebius_ladder(520)),
                                       ("sparse", lambda: nb.gen_dense_maxcut(400, 0.02, 1))])
def test_plan_run_is_graph_capturable(path, make):
    """nmfa_plan_run allocates nothing and only enqueues (include/nmfa_b200.h):
    captured in a CUDA graph and replayed, it reproduces a direct run bitwise."""
    p = make()
    p.device_handle().set_path(path)
    params = nb.NmfaParams(t_f=40, seed=9)
    R = 96
    plan = nb.Plan(p, R, params.schedule.temperatures(params.t_f), params.alpha, params.sigma)
    cfg0 = torch.empty((R, p.n), dtype=torch.int8, device="cuda")
    e0 = torch.empty(R, dtype=torch.float64, device="cuda")
    plan.run(params.seed, 0, config=cfg0, energy=e0)
    torch.cuda.synchronize()
    cfg1 = torch.zeros_like(cfg0)
    e1 = torch.zeros_like(e0)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        plan.run(params.seed, 0, config=cfg1, energy=e1, stream=s)  # warm-up on the side stream
        torch.cuda.synchronize()
        cfg1.zero_()
        e1.zero_()
        with torch.cuda.graph(g, stream=s):
            plan.run(params.seed, 0, config=cfg1, energy=e1, stream=s)
    torch.cuda.synchronize()
    for _ in range(2):
        cfg1.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(cfg1, cfg0) and torch.equal(e1, e0)
