"""The ELL sparse kernel (graphs of max degree <= 4) against the CSR kernel.

Both kernels sum each row in CSR order from +0, and the ELL pads are (own
index, weight 0), so the two must agree BIT-EXACTLY on every graph: regular
degree 3 and 4, mixed degrees with padded rows, isolated spins, n not a
multiple of 8, one or two replicas per lane, injected and in-kernel noise,
trajectories. NMFA_SPARSE_CSR=1 forces the CSR kernel (anneal_sparse.cu).
The CSR kernel itself is pinned to the oracle by test_gpu_parity.py.
"""

import os

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


def torus(rows, cols):
    """2-D toroidal grid (G-set's degree-4 class), +-1 couplers."""
    v = np.arange(rows * cols).reshape(rows, cols)
    a = np.concatenate([v.ravel(), v.ravel()])
    b = np.concatenate([np.roll(v, -1, 1).ravel(), np.roll(v, -1, 0).ravel()])
    w = np.where(np.random.default_rng(rows * cols).random(a.size) < 0.5, 1.0, -1.0)
    return nb.IsingProblem.from_arrays(rows * cols, np.minimum(a, b), np.maximum(a, b), w)


def mixed(n, seed, h=False):
    """Random graph of max degree 3 with degree-0/1/2 spins and real weights."""
    rng = np.random.default_rng(seed)
    deg = np.zeros(n, dtype=int)
    pairs = set()
    for _ in range(n):
        i, j = rng.integers(0, n, 2)
        if i != j and deg[i] < 3 and deg[j] < 3 and (min(i, j), max(i, j)) not in pairs:
            pairs.add((min(i, j), max(i, j)))
            deg[i] += 1
            deg[j] += 1
    e = np.array(sorted(pairs))
    hv = rng.normal(size=n) if h else None
    return nb.IsingProblem.from_arrays(n, e[:, 0], e[:, 1], rng.normal(size=len(e)), hv)


def random_degree(n, d, seed):
    """About n*d/2 distinct random couplers (mean degree ~d), +1 weights."""
    rng = np.random.default_rng(seed)
    a = rng.integers(0, n, n * d // 2)
    b = rng.integers(0, n, n * d // 2)
    keep = a != b
    key = np.unique(np.minimum(a, b)[keep] * n + np.maximum(a, b)[keep])
    return nb.IsingProblem.from_arrays(n, key // n, key % n, np.ones(key.size))


GRAPHS = {
    "moebius_1000": lambda: nb.moebius_ladder(1000),
    "cubic_302": lambda: nb.gen_cubic_maxcut(302, 4),
    "torus_13x11": lambda: torus(13, 11),
    "mixed_301_h": lambda: mixed(301, 7, h=True),
    "mixed_77": lambda: mixed(77, 3),
}


def _both(fn):
    old = os.environ.get("NMFA_SPARSE_CSR")
    try:
        os.environ["NMFA_SPARSE_CSR"] = "1"
        csr = fn()
        os.environ["NMFA_SPARSE_CSR"] = "0"
        ell = fn()
    finally:
        if old is None:
            os.environ.pop("NMFA_SPARSE_CSR", None)
        else:
            os.environ["NMFA_SPARSE_CSR"] = old
    return csr, ell


@pytest.mark.parametrize("graph", sorted(GRAPHS))
@pytest.mark.parametrize("R", [1, 37, 64, 96, 300])  # 1 and 96: one replica per lane
def test_ell_equals_csr_seeded(graph, R):
    p = GRAPHS[graph]()
    p.device_handle().set_path("sparse")
    params = nb.NmfaParams(t_f=60, seed=11)

    def run():
        res = nb.sample(p, params, R)
        return res.configs.cpu().numpy(), res.energies.cpu().numpy()

    (c0, e0), (c1, e1) = _both(run)
    assert np.array_equal(c0, c1) and np.array_equal(e0, e1)


@pytest.mark.parametrize("graph", sorted(GRAPHS))
def test_ell_equals_csr_injected_trajectory(graph):
    p = GRAPHS[graph]()
    p.device_handle().set_path("sparse")
    t_f, R = 25, 5
    temps = O.temperatures(t_f)
    noise = np.random.default_rng(1).standard_normal((R, t_f, p.n)) * 0.15

    def run():
        s, trs = nb.run_with_noise(p, temps, noise, 0.15, record_trajectory=True)
        return s, np.stack([tr.spins for tr in trs])

    (s0, h0), (s1, h1) = _both(run)
    assert np.array_equal(s0, s1) and np.array_equal(h0, h1)


def test_ell_torus_matches_oracle():
    """Degree-4 ELL rows against the float64 oracle under injected noise."""
    p = torus(16, 9)
    p.device_handle().set_path("sparse")
    t_f, R = 40, 33
    temps = O.temperatures(t_f)
    noise = np.random.default_rng(2).standard_normal((R, t_f, p.n)) * 0.15
    S, _ = nb.run_with_noise(p, temps, noise, 0.15)
    op = O.problem_from_edges(p.n, p.edges_i, p.edges_j, p.edge_weights)
    ref = np.stack([O.anneal(op, np.zeros(p.n), temps, noise[r], 0.15)[0] for r in range(R)])
    assert np.abs(S - ref).max() <= 2e-2
    firm = np.abs(ref) > 2e-2
    assert np.array_equal(np.sign(S[firm]), np.sign(ref[firm]))


@pytest.mark.parametrize("make,path,slots", [
    (lambda: nb.gen_cubic_maxcut(512, 1), "sparse", 3),
    (lambda: nb.moebius_ladder(1000), "sparse", 3),
    (lambda: torus(23, 23), "sparse", 4),
    (lambda: mixed(301, 7), "sparse", 3),
    (lambda: nb.gen_dense_maxcut(2000, 0.01, 7), "dense", 0),     # G2000 stand-in (C4)
    (lambda: random_degree(16384, 10, 1), "sparse", 0),  # n^2 > 611 nnz: CSR
    (lambda: random_degree(8192, 10, 1), "sparse", 0),
    (lambda: random_degree(8192, 20, 1), "dense", 0),
    (lambda: random_degree(4096, 10, 1), "dense", 0),
])
def test_path_router(make, path, slots):
    """capi.cu prefer_dense, refit from profiles/r01/path_crossover.log: max degree
    <= 4 always takes the ELL kernel; otherwise dense while n^2 < 611 nnz."""
    info = make().device_info()
    assert info["path"] == path and info["ell_slots"] == slots, info


@pytest.mark.parametrize("integer_h", [True, False])
def test_energy_field_term_in_chunks(integer_h):
    """n = 5000 > 2048: the field term h.c runs as three spin chunks
    (energy.cu). Integer fields stay bit-exact; real fields within 1e-12."""
    n = 5000
    rng = np.random.default_rng(3)
    base = nb.gen_cubic_maxcut(n, 2)
    h = rng.integers(-3, 4, n).astype(np.float64) if integer_h else rng.normal(size=n)
    p = nb.IsingProblem.from_arrays(n, base.edges_i, base.edges_j, base.edge_weights, h)
    res = nb.sample(p, nb.NmfaParams(t_f=30, seed=4), 96)
    cfg = res.configs.cpu().numpy().astype(np.float64)
    op = O.problem_from_edges(n, p.edges_i, p.edges_j, p.edge_weights, h)
    want = O.energies(op, cfg)
    got = res.energies.cpu().numpy()
    if integer_h:
        assert np.array_equal(got, want)
    else:
        assert np.allclose(got, want, rtol=1e-12, atol=1e-9)


def test_graph_replay_equals_direct_launches():
    """The sparse path replays its t_f steps from a per-plan CUDA graph; the key
    base, s0 and the last step's outputs change per run (init / last node
    re-pointed). Runs of one plan with changing seeds, outputs and s0 must equal
    direct stream launches (NMFA_SPARSE_GRAPH=0) bit for bit."""
    p = nb.gen_cubic_maxcut(300, 3)
    p.device_handle().set_path("sparse")
    params = nb.NmfaParams(t_f=50, seed=1)
    R = 128
    plan = nb.Plan(p, R, params.schedule.temperatures(params.t_f), params.alpha, params.sigma)
    s0 = torch.as_tensor(np.random.default_rng(0).uniform(-0.5, 0.5, (R, p.n)),
                         dtype=torch.float32, device="cuda")
    runs = [(1, None), (2, s0), (1, None), (3, s0), (3, None)]

    def go():
        outs = []
        for seed, init in runs:
            cfg = torch.empty((R, p.n), dtype=torch.int8, device="cuda")  # fresh buffers
            sf = torch.empty((R, p.n), dtype=torch.float32, device="cuda")
            plan.run(seed, 0, s0=init, config=cfg, s_final=sf)
            torch.cuda.synchronize()
            outs.append((cfg.cpu(), sf.cpu()))
        return outs

    old = os.environ.get("NMFA_SPARSE_GRAPH")
    try:
        os.environ["NMFA_SPARSE_GRAPH"] = "1"
        graph = go()
        os.environ["NMFA_SPARSE_GRAPH"] = "0"
        direct = go()
    finally:
        if old is None:
            os.environ.pop("NMFA_SPARSE_GRAPH", None)
        else:
            os.environ["NMFA_SPARSE_GRAPH"] = old
    for (c1, s1), (c2, s2) in zip(graph, direct):
        assert torch.equal(c1, c2) and torch.equal(s1, s2)
    assert torch.equal(graph[0][0], graph[2][0]) and not torch.equal(graph[0][0], graph[1][0])


def test_sample_many_on_the_sparse_path_equals_single_runs():
    """nmfa_anneal_many with instances above the small-path size loops over the
    per-problem plans (sparse graph replay here); each instance must equal its
    own sample() call with the bench-loop seed."""
    from dataclasses import replace
    probs = [nb.gen_cubic_maxcut(400, s) for s in range(3)] + [mixed(400, 9)]
    params = nb.NmfaParams(t_f=40, seed=21)
    R = 64
    cfg, en, _ = nb.sample_many(probs, params, R)
    for k, p in enumerate(probs):
        assert p.device_info()["path"] == "sparse"
        one = nb.sample(p, replace(params, seed=params.seed + k * R), R)
        assert torch.equal(cfg[k], one.configs) and torch.equal(en[k], one.energies)
