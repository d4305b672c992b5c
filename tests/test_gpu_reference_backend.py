"""The B200 kernels behind the REFERENCE's own operator API.

The reference package, installed unmodified into baseline/_ref (git-ignored;
`pip install --no-deps --target baseline/_ref <reference>/pkg`), gets its
kernel backend pointed at paper_1806_08422_b200.kernels (three assignments,
kernels.py:30-32).  Its own entry points -- run_with_noise, nmfa_batch,
brute_force_ground -- then run on the GPU and are compared with the outputs
the reference produced with its numba backend (tests/golden/).  Skipped when
baseline/_ref is absent.
"""

import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)
if not os.path.isdir(os.path.join(REF, "nmfa")):
    pytest.skip("reference package not installed in baseline/_ref", allow_module_level=True)


@pytest.fixture(scope="module")
def nmfa():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_ref_backend")
    sys.path.insert(0, REF)
    import nmfa as ref

    from paper_1806_08422_b200 import kernels as b200
    b200.install(ref.kernels)
    assert ref.kernels.BACKEND == "b200"
    return ref


def load(name):
    return np.load(os.path.join(os.path.dirname(__file__), "golden", name))


def test_reference_run_with_noise_on_b200(nmfa):
    """solver.py:188-218 with caller noise: trajectories within the parity bound."""
    from nmfa.solver import DEFAULT_SCHEDULE, noise_stream
    T = load("trajectories.npz")
    specs = {"moebius16": nmfa.moebius_ladder(16), "sk30_s2": nmfa.gen_sk(30, 2),
             "cubic40_s1": nmfa.gen_cubic_maxcut(40, 1), "sk100_s0": nmfa.gen_sk(100, 0),
             "dense60_p03_s3": nmfa.gen_dense_maxcut(60, 0.3, 3)}
    for name, p in specs.items():
        t_f, seed = int(T[name + "_tf"]), int(T[name + "_seed"])
        temps = DEFAULT_SCHEDULE.temperatures(t_f)
        noise = noise_stream(seed).standard_normal((t_f, p.n)) * 0.15
        s, tr = nmfa.run_with_noise(p, temps, noise, 0.15, record_trajectory=True)
        ref = T[name + "_s"]
        # the backend runs the HILO field (the full state through the GEMM) and these
        # J are exact in fp16: within 1e-5 of the reference's float64 kernel
        assert np.max(np.abs(s - ref)) <= 1e-5, (name, np.max(np.abs(s - ref)))
        assert np.array_equal(np.sign(s), np.sign(ref)), name
        assert np.mean(tr.energies == T[name + "_e_hist"]) >= 0.99, name


def test_reference_nmfa_batch_on_b200(nmfa):
    """nmfa_batch (solver.py:262-280): same per-run numpy noise streams as the
    reference's numba run, so (HILO field) all but at most one run in 32 end
    in the same energy; every returned energy is the reference's own energy()
    of the returned config."""
    B = load("batches.npz")
    for name, p, t_f, R in [("moebius16_tf100", nmfa.moebius_ladder(16), 100, 100),
                            ("cubic40_tf300", nmfa.gen_cubic_maxcut(40, 1), 300, 32),
                            ("sk100_tf1000", nmfa.gen_sk(100, 0), 1000, 32)]:
        res = nmfa.nmfa_batch(p, nmfa.NmfaParams(t_f=t_f, seed=0), R)
        e = np.array([r.final_energy for r in res])
        assert [r.seed for r in res] == list(range(R))
        assert all(r.final_energy == nmfa.energy(p, r.final_config) for r in res)
        assert np.mean(e == B[name + "_E"]) >= 0.95, (name, np.mean(e == B[name + "_E"]))


def test_reference_brute_force_ground_on_b200(nmfa):
    G = load("ground.npz")
    for name in ["moebius16", "sk20_s3", "real16_h", "w2_18", "triangle"]:
        p = nmfa.IsingProblem(int(G[name + "_n"]),
                              list(zip(G[name + "_ei"], G[name + "_ej"], G[name + "_w"])),
                              h=G[name + "_h"])
        gt = nmfa.brute_force_ground(p)
        assert abs(gt.energy - float(G[name + "_E"])) <= 1e-9 and gt.degeneracy == int(G[name + "_deg"])


def test_reference_cli_runs_on_b200(nmfa, tmp_path):
    """The reference's own CLI (cli.py:384-406) end to end on the B200 backend:
    `generate` -> `exact` (gray_ground) and `bench` (nmfa_batch per instance +
    brute_force_ground), checked against this package's mirrors."""
    from nmfa import cli

    import paper_1806_08422_b200 as nb
    from paper_1806_08422_b200.experiments import bench
    inst = tmp_path / "sk14.txt"
    assert cli.main(["generate", "--class", "sk", "--n", "14", "--seed", "3", "--out", str(inst)]) == 0
    gt = nb.brute_force_ground(nb.load_gset(str(inst)))
    assert cli.main(["exact", str(inst)]) == 0
    out = tmp_path / "bench.csv"
    assert cli.main(["bench", "--class", "sk", "--sizes", "10,12", "--instances", "3", "--runs", "64",
                     "--out", str(out)]) == 0
    rows = [l.split(",") for l in out.read_text().strip().splitlines()]
    ours_rows, _, _ = bench("sk", [10, 12], 3, 64, nb.NmfaParams())
    assert rows[0][:4] == ["class", "n", "instances", "runs"]
    for ref_row, our_row in zip(rows[1:], ours_rows):
        assert ref_row[:4] == [str(x) for x in our_row[:4]]
        # small SK: both the reference pipeline on the B200 kernels and the batched
        # sampler find the exact ground state almost always
        assert float(ref_row[5]) >= 0.9 and float(our_row[5]) >= 0.9
    assert gt.source == "EXACT" and gt.degeneracy >= 2
