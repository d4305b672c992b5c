"""Generate golden fixtures by running the REFERENCE package itself.

Runs only in the build container, where the read-only reference lives at
/root/reference (it does not exist on the GPU box).  Outputs go to
tests/golden/*.npz and are committed; tests never import the reference.

    OPENBLAS_NUM_THREADS=1 NUMBA_CACHE_DIR=/tmp/nb python tests/golden/make_golden.py

Every fixture records which reference call produced it (file:line in the
reference package under pkg/src/nmfa/).
"""

import hashlib
import os
import sys
import time

os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, "/root/reference/pkg/src")

import numpy as np  # noqa: E402

import nmfa  # noqa: E402
from nmfa import kernels  # noqa: E402
from nmfa.solver import DEFAULT_SCHEDULE, noise_stream, run_with_noise  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
THREADS = os.cpu_count() or 8


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def edges(p):
    return p.edges_i.astype(np.int32), p.edges_j.astype(np.int32), p.edge_weights.copy()


def save(name, **kw):
    np.savez_compressed(os.path.join(OUT, name), **kw)
    print("wrote", name, sorted(kw))


def instances():
    """Generator outputs (generators.py:27-86) and problem arithmetic (problem.py)."""
    out = {}
    specs = {
        "sk100_s0": nmfa.gen_sk(100, 0),
        "sk30_s2": nmfa.gen_sk(30, 2),
        "moebius16": nmfa.moebius_ladder(16),
        "moebius100": nmfa.moebius_ladder(100),
        "cubic40_s1": nmfa.gen_cubic_maxcut(40, 1),
        "dense60_p03_s3": nmfa.gen_dense_maxcut(60, 0.3, 3),
    }
    for k, p in specs.items():
        ei, ej, w = edges(p)
        out[k + "_ei"], out[k + "_ej"], out[k + "_w"] = ei, ej, w
        out[k + "_norm"] = p.normalizers_safe.copy()
        out[k + "_is_dense"] = np.array(p.is_dense)
    # large stand-ins: store only checksums + counts (calibrate.py:41,44)
    for k, p in {"sk2000_s7": nmfa.gen_sk(2000, 7),
                 "g2000_p001_s7": nmfa.gen_dense_maxcut(2000, 0.01, 7)}.items():
        ei, ej, w = edges(p)
        out[k + "_nedges"] = np.array(ei.size)
        out[k + "_sha_ei"] = np.array(sha(ei.astype(np.int64)))
        out[k + "_sha_ej"] = np.array(sha(ej.astype(np.int64)))
        out[k + "_sha_w"] = np.array(sha(w))
        out[k + "_is_dense"] = np.array(p.is_dense)
    return specs, out


def main():
    t0 = time.time()
    print("reference backend:", kernels.BACKEND)
    specs, inst = instances()
    save("instances.npz", **inst)

    # ---- schedule (solver.py:70-84) ----
    sched = {}
    for t_f in (1, 2, 37, 101, 1000):
        sched[f"default_{t_f}"] = DEFAULT_SCHEDULE.temperatures(t_f)
    custom = nmfa.Schedule([(0.0, 1.0), (1.0, 0.01)])
    sched["custom_3"] = custom.temperatures(3)
    sched["custom3pt_50"] = nmfa.Schedule([(0.0, 2.0), (0.3, 0.7), (1.0, 0.02)]).temperatures(50)
    save("schedule.npz", **sched)

    # ---- noise stream identity (solver.py:182-185) ----
    save("noise.npz", seed5=noise_stream(5).standard_normal((3, 4)),
         seed0_sigma=noise_stream(0).standard_normal((2, 100)) * 0.15)

    # ---- energies of random configs (problem.py:150-154), incl. int h and real weights ----
    rng = np.random.Generator(np.random.Philox(key=424242))
    en = {}
    probs = dict(specs)
    # integer weights + integer fields
    n = 40
    cpl = [(i, j, float(rng.integers(1, 6)) * (1.0 if rng.random() < 0.5 else -1.0))
           for i in range(n) for j in range(i + 1, n) if rng.random() < 0.6]
    probs["int40_h"] = nmfa.IsingProblem(n, cpl, h=rng.integers(-3, 4, size=n).astype(float))
    # real weights + real fields
    n = 24
    cpl = [(i, j, float(rng.standard_normal())) for i in range(n) for j in range(i + 1, n)
           if rng.random() < 0.6]
    probs["real24_h"] = nmfa.IsingProblem(n, cpl, h=rng.standard_normal(n))
    for k, p in probs.items():
        cfgs = np.where(rng.random((16, p.n)) < 0.5, 1.0, -1.0)
        en[k + "_cfg"] = cfgs.astype(np.int8)
        en[k + "_E"] = np.array([nmfa.energy(p, c) for c in cfgs])
        en[k + "_h"] = p.h.copy()
        ei, ej, w = edges(p)
        en[k + "_ei"], en[k + "_ej"], en[k + "_w"] = ei, ej, w
        en[k + "_n"] = np.array(p.n)
        if not np.any(p.h != 0):
            en[k + "_cut"] = np.array([nmfa.cut_value(p, c) for c in cfgs])
    save("energies.npz", **en)

    # ---- run_with_noise trajectories (solver.py:188-218), injected noise ----
    traj = {}
    cases = [("moebius16", 100, 33), ("cubic40_s1", 80, 1), ("sk30_s2", 80, 2),
             ("sk100_s0", 1000, 7), ("dense60_p03_s3", 200, 4), ("int40_h", 150, 9),
             ("real24_h", 120, 11)]
    for name, t_f, seed in cases:
        p = probs[name]
        temps = DEFAULT_SCHEDULE.temperatures(t_f)
        noise = noise_stream(seed).standard_normal((t_f, p.n)) * 0.15
        s, tr = run_with_noise(p, temps, noise, 0.15, record_trajectory=True)
        traj[name + "_tf"] = np.array(t_f)
        traj[name + "_seed"] = np.array(seed)
        traj[name + "_s"] = s
        traj[name + "_e_hist"] = tr.energies
        traj[name + "_s_hist_sha"] = np.array(sha(tr.spins))
        traj[name + "_s_hist_last10"] = tr.spins[-10:]
    # single-step KATs (test_solver.py:115-121)
    p2 = nmfa.IsingProblem(2, [(0, 1, 1.0)])
    traj["kat_tanh"] = nmfa.nmfa_step(p2, np.array([0.9, 0.9]), 0.5,
                                      nmfa.NmfaParams(alpha=1.0, sigma=0.0, t_f=1), noise_stream(0))
    save("trajectories.npz", **traj)

    # ---- seeded batches (solver.py:262-280) ----
    bat = {}
    for name, p, t_f, R in [("moebius16_tf100", specs["moebius16"], 100, 100),
                            ("sk100_tf1000", specs["sk100_s0"], 1000, 32),
                            ("moebius100_tf1000", specs["moebius100"], 1000, 32),
                            ("cubic40_tf300", specs["cubic40_s1"], 300, 32)]:
        res = nmfa.nmfa_batch(p, nmfa.NmfaParams(t_f=t_f, seed=0), R, threads=THREADS)
        bat[name + "_E"] = np.array([r.final_energy for r in res])
        bat[name + "_cfg"] = np.array([r.final_config for r in res]).astype(np.int8)
    g2000 = nmfa.gen_dense_maxcut(2000, 0.01, 7)
    res = nmfa.nmfa_batch(g2000, nmfa.NmfaParams(t_f=300, seed=0), 8, threads=THREADS)
    bat["g2000_tf300_E"] = np.array([r.final_energy for r in res])
    save("batches.npz", **bat)

    # ---- success statistics (metrics.py:70-94) ----
    st = {}
    for name, p, t_f, R in [("sk100", specs["sk100_s0"], 1000, 10000),
                            ("moebius100", specs["moebius100"], 1000, 4096),
                            ("moebius16_tf100", specs["moebius16"], 100, 1000),
                            ("g2000", g2000, 1000, 256),
                            ("sk2000", nmfa.gen_sk(2000, 7), 1000, 64)]:
        t1 = time.time()
        res = nmfa.nmfa_batch(p, nmfa.NmfaParams(t_f=t_f, seed=0), R, threads=THREADS)
        wall = time.time() - t1
        st[name + "_E"] = np.array([r.final_energy for r in res])
        st[name + "_wall"] = np.array(wall)
        st[name + "_threads"] = np.array(THREADS)
        print(f"  stats {name}: R={R} wall={wall:.1f}s min={st[name + '_E'].min()}")
    gt = nmfa.brute_force_ground(specs["moebius16"])
    st["moebius16_ground"] = np.array(gt.energy)
    st["tts_kat"] = np.array(nmfa.time_to_solution(0.5, 12.3e-6))
    save("stats.npz", **st)
    print(f"done in {time.time() - t0:.1f}s")


if __name__ == "__main__":
    main()
