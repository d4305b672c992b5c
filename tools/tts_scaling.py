"""Fig. 4-style TTS99 scaling on SK instances (the reference's `bench` command,
cli.py:280-347): per size, 16 instances with exact ground truth from the GPU
enumerator; the GPU side is experiments.bench (one grouped launch per size); the
CPU side is the jitted port of the reference's per-run loop on the first 4
instances (256 runs each, all host cores), tau = batch wall / runs as in the
reference."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
import math
import numpy as np
import nmfa_oracle as O
import paper_1806_08422_b200 as nb
from paper_1806_08422_b200 import experiments as X

sizes = [10, 14, 18, 22, 26]
inst, runs, cpu_inst, cpu_runs = 16, 4096, 4, 256
params = nb.NmfaParams(t_f=1000, seed=0)
threads = os.cpu_count() or 1
rows, _, per_size = X.bench("sk", sizes, inst, runs, params)
O.batch(O.problem_from_edges(10, *O.gen_sk_edges(10, 0)), 0, threads, t_f=20, threads=threads)  # warm
print(f"{'n':>3} {'GPU p med':>9} {'GPU TTS99 med':>14} {'CPU p med':>9} {'CPU TTS99 med':>14} {'ratio':>8}")
counter = 0
for k, n in enumerate(sizes):
    gpu_p = np.median([s.p_success for s in per_size[n]])
    gpu_tts = np.median([s.tts_seconds for s in per_size[n]])
    cpu_p, cpu_tts = [], []
    for g in range(cpu_inst):
        prob = X.make_instance("sk", n, 0.5, params.seed + k * inst + g)
        e_ref = nb.brute_force_ground(prob).energy
        op = O.problem_from_edges(n, prob.edges_i, prob.edges_j, prob.edge_weights)
        t0 = time.perf_counter()
        _, e = O.batch(op, 0, cpu_runs, t_f=1000, threads=threads)
        tau = (time.perf_counter() - t0) / cpu_runs
        p = float(np.mean(e <= e_ref + 1e-9))
        cpu_p.append(p)
        cpu_tts.append(O.time_to_solution(p, tau))
    cp, ct = np.median(cpu_p), np.median(cpu_tts)
    print(f"{n:3d} {gpu_p:9.3f} {gpu_tts*1e6:11.2f} us {cp:9.3f} {ct*1e6:11.1f} us {ct/gpu_tts:8.0f}x", flush=True)
print(f"(GPU: {inst} instances x {runs} runs per size in one grouped launch; CPU: {cpu_inst} instances x "
      f"{cpu_runs} runs, {threads} threads)")
