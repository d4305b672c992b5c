"""CSR path on large sparse instances: us/step and HBM roofline fraction.
Algorithmic bytes per step: R*N*8 + nnz_dir*8 + (N+1)*4."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_08422_b200 as nb

peaks = json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json")))
hbm = next(v for k, v in peaks.items() if "hbm" in k.lower() and isinstance(v, (int, float)))
def torus(n):
    import numpy as np
    c = int(round(n ** 0.5))
    v = np.arange(c * c).reshape(c, c)
    a = np.concatenate([v.ravel(), v.ravel()])
    b = np.concatenate([np.roll(v, -1, 1).ravel(), np.roll(v, -1, 0).ravel()])
    w = np.where(np.random.default_rng(c).random(a.size) < 0.5, 1.0, -1.0)
    return nb.IsingProblem.from_arrays(c * c, np.minimum(a, b), np.maximum(a, b), w)


cases = [("moebius", lambda n: nb.moebius_ladder(n)), ("cubic", lambda n: nb.gen_cubic_maxcut(n, 1))]
def er(n, d, seed=1):
    """about n*d/2 random couplers (Poisson degrees, mean d), +1 weights"""
    import numpy as np
    rng = np.random.default_rng(seed)
    a, b = rng.integers(0, n, n * d // 2), rng.integers(0, n, n * d // 2)
    keep = a != b
    key = np.unique(np.minimum(a, b)[keep] * n + np.maximum(a, b)[keep])
    return nb.IsingProblem.from_arrays(n, key // n, key % n, np.ones(key.size))


if os.environ.get("PROF_TORUS"):
    cases = [("torus", torus)]
if os.environ.get("PROF_ER"):
    cases = [(f"er_d{d}", (lambda d: lambda n: er(n, d))(d)) for d in map(int, os.environ["PROF_ER"].split(","))]
n = int(sys.argv[1]) if len(sys.argv) > 1 else 131072
R = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
t_f = 100
for name, mk in cases:
    p = mk(n)
    info = p.device_info()
    params = nb.NmfaParams(t_f=t_f, seed=0)
    plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
    cfg = torch.empty((R, n), dtype=torch.int8, device="cuda")
    plan.run(0, 0, config=cfg); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(3):
        plan.run(k, 0, config=cfg)
    b.record(); torch.cuda.synchronize()
    us = a.elapsed_time(b) * 1e3 / (3 * t_f)
    nnz = 2 * p.num_edges
    byts = R * n * 8 + nnz * 8 + (n + 1) * 4
    gbs = byts / (us * 1e-6) / 1e9
    print(f"{name} n={p.n} R={R} path={info['path']}: {us:.1f} us/step  {n*R/(us*1e-6):.3g} su/s  "
          f"{gbs:.0f} GB/s algorithmic = {gbs/hbm:.2f} of HBM {hbm:.0f}", flush=True)
