"""Quick device timings of the sampling paths (development probe, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1806_08422_b200 as nb

def timeit(p, R, t_f=1000, reps=3, path=None):
    if path: p.device_handle().set_path(path)
    params = nb.NmfaParams(t_f=t_f, seed=0)
    plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
    cfg = torch.empty((R, p.n), dtype=torch.int8, device="cuda")
    en = torch.empty(R, dtype=torch.float64, device="cuda")
    plan.run(0, 0, config=cfg, energy=en); torch.cuda.synchronize()
    ts = []
    for k in range(reps):
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(); plan.run(k, 0, config=cfg, energy=en); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e-3)
    t = min(ts)
    su = p.n * R * t_f / t
    print(f"{p!r:32s} path={p.device_info()['path']:6s} R={R:7d} t_f={t_f} time={t*1e3:9.3f} ms "
          f"spin-updates/s={su:.3e} best={en.min().item()}", flush=True)
    return t

cases = sys.argv[1:] or ["sk100", "moebius100", "g2000"]
for c in cases:
    if c == "sk100":
        p = nb.gen_sk(100, 0)
        for R in (100, 4096, 37888, 151552): timeit(p, R)
    elif c == "moebius100":
        p = nb.moebius_ladder(100)
        for R in (4096, 37888): timeit(p, R)
        timeit(nb.moebius_ladder(100), 4096, path="sparse")
    elif c == "g2000":
        p = nb.gen_dense_maxcut(2000, 0.01, 7)
        timeit(p, 4096, reps=1)
    elif c == "k2000":
        p = nb.gen_sk(2000, 7)
        timeit(p, 8192, reps=2)
