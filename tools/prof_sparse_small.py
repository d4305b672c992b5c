"""Small ELL graphs: per-step wall time (events over t_f launches) for the ncu launch list."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_08422_b200 as nb
for n in (512, 1024, 2048, 4096, 8192, 16384):
    p = nb.gen_cubic_maxcut(n, 1)
    R, t_f = 1024, 200
    params = nb.NmfaParams(t_f=t_f, seed=0)
    plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
    cfg = torch.empty((R, n), dtype=torch.int8, device="cuda")
    plan.run(0, 0, config=cfg); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); plan.run(1, 0, config=cfg); b.record(); torch.cuda.synchronize()
    print(f"cubic n={n} R={R}: {a.elapsed_time(b) * 1e3 / t_f:.2f} us/step (events)", flush=True)
