"""Per-step cost of the sparse path launched directly vs replayed from a CUDA graph."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_08422_b200 as nb
for n in (512, 2048, 8192):
    p = nb.gen_cubic_maxcut(n, 1)
    R, t_f = 1024, 200
    params = nb.NmfaParams(t_f=t_f, seed=0)
    plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
    cfg = torch.empty((R, n), dtype=torch.int8, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        plan.run(0, 0, config=cfg, stream=s); torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            plan.run(0, 0, config=cfg, stream=s)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(); plan.run(1, 0, config=cfg); ev[1].record()
    ev[2].record(); g.replay(); ev[3].record(); torch.cuda.synchronize()
    d, gr = ev[0].elapsed_time(ev[1]) * 1e3 / t_f, ev[2].elapsed_time(ev[3]) * 1e3 / t_f
    print(f"cubic n={n}: direct {d:.2f} us/step, graph replay {gr:.2f} us/step", flush=True)
