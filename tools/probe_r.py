"""K2000 dense anneal timing vs replicas per GPU (L2 working-set study)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_08422_b200 as nb
p = nb.gen_sk(2000, 7)
for R in [int(x) for x in (sys.argv[1:] or ["2048", "4096", "8192", "16384"])]:
    params = nb.NmfaParams(t_f=200, seed=0)
    plan = nb.Plan(p, R, params.schedule.temperatures(200), params.alpha, params.sigma)
    cfg = torch.empty((R, 2000), dtype=torch.int8, device="cuda")
    plan.run(0, 0, config=cfg); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); plan.run(1, 0, config=cfg); b.record(); torch.cuda.synchronize()
    t = a.elapsed_time(b) / 200
    ws = (2 * 2048 * R * 2 + 2048 * R * 2 + 2000 * 2048 * 2) / 2**20
    print(f"R={R:6d} working set {ws:6.0f} MB  {t*1e3:7.1f} us/step  {2*2000*2000*R/t/1e9:7.1f} TFLOP/s  "
          f"{2000*R/t/1e3:.3e} su/s", flush=True)
    del plan
