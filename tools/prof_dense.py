"""One short K2000 dense anneal (for ncu): n=2000, R=8192 (or argv[2]), t_f=20 (or argv[1])."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_08422_b200 as nb
t_f = int(sys.argv[1]) if len(sys.argv) > 1 else 20
R = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
p = nb.gen_sk(2000, 7)
params = nb.NmfaParams(t_f=t_f, seed=0)
plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
cfg = torch.empty((R, 2000), dtype=torch.int8, device="cuda")
en = torch.empty(R, dtype=torch.float64, device="cuda")
for k in range(2):
    plan.run(k, 0, config=cfg, energy=en)
torch.cuda.synchronize()
print("ok", en.min().item())
