"""Short runs of each kernel path for ncu captures: small (SK100), sparse (Moebius 131072), dense (K2000)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_08422_b200 as nb
which = sys.argv[1]
if which == "small":
    p, R, t_f = nb.gen_sk(100, 0), 37888, 1000
elif which == "sparse":
    p, R, t_f = nb.moebius_ladder(131072), 1024, 8
else:
    p, R, t_f = nb.gen_sk(2000, 7), 8192, int(os.environ.get("PROF_TF", "3"))
params = nb.NmfaParams(t_f=t_f, seed=0)
plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
cfg = torch.empty((R, p.n), dtype=torch.int8, device="cuda")
en = torch.empty(R, dtype=torch.float64, device="cuda")
use_e = os.environ.get("PROF_NO_ENERGY") is None
for k in range(2):
    plan.run(k, 0, config=cfg, energy=en if use_e else None)
torch.cuda.synchronize()
print(which, "ok", en.min().item())
