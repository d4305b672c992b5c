"""A few steps of the sparse path on moebius_ladder(131072) or gen_cubic_maxcut(131072), R=1024 (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_08422_b200 as nb
n, R, t_f = 131072, 1024, 8
p = nb.gen_cubic_maxcut(n, 1) if sys.argv[1:] == ["cubic"] else nb.moebius_ladder(n)
params = nb.NmfaParams(t_f=t_f, seed=0)
plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
cfg = torch.empty((R, n), dtype=torch.int8, device="cuda")
plan.run(0, 0, config=cfg); torch.cuda.synchronize(); print("ok")
