"""Per-run time (tau) on the paper's timing instance: dense MAX-CUT N=100, p=0.5
(12.3 us/run on a GTX 1080 Ti), default schedule, t_f = 1000."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_08422_b200 as nb
p = nb.gen_dense_maxcut(100, 0.5, 0)
params = nb.NmfaParams(t_f=1000, seed=0)
R = 37888
nb.sample(p, params, R); torch.cuda.synchronize()
ts = []
for k in range(5):
    t = time.perf_counter(); r = nb.sample(p, params, R); torch.cuda.synchronize(); ts.append(time.perf_counter() - t)
tau = min(ts) / R
print(f"dense MAX-CUT N=100, p=0.5, t_f=1000, {R} reads per call: tau = {tau*1e6:.3f} us/run "
      f"(paper, GTX 1080 Ti: 12.3 us/run -> {12.3e-6/tau:.0f}x); best energy {r.energies.min().item()}")
