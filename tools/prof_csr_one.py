"""One CSR-kernel run for ncu: G-set-like random graph n = 10000, mean degree 5, 1024 reads."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1806_08422_b200 as nb  # noqa: E402

p = nb.gen_dense_maxcut(10000, 5 / 9999, 1)
R, t_f = 1024, 8
params = nb.NmfaParams(t_f=t_f, seed=0)
plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
cfg = torch.empty((R, p.n), dtype=torch.int8, device="cuda")
for k in range(2):
    plan.run(k, 0, config=cfg)
torch.cuda.synchronize()
print("ok", p.device_info()["path"])
