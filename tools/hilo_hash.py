"""Configuration + energy hash of a K2000 HILO-field anneal (bitwise A/B of
HILO kernel variants) and its sweep time."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1806_08422_b200 as nb  # noqa: E402

p = nb.gen_sk(2000, 7)
p.device_handle().set_path("dense")
p.device_handle().set_field_precision("hilo")
R, t_f = 8192, int(sys.argv[1]) if len(sys.argv) > 1 else 200
params = nb.NmfaParams(t_f=t_f, seed=0)
plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
cfg = torch.empty((R, 2000), dtype=torch.int8, device="cuda")
en = torch.empty(R, dtype=torch.float64, device="cuda")
plan.run(0, 0, config=cfg, energy=en)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for k in range(3):
    plan.run(0, 0, config=cfg, energy=en)
b.record()
torch.cuda.synchronize()
h = hashlib.sha1(cfg.cpu().numpy().tobytes() + en.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"HILO K2000 t_f={t_f}: {a.elapsed_time(b) / 3 / t_f * 1e3:.1f} us/sweep  hash {h}")
