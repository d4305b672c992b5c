"""Configuration/energy hash and throughput of the small kernel on SK100 and
Moebius-100 (37,888 reads, t_f = 1000): bitwise A/B of small-kernel variants."""
import hashlib
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1806_08422_b200 as nb  # noqa: E402

for name, p in [("sk100", nb.gen_sk(100, 0)), ("moebius100", nb.moebius_ladder(100))]:
    p.device_handle().set_path("small")
    R, t_f = 37888, 1000
    params = nb.NmfaParams(t_f=t_f, seed=3)
    plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
    cfg = torch.empty((R, p.n), dtype=torch.int8, device="cuda")
    en = torch.empty(R, dtype=torch.float64, device="cuda")
    plan.run(3, 0, config=cfg, energy=en)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(5):
        plan.run(3, 0, config=cfg, energy=en)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    h = hashlib.sha1(cfg.cpu().numpy().tobytes() + en.cpu().numpy().tobytes()).hexdigest()[:12]
    print(f"{name} table={os.environ.get('NMFA_SMALL_TABLE', 'auto')}: {ms:.3f} ms/anneal  "
          f"{p.n * R * t_f / (ms * 1e-3):.3e} su/s  hash {h}", flush=True)
