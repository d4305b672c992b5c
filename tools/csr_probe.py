"""CSR-path sweep time on G-set-like random graphs (mean degree 2-10, the
G55/G60/G70 class that the router sends to the CSR kernel) against the
per-step algorithmic bytes of SURVEY 8(d)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1806_08422_b200 as nb  # noqa: E402

HBM = 6545e9
for n, d in [(5000, 5), (7000, 5), (10000, 2), (10000, 5), (16384, 10), (16384, 16), (16384, 20)]:
    p = nb.gen_dense_maxcut(n, d / (n - 1), 1)
    info = p.device_info()
    for R in (1024, 4096):
        t_f = 100
        params = nb.NmfaParams(t_f=t_f, seed=0)
        plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
        cfg = torch.empty((R, n), dtype=torch.int8, device="cuda")
        plan.run(0, 0, config=cfg)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for k in range(3):
            plan.run(k, 0, config=cfg)
        b.record()
        torch.cuda.synchronize()
        us = a.elapsed_time(b) * 1e3 / (3 * t_f)
        nnz = 2 * p.num_edges
        byts = R * n * 8 + nnz * 8 + (n + 1) * 4
        import hashlib
        h = hashlib.sha1(cfg.cpu().numpy().tobytes()).hexdigest()[:10]
        print(f"n={n:6d} deg={nnz / n:5.1f} path={info['path']} ell={info['ell_slots']} R={R:5d}: "
              f"{us:7.1f} us/step  {n * R / (us * 1e-6):.3e} su/s  {byts / (us * 1e-6) / HBM:.3f} of HBM"
              f"  cfg {h}", flush=True)
        del plan
