"""Dense-kernel throughput across spin count N and replica count R (SK
instances, t_f = 100 sweeps + energy pass, CUDA events, no L2 flush): the
sustained-peak fraction the tile geometry and the schedule reach per shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1806_08422_b200 as nb  # noqa: E402

PEAK = 1363.6  # MEASURED_PEAKS bf16 sustained TFLOP/s
# optional: tools/dense_size_sweep.py N1,N2,.. R1,R2,.. t_f
NS = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else (1000, 2000, 4000, 8000)
RS = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else (4096, 8192, 16384)
t_f = int(sys.argv[3]) if len(sys.argv) > 3 else 100
for n in NS:
    p = nb.gen_sk(n, 3)
    p.device_handle().set_path("dense")
    for R in RS:
        params = nb.NmfaParams(t_f=t_f, seed=0)
        plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
        cfg = torch.empty((R, n), dtype=torch.int8, device="cuda")
        en = torch.empty(R, dtype=torch.float64, device="cuda")
        plan.run(0, 0, config=cfg, energy=en)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for k in range(3):
            plan.run(k + 1, 0, config=cfg, energy=en)
        b.record()
        torch.cuda.synchronize()
        sweep_s = a.elapsed_time(b) * 1e-3 / (3 * t_f)
        tf = 2.0 * n * n * R / sweep_s / 1e12
        print(f"N={n:5d} R={R:6d}: {sweep_s * 1e6:8.1f} us/sweep  {tf:7.0f} TFLOP/s  "
              f"{tf / PEAK:.3f} of sustained  {n * R / sweep_s:.3e} spin-updates/s", flush=True)
        del plan
