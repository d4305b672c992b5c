"""ELL step time with the replica slices annealed in groups (NMFA_SPARSE_GROUPS,
direct launches) against one launch per step over all slices (also direct):
Moebius n = 131,072 and the 362x362 torus, 1024 reads, t_f = 200.  The
NMFA_SPARSE_GROUPS patch of anneal_sparse.cu was reverted after this study
(profiles/r02/sparse_replica_groups.log); without it the variable is ignored."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1806_08422_b200 as nb  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "moebius"
p = nb.moebius_ladder(131072) if name == "moebius" else nb.toroidal_grid(362, 362, 1)
R, t_f = 1024, 200
params = nb.NmfaParams(t_f=t_f, seed=0)
plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
cfg = torch.empty((R, p.n), dtype=torch.int8, device="cuda")
plan.run(0, 0, config=cfg)
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for k in range(3):
    plan.run(0, 0, config=cfg)
b.record()
torch.cuda.synchronize()
ms = a.elapsed_time(b) / 3
import hashlib  # noqa: E402
h = hashlib.sha1(cfg.cpu().numpy().tobytes()).hexdigest()[:12]
print(f"{name} groups={os.environ.get('NMFA_SPARSE_GROUPS', '1')}: {ms / t_f * 1e3:.1f} us/step  "
      f"{p.n * R * t_f / (ms * 1e-3):.3e} su/s  cfg {h}", flush=True)
