"""One short anneal on every kernel path, for compute-sanitizer (memcheck,
racecheck, synccheck).  Small sizes and short t_f: the sanitizer slows
kernels by 10-100x.

    compute-sanitizer --tool memcheck python tools/sanitize_paths.py
"""

import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1806_08422_b200 as nb  # noqa: E402

which = sys.argv[1:] or ["small", "dense", "ell", "csr", "energy", "ground", "many"]
params = nb.NmfaParams(t_f=int(os.environ.get("SAN_TF", "6")), seed=3)
if "small" in which:
    p = nb.gen_sk(100, 0)
    p.device_handle().set_path("small")
    r = nb.sample(p, params, 256, return_s=True, record_trajectory=True)
    print("small", float(r.energies.min()))
if "dense" in which:
    p = nb.gen_sk(600, 1)          # 3 spin tiles, ragged, two replica blocks
    p.device_handle().set_path("dense")
    r = nb.sample(p, params, 300, return_s=True)
    print("dense", float(r.energies.min()))
    noise = np.random.default_rng(1).standard_normal((20, params.t_f, 600)) * 0.15
    S, _ = nb.run_with_noise(p, nb.DEFAULT_SCHEDULE.temperatures(params.t_f), noise, 0.15)
    print("dense injected", float(np.abs(S).mean()))
if "ell" in which:
    p = nb.moebius_ladder(1000)
    assert p.device_info()["ell_slots"] > 0
    r = nb.sample(p, params, 100, return_s=True)
    print("ell", float(r.energies.min()))
if "csr" in which:
    p = nb.gen_dense_maxcut(1200, 0.01, 2)
    p.device_handle().set_path("sparse")
    r = nb.sample(p, params, 70, return_s=True)
    print("csr", float(r.energies.min()))
if "energy" in which:
    p = nb.gen_dense_maxcut(300, 0.2, 4)
    cfg = np.where(np.random.default_rng(2).random((33, 300)) < 0.5, -1.0, 1.0)
    print("energy", nb.energies(p, cfg)[:3])
if "ground" in which:
    g = nb.brute_force_ground(nb.gen_sk(14, 2))
    print("ground", g.energy, g.degeneracy)
if "many" in which:
    ps = [nb.gen_sk(40, k) for k in range(3)]
    cfg, en, _ = nb.sample_many(ps, params, 64)
    print("many", en.min(dim=1).values.tolist())
torch.cuda.synchronize()
print("ok")
