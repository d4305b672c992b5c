"""max|dS| of every injected-noise trajectory fixture on every path (the
numbers behind tests/test_gpu_parity.py's tolerance)."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for d in (REPO, os.path.join(REPO, "oracle"), os.path.join(REPO, "tests")):
    sys.path.insert(0, d)
import numpy as np  # noqa: E402

import nmfa_oracle as O  # noqa: E402
import paper_1806_08422_b200 as nb  # noqa: E402
from conftest import golden  # noqa: E402

T, E = golden("trajectories.npz"), golden("energies.npz")
for name in ["moebius16", "cubic40_s1", "sk30_s2", "dense60_p03_s3", "int40_h", "real24_h", "sk100_s0"]:
    for path in ["small", "sparse", "dense"]:
        p = nb.IsingProblem.from_arrays(int(E[name + "_n"]), E[name + "_ei"], E[name + "_ej"],
                                        E[name + "_w"], E[name + "_h"])
        p.device_handle().set_path(path)
        t_f, seed = int(T[name + "_tf"]), int(T[name + "_seed"])
        noise = O.run_noise(seed, t_f, p.n, 0.15)
        s, tr = nb.run_with_noise(p, O.temperatures(t_f), noise, 0.15, record_trajectory=True)
        d1 = np.abs(s - T[name + "_s"]).max()
        d2 = np.abs(tr.spins[-10:] - T[name + "_s_hist_last10"]).max()
        print(f"{name:16s} {path:7s} n={p.n:4d} t_f={t_f:5d} max|dS| final {d1:.2e} last10 {d2:.2e}", flush=True)
