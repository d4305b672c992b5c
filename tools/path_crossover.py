"""Dense (tcgen05) vs sparse (ELL / CSR) per-sweep time across n and degree, to
fit the path-choice cost model of capi.cu (prefer_dense).  R=1024, t_f=100."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1806_08422_b200 as nb


def random_regular_ish(n, d, seed):
    """Erdos-Renyi with mean degree d (p = d / (n - 1))."""
    return nb.gen_dense_maxcut(n, min(1.0, d / (n - 1)), seed)


def torus(n):
    c = int(round(np.sqrt(n)))
    v = np.arange(c * c).reshape(c, c)
    a = np.concatenate([v.ravel(), v.ravel()])
    b = np.concatenate([np.roll(v, -1, 1).ravel(), np.roll(v, -1, 0).ravel()])
    return nb.IsingProblem.from_arrays(c * c, np.minimum(a, b), np.maximum(a, b), np.ones(a.size))


def sweep_us(p, path, R=1024, t_f=100):
    p.device_handle().set_path(path)
    params = nb.NmfaParams(t_f=t_f, seed=0)
    plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
    cfg = torch.empty((R, p.n), dtype=torch.int8, device="cuda")
    plan.run(0, 0, config=cfg); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for k in range(3):
        plan.run(k, 0, config=cfg)
    b.record(); torch.cuda.synchronize()
    del plan
    return a.elapsed_time(b) * 1e3 / (3 * t_f)


cases = []
for n in (512, 1024, 2048, 4096, 8192, 16384):
    cases += [("cubic", n, lambda n=n: nb.gen_cubic_maxcut(n, 1)), ("torus", n, lambda n=n: torus(n)),
              ("er_d10", n, lambda n=n: random_regular_ish(n, 10, 1)),
              ("er_d20", n, lambda n=n: random_regular_ish(n, 20, 1)),
              ("er_d60", n, lambda n=n: random_regular_ish(n, 60, 1))]
for name, n, mk in cases:
    p = mk()
    auto = p.device_info()["path"]
    d = sweep_us(p, "dense")
    s = sweep_us(p, "sparse")
    deg = 2 * p.num_edges / p.n
    print(f"{name:7s} n={p.n:6d} deg={deg:5.1f} auto={auto:6s} dense {d:8.1f} us  sparse {s:8.1f} us  "
          f"-> {'dense' if d < s else 'sparse'} ({max(d, s) / min(d, s):.2f}x)", flush=True)
