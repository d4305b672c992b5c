"""Fig. 4-style sweep cost: K instances x R reads at size n, grouped launch vs one call per instance."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from dataclasses import replace
import torch
import paper_1806_08422_b200 as nb
from paper_1806_08422_b200.experiments import make_instance, bench
params = nb.NmfaParams(t_f=1000, seed=0)
for n, K, R in [(32, 100, 1000), (64, 100, 1000), (128, 50, 1000)]:
    probs = [make_instance("sk", n, 0.5, k) for k in range(K)]
    nb.sample_many(probs[:2], params, R); torch.cuda.synchronize()
    _, _, wall = nb.sample_many(probs, params, R)
    for p in probs[:2]:
        nb.sample(p, params, R)
    torch.cuda.synchronize(); t = time.perf_counter()
    for k, p in enumerate(probs):
        nb.sample(p, replace(params, seed=k * R), R)
    torch.cuda.synchronize(); loop = time.perf_counter() - t
    print(f"n={n} K={K} R={R}: grouped {wall*1e3:.1f} ms ({n*K*R*1000/wall:.3g} su/s)  "
          f"per-instance loop {loop*1e3:.1f} ms  speed-up {loop/wall:.1f}x", flush=True)
t = time.perf_counter()
rows, text, _ = bench("sk", [16, 20, 24], 20, 1000, params)
print(f"bench sk 16,20,24 x 20 instances x 1000 runs: {time.perf_counter()-t:.2f} s")
print(text)
