import sys, os
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import numpy as np, nmfa_oracle as O, paper_1806_08422_b200 as nb
n, R = 129, 256
for path in ["small", "dense", "sparse"]:
    rng = np.random.default_rng(n * 1000 + R)
    p = nb.gen_sk(n, n); p.device_handle().set_path(path)
    t_f = 40; temps = O.temperatures(t_f)
    noise = rng.standard_normal((R, t_f, n)) * 0.15
    S, _ = nb.run_with_noise(p, temps, noise, 0.15)
    op = O.problem_from_edges(n, p.edges_i, p.edges_j, p.edge_weights)
    ref = np.stack([O.anneal(op, np.zeros(n), temps, noise[r], 0.15)[0] for r in range(R)])
    err = np.abs(S - ref)
    big = np.argwhere(err > 2e-2)
    print(path, "max", err.max(), "mean", err.mean(), "n>2e-2", len(big), "replicas", sorted(set(big[:,0].tolist()))[:10], "spins", sorted(set(big[:,1].tolist()))[:10],
          "flips", np.mean(np.sign(S) != np.sign(ref)))
