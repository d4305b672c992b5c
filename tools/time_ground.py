import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import paper_1806_08422_b200 as nb
import nmfa_oracle as O
for n, mx in [(26, 26), (30, 30), (34, 34)]:
    p = nb.gen_sk(n, 1)
    nb.brute_force_ground(nb.gen_sk(20, 1))  # warm
    t = time.perf_counter(); gt = nb.brute_force_ground(p, max_n=mx); dt = time.perf_counter() - t
    print(f"GPU n={n}: E={gt.energy} deg={gt.degeneracy} {dt*1e3:.1f} ms  {2**n/dt:.3g} configs/s", flush=True)
op = O.problem_from_edges(26, *nb.gen_sk(26, 1).edges_i[None], ) if False else None
p = nb.gen_sk(24, 1)
opp = O.problem_from_edges(24, p.edges_i, p.edges_j, p.edge_weights)
O.gray_ground_fast(O.problem_from_edges(8, p.edges_i[:3], p.edges_j[:3], p.edge_weights[:3]))
t = time.perf_counter(); r = O.gray_ground_fast(opp); dt = time.perf_counter() - t
print(f"CPU port (1 thread) n=24: {r} {dt:.2f} s  {2**24/dt:.3g} configs/s", flush=True)
