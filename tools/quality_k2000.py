"""Cut quality on the K2000 stand-in gen_sk(2000,7) vs the reference's published
20-run numbers (pkg/README.md:171: t_f=1000 mean 33311 / best 33654;
t_f=2000 mean 33624 / best 33920)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_1806_08422_b200 as nb
p = nb.gen_sk(2000, 7)
W = float(p.edge_weights.sum())
for t_f, ref in [(1000, (33311, 33654)), (2000, (33624, 33920))]:
    res = nb.sample(p, nb.NmfaParams(t_f=t_f, seed=0), 4096)
    e = res.energies.cpu().numpy()
    cut = (W - e) / 2.0          # cut_value = sum w (1 - c_i c_j) / 2 (problem.py:157-163), h = 0
    first20 = cut[:20]
    print(f"t_f={t_f}: 4096 reads mean cut {cut.mean():.1f} (SE {cut.std()/np.sqrt(cut.size):.1f}), "
          f"best {cut.max():.0f}; first 20 reads mean {first20.mean():.1f} best {first20.max():.0f} | "
          f"reference 20 runs: mean {ref[0]} best {ref[1]}")
