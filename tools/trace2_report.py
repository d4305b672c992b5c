"""Analyse NMFA_TRACE2 timelines: per-tile MMA spans, readiness waits and the
publish times of the slices each tile consumed (globaltimer, ns)."""
import sys
import numpy as np

d = np.loadtxt(sys.argv[1], dtype=np.int64)
q, j, m, n0, nl = d[:, 0], d[:, 1], d[:, 2], d[:, 3], d[:, 4]
T = d[:, 5:].astype(np.float64)
t0 = T[T > 0].min()
T = np.where(T > 0, (T - t0) / 1000.0, np.nan)   # us
ps, last_ready, ms, me, ee, first_ready = T.T
pairs = q.max() + 1
ntile = np.bincount(q)
tps = {p: int((q == p).sum()) for p in range(pairs)}
# tiles per sweep per pair = number of distinct j per sweep; infer from the schedule (j % nt)
nt = np.array([len(set(zip(m[q == p], n0[q == p]))) for p in range(pairs)])
sweep = j // nt[q]
print(f"pairs {pairs}, tiles/pair per sweep {np.bincount(nt)}")
span = me - ms
print(f"MMA span per tile (us): median {np.nanmedian(span):.2f}  (sweep>=2)")
# sweep period from the end of epilogues
ends = [np.nanmax(ee[sweep == s]) for s in range(sweep.max() + 1)]
print("sweep ends (us):", np.round(ends, 1))
print("sweep periods:", np.round(np.diff(ends), 2))
# readiness: time from producer tile start to all slices ready
w_all = last_ready - ps
w_first = first_ready - ps
for s in range(2, min(sweep.max(), 6)):
    sel = sweep == s
    pos = j[sel] % nt[q[sel]]
    print(f"sweep {s}: wait first-slice by position", [f"{np.nanmedian(w_first[sel][pos == p]):.1f}" for p in range(4)],
          " wait all-slices", [f"{np.nanmedian(w_all[sel][pos == p]):.1f}" for p in range(4)])
# publish time of slice (m, kb) in sweep s = max epilogue end of tiles of block m covering kb
pub = {}
for i in range(len(d)):
    for kb in range(n0[i] // 128, (n0[i] + nl[i] - 1) // 128 + 1):
        key = (sweep[i], m[i], kb)
        pub[key] = max(pub.get(key, -1), ee[i])
# for tiles at position 0 of sweep s: when was each slice published (relative to the tile's producer start)
s = 4
sel = np.where((sweep == s) & (j % nt[q] == 0))[0]
lag = []
for i in sel[:6]:
    kbs = range(0, 16)
    p = [pub.get((s - 1, m[i], kb), np.nan) - ps[i] for kb in kbs]
    print(f"pair {q[i]} tile m={m[i]} n0={n0[i]}: prod_start {ps[i]:.1f} slices published at (rel):",
          " ".join(f"{x:5.1f}" for x in p), f"| all ready {w_all[i]:.1f} mma {ms[i]-ps[i]:.1f}..{me[i]-ps[i]:.1f}")
