import numpy as np, sys
d = np.loadtxt(sys.argv[1]).astype(np.float64)
valid = d[:, 2] > 0
d = d[valid]
t0 = d[d > 0].min()
d = np.where(d > 0, d - t0, np.nan)
# columns: 0 producer tile start, 1 producer last slice, 2 mma start, 3 mma end, 4 epi start, 5 epi end
n = len(d)
mma = d[:, 3] - d[:, 2]; epi = d[:, 5] - d[:, 4]
gap = d[1:, 2] - d[:-1, 3]
print(f"tiles traced {n}")
print("first 12 tiles [prod_start, prod_last, mma_start, mma_end, epi_start, epi_end]:")
for r in d[:12]: print("  ", np.round(r).astype(int))
print(f"MMA per tile median {np.nanmedian(mma):.0f}  epilogue per tile median {np.nanmedian(epi):.0f}")
print(f"MMA idle gap between tiles: median {np.nanmedian(gap):.0f} mean {np.nanmean(gap):.0f} max {np.nanmax(gap):.0f}")
tiles_per_sweep = int(sys.argv[2]) if len(sys.argv) > 2 else 4
sw = d[::tiles_per_sweep, 2]
print("sweep start deltas (cycles):", np.round(np.diff(sw)[:10]).astype(int), "median", np.nanmedian(np.diff(sw)))
busy = np.nansum(mma) / (np.nanmax(d[:, 3]) - np.nanmin(d[:, 2]))
print(f"MMA busy fraction over traced window: {busy:.2f}")
