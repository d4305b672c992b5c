import numpy as np, sys
d = np.loadtxt(sys.argv[1]).astype(np.float64)
d = d[d[:, 2] > 0]
t0 = np.nanmin(np.where(d > 0, d, np.nan))
d = np.where(d > 0, d - t0, np.nan)
# cols: 0 producer tile start, 1 producer last slice, 2 mma start (tempty ok), 3 mma last commit, 4 epi start (tfull), 5 epi end (max over warps)
mma = d[:, 3] - d[:, 2]; epi = d[:, 5] - d[:, 4]
gap = d[1:, 2] - d[:-1, 3]
tps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
print(f"tiles {len(d)}; first 9 rows [prod_start prod_last mma_start mma_end epi_start epi_end]:")
for r in d[:9]: print("  ", np.round(r).astype(int))
print(f"MMA issue span per tile: median {np.nanmedian(mma):.0f}; epilogue per tile: median {np.nanmedian(epi):.0f}")
print(f"MMA idle between tiles: median {np.nanmedian(gap):.0f}, mean {np.nanmean(gap):.0f}")
print(f"  idle at sweep boundaries: mean {np.nanmean(gap[tps-1::tps]):.0f}; inside sweeps: mean {np.nanmean(np.delete(gap, np.s_[tps-1::tps])):.0f}")
print(f"mma waited for epilogue (mma_start - prev-prev epi_end): median {np.nanmedian(d[2:,2]-d[:-2,5]):.0f}")
sweep = np.diff(d[::tps, 2]); print(f"sweep period median {np.nanmedian(sweep):.0f} cycles")
if d.shape[1] >= 8:
    print(f"per tile: MMA waited for TMA data median {np.nanmedian(d[:,6]+t0):.0f} cycles; "
          f"producer waited for a free stage median {np.nanmedian(d[:,7]+t0):.0f}")
