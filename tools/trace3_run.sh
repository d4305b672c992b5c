#!/bin/bash
# per-k-slice clock64 (CTA 0, k-slices 256..319): TMA issue, MMA sees data, MMA committed
for v in "$@"; do
  if [ "$v" = full ]; then defs=""; else defs=$(echo "$v" | tr "+" " " | sed "s/\([A-Z_=0-9]*\)/-D\1/g"); fi
  NMFA_NVCC_DEFS="$defs" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1 || { echo "$v build failed"; continue; }
  tag=$(echo "$v" | tr '+' '_')
  NMFA_TRACE3=gpurun_out/t3_$tag.txt timeout 100 python tools/prof_dense.py 12 > /dev/null 2>&1
  echo "== $v"; python - gpurun_out/t3_$tag.txt <<'PY'
import sys, numpy as np
d = np.loadtxt(sys.argv[1]).astype(float)
iss, see, com = d[:, 0], d[:, 1], d[:, 2]
lat = see - iss                  # TMA issue -> MMA thread sees the stage full
mma = com - see                  # MMA issue time for the slice (8 instructions + commit)
gap = np.diff(see)               # k-slice period seen by the MMA thread
print(f"TMA issue->full median {np.median(lat):.0f} p90 {np.percentile(lat,90):.0f} | MMA issue median {np.median(mma):.0f} | slice period median {np.median(gap):.0f} mean {gap.mean():.0f}")
print("first 20 lat:", lat[:20].astype(int))
print("first 20 gap:", gap[:20].astype(int))
PY
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
