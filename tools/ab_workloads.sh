#!/bin/bash
# A/B of compile-time variants over several bench workloads (alternating, twice each):
#   bash tools/ab_workloads.sh "k2000 sk100 moebius131072" "" "-DNMFA_TANH_FOLD" ...
mkdir -p gpurun_out
wls="$1"; shift
for rep in 1 2; do
  for v in "$@"; do
    NMFA_NVCC_DEFS="$v" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1 || { echo "build '$v' failed"; continue; }
    for w in $wls; do
      timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-tts --no-stats > gpurun_out/ab.json 2> /dev/null
      python - "$v" "$w" <<'PY'
import json, sys
d = json.loads([l for l in open("gpurun_out/ab.json") if l.startswith("{")][0])
print(f"[{sys.argv[1] or 'default'}] {sys.argv[2]:14s} {d['value']:.4e} su/s  frac {d['roofline']['frac']:.3f}  "
      f"clock {d['clocks']['sm_mhz']} MHz  {d['clocks']['reasons']}", flush=True)
PY
    done
  done
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
