#!/bin/bash
# A/B of compile-time variants on the K2000 bench line (alternating, twice each):
#   bash tools/ab_bench.sh "" "-DNMFA_EPI_SPIN"      (first = default build)
# prints value, ms/step, median SM clock and power for each run
mkdir -p gpurun_out
for rep in 1 2; do
  for v in "$@"; do
    NMFA_NVCC_DEFS="$v" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1 || { echo "build '$v' failed"; continue; }
    timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-tts --no-stats > gpurun_out/ab.json 2> /dev/null
    python - "$v" <<'PY'
import json, sys
d = json.loads([l for l in open("gpurun_out/ab.json") if l.startswith("{")][0])
print(f"[{sys.argv[1] or 'default'}] {d['value']:.4e} su/s  {d['ms_per_step']:.2f} ms/step  frac {d['roofline']['frac']:.3f}  "
      f"clock {d['clocks']['sm_mhz']} MHz  power {d['clocks'].get('power_w_median')} W  {d['clocks']['reasons']}", flush=True)
PY
  done
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
