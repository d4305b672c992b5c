#!/bin/bash
# A/B of runtime environment knobs on the K2000 bench line (alternating, twice each):
#   bash tools/ab_env.sh "" "NMFA_TILE_W=16"
for rep in 1 2; do
  for v in "$@"; do
    env $v timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-tts --no-stats > gpurun_out/ab.json 2> /dev/null
    python - "$v" <<'PY'
import json, sys
d = json.loads([l for l in open("gpurun_out/ab.json") if l.startswith("{")][0])
print(f"[{sys.argv[1] or 'default'}] {d['value']:.4e} su/s  {d['ms_per_step']:.2f} ms/step  frac {d['roofline']['frac']:.3f}  "
      f"clock {d['clocks']['sm_mhz']} MHz  {d['clocks']['reasons']}", flush=True)
PY
  done
done
