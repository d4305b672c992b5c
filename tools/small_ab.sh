# small kernel occupancy A/B: NMFA_SMALL_MINB (compile) x NMFA_SMALL_CS (warps per lane quarter)
mkdir -p gpurun_out
for mb in 1 2; do
  NMFA_NVCC_DEFS="-DNMFA_SMALL_MINB=$mb" python -m paper_1806_08422_b200.build --force 2>&1 | grep -A2 "small_anneal_kernelILb0" | grep -E "spill|Used" | tr '\n' ' '; echo
  for cs in 2 4; do
    echo "-- minB=$mb cs=$cs"
    NMFA_SMALL_CS=$cs timeout 300 python bench.py --workload sk100 --steps 5 --warmup 3 --no-tts --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('sk100', '%.4g'%d['value'], 'su/s', d['ms_per_step'], 'ms/step')"
    NMFA_SMALL_CS=$cs timeout 300 python bench.py --workload moebius100 --steps 5 --warmup 3 --no-tts --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('moebius100', '%.4g'%d['value'], 'su/s', d['ms_per_step'], 'ms/step')"
  done
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
