# small kernel: start stagger of the grid's second half (NMFA_SMALL_STAGGER ns)
mkdir -p gpurun_out
python -m paper_1806_08422_b200.build > /dev/null 2>&1
for st in 0 800 1600 2400 0 1600; do
  echo "-- stagger=$st ns"
  for w in sk100 moebius100; do
    NMFA_SMALL_STAGGER=$st timeout 300 python bench.py --workload $w --steps 5 --warmup 3 --no-tts --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$w', '%.4g'%d['value'], 'su/s', '%.3f'%d['ms_per_step'], 'ms/step')"
  done
done
