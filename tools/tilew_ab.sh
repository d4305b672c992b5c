# dense tile width (NMFA_TILE_W, 16-spin units) at the G2000 config (R=4096) and K2000 (R=8192)
mkdir -p gpurun_out
python -m paper_1806_08422_b200.build > /dev/null 2>&1
for w in 14 8 10 12 16 7 14; do
  NMFA_TILE_W=$w timeout 300 python bench.py --workload g2000 --steps 3 --warmup 3 --no-tts --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('g2000 w=$w', '%.4g'%d['value'], 'frac %.3f'%d['roofline']['frac'], '%.2f ms/step'%d['ms_per_step'], d['clocks']['sm_mhz'])"
done
