# HILO on the small path too: tests, and the cost on SK100 / Moebius-100 (small kernel)
set -x
timeout 1500 python -m pytest tests/test_gpu_hilo.py tests/test_gpu_properties.py tests/test_gpu_refnoise.py tests/test_gpu_parity.py -q -s > gpurun_out/pytest_hilo2.log 2>&1; echo "tests rc=$?"
grep -E "HILO|seeds|passed|failed|Error" gpurun_out/pytest_hilo2.log | tail -30
for f in fp16 hilo; do
  timeout 600 python bench.py --workload sk100 --field $f --steps 5 --warmup 3 --no-cpu-baseline --no-tts --no-stats > gpurun_out/bench_sk100_$f.json 2>/dev/null; echo "sk100 $f rc=$?"
done
python -c "
import json
for f in ['fp16','hilo']:
    d=json.loads(open(f'gpurun_out/bench_sk100_{f}.json').read().splitlines()[-1]); print('sk100', f, d['value'], d['dtype'])"
