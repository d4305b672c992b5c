# full GPU test suite + moebius131072 / k2000 bench lines
mkdir -p gpurun_out
python -m paper_1806_08422_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python bench.py --workload moebius131072 --steps 5 --warmup 3 --no-tts > gpurun_out/bench_moebius131072.json 2> gpurun_out/bench_m.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_moebius131072.json').read().strip().splitlines()[-1])
print('moebius131072', d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['traffic'], d['e2e']['value'])"
