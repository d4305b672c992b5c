# HILO field: the new tests, the headline trajectory cases, the per-seed replay, and its throughput
set -x
timeout 1500 python -m pytest tests/test_gpu_hilo.py tests/test_gpu_headline_trajectory.py -q -s > gpurun_out/pytest_hilo.log 2>&1; echo "hilo tests rc=$?"
grep -E "HILO|hilo|flips|passed|failed|Error" gpurun_out/pytest_hilo.log | head -40
timeout 600 python bench.py --field hilo --steps 5 --warmup 3 --no-cpu-baseline --no-tts --no-stats > gpurun_out/bench_k2000_hilo.json 2> gpurun_out/bench_k2000_hilo.err; echo "bench hilo rc=$?"
