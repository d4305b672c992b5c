# replica groups: new test, K2000 with all 65,536 reads on one GPU, the default bench line
set -x
timeout 600 python -m pytest tests/test_gpu_dense_groups.py -q > gpurun_out/pytest_groups.log 2>&1; echo "groups test rc=$?"; tail -2 gpurun_out/pytest_groups.log
timeout 900 python bench.py --reads 65536 --steps 5 --warmup 3 --no-cpu-baseline --no-tts --no-stats > gpurun_out/bench_k2000_65536.json 2> gpurun_out/bench_k2000_65536.err; echo "bench65536 rc=$?"
timeout 900 python bench.py > gpurun_out/bench_k2000_default.json 2> gpurun_out/bench_k2000_default.err; echo "bench rc=$?"
