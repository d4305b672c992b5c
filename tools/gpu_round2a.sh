set -x
python -m pytest tests/test_gpu_statistics.py tests/test_gpu_regressions.py -m gpu -q -s > gpurun_out/t2.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b2.log 2>&1
for tool in memcheck racecheck synccheck; do
  SAN_TF=4 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_paths.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?" >> gpurun_out/san_$tool.log
done
tail -3 gpurun_out/t2.log; tail -2 gpurun_out/san_*.log
