# round 2, first GPU pass: full -m gpu suite (statistics printed), default bench,
# reference arm, sanitizers on every path.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs -s -p no:cacheprovider > gpurun_out/gputests.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/bench_ref.log
for tool in memcheck racecheck synccheck; do
  SAN_TF=4 timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_paths.py > gpurun_out/san_$tool.log 2>&1; echo "$tool rc=$?" >> gpurun_out/san_$tool.log
done
grep -E "passed|failed|rc=" gpurun_out/gputests.log | tail -3; grep -E "^\{|rc=" gpurun_out/bench.log gpurun_out/bench_ref.log | cut -c1-400; tail -n2 gpurun_out/san_*.log
