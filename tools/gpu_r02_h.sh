# full GPU suite + default bench + reference arm after the skew/prefetch change
set -x
timeout 1500 python -m pytest tests -m gpu -q -rs -s -p no:cacheprovider > gpurun_out/gputests_h.log 2>&1; echo "tests rc=$?" >> gpurun_out/gputests_h.log
timeout 600 python bench.py > gpurun_out/bench_h.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_h.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_h.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_h.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_h.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-tts --no-stats > gpurun_out/ncu_h.log 2>&1; echo "ncu rc=$?"
grep -E "passed|failed|rc=" gpurun_out/gputests_h.log | tail -3; grep -E "^\{" gpurun_out/bench_h.log | cut -c1-300; tail -2 gpurun_out/smoke_h.log
