# round-2 final evidence: default bench line, reference arm, launch list, smoke
set -x
mkdir -p gpurun_out/fin
timeout 900 python bench.py > gpurun_out/fin/bench_k2000.json 2> gpurun_out/fin/k2000.err
timeout 600 python bench.py --impl reference > gpurun_out/fin/bench_k2000_reference_arm.json 2> gpurun_out/fin/ref.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/fin/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin/launches_bench_k2000.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-tts --no-stats > gpurun_out/fin/ncu.log 2>&1; echo "ncu rc=$?"
head -c 600 gpurun_out/fin/bench_k2000.json; tail -2 gpurun_out/fin/smoke.log
