# final-build evidence: full GPU suite, smoke, default bench line, reference arm, every workload line
set -x
mkdir -p gpurun_out/ev3
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/ev3/gputests.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ev3/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev3/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev3/smoke.log
timeout 900 python bench.py > gpurun_out/ev3/bench_k2000.json 2> gpurun_out/ev3/k2000.err
timeout 600 python bench.py --impl reference > gpurun_out/ev3/bench_k2000_reference_arm.json 2> gpurun_out/ev3/k2000_ref.err
for w in sk100 moebius100 g2000 moebius131072 torus gset5000 sk65536 ground26; do
  timeout 900 python bench.py --workload $w --no-stats --no-tts > gpurun_out/ev3/bench_$w.json 2> gpurun_out/ev3/$w.err
done
for f in gpurun_out/ev3/*.json; do echo "$f $(head -c 150 $f)"; done
tail -2 gpurun_out/ev3/smoke.log
