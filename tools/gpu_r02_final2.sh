# round-2 final evidence (after replica groups + HILO): every workload's bench line and reference
# arm, the default K2000 line, smoke, and the launch list of the bench command
set -x
mkdir -p gpurun_out/ev2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev2/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/ev2/smoke.log
timeout 900 python bench.py > gpurun_out/ev2/bench_k2000.json 2> gpurun_out/ev2/k2000.err
timeout 600 python bench.py --impl reference > gpurun_out/ev2/bench_k2000_reference_arm.json 2> gpurun_out/ev2/k2000_ref.err
for w in sk100 moebius100 g2000 moebius131072 torus sk65536 ground26; do
  timeout 900 python bench.py --workload $w --no-stats --no-tts > gpurun_out/ev2/bench_$w.json 2> gpurun_out/ev2/$w.err
done
for w in sk100 moebius100 g2000 moebius131072 torus; do
  timeout 900 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > gpurun_out/ev2/bench_${w}_reference_arm.json 2> gpurun_out/ev2/ref_$w.err
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ev2/launches_bench_k2000.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-tts --no-stats > gpurun_out/ev2/ncu.log 2>&1; echo "ncu rc=$?"
for f in gpurun_out/ev2/*.json; do echo "$f $(head -c 160 $f)"; done
tail -2 gpurun_out/ev2/smoke.log
