# round-2 evidence refresh: every workload's bench line and reference arm
set -x
mkdir -p gpurun_out/ev
timeout 900 python bench.py > gpurun_out/ev/bench_k2000.json 2> gpurun_out/ev/k2000.err
timeout 600 python bench.py --impl reference > gpurun_out/ev/bench_k2000_reference_arm.json 2> gpurun_out/ev/k2000_ref.err
for w in sk100 moebius100 g2000 moebius131072 torus sk65536 ground26; do
  timeout 900 python bench.py --workload $w --no-stats --no-tts > gpurun_out/ev/bench_$w.json 2> gpurun_out/ev/$w.err
done
for w in sk100 moebius100 g2000 moebius131072 torus; do
  timeout 900 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > gpurun_out/ev/bench_${w}_reference_arm.json 2> gpurun_out/ev/ref_$w.err
done
for f in gpurun_out/ev/*.json; do echo "$f $(head -c 200 $f)"; done
