# the reference arm (--impl reference) for every BASELINE workload line
mkdir -p gpurun_out
for w in sk100 moebius100 g2000 moebius131072 torus; do
  timeout 900 python bench.py --impl reference --workload $w --steps 3 --warmup 1 > gpurun_out/bench_${w}_reference_arm.json 2> gpurun_out/ref_$w.err
  tail -c 300 gpurun_out/bench_${w}_reference_arm.json; echo
done
