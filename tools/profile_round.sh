#!/bin/bash
# Evidence for profiles/: GPU tests, bench lines, launch list of the bench command, ncu --set full per path.
mkdir -p gpurun_out
python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_k2000.json 2> gpurun_out/bench_k2000.err; tail -c 300 gpurun_out/bench_k2000.json
python bench.py --workload moebius131072 --steps 5 --warmup 3 --no-tts > gpurun_out/bench_moebius131072.json 2> gpurun_out/bench_m.err
python bench.py --workload sk100 --steps 5 --warmup 3 --no-tts --no-cpu-baseline > gpurun_out/bench_sk100.json 2> gpurun_out/bench_s.err
python bench.py --workload g2000 --steps 5 --warmup 3 --no-tts --no-cpu-baseline > gpurun_out/bench_g2000.json 2> gpurun_out/bench_g.err
python bench.py --workload torus --steps 5 --warmup 3 --no-tts > gpurun_out/bench_torus.json 2> gpurun_out/bench_t.err
python bench.py --workload moebius100 --steps 5 --warmup 3 --no-tts --no-cpu-baseline > gpurun_out/bench_moebius100.json 2> gpurun_out/bench_m100.err
python bench.py --workload ground26 --steps 5 --warmup 3 > gpurun_out/bench_ground26.json 2> gpurun_out/bench_gr.err
python bench.py --workload sk65536 --steps 2 --warmup 1 > gpurun_out/bench_sk65536_g1.json 2> gpurun_out/bench_sk.err
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-tts > gpurun_out/plain.json 2> gpurun_out/plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-tts > gpurun_out/ncu_launch.log 2>&1
for w in dense small sparse; do
  python tools/prof_paths.py $w > gpurun_out/plain_$w.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"dense_anneal|small_anneal|sparse_step|sparse_ell" -s 1 -c 1 \
      -o gpurun_out/prof_$w python tools/prof_paths.py $w > gpurun_out/ncu_$w.log 2>&1
done
echo done
