#!/bin/bash
# Evidence for profiles/: plain bench, launch list of the same command, ncu --set full per path.
set -x
python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/plain.json 2> gpurun_out/plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
for w in dense small sparse; do
  python tools/prof_paths.py $w > gpurun_out/plain_$w.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"dense_anneal|small_anneal|sparse_step" -s 1 -c 1 \
      -o gpurun_out/prof_$w python tools/prof_paths.py $w > gpurun_out/ncu_$w.log 2>&1
done
echo done
