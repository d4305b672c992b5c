#!/bin/bash
# sweep time for tile order x K order (runtime knobs), full kernel
for o in mmajor sorted spin; do
  for k in early natural; do
    NMFA_TILE_ORDER=$o NMFA_KORDER=$k timeout 100 python tools/probe_clk.py "$o/$k"
  done
done
NMFA_TILE_ORDER=mmajor NMFA_TRACE2=gpurun_out/t2_full_mmajor_early.txt timeout 100 python tools/prof_dense.py 12 > /dev/null 2>&1
