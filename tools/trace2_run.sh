#!/bin/bash
# cross-SM globaltimer timelines (NMFA_TRACE2) + sweep timing for each tile order
mkdir -p gpurun_out
for v in full noepi; do
  if [ $v = noepi ]; then NMFA_NVCC_DEFS="-DNMFA_DBG_NOEPI" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1; fi
  for o in mmajor sorted spin; do
    NMFA_TILE_ORDER=$o NMFA_TRACE2=gpurun_out/t2_${v}_${o}.txt timeout 100 python tools/prof_dense.py 12 > /dev/null 2>&1
    NMFA_TILE_ORDER=$o timeout 100 python tools/probe_clk.py "$v/$o"
  done
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
