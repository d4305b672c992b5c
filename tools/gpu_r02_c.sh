# dense schedule study: sweep time per (tile order, K order), then NMFA_TRACE2 timelines
set -x
for cfg in mmajor:natural block:natural block:rotate block:rotm block:rotmn mmajor:rotm; do
  o=${cfg%%:*}; k=${cfg##*:}
  if [ $k = natural ]; then NMFA_TILE_ORDER=$o timeout 120 python tools/probe_clk.py "$o/$k"; else NMFA_TILE_ORDER=$o NMFA_KORDER=$k timeout 120 python tools/probe_clk.py "$o/$k"; fi
done > gpurun_out/sched_study.log 2>&1
for cfg in mmajor:natural block:rotmn; do
  o=${cfg%%:*}; k=${cfg##*:}
  if [ $k = natural ]; then NMFA_TILE_ORDER=$o NMFA_TRACE2=gpurun_out/t2_${o}_${k}.txt timeout 100 python tools/prof_dense.py 12 > /dev/null 2>&1
  else NMFA_TILE_ORDER=$o NMFA_KORDER=$k NMFA_TRACE2=gpurun_out/t2_${o}_${k}.txt timeout 100 python tools/prof_dense.py 12 > /dev/null 2>&1; fi
done
ls -la gpurun_out/; cat gpurun_out/sched_study.log | grep us/sweep
