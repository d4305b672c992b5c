# skewed E/L dealing vs m-major: sweep time at several R (cfg hashes must match), trace, dense tests
set -x
for R in 4096 6144 8192 12288; do
  for o in mmajor skew; do NMFA_PROBE_R=$R NMFA_TILE_ORDER=$o timeout 120 python tools/probe_clk.py "R=$R $o"; done
done > gpurun_out/skew_study.log 2>&1
NMFA_TILE_ORDER=skew NMFA_TRACE2=gpurun_out/t2_skew.txt timeout 100 python tools/prof_dense.py 12 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_sharded.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_d.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_d.log
grep -E "us/sweep|sha1" gpurun_out/skew_study.log; tail -3 gpurun_out/t_d.log
