# readiness prefetch: timing for m-major vs skew dealing, trace, dense parity + checked build
set -x
for R in 4096 8192 12288; do
  for o in mmajor skew; do NMFA_PROBE_R=$R NMFA_TILE_ORDER=$o timeout 120 python tools/probe_clk.py "R=$R $o"; done
done > gpurun_out/prefetch_study.log 2>&1
NMFA_TILE_ORDER=skew NMFA_TRACE2=gpurun_out/t2_skew_pf.txt timeout 100 python tools/prof_dense.py 12 > /dev/null 2>&1
NMFA_TILE_ORDER=mmajor NMFA_TRACE2=gpurun_out/t2_mmajor_pf.txt timeout 100 python tools/prof_dense.py 12 > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_sharded.py tests/test_gpu_guarded.py tests/test_gpu_refnoise.py -m gpu -q -x -p no:cacheprovider > gpurun_out/t_g.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_g.log
grep -E "us/sweep|sha1" gpurun_out/prefetch_study.log; tail -3 gpurun_out/t_g.log
