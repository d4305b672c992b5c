# replay-mode tests + ncu of mmajor vs skew dealing (12-sweep K2000 launches)
set -x
timeout 900 python -m pytest tests/test_gpu_refnoise.py -m gpu -q -s -p no:cacheprovider > gpurun_out/t_f.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_f.log
for o in mmajor skew; do
  NMFA_TILE_ORDER=$o timeout 600 ncu --set full --clock-control none -k regex:dense_anneal --launch-skip 1 -c 1 -f -o gpurun_out/ncu_$o python tools/prof_dense.py 12 > gpurun_out/ncu_$o.log 2>&1; echo "ncu $o rc=$?"
done
grep -E "passed|failed|identical|rc=|Error" gpurun_out/t_f.log | tail -12
