# round 2 pass b: checked-build test, headline trajectories (R=256), ncu --set full of a 64-sweep dense launch
set -x
timeout 1200 python -m pytest tests/test_gpu_guarded.py tests/test_gpu_headline_trajectory.py -m gpu -q -s -p no:cacheprovider > gpurun_out/t_b.log 2>&1; echo "tests rc=$?" >> gpurun_out/t_b.log
timeout 600 python tools/prof_dense.py 64 > gpurun_out/prof_dense64.log 2>&1; echo "plain rc=$?" >> gpurun_out/prof_dense64.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_anneal --launch-skip 1 -c 1 -f -o gpurun_out/ncu_dense64 python tools/prof_dense.py 64 > gpurun_out/ncu_dense64.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_dense64.log
grep -E "passed|failed|rc=|flips|guard|product" gpurun_out/t_b.log | tail -12; tail -2 gpurun_out/ncu_dense64.log
