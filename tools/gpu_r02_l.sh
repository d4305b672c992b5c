# replica groups where J itself outgrows L2: large N, and the row-sharded SK65536 line at G = 1
set -x
export NMFA_DENSE_VERBOSE=1
timeout 600 python bench.py --workload sk65536 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sk65536_auto.json 2> gpurun_out/sk65536_auto.err; echo rc=$?
NMFA_DENSE_GROUPS=1 timeout 600 python bench.py --workload sk65536 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/sk65536_g1.json 2> gpurun_out/sk65536_g1.err; echo rc=$?
grep "dense plan" gpurun_out/sk65536_*.err | sort | uniq -c
echo "== large N, automatic"; timeout 900 python tools/dense_size_sweep.py 10000,12000 4096,8192 20 2>&1
echo "== large N, one group"; NMFA_DENSE_GROUPS=1 timeout 900 python tools/dense_size_sweep.py 10000,12000 4096,8192 20 2>&1
