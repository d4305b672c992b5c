# SK N=65,536 at 8192 reads (SURVEY 8(d) C5's larger R) on one GPU: automatic replica groups vs forced
set -x
for g in "" 1 4 8; do
  NMFA_DENSE_VERBOSE=1 NMFA_DENSE_GROUPS=$g timeout 900 python bench.py --workload sk65536 --reads 8192 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/sk65536_r8192_g${g:-auto}.json 2> gpurun_out/sk65536_r8192_g${g:-auto}.err
  grep "dense plan" gpurun_out/sk65536_r8192_g${g:-auto}.err | head -1
  python -c "import json; d=json.loads(open('gpurun_out/sk65536_r8192_g${g:-auto}.json').read().splitlines()[-1]); print('groups=${g:-auto}', d['value'], d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
