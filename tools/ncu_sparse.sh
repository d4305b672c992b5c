# ncu --set full of the V=2 CSR kernel on moebius_ladder(131072), R=1024 (one launch)
set -e
mkdir -p gpurun_out
timeout 300 python tools/prof_sparse_one.py
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_step_kernel -s 2 -c 1 \
  -o gpurun_out/sparse_v2 -f python tools/prof_sparse_one.py > gpurun_out/ncu_sparse.log 2>&1
