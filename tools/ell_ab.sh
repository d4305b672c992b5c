# ELL vs CSR sparse kernels: bit-identity tests, timing on large Moebius / cubic graphs
mkdir -p gpurun_out
python -m paper_1806_08422_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_sparse_ell.py -m gpu -x -q 2>&1 | tail -5
for rep in 1 2; do
  echo "-- CSR"; NMFA_SPARSE_CSR=1 timeout 200 python tools/prof_sparse_large.py 131072 1024
  echo "-- ELL"; timeout 200 python tools/prof_sparse_large.py 131072 1024
done
echo "-- ELL R=4096"; timeout 200 python tools/prof_sparse_large.py 131072 4096
