# ELL look-ahead A/B (NMFA_ELL_LOOKAHEAD compile switch) + identity tests
mkdir -p gpurun_out
P="timeout 200 python tools/prof_sparse_large.py"
for la in 0 1; do
  NMFA_NVCC_DEFS="-DNMFA_ELL_LOOKAHEAD=$la" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
  echo "-- lookahead=$la V=2"; $P 131072 1024
  echo "-- lookahead=$la V=1"; NMFA_SPARSE_V=1 $P 131072 1024
  timeout 600 python -m pytest tests/test_gpu_sparse_ell.py -m gpu -x -q 2>&1 | tail -1
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
