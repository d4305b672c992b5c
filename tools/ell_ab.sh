# ELL sparse kernel occupancy A/B: NMFA_ELL_MINB (blocks per SM, compile time) x replicas per lane
mkdir -p gpurun_out
P="timeout 200 python tools/prof_sparse_large.py"
for mb in 2 3 4; do
  NMFA_NVCC_DEFS="-DNMFA_ELL_MINB=$mb" python -m paper_1806_08422_b200.build --force 2>&1 | grep -A2 "Compiling entry.*sparse_ell" | grep -E "spill" | tr '\n' ' '; echo
  echo "-- minB=$mb V=2"; $P 131072 1024
  echo "-- minB=$mb V=1"; NMFA_SPARSE_V=1 $P 131072 1024
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_sparse_ell.py -m gpu -x -q 2>&1 | tail -1
NMFA_SPARSE_V=1 timeout 600 python -m pytest tests/test_gpu_sparse_ell.py -m gpu -x -q 2>&1 | tail -1
