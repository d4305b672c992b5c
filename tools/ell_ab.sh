# CSR general path: entries per row per round (NMFA_CSR_ROUNDS) 1 (old .so) vs 2 vs 4
mkdir -p gpurun_out
P="timeout 300 python tools/prof_sparse_large.py"
cp tools/_ab/old.so paper_1806_08422_b200/libnmfa_b200.so
echo "-- rounds=1"; PROF_ER=5,10,20 $P 65536 1024; PROF_TORUS=1 NMFA_SPARSE_CSR=1 $P 65536 1024
for r in 4 2; do
  NMFA_NVCC_DEFS="-DNMFA_CSR_ROUNDS=$r" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
  echo "-- rounds=$r"; PROF_ER=5,10,20 $P 65536 1024; PROF_TORUS=1 NMFA_SPARSE_CSR=1 $P 65536 1024
done
timeout 600 python -m pytest tests/test_gpu_sparse_ell.py -m gpu -x -q 2>&1 | tail -1
