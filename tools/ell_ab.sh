# CSR general path: rows longer than 3 interleaved across the group's 8 rows (new) vs serial (old .so)
mkdir -p gpurun_out
P="timeout 300 python tools/prof_sparse_large.py"
cp tools/_ab/old.so paper_1806_08422_b200/libnmfa_b200.so
echo "-- OLD"; PROF_ER=5,10,20 $P 65536 1024; PROF_TORUS=1 NMFA_SPARSE_CSR=1 $P 65536 1024
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
echo "-- NEW"; PROF_ER=5,10,20 $P 65536 1024; PROF_TORUS=1 NMFA_SPARSE_CSR=1 $P 65536 1024
timeout 600 python -m pytest tests/test_gpu_sparse_ell.py -m gpu -x -q 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sparse or g2000 or ragged" 2>&1 | tail -1
