# sparse kernels after a change: ELL==CSR identity + sparse parity tests, then timing
mkdir -p gpurun_out
python -m paper_1806_08422_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_sparse_ell.py -m gpu -x -q 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "sparse" 2>&1 | tail -1
P="timeout 200 python tools/prof_sparse_large.py"
echo "-- CSR"; NMFA_SPARSE_CSR=1 $P 131072 1024
echo "-- ELL"; $P 131072 1024
echo "-- ELL"; $P 131072 1024
