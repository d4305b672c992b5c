# unit-weight ELL A/B (NMFA_ELL_UNIT=0 keeps the weighted kernel) + identity tests
mkdir -p gpurun_out
python -m paper_1806_08422_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_sparse_ell.py -m gpu -x -q 2>&1 | tail -1
P="timeout 200 python tools/prof_sparse_large.py"
for rep in 1 2; do
  echo "-- ELL weighted"; NMFA_ELL_UNIT=0 $P 131072 1024
  echo "-- ELL unit"; $P 131072 1024
done
