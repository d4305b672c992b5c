# sparse path: CUDA-graph replay of the t_f steps (default) vs direct launches (NMFA_SPARSE_GRAPH=0)
mkdir -p gpurun_out
python -m paper_1806_08422_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_sparse_ell.py tests/test_gpu_noise.py tests/test_gpu_fuzz.py -m gpu -x -q 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
for g in 1 0; do
  echo "-- graph=$g"
  NMFA_SPARSE_GRAPH=$g python tools/prof_sparse_small.py
  NMFA_SPARSE_GRAPH=$g timeout 200 python tools/prof_sparse_large.py 131072 1024
done
