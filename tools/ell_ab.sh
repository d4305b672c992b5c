# ELL interior-group fast path (NMFA_ELL_FULL_GROUPS) A/B
mkdir -p gpurun_out
for fg in 0 1 0 1; do
  NMFA_NVCC_DEFS="-DNMFA_ELL_FULL_GROUPS=$fg" python -m paper_1806_08422_b200.build --force 2>&1 | grep -A2 "sparse_ell_kernelILi2ELi3" | grep -E "spill" | tr '\n' ' '
  echo "-- full_groups=$fg"; timeout 200 python tools/prof_sparse_large.py 131072 1024
done
NMFA_NVCC_DEFS="-DNMFA_ELL_FULL_GROUPS=1" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_sparse_ell.py -m gpu -x -q 2>&1 | tail -1
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
