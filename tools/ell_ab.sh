# interior-group stores fast path (NMFA_FULL_GROUP_STORES) A/B
mkdir -p gpurun_out
for fg in 0 1 0 1; do
  NMFA_NVCC_DEFS="-DNMFA_FULL_GROUP_STORES=$fg" python -m paper_1806_08422_b200.build --force 2>&1 | grep -A2 "sparse_ell_kernelILi2ELi3" | grep -E "spill" | tr '\n' ' '
  echo "-- group_stores=$fg"; timeout 200 python tools/prof_sparse_large.py 131072 1024
done
NMFA_NVCC_DEFS="-DNMFA_FULL_GROUP_STORES=1" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_sparse_ell.py tests/test_gpu_fuzz.py -m gpu -x -q 2>&1 | tail -1
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
