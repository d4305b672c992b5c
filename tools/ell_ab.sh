# degree-4 ELL register budget: NMFA_ELL4_MINB 2 (128 regs, spills) vs 1 (no cap)
mkdir -p gpurun_out
for mb in 2 1; do
  NMFA_NVCC_DEFS="-DNMFA_ELL4_MINB=$mb" python -m paper_1806_08422_b200.build --force 2>&1 | grep -A2 "sparse_ell_kernelILi2ELi4" | grep -E "spill|Used" | tr '\n' ' '; echo
  echo "-- ELL4 minB=$mb"; PROF_TORUS=1 timeout 200 python tools/prof_sparse_large.py 131044 1024
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
