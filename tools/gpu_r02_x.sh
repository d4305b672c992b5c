set -x
for v in "-DNMFA_CSR_BATCH=16" "-DNMFA_CSR_BATCH=24" "-DNMFA_CSR_BATCH=32"; do
  NMFA_NVCC_DEFS="$v" python -m paper_1806_08422_b200.build --force 2>&1 | grep -E "sparse_step_kernelILi2" -A3 | grep spill
  echo "== $v"; timeout 300 python tools/csr_probe.py 2>&1 | grep n= | head -8
done
