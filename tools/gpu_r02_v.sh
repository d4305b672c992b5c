# CSR staged path: rounds of 1 / 2 / 3 entries per row per round trip
set -x
for v in "-DNMFA_CSR_ROUNDS=1" "-DNMFA_CSR_ROUNDS=3" "-DNMFA_CSR_ROUNDS=4"; do
  NMFA_NVCC_DEFS="$v" python -m paper_1806_08422_b200.build --force 2>&1 | grep -E "sparse_step_kernelILi2" -A3 | grep -E "spill" 
  echo "== $v"; timeout 300 python tools/csr_probe.py 2>&1 | grep n=
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
