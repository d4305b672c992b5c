# CSR staged segment (two registers per lane, unconditional shuffles) against the unstaged kernel
set -x
for v in "-DNMFA_CSR_UNSTAGED" ""; do
  NMFA_NVCC_DEFS="$v" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
  echo "== ${v:-staged}"; timeout 300 python tools/csr_probe.py 2>&1 | grep n=
  NMFA_SPARSE_CSR=1 timeout 120 python tools/sparse_groups_ab.py moebius
done
