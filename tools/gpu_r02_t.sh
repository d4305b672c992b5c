# CSR staged segment: registers per lane (2, 3, 4) against the unstaged kernel
set -x
for v in "-DNMFA_CSR_UNSTAGED" "-DNMFA_CSR_STAGE_REGS=2" "-DNMFA_CSR_STAGE_REGS=3" "-DNMFA_CSR_STAGE_REGS=4"; do
  NMFA_NVCC_DEFS="$v" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
  echo "== $v"; timeout 300 python tools/csr_probe.py 2>&1 | grep n=
  NMFA_SPARSE_CSR=1 timeout 120 python tools/sparse_groups_ab.py moebius
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
