# CSR kernel: staged segment path (default) against the unstaged kernel (-DNMFA_CSR_UNSTAGED)
set -x
NMFA_NVCC_DEFS="-DNMFA_CSR_UNSTAGED" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
echo "== unstaged"; timeout 300 python tools/csr_probe.py 2>&1 | grep n=
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
echo "== staged"; timeout 300 python tools/csr_probe.py 2>&1 | grep n=
