# CSR: a third staged register (segments up to 96 entries) against two
set -x
for rep in 1 2; do
for v in "" "-DNMFA_CSR_STAGED96=1"; do
  NMFA_NVCC_DEFS="$v" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
  echo "== ${v:-two}"; timeout 300 python tools/csr_probe.py 2>&1 | grep n=
done
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
