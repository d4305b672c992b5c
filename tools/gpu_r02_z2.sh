set -x
for rep in 1 2 3; do
for v in "" "-DNMFA_PF_SLEEP_NS=0" "-DNMFA_PF_SLEEP_NS=0 -DNMFA_POLL_SLEEP_NS=0"; do
  NMFA_NVCC_DEFS="$v" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
  timeout 120 python tools/probe_clk.py "${v:-default}" 2>&1 | head -1
done
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
