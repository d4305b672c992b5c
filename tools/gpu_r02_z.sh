# dense kernel back-off constants: producer mailbox poll and prefetch-thread readiness poll (K2000 probe)
set -x
for rep in 1 2; do
for v in "" "-DNMFA_PF_SLEEP_NS=0" "-DNMFA_PF_SLEEP_NS=100" "-DNMFA_POLL_SLEEP_NS=0" "-DNMFA_POLL_SLEEP_NS=128" "-DNMFA_POLL_SLEEP_NS=512"; do
  NMFA_NVCC_DEFS="$v" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
  timeout 120 python tools/probe_clk.py "${v:-default}" 2>&1 | head -1
done
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
