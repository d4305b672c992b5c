# experiment: persisting L2 window over the two hi images (NMFA_L2_PERSIST), with and without the epilogue's
# explicit cache-policy hints (-DNMFA_DBG_PLAINMEM); K2000 probe, alternating
set -x
for rep in 1 2; do
  python -m paper_1806_08422_b200.build > /dev/null 2>&1
  timeout 120 python tools/probe_clk.py "default" 2>&1 | tr '\n' ' '; echo
  NMFA_L2_PERSIST=1 timeout 120 python tools/probe_clk.py "persist" 2>&1 | tr '\n' ' '; echo
  NMFA_NVCC_DEFS="-DNMFA_DBG_PLAINMEM" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
  NMFA_L2_PERSIST=1 timeout 120 python tools/probe_clk.py "persist+plainmem" 2>&1 | tr '\n' ' '; echo
  timeout 120 python tools/probe_clk.py "plainmem" 2>&1 | tr '\n' ' '; echo
  python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
done
