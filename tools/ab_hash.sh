#!/bin/bash
# configuration hash + sweep time of the K2000 probe per compile-time variant (bitwise-equality A/B)
for v in "$@"; do
  NMFA_NVCC_DEFS="$v" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1 || { echo "build '$v' failed"; continue; }
  timeout 120 python tools/probe_clk.py "${v:-default}" 2>&1 | tr '\n' ' '; echo
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
