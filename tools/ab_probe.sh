#!/bin/bash
# timing-only ablations of the dense kernel (results are wrong for DBG builds): probe_clk at K2000/8192
for v in "$@"; do
  NMFA_NVCC_DEFS="$v" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1 || { echo "build '$v' failed"; continue; }
  timeout 120 python tools/probe_clk.py "${v:-default}" | head -1
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
