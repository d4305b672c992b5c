#!/bin/bash
# per-tile MMA span (NMFA_TRACE2) and sweep time for epilogue ablations; args = define sets
for v in "$@"; do
  if [ "$v" = full ]; then defs=""; else defs=$(echo "$v" | tr "+" " " | sed "s/\([A-Z_=0-9]*\)/-D\1/g"); fi
  NMFA_NVCC_DEFS="$defs" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1 || { echo "$v build failed"; continue; }
  tag=$(echo "$v" | tr '+' '_')
  NMFA_TRACE2=gpurun_out/t2_$tag.txt timeout 100 python tools/prof_dense.py 12 > /dev/null 2>&1
  timeout 100 python tools/probe_clk.py "$v"
  python tools/trace2_report.py gpurun_out/t2_$tag.txt | grep -E "MMA span"
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
