#!/bin/bash
# A/B of dense-kernel variants (compile-time switches) at K2000 / 8192 reads
run() { NMFA_NVCC_DEFS="$2" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1 || { echo build failed; return; }; timeout 100 python tools/probe_clk.py "$1"; }
for v in "$@"; do
  case $v in
    full) run full "";;
    noepi) run noepi "-DNMFA_DBG_NOEPI";;
    nomem) run nomem "-DNMFA_DBG_NOMEM";;
    epi12) run epi12 "-DNMFA_EPI_WARPS=12";;
    *) run "$v" "$v";;
  esac
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
