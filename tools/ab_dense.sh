#!/bin/bash
run() { NMFA_NVCC_DEFS="$2" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1 || { echo build failed; return; }; timeout 100 python tools/probe_clk.py "$1"; }
run noepi "-DNMFA_DBG_NOEPI"
run nomem "-DNMFA_DBG_NOMEM"
run full ""
run noepi "-DNMFA_DBG_NOEPI"
run nomem "-DNMFA_DBG_NOMEM"
run full ""
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
