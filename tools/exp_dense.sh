#!/bin/bash
# dense-kernel experiment matrix (timing only); leaves the default build in place
run() { echo "== $1"; NMFA_NVCC_DEFS="$2" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1 || { echo build failed; return; }; timeout 120 python tools/probe.py k2000; }
run "16 epi warps (default)" ""
run "12 epi warps" "-DNMFA_EPI_WARPS=12"
run "no epilogue math" "-DNMFA_DBG_NOEPI"
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
