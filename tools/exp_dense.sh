#!/bin/bash
# dense-kernel experiment matrix (timing only); leaves the default build in place
run() { echo "== $1"; NMFA_NVCC_DEFS="$2" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1 || { echo build failed; return; }; timeout 120 python tools/probe.py k2000; }
run "no master ld/st" "-DNMFA_DBG_NOMASTER"
run "no image store" "-DNMFA_DBG_NOIMG"
run "no math" "-DNMFA_DBG_NOMATH"
run "no master, no image" "-DNMFA_DBG_NOMASTER -DNMFA_DBG_NOIMG"
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
