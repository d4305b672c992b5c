#!/bin/bash
NMFA_NVCC_DEFS="$1 -DNMFA_DBG_TRACE" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1 || echo build failed
timeout 100 python tools/prof_dense.py 3
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
