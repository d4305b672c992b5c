#!/bin/bash
# per-tile clock64 traces of CTA 0 for the full kernel and the no-epilogue variant
mkdir -p gpurun_out
NMFA_TRACE=gpurun_out/trace_full.txt timeout 100 python tools/prof_dense.py 40 > /dev/null 2>&1
NMFA_NVCC_DEFS="-DNMFA_DBG_NOEPI" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
NMFA_TRACE=gpurun_out/trace_noepi.txt timeout 100 python tools/prof_dense.py 40 > /dev/null 2>&1
NMFA_NVCC_DEFS="-DNMFA_DBG_NOMEM" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
NMFA_TRACE=gpurun_out/trace_nomem.txt timeout 100 python tools/prof_dense.py 40 > /dev/null 2>&1
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
for v in full noepi nomem; do echo "== $v"; python tools/trace_persist.py gpurun_out/trace_$v.txt 3; done
