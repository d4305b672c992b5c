# L2-aware replica groups: bitwise identity (cfg hash) across forced group
# counts, then throughput with the automatic split vs one group
set -x
python -m paper_1806_08422_b200.build > /dev/null 2>&1
export NMFA_DENSE_VERBOSE=1
for g in "" 1 2 4; do NMFA_DENSE_GROUPS=$g timeout 120 python tools/probe_clk.py "K2000 R=8192 groups=${g:-auto}" 2>&1 | tr '\n' ' '; echo; done
for g in "" 1 2; do NMFA_PROBE_R=65536 NMFA_DENSE_GROUPS=$g timeout 300 python tools/probe_clk.py "K2000 R=65536 groups=${g:-auto}" 2>&1 | tr '\n' ' '; echo; done
echo "== size sweep, automatic groups"; timeout 900 python tools/dense_size_sweep.py 2>&1
echo "== size sweep, one group"; NMFA_DENSE_GROUPS=1 timeout 900 python tools/dense_size_sweep.py 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_j.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu_j.log
