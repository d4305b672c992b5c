# ncu --set full of the round-2 dense kernel: one full K2000 launch (t_f = 1000, 8192 reads,
# the bench's launch) and a 64-sweep launch; the ELL kernel on Moebius-131072; power limit
set -x
nvidia-smi -q -d POWER > gpurun_out/power.txt 2>&1
PROF_TF=1000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_anneal --launch-skip 1 -c 1 -f -o gpurun_out/ncu_dense_k2000 python tools/prof_paths.py dense > gpurun_out/ncu_dense_k2000.log 2>&1; echo "ncu dense rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_anneal --launch-skip 1 -c 1 -f -o gpurun_out/ncu_dense64_r2 python tools/prof_dense.py 64 > gpurun_out/ncu_dense64_r2.log 2>&1; echo "ncu dense64 rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_ell --launch-skip 2 -c 1 -f -o gpurun_out/ncu_ell python tools/prof_paths.py sparse > gpurun_out/ncu_ell.log 2>&1; echo "ncu ell rc=$?"
grep -E "Power Limit|Enforced|Default" gpurun_out/power.txt | head
