# ncu --set full of the final round-2 kernels: the dense kernel over one full K2000 bench launch
# (t_f = 1000 + energy pass) and the small kernel over one SK100 launch (37,888 reads, t_f = 1000)
set -x
PROF_TF=1000 timeout 900 ncu --set full --clock-control none --import-source on -k regex:dense_anneal --launch-skip 1 -c 1 -f -o gpurun_out/ncu_dense_k2000_final python tools/prof_paths.py dense > gpurun_out/ncu_dense_final.log 2>&1; echo "dense rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:small_anneal --launch-skip 1 -c 1 -f -o gpurun_out/ncu_small_sk100_final python tools/prof_paths.py small > gpurun_out/ncu_small_final.log 2>&1; echo "small rc=$?"
