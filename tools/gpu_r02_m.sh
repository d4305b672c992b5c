# DRAM traffic and L2 hit rate of the K2000 65,536-read anneal (t_f = 50): one launch vs 8 replica groups
set -x
M=dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,gpu__time_duration.sum
NMFA_DENSE_GROUPS=1 timeout 900 ncu --metrics $M --clock-control none -k regex:dense_anneal --launch-skip 1 -c 1 --csv python tools/prof_dense.py 50 65536 > gpurun_out/ncu_groups1.csv 2> gpurun_out/ncu_groups1.err; echo rc=$?
timeout 900 ncu --metrics $M --clock-control none -k regex:dense_anneal --launch-skip 8 -c 8 --csv python tools/prof_dense.py 50 65536 > gpurun_out/ncu_groups8.csv 2> gpurun_out/ncu_groups8.err; echo rc=$?
