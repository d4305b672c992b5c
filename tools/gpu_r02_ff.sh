# ring stages sized per plan (default) against kMaxW-sized stages (NMFA_STAGE_FULL=1): K2000 probe + small-N sweep
set -x
for rep in 1 2; do
for f in 1 0; do
  NMFA_STAGE_FULL=$f timeout 120 python tools/probe_clk.py "full=$f" 2>&1 | tr '\n' ' '; echo
  NMFA_STAGE_FULL=$f timeout 300 python tools/dense_size_sweep.py 800,1000,1500 8192,16384 100 2>&1 | grep N= | sed "s/^/full=$f /"
done
done
