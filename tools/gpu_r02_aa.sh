# sincos table in the dense epilogue: K2000 probe (hash) and small-N sweeps, with and without (-DNMFA_DENSE_TABLE=0)
set -x
for rep in 1 2; do
for v in "-DNMFA_DENSE_TABLE=0" ""; do
  NMFA_NVCC_DEFS="$v" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
  timeout 120 python tools/probe_clk.py "${v:-table}" 2>&1 | tr '\n' ' '; echo
  [ $rep = 1 ] && timeout 300 python tools/dense_size_sweep.py 800,1000,2000 8192,16384 100 2>&1 | grep N=
done
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
