# k-slice stride padding x tile dealing at K2000/8192 (cfg hashes must match within an order)
set -x
for pad in 0 1 9 40; do
  for o in mmajor skew block; do NMFA_SLICE_PAD=$pad NMFA_TILE_ORDER=$o timeout 120 python tools/probe_clk.py "pad=$pad $o"; done
done > gpurun_out/pad_study.log 2>&1
grep -E "us/sweep|sha1" gpurun_out/pad_study.log
