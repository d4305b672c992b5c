# timing-only: tile order (mmajor / block) x K order (natural / rotate) at K2000, 8192 reads
mkdir -p gpurun_out
python -m paper_1806_08422_b200.build > /dev/null 2>&1
for rep in 1 2; do
for to in mmajor block; do
  for ko in natural rotate; do
    NMFA_TILE_ORDER=$to NMFA_KORDER=$ko timeout 120 python tools/probe_clk.py "$to/$ko" 2>&1 | head -1
  done
done
done
