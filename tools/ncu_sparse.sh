# ncu --set full of the sparse kernel (ELL when max degree <= 4) on moebius_ladder(131072), R=1024 (one launch)
# usage: bash tools/ncu_sparse.sh [tag] [extra env assignments...]
set -e
mkdir -p gpurun_out
tag=${1:-sparse_ell}; shift || true
env "$@" timeout 300 python tools/prof_sparse_one.py ${PROF_GRAPH:-moebius}
env "$@" timeout 900 ncu --set full --clock-control none --import-source on -k regex:sparse_ -s 2 -c 1 \
  -o gpurun_out/$tag -f python tools/prof_sparse_one.py ${PROF_GRAPH:-moebius} > gpurun_out/ncu_$tag.log 2>&1
