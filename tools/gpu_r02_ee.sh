# ELL kernel: separate seeded / injected instances (default) against one instance with a run-time branch
set -x
for rep in 1 2; do
for v in "-DNMFA_ELL_SPLIT_INJ=0" ""; do
  NMFA_NVCC_DEFS="$v" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
  for w in moebius torus; do timeout 120 python tools/sparse_groups_ab.py $w | sed "s/^/${v:-split} /"; done
done
done
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
