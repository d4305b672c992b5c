# global sincos table in the sparse kernels (NMFA_SPARSE_TABLE=0: inline MUFU)
set -x
for rep in 1 2; do
for t in 0 1; do
  NMFA_SPARSE_TABLE=$t timeout 120 python tools/sparse_groups_ab.py moebius
  NMFA_SPARSE_TABLE=$t timeout 120 python tools/sparse_groups_ab.py torus
  NMFA_SPARSE_TABLE=$t timeout 300 python tools/csr_probe.py 2>&1 | grep "R=  4096" | head -3
done
done
