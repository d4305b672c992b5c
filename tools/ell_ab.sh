# CSR kernel on long rows: two replicas per lane (16 warps/SM) vs one (32 warps/SM)
mkdir -p gpurun_out
python -m paper_1806_08422_b200.build > /dev/null 2>&1
P="timeout 300 python tools/prof_sparse_large.py"
echo "-- V=2"; PROF_ER=5,10,20 $P 65536 1024
echo "-- V=1"; PROF_ER=5,10,20 NMFA_SPARSE_V=1 $P 65536 1024
