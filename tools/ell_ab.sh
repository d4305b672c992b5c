# toroidal (degree 4) graphs: ELL K=4 (V=2 / V=1) vs CSR
mkdir -p gpurun_out
python -m paper_1806_08422_b200.build > /dev/null 2>&1
P="timeout 200 python tools/prof_sparse_large.py"
echo "-- torus ELL V=2"; PROF_TORUS=1 $P 131044 1024
echo "-- torus ELL V=1"; PROF_TORUS=1 NMFA_SPARSE_V=1 $P 131044 1024
echo "-- torus CSR"; PROF_TORUS=1 NMFA_SPARSE_CSR=1 $P 131044 1024
echo "-- torus ELL G sweep"; for g in 2 4 8; do PROF_TORUS=1 NMFA_ELL_G=$g $P 131044 1024; done
