# NOTE: the NMFA_EPI_INTERLEAVE code was reverted after this run (profiles/r01/korder_ab.log); kept for the record
set -x
bash tools/epi_variants.sh full NMFA_EPI_INTERLEAVE full NMFA_EPI_INTERLEAVE 2>&1 | tee gpurun_out/interleave.log
NMFA_NVCC_DEFS="-DNMFA_EPI_INTERLEAVE" python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sharded.py -m gpu -x -q 2>&1 | tail -3 | tee -a gpurun_out/interleave.log
python -m paper_1806_08422_b200.build --force > /dev/null 2>&1
