# full GPU test suite + the sparse timing and path crossover + moebius131072 bench line
mkdir -p gpurun_out
python -m paper_1806_08422_b200.build > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/prof_sparse_large.py 131072 1024
timeout 600 python tools/path_crossover.py > gpurun_out/path_crossover2.log 2>&1
timeout 600 python bench.py --workload moebius131072 --steps 5 --warmup 3 > gpurun_out/bench_moebius131072.json 2> gpurun_out/bench_moebius131072.err
tail -c 1500 gpurun_out/bench_moebius131072.json
