# functional check of bench.py's N > 1 code path on the one-GPU box (both ranks on cuda:0, host gloo
# collectives; NOT a timing), final build: K2000 replica mode, SK65536 row-sharded mode, the reference arm
set -x
export NMFA_BENCH_SHARED_GPU=1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline --no-tts --no-stats > gpurun_out/n2_k2000.json 2> gpurun_out/n2_k2000.err; echo "k2000 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29532 bench.py --gpus 2 --workload sk65536 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/n2_sk65536.json 2> gpurun_out/n2_sk65536.err; echo "sk65536 rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --impl reference --steps 3 --warmup 3 > gpurun_out/n2_ref.json 2> gpurun_out/n2_ref.err; echo "ref rc=$?"
wc -l gpurun_out/n2_*.json; for f in gpurun_out/n2_*.json; do head -c 300 $f; echo; done
