# replica groups, refined rule (>= 3.75 tiles per pair per group): the size sweeps again
set -x
export NMFA_DENSE_VERBOSE=1
timeout 900 python tools/dense_size_sweep.py 2>&1 | grep -v "^$" | paste - - | sed "s/dense plan: //"
timeout 600 python tools/dense_size_sweep.py 1000,1200,1500 16384,32768 100 2>&1 | grep -v "^$" | paste - - | sed "s/dense plan: //"
timeout 900 python tools/dense_size_sweep.py 10000,12000 4096,8192 20 2>&1 | grep -v "^$" | paste - - | sed "s/dense plan: //"
NMFA_PROBE_R=65536 timeout 300 python tools/probe_clk.py "K2000 R=65536 auto" 2>&1 | tr '\n' ' '; echo
timeout 600 python bench.py --workload sk65536 --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().splitlines()[-1]); print('sk65536', d['value'], d['clocks']['sm_mhz'])"
