# small-kernel sincos table: full GPU suite, the default bench line (TTS99 SK100), SK100 / Moebius-100 lines
set -x
timeout 2000 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu_full6.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu_full6.log
timeout 900 python bench.py > gpurun_out/bench_k2000_t.json 2>/dev/null; echo "bench rc=$?"
for w in sk100 moebius100; do timeout 900 python bench.py --workload $w --no-stats --no-tts > gpurun_out/bench_${w}_t.json 2>/dev/null; done
python - <<'PY'
import json
for f in ["gpurun_out/bench_k2000_t.json", "gpurun_out/bench_sk100_t.json", "gpurun_out/bench_moebius100_t.json"]:
    d = json.loads(open(f).read().splitlines()[-1])
    print(f, d["value"], d["roofline"]["frac"], d["e2e"]["value"], d.get("tts99_sk100", {}).get("gpu", {}).get("tts99_s"))
PY
