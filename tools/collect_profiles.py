"""Copy a profile_round.sh run from gpurun_out/ into profiles/r01/ and
refresh profiles/ncu_summary.json (per-launch DRAM bytes the bench reads)."""
import json, os, shutil, subprocess, sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
G, P = os.path.join(REPO, "gpurun_out"), os.path.join(REPO, "profiles", "r01")
for f in ["bench_k2000", "bench_moebius131072", "bench_torus", "bench_sk100", "bench_g2000", "bench_moebius100",
          "bench_ground26", "bench_sk65536_g1"]:
    src = os.path.join(G, f + ".json")
    if os.path.exists(src):
        lines = [l for l in open(src).read().splitlines() if l.startswith("{")]
        if lines:
            open(os.path.join(P, f + ".json"), "w").write(lines[-1] + "\n")
if os.path.exists(os.path.join(G, "launches.csv")):
    shutil.copy(os.path.join(G, "launches.csv"), os.path.join(P, "launches_bench_k2000.csv"))
args = []
for w in ("dense", "small", "sparse"):
    rep = os.path.join(G, f"prof_{w}.ncu-rep")
    if os.path.exists(rep):
        args += [w, rep]
        with open(os.path.join(P, f"ncu_details_{w}.csv"), "w") as fh:
            subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], stdout=fh, check=True)
summ = subprocess.run([sys.executable, os.path.join(REPO, "tools", "ncu_summary.py"), *args],
                      capture_output=True, text=True, check=True).stdout
open(os.path.join(P, "ncu_full_summary.json"), "w").write(summ)
d = json.loads(summ)
out = json.load(open(os.path.join(REPO, "profiles", "ncu_summary.json")))
if "dense" in d:
    out["k2000"]["dram_bytes_per_launch"] = (d["dense"]["dram_read"] + d["dense"]["dram_write"]) / 4
if "sparse" in d:
    out["moebius131072"]["dram_bytes_per_launch"] = d["sparse"]["dram_read"] + d["sparse"]["dram_write"]
if "small" in d:
    out["sk100"]["dram_bytes_per_launch"] = (d["small"]["dram_read"] + d["small"]["dram_write"]) / 1000
json.dump(out, open(os.path.join(REPO, "profiles", "ncu_summary.json"), "w"), indent=1)
print({k: v["dram_bytes_per_launch"] for k, v in out.items()})
