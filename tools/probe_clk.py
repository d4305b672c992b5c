"""K2000 dense sweep time with nvidia-smi clock/power sampling during the run."""
import sys, os, subprocess, threading, time, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1806_08422_b200 as nb
rows = []
proc = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits", "-lms", "50"],
                        stdout=subprocess.PIPE, text=True)
threading.Thread(target=lambda: [rows.append(l) for l in proc.stdout], daemon=True).start()
p = nb.gen_sk(2000, 7)
R, t_f = int(os.environ.get("NMFA_PROBE_R", 8192)), 1000
params = nb.NmfaParams(t_f=t_f, seed=0)
plan = nb.Plan(p, R, params.schedule.temperatures(t_f), params.alpha, params.sigma)
cfg = torch.empty((R, 2000), dtype=torch.int8, device="cuda")
plan.run(0, 0, config=cfg); torch.cuda.synchronize()
time.sleep(0.3); n0 = len(rows)
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record()
for k in range(4): plan.run(k, 0, config=cfg)
b.record(); torch.cuda.synchronize()
n1 = len(rows); proc.terminate()
t = a.elapsed_time(b) / (4 * t_f)
vals = [l.strip().split(",") for l in rows[n0:n1]]
clk = statistics.median(float(v[0]) for v in vals); pw = statistics.median(float(v[1]) for v in vals)
print(f"{sys.argv[1] if len(sys.argv)>1 else ''}: {t*1e3:.1f} us/sweep  {2*2000*2000*R/(t*1e-3)/1e12:.0f} TFLOP/s  sm_clock {clk:.0f} MHz  power {pw:.0f} W  ({len(vals)} samples)", flush=True)
import hashlib
print(f"  cfg sha1 {hashlib.sha1(cfg.cpu().numpy().tobytes()).hexdigest()[:16]}", flush=True)
