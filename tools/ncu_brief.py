"""One-screen summary of .ncu-rep files: time, DRAM bytes, hit rates, issue, top stalls."""
import csv, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size"]
for f in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", f, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u = rows[0], rows[1]
    for v in rows[2:]:
        d = dict(zip(h, v)); un = dict(zip(h, u))
        print(f"== {f}: {d.get('Kernel Name')}")
        for k in KEYS:
            print(f"  {k} = {d.get(k)} {un.get(k, '')}")
        st = sorted(((float(x), k.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""))
                     for k, x in d.items() if k.startswith("smsp__average_warps_issue_stalled_")
                     and k.endswith("_per_issue_active.ratio") and x not in ("", "n/a")), reverse=True)
        print("  stalls/issue:", ", ".join(f"{k} {x:.2f}" for x, k in st[:7]))
