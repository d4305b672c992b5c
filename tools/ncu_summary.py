"""Summarise ncu --set full captures into profiles/ (markdown + json)."""
import csv, io, json, subprocess, sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "gpc__cycles_elapsed.max": "cycles_elapsed",
    "sm__cycles_active.avg": "sm_active_cycles",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum": "tma_load_bytes",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
}

def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    h, u, v = r[0], r[1], r[2]
    d = {}
    for name, unit, val in zip(h, u, v):
        if name in METRICS:
            d[METRICS[name]] = (val, unit)
        if name == "Kernel Name":
            d["kernel"] = (val, "")
    return d

def scale(val, unit):
    m = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
         "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9}
    try:
        return float(val.replace(",", "")) * m.get(unit, 1)
    except ValueError:
        return val

res = {}
for tag, rep in zip(sys.argv[1::2], sys.argv[2::2]):
    d = raw(rep)
    res[tag] = {k: scale(*v) for k, v in d.items()}
print(json.dumps(res, indent=1))
