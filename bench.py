"""Benchmark: NMFA spin-updates/s on the K2000 stand-in (BASELINE.json metric).

A "step" is one full NMFA anneal (t_f = 1000 synchronous sweeps, default
schedule, alpha = sigma = 0.15) over one batch of replicas of gen_sk(2000, 7)
(the reference's own K2000 stand-in, calibrate.py:44), including exact
energies and the best-of-reads reduction.  Per GPU the batch is 8192 reads, so
8 GPUs run the 65,536-read K2000 configuration (weak scaling: replicas are
sharded with no data-path collective; one all-gather of each rank's best at
the end).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload k2000|sk100|moebius100|g2000|moebius131072|torus|gset5000|ground26|sk65536]
                    [--reads R] [--field fp16|hilo]

Prints ONE JSON line on rank 0.  --impl reference times the reference's own
per-run loop (`nmfa.nmfa_batch` from the unmodified install in baseline/_ref,
solver.py:236-280 / _kernels_numba.py:64-80; when that install is missing,
the oracle's jitted restatement, oracle/nmfa_oracle.py) on this host's cores,
on a bounded sample of the same workload.  --field hilo measures the dense
path's fidelity mode (NMFA_FIELD_HILO) instead of the default fp16 operand.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

WORKLOADS = {
    # name: (builder, n, reads per GPU, t_f, description)
    "k2000": ("gen_sk(2000, 7)", 2000, 8192, 1000,
              "K2000 stand-in gen_sk(2000,7) (calibrate.py:44), 8192 reads/GPU (65536 on 8), t_f=1000"),
    "sk100": ("gen_sk(100, 0)", 100, 37888, 1000, "SK100 gen_sk(100,0), 37888 reads/GPU, t_f=1000"),
    "moebius100": ("moebius_ladder(100)", 100, 37888, 1000,
                   "Moebius ladder n=100, 37888 reads/GPU, t_f=1000"),
    "g2000": ("gen_dense_maxcut(2000, 0.01, 7)", 2000, 4096, 1000,
              "G-set-style gen_dense_maxcut(2000,0.01,7), 4096 reads/GPU, t_f=1000"),
    # the sparse path where it is the routed one (large, low-degree instance: ELL kernel)
    "moebius131072": ("moebius_ladder(131072)", 131072, 1024, 200,
                      "Moebius ladder n=131072 (sparse ELL path), 1024 reads/GPU, t_f=200"),
    # the G-set toroidal class at scale (degree 4: ELL kernel with 4 slots)
    "torus": ("toroidal_grid(362, 362, 1)", 131044, 1024, 200,
              "toroidal grid 362x362 (n=131044, +-1 couplers, sparse ELL path), 1024 reads/GPU, t_f=200"),
    # the G-set random class beyond the dense crossover (G55/G60 shape: n = 5000, mean degree 5,
    # max degree > 4): the CSR kernel with staged segments
    "gset5000": ("gen_dense_maxcut(5000, 5.0 / 4999, 1)", 5000, 4096, 1000,
                 "G-set-class random graph gen_dense_maxcut(5000, 0.001, 1) (mean degree 5, sparse CSR "
                 "path), 4096 reads/GPU, t_f=1000"),
    # exhaustive ground state (brute_force_ground) at the reference's limit
    "ground26": ("gen_sk(26, 1)", 26, 1, 1, "exact ground state of gen_sk(26,1) by Gray-code enumeration"),
    # config 5: J generated on device, row-sharded over the ranks (strong scaling)
    "sk65536": (None, 65536, 1024, 200,
                "synthetic SK N=65536 (on-device Philox J, seed 7), 1024 reads total, t_f=200, "
                "J row-sharded, S all-gathered each sweep"),
}


DTYPES = {
    "dense": "f16 operand / f16 hi+lo state (~22-bit) / f32 accumulate",
    "dense_hilo": "f16 hi+lo operands (HILO field, ~22-bit) / f16 hi+lo state / f32 accumulate",
    "small_hilo": "f16 hi+lo operands (HILO field, ~22-bit) / f32 state / f32 accumulate",
    "small": "f16 operand / f32 state / f32 accumulate",
    "sparse": "f32 state / f32 accumulate",
}


def metric_name(workload):
    return ("spin-updates/s (N*reads*steps/s) on K2000" if workload == "k2000"
            else f"spin-updates/s (N*reads*steps/s) on {workload}")


def build_problem(nb, name):
    expr = WORKLOADS[name][0]
    return eval("nb." + expr, {"nb": nb})


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
            # nvidia-smi needs ~0.1 s for its first row; wait for it so that a
            # timed region shorter than the sampling period still gets sampled
            t_end = time.time() + 3.0
            while not self.rows and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.proc.wait()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k] == "Active"})
        pw = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w_median": statistics.median(pw) if pw else None, "samples": len(self.rows)}


def load_peaks():
    try:
        with open(os.path.join(REPO, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


def load_traffic(workload, reads_override=None):
    """ncu DRAM bytes of one launch of the workload's default shape
    (profiles/ncu_summary.json); null when --reads changes the shape."""
    if reads_override is not None:
        return None
    path = os.path.join(REPO, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return d.get(workload, {}).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        if os.environ.get("NMFA_BENCH_SHARED_GPU") == "1":
            # functional check of the N > 1 code path on a one-GPU box: every rank
            # on cuda:0, host-side gloo collectives (no kernel waits on another
            # rank); timings from such a run are not bench numbers
            local = 0
            torch.cuda.set_device(0)
            dist.init_process_group("gloo")
        else:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    return world, rank, local


def reference_package():
    """The UNMODIFIED reference package installed into baseline/_ref (pip
    --target), or None when it is absent."""
    ref = os.path.join(REPO, "baseline", "_ref")
    if not os.path.isfile(os.path.join(ref, "nmfa", "solver.py")):
        return None
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nmfa_ref_numba_cache")
    if ref not in sys.path:
        sys.path.insert(0, ref)
    try:
        import nmfa
    except Exception:  # pragma: no cover - broken install: fall back to the port
        return None
    return nmfa


def cpu_reference(workload, sample_runs=None, threads=None):
    """Time the reference's own per-run loop on a bounded sample (host cores).

    Preferred: the installed reference itself, `nmfa.nmfa_batch(problem,
    NmfaParams(t_f, seed=0), runs, threads)` with OPENBLAS_NUM_THREADS=1
    (solver.py:262-280; kind "reference").  Fallback when baseline/_ref is
    missing: the oracle's jitted restatement of the same loop (kind "port",
    bit-exact with the reference's seeded energies, tests/test_oracle.py)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    import numpy as np

    import paper_1806_08422_b200.instances as inst  # input construction only

    _, n, _, t_f, _ = WORKLOADS[workload]
    p = build_problem(inst, workload)
    threads = threads or os.cpu_count() or 1
    if sample_runs is None:
        sample_runs = {"k2000": 2 * threads, "g2000": 8 * threads, "gset5000": 8 * threads,
                       "moebius131072": threads, "torus": threads}.get(workload, 64 * threads)
    nmfa = reference_package()
    if nmfa is not None:
        cpl = np.column_stack([p.edges_i, p.edges_j, p.edge_weights])
        rp = nmfa.IsingProblem(p.n, cpl, h=np.asarray(p.h, dtype=np.float64))
        nmfa.nmfa_batch(rp, nmfa.NmfaParams(t_f=20, seed=10**6), threads, threads=threads)  # jit
        t0 = time.perf_counter()
        res = nmfa.nmfa_batch(rp, nmfa.NmfaParams(t_f=t_f, seed=0), sample_runs, threads=threads)
        wall = time.perf_counter() - t0
        best = min(r.final_energy for r in res)
        kind, what = "reference", (f"the reference's nmfa.nmfa_batch (baseline/_ref, backend "
                                   f"{nmfa.kernels.BACKEND}, OPENBLAS_NUM_THREADS=1)")
    else:
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import nmfa_oracle as O
        op = O.problem_from_edges(p.n, p.edges_i, p.edges_j, p.edge_weights, p.h)
        O.batch(op, 10**6, threads, t_f=20, threads=threads)  # warm BLAS / thread pool
        t0 = time.perf_counter()
        _, e = O.batch(op, 0, sample_runs, t_f=t_f, threads=threads)
        wall = time.perf_counter() - t0
        best = float(e.min())
        kind, what = "port", "oracle per-run float64 loop (dgemv/CSR, numpy Philox noise)"
    return {"value": n * sample_runs * t_f / wall, "unit": "spin-updates/s", "cores": threads,
            "kind": kind,
            "sample": f"{sample_runs} runs x t_f={t_f} of the {workload} instance, {what}, "
                      f"{threads} threads, {wall:.1f} s wall, best E={best:.0f}",
            "wall_s": wall}


def measure_tts_sk100(nb, dev, skip_cpu=False):
    """TTS99 on the 100-spin SK instance (the metric's second half).

    GPU: batches of 37,888 reads (2 per SM-resident CTA of 128) through the
    plan API, tau = batch time (CUDA events, mean of 3) / reads, p = P(E <= -730), -730 being the best of 10,000 reference
    runs (tests/golden/stats.npz).  CPU: tau of the jitted reference port on
    the host cores; p from the reference's own 10,000-run statistics.
    """
    import math

    import numpy as np
    import torch

    e_ref = -730.0
    p = nb.gen_sk(100, 0)
    R = 37888
    params = nb.NmfaParams(t_f=1000, seed=777)
    # the batch through the plan API (device buffers allocated once, as a sampling
    # service would hold them): anneal + exact energies of all R reads per batch
    plan = nb.Plan(p, R, params.schedule.temperatures(params.t_f), params.alpha, params.sigma,
                   device=dev.index)
    cfg = torch.empty((R, p.n), dtype=torch.int8, device=dev)
    en = torch.empty(R, dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    plan.run(12345, 0, config=cfg, energy=en, stream=stream)       # warm
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    reps = 3
    with ClockSampler(dev.index) as clk:  # the state the K2000 steps left the GPU in is recorded
        ev[0].record(stream)
        for k in range(reps):
            plan.run(params.seed + k * R, 0, config=cfg, energy=en, stream=stream)
        ev[1].record(stream)
        torch.cuda.synchronize(dev)
    wall = ev[0].elapsed_time(ev[1]) * 1e-3 / reps
    e = en.cpu().numpy()
    k = int(np.count_nonzero(e <= e_ref + 1e-9))
    pg = k / R
    tau = wall / R
    out = {"instance": "gen_sk(100,0), t_f=1000, E_ref=-730 (best of 65,536 reference runs)",
           "gpu": {"reads": R, "p": pg, "tau_s": tau,
                   "tts99_s": tau * math.log(0.01) / math.log(1 - pg) if 0 < pg < 0.99 else None,
                   "clocks": clk.summary()}}
    try:
        golden = np.load(REF_STATS)
        pref = float(np.mean(golden["sk100_E"] <= e_ref + 1e-9))
        out["reference_p"] = pref
        out["reference_reads"] = int(golden["sk100_E"].size)
    except OSError:
        pref = None
    if not skip_cpu and pref:
        threads = os.cpu_count() or 1
        runs = 32 * threads
        nmfa = reference_package()
        if nmfa is not None:     # the installed reference itself
            rp = nmfa.gen_sk(100, 0)
            nmfa.nmfa_batch(rp, nmfa.NmfaParams(t_f=50, seed=0), threads, threads=threads)
            t0 = time.perf_counter()
            nmfa.nmfa_batch(rp, nmfa.NmfaParams(t_f=1000, seed=0), runs, threads=threads)
            kind = "reference"
        else:
            sys.path.insert(0, os.path.join(REPO, "oracle"))
            import nmfa_oracle as O
            op = O.problem_from_edges(100, p.edges_i, p.edges_j, p.edge_weights)
            O.batch(op, 0, threads, t_f=50, threads=threads)
            t0 = time.perf_counter()
            O.batch(op, 0, runs, t_f=1000, threads=threads)
            kind = "port"
        tau_c = (time.perf_counter() - t0) / runs
        out["cpu_reference"] = {"runs": runs, "threads": threads, "tau_s": tau_c, "p": pref,
                                "kind": kind,
                                "tts99_s": tau_c * math.log(0.01) / math.log(1 - pref)}
    return out


REF_STATS = os.path.join(REPO, "tests", "golden", "stats_large.npz")


def binomial(k, n):
    """k successes of n with the 95% Wilson score interval."""
    import math
    z = 1.96
    ph = k / n
    den = 1.0 + z * z / n
    c = (ph + z * z / (2 * n)) / den
    half = z * math.sqrt(ph * (1 - ph) / n + z * z / (4 * n * n)) / den
    return {"k": int(k), "n": int(n), "p": ph, "ci95": [c - half, c + half]}


def compare_p(k_gpu, n_gpu, k_ref, n_ref):
    """North-star statistics criterion: the GPU's success probability inside the
    reference's 95% binomial (Wilson) interval; the pooled two-proportion z is
    reported beside it."""
    import math
    ref, gpu = binomial(k_ref, n_ref), binomial(k_gpu, n_gpu)
    pool = (k_gpu + k_ref) / (n_gpu + n_ref)
    se = math.sqrt(max(pool * (1 - pool), 1e-300) * (1 / n_gpu + 1 / n_ref))
    return {"reference": ref, "gpu": gpu,
            "gpu_p_in_reference_ci": ref["ci95"][0] <= gpu["p"] <= ref["ci95"][1],
            "z": (gpu["p"] - ref["p"]) / se}


def measure_statistics(nb, dev, workload, last_energies):
    """Success probabilities against the reference's own large samples
    (tests/golden/stats_large.npz, make_golden_stats.py: the reference's streams
    and arithmetic, identical to nmfa_batch on every shared seed).

    SK100 / Moebius-100: p(E <= ground) with the reference's best energy.
    G2000 / K2000: p(E <= E*), E* = the 10th-percentile energy of the first
    4096 reference reads, the reference's p scored on the
    reads after those (tests/test_gpu_statistics.py explains why).  K2000 uses
    the timed steps' own last energies."""
    import numpy as np

    try:
        ref = np.load(REF_STATS)
    except OSError:
        return None
    out = {}
    cases = [("sk100", "gen_sk(100, 0)", 65536, None), ("moebius100", "moebius_ladder(100)", 32768, None),
             ("g2000", "gen_dense_maxcut(2000, 0.01, 7)", 16384, 0.1)]
    def reference_success(e_ref, q):
        if q is None:
            return float(e_ref.min()), e_ref
        thr = float(np.quantile(e_ref[:4096], q, method="lower"))
        return thr, (e_ref[4096:] if e_ref.size > 4096 else e_ref)

    # Moebius-100 also on the CSR/ELL gather path BASELINE config 2 names (the router
    # sends n <= 256 to the on-chip small kernel, which is faster)
    cases.append(("moebius100", "moebius_ladder(100)", 32768, None, "sparse"))
    for name, expr, reads, q, *force in cases:
        thr, e_ref = reference_success(ref[name + "_E"].astype(np.float64), q)
        p = eval("nb." + expr, {"nb": nb})
        if force:
            p.device_handle(dev.index).set_path(force[0])
        ev = (torch_event(), torch_event())
        nb.sample(p, nb.NmfaParams(t_f=1000, seed=0), reads, device=dev.index)   # warm the plan
        ev[0].record()
        res = nb.sample(p, nb.NmfaParams(t_f=1000, seed=0), reads, device=dev.index)
        ev[1].record()
        ev[1].synchronize()
        e = res.energies.cpu().numpy()
        wall = ev[0].elapsed_time(ev[1]) * 1e-3
        out[name + ("_" + force[0] if force else "")] = {"threshold_E": thr, "threshold": "reference minimum" if q is None else
                     "10th percentile of the first 4096 reference reads; reference p over the rest", "path": p.device_info(dev.index)["path"],
                     "spin_updates_per_s": p.n * reads * 1000 / wall, "seed": 0,
                     **compare_p(int(np.count_nonzero(e <= thr + 1e-9)), reads,
                                 int(np.count_nonzero(e_ref <= thr + 1e-9)), e_ref.size)}
    if workload == "k2000" and last_energies is not None:
        thr, e_ref = reference_success(ref["sk2000_E"].astype(np.float64), 0.1)
        e = np.asarray(last_energies)
        out["k2000"] = {"threshold_E": thr, "threshold": "10th percentile of the first 4096 reference reads; reference p over the rest",
                        "note": "energies of the last timed step",
                        **compare_p(int(np.count_nonzero(e <= thr + 1e-9)), e.size,
                                    int(np.count_nonzero(e_ref <= thr + 1e-9)), e_ref.size)}
    return out


def torch_event():
    import torch
    return torch.cuda.Event(enable_timing=True)


def run_reference(args):
    # no process group: the reference arm has no collective, rank 0 alone runs
    # it on the host cores and the other ranks exit 0 at once
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    desc = WORKLOADS[args.workload][4]
    steps = []
    cb = None
    for k in range(args.warmup + args.steps):
        r = cpu_reference(args.workload, sample_runs=args.ref_runs)
        if k >= args.warmup:
            steps.append(r)
            cb = r
    value = statistics.median(s["value"] for s in steps)
    line = {"metric": metric_name(args.workload), "value": value,
            "unit": "spin-updates/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * statistics.median(s["wall_s"] for s in steps),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (reference generator stream)", "impl": "reference",
            "config": {"workload": desc, "sample": cb["sample"]},
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")} |
            {"value": value},
            "e2e": {"value": value, "unit": "spin-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_sk65536(args):
    """Config 5: row-sharded J; a step is one anneal (t_f sweeps) of all reads."""
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1806_08422_b200 import NmfaParams
    from paper_1806_08422_b200.sharded import RowShardedSK

    world, rank, local = dist_init()
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    _, n, R, t_f, desc = WORKLOADS["sk65536"]
    R = args.reads or R
    params = NmfaParams(t_f=t_f, seed=args.seed)
    t0 = time.perf_counter()
    sk = RowShardedSK(n, 7, R, params, device=local, exchange=args.exchange)
    torch.cuda.synchronize(dev)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream(dev)
    for k in range(args.warmup):
        sk.run(params.seed + k)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    with ClockSampler(local) as clk:
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for k in range(args.steps):
            res = sk.run(params.seed + args.warmup + k)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    ms = torch.tensor([ev0.elapsed_time(ev1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    value = n * R * t_f * args.steps / (ms * 1e-3)
    launches = args.steps * (1 if world == 1 else t_f + 1) + args.steps  # sweeps + read_config
    # e2e: the same call plus D2H of configs and energies into pinned host memory
    cfg_h = torch.empty((R, n), dtype=torch.int8).pin_memory()
    en_h = torch.empty(R, dtype=torch.float64).pin_memory()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 3))
    for k in range(e2e_steps):
        res = sk.run(params.seed + k)
        cfg_h.copy_(res.configs, non_blocking=True)
        en_h.copy_(res.energies, non_blocking=True)
        torch.cuda.synchronize(dev)
    et = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_value = n * R * t_f * e2e_steps / float(et.item())
    # per-sweep roofline on this GPU's shard: 2 * N * (N/G) * R FLOP
    flop = 2.0 * n * (n // world) * R
    per_sweep_s = ms * 1e-3 / (args.steps * t_f)
    peaks, peak_src = load_peaks()
    peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
    achieved = flop / per_sweep_s / 1e12
    best = float(en_h.min())
    if rank == 0:
        print(json.dumps({
            "metric": "spin-updates/s (N*reads*steps/s) on synthetic SK N=65536", "value": value,
            "unit": "spin-updates/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": DTYPES["dense"],
            "data": "synthetic (on-device Philox SK couplings)",
            "config": {"workload": desc, "reads_total": R, "n": n, "t_f": t_f,
                       "parallelism": f"J row-sharded x{world}", "setup_s": setup_s,
                       "exchange": (f"{sk.exchange}: " + ("epilogue peer stores into symmetric "
                                    "memory + device barrier per sweep" if sk.exchange == "p2p"
                                    else "NCCL all_gather_into_tensor per sweep")),
                       "l2": "J shard (8.6/G GB) exceeds L2; no flush needed",
                       "best_energy": best, "best_energy_per_spin": best / n},
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": peak,
                         "unit": "TFLOP/s", "frac": achieved / peak, "traffic": None,
                         "kernel": "dense NMFA sweep on the J row shard (tcgen05)",
                         "algorithmic_per_launch": f"2*N*(N/G)*R = {flop:.4g} FLOP per sweep",
                         "avg_sweep_us": per_sweep_s * 1e6,
                         "peak_source": f"{peak_src} bf16 sustained"},
            "cpu_baseline": None,
            "e2e": {"value": e2e_value, "unit": "spin-updates/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": int(R * n + R * 8),
                    "api": "RowShardedSK.run + D2H of configs/energies"},
            "gpu_launches": launches, "clocks": clk.summary()}), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def run_ground(args, impl):
    """brute_force_ground on gen_sk(26, 1): one step = one full enumeration of
    2^26 configurations; metric configurations/s.  The reference arm times the
    oracle's numba restatement of the reference's sequential Gray walk
    (_kernels_numba.py:83-114) on one host core (the reference is sequential)."""
    import numpy as np

    import paper_1806_08422_b200 as nb

    world, rank, _ = dist_init()
    p = nb.gen_sk(26, 1)
    n = p.n
    desc = WORKLOADS["ground26"][4]
    if impl == "reference":
        if rank == 0:
            sys.path.insert(0, os.path.join(REPO, "oracle"))
            import nmfa_oracle as O
            op = O.problem_from_edges(n, p.edges_i, p.edges_j, p.edge_weights)
            O.gray_ground_fast(O.problem_from_edges(4, [0], [1], [1.0]))  # jit
            times = []
            for _ in range(args.warmup + args.steps):
                t0 = time.perf_counter()
                e, c = O.gray_ground_fast(op)
                times.append(time.perf_counter() - t0)
            dt = statistics.median(times[args.warmup:])
            v = 2.0 ** n / dt
            print(json.dumps({
                "metric": "configurations/s (2^n / enumeration time), exact ground state", "value": v,
                "unit": "configurations/s", "n_gpus": args.gpus, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "impl": "reference", "config": {"workload": desc, "energy": e, "degeneracy": c},
                "cpu_baseline": {"value": v, "unit": "configurations/s", "cores": 1, "kind": "port",
                                 "sample": "full 2^26 enumeration"},
                "e2e": {"value": v, "unit": "configurations/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}), flush=True)
        return
    import torch
    nb.brute_force_ground(p)  # warm-up: builds the device problem
    with ClockSampler(0) as clk:
        times = []
        for _ in range(args.warmup + args.steps):
            t0 = time.perf_counter()
            gt = nb.brute_force_ground(p)   # synchronous host API (host in, host out)
            times.append(time.perf_counter() - t0)
    dt = statistics.median(times[args.warmup:])
    value = 2.0 ** n / dt
    cpu_bl = None
    if not args.no_cpu_baseline:
        sys.path.insert(0, os.path.join(REPO, "oracle"))
        import nmfa_oracle as O
        op = O.problem_from_edges(n, p.edges_i, p.edges_j, p.edge_weights)
        O.gray_ground_fast(O.problem_from_edges(4, [0], [1], [1.0]))
        t0 = time.perf_counter()
        O.gray_ground_fast(op)
        cdt = time.perf_counter() - t0
        cpu_bl = {"value": 2.0 ** n / cdt, "unit": "configurations/s", "cores": 1, "kind": "port",
                  "sample": "full 2^26 enumeration (numba restatement of gray_ground)"}
    if rank == 0:
        print(json.dumps({
            "metric": "configurations/s (2^n / enumeration time), exact ground state", "value": value,
            "unit": "configurations/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "int64 (popcount fields)", "data": "synthetic",
            "config": {"workload": desc, "n": n, "energy": gt.energy, "degeneracy": gt.degeneracy,
                       "timing": "host wall clock around the synchronous C-ABI call"},
            "roofline": None,
            "cpu_baseline": cpu_bl,
            "e2e": {"value": value, "unit": "configurations/s", "h2d_bytes_per_step": n * n * 8 + n * 40,
                    "d2h_bytes_per_step": 24 * max(1, (1 << (n - 1 - 9)) // 256),
                    "api": "brute_force_ground -> nmfa_ground_state (C ABI, host buffers)"},
            "gpu_launches": 1, "clocks": clk.summary()}), flush=True)


def run_ours(args):
    import ctypes

    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1806_08422_b200 as nb
    from paper_1806_08422_b200 import _native

    world, rank, local = dist_init()
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    _, n, R, t_f, desc = WORKLOADS[args.workload]
    if args.reads:
        R = args.reads
    p = build_problem(nb, args.workload)
    if args.field != "fp16":
        p.device_handle(local).set_field_precision(args.field)
    params = nb.NmfaParams(t_f=t_f, seed=args.seed)
    temps = params.schedule.temperatures(t_f)
    plan = nb.Plan(p, R, temps, params.alpha, params.sigma, device=local)
    r0 = rank * R                       # global replica offset: sharding-invariant noise keys
    cfg = torch.empty((R, n), dtype=torch.int8, device=dev)
    en = torch.empty(R, dtype=torch.float64, device=dev)
    best_e = torch.empty(1, dtype=torch.float64, device=dev)
    best_i = torch.empty(1, dtype=torch.int64, device=dev)
    lib = _native.load()
    stream = torch.cuda.current_stream(dev)

    def step(k, mid=None):
        launches = plan.run(params.seed + 1000003 * k, r0, config=cfg, energy=en, stream=stream)
        if mid is not None:
            mid.record(stream)
        _native.check(lib.nmfa_best_of(_native.ptr(en), R, _native.ptr(best_e), _native.ptr(best_i),
                                       ctypes.c_void_p(stream.cuda_stream)))
        return launches + 1

    for k in range(args.warmup):
        step(k)
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    launches = 0
    # L2 is flushed between timed steps (a 256 MB write, outside the per-step
    # CUDA-event brackets), so no step starts with the previous step's J/state hot
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    # three events per step on the launching stream: start, after the anneal
    # launch (the dominant kernel: all t_f sweeps + energies), after best-of
    evs = [tuple(torch.cuda.Event(enable_timing=True) for _ in range(3)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize(dev)
        for k in range(args.steps):
            flush.fill_(k & 0xFF)
            evs[k][0].record(stream)
            launches += step(args.warmup + k, mid=evs[k][1])
            evs[k][2].record(stream)
        torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    ms = sum(e0.elapsed_time(e2) for e0, _, e2 in evs)
    anneal_ms = sum(e0.elapsed_time(e1) for e0, e1, _ in evs) / args.steps
    last_energies = en.double().cpu().numpy()
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    # global best-of-reads across ranks (the only collective: one small all-gather)
    pair = torch.stack([best_e[0], (best_i[0] + r0).double()])
    if world > 1:
        allp = [torch.empty_like(pair) for _ in range(world)]
        dist.all_gather(allp, pair)
        allp = torch.stack(allp).cpu().numpy()
    else:
        allp = pair[None].cpu().numpy()
    gbest = allp[np.lexsort((allp[:, 1], allp[:, 0]))[0]]
    value = world * n * R * t_f * args.steps / (ms_max * 1e-3)

    # ---- roofline of the dominant kernel, from the timed steps themselves: the
    # anneal launch's CUDA-event time (same L2-flushed steps as `value`)
    info = p.device_info(local)
    per_launch_s = anneal_ms * 1e-3 / t_f
    peaks, peak_src = load_peaks()
    sm_mhz = clk.summary().get("sm_mhz")
    if info["path"] in ("dense", "small"):
        npad = (n + 15) // 16 * 16
        flop = 2.0 * n * n * R
        achieved = flop / per_launch_s / 1e12
        peak = peaks.get("bf16_tflops_sustained", peaks.get("bf16_tflops"))
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved / peak, "traffic": load_traffic(args.workload, args.reads),
                "kernel": f"{info['path']} NMFA anneal (tcgen05, fused epilogue; one launch = t_f sweeps "
                          "+ exact energies)",
                "algorithmic_per_launch": f"2*N^2*R*t_f = {flop * t_f:.4g} FLOP (N={n}, R={R}, "
                                          f"t_f={t_f}; padded N={npad}; energy pass not counted)",
                "avg_launch_us": anneal_ms * 1e3, "avg_sweep_us": per_launch_s * 1e6,
                "timing": "CUDA events around the anneal launch inside the timed, L2-flushed steps",
                "peak_source": f"{peak_src} bf16 sustained (fp16 runs at the bf16 rate)",
                "frac_of_burst": achieved / peaks.get("bf16_tflops", peak)}
        if sm_mhz:
            # tensor duty per clock: FLOP/clk/SM over the 8192 dense f16 FLOP/clk/SM
            roof["per_clock_duty"] = achieved * 1e12 / (148 * sm_mhz * 1e6) / 8192
            roof["per_clock_sm_mhz"] = sm_mhz
        if args.field == "hilo":
            roof["note_hilo"] = ("HILO field: the kernel issues two MMAs per k-slice (hi and lo), so the "
                                 "tensor work executed is 2x the algorithmic FLOP counted here "
                                 f"(executed-FLOP fraction {2 * achieved / peak:.3f})")
        if info["path"] == "small":
            roof["note"] = ("n <= 256 runs on chip for all t_f steps; the binding resource is the fused "
                            "update's instruction issue (ncu: 28 instructions per spin-update, IPC 2.1 "
                            "of 4), not the tensor pipe (profiles/r01/ncu_full_summary.json)")
    else:
        nnz = 2 * p.num_edges
        byts = R * n * 8 + nnz * 8 + (n + 1) * 4
        achieved = byts / per_launch_s / 1e9
        peak = peaks.get("hbm_gbs")
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": load_traffic(args.workload, args.reads),
                "timing": "CUDA events around the anneal launches inside the timed, L2-flushed steps",
                "kernel": ("sparse NMFA step (ELL gather, %d slots per row, fused epilogue)" % info["ell_slots"]
                           if info.get("ell_slots") else "sparse NMFA step (CSR gather, fused epilogue)"),
                "algorithmic_per_launch": f"R*N*8 + nnz*8 + (N+1)*4 = {byts:.4g} B",
                "avg_launch_us": per_launch_s * 1e6, "peak_source": f"{peak_src} HBM copy"}

    # SURVEY 8(d) defines the sparse-class configs (C2 Moebius-100, C4 G2000: the
    # reference's is_dense = False) by the HBM roofline of a gather step.  When the
    # router sends them to the on-chip small kernel or the tensor-core kernel, the
    # roofline above is that kernel's; this is the 8(d) figure for the same launches.
    roof_8d = None
    if not info["is_dense"] and info["path"] != "sparse":
        nnz = 2 * p.num_edges
        byts = R * n * 8 + nnz * 8 + (n + 1) * 4
        ach = byts / per_launch_s / 1e9
        roof_8d = {"bound": "hbm", "achieved": ach, "peak": peaks.get("hbm_gbs"), "unit": "GB/s",
                   "frac": ach / peaks.get("hbm_gbs"),
                   "algorithmic_per_launch": f"R*N*8 + nnz*8 + (N+1)*4 = {byts:.4g} B",
                   "note": f"SURVEY 8(d) sparse-step definition; the instance runs on the {info['path']} "
                           "kernel, which keeps the state on chip (small) or streams J through the "
                           "tensor cores (dense) instead of gathering from HBM"}

    # ---- end to end through the C ABI with HOST buffers (nmfa_anneal_host)
    cfg_h = torch.empty((R, n), dtype=torch.int8).pin_memory()
    en_h = torch.empty(R, dtype=torch.float64).pin_memory()
    temps_h = torch.from_numpy(np.ascontiguousarray(temps)).pin_memory()
    handle = p.device_handle(local).handle
    e2e_steps = max(1, min(args.steps, 5))
    _native.check(lib.nmfa_anneal_host(handle, R, t_f, _native.ptr(temps_h), params.alpha,
                                       params.sigma, params.seed, r0, _native.ptr(cfg_h),
                                       _native.ptr(en_h)))  # warm-up: builds the cached plan
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(e2e_steps):
        _native.check(lib.nmfa_anneal_host(handle, R, t_f, _native.ptr(temps_h), params.alpha,
                                           params.sigma, params.seed + k, r0, _native.ptr(cfg_h),
                                           _native.ptr(en_h)))
    e2e_wall = time.perf_counter() - t0
    et = torch.tensor([e2e_wall], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(et, op=dist.ReduceOp.MAX)
    e2e_value = world * n * R * t_f * e2e_steps / float(et.item())

    # ---- the reference-compatible Python entry itself: nb.nmfa_batch returns the
    # reference's list[RunResult] (float64 +-1 configs, one dataclass per run)
    e2e_py = None
    if rank == 0 and world == 1:
        nb.nmfa_batch(p, params, R, device=local)          # warm
        t0 = time.perf_counter()
        runs = nb.nmfa_batch(p, params, R, device=local)
        py_wall = time.perf_counter() - t0
        e2e_py = {"value": n * R * t_f / py_wall, "unit": "spin-updates/s",
                  "wall_s": py_wall, "runs": len(runs),
                  "api": "nb.nmfa_batch(problem, params, n_runs) -> list[RunResult] (the reference's "
                         "return type: float64 configs, one dataclass per run; solver.py:262-280)"}
        del runs

    # the dense path's fidelity mode on the same workload (side measurement, K2000 line
    # only): HILO field, 3 anneals, CUDA events; the algorithmic FLOP as in `roofline`
    hilo_side = None
    if (rank == 0 and args.workload == "k2000" and args.field == "fp16" and not args.no_stats
            and p.device_info(local)["path"] == "dense"):
        q = build_problem(nb, args.workload)
        q.device_handle(local).set_field_precision("hilo")
        hplan = nb.Plan(q, R, temps, params.alpha, params.sigma, device=local)
        hplan.run(1, r0, config=cfg, energy=en, stream=stream)
        hev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        hev[0].record(stream)
        for k in range(3):
            hplan.run(2 + k, r0, config=cfg, energy=en, stream=stream)
        hev[1].record(stream)
        torch.cuda.synchronize(dev)
        hs = hev[0].elapsed_time(hev[1]) * 1e-3 / 3
        hilo_side = {"value": n * R * t_f / hs, "unit": "spin-updates/s",
                     "frac_of_sustained_algorithmic": 2.0 * n * n * R * t_f / hs / 1e12 / peak
                     if info["path"] == "dense" else None,
                     "note": "HILO field (hi + lo state through the GEMM, NMFA_FIELD_HILO): the "
                             "fidelity mode; two MMAs per k-slice, so the executed tensor work is 2x "
                             "the algorithmic FLOP"}
        del hplan

    tts = None
    if rank == 0 and not args.no_tts:
        tts = measure_tts_sk100(nb, dev, args.no_cpu_baseline)
    stats = None
    if rank == 0 and not args.no_stats:
        stats = measure_statistics(nb, dev, args.workload, last_energies)

    cpu_bl = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = cpu_reference(args.workload, sample_runs=args.ref_runs)
        cpu_bl = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}

    if rank == 0:
        line = {
            "metric": metric_name(args.workload), "value": value,
            "unit": "spin-updates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": DTYPES[info["path"] + "_hilo"] if info.get("field") == "hilo" and
            info["path"] + "_hilo" in DTYPES else DTYPES[info["path"]],
            "data": f"synthetic (reference generator stream, {WORKLOADS[args.workload][0]})",
            "config": {"workload": desc, "reads_per_gpu": R, "reads_total": R * world,
                       "n": n, "t_f": t_f, "path": info["path"],
                       **({"field": "hilo (2 MMAs per k-slice; roofline counts the algorithmic "
                                    "2 N^2 R FLOP per sweep)"} if args.field == "hilo" else {}),
                       "parallelism": f"replica-sharded x{world}",
                       "l2": "flushed between timed steps (256 MB write outside the per-step "
                             "event brackets); value = steps x work / sum of step times",
                       "best_energy": float(gbest[0]), "best_replica": int(gbest[1])},
            "roofline": roof,
            **({"roofline_8d_hbm": roof_8d} if roof_8d else {}),
            "cpu_baseline": cpu_bl,
            "e2e": {"value": e2e_value, "unit": "spin-updates/s",
                    "h2d_bytes_per_step": int(temps.nbytes),
                    "d2h_bytes_per_step": int(R * n + R * 8),
                    "api": "nmfa_anneal_host (C ABI, host buffers)"},
            **({"e2e_python_api": e2e_py} if e2e_py else {}),
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "tts99_sk100": tts,
            "statistics": stats,
            **({"hilo_field": hilo_side} if hilo_side else {}),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="k2000")
    ap.add_argument("--reads", type=int, default=None, help="reads per GPU override")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--ref-runs", type=int, default=None)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-tts", action="store_true", help="skip the SK100 TTS99 side measurement")
    ap.add_argument("--no-stats", action="store_true",
                    help="skip the success-probability side measurements (SK100, Moebius-100, G2000)")
    ap.add_argument("--field", choices=["fp16", "hilo"], default="fp16",
                    help="dense path GEMM operand: fp16 hi (default, the throughput mode) or the "
                         "HILO fidelity mode (hi + lo; NMFA_FIELD_HILO)")
    ap.add_argument("--exchange", choices=["p2p", "nccl"], default="nccl",
                    help="sk65536: NCCL all-gather per sweep (default) or the fused peer-store "
                         "exchange (p2p; falls back to NCCL when symmetric memory is unavailable)")
    args = ap.parse_args()
    if args.impl != "reference":
        # the CUDA library ships prebuilt with the snapshot; build it if it is
        # missing or stale (no-op otherwise)
        from paper_1806_08422_b200 import build as _nbuild
        _nbuild.build()
    if args.workload == "ground26":
        run_ground(args, args.impl)
        return
    if args.workload == "sk65536":
        if args.impl == "reference":
            if int(os.environ.get("RANK", "0")) == 0:
                print(json.dumps({"impl": "reference", "unavailable":
                                  "the reference builds J as a dense n x n float64 host matrix "
                                  "(problem.py:100-104): 34 GB at N=65536"}), flush=True)
            return
        run_sk65536(args)
    elif args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
