"""Size sweeps over many small instances (the reference's `nmfa bench`,
cli.py:280-347; Fig. 4 of arXiv 1806.08422), batched on the GPU.

The reference loops instance by instance: generate, exact ground truth
(brute_force_ground for n <= 26, else a supplied best-known energy), then one
nmfa_batch of n_runs reads seeded seed + instance_counter * n_runs.  Here all
instances of one size are annealed in one nmfa_anneal_many call (one launch
for n <= 256) with exactly those seeds, and the ground truths come from the
GPU enumerator.  Rows and CSV text match cmd_bench's columns.
"""

from __future__ import annotations

import csv
import io

from .instances import gen_cubic_maxcut, gen_dense_maxcut, gen_sk, moebius_ladder
from .metrics import MAX_EXACT_N, GroundTruth, aggregate, brute_force_ground, instance_stats
from .solver import MASK64, NmfaParams, sample_many

BENCH_COLUMNS = ["class", "n", "instances", "runs", "p_success_q1", "p_success_median",
                 "p_success_q3", "tts_q1", "tts_median", "tts_q3"]


_CLASSES = {
    "sk": lambda n, p, seed: gen_sk(n, seed),
    "dense": gen_dense_maxcut,
    "cubic": lambda n, p, seed: gen_cubic_maxcut(n, seed),
    "moebius": lambda n, p, seed: moebius_ladder(n),
}


def make_instance(cls, n, p, seed):
    """One generated instance of a benchmark class (the classes of cli.py:172-184)."""
    build = _CLASSES.get(cls)
    if build is None:
        raise ValueError(f"unknown instance class {cls!r}")
    return build(n, p, seed)


def bench(cls, sizes, instances, n_runs, params=None, p=0.5, reference_energies=None,
          timings=True, device=0):
    """Per-size median/IQR of success probability and TTS99 over `instances`
    random instances (cli.py:280-347).  Returns (rows, csv_text, per_size_stats).

    tau (the time per run in TTS) is the wall time of the whole batched call
    divided by instances x n_runs when `timings`, else 1.0 as in the reference.
    """
    params = NmfaParams() if params is None else params
    if n_runs < 1 or instances < 1:
        raise ValueError("--runs and --instances must be at least 1")
    sizes = [int(s) for s in sizes]
    if not sizes:
        raise ValueError("--sizes must list at least one size")
    needs_ref = [n for n in sizes if n > MAX_EXACT_N]
    if needs_ref and reference_energies is None:
        raise ValueError(f"sizes {needs_ref} exceed the enumeration bound {MAX_EXACT_N}; "
                         "supply --reference-energy")
    rows, per_size = [], {}
    counter = 0
    for n in sizes:
        probs, grounds, seeds = [], [], []
        for g in range(instances):
            prob = make_instance(cls, n, p, params.seed + counter)
            if n <= MAX_EXACT_N:
                grounds.append(brute_force_ground(prob, device=device))
            else:
                try:
                    grounds.append(GroundTruth(reference_energies[(n, g)], 0, "BEST_KNOWN"))
                except KeyError:
                    raise ValueError(f"no reference energy for size {n} instance {g}") from None
            seeds.append((params.seed + counter * n_runs) & MASK64)
            probs.append(prob)
            counter += 1
        _, energies, wall = sample_many(probs, params, n_runs, seeds=seeds, device=device)
        tau = wall / (instances * n_runs) if timings else 1.0
        e = energies.cpu().numpy()
        stats = [instance_stats(e[k], grounds[k], tau) for k in range(instances)]
        agg = aggregate(stats)
        per_size[n] = stats
        rows.append([cls, n, instances, n_runs,
                     repr(agg.p_success_q1), repr(agg.p_success_median), repr(agg.p_success_q3),
                     repr(agg.tts_q1), repr(agg.tts_median), repr(agg.tts_q3)])
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(BENCH_COLUMNS)
    w.writerows(rows)
    return rows, buf.getvalue(), per_size
