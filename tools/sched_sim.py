"""Discrete-event model of the persistent dense kernel's cross-sweep schedule.

Per pair: a TMA producer (3 stages, latency L per k-slice load, waits for the
slice to be published), an MMA stream (cost per k-slice proportional to the
tile width), two TMEM accumulators, and an epilogue of duration E per tile that
publishes the tile's spins when it ends.  Reports the steady-state sweep
period for a tile order and a K order.  No L2 effects are modelled.
"""
import sys
import numpy as np


def tiles_for(n=2000, R=8192, pairs=74, w=None):
    upm, mb = (n + 15) // 16, (R + 255) // 256
    if w is None:
        best = None
        for ww in range(1, 17):
            tpm = -(-upm // ww); T = tpm * mb; pu = min(pairs, T)
            cost = -(-T // pu) * max(64 * ww, 563 + 22.6 * ww)
            if best is None or cost < best[0] - 1e-9: best = (cost, ww)
        w = best[1]
    tpm = -(-upm // w)
    tiles = []
    for m in range(mb):
        for k in range(tpm):
            a0, a1 = upm * k // tpm, upm * (k + 1) // tpm
            tiles.append((m, k, a0 * 16, (a1 - a0) * 16))
    return tiles, mb, tpm


def assign(tiles, pairs, mode, mb, tpm):
    T = len(tiles)
    if mode == "mmajor":
        off = [T * q // pairs for q in range(pairs + 1)]
        return [tiles[off[q]:off[q + 1]] for q in range(pairs)]
    if mode == "mmajor_sorted":
        off = [T * q // pairs for q in range(pairs + 1)]
        return [sorted(tiles[off[q]:off[q + 1]], key=lambda t: (t[1], t[0])) for q in range(pairs)]
    if mode == "spinmajor":
        s = sorted(tiles, key=lambda t: (t[1], t[0]))
        return [s[q::pairs] for q in range(pairs)]
    raise ValueError(mode)


def simulate(n=2000, R=8192, pairs=74, mode="mmajor", korder="natural", E=19000, slow=1.43,
             L=1500, stages=3, sweeps=8, w=None, pub="tile"):
    tiles, mb, tpm = tiles_for(n, R, pairs, w)
    per = assign(tiles, pairs, mode, mb, tpm)
    kb = -(-n // 128)
    # slice -> tiles of each block that cover it: readiness time = max of their publish times
    ready = {}          # (sweep, m, k) -> time (sweep -1 = initial state)
    cover = {}
    for t in tiles:
        m, a, n0, nl = t
        for k in range(n0 // 128, (n0 + nl - 1) // 128 + 1):
            cover.setdefault((m, k), []).append(t)
    pub_time = {}       # (sweep, tile) -> publish time
    # event-free approximation: iterate sweeps; within a sweep process pairs independently
    # given readiness of the previous sweep (exact because sweep t only needs sweep t-1)
    state = [dict(mma_free=0.0, acc_free=[0.0, 0.0], epi_free=0.0, stage_free=[0.0] * stages, it=0, jj=0)
             for _ in range(pairs)]
    periods = []
    first_start = []
    for sw in range(sweeps):
        def slice_ready(m, k):
            if sw == 0:
                return 0.0
            return max(pub_time[(sw - 1, t)] for t in cover[(m, k)])
        starts = []
        for q in range(pairs):
            st = state[q]
            for t in per[q]:
                m, a, n0, nl = t
                ks = list(range(kb))
                if korder == "early":
                    ks.sort(key=lambda k: slice_ready(m, k))
                cost = 64 * (nl / 16) * slow
                slot = st["jj"] & 1
                mma_t = max(st["mma_free"], st["acc_free"][slot])
                starts.append(mma_t)
                for k in ks:
                    s = st["it"] % stages
                    load_issue = max(slice_ready(m, k), st["stage_free"][s])
                    data = load_issue + L
                    mma_t = max(mma_t, data) + cost
                    st["stage_free"][s] = mma_t
                    st["it"] += 1
                st["mma_free"] = mma_t
                e0 = max(mma_t, st["epi_free"])
                st["epi_free"] = e0 + E
                st["acc_free"][slot] = e0 + E
                pub_time[(sw, t)] = e0 + E
                st["jj"] += 1
        first_start.append(min(starts))
    end = [max(pub_time[(sw, t)] for t in tiles) for sw in range(sweeps)]
    per_sweep = np.diff(end)[2:].mean()
    return per_sweep


if __name__ == "__main__":
    for E, slow, label in [(19000, 1.43, "full"), (700, 1.0, "noepi"), (13000, 1.25, "nomem")]:
        print(f"== {label}: E={E}, MMA slowdown x{slow}")
        for mode in ("mmajor", "mmajor_sorted", "spinmajor"):
            for ko in ("natural", "early"):
                p = simulate(mode=mode, korder=ko, E=E, slow=slow)
                print(f"  {mode:14s} {ko:8s} sweep {p:8.0f} cycles = {p/1965:6.1f} us @1965MHz")
        ideal = 4 * 16 * 64 * 14 * slow
        print(f"  bound 4 tiles x 16 slices x 896 x slow = {ideal:.0f}")
