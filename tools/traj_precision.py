"""How far do injected-noise trajectories drift from float64 under a given
GEMM-operand precision?  (CPU emulation, SURVEY 8(c) / Appendix A method.)

Replica r gets the reference's own noise stream noise_stream(r) (solver.py:
236-241); every variant steps the same noise:

  f64        the reference arithmetic (batched; == run_with_noise)
  f16op      state kept to ~22 bits (f32 here), GEMM operand fp16(s), fp32 sums
             -- the dense kernel's arithmetic up to MUFU tanh / sum order
  bf16op     same with a bf16 operand (the north star's stated format)
  f32op      fp32 operand (an upper bound on what a 3-pass split could give)

and reports, against f64, the mean over replicas of the final-sign mismatch
fraction, its max replica, and mean |dS|.

    python tools/traj_precision.py --inst k2000 --reads 64 --t_f 1000
"""

import argparse
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))

import numpy as np  # noqa: E402

import nmfa_oracle as O  # noqa: E402


def bf16(x):
    u = np.asarray(x, dtype=np.float32).view(np.uint32)
    r = ((u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000))
    return r.view(np.float32)


def instance(name):
    if name == "k2000":
        return O.problem_from_edges(2000, *O.gen_sk_edges(2000, 7))
    if name == "sk520":
        return O.problem_from_edges(520, *O.gen_sk_edges(520, 5))
    raise ValueError(name)


def run(p, noise, temps, variant, alpha=0.15):
    R = noise.shape[0]
    if variant == "f64":
        return O.batched_anneal(p, None, temps=temps, noise=noise)
    J = p.dense.astype(np.float32)
    invn = (1.0 / p.normalizers_safe).astype(np.float32)[:, None]
    S = np.zeros((p.n, R), dtype=np.float32)
    q = {"f16op": lambda s: s.astype(np.float16).astype(np.float32), "bf16op": bf16,
         "f32op": lambda s: s, "f16op_lo8": lambda s: s.astype(np.float16).astype(np.float32),
         "f16op_lo16": lambda s: s.astype(np.float16).astype(np.float32),
         "f16op_sr16": lambda s: s.astype(np.float16).astype(np.float32),
         "f16op_fx8": lambda s: s.astype(np.float16).astype(np.float32)}[variant]
    rng = np.random.default_rng(12345)

    def store(S):  # the state as the dense kernel stores it between sweeps
        if variant == "f16op_lo16":   # hi = fp16(s), lo = fp16(s - hi)  (today's kernel)
            hi = S.astype(np.float16).astype(np.float32)
            return hi + (S - hi).astype(np.float16).astype(np.float32)
        if variant == "f16op_fx8":    # hi = fp16(s), lo = int8 fixed point, scale 2^-19
            hi = S.astype(np.float16).astype(np.float32)
            qv = np.clip(np.rint((S - hi) * np.float32(2.0 ** 19)), -127, 127)
            return (hi + qv.astype(np.float32) * np.float32(2.0 ** -19)).astype(np.float32)
        if variant == "f16op_sr16":   # fp16 state, stochastic rounding (no residual)
            lo = S.astype(np.float16)
            lo32 = lo.astype(np.float32)
            nxt = np.where(S >= lo32, np.nextafter(lo, np.float16(np.inf)),
                           np.nextafter(lo, np.float16(-np.inf))).astype(np.float32)
            gap = np.abs(nxt - lo32)
            frac = np.where(gap > 0, np.abs(S - lo32) / np.where(gap > 0, gap, 1), 0)
            up = rng.random(S.shape) < frac
            return np.where(up, nxt, lo32).astype(np.float32)
        if variant == "f16op_lo8":    # hi = fp16(s), lo = int8 in units of ulp(hi)/254
            hi = S.astype(np.float16)
            ulp = np.spacing(np.abs(hi)).astype(np.float32)
            ulp = np.where(ulp == 0, np.float32(2.0 ** -24), ulp)
            qv = np.clip(np.rint((S - hi.astype(np.float32)) / ulp * 254.0), -127, 127)
            return (hi.astype(np.float32) + qv.astype(np.float32) * ulp / 254.0).astype(np.float32)
        return S
    for t in range(len(temps)):
        phi = (J @ q(S)) * invn + noise[:, t, :].T.astype(np.float32)
        sh = -np.tanh(phi * np.float32(1.0 / temps[t]))
        S = store((np.float32(alpha) * sh + np.float32(1.0 - alpha) * S).astype(np.float32))
    return S.T.astype(np.float64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--inst", default="k2000")
    ap.add_argument("--reads", type=int, default=64)
    ap.add_argument("--t_f", type=int, default=1000)
    ap.add_argument("--variants", default="f16op,bf16op,f32op")
    a = ap.parse_args()
    p = instance(a.inst)
    temps = O.temperatures(a.t_f)
    noise = np.stack([O.run_noise(r, a.t_f, p.n, 0.15) for r in range(a.reads)])
    t0 = time.time()
    ref = run(p, noise, temps, "f64")
    print(f"{a.inst}: f64 reference in {time.time() - t0:.0f} s", flush=True)
    for v in a.variants.split(","):
        t0 = time.time()
        S = run(p, noise, temps, v)
        fl = np.mean(np.sign(S) != np.sign(ref), axis=1)
        print(f"{a.inst} {v:7s}: mean sign flips {fl.mean():.2e}  max replica {fl.max():.2e}  "
              f"replicas with any flip {np.mean(fl > 0):.2f}  mean|dS| {np.abs(S - ref).mean():.2e}  "
              f"({time.time() - t0:.0f} s)", flush=True)


if __name__ == "__main__":
    main()
