"""CPU study for the next-round exact-integer contraction (DESIGN §8 item 1):
final-sign flips against the float64 oracle when the J.s operand is quantized.
Same setup as tests/test_gpu_parity.py::test_dense_large_injected_noise_matches_oracle
(gen_sk(520, 5), t_f=120, R=300, injected noise sigma=0.15). Modes:
  bf16      : s -> bf16(s)                          (the north star's "S in bf16")
  f16       : s -> fp16(s)                          (today's operand)
  f16hilo   : fp16(s) + fp16(s - fp16(s))           (hi+lo both as operands)
  fixK      : s -> round(s * 2^K) / 2^K             (fixed point, K fractional bits)
  tanh11    : exact operand, tanh rounded to ~11 bits (a tanh.approx.f32 stand-in)
The sum itself is exact float64 here (the int32 accumulation is exact too)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import nmfa_oracle as O
import paper_1806_08422_b200 as nb

p = nb.gen_sk(int(sys.argv[1]) if len(sys.argv) > 1 else 520, 5)
n = p.n
op = O.problem_from_edges(n, p.edges_i, p.edges_j, p.edge_weights)
J = np.zeros((n, n))
J[p.edges_i, p.edges_j] = p.edge_weights
J[p.edges_j, p.edges_i] = p.edge_weights
norm = np.sqrt((J * J).sum(1))
norm[norm == 0] = 1.0
t_f, R, alpha = 120, 300, 0.15
temps = O.temperatures(t_f)
rng = np.random.Generator(np.random.Philox(key=99))
noise = rng.standard_normal((R, t_f, n)) * 0.15


def tanh11(x):
    """tanh with ~2^-11 relative error (float16 rounding), a stand-in for tanh.approx.f32"""
    return np.tanh(x).astype(np.float16).astype(np.float64)


def run(q, th=np.tanh):
    S = np.zeros((R, n))
    for t in range(t_f):
        phi = (q(S) @ J) / norm + noise[:, t, :]
        S = alpha * (-th(phi / temps[t])) + (1 - alpha) * S
    return S


ref = run(lambda s: s)
def bf16(x):
    """round-to-nearest-even to bfloat16 (8-bit significand)"""
    b = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0x7FFF + ((b >> 16) & 1)) & 0xFFFF0000
    return b.astype(np.uint32).view(np.float32).astype(np.float64)


modes = {"bf16": bf16,
         "f16": lambda s: s.astype(np.float16).astype(np.float64),
         "f16hilo": lambda s: (lambda h: h + (s - h).astype(np.float16).astype(np.float64))(
             s.astype(np.float16).astype(np.float64))}
for K in (11, 13, 14, 15, 16, 20):
    modes[f"fix{K}"] = (lambda K: lambda s: np.clip(np.round(s * 2.0 ** K), -2.0 ** K, 2.0 ** K - 1) / 2.0 ** K)(K)
f16 = modes["f16"]
modes["tanh11"] = None
modes["f16+tanh11"] = None
for name, q in modes.items():
    if name == "tanh11":
        S = run(lambda s: s, tanh11)
    elif name == "f16+tanh11":
        S = run(f16, tanh11)
    else:
        S = run(q)
    err = np.abs(S - ref)
    flips = np.mean(np.sign(S) != np.sign(ref))
    print(f"n={n} {name:8s} mean|dS|={err.mean():.2e}  frac(|dS|>2e-2)={np.mean(err > 2e-2):.2e}  "
          f"sign flips={flips:.2e}", flush=True)
