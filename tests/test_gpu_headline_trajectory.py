"""Injected-noise trajectory parity at the headline configurations (SURVEY
8(c), north star correctness leg 2): K2000 stand-in gen_sk(2000, 7) and the
G-set-style gen_dense_maxcut(2000, 0.01, 7), t_f = 1000, 256 replicas.

Replica r is driven by the reference's own per-run noise stream,
`noise_stream(r).standard_normal((t_f, n)) * sigma` (solver.py:236-241),
injected through `run_with_noise` (solver.py:188-218) on the GPU and through
the float64 batched oracle (the reference's anneal loop, _kernels_numba.py:
40-80) on the host.

Stated tolerance (N = 2000, the MEAN over replicas of the fraction of spins
whose final sign differs from float64 -- a mean, because a replica that sits
on a bifurcation late in the anneal flips a correlated cluster of spins):

* sparse path (fp32 state and sums): <= 1e-4.
* dense path (fp16 GEMM operand, ~22-bit state, fp32 sums): <= 2e-3.
  SURVEY 8(c) proposed 1e-3 from an 8-replica emulation; the same emulation
  over 256 replicas (tools/traj_precision.py, profiles/r02/traj_precision.log)
  measures 9.6e-4 for an fp16 operand, 6.9e-3 for the north star's own
  "bf16 S" operand and 7.8e-6 for fp32, so 1e-3 sits ON the fp16 design's
  mean rather than above it.  2e-3 is 2x the fp16 design and 3.5x below the
  north star's bf16 format.
* the GPU tracks its design arithmetic: the dense path's flips are at most
  2x (+2e-4) those of an fp32-state / fp16-operand emulation stepped on the
  same noise here (`_f16_operand_emulation`).
* dense path with the HILO field (hi + lo state as the GEMM operand, the
  fidelity mode, include/nmfa_b200.h NMFA_FIELD_HILO): <= 2e-4, 5x inside
  SURVEY 8(c)'s own 1e-3 (measured 8.6e-5 on K2000, 3.9e-6 on G2000; the
  remaining gap to float64 is the ~22-bit state and the fp32 sums).
"""

import numpy as np
import pytest

import nmfa_oracle as O

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover - CPU container
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1806_08422_b200 as nb  # noqa: E402
from paper_1806_08422_b200 import _native  # noqa: E402

R, T_F, SIGMA, ALPHA = 256, 1000, 0.15, 0.15
MAKE = {"k2000": lambda: nb.gen_sk(2000, 7),
        "g2000": lambda: nb.gen_dense_maxcut(2000, 0.01, 7)}


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_1806_08422_b200 import build
    build.build()
    _native.load()


_CACHE = {}


def _f16_operand_emulation(op, noise, temps):
    """fp32 state, fp16-rounded GEMM operand, fp32 products: the dense
    kernel's arithmetic up to MUFU tanh and tensor-core summation order."""
    J = op.dense.astype(np.float32)
    invn = (1.0 / op.normalizers_safe).astype(np.float32)[:, None]
    S = np.zeros((op.n, noise.shape[0]), dtype=np.float32)
    for t in range(len(temps)):
        phi = (J @ S.astype(np.float16).astype(np.float32)) * invn + noise[:, t, :].T.astype(np.float32)
        S = (np.float32(ALPHA) * -np.tanh(phi * np.float32(1.0 / temps[t]))
             + np.float32(1.0 - ALPHA) * S).astype(np.float32)
    return S.T.astype(np.float64)


def reference_run(name):
    """(problem, oracle problem, noise (R, t_f, n), float64 final S (R, n))."""
    if name not in _CACHE:
        p = MAKE[name]()
        op = O.problem_from_edges(p.n, p.edges_i, p.edges_j, p.edge_weights)
        noise = np.stack([O.run_noise(r, T_F, p.n, SIGMA) for r in range(R)])
        S = O.batched_anneal(op, None, t_f=T_F, temps=O.temperatures(T_F), noise=noise)
        _CACHE[name] = (op, noise, S)
    return _CACHE[name]


def flips(S, Sref):
    return np.mean(np.sign(S) != np.sign(Sref), axis=1)


@pytest.mark.parametrize("name,path", [("k2000", "dense"), ("g2000", "dense"), ("g2000", "sparse"),
                                       ("k2000", "dense-hilo"), ("g2000", "dense-hilo")])
def test_headline_trajectory_matches_float64_reference(name, path):
    op, noise, Sref = reference_run(name)
    q = MAKE[name]()
    q.device_handle().set_path(path.split("-")[0])
    field = "hilo" if path.endswith("hilo") else None
    S, _ = nb.run_with_noise(q, O.temperatures(T_F), noise, SIGMA, field=field)
    fl = flips(S, Sref)
    err = np.abs(S - Sref)
    e_gpu = O.energies(op, O.sign_round(S))
    e_ref = O.energies(op, O.sign_round(Sref))
    print(f"\n{name}/{path}: mean final-sign flips {fl.mean():.2e} (max replica {fl.max():.2e}, "
          f"replicas with any flip {np.mean(fl > 0):.2f}), mean|dS| {err.mean():.2e}; "
          f"identical final energy on {np.mean(e_gpu == e_ref):.2%} of replicas")
    if path in ("sparse", "dense-hilo"):
        assert fl.mean() <= (1e-4 if path == "sparse" else 2e-4), fl.mean()
        return
    emu = flips(_f16_operand_emulation(op, noise, O.temperatures(T_F)), Sref)
    print(f"{name}/{path}: fp16-operand emulation on the same noise: mean flips {emu.mean():.2e}")
    assert fl.mean() <= 2e-3, fl.mean()
    assert fl.mean() <= 2.0 * emu.mean() + 2e-4, (fl.mean(), emu.mean())
