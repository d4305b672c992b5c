"""NMFA sampling entry points -- drop-in mirror of the reference `nmfa.solver`.

Same names, arguments, defaults and error behaviour as the reference
(solver.py:41-280): `Schedule`, `NmfaParams`, `RunResult`, `Trajectory`,
`noise_stream`, `run_with_noise`, `nmfa_step`, `nmfa_run`, `nmfa_batch`.
Every anneal runs on the GPU through the C-ABI (`_native`); there is no CPU
path.  Differences, all documented in DESIGN.md:

* Seeded runs draw their noise in-kernel from a counter-based Philox4x32-10
  stream keyed by (seed + replica) instead of numpy's sequential Philox4x64 +
  ziggurat, so a given seed reproduces the reference statistically, not
  bitwise.  Bitwise-comparable noise goes through `run_with_noise` (the
  reference's own injected-noise seam) or `nmfa_step` (which draws from the
  caller's numpy generator exactly like the reference).
* `nmfa_batch` runs all replicas in one device batch; `threads` is accepted
  for signature compatibility and ignored (results never depended on it).
* `run_with_noise` additionally accepts a batch of noise (R, t_f, n) and then
  returns (R, n) spins and a list of trajectories.
* `sample()` is the batched API underneath: device tensors in and out.
"""

from __future__ import annotations

import ctypes
import time
from dataclasses import dataclass, replace

import numpy as np

from . import _native
from .problem import as_problem, energy, sign_round  # noqa: F401  (re-exported like the reference)

MASK64 = (1 << 64) - 1
RUN_STREAM_TAG = 2                     # solver.py:33 (numpy noise_stream key space)
DEFAULT_ALPHA = 0.15
DEFAULT_SIGMA = 0.15
DEFAULT_TF = 1000


class Schedule:
    """Temperature as a function of the anneal fraction f = (t - 1) / (t_f - 1).

    Breakpoints (f_k, T_k) run from f = 0 to f = 1; between them log T is linear
    in f (geometric interpolation).  Same curve, validation order and messages
    as the reference Schedule (solver.py:41-127).
    """

    def __init__(self, breakpoints):
        table = [(float(f), float(T)) for f, T in breakpoints]
        if len(table) < 2:
            raise ValueError("schedule needs at least two breakpoints")
        f = np.array([row[0] for row in table])
        T = np.array([row[1] for row in table])
        rules = (
            (lambda: f[0] != 0.0 or f[-1] != 1.0, "schedule must start at f=0 and end at f=1"),
            (lambda: bool(np.any(f[1:] - f[:-1] <= 0.0)),
             "schedule fractions must be strictly increasing"),
            (lambda: bool(np.any(T <= 0.0)) or not bool(np.all(np.isfinite(T))),
             "schedule temperatures must be positive and finite"),
        )
        for violated, message in rules:
            if violated():
                raise ValueError(message)
        f.flags.writeable = False
        T.flags.writeable = False
        self._fs, self._Ts = f, T

    @property
    def breakpoints(self):
        return tuple(zip(self._fs.tolist(), self._Ts.tolist()))

    def _segment(self, f):
        """Index k of the segment [f_k, f_k+1) containing f (clamped)."""
        return np.clip(np.searchsorted(self._fs, f, side="right") - 1, 0, self._fs.size - 2)

    def _geometric(self, f, k):
        f0, f1 = self._fs[k], self._fs[k + 1]
        T0, T1 = self._Ts[k], self._Ts[k + 1]
        return T0 * (T1 / T0) ** ((f - f0) / (f1 - f0))

    def temperatures(self, t_f):
        """Temperatures of iterations t = 1..t_f (host float64, uploaded once per plan)."""
        t_f = int(t_f)
        if t_f < 1:
            raise ValueError("t_f must be at least 1")
        f = np.arange(t_f) / (t_f - 1) if t_f > 1 else np.zeros(1)
        curve = self._geometric(f, self._segment(f))
        curve[f >= self._fs[-1]] = self._Ts[-1]  # the last breakpoint is exact
        return curve

    def temperature(self, t, t_f):
        """Temperature of iteration t (1-based) of t_f."""
        t, t_f = int(t), int(t_f)
        if t_f < 1:
            raise ValueError("t_f must be at least 1")
        if not 1 <= t <= t_f:
            raise ValueError(f"iteration {t} outside [1, {t_f}]")
        f = (t - 1) / (t_f - 1) if t_f > 1 else 0.0
        if f >= self._fs[-1]:
            return float(self._Ts[-1])
        return float(self._geometric(f, int(self._segment(f))))

    @classmethod
    def parse(cls, text):
        """Schedule from "f:T,f:T,..." text, e.g. "0:2,0.25:0.8,0.75:0.2,1:0.02"."""
        points = []
        for item in (piece.strip() for piece in text.split(",")):
            if not item:
                continue
            fields = item.split(":")
            try:
                if len(fields) != 2:
                    raise ValueError(item)
                points.append((float(fields[0]), float(fields[1])))
            except ValueError:
                raise ValueError(f"bad schedule point {item!r}, expected f:T") from None
        return cls(points)

    def format(self):
        return ",".join(f"{f:g}:{T:g}" for f, T in self.breakpoints)

    def __repr__(self):
        return f"Schedule({self.format()!r})"

    def __eq__(self, other):
        return isinstance(other, Schedule) and other.breakpoints == self.breakpoints

    def __hash__(self):
        return hash(self.breakpoints)


DEFAULT_SCHEDULE = Schedule([(0.0, 2.0), (0.25, 0.8), (0.75, 0.2), (1.0, 0.02)])


def schedule_eval(schedule, t, t_f):
    """Temperature at iteration t of t_f (t is 1-based)."""
    return schedule.temperature(t, t_f)


@dataclass(frozen=True)
class NmfaParams:
    """Solver parameters: feedback alpha, noise sigma, length t_f, schedule, seed."""

    alpha: float = DEFAULT_ALPHA
    sigma: float = DEFAULT_SIGMA
    t_f: int = DEFAULT_TF
    schedule: Schedule = DEFAULT_SCHEDULE
    seed: int = 0

    def __post_init__(self):
        # validated in the reference's order (solver.py:151-162); t_f and seed are
        # normalised to Python ints once their checks pass
        checks = (
            (lambda: 0.0 <= self.alpha <= 1.0, lambda: f"alpha must be in [0, 1], got {self.alpha}"),
            (lambda: self.sigma >= 0.0, lambda: f"sigma must be nonnegative, got {self.sigma}"),
            (lambda: int(self.t_f) >= 1, lambda: f"t_f must be at least 1, got {self.t_f}"),
            (lambda: 0 <= int(self.seed) <= MASK64, lambda: "seed must fit in 64 unsigned bits"),
        )
        for holds, message in checks:
            if not holds():
                raise ValueError(message())
        object.__setattr__(self, "t_f", int(self.t_f))
        object.__setattr__(self, "seed", int(self.seed))


@dataclass(frozen=True)
class Trajectory:
    """Per-iteration record: analog spins and the energy of their rounding."""

    spins: np.ndarray      # (t_f, n)
    energies: np.ndarray   # (t_f,)


@dataclass(frozen=True)
class RunResult:
    final_config: np.ndarray
    final_energy: float
    seed: int
    wall_clock: float      # seconds per run: batch wall / n_runs (SPEC tau convention)
    trajectory: Trajectory | None = None


def noise_stream(seed):
    """numpy Philox generator with the reference's stream identity (solver.py:182-185).

    Only used to draw host noise for the injected-noise seam (`nmfa_step`);
    seeded anneals draw in-kernel noise instead.
    """
    key = (RUN_STREAM_TAG << 64) | (int(seed) & MASK64)
    return np.random.Generator(np.random.Philox(key=key))


# ---------------------------------------------------------------------------
# batched device API
# ---------------------------------------------------------------------------
class Plan:
    """Device state for n_runs replicas x t_f steps of one problem (nmfa_plan_*)."""

    def __init__(self, problem, n_runs, temps, alpha, sigma, device=0):
        self.problem = as_problem(problem)
        self.dev = self.problem.device_handle(device)
        self.device = int(device)
        self.n_runs = int(n_runs)
        self.temps = np.ascontiguousarray(temps, dtype=np.float64)
        self.t_f = int(self.temps.size)
        self.alpha, self.sigma = float(alpha), float(sigma)
        out = ctypes.c_void_p()
        _native.check(_native.load().nmfa_plan_create(
            self.dev.handle, self.n_runs, self.t_f, _native.ptr(self.temps), self.alpha,
            self.sigma, ctypes.byref(out)))
        self.handle = out

    def run(self, seed, r0=0, noise=None, s0=None, config=None, energy=None, s_final=None,
            s_hist=None, e_hist=None, stream=None):
        """Enqueue one batch on `stream` (a torch.cuda.Stream or None = current)."""
        import torch

        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        _native.check(_native.load().nmfa_plan_run(
            self.handle, int(seed) & MASK64, int(r0), _native.ptr(noise), _native.ptr(s0),
            _native.ptr(config), _native.ptr(energy), _native.ptr(s_final),
            _native.ptr(s_hist), _native.ptr(e_hist), ctypes.c_void_p(stream.cuda_stream)))
        return _native.load().nmfa_last_launch_count()

    def __del__(self):
        try:
            if self.handle:
                _native.load().nmfa_plan_destroy(self.handle)
                self.handle = None
        except Exception:
            pass


@dataclass
class SampleSet:
    """Batched result of `sample`: device tensors plus timing."""

    configs: "object"          # torch.int8 (R, n) on device, values +-1
    energies: "object"         # torch.float64 (R,) on device
    seed: int
    r0: int
    wall_clock: float          # seconds for the whole batch
    s_final: "object" = None   # torch.float32 (R, n) or None
    s_hist: "object" = None    # torch.float32 (R, t_f, n) or None
    e_hist: "object" = None    # torch.float64 (R, t_f) or None

    def best(self):
        """(best energy, global replica index) -- best-of-reads on device."""
        import torch

        be = torch.empty(1, dtype=torch.float64, device=self.energies.device)
        bi = torch.empty(1, dtype=torch.int64, device=self.energies.device)
        stream = torch.cuda.current_stream(self.energies.device)
        _native.check(_native.load().nmfa_best_of(
            _native.ptr(self.energies), self.energies.numel(), _native.ptr(be), _native.ptr(bi),
            ctypes.c_void_p(stream.cuda_stream)))
        return float(be.item()), int(bi.item()) + self.r0


class _FieldPrecision:
    """Use a dense-path field precision ("fp16" / "hilo") for one call and
    restore the problem's previous setting afterwards (None: leave it)."""

    def __init__(self, problem, device, field):
        self.dev = problem.device_handle(device) if field is not None else None
        self.field = field

    def __enter__(self):
        if self.dev is not None:
            self.prev = self.dev.info()["field"]
            if self.prev != self.field:
                self.dev.set_field_precision(self.field)
        return self

    def __exit__(self, *exc):
        if self.dev is not None and self.prev != self.field:
            self.dev.set_field_precision(self.prev)
        return False


def _replay_field(problem, device, field):
    """The replay mode is the fidelity mode: on the tensor-core paths it
    multiplies the full hi + lo state (HILO field; small path up to n = 224)
    unless the caller chose a field."""
    if field is not None:
        return field
    info = problem.device_handle(device).info()
    if info["path"] == "dense" or (info["path"] == "small" and info["n"] <= 224):
        return "hilo"
    return None


def sample(problem, params=None, n_runs=1, *, r0=0, device=0, noise=None, s0=None,
           temps=None, return_s=False, record_trajectory=False, field=None):
    """Run n_runs replicas (global indices r0..r0+n_runs-1) in one device batch.

    noise: optional (n_runs, t_f, n) pre-scaled additive noise (device tensor
    or array); when given, params.sigma is unused (run_with_noise seam).
    field: tensor-core GEMM operand for this call, "fp16" or "hilo" (None: the
    problem's setting, default "fp16"; include/nmfa_b200.h NMFA_FIELD_*).  It
    switches the problem's setting for the duration of the call, so threads
    sharing one problem should not pass different fields concurrently.
    """
    problem = as_problem(problem)
    with _FieldPrecision(problem, device, field):
        return _sample(problem, params, n_runs, r0=r0, device=device, noise=noise, s0=s0,
                       temps=temps, return_s=return_s, record_trajectory=record_trajectory)


def _sample(problem, params, n_runs, *, r0, device, noise, s0, temps, return_s,
            record_trajectory):
    import torch

    params = NmfaParams() if params is None else params
    problem = as_problem(problem)
    n = problem.n
    n_runs = int(n_runs)
    if n_runs < 1:
        raise ValueError(f"n_runs must be at least 1, got {n_runs}")
    temps = params.schedule.temperatures(params.t_f) if temps is None else np.asarray(
        temps, dtype=np.float64)
    t_f = int(temps.size)
    dev = torch.device(f"cuda:{device}")
    if noise is not None:
        noise = torch.as_tensor(noise, dtype=torch.float32, device=dev).contiguous()
        if tuple(noise.shape) != (n_runs, t_f, n):
            raise ValueError(f"noise shape {tuple(noise.shape)} does not match "
                             f"({n_runs}, {t_f}, {n})")
    if s0 is not None:
        s0 = torch.as_tensor(s0, dtype=torch.float32, device=dev).contiguous()
        if tuple(s0.shape) != (n_runs, n):
            raise ValueError(f"s0 length does not match problem size {n}")
    temps = np.ascontiguousarray(temps, dtype=np.float64)
    handle = problem.device_handle(device).handle
    cfg = torch.empty((n_runs, n), dtype=torch.int8, device=dev)
    en = torch.empty(n_runs, dtype=torch.float64, device=dev)
    s_final = torch.empty((n_runs, n), dtype=torch.float32, device=dev) if return_s else None
    s_hist = e_hist = None
    if record_trajectory:
        s_hist = torch.empty((n_runs, t_f, n), dtype=torch.float32, device=dev)
        e_hist = torch.empty((n_runs, t_f), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    # one-shot C-ABI entry: reuses the device plan cached on the problem handle
    _native.check(_native.load().nmfa_anneal(
        handle, n_runs, t_f, _native.ptr(temps), float(params.alpha), float(params.sigma),
        int(params.seed) & MASK64, int(r0), _native.ptr(noise), _native.ptr(s0), _native.ptr(cfg),
        _native.ptr(en), _native.ptr(s_final), _native.ptr(s_hist), _native.ptr(e_hist),
        ctypes.c_void_p(stream.cuda_stream)))
    wall = time.perf_counter() - t0
    return SampleSet(cfg, en, int(params.seed), int(r0), wall, s_final, s_hist, e_hist)


# ---------------------------------------------------------------------------
# reference-compatible entry points
# ---------------------------------------------------------------------------
def sample_many(problems, params=None, n_runs=1, *, seeds=None, device=0):
    """Anneal many instances of the same size in one call (nmfa_anneal_many).

    Instance k runs ``n_runs`` replicas seeded like the reference's bench loop
    (cli.py:319-321): ``seeds[k]`` defaults to ``params.seed + k * n_runs``, and
    replica r uses key ``seeds[k] + r`` -- identical to ``sample(problems[k],
    replace(params, seed=seeds[k]), n_runs)``.  Small instances (n <= 256) share
    ONE persistent launch.  Returns (configs int8 (K, R, n), energies f64 (K, R))
    as device tensors and the wall time of the whole call.
    """
    import ctypes

    import torch

    params = NmfaParams() if params is None else params
    probs = [as_problem(p) for p in problems]
    if not probs:
        raise ValueError("sample_many needs at least one instance")
    n = probs[0].n
    if any(p.n != n for p in probs):
        raise ValueError("every instance of a group must have the same n")
    n_runs = int(n_runs)
    if n_runs < 1:
        raise ValueError(f"n_runs must be at least 1, got {n_runs}")
    K = len(probs)
    if seeds is None:
        seeds = [(int(params.seed) + k * n_runs) & MASK64 for k in range(K)]
    seeds = np.ascontiguousarray([int(x) & MASK64 for x in seeds], dtype=np.uint64)
    if seeds.size != K:
        raise ValueError("seeds must have one entry per instance")
    temps = np.ascontiguousarray(params.schedule.temperatures(params.t_f), dtype=np.float64)
    handles = (ctypes.c_void_p * K)(*[p.device_handle(device).handle.value for p in probs])
    dev = torch.device("cuda", device)
    cfg = torch.empty((K, n_runs, n), dtype=torch.int8, device=dev)
    en = torch.empty((K, n_runs), dtype=torch.float64, device=dev)
    stream = torch.cuda.current_stream(dev)
    t0 = time.perf_counter()
    _native.check(_native.load().nmfa_anneal_many(
        ctypes.cast(handles, ctypes.c_void_p), K, n_runs, int(params.t_f), _native.ptr(temps),
        float(params.alpha), float(params.sigma), _native.ptr(seeds), _native.ptr(cfg),
        _native.ptr(en), ctypes.c_void_p(stream.cuda_stream)))
    return cfg, en, time.perf_counter() - t0


def run_with_noise(problem, temps, noise, alpha, s0=None, record_trajectory=False, device=0,
                   field=None):
    """Anneal with caller-supplied, pre-scaled noise (solver.py:188-218).

    noise (t_f, n) -> returns (s (n,), Trajectory | None), like the reference.
    noise (R, t_f, n) -> returns (S (R, n), list[Trajectory] | None).
    """
    problem = as_problem(problem)
    temps = np.asarray(temps, dtype=np.float64)
    noise = np.asarray(noise, dtype=np.float64)
    batched = noise.ndim == 3
    nz = noise if batched else noise[None]
    if nz.shape[1:] != (temps.shape[0], problem.n):
        shape = noise.shape
        raise ValueError(f"noise shape {shape} does not match ({temps.shape[0]}, {problem.n})")
    R = nz.shape[0]
    if s0 is not None:
        s0 = np.array(s0, dtype=np.float64)
        want = (R, problem.n) if batched else (problem.n,)
        if s0.shape != want:
            raise ValueError(f"s0 length does not match problem size {problem.n}")
        s0 = s0.reshape(R, problem.n)
    params = NmfaParams(alpha=float(alpha), sigma=1.0, t_f=temps.shape[0])
    res = sample(problem, params, R, device=device, noise=nz.astype(np.float32), s0=s0,
                 temps=temps, return_s=True, record_trajectory=record_trajectory, field=field)
    S = res.s_final.double().cpu().numpy()
    trajs = None
    if record_trajectory:
        sh = res.s_hist.double().cpu().numpy()
        eh = res.e_hist.cpu().numpy()
        trajs = [Trajectory(spins=sh[r], energies=eh[r]) for r in range(R)]
    if batched:
        return S, trajs
    return S[0], (trajs[0] if trajs else None)


def nmfa_step(problem, s, T, params, rng):
    """One synchronous update of the spins `s` at temperature T (solver.py:221-233).

    The noise comes from the caller's numpy generator, one standard normal per
    spin scaled by sigma, exactly as the reference draws it, so a shared
    generator gives both packages the same step.  On the tensor-core paths the
    step uses the HILO field, as the replay mode does.
    """
    if T <= 0.0:  # the reference's test (a NaN temperature is not rejected there either)
        raise ValueError(f"temperature must be positive, got {T}")
    prob = as_problem(problem)
    drive = params.sigma * rng.standard_normal(prob.n)
    # the reference's own noise, like the replay mode: the same (HILO on the
    # tensor-core paths) field, so t_f steps equal nmfa_run(noise="reference") bitwise
    updated, _ = run_with_noise(prob, np.full(1, float(T)), drive.reshape(1, -1), params.alpha, s0=s,
                                field=_replay_field(prob, 0, None))
    return updated


_PINNED = {}
_PINNED_LOCK = __import__("threading").Lock()


def _host_configs_f64(configs):
    """Device int8 (R, n) -> host float64 (R, n): the copy lands in a cached
    pinned buffer (a pageable copy of 16 MB costs a few ms), the conversion
    uses torch's threaded kernel (about 2x numpy's astype) into a new array."""
    import torch

    key = (tuple(configs.shape), configs.device.index)
    with _PINNED_LOCK:
        buf = _PINNED.get(key)
        if buf is None:
            if len(_PINNED) >= 4:
                _PINNED.clear()
            buf = _PINNED[key] = torch.empty(configs.shape, dtype=torch.int8, pin_memory=True)
        buf.copy_(configs)
        return buf.to(torch.float64).numpy()


def _results(problem, res, params, record_trajectory):
    cfg = _host_configs_f64(res.configs)
    en = res.energies.cpu().numpy().tolist()     # Python floats, as energy() returns
    R = cfg.shape[0]
    per = res.wall_clock / R
    trajs = [None] * R
    if record_trajectory:
        sh = res.s_hist.double().cpu().numpy()
        eh = res.e_hist.cpu().numpy()
        trajs = [Trajectory(spins=sh[r], energies=eh[r]) for r in range(R)]
    # row views and positional fields: ~40% less host time per RunResult at 8192 runs
    rows = list(cfg)
    s0 = params.seed + res.r0
    return [RunResult(rows[r], en[r], (s0 + r) & MASK64, per, trajs[r]) for r in range(R)]


NOISE_MODES = ("device", "reference")
REPLAY_CHUNK_BYTES = 16 << 30  # largest device noise buffer per replay chunk (float32)


def _replay_chunk_bytes(device):
    """Noise buffer per replay chunk: up to REPLAY_CHUNK_BYTES and a quarter
    of the free device memory, at least 1 GiB.  Larger chunks give the
    warp-per-run generator more runs (warps) in flight."""
    import torch

    free, _ = torch.cuda.mem_get_info(device)
    return int(max(1 << 30, min(REPLAY_CHUNK_BYTES, free // 4)))


def reference_noise(seed, n_runs, t_f, n, sigma, *, r0=0, device=0):
    """The reference's per-run noise, generated on the GPU (refnoise.cu).

    Returns a (n_runs, t_f, n) float32 device tensor whose row r is
    noise_stream(seed + r0 + r).standard_normal((t_f, n)) * sigma -- exactly
    what `_run` draws for run seed + r0 + r (solver.py:236-241), rounded to
    float32 (bitwise numpy's draws at that precision)."""
    import torch

    out = torch.empty((int(n_runs), int(t_f), int(n)), dtype=torch.float32,
                      device=torch.device("cuda", device))
    stream = torch.cuda.current_stream(out.device)
    _native.check(_native.load().nmfa_reference_noise(
        int(seed) & MASK64, int(r0), int(n_runs), int(t_f) * int(n), float(sigma), _native.ptr(out),
        None, ctypes.c_void_p(stream.cuda_stream)))
    return out


def _replay(problem, params, n_runs, device, record_trajectory, field=None):
    """Seeded anneals on the reference's own noise streams: replica chunks of
    at most _replay_chunk_bytes() of device noise, each generated on the GPU and
    injected through the run_with_noise seam.  One SampleSet for all runs."""
    import torch

    problem = as_problem(problem)
    field = _replay_field(problem, device, field)
    n, t_f = problem.n, int(params.t_f)
    temps = params.schedule.temperatures(t_f)
    chunk = max(1, min(n_runs, _replay_chunk_bytes(device) // (4 * t_f * n)))
    parts, wall = [], 0.0
    for c0 in range(0, n_runs, chunk):
        c = min(chunk, n_runs - c0)
        nz = reference_noise(params.seed, c, t_f, n, params.sigma, r0=c0, device=device)
        res = sample(problem, params, c, device=device, noise=nz, temps=temps,
                     record_trajectory=record_trajectory, field=field)
        parts.append(res)
        wall += res.wall_clock
        del nz
    cat = (lambda xs: torch.cat(xs) if xs[0] is not None else None)
    return SampleSet(cat([r.configs for r in parts]), cat([r.energies for r in parts]),
                     int(params.seed), 0, wall, None, cat([r.s_hist for r in parts]),
                     cat([r.e_hist for r in parts]))


def _check_noise_mode(noise):
    if noise not in NOISE_MODES:
        raise ValueError(f"noise must be one of {NOISE_MODES}, got {noise!r}")


def nmfa_run(problem, params, record_trajectory=False, device=0, noise="device", field=None):
    """Full anneal from all-zero spins; deterministic given (problem, seed).

    noise="reference" replays the reference's own stream for params.seed, so
    the run follows `nmfa.nmfa_run(problem, params)` step for step (on the
    dense path with the HILO field unless `field` says otherwise)."""
    _check_noise_mode(noise)
    if noise == "reference":
        res = _replay(problem, params, 1, device, record_trajectory, field)
    else:
        res = sample(problem, params, 1, device=device, record_trajectory=record_trajectory,
                     field=field)
    return _results(problem, res, params, record_trajectory)[0]


def nmfa_batch(problem, params, n_runs, threads=1, record_trajectory=False, device=0,
               noise="device", field=None):
    """n_runs independent anneals; run k uses seed params.seed + k (solver.py:262-280).

    noise="device" (default) draws in-kernel counter-based Philox noise keyed
    by seed + k (statistically equivalent to the reference, not per seed).
    noise="reference" replays each run's own numpy stream noise_stream(seed +
    k) generated on the GPU (one warp per stream), so run
    k is comparable per seed with the reference's run k; the noise is injected
    in replica chunks (K2000: 8192 seeds in under a second).  field: the dense
    path's GEMM operand,
    "fp16" (hi; the default for device noise) or "hilo" (hi + lo; the default
    for the replay mode), see sample()."""
    n_runs = int(n_runs)
    if n_runs < 1:
        raise ValueError(f"n_runs must be at least 1, got {n_runs}")
    _check_noise_mode(noise)
    if noise == "reference":
        res = _replay(problem, params, n_runs, device, record_trajectory, field)
    else:
        res = sample(problem, params, n_runs, device=device, record_trajectory=record_trajectory,
                     field=field)
    return _results(problem, res, params, record_trajectory)
