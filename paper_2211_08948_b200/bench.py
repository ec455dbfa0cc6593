"""Work-precision harness on the device engines.

Drop-in for `expkit.bench` (bench.py:1-246): the same names, CSV layout
(header pinned by test_bench.py:14-18, plus the trailing `error` column),
`.ref` cache format (little-endian u64 count + fp64 payload,
bench.py:85-101; file name = sha256 of "problem|param!r|n|t_final!r") and
failure semantics (a failed run is recorded, not raised). Every run goes
through this package's `adaptive_loop`, i.e. the sm_100a Leja / KIOPS /
LeKry engines; only the bookkeeping is host code.

    from paper_2211_08948_b200.bench import SweepConfig, expand_matrix, run_sweep
"""

import csv
import hashlib
import math
import struct
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from .errors import StepFailure
from .integrators import INTEGRATORS, LEKRY_INTEGRATORS, SCHEMES, EngineContext
from .linalg import norm_l2
from .problems import PROBLEMS, make_problem
from .timestep import adaptive_loop

_COLUMNS = ("problem", "param", "n", "integrator", "scheme", "tol", "steps_accepted",
            "steps_rejected", "rhs_evals", "leja_iters", "krylov_matvecs", "substeps",
            "wall_time_s", "l2_error")
CSV_HEADER = ",".join(_COLUMNS)
DEFAULT_TOLS = tuple(10.0 ** -e for e in range(3, 10))  # 1e-3 .. 1e-9
REFERENCE_TOL = 1e-12

# Trajectory counters copied into a RunRecord (bench.py:153-158)
_COUNTERS = ("steps_accepted", "steps_rejected", "rhs_evals", "leja_iters",
             "krylov_matvecs", "substeps")


def _isnan(x):
    return isinstance(x, float) and math.isnan(x)


@dataclass(frozen=True)
class RunConfig:
    """One cell of the work-precision matrix (bench.py:31-54)."""

    problem: str
    param: float  # diffusion coefficient; NaN for parameter-free problems
    n: int
    integrator: str
    scheme: str
    tol: float
    t_final: float = None
    seed: int = 0

    def validate(self):
        checks = ((self.problem in PROBLEMS, f"unknown problem '{self.problem}'"),
                  (self.integrator in INTEGRATORS, f"unknown integrator '{self.integrator}'"),
                  (self.scheme in SCHEMES, f"unknown scheme '{self.scheme}'"),
                  (self.scheme != "lekry" or self.integrator in LEKRY_INTEGRATORS,
                   f"integrator '{self.integrator}' has no lekry scheme"),
                  (0.0 < self.tol < 1.0, "tol must be in (0, 1)"))
        for ok, msg in checks:
            if not ok:
                raise ValueError(msg)


@dataclass
class RunRecord:
    """Counters, timing and error of one run (bench.py:57-71)."""

    config: RunConfig
    steps_accepted: int = 0
    steps_rejected: int = 0
    rhs_evals: int = 0
    leja_iters: int = 0
    krylov_matvecs: int = 0
    substeps: int = 0
    wall_time_s: float = 0.0
    l2_error: float = math.nan
    error: str = ""

    @property
    def failed(self):
        return self.error != ""


def _make(config):
    """The problem instance of a config; semilinear takes no alpha
    (bench.py:74-82)."""
    kw = {"n": config.n}
    if config.problem != "semilinear":
        kw["alpha"] = config.param
    prob = make_problem(config.problem, **kw)
    if config.t_final is not None:
        prob.t_final = config.t_final
    return prob


def _ref_key(problem, param, n, t_final):
    return hashlib.sha256(f"{problem}|{param!r}|{n}|{t_final!r}".encode()).hexdigest()


def _ref_write(path, u):
    a = np.ascontiguousarray(np.asarray(u, dtype=np.float64)).astype("<f8", copy=False)
    Path(path).write_bytes(struct.pack("<Q", a.size) + a.tobytes())


def _ref_read(path):
    raw = Path(path).read_bytes()
    if len(raw) < 8:
        raise ValueError(f"corrupt reference file {path}")
    count = struct.unpack("<Q", raw[:8])[0]
    if len(raw) - 8 < 8 * count:
        raise ValueError(f"corrupt reference file {path}")
    return np.frombuffer(raw, dtype="<f8", count=count, offset=8).astype(np.float64)


def _loop(prob, integrator, scheme, tol):
    return adaptive_loop(prob.rhs, prob.u0, prob.t_final, integrator, scheme, tol,
                         jac_factory=prob.jac_factory, ctx=EngineContext())


def build_reference(problem, param, n, cache_dir=None, t_final=None,
                    reference_tol=REFERENCE_TOL):
    """Reference state: the exact solution if the problem has one, else a
    tight EPIRK5P1 + KIOPS run, cached as a `.ref` file (bench.py:104-135)."""
    prob = _make(RunConfig(problem, param, n, "epirk5p1", "kiops", reference_tol,
                           t_final=t_final))
    if prob.exact is not None:
        return prob.exact(prob.t_final)
    path = None
    if cache_dir is not None:
        cache = Path(cache_dir)
        cache.mkdir(parents=True, exist_ok=True)
        path = cache / f"{_ref_key(problem, param, n, prob.t_final)}.ref"
        if path.exists():
            return _ref_read(path)
    try:
        traj = _loop(prob, "epirk5p1", "kiops", reference_tol)
    except StepFailure as exc:
        raise StepFailure(f"reference run failed for {problem} (param={param}, n={n}); "
                          f"retry with a looser reference_tol", cause=exc) from exc
    u_ref = np.asarray(prob.extract(traj.u), dtype=np.float64)
    if path is not None:
        _ref_write(path, u_ref)
    return u_ref


def run_one(config, u_ref=None, ref_cache_dir=None):
    """Run one config through the device engines; StepFailure /
    FloatingPointError are recorded in `error` (bench.py:138-164)."""
    config.validate()
    if u_ref is None:
        u_ref = build_reference(config.problem, config.param, config.n,
                                cache_dir=ref_cache_dir, t_final=config.t_final)
    prob = _make(config)
    rec = RunRecord(config=config)
    start = time.perf_counter()
    try:
        traj = _loop(prob, config.integrator, config.scheme, config.tol)
    except (StepFailure, FloatingPointError) as exc:
        rec.wall_time_s = time.perf_counter() - start
        rec.error = f"{type(exc).__name__}: {exc}"
        return rec
    rec.wall_time_s = time.perf_counter() - start
    for name in _COUNTERS:
        setattr(rec, name, getattr(traj, name))
    u = prob.extract(traj.u)
    rec.l2_error = norm_l2(u - u_ref) / norm_l2(u_ref)
    return rec


def _fmt(x):
    """Floats round-trip (%.17g), NaN as 'nan' (bench.py:167-170)."""
    if isinstance(x, float):
        return "nan" if math.isnan(x) else "%.17g" % x
    return str(x)


def record_row(rec):
    c = rec.config
    param = "" if _isnan(c.param) else _fmt(float(c.param))
    head = [c.problem, param, str(c.n), c.integrator, c.scheme, _fmt(c.tol)]
    counts = [str(getattr(rec, name)) for name in _COUNTERS]
    return head + counts + [_fmt(rec.wall_time_s), _fmt(rec.l2_error), rec.error]


def write_csv(records, out_path):
    with Path(out_path).open("w", encoding="utf-8", newline="") as fh:
        fh.write(CSV_HEADER + ",error\n")
        w = csv.writer(fh, lineterminator="\n")
        w.writerows(record_row(r) for r in records)


@dataclass
class SweepConfig:
    """Axes of a work-precision sweep (bench.py:195-203)."""

    problems: list
    params: dict = field(default_factory=dict)  # problem -> [alpha, ...]
    n: int = 64
    integrators: list = field(default_factory=lambda: list(INTEGRATORS))
    schemes: list = field(default_factory=lambda: list(SCHEMES))
    tols: tuple = DEFAULT_TOLS
    t_final: float = None


def expand_matrix(sweep):
    """Cartesian product problem x param x integrator x scheme x tol, in that
    nesting order, without the lekry cells an integrator lacks
    (bench.py:206-223)."""
    out = []
    for problem in sweep.problems:
        params = [math.nan] if problem == "semilinear" else sweep.params.get(problem, [math.nan])
        for param in params:
            for integ in sweep.integrators:
                schemes = [s for s in sweep.schemes
                           if s != "lekry" or integ in LEKRY_INTEGRATORS]
                for scheme in schemes:
                    out.extend(RunConfig(problem, param, sweep.n, integ, scheme, tol,
                                         t_final=sweep.t_final) for tol in sweep.tols)
    return out


def run_sweep(configs, out_path, ref_cache_dir=None):
    """Validate all configs, build each distinct reference once, run every
    config in order and write the CSV (bench.py:226-246)."""
    def key(cfg):
        return (cfg.problem, None if _isnan(cfg.param) else cfg.param, cfg.n, cfg.t_final)

    refs = {}
    for cfg in configs:
        cfg.validate()
        k = key(cfg)
        if k not in refs:
            refs[k] = build_reference(cfg.problem, cfg.param, cfg.n,
                                      cache_dir=ref_cache_dir, t_final=cfg.t_final)
    records = [run_one(cfg, u_ref=refs[key(cfg)]) for cfg in configs]
    write_csv(records, out_path)
    return records
