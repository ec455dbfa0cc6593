"""Real-Leja interpolation of phi-function actions on the GPU.

Drop-in for `expkit.leja` (leja.py:1-189). Host side (unchanged semantics):
the Leja point sequence and its text cache, and the divided differences at
the Leja points (first column of phi_l of a bidiagonal node matrix, scipy
`expm` — BASELINE.json north_star keeps them on the host). Device side: the
Newton-Leja recurrence.

For a native stencil Jacobian every iteration is ONE fused kernel
(`ek_leja_run`): the Jacobian stencil (FD or analytic), the shifted/scaled
recurrence y' = J y / gamma - (c/gamma + xi[m-1]) y, all k polynomial
accumulators p_i += d_i[m] y', the deterministic ||y'||^2 reduction and the
per-coefficient freeze test |d_i[m]| ||y'|| < tol — decided on the device
with the reference's own fp64 expression. The host uploads one 32-column
coefficient chunk at a time (the reference recomputes its divided
differences per 32-point chunk, leja.py:168-171) and synchronises once per
launch batch, never per iteration.
"""

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _ddpool
from . import _device as D
from . import _native as N
from .errors import NonConvergence
from ._dense import phi_divided_differences, phi_divided_differences_many
from .linalg import MatrixFreeOperator, fused_target
from .spectrum import SpectrumEstimate

DEFAULT_NUM_POINTS = 400
DEFAULT_CANDIDATES = 100_000
_CHUNK = 32

_cached_points = None

# Optional measurement hook (bench.py): when a list, each fused call
# appends {"events": [(start, end), ...], "iters", "freeze", "k", "n", "fd"}
# with CUDA events bracketing its ek_leja_run launch batches.
PROFILE = None
_FASTCALL = os.environ.get("EK_LEJA_FASTCALL", "1") != "0"  # A/B switch (tools)
# the iterations of a whole-grid fused call as ONE launch
# of a CUDA graph with a device-side WHILE loop (ek_leja_run_graph): the call
# runs to its end or to the 32-point chunk boundary with no launch batch to
# size. "0" keeps the launch batches (A/B runs, tools).
_GRAPH = [os.environ.get("EK_LEJA_GRAPH", "1") != "0"]
# Deferred accumulation (ek_leja_run_seq / ek_leja_combine): on large grids the
# iterations keep every iterate in its own buffer and one pass forms the
# accumulators at the end — M + 1 + k vector transfers per call instead of
# 2kM, the same bits. [on, smallest vector length, smallest group (analytic
# Jacobian), byte budget of the iterate buffers of one call, smallest group
# (FD Jacobian: the K = 0 iteration saves the second f evaluation's traffic
# too, so a single accumulator already pays: config 4 k = 1 call 5.56 -> 5.05 ms)]
_DEFER = [os.environ.get("EK_LEJA_DEFER", "1") != "0",
          int(os.environ.get("EK_LEJA_DEFER_MIN_N", str(1 << 22))),
          int(os.environ.get("EK_LEJA_DEFER_MIN_K", "2")),
          int(os.environ.get("EK_LEJA_DEFER_BYTES", str(48 << 30))),
          int(os.environ.get("EK_LEJA_DEFER_MIN_K_FD", "1"))]


def generate_leja_points(m=DEFAULT_NUM_POINTS, n_candidates=DEFAULT_CANDIDATES):
    """Greedy Leja sequence on [-2, 2] from xi_0 = 2 (leja.py:32-50): each
    point maximises the log-product of distances on a uniform candidate grid,
    ties toward the smaller candidate."""
    if m < 1:
        raise ValueError("need at least one point")
    cand = np.linspace(-2.0, 2.0, n_candidates)
    pts = np.empty(m)
    pts[0] = 2.0
    with np.errstate(divide="ignore"):
        score = np.log(np.abs(cand - pts[0]))
        for k in range(1, m):
            pts[k] = cand[int(np.argmax(score))]
            score += np.log(np.abs(cand - pts[k]))
    return pts


def _default_cache_path():
    root = os.environ.get("XDG_CACHE_HOME") or str(Path.home() / ".cache")
    return Path(root) / "expkit" / "leja_points.txt"


def get_leja_points(m=DEFAULT_NUM_POINTS, cache_path=None):
    """Leja points from the in-process / text cache (leja.py:58-76); the
    text format (%.17g per line) round-trips exactly."""
    global _cached_points
    if _cached_points is not None and len(_cached_points) >= m:
        return _cached_points[:m]
    path = Path(cache_path) if cache_path is not None else _default_cache_path()
    if path.exists():
        pts = np.loadtxt(path, ndmin=1)
        if len(pts) >= m:
            _cached_points = pts
            return pts[:m]
    pts = generate_leja_points(max(m, DEFAULT_NUM_POINTS))
    try:
        path.parent.mkdir(parents=True, exist_ok=True)
        np.savetxt(path, pts, fmt="%.17g")
    except OSError:
        pass
    _cached_points = pts
    return pts[:m]


@dataclass(frozen=True)
class DividedDifferences:
    d: np.ndarray
    l: int
    h: float
    c: float
    gamma: float


_DD_CACHE = {}
_DD_CACHE_MAX = 128


def _dd_key(l, h, est, xi, m_max):
    return (l, h, est.c, est.gamma, min(m_max, len(xi)), id(xi), len(xi),
            float(xi[0]), float(xi[-1]))


def _dd_store(key, d):
    if len(_DD_CACHE) >= _DD_CACHE_MAX:
        _DD_CACHE.pop(next(iter(_DD_CACHE)))
    _DD_CACHE[key] = d


def _dd_prefetch(l, h, est, xi, m_max):
    """Start computing a later chunk's table in the worker pool (`_ddpool`):
    tables beyond the first chunk (m > 32) are always computed there, one
    BLAS thread each, so the bits do not depend on the caller's BLAS
    threading and the host work runs beside the device work."""
    m = min(m_max, len(xi))
    if m <= _CHUNK or not 0 <= l <= 4 or h < 0:
        return
    key = _dd_key(l, h, est, xi, m)
    if key in _DD_CACHE:
        return
    pool = _ddpool.existing()
    if pool is not None:
        try:
            pool.submit(key, (l, h, est.c, est.gamma, np.asarray(xi, dtype=np.float64), m))
        except Exception:  # noqa: BLE001 - worker trouble: compute in-process
            _ddpool.disable()


def _dd_cached(l, h, est, xi, m_max):
    """divided_differences(...).d memoised on its exact inputs: fixed-dt
    stepping and the 50-step spectrum reuse hit the same tables every step,
    so the host expm (0.2-2.7 ms per table) is paid once. Tables beyond the
    first chunk come from the worker pool (submitted ahead by the Leja loop
    when it can)."""
    key = _dd_key(l, h, est, xi, m_max)
    d = _DD_CACHE.get(key)
    if d is not None:
        return d
    _dd_prefetch(l, h, est, xi, m_max)
    pool = _ddpool.existing()
    if pool is not None and pool.pending(key):
        try:
            ok, val = pool.collect(key)
        except Exception:  # noqa: BLE001 - worker trouble: compute in-process
            _ddpool.disable()
            ok, val = False, None
        if ok:
            if not np.isfinite(val).all():  # as divided_differences()
                raise NonConvergence("non-finite divided differences; spectral estimate invalid")
            _dd_store(key, val)
            return val
    if min(m_max, len(xi)) > _CHUNK:
        with _one_blas_thread():
            d = divided_differences(l, h, est, xi, m_max).d
        _ddpool.pool()  # a chunk crossing: have the workers ready for the next ones
    else:
        d = divided_differences(l, h, est, xi, m_max).d
    _dd_store(key, d)
    return d


def _dd_group(l, hs, est, xi, m_max):
    """_dd_cached for the scales of one vertical group: first-chunk tables
    that miss the memo are computed in one batched exponential call
    (`_dense.phi_divided_differences_many`, the same bits per table)."""
    m = min(m_max, len(xi))
    keys = [_dd_key(l, h, est, xi, m_max) for h in hs]
    miss = [i for i, k in enumerate(keys) if k not in _DD_CACHE]
    if miss and m <= _CHUNK and 0 <= l <= 4 and min(hs) >= 0:
        ds = phi_divided_differences_many(l, [hs[i] for i in miss], est.c, est.gamma, xi, m)
        for i, d in zip(miss, ds):
            if not np.isfinite(d).all():  # as divided_differences()
                raise NonConvergence("non-finite divided differences; spectral estimate invalid")
            _dd_store(keys[i], d)
    return [_dd_cached(l, h, est, xi, m_max) for h in hs]


def _one_blas_thread():
    """In-process fallback for large tables: the pool's one-thread BLAS."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=1, user_api="blas")
    except ImportError:
        import contextlib
        return contextlib.nullcontext()


def divided_differences(l, h, est: SpectrumEstimate, xi, m_max):
    """Newton divided differences of z -> phi_l(h (c + gamma z)) at xi[:m_max]
    (leja.py:88-111), read off the first column of phi_l of the lower
    bidiagonal matrix diag(h (c + gamma xi)) + h gamma * subdiag."""
    if not 0 <= l <= 4:
        raise ValueError("phi order must be in 0..4")
    if h < 0:
        raise ValueError("scale h must be >= 0")
    m_max = min(m_max, len(xi))
    d = phi_divided_differences(l, h, est.c, est.gamma, xi, m_max)
    if not np.isfinite(d).all():
        raise NonConvergence("non-finite divided differences; spectral estimate invalid")
    return DividedDifferences(d=d, l=l, h=h, c=est.c, gamma=est.gamma)


@dataclass
class LejaResult:
    vectors: list
    iters: int
    freeze_iters: list


_KMAX = 8  # accumulators one fused pass / state block carries


def _vertical_wide(J, b, bd, l, coeffs, h, est, tol, xi, max_points):
    """A vertical group of more than _KMAX coefficients (the reference has
    no cap, leja.py:144-150): the shared recurrence runs once per iteration
    (one J.apply_dev, so the counter sees exactly the reference's charges),
    and the accumulators are updated in blocks of _KMAX, each with its own
    state block (same ||y_m||, its own freeze decisions); the loop ends when
    every block has frozen, at the largest freeze point — leja.py:167-189
    unchanged."""
    n = bd.numel()
    k = len(coeffs)
    c, gamma = est.c, est.gamma
    blocks = [list(range(i, min(k, i + _KMAX))) for i in range(0, k, _KMAX)]
    m_avail = min(_CHUNK, max_points)
    dds = _dd_group(l, [ci * h for ci in coeffs], est, xi, m_avail)
    ps = [D.empty(n) for _ in range(k)]
    tabs, sts = [], []
    ws = D.work_ptr()
    for blk in blocks:
        t = _CoefTable(len(blk))
        t.load(0, m_avail, [dds[i] for i in blk], c, gamma, xi)
        st = D.DevState(N.LejaState, tol=float(tol), nu=0.0, k=len(blk), p_init=0)
        N.check(N.lib().ek_leja_begin_len(n, C.c_void_p(bd.data_ptr()),
                                          N.ptrs([ps[i] for i in blk]), len(blk),
                                          C.c_void_p(t.dev.data_ptr()), st.ptr, ws, D.stream()),
                "ek_leja_begin_len")
        tabs.append(t)
        sts.append(st)
    hs = [st.read() for st in sts]
    done = [bool(hh.done) for hh in hs]
    ybuf = [D.empty(n), D.empty(n)]
    m, base = 1, 0
    while not all(done) and m < max_points:
        if m >= m_avail:  # next 32-point chunk (leja.py:168-171)
            m_avail = min(m_avail + _CHUNK, max_points)
            dds = _dd_group(l, [ci * h for ci in coeffs], est, xi, m_avail)
            base = m
            for blk, t in zip(blocks, tabs):
                t.load(base, m_avail, [dds[i] for i in blk], c, gamma, xi)
        y = bd if m == 1 else ybuf[(m - 1) & 1]
        jv = J.apply_dev(y)
        for bi, (blk, t, st) in enumerate(zip(blocks, tabs, sts)):
            if done[bi]:
                continue
            N.check(N.lib().ek_leja_update(
                n, C.c_void_p(jv.data_ptr()), C.c_void_p(y.data_ptr()),
                C.c_void_p(ybuf[m & 1].data_ptr()), N.ptrs([ps[i] for i in blk]), len(blk),
                C.c_void_p(t.dev.data_ptr()), base, m, float(gamma), 0, st.ptr, ws,
                D.stream()), "ek_leja_update")
        for bi, st in enumerate(sts):
            if not done[bi]:
                hs[bi] = st.read()
                if hs[bi].status == N.ST_NORM_NONFINITE:
                    raise NonConvergence("polynomial iteration diverged", iters=int(hs[bi].iters))
                done[bi] = bool(hs[bi].done)
        m += 1
    if not all(done):
        stalled = [coeffs[i] for bi, blk in enumerate(blocks) for j, i in enumerate(blk)
                   if (hs[bi].active >> j) & 1]
        raise NonConvergence(f"no convergence in {max_points} Leja points",
                             iters=max_points, detail={"stalled_coefficients": stalled})
    freeze = [int(hs[bi].freeze[j]) for bi, blk in enumerate(blocks) for j in range(len(blk))]
    return LejaResult(vectors=[D.like_input(p, b) for p in ps], iters=max(freeze),
                      freeze_iters=freeze)


def leja_interpolate(J: MatrixFreeOperator, b, l, h, est, tol,
                     xi=None, max_points=DEFAULT_NUM_POINTS):
    """p ~ phi_l(h J) b; returns (p, iters) (leja.py:121-130)."""
    res = leja_interpolate_vertical(J, b, l, [1.0], h, est, tol,
                                    xi=xi, max_points=max_points)
    return res.vectors[0], res.iters


class _CoefTable:
    """(k+1) x 32 device table of one chunk: row 0 the shifts
    c/gamma + xi[m-1] (Python-evaluated, leja.py:172), rows 1..k the divided
    differences d_i[m]."""

    def __init__(self, k):
        self.k = k
        self.dev = D.empty((k + 1) * _CHUNK)
        self.host = np.zeros((k + 1) * _CHUNK)

    def load(self, base, hi, dds, c, gamma, xi):
        self.fill(base, hi, dds, c, gamma, xi)
        self.upload()

    def upload(self):
        h = self.host
        N.check(N.lib().ek_copy(C.c_void_p(self.dev.data_ptr()),
                                h.ctypes.data_as(C.c_void_p), h.nbytes, 1, D.stream()),
                "coef upload")

    def fill(self, base, hi, dds, c, gamma, xi):
        h = self.host
        h[:] = 0.0
        lo = max(base, 1)
        if hi > lo:  # c/gamma + xi[m-1]: one Python-float quotient, then fp64 adds
            h[lo - base:hi - base] = (c / gamma) + np.asarray(xi[lo - 1:hi - 1], dtype=np.float64)
        for i, d in enumerate(dds):
            h[(1 + i) * _CHUNK:(1 + i) * _CHUNK + (hi - base)] = d[base:hi]


def _part_view(st):
    """The `part` field (EK_PART_SLOTS 8-byte slots) of a device state block,
    as a tensor."""
    fld = type(st.host).part
    return st.buf[fld.offset:fld.offset + fld.size].view(D.F64)


def _slab_decide(st, Jn, table, base, m, k, begin):
    comm = Jn.comm
    gathered = comm.allgather_pairs(_part_view(st))
    N.check(N.lib().ek_leja_decide(st.ptr, C.c_void_p(gathered.data_ptr()), comm.world,
                                   C.c_void_p(table.dev.data_ptr()), base, m, k,
                                   1 if Jn.jac == N.JAC_FD else 0, 1 if begin else 0,
                                   D.stream()), "ek_leja_decide")
    return gathered


class SpecMiss(Exception):
    """A speculative phi-call (see `leja_interpolate_vertical` _spec) did
    not finish inside its launch batch, or stopped on an error status: the
    step that used its vectors must be recomputed without speculation."""


def leja_interpolate_vertical(J: MatrixFreeOperator, b, l, coeffs, h, est, tol,
                              xi=None, max_points=DEFAULT_NUM_POINTS, _lazy_m0=False,
                              _first_batch=8, _spec=None, _spec_zero=False):
    """phi_l(c_i h J) b for several scale factors c_i sharing one Newton
    basis recurrence (leja.py:133-189). Accumulator i freezes once
    |d_i[m]| ||y_m|| < tol; the loop runs until all are frozen.

    Returns LejaResult(vectors, iters, freeze_iters); raises NonConvergence
    after `max_points` terms or on a non-finite ||y||.

    _first_batch: iterations enqueued before the first host check (the
    engines pass the previous count of the same group + 1, so a call usually
    needs one check; later iterations of a batch early-exit on the device).

    _lazy_m0 (integrator engines only, device b): if every accumulator
    freezes at m = 0 the results d_i[0]*b are returned as expressions
    (`_device.Expr`) that the stage algebra evaluates in registers with the
    same rounding, instead of being written to HBM.

    _spec (integrator engines only, fused single-GPU path): speculative call.
    The begin pass and ONE launch batch of `_first_batch` iterations are
    enqueued and the accumulators are returned at once, without a host
    synchronisation; the termination test already runs on the device (the
    kernels after termination early-exit), so the vectors are final if the
    call finished inside the batch. `_spec(iters, freeze_iters, fd_evals)`
    is called when the state block is read at the stream's next host sync
    (`_device.flush_checks`, in program order); if the call did not finish
    in the batch, or stopped on an error status, that read raises SpecMiss
    and the engines' caller recomputes the step without speculation
    (integrators.run_stepper), so results, counters and exceptions are
    those of the synchronous path. _spec_zero: the engines predict that
    every accumulator freezes at m = 0 (it did last time for this group);
    only the begin pass is enqueued and the results are the lazy
    expressions d_i[0]*b — the read checks iters == 0."""
    if tol <= 0:
        raise ValueError("tolerance must be positive")
    if len(coeffs) < 1:
        raise ValueError("need at least one coefficient")
    for ci in coeffs:
        if not 0.0 < ci <= 1.0:
            raise ValueError("coefficients must lie in (0, 1]")
    if xi is None:
        xi = get_leja_points(max_points)
    k = len(coeffs)
    c, gamma = est.c, est.gamma
    bd = D.to_dev(b)
    n = bd.numel()
    if n != J.dim:
        raise ValueError(f"expected vector of length {J.dim}, got {n}")
    if k > _KMAX:
        return _vertical_wide(J, b, bd, l, coeffs, h, est, tol, xi, max_points)

    m_avail = min(_CHUNK, max_points)
    # a group that needed more than one chunk last time (the engines pass its
    # previous count + 1 as _first_batch) gets its later tables started now
    ahead = min(max_points, (int(_first_batch) + _CHUNK // 2) // _CHUNK * _CHUNK + _CHUNK)
    for mm in range(2 * _CHUNK, ahead + 1, _CHUNK):
        for ci in coeffs:
            _dd_prefetch(l, ci * h, est, xi, mm)
    dds = _dd_group(l, [ci * h for ci in coeffs], est, xi, m_avail)
    table = _CoefTable(k)
    table.fill(0, min(_CHUNK, m_avail), dds, c, gamma, xi)

    fused = fused_target(J)
    if fused is not None and (fused[1] != 1.0 or fused[0].grid.problem == N.P_SEMILINEAR):
        fused = None
    Jn = fused[0] if fused else None
    nu, nu_dev = 0.0, None
    if Jn is not None and Jn.jac == N.JAC_FD:
        if Jn._nu is None and getattr(Jn, "_nu_state", None) is not None and D.COMM is None:
            nu_dev = Jn._nu_state  # ||u|| from the RHS pass: device copy, no host sync
        else:
            nu = Jn.nu

    slab = Jn is not None and Jn.comm is not None
    ps = [D.empty(n) for _ in range(k)]
    # fused single-GPU path: the begin pass only takes ||b|| and the m = 0
    # decisions; the first iteration writes p_i = d_i[0] b + d_i[1] y_1
    fold = Jn is not None and not slab and max_points > 1
    # deferred accumulation: large whole-grid calls (bandwidth-bound); the
    # iterate buffers of one chunk must fit the byte budget
    da = bool(fold and _DEFER[0] and n >= _DEFER[1]
              and k >= (_DEFER[4] if Jn.jac == N.JAC_FD else _DEFER[2])
              and min(_CHUNK, max_points) * n * 8 <= _DEFER[3])
    # graph mode: one graph launch covers the whole first chunk
    graph = fold and _FASTCALL and _GRAPH[0] and not da
    # (speculate only when the group's previous count fits the first chunk: a
    # call that crosses a chunk needs the host for its next table)
    spec = _spec is not None and fold and min(_CHUNK, max_points) > int(_first_batch)
    spec_zero = spec and _spec_zero and _lazy_m0 and isinstance(b, torch.Tensor)
    lazy = bool(_lazy_m0 and fold and (spec_zero or not spec) and isinstance(b, torch.Tensor))
    # whole-grid fused call without profiling: table upload, state init,
    # begin pass and the first launch batch in ONE native call
    fast = fold and PROFILE is None and _FASTCALL
    first_hi = m_avail if graph else min(m_avail, 1 + max(1, int(_first_batch)))
    st = D.DevState(N.LejaState, upload=not fast, tol=float(tol), nu=nu, k=k,
                    defer=1 if slab else 0, p_init=-1 if fold else 0, lazy0=1 if lazy else 0)
    nu_ptr = None if nu_dev is None else \
        C.c_void_p(nu_dev.buf.data_ptr() + N.ScalarState.val.offset + 8)
    ws = D.work_ptr(N.lib().ek_workspace_bytes(C.byref(Jn.grid)) if Jn else None)
    pp = N.ptrs(ps)
    ybuf = None
    # deferred accumulation: Y[j] = the iterate of table column j of the
    # current chunk (first chunk: Y[0] = b), yprev = the last iterate of the
    # previous chunk, pool = buffers free for reuse
    Y, yprev, pool = [bd] + [None] * (_CHUNK - 1), None, []

    def seq_buffers(m0, m1, base_):
        """Input / output buffers of iterations m0 .. m1-1 (chunk base base_)."""
        yin, yout = [], []
        for mm in range(m0, m1):
            j = mm - base_
            yin.append(Y[j - 1] if j >= 1 else yprev)
            Y[j] = pool.pop() if pool else D.empty(n)
            yout.append(Y[j])
        return N.ptrs(yin), N.ptrs(yout)

    def combine(base_, timed=True):
        """Form the sums over the current chunk's iterates (the freeze points
        are read from the state block on the device)."""
        ny = max(j for j in range(_CHUNK) if Y[j] is not None) + 1
        cev = None
        if timed and prof is not None:
            cev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            cev[0].record()
        N.check(N.lib().ek_leja_combine(
            n, N.ptrs(Y[:ny]), ny, pp, k, C.c_void_p(table.dev.data_ptr()), base_,
            1 if base_ > 0 else 0, st.ptr, D.stream()), "ek_leja_combine")
        if cev is not None:
            cev[1].record()
            prof["combine_events"].append(cev)

    if fast and da and not spec_zero:
        yin0, yout0 = seq_buffers(1, first_hi, 0)
        N.check(N.lib().ek_leja_call_seq(
            C.byref(Jn.grid), Jn.jac, C.c_void_p(Jn.u.data_ptr()), C.c_void_p(Jn.fu.data_ptr()),
            C.c_void_p(bd.data_ptr()), yin0, yout0, first_hi - 1, pp, k,
            table.host.ctypes.data_as(C.c_void_p), C.c_void_p(table.dev.data_ptr()), float(tol),
            nu, nu_ptr, 1 if lazy else 0, float(gamma), st.ptr, ws, D.stream()),
            "ek_leja_call_seq")
    elif fast:
        ybuf = None if spec_zero else [D.empty(n), D.empty(n)]
        N.check(N.lib().ek_leja_call(
            C.byref(Jn.grid), Jn.jac, C.c_void_p(Jn.u.data_ptr()), C.c_void_p(Jn.fu.data_ptr()),
            C.c_void_p(bd.data_ptr()), N.ptrs(ybuf or []), pp, k, table.host.ctypes.data_as(C.c_void_p),
            C.c_void_p(table.dev.data_ptr()), float(tol), nu, nu_ptr, 1, 1 if lazy else 0,
            1 if spec_zero else (-first_hi if graph else first_hi), float(gamma), st.ptr, ws,
            D.stream()), "ek_leja_call")
    else:
        table.upload()
        if nu_ptr is not None:
            N.check(N.lib().ek_copy(C.c_void_p(st.buf.data_ptr() + N.LejaState.nu.offset),
                                    nu_ptr, 8, 3, D.stream()), "nu copy")
        N.check(N.lib().ek_leja_begin_len(n, C.c_void_p(bd.data_ptr()), pp, k,
                                          C.c_void_p(table.dev.data_ptr()), st.ptr, ws,
                                          D.stream()), "ek_leja_begin_len")
    if slab:
        _slab_decide(st, Jn, table, 0, 0, k, begin=True)
    if Jn is None or max_points <= 1:
        # a generic action must not run (and charge) after termination
        hst = st.read()
        if hst.done:
            return LejaResult(vectors=[D.like_input(p, b) for p in ps], iters=0,
                              freeze_iters=[0] * k)
    # fused path: the first launch batch follows without a host round trip;
    # its kernels early-exit if everything froze at m = 0
    if spec_zero:
        def on_begin(hst):
            if hst.status != N.ST_OK or not hst.done or int(hst.iters) != 0:
                raise SpecMiss("phi-call predicted to stop at m = 0 did not")
            _spec(0, [0] * k, 0)
        D.defer_fn(st, on_begin)
        return LejaResult(vectors=[float(dds[i][0]) * D.V(bd) for i in range(k)],
                          iters=None, freeze_iters=None)

    if ybuf is None and not da:
        ybuf = [D.empty(n), D.empty(n)]
    yp = N.ptrs(ybuf or [])
    fd_seen = 0
    m = 1
    base = 0
    prof = None
    if PROFILE is not None and Jn is not None:
        prof = {"events": [], "k": k, "n": n, "fd": Jn.jac == N.JAC_FD, "deferred": da,
                "graph": bool(graph), "launches": [], "combine_events": []}
        PROFILE.append(prof)
    while m < max_points:
        if m >= m_avail:  # next 32-point chunk (leja.py:168-171)
            m_avail = min(m_avail + _CHUNK, max_points)
            for ci in coeffs:  # keep the pool one chunk ahead
                _dd_prefetch(l, ci * h, est, xi, min(m_avail + _CHUNK, max_points))
            dds = [_dd_cached(l, ci * h, est, xi, m_avail) for ci in coeffs]
            if da:  # fold the finished chunk into the sums before its table goes
                combine(base, timed=False)
                yprev = Y[m - 1 - base]
                pool.extend(y for j, y in enumerate(Y)
                            if y is not None and y is not yprev and y is not bd)
                Y = [None] * _CHUNK
            base = m
            table.load(base, m_avail, dds, c, gamma, xi)
        if Jn is not None:
            # launch batch: short first batch (most calls finish early), then
            # the rest of the chunk; kernels after termination early-exit
            hi = first_hi if m == 1 else m_avail
            if prof is not None:
                ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                ev[0].record()
            if prof is not None:
                prof["launches"].append(hi - m)
            if fast and m == 1:
                pass  # launched by ek_leja_call / ek_leja_call_seq
            elif da:
                yin_, yout_ = seq_buffers(m, hi, base)
                N.check(N.lib().ek_leja_run_seq(
                    C.byref(Jn.grid), Jn.jac, C.c_void_p(Jn.u.data_ptr()),
                    C.c_void_p(Jn.fu.data_ptr()), yin_, yout_, hi - m,
                    C.c_void_p(table.dev.data_ptr()), base, m, float(gamma), st.ptr, ws,
                    D.stream()), "ek_leja_run_seq")
            elif slab and Jn.comm.peer:
                # peer mode: ghost rows of b once (NCCL), then every pass
                # stores its boundary rows into the neighbours' windows and
                # a decide kernel waits for the pass flags: no host work
                win = Jn.comm.window(Jn.grid)
                N.check(N.lib().ek_leja_run_peer(
                    C.byref(Jn.grid), Jn.jac, C.c_void_p(Jn.u.data_ptr()),
                    C.c_void_p(Jn.fu.data_ptr()), C.c_void_p(bd.data_ptr()), yp, pp, k,
                    C.c_void_p(table.dev.data_ptr()), base, m, hi, float(gamma), st.ptr, ws,
                    Jn.halos(v=bd) if m == 1 else Jn.halos(), win.ptr,
                    C.c_void_p(win.local), win.take(hi - m), D.stream()), "ek_leja_run_peer")
            elif slab:
                # per iteration: ghost rows of y_{m-1}, local fused pass,
                # all-gather of the local sums, device decision (all ranks
                # reach the same one, so they stay in lockstep)
                for mm in range(m, hi):
                    yprev = bd if mm == 1 else ybuf[(mm - 1) & 1]
                    N.check(N.lib().ek_leja_run(
                        C.byref(Jn.grid), Jn.jac, C.c_void_p(Jn.u.data_ptr()),
                        C.c_void_p(Jn.fu.data_ptr()), C.c_void_p(bd.data_ptr()), yp, pp, k,
                        C.c_void_p(table.dev.data_ptr()), base, mm, mm + 1, float(gamma),
                        st.ptr, ws, Jn.halos(v=yprev), D.stream()), "ek_leja_run")
                    _slab_decide(st, Jn, table, base, mm, k, begin=False)
            elif graph:
                N.check(N.lib().ek_leja_run_graph(
                    C.byref(Jn.grid), Jn.jac, C.c_void_p(Jn.u.data_ptr()),
                    C.c_void_p(Jn.fu.data_ptr()), C.c_void_p(bd.data_ptr()), yp, pp, k,
                    C.c_void_p(table.dev.data_ptr()), base, m, hi, float(gamma), st.ptr,
                    ws, D.stream()), "ek_leja_run_graph")
            else:
                N.check(N.lib().ek_leja_run(
                    C.byref(Jn.grid), Jn.jac, C.c_void_p(Jn.u.data_ptr()),
                    C.c_void_p(Jn.fu.data_ptr()), C.c_void_p(bd.data_ptr()), yp, pp, k,
                    C.c_void_p(table.dev.data_ptr()), base, m, hi, float(gamma), st.ptr,
                    ws, None, D.stream()), "ek_leja_run")
            if prof is not None:
                ev[1].record()
                prof["events"].append(ev)
            if spec and da:
                combine(base)
            if spec:
                def on_state(hst, prof=prof):
                    if hst.status != N.ST_OK or not hst.done:
                        raise SpecMiss("phi-call did not finish in its launch batch")
                    iters = int(hst.iters)
                    freeze = [int(hst.freeze[i]) for i in range(k)]
                    if prof is not None:
                        prof["iters"], prof["freeze"] = iters, freeze
                    _spec(iters, freeze, int(hst.fd_evals) if Jn.jac == N.JAC_FD else 0)
                D.defer_fn(st, on_state)
                return LejaResult(vectors=ps, iters=None, freeze_iters=None)
            if hi == m_avail < max_points:
                # the next chunk's tables start in the
                # worker pool while this batch runs on the device
                for ci in coeffs:
                    _dd_prefetch(l, ci * h, est, xi, min(m_avail + _CHUNK, max_points))
            hst = st.read()
            if prof is not None:
                prof["iters"] = int(hst.m)
                prof["freeze"] = [int(hst.freeze[i]) if not (hst.active >> i) & 1
                                  else int(hst.m) for i in range(k)]
            if Jn.jac == N.JAC_FD:
                Jn.rhs.counter.charge(hst.fd_evals - fd_seen)
                fd_seen = hst.fd_evals
        else:
            # generic operator: its action runs elsewhere, one sync per step
            hi = m + 1
            y = bd if m == 1 else ybuf[(m - 1) & 1]
            jv = J.apply_dev(y)
            N.check(N.lib().ek_leja_update(
                n, C.c_void_p(jv.data_ptr()), C.c_void_p(y.data_ptr()),
                C.c_void_p(ybuf[m & 1].data_ptr()), pp, k,
                C.c_void_p(table.dev.data_ptr()), base, m, float(gamma), 0, st.ptr,
                ws, D.stream()), "ek_leja_update")
            hst = st.read()
        if hst.status == N.ST_JV_NONFINITE:
            raise FloatingPointError("non-finite Jacobian action")
        if hst.status == N.ST_NORM_NONFINITE:
            raise NonConvergence("polynomial iteration diverged", iters=int(hst.iters))
        if hst.status == N.ST_PEER_TIMEOUT:
            raise RuntimeError("peer mode: a rank's pass flag did not arrive (dead peer?)")
        if hst.done:
            if lazy and int(hst.iters) == 0:
                # everything froze at m = 0: ps[i] = dds[i][0] * y (leja.py:161)
                return LejaResult(vectors=[float(dds[i][0]) * D.V(bd) for i in range(k)],
                                  iters=0, freeze_iters=[0] * k)
            if da:
                combine(base)
            return LejaResult(vectors=[D.like_input(p, b) for p in ps],
                              iters=int(hst.iters),
                              freeze_iters=[int(hst.freeze[i]) for i in range(k)])
        m = hi

    stalled = [coeffs[i] for i in range(k) if (hst.active >> i) & 1]
    raise NonConvergence(
        f"no convergence in {max_points} Leja points",
        iters=max_points, detail={"stalled_coefficients": stalled})
