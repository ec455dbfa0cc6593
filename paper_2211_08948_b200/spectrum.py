"""Spectrum estimate for the Leja scaling (drop-in for `expkit.spectrum`,
spectrum.py:1-96).

`power_iterate` runs on the GPU. For a native stencil Jacobian the whole
iteration is device-resident: one fused Jacobian+norm kernel per iteration
and a device-side convergence test (`ek_power_run`), so the host only
synchronises every few iterations. The seeded PCG64 start vector is drawn
on the host once per (seed, dim) — exactly the reference's
`default_rng(seed).standard_normal(dim)` — and cached on the device.
"""

import ctypes as C
from dataclasses import dataclass, replace

import numpy as np

from . import _device as D
from . import _native as N
from .linalg import MatrixFreeOperator, fused_target

GAMMA_MIN = 1e-13


@dataclass(frozen=True)
class SpectrumEstimate:
    """Interval [alpha, beta], midpoint c, quarter-width gamma (spectrum.py:19-31)."""

    alpha: float
    beta: float
    c: float
    gamma: float
    safety: float
    age_steps: int = 0

    def aged(self):
        return replace(self, age_steps=self.age_steps + 1)


@dataclass(frozen=True)
class RefreshPolicy:
    """spectrum.py:34-40."""

    n_recompute: int = 50
    safety: float = 1.1
    tol_pi: float = 1e-2
    max_it: int = 1000
    seed: int = 0


_START = {}


def _start_vector(seed, dim):
    key = (seed, dim, D.device().index)
    v = _START.get(key)
    if v is None:
        host = np.random.default_rng(seed).standard_normal(dim)
        v = D.to_dev(host)
        if len(_START) > 8:
            _START.clear()
        _START[key] = v
    return v


# iterations launched per host sync on the fused path
_POWER_BATCH = 8


def power_iterate(J: MatrixFreeOperator, tol_pi=1e-2, max_it=1000, seed=0):
    """Dominant |lambda| of J by power iteration (spectrum.py:43-63).
    Returns (estimate, converged)."""
    if max_it <= 0:  # the reference's loop body never runs (spectrum.py:53-63)
        return 0.0, False
    fused = fused_target(J)
    if fused is not None and fused[0].comm is not None:
        # slab mode: this rank's rows of the global seeded start vector
        sten = fused[0].stencil
        key = (seed, "slab", sten.comm.rank, int(sten.grid.row0), J.dim)
        v0 = _START.get(key)
        if v0 is None:
            glen = int(N.lib().ek_grid_len(C.byref(sten.global_grid)))
            host = np.random.default_rng(seed).standard_normal(glen)
            v0 = D.to_dev(sten.comm.scatter(host, sten.global_grid))
            _START[key] = v0
    else:
        v0 = _start_vector(seed, J.dim)
    if fused is not None and fused[1] == 1.0 and fused[0].grid.problem != N.P_SEMILINEAR:
        return _power_fused(fused[0], v0, tol_pi, max_it)
    # generic operator: the action runs per iteration on the host's request
    nv0 = D.norm2(v0)[0]
    v = D.ev(D.V(v0) / nv0)
    lam = 0.0
    for _ in range(max_it):
        w = J.apply_dev(v)
        nw = D.norm2(w)[0]
        if nw == 0.0:
            return 0.0, True
        v = D.ev(D.V(w) / nw)
        if abs(nw - lam) <= tol_pi * nw:
            return float(nw), True
        lam = nw
    return float(lam), False


def _part(st):
    fld = type(st.host).part
    return st.buf[fld.offset:fld.offset + fld.size].view(D.F64)


def _slab_decide(st, J, which):
    g = J.comm.allgather_pairs(_part(st))
    N.check(N.lib().ek_power_decide(st.ptr, C.c_void_p(g.data_ptr()), J.comm.world,
                                    1 if J.jac == N.JAC_FD else 0, which, D.stream()),
            "ek_power_decide")


def _slab_norm(st, J, x, scaled, ws):
    N.check(N.lib().ek_power_norm(x.numel(), C.c_void_p(x.data_ptr()), scaled, st.ptr, ws,
                                  D.stream()), "ek_power_norm")
    _slab_decide(st, J, 2 if scaled else 1)


def _power_fused(J, v0, tol_pi, max_it):
    slab = J.comm is not None
    st = D.DevState(N.PowerState, lam=0.0, nu=J.nu, tol_pi=tol_pi, max_it=max_it,
                    defer=1 if slab else 0)
    wbuf = [D.empty(J.dim), D.empty(J.dim)]
    wp = N.ptrs(wbuf)
    ws = D.work_ptr(N.lib().ek_workspace_bytes(C.byref(J.grid)))
    it = 0
    h = None
    fd_seen = 0
    fd = J.jac == N.JAC_FD
    if slab:
        # v = v0 / ||v0|| with the global norm (and ||v|| for the FD increment)
        _slab_norm(st, J, v0, 0, ws)
        if fd:
            _slab_norm(st, J, v0, 1, ws)
    while it < max_it:
        hi = min(max_it, it + (_POWER_BATCH if it else 4))
        if slab:
            for i in range(it, hi):
                vin = v0 if i == 0 else wbuf[(i - 1) & 1]
                N.check(N.lib().ek_power_run(
                    C.byref(J.grid), J.jac, C.c_void_p(J.u.data_ptr()),
                    C.c_void_p(J.fu.data_ptr()), C.c_void_p(v0.data_ptr()), wp, i, i + 1,
                    st.ptr, ws, J.halos(v=vin), D.stream()), "ek_power_run")
                _slab_decide(st, J, 0)
                if fd:
                    _slab_norm(st, J, wbuf[i & 1], 1, ws)
        else:
            N.check(N.lib().ek_power_run(
                C.byref(J.grid), J.jac, C.c_void_p(J.u.data_ptr()),
                C.c_void_p(J.fu.data_ptr()), C.c_void_p(v0.data_ptr()), wp, it, hi,
                st.ptr, ws, None, D.stream()), "ek_power_run")
        h = st.read()
        if J.jac == N.JAC_FD:
            J.rhs.counter.charge(h.fd_evals - fd_seen)
            fd_seen = h.fd_evals
        if h.status == N.ST_JV_NONFINITE:
            raise FloatingPointError("non-finite Jacobian action")
        if h.done:
            break
        it = hi
    return float(h.lam), bool(h.converged)


def make_estimate(lam, safety=1.1):
    """alpha = -safety |lam|, beta = 0 (spectrum.py:66-78)."""
    if not np.isfinite(lam):
        raise ValueError("non-finite eigenvalue estimate")
    alpha = -safety * abs(lam)
    beta = 0.0
    c = (alpha + beta) / 2.0
    gamma = max(abs(beta - alpha) / 4.0, GAMMA_MIN)
    return SpectrumEstimate(alpha=alpha, beta=beta, c=c, gamma=gamma,
                            safety=safety, age_steps=0)


def maybe_refresh(est: SpectrumEstimate, J: MatrixFreeOperator,
                  policy: RefreshPolicy, force=False):
    """Re-run the power iteration when stale or forced (spectrum.py:81-96)."""
    if force or est is None or est.age_steps >= policy.n_recompute:
        lam, converged = power_iterate(J, tol_pi=policy.tol_pi,
                                       max_it=policy.max_it, seed=policy.seed)
        base = est.safety if est is not None else policy.safety
        safety = base if converged else base * 1.5
        return make_estimate(lam, safety=safety)
    return est.aged()
