"""BASELINE.json plugins the reference does not define.

Kept in their own registry so the reference's pinned registries
(`problems.PROBLEMS`, `integrators.INTEGRATORS`, `make_problem`) stay
unchanged:

  problems   advdiff2d_problem            config 1: periodic upwind adv-diff 2-D
             allen_cahn_periodic_problem  config 2: periodic Allen-Cahn, noise IC
             burgers2d_problem            config 3: 2-D viscous Burgers, exact Jv
             brusselator_periodic_problem config 4: periodic 2-species Brusselator
             advdiff3d_problem            config 5: periodic upwind adv-diff 3-D
  steppers   exprb2   exponential Rosenbrock-Euler (no embedded pair)
             exprb32  u3 = a + 2 phi_3(dt J) R(a) dt, a = u + phi_1(dt J) f dt,
                      err = ||u3 - a||

The right-hand sides and ICs are defined in DESIGN.md §3; the NumPy
restatement used to pin them lives in oracle/np_fields.py.
"""

import math

import numpy as np

from . import _device as D
from . import _native as N
from .integrators import (INTEGRATOR_ORDER, StepResult, StepStats, _Engines,
                          _check_scheme, run_stepper, take_step)
from .problems import NativeJacFactory, Problem, StencilRhs, make_grid

X = D.V

EXT_PROBLEMS = ("advdiff2d", "allen_cahn_periodic", "burgers2d",
                "brusselator_periodic", "advdiff3d")
EXT_INTEGRATORS = ("exprb2", "exprb32")
EXT_ORDER = {"exprb2": 2, "exprb32": 3}
EXT_EMBEDDED_ORDER = {"exprb2": None, "exprb32": 2}


def _periodic_axis(n, length=1.0, lo=0.0):
    h = length / n
    return lo + h * np.arange(n), h


def advdiff2d_problem(n=64, D_=1.0, peclet=1.0, L=1.0):
    """u_t = D Lap u + v.grad u on the periodic unit square, upwind
    advection following the sign of +v.grad u, v = Pe D/L (1, 1). Linear,
    exact Jacobian = the same stencil."""
    x, h = _periodic_axis(n)
    vel = peclet * D_ / L
    X_, Y_ = np.meshgrid(x, x, indexing="ij")
    u0 = np.exp(-((X_ - 0.5)**2 + (Y_ - 0.5)**2) / 0.01).ravel()
    g = make_grid(N.P_ADVDIFF2D, N.BC_PERIODIC, 2, 1, n, h, (D_, vel, vel))
    rhs = StencilRhs("advdiff2d", g, analytic=True)
    dt_cfl = 1.0 / (4.0 * D_ / h**2 + (abs(vel) + abs(vel)) / h)
    return Problem("advdiff2d", rhs, u0, 1.0, n=n, jac_factory=NativeJacFactory(rhs),
                   params={"D": D_, "vx": vel, "vy": vel, "peclet": peclet,
                           "dt_cfl": dt_cfl})


def allen_cahn_periodic_problem(n=256, eps=1e-2, seed=0):
    """u_t = eps Lap u + u - u^3, periodic [-1,1)^2 (h = 2/n), IC
    0.1 * uniform(-1, 1) from default_rng(seed). FD Jacobian."""
    h = 2.0 / n
    u0 = 0.1 * np.random.default_rng(seed).uniform(-1.0, 1.0, n * n)
    g = make_grid(N.P_ALLEN_CAHN, N.BC_PERIODIC, 2, 1, n, h, (eps,))
    return Problem("allen_cahn_periodic", StencilRhs("allen_cahn_periodic", g), u0, 1.0,
                   n=n, params={"alpha": eps})


def _bump(x, c, w2):
    return np.exp(-(x - c)**2 / w2)


def burgers2d_problem(n=1024, eta=1e-2, seed=0):
    """u_t = eta Lap u + 1/2 d_x(u^2) + 1/2 d_y(u^2), periodic unit square,
    centred differences; exact Jv = eta Lap v + d_x(u v) + d_y(u v).
    IC: sin(2 pi x) sin(2 pi y) + 8 seeded separable Gaussian bumps."""
    x, h = _periodic_axis(n)
    rng = np.random.default_rng(seed)
    amps = rng.uniform(0.1, 0.5, 8)
    cen = rng.uniform(0.0, 1.0, (8, 2))
    s = np.sin(2.0 * np.pi * x)
    u = np.outer(s, s)
    w2 = 2.0 * 0.05**2
    for k in range(8):
        u = u + amps[k] * np.outer(_bump(x, cen[k, 0], w2), _bump(x, cen[k, 1], w2))
    g = make_grid(N.P_BURGERS2D, N.BC_PERIODIC, 2, 1, n, h, (eta,))
    rhs = StencilRhs("burgers2d", g, analytic=True)
    return Problem("burgers2d", rhs, u.ravel(), 1.0, n=n,
                   jac_factory=NativeJacFactory(rhs), params={"eta": eta})


def _smooth(rng, x, terms=4):
    kk = rng.integers(1, 5, size=(terms, 2))
    ph = rng.uniform(0.0, 2.0 * np.pi, size=(terms, 2))
    amp = rng.uniform(0.5, 1.0, size=terms)
    s = np.zeros((len(x), len(x)))
    for q in range(terms):
        s = s + amp[q] * np.outer(np.sin(2.0 * np.pi * kk[q, 0] * x + ph[q, 0]),
                                  np.sin(2.0 * np.pi * kk[q, 1] * x + ph[q, 1]))
    return s / terms


def brusselator_periodic_problem(n=4096, alpha=0.02, seed=0):
    """Standard-form Brusselator (u^2 w) with the periodic Laplacian on the
    unit square; IC = steady state (1, 3) + 0.05 * seeded smooth fields.
    FD Jacobian (the reference has no analytic Brusselator Jacobian)."""
    x, h = _periodic_axis(n)
    rng = np.random.default_rng(seed)
    su = _smooth(rng, x)
    sw = _smooth(rng, x)
    u0 = np.concatenate([(1.0 + 0.05 * su).ravel(), (3.0 + 0.05 * sw).ravel()])
    g = make_grid(N.P_BRUSS_STANDARD, N.BC_PERIODIC, 2, 2, n, h, (alpha,))
    return Problem("brusselator_periodic", StencilRhs("brusselator_periodic", g), u0, 1.0,
                   n=n, n_components=2, params={"alpha": alpha, "form": "standard"})


def advdiff3d_problem(n=512, D_=1.0, peclet=50.0, L=1.0, seed=0):
    """Periodic 3-D advection-diffusion, 7-point Laplacian + upwind,
    v = Pe D/L (1,1,1)/sqrt(3); IC = 6 seeded separable Gaussians. Linear."""
    x, h = _periodic_axis(n)
    vel = peclet * D_ / L / math.sqrt(3.0)
    rng = np.random.default_rng(seed)
    cen = rng.uniform(0.0, 1.0, (6, 3))
    u = np.zeros((n, n, n))
    for k in range(6):
        gx = _bump(x, cen[k, 0], 0.005)
        gy = _bump(x, cen[k, 1], 0.005)
        gz = _bump(x, cen[k, 2], 0.005)
        u = u + gx[:, None, None] * gy[None, :, None] * gz[None, None, :]
    g = make_grid(N.P_ADVDIFF3D, N.BC_PERIODIC, 3, 1, n, h, (D_, vel, vel, vel))
    rhs = StencilRhs("advdiff3d", g, analytic=True)
    dt_cfl = 1.0 / (6.0 * D_ / h**2 + 3.0 * abs(vel) / h)
    return Problem("advdiff3d", rhs, u.ravel(), 1.0, n=n,
                   jac_factory=NativeJacFactory(rhs),
                   params={"D": D_, "v": vel, "peclet": peclet, "dt_cfl": dt_cfl})


def make_ext_problem(name, **kw):
    makers = {"advdiff2d": advdiff2d_problem,
              "allen_cahn_periodic": allen_cahn_periodic_problem,
              "burgers2d": burgers2d_problem,
              "brusselator_periodic": brusselator_periodic_problem,
              "advdiff3d": advdiff3d_problem}
    if name not in makers:
        raise ValueError(f"unknown BASELINE problem '{name}'")
    return makers[name](**kw)


# ---------------------------------------------------------------- steppers

_NO_LEKRY = frozenset()


def step_exprb2(sys, dt, scheme, tol, ctx):
    """Exponential Rosenbrock-Euler u1 = u + phi_1(dt J) f dt (config 1).
    No embedded pair: err_est = 0 (use fixed steps)."""
    _check_scheme("exprb2", scheme, _NO_LEKRY)
    stats = StepStats()
    eng = _Engines(sys, ctx, tol, stats)
    u = sys._u
    fdt = D.ev(X(sys._f) * dt)
    if scheme == "leja":
        t1 = eng.leja_single("internal", fdt, 1, dt)
    else:
        t1 = eng.kiops_combo("internal", [None, fdt], dt)
    return StepResult(D.ev(X(u) + X(t1)), 0.0, stats, sys._as_numpy)


def step_exprb32(sys, dt, scheme, tol, ctx):
    """EXPRB32 (config 5): a = u + phi_1(dt J) f dt (2nd order),
    u3 = a + 2 phi_3(dt J) R(a) dt, err_est = ||u3 - a||."""
    _check_scheme("exprb32", scheme, _NO_LEKRY)
    stats = StepStats()
    eng = _Engines(sys, ctx, tol, stats)
    u = sys._u
    n = u.numel()
    fdt = D.ev(X(sys._f) * dt)
    if scheme == "leja":
        a, (_, (r2,)) = eng.stage_remainder(
            X(u) + X(eng.leja_single("internal", fdt, 1, dt)), keep=True,
            combos=[(None, 0.0, 2.0, dt)], store=False)  # (2 R(a)) dt
        t3 = eng.leja_single("stage3", r2, 3, dt)
    else:
        a, (_, (r2,)) = eng.stage_remainder(
            X(u) + X(eng.kiops_combo("internal", [None, fdt], dt)), keep=True,
            combos=[(None, 0.0, 2.0, dt)], store=False)
        t3 = eng.kiops_combo("stage3", [None, None, None, r2], dt)
    u3 = D.ev(X(a) + X(t3))
    err = D.evaluate([(X(u3) - X(a), None)], n, norm=True)[0]
    return StepResult(u3, err, stats, sys._as_numpy)


EXT_STEPPERS = {"exprb2": step_exprb2, "exprb32": step_exprb32}


def take_step_ext(name, sys, dt, scheme, tol, ctx):
    """take_step over the reference integrators plus EXPRB2 / EXPRB32."""
    if name in EXT_STEPPERS:
        if dt <= 0:
            raise ValueError("dt must be positive")
        return run_stepper(EXT_STEPPERS[name], sys, dt, scheme, tol, ctx)
    return take_step(name, sys, dt, scheme, tol, ctx)


def order_of(name):
    return EXT_ORDER.get(name, INTEGRATOR_ORDER.get(name))
