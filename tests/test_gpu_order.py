"""Pinning of the BASELINE plugin right-hand sides.

The five BASELINE problems (advdiff2d, allen_cahn_periodic, burgers2d,
brusselator_periodic, advdiff3d) do not exist in the reference, so no
reference test pins their definitions. These tests pin them on the device
kernels against analytic fields, the way the reference pins its own
stencils (/root/reference/pkg/tests/test_problems.py:37-53 second order of
the ADR stencils on cos*cos; :145-165 periodic Laplacian second order and
the null space of constant fields):

* every periodic Laplacian (2-D 5-point, 3-D 7-point) is second order;
* the centred Burgers flux 1/2 d(u^2) and its exact Jacobian action
  d(u v) are second order;
* the upwind advection is first order, and its leading error is the
  numerical diffusion (h/2) sum_a |v_a| d_aa u for either sign of v_a —
  i.e. the one-sided difference follows the sign of +v.grad u (forward
  difference for v_a > 0). The wrong direction would give the opposite
  sign (anti-diffusion);
* constant fields are in the null space of the transport operators.
"""

import math

import numpy as np
import pytest

from paper_2211_08948_b200 import _native as N, ext
from paper_2211_08948_b200.problems import NativeJacFactory, StencilRhs, make_grid

pytestmark = pytest.mark.gpu

TWO_PI = 2.0 * math.pi


def _field2(n, lo=0.0, L=1.0):
    """Smooth periodic test field on [lo, lo+L)^2 with its derivatives."""
    h = L / n
    x = lo + h * np.arange(n)
    X, Y = np.meshgrid(x, x, indexing="ij")
    k = TWO_PI / L
    a, b = k * (X - lo), k * (Y - lo)
    u = np.sin(a) * np.cos(2 * b) + 0.5 * np.cos(a + b) + 0.2
    ux = k * np.cos(a) * np.cos(2 * b) - 0.5 * k * np.sin(a + b)
    uy = -2 * k * np.sin(a) * np.sin(2 * b) - 0.5 * k * np.sin(a + b)
    uxx = -k * k * np.sin(a) * np.cos(2 * b) - 0.5 * k * k * np.cos(a + b)
    uyy = -4 * k * k * np.sin(a) * np.cos(2 * b) - 0.5 * k * k * np.cos(a + b)
    return h, dict(u=u, ux=ux, uy=uy, uxx=uxx, uyy=uyy)


def _field3(n):
    h = 1.0 / n
    x = h * np.arange(n)
    X, Y, Z = np.meshgrid(x, x, x, indexing="ij")
    a, b, c = TWO_PI * X, TWO_PI * Y, TWO_PI * Z
    k = TWO_PI
    u = np.sin(a) * np.cos(b) * np.sin(2 * c) + 0.3 * np.cos(a + 2 * b) + 0.1
    ux = k * np.cos(a) * np.cos(b) * np.sin(2 * c) - 0.3 * k * np.sin(a + 2 * b)
    uy = -k * np.sin(a) * np.sin(b) * np.sin(2 * c) - 0.6 * k * np.sin(a + 2 * b)
    uz = 2 * k * np.sin(a) * np.cos(b) * np.cos(2 * c)
    uxx = -k * k * np.sin(a) * np.cos(b) * np.sin(2 * c) - 0.3 * k * k * np.cos(a + 2 * b)
    uyy = -k * k * np.sin(a) * np.cos(b) * np.sin(2 * c) - 1.2 * k * k * np.cos(a + 2 * b)
    uzz = -4 * k * k * np.sin(a) * np.cos(b) * np.sin(2 * c)
    return h, dict(u=u, ux=ux, uy=uy, uz=uz, uxx=uxx, uyy=uyy, uzz=uzz)


def _advdiff2(n, D_, vx, vy):
    h = 1.0 / n
    g = make_grid(N.P_ADVDIFF2D, N.BC_PERIODIC, 2, 1, n, h, (D_, vx, vy))
    return StencilRhs("advdiff2d", g, analytic=True)


def _advdiff3(n, D_, vx, vy, vz):
    h = 1.0 / n
    g = make_grid(N.P_ADVDIFF3D, N.BC_PERIODIC, 3, 1, n, h, (D_, vx, vy, vz))
    return StencilRhs("advdiff3d", g, analytic=True)


def _ratio(errs):
    return [errs[i] / errs[i + 1] for i in range(len(errs) - 1)]


# ------------------------------------------------------------ Laplacians

def test_advdiff2d_laplacian_second_order():
    errs = []
    for n in (32, 64, 128):
        h, f = _field2(n)
        got = _advdiff2(n, 1.0, 0.0, 0.0)(f["u"].ravel()).reshape(n, n)
        errs.append(np.max(np.abs(got - (f["uxx"] + f["uyy"]))))
    for r in _ratio(errs):
        assert 3.6 <= r <= 4.4, errs


def test_advdiff3d_laplacian_second_order():
    errs = []
    for n in (16, 32, 64):
        h, f = _field3(n)
        got = _advdiff3(n, 1.0, 0.0, 0.0, 0.0)(f["u"].ravel()).reshape(n, n, n)
        errs.append(np.max(np.abs(got - (f["uxx"] + f["uyy"] + f["uzz"]))))
    for r in _ratio(errs):
        assert 3.6 <= r <= 4.4, errs


def test_allen_cahn_periodic_second_order():
    """eps Lap u + u - u^3 on the periodic [-1, 1)^2 grid of config 2
    (h = 2/n); the pointwise reaction is exact up to rounding."""
    eps = 1e-2
    errs = []
    for n in (32, 64, 128):
        p = ext.allen_cahn_periodic_problem(n=n, eps=eps)
        h, f = _field2(n, lo=-1.0, L=2.0)
        assert p.rhs.grid.h == h
        u = f["u"]
        got = p.rhs(u.ravel()).reshape(n, n)
        exact = eps * (f["uxx"] + f["uyy"]) + u - u**3
        errs.append(np.max(np.abs(got - exact)))
    for r in _ratio(errs):
        assert 3.6 <= r <= 4.4, errs


def test_brusselator_periodic_second_order():
    """Standard-form Brusselator: alpha Lap u + 1 - 4u + u^2 w,
    alpha Lap w + 3u - u^2 w (problems.py:118-120 form 'standard')."""
    alpha = 0.02
    errs = []
    for n in (32, 64, 128):
        p = ext.brusselator_periodic_problem(n=n, alpha=alpha)
        h, fu = _field2(n)
        u = 1.0 + 0.1 * fu["u"]
        w = 3.0 - 0.2 * fu["u"].T
        lu = 0.1 * (fu["uxx"] + fu["uyy"])
        lw = -0.2 * (fu["uxx"] + fu["uyy"]).T   # Laplacian of the transpose
        got = p.rhs(np.concatenate([u.ravel(), w.ravel()]))
        ex_u = alpha * lu + 1.0 - 4.0 * u + u * u * w
        ex_w = alpha * lw + 3.0 * u - u * u * w
        err = max(np.max(np.abs(got[:n * n].reshape(n, n) - ex_u)),
                  np.max(np.abs(got[n * n:].reshape(n, n) - ex_w)))
        errs.append(err)
    for r in _ratio(errs):
        assert 3.6 <= r <= 4.4, errs


# ------------------------------------------------------------ Burgers

def test_burgers2d_centred_flux_and_jacobian_second_order():
    eta = 1e-2
    errs_f, errs_j = [], []
    for n in (32, 64, 128):
        p = ext.burgers2d_problem(n=n, eta=eta)
        h, f = _field2(n)
        u = f["u"]
        got = p.rhs(u.ravel()).reshape(n, n)
        exact = eta * (f["uxx"] + f["uyy"]) + u * f["ux"] + u * f["uy"]
        errs_f.append(np.max(np.abs(got - exact)))
        # exact Jacobian action J(u) v = eta Lap v + d_x(u v) + d_y(u v)
        _, g = _field2(n)
        v = np.cos(TWO_PI * np.arange(n) / n)[:, None] * np.ones((1, n))
        vx = -TWO_PI * np.sin(TWO_PI * np.arange(n) / n)[:, None] * np.ones((1, n))
        vxx = -(TWO_PI ** 2) * v
        jv = NativeJacFactory(p.rhs)(u.ravel())(v.ravel()).reshape(n, n)
        jex = eta * vxx + (f["ux"] * v + u * vx) + (f["uy"] * v)
        errs_j.append(np.max(np.abs(jv - jex)))
    for r in _ratio(errs_f) + _ratio(errs_j):
        assert 3.6 <= r <= 4.4, (errs_f, errs_j)


# ------------------------------------------------------------ upwind

@pytest.mark.parametrize("vx,vy", [(1.5, 0.7), (-1.5, 0.7), (1.5, -0.7), (-1.5, -0.7)])
def test_advdiff2d_upwind_first_order_follows_velocity(vx, vy):
    errs, lead = [], []
    for n in (64, 128, 256):
        h, f = _field2(n)
        got = _advdiff2(n, 0.0, vx, vy)(f["u"].ravel()).reshape(n, n)
        err = got - (vx * f["ux"] + vy * f["uy"])
        errs.append(np.max(np.abs(err)))
        # leading term of a one-sided difference in the upwind direction of
        # +v.grad u: + (h/2) |v| u'' per axis (numerical diffusion)
        pred = 0.5 * h * (abs(vx) * f["uxx"] + abs(vy) * f["uyy"])
        lead.append(np.max(np.abs(err - pred)) / np.max(np.abs(pred)))
    for r in _ratio(errs):
        assert 1.8 <= r <= 2.2, errs
    assert lead[-1] <= 0.1, lead                     # the error IS the upwind term
    assert lead[-1] < lead[0] * 0.6, lead            # and the rest is higher order


@pytest.mark.parametrize("v", [(1.0, 0.6, 0.3), (-1.0, 0.6, -0.3), (-1.0, -0.6, -0.3)])
def test_advdiff3d_upwind_first_order_follows_velocity(v):
    """(+, +, +) runs the select-free instantiation (PAdvDiff3T<true>), the
    mixed signs the general one."""
    vx, vy, vz = v
    errs, lead = [], []
    for n in (32, 64, 128):
        h, f = _field3(n)
        got = _advdiff3(n, 0.0, vx, vy, vz)(f["u"].ravel()).reshape(n, n, n)
        err = got - (vx * f["ux"] + vy * f["uy"] + vz * f["uz"])
        errs.append(np.max(np.abs(err)))
        pred = 0.5 * h * (abs(vx) * f["uxx"] + abs(vy) * f["uyy"] + abs(vz) * f["uzz"])
        lead.append(np.max(np.abs(err - pred)) / np.max(np.abs(pred)))
    for r in _ratio(errs):
        assert 1.75 <= r <= 2.25, errs
    assert lead[-1] <= 0.12, lead
    assert lead[-1] < lead[0] * 0.6, lead


def test_advdiff_full_operator_matches_sum_of_parts():
    """D Lap + v.grad with both parts on: the kernel's value is the sum of
    the diffusion-only and advection-only values up to rounding."""
    n = 64
    h, f = _field2(n)
    u = f["u"].ravel()
    full = _advdiff2(n, 1.0, 2.0, -3.0)(u)
    parts = _advdiff2(n, 1.0, 0.0, 0.0)(u) + _advdiff2(n, 0.0, 2.0, -3.0)(u)
    assert np.max(np.abs(full - parts)) <= 1e-12 * np.max(np.abs(full))


# ------------------------------------------------------------ null space

@pytest.mark.parametrize("c", [0.75, -1.25, 0.7])
def test_constant_fields_in_null_space(c):
    n = 32
    u2 = np.full(n * n, c)
    u3 = np.full(n ** 3, c)
    # the upwind differences of a constant are exactly 0; the Laplacian's
    # neighbour sum of a non-dyadic constant can round by an ulp, which
    # 1/h^2 scales: the bound is that rounding, nothing more
    tol = 8.0 * np.finfo(float).eps * abs(c) * n * n
    for rhs in (_advdiff2(n, 1.0, 2.0, -3.0), _advdiff2(n, 1.0, 5.0, 5.0)):
        assert np.max(np.abs(rhs(u2))) <= tol
        assert not np.any(_advdiff2(n, 0.0, 2.0, -3.0)(u2))
    for rhs in (_advdiff3(n, 1.0, 1.0, -2.0, 3.0), _advdiff3(n, 1.0, 1.0, 2.0, 3.0)):
        assert np.max(np.abs(rhs(u3))) <= tol
    assert not np.any(_advdiff3(n, 0.0, 1.0, -2.0, 3.0)(u3))
    assert not np.any(_advdiff3(n, 0.0, 1.0, 2.0, 3.0)(u3))
    # Burgers: transport of a constant is zero; its Jacobian maps constants
    # to zero as well (d(c v) of a constant v)
    pb = ext.burgers2d_problem(n=n)
    assert np.allclose(pb.rhs(u2), 0.0, atol=1e-15)
    assert np.allclose(NativeJacFactory(pb.rhs)(u2)(np.ones(n * n)), 0.0, atol=1e-15)
    # reaction problems: only the pointwise reaction survives
    pa = ext.allen_cahn_periodic_problem(n=n)
    assert np.allclose(pa.rhs(u2), c - c ** 3, atol=1e-15)
    pr = ext.brusselator_periodic_problem(n=n)
    w = 2.0
    got = pr.rhs(np.concatenate([u2, np.full(n * n, w)]))
    assert np.allclose(got[:n * n], 1.0 - 4.0 * c + c * c * w, atol=1e-15)
    assert np.allclose(got[n * n:], 3.0 * c - c * c * w, atol=1e-15)
    if c == 0.75:  # dyadic constant: the stencil sums are exact, so are the zeros
        assert not np.any(_advdiff2(n, 1.0, 2.0, -3.0)(u2))
        assert not np.any(_advdiff3(n, 1.0, 1.0, 2.0, 3.0)(u3))
