"""NumPy restatement of the PDE right-hand sides on the phi-action path.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Never imported by the
product package.

Part 1 restates the five reference problems of
`/root/reference/pkg/src/expkit/problems.py` with the reference's exact
elementwise evaluation order (SURVEY.md §8(a) "per-element evaluation
order"), so outputs are bit-identical to the reference on the same host.

Part 2 defines the BASELINE.json problems the reference does not have
(SURVEY.md Appendix A): periodic upwind advection-diffusion (2-D, 3-D),
periodic Allen-Cahn with a seeded noise IC, 2-D viscous Burgers with an
analytic Jacobian, and the periodic two-species Brusselator. Their RHS
definitions are this project's; the GPU kernels in
`paper_2211_08948_b200/csrc/stencils.cuh` follow the same op order.

A problem is returned as a `Spec` (fields mirror `problems.py:46-60`).
"""

import math
from dataclasses import dataclass, field

import numpy as np

MACH_EPS = float(np.finfo(np.float64).eps)  # linalg.py:18


@dataclass
class Spec:
    name: str
    rhs: object
    u0: np.ndarray
    t_final: float
    n: int
    n_components: int = 1
    extract: object = None
    exact: object = None
    params: dict = field(default_factory=dict)
    jac_factory: object = None
    dim: int = 2

    def __post_init__(self):
        if self.extract is None:
            self.extract = lambda u: u


# --------------------------------------------------------------- stencils


def _ring(f, mode):
    """Neighbour views (i-1, i+1, j-1, j+1) of a 2-D field with one ghost
    layer. mode 'reflect' mirrors without repeating the edge (Neumann,
    problems.py:27), 'wrap' is periodic (problems.py:41)."""
    g = np.pad(f, 1, mode=mode)
    return g[:-2, 1:-1], g[2:, 1:-1], g[1:-1, :-2], g[1:-1, 2:]


def five_point(f, h, mode):
    """((((f[i-1]+f[i+1])+f[j-1])+f[j+1]) - 4f) / h**2  (problems.py:26-29,
    40-43). `h**2` is evaluated as a Python float like the reference."""
    im, ip, jm, jp = _ring(f, mode)
    return (im + ip + jm + jp - 4.0 * f) / h**2


def centered_sum_grad(f, h, mode):
    """(f[i+1]-f[i-1])/(2h) + (f[j+1]-f[j-1])/(2h)  (problems.py:32-37)."""
    im, ip, jm, jp = _ring(f, mode)
    return (ip - im) / (2.0 * h) + (jp - jm) / (2.0 * h)


def _neumann_axis(n, lo, hi):
    # problems.py:63-66
    h = (hi - lo) / (n - 1)
    return lo + h * np.arange(n), h


# ------------------------------------------------- reference problem set


def adr(alpha, n, beta=-10.0, gamma=100.0):
    """problems.py:69-83 (Neumann, centered advection, cubic reaction)."""
    x, h = _neumann_axis(n, 0.0, 1.0)
    X, Y = np.meshgrid(x, x, indexing="ij")
    u0 = (256.0 * (X * Y * (1.0 - X) * (1.0 - Y))**2 + 0.3).ravel()

    def rhs(u):
        f = u.reshape(n, n)
        return (alpha * five_point(f, h, "reflect")
                + beta * centered_sum_grad(f, h, "reflect")
                + gamma * f * (1.0 - f) * (f - 0.5)).ravel()

    return Spec("adr", rhs, u0, 0.01, n,
                params={"alpha": alpha, "beta": beta, "gamma": gamma})


def allen_cahn(alpha, n):
    """problems.py:86-97 (Neumann on [-1,1]^2, cosine IC)."""
    x, h = _neumann_axis(n, -1.0, 1.0)
    X, Y = np.meshgrid(x, x, indexing="ij")
    u0 = (0.1 + 0.1 * np.cos(2.0 * np.pi * X) * np.cos(2.0 * np.pi * Y)).ravel()

    def rhs(u):
        f = u.reshape(n, n)
        return (alpha * five_point(f, h, "reflect") + f - f**3).ravel()

    return Spec("allen_cahn", rhs, u0, 1.0, n, params={"alpha": alpha})


def brusselator(alpha, n, form="printed"):
    """problems.py:100-124 (two species, component-major, Neumann)."""
    if form not in ("printed", "standard"):
        raise ValueError(f"unknown brusselator form '{form}'")
    x, h = _neumann_axis(n, 0.0, 1.0)
    X, Y = np.meshgrid(x, x, indexing="ij")
    u0 = np.concatenate([(2.0 + 0.25 * Y).ravel(), (1.0 + 0.8 * X).ravel()])
    nn = n * n

    def rhs(w):
        a = w[:nn].reshape(n, n)
        b = w[nn:].reshape(n, n)
        react = a * b**2 if form == "printed" else a**2 * b
        da = alpha * five_point(a, h, "reflect") + react - 4.0 * a + 1.0
        db = alpha * five_point(b, h, "reflect") - a**2 * b + 3.0 * a
        return np.concatenate([da.ravel(), db.ravel()])

    return Spec("brusselator", rhs, u0, 1.0, n, n_components=2,
                params={"alpha": alpha, "form": form})


def gray_scott(alpha, n, a=0.04, b=0.06):
    """problems.py:127-145 (periodic unit square)."""
    h = 1.0 / n
    x = h * np.arange(n)
    X, Y = np.meshgrid(x, x, indexing="ij")
    u0u = 1.0 - np.exp(-150.0 * ((X - 0.5)**2 + (Y - 0.5)**2))
    u0v = np.exp(-150.0 * ((X - 0.5)**2 + 2.0 * (Y - 0.5)**2))
    u0 = np.concatenate([u0u.ravel(), u0v.ravel()])
    nn = n * n

    def rhs(w):
        u = w[:nn].reshape(n, n)
        v = w[nn:].reshape(n, n)
        uvv = u * v**2
        du = alpha * five_point(u, h, "wrap") - uvv + a * (1.0 - u)
        dv = alpha * five_point(v, h, "wrap") + uvv - (a + b) * v
        return np.concatenate([du.ravel(), dv.ravel()])

    return Spec("gray_scott", rhs, u0, 0.1, n, n_components=2,
                params={"alpha": alpha, "a": a, "b": b})


def semilinear_forcing(x, t):
    """problems.py:148-151."""
    return np.exp(t) * (x * (1.0 - x) + 2.0 - 1.0 / 6.0)


def semilinear(n):
    """problems.py:154-196: 1-D Dirichlet, nonlocal trapezoid term with
    Euler-Maclaurin end correction, time carried as the last component,
    analytic Jacobian factory."""
    h = 1.0 / (n + 1)
    x = h * np.arange(1, n + 1)
    u0 = np.concatenate([x * (1.0 - x), [0.0]])

    def integral(u):
        corr = h / 24.0 * (4.0 * u[0] - u[1] + 4.0 * u[-1] - u[-2])
        return h * np.sum(u) + corr

    def d2(u):
        g = np.pad(u, 1)
        return (g[:-2] - 2.0 * u + g[2:]) / h**2

    def rhs(w):
        u, t = w[:-1], w[-1]
        return np.concatenate(
            [d2(u) + integral(u) + semilinear_forcing(x, t), [1.0]])

    def jac_factory(w_n):
        slope = semilinear_forcing(x, w_n[-1])

        def apply_fn(v):
            vu, vt = v[:-1], v[-1]
            return np.concatenate([d2(vu) + integral(vu) + slope * vt, [0.0]])
        return apply_fn

    return Spec("semilinear", rhs, u0, 1.0, n, extract=lambda w: w[:-1],
                exact=lambda t: x * (1.0 - x) * np.exp(t),
                jac_factory=jac_factory, dim=1)


def make(name, *, alpha=None, n=64, **kw):
    """problems.py:199-210 registry (reference defaults for alpha)."""
    if name == "adr":
        return adr(0.1 if alpha is None else alpha, n, **kw)
    if name == "allen_cahn":
        return allen_cahn(1e-2 if alpha is None else alpha, n, **kw)
    if name == "brusselator":
        return brusselator(1e-3 if alpha is None else alpha, n, **kw)
    if name == "gray_scott":
        return gray_scott(1e-3 if alpha is None else alpha, n, **kw)
    if name == "semilinear":
        return semilinear(n, **kw)
    raise ValueError(f"unknown problem '{name}'")


# ------------------------------------------- BASELINE plugin problems (ext)


def upwind_diff(f, h, vel, axis):
    """One-sided difference along `axis` following the sign of +v.grad(u):
    forward (f[+1]-f)/h for v >= 0, backward (f-f[-1])/h otherwise. Periodic."""
    if vel >= 0.0:
        return (np.roll(f, -1, axis=axis) - f) / h
    return (f - np.roll(f, 1, axis=axis)) / h


def _periodic_axis(n, lo=0.0, length=1.0):
    h = length / n
    return lo + h * np.arange(n), h


def advdiff2d(n=64, D=1.0, peclet=1.0, L=1.0):
    """Config 1: u_t = D Lap u + v.grad u, periodic [0,1)^2, upwind, linear.
    v = Pe*D/L*(1,1). Order: ((D*lap) + vx*dx) + vy*dy."""
    x, h = _periodic_axis(n)
    vel = peclet * D / L
    vx = vy = vel
    X, Y = np.meshgrid(x, x, indexing="ij")
    u0 = np.exp(-((X - 0.5)**2 + (Y - 0.5)**2) / 0.01).ravel()

    def rhs(u):
        f = u.reshape(n, n)
        out = (D * five_point(f, h, "wrap") + vx * upwind_diff(f, h, vx, 0)
               + vy * upwind_diff(f, h, vy, 1))
        return out.ravel()

    dt_cfl = 1.0 / (4.0 * D / h**2 + (abs(vx) + abs(vy)) / h)
    return Spec("advdiff2d", rhs, u0, 1.0, n, jac_factory=lambda u: rhs,
                params={"D": D, "vx": vx, "vy": vy, "peclet": peclet,
                        "dt_cfl": dt_cfl})


def allen_cahn_periodic(n=256, eps=1e-2, seed=0):
    """Config 2: u_t = eps Lap u + u - u^3, periodic [-1,1)^2 (h = 2/n, the
    reference's stiffness scale), IC 0.1*uniform(-1,1) from default_rng(seed)."""
    h = 2.0 / n
    u0 = 0.1 * np.random.default_rng(seed).uniform(-1.0, 1.0, n * n)

    def rhs(u):
        f = u.reshape(n, n)
        return (eps * five_point(f, h, "wrap") + f - f**3).ravel()

    return Spec("allen_cahn_periodic", rhs, u0, 1.0, n,
                params={"alpha": eps})


def _bumps_1d(x, c, width2):
    return np.exp(-(x - c)**2 / width2)


def burgers2d(n=1024, eta=1e-2, seed=0):
    """Config 3: u_t = eta Lap u + 1/2 d_x(u^2) + 1/2 d_y(u^2), periodic
    [0,1)^2, centered differences. Analytic Jv = eta Lap v + d_x(uv) + d_y(uv).
    IC: sin(2 pi x) sin(2 pi y) + sum_k a_k exp(-|x-x_k|^2/(2*0.05^2)) with
    a_k ~ U(0.1,0.5), x_k ~ U(0,1)^2 from default_rng(seed); the Gaussian is
    formed as a separable product."""
    x, h = _periodic_axis(n)
    rng = np.random.default_rng(seed)
    amps = rng.uniform(0.1, 0.5, 8)
    cen = rng.uniform(0.0, 1.0, (8, 2))
    sx = np.sin(2.0 * np.pi * x)
    u = np.outer(sx, sx)
    w2 = 2.0 * 0.05**2
    for k in range(8):
        u = u + amps[k] * np.outer(_bumps_1d(x, cen[k, 0], w2),
                                   _bumps_1d(x, cen[k, 1], w2))
    u0 = u.ravel()
    two_h = 2.0 * h

    def ddx_sum(g):
        im, ip, jm, jp = _ring(g, "wrap")
        return (ip - im) / two_h, (jp - jm) / two_h

    def rhs(w):
        f = w.reshape(n, n)
        gx, gy = ddx_sum(f * f)
        return (eta * five_point(f, h, "wrap") + 0.5 * gx + 0.5 * gy).ravel()

    def jac_factory(w_n):
        base = w_n.reshape(n, n)

        def apply_fn(v):
            g = v.reshape(n, n)
            gx, gy = ddx_sum(base * g)
            return (eta * five_point(g, h, "wrap") + gx + gy).ravel()
        return apply_fn

    return Spec("burgers2d", rhs, u0, 1.0, n, jac_factory=jac_factory,
                params={"eta": eta})


def _smooth_field(rng, x, terms=4):
    """Sum of `terms` random low-mode separable sines, scaled to |s| <= 1."""
    kk = rng.integers(1, 5, size=(terms, 2))
    ph = rng.uniform(0.0, 2.0 * np.pi, size=(terms, 2))
    amp = rng.uniform(0.5, 1.0, size=terms)
    s = np.zeros((len(x), len(x)))
    for q in range(terms):
        s = s + amp[q] * np.outer(np.sin(2.0 * np.pi * kk[q, 0] * x + ph[q, 0]),
                                  np.sin(2.0 * np.pi * kk[q, 1] * x + ph[q, 1]))
    return s / terms


def brusselator_periodic(n=4096, alpha=0.02, seed=0):
    """Config 4: standard-form two-species Brusselator (problems.py:104-107,
    118-120 op order) with the periodic Laplacian (problems.py:40-43) on
    [0,1)^2. IC: steady state (1, 3) + 0.05 * seeded smooth fields."""
    x, h = _periodic_axis(n)
    rng = np.random.default_rng(seed)
    su = _smooth_field(rng, x)
    sw = _smooth_field(rng, x)
    u0 = np.concatenate([(1.0 + 0.05 * su).ravel(), (3.0 + 0.05 * sw).ravel()])
    nn = n * n

    def rhs(w):
        a = w[:nn].reshape(n, n)
        b = w[nn:].reshape(n, n)
        da = alpha * five_point(a, h, "wrap") + a**2 * b - 4.0 * a + 1.0
        db = alpha * five_point(b, h, "wrap") - a**2 * b + 3.0 * a
        return np.concatenate([da.ravel(), db.ravel()])

    return Spec("brusselator_periodic", rhs, u0, 1.0, n, n_components=2,
                params={"alpha": alpha, "form": "standard"})


def seven_point(f, h):
    """Periodic 3-D Laplacian, neighbour order (i-1,i+1,j-1,j+1,k-1,k+1)."""
    s = (np.roll(f, 1, 0) + np.roll(f, -1, 0) + np.roll(f, 1, 1)
         + np.roll(f, -1, 1) + np.roll(f, 1, 2) + np.roll(f, -1, 2))
    return (s - 6.0 * f) / h**2


def advdiff3d(n=512, D=1.0, peclet=50.0, L=1.0, seed=0):
    """Config 5: periodic 3-D advection-diffusion, 7-point Laplacian plus
    upwind advection, v = Pe*D/L*(1,1,1)/sqrt(3). IC: sum of 6 separable
    Gaussians exp(-|x-x_k|^2/0.005), centres ~ U(0,1)^3 from default_rng(seed)."""
    x, h = _periodic_axis(n)
    vel = peclet * D / L / math.sqrt(3.0)
    rng = np.random.default_rng(seed)
    cen = rng.uniform(0.0, 1.0, (6, 3))
    u = np.zeros((n, n, n))
    for k in range(6):
        gx = _bumps_1d(x, cen[k, 0], 0.005)
        gy = _bumps_1d(x, cen[k, 1], 0.005)
        gz = _bumps_1d(x, cen[k, 2], 0.005)
        u = u + gx[:, None, None] * gy[None, :, None] * gz[None, None, :]
    u0 = u.ravel()

    def rhs(w):
        f = w.reshape(n, n, n)
        out = (D * seven_point(f, h) + vel * upwind_diff(f, h, vel, 0)
               + vel * upwind_diff(f, h, vel, 1)
               + vel * upwind_diff(f, h, vel, 2))
        return out.ravel()

    dt_cfl = 1.0 / (6.0 * D / h**2 + 3.0 * abs(vel) / h)
    return Spec("advdiff3d", rhs, u0, 1.0, n, jac_factory=lambda u: rhs,
                params={"D": D, "v": vel, "peclet": peclet, "dt_cfl": dt_cfl},
                dim=3)


# ------------------------------------------------------- Jacobian actions


def fd_jv(f, u, v, fu=None):
    """Forward-difference Jacobian action, linalg.py:111-129."""
    if u.shape != v.shape:
        raise ValueError("u and v must have equal length")
    nv = np.linalg.norm(v)
    if nv == 0.0:
        raise ValueError("degenerate direction: v = 0")
    eps = math.sqrt(MACH_EPS) * (1.0 + np.linalg.norm(u)) / nv
    if fu is None:
        fu = f(u)
    out = (f(u + eps * v) - fu) / eps
    if not np.all(np.isfinite(out)):
        raise FloatingPointError("non-finite Jacobian action")
    return out
