"""Benchmark PDE problems with GPU stencil right-hand sides.

Drop-in for `expkit.problems` (problems.py:1-210): the same registry,
constructors, initial conditions and `Problem` fields. The difference is
`Problem.rhs`: a `StencilRhs` that evaluates the discretised right-hand side
with the fp64 sm_100a stencil kernels of libexpkit_sm100.so (NumPy array in
-> NumPy array out; CUDA tensor in -> CUDA tensor out). The engines detect
it and fuse the Jacobian action into their iteration kernels.

Initial conditions are set-up data, built on the host with the reference's
own NumPy expressions (bit-identical).
"""

import ctypes as C

import numpy as np

from . import _device as D
from . import _native as N

PROBLEMS = ("adr", "allen_cahn", "brusselator", "gray_scott", "semilinear")

GS_A = 0.04
GS_B = 0.06


def make_grid(problem, bc, dim, ncomp, n, h, prm=()):
    """ek_grid for a single-GPU problem. h2 = h**2 and two_h = 2.0*h are
    evaluated in Python exactly as the reference's stencils do."""
    g = N.Grid()
    g.problem, g.bc, g.dim, g.ncomp = problem, bc, dim, ncomp
    g.n, g.rows, g.row0, g.slab = n, n, 0, 0
    g.h, g.h2, g.two_h = h, h**2, 2.0 * h
    for i, v in enumerate(prm):
        g.prm[i] = float(v)
    return g


class StencilRhs:
    """du/dt = f(u) evaluated by the native stencil kernel (`ek_rhs`)."""

    def __init__(self, name, grid, analytic=False):
        self.name = name
        self.grid = grid
        self.analytic = analytic
        self.comm = None          # slab.SlabComm when this is a rank's slab
        self.global_grid = None
        self.length = int(N.lib().ek_grid_len(C.byref(grid))) if N.lib_path().exists() \
            else None

    def halo(self, x):
        """Ghost rows of the local field x (slab mode): flat device buffer."""
        from .slab import halo_buffer
        return self.comm.exchange(x, self.grid, halo_buffer(self.grid))

    def __call__(self, u):
        ud = D.to_dev(u)
        if self.length is None:
            self.length = int(N.lib().ek_grid_len(C.byref(self.grid)))
        if ud.numel() != self.length:
            raise ValueError(f"{self.name}: state length {ud.numel()} != {self.length}")
        out = D.empty(self.length)
        halo = None
        if self.comm is not None:
            hb = self.halo(ud)
            halo = N.ptrs([hb, None, None])
        N.check(N.lib().ek_rhs(C.byref(self.grid), C.c_void_p(ud.data_ptr()),
                               C.c_void_p(out.data_ptr()), halo, D.stream()), "ek_rhs")
        return D.like_input(out, u)

    def eval_with_norm(self, ud):
        """(f(u), state block holding ||u||^2 of the local slab) in one pass
        (ek_rhs_norm); device in, device out. Not charged: the caller
        charges its counter."""
        if ud.numel() != self.length:
            raise ValueError(f"{self.name}: state length {ud.numel()} != {self.length}")
        out = D.empty(self.length)
        halo = None
        if self.comm is not None:
            hb = self.halo(ud)
            halo = N.ptrs([hb, None, None])
        st = D.scalar_state()
        N.check(N.lib().ek_rhs_norm(C.byref(self.grid), C.c_void_p(ud.data_ptr()),
                                    C.c_void_p(out.data_ptr()), st.ptr,
                                    D.work_ptr(N.lib().ek_workspace_bytes(C.byref(self.grid))),
                                    halo, D.stream()), "ek_rhs_norm")
        return out, st


class NativeJacFactory:
    """`jac_factory` of a problem with an exact Jacobian stencil: called with
    the linearisation point it returns the action v -> J(u) v on the GPU
    (problems.py:177-189 for the semilinear problem)."""

    def __init__(self, stencil):
        self.stencil = stencil

    def __call__(self, u):
        ud = D.to_dev(u, copy=True)
        grid = self.stencil.grid

        def apply_fn(v):
            vd = D.to_dev(v)
            out = D.empty(vd.numel())
            N.check(N.lib().ek_jv(C.byref(grid), N.JAC_ANALYTIC, C.c_void_p(ud.data_ptr()),
                                  None, C.c_void_p(vd.data_ptr()), 0.0,
                                  C.c_void_p(out.data_ptr()), None, None, None,
                                  D.stream()), "ek_jv")
            return D.like_input(out, v)
        apply_fn.native_factory = self
        apply_fn.u = ud
        return apply_fn


class Problem:
    """A discretised initial-value problem du/dt = rhs(u) (problems.py:46-60)."""

    def __init__(self, name, rhs, u0, t_final, *, n, n_components=1,
                 extract=None, exact=None, params=None, jac_factory=None):
        self.name = name
        self.rhs = rhs
        self.u0 = u0
        self.t_final = t_final
        self.n = n
        self.n_components = n_components
        self.extract = extract if extract is not None else (lambda u: u)
        self.exact = exact
        self.params = dict(params or {})
        self.jac_factory = jac_factory


def _node_axis(n, lo, hi):
    """Neumann node-centred axis, h = (hi-lo)/(n-1) (problems.py:63-66)."""
    h = (hi - lo) / (n - 1)
    return lo + h * np.arange(n), h


def adr_problem(alpha, n, beta=-10.0, gamma=100.0):
    """u_t = alpha Lap u + beta (u_x + u_y) + gamma u (1-u)(u-1/2), [0,1]^2,
    homogeneous Neumann (problems.py:69-83)."""
    x, h = _node_axis(n, 0.0, 1.0)
    X, Y = np.meshgrid(x, x, indexing="ij")
    u0 = (256.0 * (X * Y * (1.0 - X) * (1.0 - Y))**2 + 0.3).ravel()
    g = make_grid(N.P_ADR, N.BC_NEUMANN, 2, 1, n, h, (alpha, beta, gamma))
    return Problem("adr", StencilRhs("adr", g), u0, 0.01, n=n,
                   params={"alpha": alpha, "beta": beta, "gamma": gamma})


def allen_cahn_problem(alpha, n):
    """u_t = alpha Lap u + u - u^3 on [-1,1]^2, Neumann (problems.py:86-97)."""
    x, h = _node_axis(n, -1.0, 1.0)
    X, Y = np.meshgrid(x, x, indexing="ij")
    u0 = (0.1 + 0.1 * np.cos(2.0 * np.pi * X) * np.cos(2.0 * np.pi * Y)).ravel()
    g = make_grid(N.P_ALLEN_CAHN, N.BC_NEUMANN, 2, 1, n, h, (alpha,))
    return Problem("allen_cahn", StencilRhs("allen_cahn", g), u0, 1.0, n=n,
                   params={"alpha": alpha})


def brusselator_problem(alpha, n, form="printed"):
    """Two-species Brusselator on [0,1]^2, Neumann (problems.py:100-124).
    form="printed": react = u v^2; form="standard": react = u^2 v."""
    if form not in ("printed", "standard"):
        raise ValueError(f"unknown brusselator form '{form}'")
    x, h = _node_axis(n, 0.0, 1.0)
    X, Y = np.meshgrid(x, x, indexing="ij")
    u0 = np.concatenate([(2.0 + 0.25 * Y).ravel(), (1.0 + 0.8 * X).ravel()])
    pid = N.P_BRUSS_PRINTED if form == "printed" else N.P_BRUSS_STANDARD
    g = make_grid(pid, N.BC_NEUMANN, 2, 2, n, h, (alpha,))
    return Problem("brusselator", StencilRhs("brusselator", g), u0, 1.0, n=n,
                   n_components=2, params={"alpha": alpha, "form": form})


def gray_scott_problem(alpha, n, a=GS_A, b=GS_B):
    """Gray-Scott on the periodic unit square (problems.py:127-145)."""
    h = 1.0 / n
    x = h * np.arange(n)
    X, Y = np.meshgrid(x, x, indexing="ij")
    u0u = 1.0 - np.exp(-150.0 * ((X - 0.5)**2 + (Y - 0.5)**2))
    u0v = np.exp(-150.0 * ((X - 0.5)**2 + 2.0 * (Y - 0.5)**2))
    u0 = np.concatenate([u0u.ravel(), u0v.ravel()])
    g = make_grid(N.P_GRAY_SCOTT, N.BC_PERIODIC, 2, 2, n, h, (alpha, a, a + b))
    return Problem("gray_scott", StencilRhs("gray_scott", g), u0, 0.1, n=n,
                   n_components=2, params={"alpha": alpha, "a": a, "b": b})


def semilinear_forcing(x, t):
    """Forcing with exact solution u = x(1-x)e^t (problems.py:148-151).
    Host formula helper (scalars / small arrays)."""
    return np.exp(t) * (x * (1.0 - x) + 2.0 - 1.0 / 6.0)


def semilinear_problem(n):
    """1-D semilinear parabolic problem, Dirichlet, nonlocal integral term,
    time as the last state component, exact Jacobian (problems.py:154-196)."""
    h = 1.0 / (n + 1)
    x = h * np.arange(1, n + 1)
    u0 = np.concatenate([x * (1.0 - x), [0.0]])
    g = make_grid(N.P_SEMILINEAR, N.BC_DIRICHLET, 1, 1, n, h, (h / 24.0,))
    rhs = StencilRhs("semilinear", g, analytic=True)

    def exact(t):
        return x * (1.0 - x) * np.exp(t)

    return Problem("semilinear", rhs, u0, 1.0, n=n,
                   extract=lambda w: w[:-1], exact=exact, params={},
                   jac_factory=NativeJacFactory(rhs))


def make_problem(name, *, alpha=None, n=64, **kwargs):
    """Registry (problems.py:199-210)."""
    if name == "adr":
        return adr_problem(0.1 if alpha is None else alpha, n, **kwargs)
    if name == "allen_cahn":
        return allen_cahn_problem(1e-2 if alpha is None else alpha, n, **kwargs)
    if name == "brusselator":
        return brusselator_problem(1e-3 if alpha is None else alpha, n, **kwargs)
    if name == "gray_scott":
        return gray_scott_problem(1e-3 if alpha is None else alpha, n, **kwargs)
    if name == "semilinear":
        return semilinear_problem(n, **kwargs)
    raise ValueError(f"unknown problem '{name}'")
