"""Operators, work counters and vector kernels of the phi-action path.

Drop-in for the reference module `expkit.linalg` (linalg.py:1-199): same
names, signatures, counter semantics and exceptions. The vector work runs
on the GPU (libexpkit_sm100.so); NumPy arrays in give NumPy arrays out,
CUDA tensors in give CUDA tensors out.

Operator kinds:
  * `NativeJacobian`   — the Jacobian of a native stencil problem at a
    linearisation point (FD or analytic); the engines fuse it into their
    iteration kernels.
  * `DenseOperator`    — `MatrixFreeOperator.from_matrix`, device GEMV.
  * `ScaledOperator`   — `op.scaled(f)`.
  * plain `MatrixFreeOperator` around a user callable — the callable runs
    where the user wrote it; the engine's vector algebra stays on the GPU.

The dense helpers (`dense_expm`, `dense_phi`, `dense_phi_action`) act on
small matrices (Hessenberg projections, divided-difference generators) and
stay on the host by design (BASELINE.json north_star).
"""

import ctypes as C
import math

import numpy as np
import scipy.linalg
import torch

from . import _device as D
from . import _native as N

EPS = float(np.finfo(np.float64).eps)


class EvalCounter:
    """Monotone count of right-hand-side evaluations (linalg.py:21-32)."""

    __slots__ = ("count",)

    def __init__(self):
        self.count = 0

    def charge(self, k=1):
        if k < 0:
            raise ValueError("counter cannot decrease")
        self.count += k


class CountingRhs:
    """Charges one evaluation per call, then calls `fn` (linalg.py:35-48)."""

    def __init__(self, fn, counter=None):
        self.fn = fn
        self.counter = counter if counter is not None else EvalCounter()

    def __call__(self, u):
        self.counter.charge()
        return self.fn(u)

    @property
    def evals(self):
        return self.counter.count


def native_rhs(rhs):
    """The native stencil behind `rhs` (a StencilRhs or a CountingRhs around
    one), else None."""
    from .problems import StencilRhs
    f = rhs.fn if isinstance(rhs, CountingRhs) else rhs
    return f if isinstance(f, StencilRhs) else None


def call_rhs(rhs, x):
    """Evaluate an RHS on a device vector. Native stencils take the tensor;
    a user callable is handed a NumPy copy (it runs where it was written)."""
    if native_rhs(rhs) is not None:
        return rhs(x)
    return D.to_dev(rhs(D.to_host(x)))


class MatrixFreeOperator:
    """Linear action v -> A v with an evaluation counter (linalg.py:51-90).

    `apply(v)` keeps the reference semantics for any v; the engines call
    `apply_dev(v)` with a CUDA tensor and get a CUDA tensor back."""

    def __init__(self, apply_fn, dim, counter=None, charge_per_apply=1):
        self.apply_fn = apply_fn
        self.dim = int(dim)
        if self.dim < 1:
            raise ValueError("operator dimension must be positive")
        self.counter = counter if counter is not None else EvalCounter()
        self.charge_per_apply = charge_per_apply

    def _check(self, v):
        if tuple(v.shape) != (self.dim,):
            raise ValueError(f"expected vector of length {self.dim}, got {tuple(v.shape)}")

    def apply(self, v):
        self._check(v)
        if isinstance(v, torch.Tensor):
            return self.apply_dev(D.to_dev(v))
        if self.charge_per_apply:
            self.counter.charge(self.charge_per_apply)
        return self.apply_fn(v)

    def apply_dev(self, v):
        self._check(v)
        if self.charge_per_apply:
            self.counter.charge(self.charge_per_apply)
        return D.to_dev(self.apply_fn(D.to_host(v)))

    @property
    def eval_counter(self):
        return self.counter.count

    def scaled(self, factor):
        """Operator v -> factor * (A v) sharing this counter."""
        return ScaledOperator(self, factor)

    @classmethod
    def from_matrix(cls, A, counter=None):
        return DenseOperator(A, counter=counter)


class ScaledOperator(MatrixFreeOperator):
    """factor * base (linalg.py:77-84); charges nothing itself."""

    def __init__(self, base, factor):
        super().__init__(None, base.dim, counter=base.counter, charge_per_apply=0)
        self.base = base
        self.factor = factor

    def apply(self, v):
        self._check(v)
        if isinstance(v, torch.Tensor):
            return self.apply_dev(D.to_dev(v))
        return D.to_host(self.apply_dev(D.to_dev(v)))

    def apply_dev(self, v):
        w = self.base.apply_dev(v)
        return D.ev(self.factor * D.V(w))


class DenseOperator(MatrixFreeOperator):
    """`from_matrix`: y = A v by the device GEMV kernel (linalg.py:87-90)."""

    def __init__(self, A, counter=None):
        A = np.asarray(A, dtype=float)
        super().__init__(None, A.shape[0], counter=counter, charge_per_apply=1)
        self.A_host = A
        self._A = None

    @property
    def A_dev(self):
        if self._A is None:
            self._A = torch.from_numpy(np.ascontiguousarray(self.A_host)).to(D.device())
        return self._A

    def apply(self, v):
        self._check(v)
        out = self.apply_dev(D.to_dev(v))
        return out if isinstance(v, torch.Tensor) else D.to_host(out)

    def apply_dev(self, v):
        self._check(v)
        if self.charge_per_apply:
            self.counter.charge(self.charge_per_apply)
        out = D.empty(self.dim)
        N.check(N.lib().ek_dense_gemv(self.dim, C.c_void_p(self.A_dev.data_ptr()),
                                      C.c_void_p(v.data_ptr()),
                                      C.c_void_p(out.data_ptr()), D.stream()),
                "ek_dense_gemv")
        return out


class NativeJacobian(MatrixFreeOperator):
    """Jacobian of a native stencil problem at u (integrators.py:80-96).

    jac == JAC_FD: forward difference around the cached f(u); each action
    charges the shared RHS counter once (zero direction: no charge,
    integrators.py:89-90). jac == JAC_ANALYTIC: exact stencil, no charge.
    The engines read `grid`, `u`, `fu`, `nu` and `jac` and run fused
    kernels; `apply_dev` is the standalone action."""

    def __init__(self, stencil, u, fu, rhs, jac):
        super().__init__(None, u.numel(), counter=rhs.counter, charge_per_apply=0)
        self.stencil = stencil
        self.grid = stencil.grid
        self.u = u
        self.fu = fu
        self.rhs = rhs
        self.jac = jac
        self._nu = None

    @property
    def nu(self):
        """||u|| (linalg.py:123), computed once per linearisation."""
        if self._nu is None:
            if self.jac != N.JAC_FD:
                self._nu = 0.0
            elif getattr(self, "_nu_state", None) is not None:  # from the RHS pass
                self._nu = D.global_norm(self._nu_state.read())[0]
            else:
                self._nu = D.norm2(self.u)[0]
        return self._nu

    @property
    def comm(self):
        return self.stencil.comm

    @property
    def u_halo(self):
        """Ghost rows of u (slab mode), exchanged once per linearisation."""
        if getattr(self, "_uh", None) is None:
            self._uh = self.stencil.halo(self.u)
        return self._uh

    def halos(self, v=None, k=None):
        """C array {u, y, k} of halo buffers, or None off slab mode; the
        buffers are kept on the object until the next call."""
        if self.comm is None:
            return None
        self._hv = self.stencil.halo(v) if v is not None else None
        self._hk = self.stencil.halo(k) if k is not None else None
        return N.ptrs([self.u_halo, self._hv, self._hk])

    def apply(self, v):
        self._check(v)
        out = self.apply_dev(D.to_dev(v))
        return out if isinstance(v, torch.Tensor) else D.to_host(out)

    def apply_dev(self, v):
        self._check(v)
        out = D.empty(self.dim)
        halo = self.halos(v=v)
        if self.jac == N.JAC_FD:
            nv, flag = D.norm2(v)
            if not flag & 1:  # `if not np.any(v)` (integrators.py:89)
                out.zero_()
                return out
            eps = math.sqrt(EPS) * (1.0 + self.nu) / nv  # linalg.py:123
            self.rhs.counter.charge()
            st = D.scalar_state()
            N.check(N.lib().ek_jv(C.byref(self.grid), N.JAC_FD,
                                  C.c_void_p(self.u.data_ptr()),
                                  C.c_void_p(self.fu.data_ptr()),
                                  C.c_void_p(v.data_ptr()), eps,
                                  C.c_void_p(out.data_ptr()), st.ptr, D.work_ptr(),
                                  halo, D.stream()), "ek_jv")
            if D.global_norm(st.read())[1] & 2:
                raise FloatingPointError("non-finite Jacobian action")
            return out
        N.check(N.lib().ek_jv(C.byref(self.grid), N.JAC_ANALYTIC,
                              C.c_void_p(self.u.data_ptr()),
                              C.c_void_p(self.fu.data_ptr()),
                              C.c_void_p(v.data_ptr()), 0.0,
                              C.c_void_p(out.data_ptr()), None, None, halo,
                              D.stream()), "ek_jv")
        return out


def fused_target(op):
    """(NativeJacobian, dt) when `op` is a native Jacobian or one scaling of
    it, so engines can run the fused kernels; else None."""
    if isinstance(op, NativeJacobian):
        return op, 1.0
    if isinstance(op, ScaledOperator) and isinstance(op.base, NativeJacobian):
        return op.base, float(op.factor)
    return None


def norm_l2(v):
    """Unnormalised Euclidean norm (linalg.py:93-95), device reduction."""
    return D.norm2(D.to_dev(v))[0]


def dot(x, y):
    """linalg.py:98-101, device reduction."""
    if tuple(x.shape) != tuple(y.shape):
        raise ValueError("length mismatch in dot")
    xd, yd = D.to_dev(x), D.to_dev(y)
    pr = D._Prog()
    pr.lower(D.V(xd) * D.V(yd))
    pr.emit(N.VX_ACC, 0)
    pr.emit(N.VX_POP)
    st = D.scalar_state()
    code = (C.c_int32 * len(pr.code))(*pr.code)
    N.check(N.lib().ek_vexpr(xd.numel(), code, len(pr.code), (C.c_double * 1)(), 0,
                             N.ptrs(pr.ins), len(pr.ins), N.ptrs([]), 0, st.ptr,
                             D.work_ptr(), D.stream()), "ek_vexpr")
    return D.global_sum_state(st.read())


def axpy(alpha, x, y):
    """alpha*x + y (linalg.py:104-108), device elementwise."""
    if tuple(x.shape) != tuple(y.shape):
        raise ValueError("length mismatch in axpy")
    out = D.ev(alpha * D.V(D.to_dev(x)) + D.V(D.to_dev(y)))
    return D.like_input(out, x)


def fd_jacobian_apply(f, u, v, fu=None):
    """Forward-difference Jacobian action (f(u + eps v) - f(u)) / eps with
    eps = sqrt(eps_mach)(1 + ||u||)/||v|| (linalg.py:111-129), on the GPU.
    A native stencil `f` runs the fused kernel; a user callable is evaluated
    where it was written. One RHS charge when `fu` is given."""
    if tuple(u.shape) != tuple(v.shape):
        raise ValueError("u and v must have equal length")
    ud, vd = D.to_dev(u), D.to_dev(v)
    nv = D.norm2(vd)[0]
    if nv == 0.0:
        raise ValueError("degenerate direction: v = 0")
    nu = D.norm2(ud)[0]
    eps = math.sqrt(EPS) * (1.0 + nu) / nv
    fud = D.to_dev(fu) if fu is not None else call_rhs(f, ud)
    st = native_rhs(f)
    if st is not None and st.grid.problem != N.P_SEMILINEAR:
        if isinstance(f, CountingRhs):
            f.counter.charge()
        out = D.empty(ud.numel())
        sst = D.scalar_state()
        N.check(N.lib().ek_jv(C.byref(st.grid), N.JAC_FD, C.c_void_p(ud.data_ptr()),
                              C.c_void_p(fud.data_ptr()), C.c_void_p(vd.data_ptr()),
                              eps, C.c_void_p(out.data_ptr()), sst.ptr, D.work_ptr(),
                              None, D.stream()), "ek_jv")
        bad = bool(sst.read().flag & 2)
    else:
        w = D.ev(D.V(ud) + eps * D.V(vd))
        fw = call_rhs(f, w)
        out = D.empty(ud.numel())
        _, flag = D.evaluate([((D.V(fw) - D.V(fud)) / eps, out)], ud.numel(),
                             check=True)
        bad = bool(flag & 2)
    if bad:
        raise FloatingPointError("non-finite Jacobian action")
    return D.like_input(out, u)


# ------------------------------------------------------- small dense (host)
# torch-free module: the divided-difference worker processes run the same code
from ._dense import _phi_taylor, dense_expm, dense_phi, dense_phi_action  # noqa: E402,F401
