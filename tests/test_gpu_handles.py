"""The handle layer of the C ABI (ek_ctx / ek_op)
against the NumPy oracle: linearisation, RHS, FD / analytic Jacobian
actions, one power-iteration step, axpby and the batched dots."""

import ctypes as C

import numpy as np
import pytest

from paper_2211_08948_b200 import _device as D, _native as N, ext
from oracle import np_fields as OF

pytestmark = pytest.mark.gpu


def _p(t):
    return C.c_void_p(t.data_ptr())


@pytest.fixture()
def ctx():
    c = N.lib().ek_ctx_create(0, D.stream())
    assert c
    yield c
    N.lib().ek_ctx_destroy(c)


def _op(ctx, grid, jac):
    op = N.lib().ek_op_create(ctx, C.byref(grid), jac)
    assert op, N.lib().ek_last_error()
    return op


def test_linearize_rhs_and_fd_jv(ctx):
    p, q = ext.brusselator_periodic_problem(n=64), OF.brusselator_periodic(n=64)
    op = _op(ctx, p.rhs.grid, N.JAC_FD)
    try:
        u = D.to_dev(p.u0, copy=True)
        fu = D.empty(u.numel())
        nu = C.c_double()
        N.check(N.lib().ek_op_linearize(op, _p(u), _p(fu), C.byref(nu)), "linearize")
        assert np.array_equal(D.to_host(fu), q.rhs(p.u0))          # bit-exact stencil
        assert nu.value == pytest.approx(np.linalg.norm(p.u0), rel=1e-15)
        out = D.empty(u.numel())
        N.check(N.lib().ek_op_rhs(op, _p(u), _p(out)), "rhs")
        assert np.array_equal(D.to_host(out), q.rhs(p.u0))
        v = np.random.default_rng(1).standard_normal(p.u0.shape)
        vd = D.to_dev(v)  # keep the device copies alive across the calls
        N.check(N.lib().ek_op_jv(op, _p(vd), _p(out)), "jv")
        ref = OF.fd_jv(q.rhs, p.u0, v)
        assert np.linalg.norm(D.to_host(out) - ref) <= 1e-7 * np.linalg.norm(ref)  # FD tier
        # zero vector: fd_jacobian_apply raises ValueError (linalg.py:121-122)
        zd = D.to_dev(np.zeros_like(v))
        with pytest.raises(ValueError):
            N.check(N.lib().ek_op_jv(op, _p(zd), _p(out)), "jv0")
        # non-finite action -> FloatingPointError (linalg.py:127-128)
        bad = v.copy()
        bad[5] = np.inf
        bd = D.to_dev(bad)
        with pytest.raises(FloatingPointError):
            N.check(N.lib().ek_op_jv(op, _p(bd), _p(out)), "jv inf")
        # one power-iteration step: w = J v, ||w||
        w = D.empty(u.numel())
        nw = C.c_double()
        N.check(N.lib().ek_power_step(op, _p(vd), _p(w), C.byref(nw)), "power")
        wh = D.to_host(w)
        assert np.linalg.norm(wh - ref) <= 1e-7 * np.linalg.norm(ref)
        assert nw.value == pytest.approx(np.linalg.norm(wh), rel=1e-14)
    finally:
        N.lib().ek_op_destroy(op)


def test_analytic_jv_bit_exact(ctx):
    p, q = ext.burgers2d_problem(n=64), OF.burgers2d(n=64)
    op = _op(ctx, p.rhs.grid, N.JAC_ANALYTIC)
    try:
        u = D.to_dev(p.u0, copy=True)
        fu = D.empty(u.numel())
        N.check(N.lib().ek_op_linearize(op, _p(u), _p(fu), None), "linearize")
        v = np.random.default_rng(2).standard_normal(p.u0.shape)
        vd, out = D.to_dev(v), D.empty(u.numel())
        N.check(N.lib().ek_op_jv(op, _p(vd), _p(out)), "jv")
        assert np.array_equal(D.to_host(out), q.jac_factory(p.u0)(v))
    finally:
        N.lib().ek_op_destroy(op)


def test_op_create_rejects_missing_analytic_jacobian(ctx):
    p = ext.brusselator_periodic_problem(n=32)   # FD only in the reference
    assert not N.lib().ek_op_create(ctx, C.byref(p.rhs.grid), N.JAC_ANALYTIC)


def test_axpby_and_dot_multi():
    rng = np.random.default_rng(3)
    n = 100_003
    x, y = rng.standard_normal(n), rng.standard_normal(n)
    xd, yd0, out = D.to_dev(x), D.to_dev(y), D.empty(n)
    N.check(N.lib().ek_axpby(n, 0.3, _p(xd), -1.7, _p(yd0), _p(out), D.stream()), "axpby")
    assert np.array_equal(D.to_host(out), (0.3 * x) + (-1.7 * y))
    ys = [rng.standard_normal(n) for _ in range(5)]
    yd = [D.to_dev(a) for a in ys]
    st = D.DevState(N.ScalarState)
    res = (C.c_double * 5)()
    N.check(N.lib().ek_dot_multi(n, _p(xd), N.ptrs(yd), 5, st.ptr, res,
                                 D.work_ptr(None), D.stream()), "dots")
    for i in range(5):
        assert res[i] == pytest.approx(float(np.dot(x, ys[i])), rel=1e-12, abs=1e-12)
