"""BASELINE.json configurations on the GPU against the CPU oracle run live on
the same seeded inputs (the oracle is pinned bit-exact to the reference in
tests/test_oracle_golden.py).

  config 1  2-D upwind adv-diff 64^2, one EXPRB2 step, dt = 50 dt_CFL, Leja 1e-10
  config 2  periodic Allen-Cahn 256^2, EXPRB43, Leja and KIOPS, tol 1e-10, 100 steps
  config 3  2-D Burgers (1024^2 Leja / LeKry; 256^2 KIOPS), EPIRK4s3, tol 1e-8, 20 steps
  config 4  periodic Brusselator: 1024^2 x 2 EPIRK5P1 Leja step; 4096^2 x 2 RHS + FD Jv
  config 5  3-D upwind adv-diff: 48^3 EXPRB32 steps vs oracle; 512^3 linearity / exactness
"""

import math

import numpy as np
import pytest
import torch

import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import _device as D, ext
from oracle import np_fields as OF, np_integrate as OI, np_phi as OP

pytestmark = pytest.mark.gpu


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.fixture(scope="module")
def xi():
    return OP.leja_points(400)


# ------------------------------------------------------------------ config 1

@pytest.mark.parametrize("pe", [1.0, 10.0])
def test_config1_exprb2_step(xi, pe):
    n = 64
    p, q = ext.advdiff2d_problem(n=n, peclet=pe), OF.advdiff2d(n=n, peclet=pe)
    dt = 50.0 * p.params["dt_cfl"]
    assert dt == 50.0 * q.params["dt_cfl"]
    rhs = ek.CountingRhs(p.rhs)
    sys_ = ek.make_linearized(rhs, p.u0, jac_factory=p.jac_factory)
    lam, _ = ek.power_iterate(sys_.J)
    orhs = OP.CountedRhs(q.rhs)
    osys = OI.linearize(orhs, q.u0, jac_factory=q.jac_factory)
    olam, _ = OP.power_iterate(osys.J)
    assert abs(lam - olam) <= 1e-12 * olam
    est = ek.make_estimate(olam)
    ctx = ek.EngineContext(est=est, xi=xi, engine_tol_factor=1.0)
    res = ext.take_step_ext("exprb2", sys_, dt, "leja", 1e-10, ctx)
    ores = OI.step("exprb2", osys, dt, "leja", 1e-10, OI.Ctx(est=est, xi=xi,
                                                              engine_tol_factor=1.0))
    assert res.stats.leja_iters == ores.stats.leja_iters
    assert rel(res.u_high, ores.u_high) <= 1e-12
    # accuracy against the exact exponential of the (oracle-assembled) operator
    import scipy.sparse.linalg as spla
    exact = spla.expm_multiply(dt * _advdiff_matrix(q, n), q.u0)
    assert rel(res.u_high, exact) <= 1e-8


def _advdiff_matrix(q, n):
    import scipy.sparse as sp
    N = n * n
    rows, cols, vals = [], [], []
    basis = np.zeros(N)
    for k in range(N):
        basis[k] = 1.0
        col = q.rhs(basis)
        nz = np.nonzero(col)[0]
        rows.extend(nz.tolist())
        cols.extend([k] * len(nz))
        vals.extend(col[nz].tolist())
        basis[k] = 0.0
    return sp.csr_matrix((vals, (rows, cols)), shape=(N, N))


# ------------------------------------------------------------------ config 2

def _counts(r):
    return [r.steps_accepted, r.steps_rejected, r.rhs_evals, r.leja_iters,
            r.krylov_matvecs, r.substeps]


def _whole_run(xi, p, q, integ, scheme, tol, max_steps):
    """GPU run, oracle run and the oracle's 1-ulp sensitivity envelope (every
    np.linalg.norm scaled by 1 + 2^-52)."""
    tr = ek.adaptive_loop(p.rhs, p.u0, 1.0, integ, scheme, tol, jac_factory=p.jac_factory,
                          ctx=ek.EngineContext(xi=xi), max_steps=max_steps)

    def oracle():
        return OI.adaptive(q.rhs, q.u0, 1.0, integ, scheme, tol, jac_factory=q.jac_factory,
                           ctx=OI.Ctx(xi=xi), max_steps=max_steps)
    otr = oracle()
    real = np.linalg.norm
    np.linalg.norm = lambda *a, **k: real(*a, **k) * (1.0 + 2.0**-52)
    try:
        ptr = oracle()
    finally:
        np.linalg.norm = real
    return tr, otr, ptr


def _check_tier_t3(tr, otr, ptr):
    # discrete decisions: identical accepted-step sequence and work counts
    assert _counts(tr) == _counts(otr)
    assert len(tr.dts) == len(otr.dts)
    # continuous values: <= 1e-10, or inside the oracle's own sensitivity
    # envelope (the same 1-ulp change of a norm moves the oracle itself)
    env_u = rel(ptr.u, otr.u)
    env_dt = rel(np.array(ptr.dts), np.array(otr.dts)) if len(ptr.dts) == len(otr.dts) else 1.0
    assert rel(tr.u, otr.u) <= max(1e-10, 10.0 * env_u), (rel(tr.u, otr.u), env_u)
    assert rel(np.array(tr.dts), np.array(otr.dts)) <= max(1e-9, 10.0 * env_dt)


@pytest.mark.parametrize("scheme", ["leja", "kiops"])
def test_config2_allen_cahn_100_steps(xi, scheme):
    n = 256
    p, q = ext.allen_cahn_periodic_problem(n=n), OF.allen_cahn_periodic(n=n)
    _check_tier_t3(*_whole_run(xi, p, q, "exprb43", scheme, 1e-10, 100))


# ------------------------------------------------------------------ config 3

@pytest.mark.parametrize("scheme,n", [("leja", 1024), ("lekry", 1024), ("kiops", 256)])
def test_config3_burgers_20_steps(xi, scheme, n):
    p, q = ext.burgers2d_problem(n=n), OF.burgers2d(n=n)
    _check_tier_t3(*_whole_run(xi, p, q, "epirk4s3", scheme, 1e-8, 20))


# ------------------------------------------------------------------ config 4

def test_config4_epirk5p1_leja_step_1024(xi):
    n = 1024
    p, q = ext.brusselator_periodic_problem(n=n), OF.brusselator_periodic(n=n)
    rhs = ek.CountingRhs(p.rhs)
    sys_ = ek.make_linearized(rhs, p.u0)
    orhs = OP.CountedRhs(q.rhs)
    osys = OI.linearize(orhs, q.u0)
    olam, _ = OP.power_iterate(osys.J, max_it=30)
    est = ek.make_estimate(olam)
    dt = 50.0 / abs(est.alpha)
    res = ek.take_step("epirk5p1", sys_, dt, "leja", 1e-8, ek.EngineContext(est=est, xi=xi))
    ores = OI.step("epirk5p1", osys, dt, "leja", 1e-8, OI.Ctx(est=est, xi=xi))
    assert res.stats.leja_iters == ores.stats.leja_iters
    assert res.stats.group_rhs_evals == ores.stats.group_rhs_evals
    assert rel(res.u_high, ores.u_high) <= 1e-10
    assert res.err_est == pytest.approx(ores.err_est, rel=1e-4)


def test_config4_full_size_rhs_and_fd_jv():
    n = 4096
    p, q = ext.brusselator_periodic_problem(n=n), OF.brusselator_periodic(n=n)
    u = torch.from_numpy(p.u0).cuda()
    f = p.rhs(u)
    fq = q.rhs(q.u0)
    assert np.array_equal(f.cpu().numpy(), fq)
    v = np.random.default_rng(4).standard_normal(p.u0.size)
    eps = math.sqrt(ek.linalg.EPS) * (1.0 + np.linalg.norm(q.u0)) / np.linalg.norm(v)
    w = q.rhs(q.u0 + eps * v)
    ref = (w - fq) / eps
    got = ek.fd_jacobian_apply(p.rhs, q.u0, v, fu=fq)
    assert rel(got, ref) <= 1e-7


# ------------------------------------------------------------------ config 5

def test_config5_exprb32_steps_48(xi):
    n = 48
    p, q = ext.advdiff3d_problem(n=n), OF.advdiff3d(n=n)
    assert np.array_equal(p.rhs(p.u0), q.rhs(q.u0))
    for mult in (5.0, 50.0):
        dt = mult * p.params["dt_cfl"]
        u = ek.fixed_step_loop(p.rhs, p.u0, 2 * dt, 2, "exprb32", "leja", 1e-10,
                               jac_factory=p.jac_factory, ctx=ek.EngineContext(xi=xi),
                               stepper=ext.take_step_ext)
        ou = _oracle_fixed(q, 2 * dt, 2, xi)
        assert rel(u, ou) <= 1e-12


def _oracle_fixed(q, t_final, steps, xi):
    rhs = OP.CountedRhs(q.rhs)
    ctx = OI.Ctx(xi=xi)
    pol = OP.Policy()
    dt = t_final / steps
    u = q.u0.copy()
    for _ in range(steps):
        sys_ = OI.linearize(rhs, u, jac_factory=q.jac_factory)
        ctx.est = OP.refresh(ctx.est, sys_.J, pol)
        u = OI.step("exprb32", sys_, dt, "leja", 1e-10, ctx).u_high
    return u


def test_config5_full_size_linearity_and_remainder():
    """512^3 (1 GB per vector): the analytic Jacobian is linear to rounding
    and equals the RHS (linear problem); the EXPRB32 remainder of a linear
    problem vanishes to rounding."""
    n = 512
    p = ext.advdiff3d_problem(n=n)
    u = torch.from_numpy(p.u0).cuda()
    rhs = ek.CountingRhs(p.rhs)
    sys_ = ek.make_linearized(rhs, u, jac_factory=p.jac_factory)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(u.numel(), dtype=torch.float64, device="cuda", generator=g)
    jx = sys_.J.apply(x)
    assert torch.equal(jx, p.rhs(x))              # J == f for a linear problem
    y = torch.randn(u.numel(), dtype=torch.float64, device="cuda", generator=g)
    lhs = sys_.J.apply(2.0 * x + y)
    rhs_lin = 2.0 * jx + sys_.J.apply(y)
    assert (torch.linalg.vector_norm(lhs - rhs_lin) / torch.linalg.vector_norm(lhs)) < 1e-13
    r = ek.remainder(sys_, u + 1e-3 * x)
    assert torch.linalg.vector_norm(r) <= 1e-9 * torch.linalg.vector_norm(sys_.f_n)
