"""Oracle parity at the sizes that are benchmarked (SURVEY.md §8(c) c4 at
BASELINE.json's full sizes). The CPU oracle (oracle/, pinned bit-exact to
the reference) runs on the GPU box's host on the same seeded inputs; these
tests take minutes of host time, not of GPU time.

* the exact bench.py loop: config 4 (periodic Brusselator 4096^2 x 2, FD
  Jacobian), dt |alpha| = 50 from the power-iteration estimate, two
  EPIRK5P1 Leja steps as `fixed_step_loop` runs them (linearise, refresh,
  take_step). T2 per step: identical Leja iterations, per-group RHS charges
  and counter deltas, ||du|| / ||u|| <= 1e-10 (reference:
  integrators.py:318-341, timestep.py:167-183, leja.py:133-189);
* config 5 at 512^3 (1.07 GB per vector): one fused linear Leja phi_1
  call, T1: identical iterations, <= 1e-13 (leja.py:167-184);
* KIOPS at size: config 3 (Burgers 1024^2, analytic Jacobian) 20 adaptive
  EPIRK4s3 steps at T3 or inside the oracle's 1-ulp envelope, and one
  config 4 KIOPS phi_1 call (4096^2 x 2, FD) at T1: identical matvecs /
  substeps / rejections, <= 1e-7 (kiops.py:106-303).
"""

import numpy as np
import pytest
import torch

import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import _device as D, ext
from oracle import np_fields as OF, np_integrate as OI, np_phi as OP

pytestmark = pytest.mark.gpu

DT_ALPHA = 50.0
TOL = 1e-8


def rel(a, b):
    a = a.cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def xi():
    return OP.leja_points(400)


# ------------------------------------------------------- config 4: bench loop

def test_config4_bench_loop_two_epirk5p1_steps(xi):
    """bench.py run_ours(): the same problem, the same dt rule and the same
    per-step calls, against the oracle's fixed-step loop on the host."""
    n = 4096
    p = ext.brusselator_periodic_problem(n=n)
    rhs = ek.CountingRhs(p.rhs)
    u = D.to_dev(p.u0, copy=True)
    lam, conv = ek.power_iterate(ek.make_linearized(rhs, u).J)
    dt = DT_ALPHA / abs(ek.make_estimate(lam).alpha)
    policy, ctx = ek.RefreshPolicy(), ek.EngineContext(xi=xi)
    gpu = []
    for _ in range(2):
        c0 = rhs.counter.count
        sys_ = ek.make_linearized(rhs, u, _as_numpy=False)
        ctx.est = ek.maybe_refresh(ctx.est, sys_.J, policy)
        res = ek.take_step("epirk5p1", sys_, dt, "leja", TOL, ctx)
        u = res._u
        gpu.append((res.stats.leja_iters, dict(res.stats.group_rhs_evals),
                    rhs.counter.count - c0, u.cpu().numpy(), res.err_est))
    del p, sys_, res, u
    torch.cuda.empty_cache()

    q = OF.brusselator_periodic(n=n)
    orhs = OP.CountedRhs(q.rhs)
    octx, opol = OI.Ctx(xi=xi), OP.Policy()
    ou = q.u0.copy()
    for step in range(2):
        c0 = orhs.counter.count
        osys = OI.linearize(orhs, ou)
        octx.est = OP.refresh(octx.est, osys.J, opol)
        if step == 0:
            # the estimate the GPU's dt came from: FD power iteration, T1
            olam = abs(octx.est.alpha) / octx.est.safety
            assert abs(lam - olam) <= 1e-7 * olam, (lam, olam)
            assert octx.est.safety == ctx.est.safety
        ores = OI.step("epirk5p1", osys, dt, "leja", TOL, octx)
        ou = ores.u_high
        iters, groups, charges, ug, err = gpu[step]
        assert iters == ores.stats.leja_iters, (step, iters, ores.stats.leja_iters)
        assert groups == ores.stats.group_rhs_evals, (step, groups)
        assert charges == orhs.counter.count - c0
        assert rel(ug, ou) <= 1e-10, (step, rel(ug, ou))
        assert err == pytest.approx(ores.err_est, rel=1e-3)


# ------------------------------------------------------- config 5: 512^3

def test_config5_full_size_leja_phi1_call(xi):
    """One phi_1 call at 512^3 through the fused 3-D TMA Leja kernel
    (linear analytic Jacobian), dt = dt_CFL, tol 1e-10: T1 against the
    oracle's leja_vertical with the same estimate."""
    n = 512
    p = ext.advdiff3d_problem(n=n)
    dt = p.params["dt_cfl"]
    rhs = ek.CountingRhs(p.rhs)
    u = D.to_dev(p.u0, copy=True)
    sys_ = ek.make_linearized(rhs, u, jac_factory=p.jac_factory, _as_numpy=False)
    lam, _ = ek.power_iterate(sys_.J)
    est = ek.make_estimate(lam)
    b = D.ev(D.V(sys_._f) * dt)
    res = ek.leja_interpolate_vertical(sys_.J, b, 1, [0.5, 1.0], dt, est, 1e-10, xi=xi)
    got = [v.cpu().numpy() for v in res.vectors]
    assert rhs.counter.count == 1                     # analytic Jv charges nothing
    del p, sys_, b, u, res.vectors
    torch.cuda.empty_cache()

    q = OF.advdiff3d(n=n)
    osys = OI.linearize(OP.CountedRhs(q.rhs), q.u0, jac_factory=q.jac_factory)
    ores = OP.leja_vertical(osys.J, osys.f_n * dt, 1, [0.5, 1.0], dt, est, 1e-10, xi)
    assert res.iters == ores.iters and res.freeze_iters == ores.freeze_iters
    for g, o in zip(got, ores.vectors):
        assert rel(g, o) <= 1e-13, rel(g, o)


# ------------------------------------------------------- KIOPS at size

def test_config3_kiops_1024_20_steps(xi):
    """Config 3 KIOPS (EPIRK4s3, tol 1e-8) at the BASELINE size: 20 adaptive
    steps, T3 or inside the oracle's own 1-ulp sensitivity envelope."""
    from test_gpu_configs import _check_tier_t3, _whole_run
    n = 1024
    p, q = ext.burgers2d_problem(n=n), OF.burgers2d(n=n)
    _check_tier_t3(*_whole_run(xi, p, q, "epirk4s3", "kiops", 1e-8, 20))


def test_config4_kiops_phi1_call_full_size():
    """One KIOPS phi_1 action at config 4 (FD Jacobian, dt |alpha| = 50,
    tol 1e-9 = the engines' 0.1 tol): identical KIOPS statistics, vectors
    within the FD tier (1e-7)."""
    n = 4096
    p = ext.brusselator_periodic_problem(n=n)
    rhs = ek.CountingRhs(p.rhs)
    sys_ = ek.make_linearized(rhs, D.to_dev(p.u0, copy=True), _as_numpy=False)
    lam, _ = ek.power_iterate(sys_.J)
    dt = DT_ALPHA / abs(ek.make_estimate(lam).alpha)
    c0 = rhs.counter.count
    w, st = ek.kiops_eval(sys_.J, [None, sys_._f], dt, 0.1 * TOL)
    charges = rhs.counter.count - c0
    got = w.cpu().numpy()
    del p, sys_, w
    torch.cuda.empty_cache()

    q = OF.brusselator_periodic(n=n)
    orhs = OP.CountedRhs(q.rhs)
    osys = OI.linearize(orhs, q.u0)
    c0 = orhs.counter.count
    ow, ost = OP.kiops_eval(osys.J, [np.zeros_like(osys.f_n), osys.f_n], dt, 0.1 * TOL)
    assert (st.matvecs, st.substeps, st.rejections, st.expms, st.m_last) == \
        (ost.matvecs, ost.substeps, ost.rejections, ost.expms, ost.m_last)
    # RHS charges: one per FD action of a nonzero direction (the oracle's
    # count, which can be below matvecs: the zero-direction shortcut of
    # integrators.py:89-90 charges nothing)
    assert charges == orhs.counter.count - c0
    assert rel(got, ow) <= 1e-7, rel(got, ow)
