"""Speculative phi-calls (integrators.run_stepper): a step whose Leja calls
are enqueued without host synchronisation must give bit-identical results,
counters and statistics to the synchronous path, both when the speculation
holds and when it misses (the step is then recomputed synchronously)."""

import numpy as np
import pytest
import torch

import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import ext, integrators as I

pytestmark = pytest.mark.gpu


@pytest.fixture
def spec_mode():
    old = I.SPECULATE
    yield
    I.SPECULATE = old


def _fixed_run(p, integ, dt, steps, xi, jac_factory=None, stepper=None):
    rhs = ek.CountingRhs(p.rhs)
    ctx = ek.EngineContext(xi=xi)
    pol = ek.RefreshPolicy()
    u = torch.from_numpy(p.u0).cuda()
    stats = []
    for _ in range(steps):
        s = ek.make_linearized(rhs, u, jac_factory=jac_factory, _as_numpy=False)
        ctx.est = ek.maybe_refresh(ctx.est, s.J, pol)
        r = (stepper or ek.take_step)(integ, s, dt, "leja", 1e-8, ctx)
        u = r._u
        stats.append((r.stats.leja_iters, r.stats.internal_stage_iters,
                      dict(r.stats.group_rhs_evals), rhs.counter.count, r.err_est))
    return u.cpu().numpy(), stats


@pytest.mark.parametrize("integ", ["epirk5p1", "epirk4s3", "exprb43", "exprb53s3"])
def test_speculative_steps_bit_identical(spec_mode, integ):
    xi = ek.get_leja_points(400)
    p = ext.brusselator_periodic_problem(n=128)
    rhs = ek.CountingRhs(p.rhs)
    lam, _ = ek.power_iterate(ek.make_linearized(rhs, p.u0).J)
    dt = 50.0 / abs(ek.make_estimate(lam).alpha)
    I.SPECULATE = False
    u0, s0 = _fixed_run(p, integ, dt, 4, xi)
    I.SPECULATE = True
    m0 = dict(I.SPEC_STATS)
    u1, s1 = _fixed_run(p, integ, dt, 4, xi)
    assert np.array_equal(u0, u1)
    assert s0 == s1
    # steps after the first (every group seen) held their speculation
    assert I.SPEC_STATS["steps"] - m0["steps"] == 4
    assert I.SPEC_STATS["misses"] - m0["misses"] == 0


def test_speculative_adaptive_run_identical(spec_mode):
    xi = ek.get_leja_points(400)
    p = ext.allen_cahn_periodic_problem(n=64)
    runs = []
    for flag in (False, True):
        I.SPECULATE = flag
        tr = ek.adaptive_loop(p.rhs, p.u0, 1.0, "exprb43", "leja", 1e-10,
                              ctx=ek.EngineContext(xi=xi), max_steps=60)
        runs.append(tr)
    a, b = runs
    assert np.array_equal(a.u, b.u)
    assert a.dts == b.dts
    assert (a.steps_accepted, a.steps_rejected, a.rhs_evals, a.leja_iters) == \
        (b.steps_accepted, b.steps_rejected, b.rhs_evals, b.leja_iters)


def test_speculation_miss_recomputes_step(spec_mode):
    """A stale batch hint (the group needed far more iterations than the
    speculative batch holds) misses; the step is recomputed synchronously
    with the same result, counters and statistics."""
    xi = ek.get_leja_points(400)
    p = ext.brusselator_periodic_problem(n=128)
    rhs0 = ek.CountingRhs(p.rhs)
    lam, _ = ek.power_iterate(ek.make_linearized(rhs0, p.u0).J)
    est = ek.make_estimate(lam)
    dt = 120.0 / abs(est.alpha)   # ~20 Leja iterations per group
    out = []
    for flag in (False, True):
        I.SPECULATE = flag
        rhs = ek.CountingRhs(p.rhs)
        ctx = ek.EngineContext(xi=xi, est=est)
        for g in ("internal", "stage2", "stage3"):
            ctx.leja_seen(g, 1)       # stale hint: batch of 8 iterations
        m0 = dict(I.SPEC_STATS)
        s = ek.make_linearized(rhs, p.u0)
        r = ek.take_step("epirk5p1", s, dt, "leja", 1e-8, ctx)
        out.append((r.u_high, r.stats.leja_iters, dict(r.stats.group_rhs_evals),
                    rhs.counter.count, r.err_est, dict(ctx._leja_last)))
        if flag:
            assert I.SPEC_STATS["misses"] - m0["misses"] == 1
    (ua, *ra), (ub, *rb) = out
    assert np.array_equal(ua, ub)
    assert ra == rb
    assert ra[0] > 3 * 8
