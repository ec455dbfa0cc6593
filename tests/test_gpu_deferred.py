"""Deferred accumulation of the Leja sums (`ek_leja_run_seq`,
`ek_leja_combine`; large whole-grid calls): the iterations keep every iterate
in its own buffer and one pass forms p_i = sum_m d_i[m] y_m at the end, term
by term in the reference's order (leja.py:161, 179). Results, iteration
counts, freeze points and RHS charges are those of the per-iteration
accumulation bit for bit — analytic and FD Jacobians, 2-D (row march) and 3-D
(plane march), groups whose members freeze at different iterations, calls
that end at m = 0, calls that cross 32-point chunks, calls cut off by
max_points — and whole steps / adaptive runs (speculative phi-calls
included) are unchanged. The mode is forced on here for small grids (its
size threshold is a performance choice, not a correctness one)."""

import numpy as np
import pytest

import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import ext, leja as L

pytestmark = pytest.mark.gpu


@pytest.fixture
def defer_switch():
    old = list(L._DEFER)
    yield
    L._DEFER[:] = old


def _mode(on):
    L._DEFER[0] = on
    L._DEFER[1] = 0   # any vector length
    L._DEFER[2] = 1   # any group size
    L._DEFER[4] = 1


def _setup(name, n, analytic):
    p = ek.make_problem(name, n=n) if name in ek.PROBLEMS else ext.make_ext_problem(name, n=n)
    rhs = ek.CountingRhs(p.rhs)
    sys_ = ek.make_linearized(rhs, p.u0, jac_factory=p.jac_factory if analytic else None)
    est = ek.make_estimate(ek.power_iterate(sys_.J)[0])
    return p, rhs, sys_, est


CALLS = [("advdiff2d", 128, True, 20.0, [0.5, 1.0]),
         ("brusselator_periodic", 96, False, 30.0, [1.0]),
         ("brusselator_periodic", 96, False, 30.0, [0.25, 0.5, 1.0]),
         ("brusselator_periodic", 200, False, 50.0, [0.2, 0.4, 0.6, 0.8, 1.0]),
         ("allen_cahn", 64, False, 15.0, [0.5, 1.0]),
         ("burgers2d", 128, True, 25.0, [1.0 / 3.0, 2.0 / 3.0, 1.0]),
         ("advdiff3d", 34, True, 20.0, [0.5, 1.0]),
         ("advdiff3d", 70, True, 40.0, [0.25, 1.0]),
         ("advdiff2d", 128, True, 400.0, [0.5, 1.0]),   # crosses 32-point chunks
         ("brusselator_periodic", 96, False, 400.0, [0.3, 0.7, 1.0]),   # FD, crosses chunks
         ("advdiff3d", 40, True, 400.0, [0.5, 1.0]),    # 3-D, crosses chunks
         ("advdiff2d", 128, True, 1e-6, [0.5, 1.0])]    # everything freezes at m = 0


@pytest.mark.parametrize("name,n,analytic,scale,coeffs", CALLS)
def test_deferred_call_equals_per_iteration_accumulation(defer_switch, name, n, analytic, scale,
                                                         coeffs):
    xi = ek.get_leja_points(400)
    p, rhs, sys_, est = _setup(name, n, analytic)
    dt = scale / abs(est.alpha)
    b = sys_.f_n * dt
    out = {}
    for mode in (False, True):
        _mode(mode)
        L._DD_CACHE.clear()
        c0 = rhs.counter.count
        tol = 1.0 if scale <= 1e-6 else 1e-10  # loose: every accumulator freezes at m = 0
        r = ek.leja_interpolate_vertical(sys_.J, b, 1, coeffs, dt, est, tol, xi=xi)
        out[mode] = (r, rhs.counter.count - c0)
    (a, ca), (d, cd) = out[False], out[True]
    assert d.iters == a.iters and d.freeze_iters == a.freeze_iters and cd == ca
    if scale >= 400.0:
        assert a.iters > 32
    if scale <= 1e-6:
        assert a.iters == 0
    if len(coeffs) >= 3 and scale >= 30.0:
        assert len(set(a.freeze_iters)) > 1   # members freeze at different iterations
    for x, y in zip(d.vectors, a.vectors):
        assert np.array_equal(x, y)


def test_deferred_call_respects_max_points(defer_switch):
    xi = ek.get_leja_points(400)
    p, rhs, sys_, est = _setup("advdiff2d", 64, True)
    dt = 100.0 / abs(est.alpha)
    b = sys_.f_n * dt
    for max_points in (2, 5, 33, 40):
        errs = {}
        for mode in (False, True):
            _mode(mode)
            with pytest.raises(ek.NonConvergence) as ei:
                ek.leja_interpolate_vertical(sys_.J, b, 1, [0.5, 1.0], dt, est, 1e-13, xi=xi,
                                             max_points=max_points)
            errs[mode] = (ei.value.iters, ei.value.detail)
        assert errs[True] == errs[False]
        assert errs[True][0] == max_points


def test_deferred_call_device_vector_in_device_vectors_out(defer_switch):
    """Device-resident b (the integrators' case): the accumulators come back
    as device tensors with the same bits."""
    import torch
    from paper_2211_08948_b200 import _device as D
    xi = ek.get_leja_points(400)
    p, rhs, sys_, est = _setup("brusselator_periodic", 128, False)
    dt = 40.0 / abs(est.alpha)
    b = D.to_dev(sys_.f_n * dt, copy=True)
    out = {}
    for mode in (False, True):
        _mode(mode)
        r = ek.leja_interpolate_vertical(sys_.J, b, 2, [0.5, 0.75, 1.0], dt, est, 1e-9, xi=xi)
        out[mode] = r
    a, d = out[False], out[True]
    assert d.iters == a.iters and d.freeze_iters == a.freeze_iters
    for x, y in zip(d.vectors, a.vectors):
        assert isinstance(x, torch.Tensor) and torch.equal(x, y)


@pytest.mark.parametrize("integrator,name,analytic",
                         [("epirk5p1", "brusselator_periodic", False),
                          ("epirk4s3", "burgers2d", True),
                          ("exprb43", "allen_cahn_periodic", False)])
def test_adaptive_runs_unchanged_by_deferred_mode(defer_switch, integrator, name, analytic):
    """Speculative steps with deferred accumulation: the same accepted /
    rejected steps, counters and solution as with per-iteration sums."""
    p = ext.make_ext_problem(name, n=96)
    xi = ek.get_leja_points(400)
    runs = {}
    for mode in (False, True):
        _mode(mode)
        L._DD_CACHE.clear()
        tr = ek.adaptive_loop(p.rhs, p.u0, 1.0, integrator, "leja", 1e-8,
                              jac_factory=p.jac_factory if analytic else None,
                              ctx=ek.EngineContext(xi=xi), max_steps=12)
        runs[mode] = tr
    a, d = runs[False], runs[True]
    assert (d.steps_accepted, d.steps_rejected) == (a.steps_accepted, a.steps_rejected)
    assert d.leja_iters == a.leja_iters and d.rhs_evals == a.rhs_evals
    assert d.t == a.t and d.dts == a.dts
    assert np.array_equal(np.asarray(d.u), np.asarray(a.u))


def test_fixed_steps_epirk5p1_unchanged_by_deferred_mode(defer_switch):
    """The bench loop in small: fixed-dt EPIRK5P1 Leja steps (speculative
    phi-calls after the first step) give the same bits and counters."""
    p = ext.brusselator_periodic_problem(n=160)
    xi = ek.get_leja_points(400)
    runs = {}
    for mode in (False, True):
        _mode(mode)
        L._DD_CACHE.clear()
        rhs = ek.CountingRhs(p.rhs)
        sys0 = ek.make_linearized(rhs, p.u0)
        est = ek.make_estimate(ek.power_iterate(sys0.J)[0])
        dt = 50.0 / abs(est.alpha)
        ctx = ek.EngineContext(est=est, xi=xi)
        u, stats = p.u0, []
        for _ in range(4):
            s = ek.make_linearized(rhs, u)
            r = ek.take_step("epirk5p1", s, dt, "leja", 1e-8, ctx)
            u = r.u_high
            stats.append((r.stats.leja_iters, dict(r.stats.group_rhs_evals), float(r.err_est)))
        runs[mode] = (u, stats, rhs.counter.count)
    (ua, sa, ca), (ud, sd, cd) = runs[False], runs[True]
    assert sd == sa and cd == ca
    assert np.array_equal(ud, ua)


def test_deferred_mode_selection(defer_switch):
    """The form is chosen per call: on by size / group thresholds, off when the
    chunk's iterate buffers would exceed the byte budget or the switch is
    off; the profile record says which ran."""
    xi = ek.get_leja_points(400)
    p, rhs, sys_, est = _setup("brusselator_periodic", 96, False)
    dt = 30.0 / abs(est.alpha)
    b = sys_.f_n * dt

    def ran_deferred():
        L.PROFILE = []
        try:
            ek.leja_interpolate_vertical(sys_.J, b, 1, [0.5, 1.0], dt, est, 1e-10, xi=xi)
            return L.PROFILE[0]["deferred"]
        finally:
            L.PROFILE = None

    _mode(True)
    assert ran_deferred() is True
    L._DEFER[3] = 8            # byte budget smaller than one iterate
    assert ran_deferred() is False
    _mode(True)
    L._DEFER[3] = 48 << 30
    L._DEFER[1] = 1 << 40      # vector length threshold above this grid
    assert ran_deferred() is False
    _mode(False)
    assert ran_deferred() is False
    _mode(True)
    L._DEFER[4] = 3            # FD calls need >= 3 coefficients: this one has 2
    assert ran_deferred() is False


@pytest.mark.parametrize("name,analytic", [("advdiff2d", True), ("brusselator_periodic", False)])
def test_deferred_call_raises_as_the_per_iteration_form(defer_switch, name, analytic):
    """A spectrum estimate far too small makes the iteration blow up: both
    forms stop at the same iteration with the same exception (overflowing
    norm -> NonConvergence, non-finite FD action -> FloatingPointError;
    leja.py:174-175, linalg.py:127-128)."""
    xi = ek.get_leja_points(400)
    p, rhs, sys_, est = _setup(name, 96, analytic)
    bad = ek.make_estimate(est.alpha * 1e-4)
    dt = 30.0 / abs(est.alpha)
    b = sys_.f_n * dt
    seen = {}
    for mode in (False, True):
        _mode(mode)
        L._DD_CACHE.clear()
        c0 = rhs.counter.count
        with pytest.raises((ek.NonConvergence, FloatingPointError)) as ei:
            ek.leja_interpolate_vertical(sys_.J, b, 1, [0.5, 1.0], dt, bad, 1e-10, xi=xi)
        seen[mode] = (type(ei.value), str(ei.value), getattr(ei.value, "iters", None),
                      rhs.counter.count - c0)
    assert seen[True] == seen[False]
