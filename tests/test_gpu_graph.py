"""The Leja iterations of a phi-call as a CUDA graph with a device-side WHILE
loop (`ek_leja_run_graph`): one graph launch per 32-point
chunk runs the call to its end. Results, iteration counts, freeze points and
RHS charges are those of the launch-batch path bit for bit — for analytic
and FD Jacobians, 2-D (row march) and 3-D (TMA plane march), calls that end
at m = 0, calls that cross chunk boundaries, calls cut off by max_points —
and whole steps / adaptive runs are unchanged."""

import numpy as np
import pytest

import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import _native as N, ext, leja as L

pytestmark = pytest.mark.gpu


@pytest.fixture
def graph_switch():
    old = L._GRAPH[0]
    yield
    L._GRAPH[0] = old


def _setup(name, n, analytic):
    p = ek.make_problem(name, n=n) if name in ek.PROBLEMS else ext.make_ext_problem(name, n=n)
    rhs = ek.CountingRhs(p.rhs)
    sys_ = ek.make_linearized(rhs, p.u0, jac_factory=p.jac_factory if analytic else None)
    est = ek.make_estimate(ek.power_iterate(sys_.J)[0])
    return p, rhs, sys_, est


CALLS = [("advdiff2d", 128, True, 20.0, [0.5, 1.0]),
         ("brusselator_periodic", 96, False, 30.0, [1.0]),
         ("brusselator_periodic", 96, False, 30.0, [0.25, 0.5, 1.0]),
         ("allen_cahn", 64, False, 15.0, [0.5, 1.0]),
         ("burgers2d", 128, True, 25.0, [1.0 / 3.0, 2.0 / 3.0, 1.0]),
         ("advdiff3d", 34, True, 20.0, [0.5, 1.0]),
         ("advdiff2d", 128, True, 400.0, [1.0]),      # crosses 32-point chunks
         ("advdiff2d", 128, True, 1e-6, [0.5, 1.0])]  # everything freezes at m = 0


@pytest.mark.parametrize("name,n,analytic,scale,coeffs", CALLS)
def test_graph_call_equals_launch_batches(graph_switch, name, n, analytic, scale, coeffs):
    xi = ek.get_leja_points(400)
    p, rhs, sys_, est = _setup(name, n, analytic)
    dt = scale / abs(est.alpha)
    b = sys_.f_n * dt
    out = {}
    for mode in (False, True):
        L._GRAPH[0] = mode
        L._DD_CACHE.clear()
        c0 = rhs.counter.count
        tol = 1.0 if scale <= 1e-6 else 1e-10  # loose: every accumulator freezes at m = 0
        r = ek.leja_interpolate_vertical(sys_.J, b, 1, coeffs, dt, est, tol, xi=xi)
        out[mode] = (r, rhs.counter.count - c0)
    (a, ca), (g, cg) = out[False], out[True]
    assert g.iters == a.iters and g.freeze_iters == a.freeze_iters and cg == ca
    if scale >= 400.0:
        assert a.iters > 32
    if scale <= 1e-6:
        assert a.iters == 0
    for x, y in zip(g.vectors, a.vectors):
        assert np.array_equal(x, y)


def test_graph_call_respects_max_points(graph_switch):
    xi = ek.get_leja_points(400)
    p, rhs, sys_, est = _setup("advdiff2d", 64, True)
    dt = 100.0 / abs(est.alpha)
    b = sys_.f_n * dt
    for max_points in (2, 5, 33, 40):
        errs = {}
        for mode in (False, True):
            L._GRAPH[0] = mode
            with pytest.raises(ek.NonConvergence) as ei:
                ek.leja_interpolate_vertical(sys_.J, b, 1, [1.0], dt, est, 1e-13, xi=xi,
                                             max_points=max_points)
            errs[mode] = (ei.value.iters, ei.value.detail)
        assert errs[True] == errs[False]
        assert errs[True][0] == max_points


@pytest.mark.parametrize("integrator,name,analytic",
                         [("epirk5p1", "brusselator_periodic", False),
                          ("epirk4s3", "burgers2d", True),
                          ("exprb43", "allen_cahn_periodic", False)])
def test_adaptive_runs_unchanged_by_graph_mode(graph_switch, integrator, name, analytic):
    """Speculative steps with the graph loop: the same accepted / rejected
    steps, counters and solution as with launch batches."""
    p = ext.make_ext_problem(name, n=96)
    xi = ek.get_leja_points(400)
    runs = {}
    for mode in (False, True):
        L._GRAPH[0] = mode
        L._DD_CACHE.clear()
        tr = ek.adaptive_loop(p.rhs, p.u0, 1.0, integrator, "leja", 1e-8,
                              jac_factory=p.jac_factory if analytic else None,
                              ctx=ek.EngineContext(xi=xi), max_steps=12)
        runs[mode] = tr
    a, g = runs[False], runs[True]
    assert (g.steps_accepted, g.steps_rejected) == (a.steps_accepted, a.steps_rejected)
    assert g.leja_iters == a.leja_iters and g.rhs_evals == a.rhs_evals
    assert g.t == a.t and g.dts == a.dts
    assert np.array_equal(np.asarray(g.u), np.asarray(a.u))
