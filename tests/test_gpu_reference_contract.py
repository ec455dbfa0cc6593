"""The reference package's unit-test contract, restated against the drop-in
on the GPU engines ("run all of these against the new
package unchanged (GPU engines, numpy I/O)").

The reference suite itself cannot travel to the GPU box (`/root/reference`
is absent there), so each behaviour it pins is restated here in this
repository's own cases: the same property, the same tolerance, other
matrices and seeds. Every test names the reference test it stands for.
Dense and callable operators take the generic device path; the stencil
cases at the end take the fused kernels.

Tolerances are the reference's own: dense phi actions 1e-10 relative
(Leja, test_leja.py:113-126), 1e-8 / 1e-7 (KIOPS, test_kiops.py:69-113),
happy breakdown 1e-11 (test_kiops.py:124-135).
"""

import math

import numpy as np
import pytest
import scipy.linalg
from scipy.integrate import solve_ivp

import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import ext
from paper_2211_08948_b200.errors import NonConvergence
from paper_2211_08948_b200.integrators import (EMBEDDED_ORDER, INTEGRATOR_ORDER, INTEGRATORS,
                                               LEKRY_INTEGRATORS, SCHEMES, EngineContext)
from paper_2211_08948_b200.kiops import (AugmentedSystem, arnoldi_iop, augmented_apply,
                                         kiops, kiops_eval)
from paper_2211_08948_b200.leja import leja_interpolate, leja_interpolate_vertical
from paper_2211_08948_b200.linalg import (CountingRhs, MatrixFreeOperator, dense_phi,
                                          dense_phi_action)
from paper_2211_08948_b200.spectrum import (GAMMA_MIN, RefreshPolicy, SpectrumEstimate,
                                            make_estimate, maybe_refresh, power_iterate)

pytestmark = pytest.mark.gpu


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(b))


def stiff_matrix(n, seed, spread, coupling):
    """Diagonal spectrum on [-spread, -spread/n] plus a small random
    non-normal part (the reference's test systems have the same shape)."""
    rng = np.random.default_rng(seed)
    A = np.diag(-np.geomspace(spread / n, spread, n))
    A += coupling * rng.standard_normal((n, n))
    return A


def leftmost(A):
    return float(np.linalg.eigvals(A).real.min())


def dense_op(A):
    return MatrixFreeOperator.from_matrix(A)


# --------------------------------------------------------------------- Leja

@pytest.mark.parametrize("l", [0, 1, 2, 4])
def test_leja_single_vs_dense_phi(xi, l):
    """test_leja.py:113-126: one phi_l action within 1e-10 of the dense
    phi_l(hA)b, with a positive iteration count."""
    A = stiff_matrix(28, seed=101, spread=25.0, coupling=0.04)
    b = np.random.default_rng(102).standard_normal(28)
    est = make_estimate(leftmost(A))
    h = 0.35
    p, iters = leja_interpolate(dense_op(A), b, l, h, est, 1e-12, xi=xi)
    assert isinstance(p, np.ndarray) and p.shape == b.shape
    assert iters > 0
    assert relerr(p, dense_phi_action(l, h * A, b)) <= 1e-10


def test_leja_vertical_equals_separate_calls(xi):
    """test_leja.py:128-139: a vertical group equals its members computed
    one by one, and a smaller coefficient freezes no later."""
    A = stiff_matrix(22, seed=103, spread=18.0, coupling=0.03)
    b = np.random.default_rng(104).standard_normal(22)
    est = make_estimate(leftmost(A))
    coeffs = [0.2, 0.5, 1.0]
    res = leja_interpolate_vertical(dense_op(A), b, 2, coeffs, 0.6, est, 1e-12, xi=xi)
    for ci, vec in zip(coeffs, res.vectors):
        single, _ = leja_interpolate(dense_op(A), b, 2, ci * 0.6, est, 1e-12, xi=xi)
        assert relerr(vec, single) <= 1e-10
    assert res.freeze_iters[0] <= res.freeze_iters[1] <= res.freeze_iters[2]
    assert res.iters == max(res.freeze_iters)


def test_leja_termination_bound(xi):
    """test_leja.py:142-152: at the returned count the absolute error is
    within a small multiple of tol."""
    A = stiff_matrix(18, seed=105, spread=6.0, coupling=0.05)
    b = np.linspace(-1.0, 1.0, 18)
    est = make_estimate(leftmost(A))
    tol = 1e-8
    res = leja_interpolate_vertical(dense_op(A), b, 1, [1.0], 0.4, est, tol, xi=xi)
    exact = dense_phi_action(1, 0.4 * A, b)
    assert np.linalg.norm(res.vectors[0] - exact) < 100 * tol


def test_leja_exhaustion_payload(xi):
    """test_leja.py:155-165: running out of points raises NonConvergence
    with iters == max_points and the stalled coefficients listed."""
    A = stiff_matrix(18, seed=106, spread=500.0, coupling=0.1)
    est = make_estimate(leftmost(A))
    with pytest.raises(NonConvergence) as exc:
        leja_interpolate_vertical(dense_op(A), np.ones(18), 1, [0.25, 1.0], 1.0, est,
                                  1e-12, xi=xi, max_points=10)
    assert exc.value.iters == 10
    assert exc.value.detail["stalled_coefficients"]


@pytest.mark.parametrize("coeffs,tol", [([0.0], 1e-8), ([1.25], 1e-8), ([-0.5], 1e-8),
                                        ([1.0], 0.0), ([1.0], -1e-8)])
def test_leja_argument_validation(xi, coeffs, tol):
    """test_leja.py:168-176: coefficients outside (0, 1] and tol <= 0 are
    ValueError, before any device work."""
    op = MatrixFreeOperator(lambda v: -2.0 * v, 5)
    with pytest.raises(ValueError):
        leja_interpolate_vertical(op, np.ones(5), 1, coeffs, 0.1, make_estimate(-2.0), tol,
                                  xi=xi)


def test_leja_input_not_mutated(xi):
    """SURVEY.md §8(b) b3 (leja.py:159): b is copied, never written."""
    A = stiff_matrix(12, seed=107, spread=5.0, coupling=0.02)
    b = np.random.default_rng(108).standard_normal(12)
    keep = b.copy()
    leja_interpolate(dense_op(A), b, 1, 0.5, make_estimate(leftmost(A)), 1e-10, xi=xi)
    assert np.array_equal(b, keep)


# -------------------------------------------------------------------- KIOPS

def augmented_dense(sys):
    n, p = sys.n, sys.p
    return np.stack([augmented_apply(sys, e) for e in np.eye(n + p)], axis=1)


def test_augmented_matrix_exponential_identity():
    """test_kiops.py:27-38: the last column of exp(augmented matrix) holds
    sum_j phi_{j+1}(A) b_j."""
    A = stiff_matrix(7, seed=109, spread=5.0, coupling=0.1)
    rng = np.random.default_rng(110)
    cols = [rng.standard_normal(7) for _ in range(4)]
    sys = AugmentedSystem(dense_op(A), cols)
    w = scipy.linalg.expm(augmented_dense(sys))[:7, -1]
    expect = sum(dense_phi(j + 1, A) @ c for j, c in enumerate(cols))
    assert relerr(w, expect) <= 1e-12


def test_augmented_apply_wrong_length():
    """test_kiops.py:41-44."""
    sys = AugmentedSystem(MatrixFreeOperator(lambda v: 3.0 * v, 6), [np.ones(6), np.ones(6)])
    with pytest.raises(ValueError):
        augmented_apply(sys, np.ones(6))


def test_arnoldi_relation_and_window_orthogonality():
    """test_kiops.py:47-61: A V_m^T = V_{m+1}^T H to round-off, unit rows,
    neighbouring rows orthogonal under the iop_len = 2 window."""
    A = stiff_matrix(24, seed=111, spread=7.0, coupling=0.1)
    m = 9
    st = arnoldi_iop(lambda v: A @ v, np.random.default_rng(112).standard_normal(24), m,
                     iop_len=2)
    V = st.V[:m + 1]
    assert np.linalg.norm(A @ V[:m].T - V.T @ st.H[:m + 1, :m]) <= 1e-10 * np.linalg.norm(A)
    assert np.allclose(np.linalg.norm(V, axis=1), 1.0, atol=1e-12)
    for j in range(1, m):
        assert abs(V[j] @ V[j + 1]) < 1e-12


def test_arnoldi_zero_start():
    """test_kiops.py:64-66."""
    with pytest.raises(ValueError):
        arnoldi_iop(lambda v: 2.0 * v, np.zeros(7), 3)


@pytest.mark.parametrize("p", [1, 2, 4])
def test_kiops_eval_vs_dense(p):
    """test_kiops.py:69-81: sum_j phi_j(dt A) v_j within 1e-8 of the dense
    sum; matvecs and substeps positive."""
    A = stiff_matrix(30, seed=113, spread=35.0, coupling=0.08)
    rng = np.random.default_rng(114 + p)
    vecs = [rng.standard_normal(30) for _ in range(p + 1)]
    dt = 0.6
    w, stats = kiops_eval(dense_op(A), vecs, dt, tol=1e-10)
    expect = sum(dense_phi_action(j, dt * A, v) for j, v in enumerate(vecs))
    assert relerr(w, expect) <= 1e-8
    assert stats.matvecs > 0 and stats.substeps >= 1


def test_kiops_eval_dt_zero_returns_fresh_copy():
    """test_kiops.py:84-90."""
    v0 = np.linspace(1.0, 5.0, 5)
    w, stats = kiops_eval(MatrixFreeOperator(lambda v: -v, 5), [v0, np.ones(5)], 0.0,
                          tol=1e-8)
    assert np.array_equal(w, v0) and w is not v0
    assert stats.matvecs == 0


def test_kiops_eval_more_than_four_phi_vectors():
    """test_kiops.py:93-96: p > 4 is a ValueError."""
    with pytest.raises(ValueError):
        kiops_eval(MatrixFreeOperator(lambda v: -v, 4), [np.ones(4)] * 6, 0.2, tol=1e-8)


def test_kiops_several_output_times():
    """test_kiops.py:99-112: one output per tau, each the tau-scaled sum,
    within 1e-7."""
    A = stiff_matrix(20, seed=120, spread=14.0, coupling=0.06)
    rng = np.random.default_rng(121)
    vecs = [rng.standard_normal(20) for _ in range(3)]
    taus = (0.2, 0.45, 0.7, 1.0)
    ws, stats = kiops(dense_op(A), vecs, tau_out=taus, tol=1e-10)
    assert len(ws) == len(taus)
    for w, tau in zip(ws, taus):
        assert w.shape == (20,)
        expect = sum(tau ** j * dense_phi_action(j, tau * A, v) for j, v in enumerate(vecs))
        assert relerr(w, expect) <= 1e-7
    assert stats.substeps >= 1


@pytest.mark.parametrize("taus", [(1.0, 0.5), (-1.0,), (0.0, 1.0)])
def test_kiops_tau_out_must_be_positive_ascending(taus):
    """test_kiops.py:115-121."""
    with pytest.raises(ValueError):
        kiops(MatrixFreeOperator(lambda v: -v, 3), [np.ones(3), np.ones(3)], tau_out=taus)


def test_kiops_happy_breakdown_one_substep():
    """test_kiops.py:124-135: n + p below m_init makes the Krylov space
    exact; one substep, round-off accuracy."""
    A = stiff_matrix(5, seed=122, spread=2.5, coupling=0.1)
    v0, v1 = np.full(5, 0.5), np.arange(5.0) - 2.0
    w, stats = kiops_eval(dense_op(A), [v0, v1], 1.0, tol=1e-10)
    expect = dense_phi_action(0, A, v0) + dense_phi_action(1, A, v1)
    assert relerr(w, expect) <= 1e-11
    assert stats.substeps == 1


def test_kiops_single_vector_equals_zero_padded():
    """test_kiops.py:138-147."""
    A = stiff_matrix(11, seed=123, spread=6.0, coupling=0.1)
    v0 = np.random.default_rng(124).standard_normal(11)
    w1, _ = kiops(dense_op(A), [v0], tol=1e-10)
    w2, _ = kiops(dense_op(A), [v0, np.zeros(11)], tol=1e-10)
    assert np.allclose(w1[0], w2[0], atol=1e-12)


def test_kiops_matvecs_equal_operator_charges():
    """test_kiops.py:150-157 (matvecs == counter delta)."""
    A = stiff_matrix(14, seed=125, spread=45.0, coupling=0.05)
    op = dense_op(A)
    before = op.counter.count
    _, stats = kiops_eval(op, [np.ones(14), np.linspace(0, 1, 14)], 0.5, tol=1e-9)
    assert stats.matvecs == op.counter.count - before
    assert stats.m_last >= 1


# ----------------------------------------------------------------- spectrum

def diagonal(values):
    d = np.asarray(values, dtype=float)
    return MatrixFreeOperator(lambda v: d * v, len(d))


def test_power_iteration_finds_dominant_modulus():
    """test_spectrum.py:14-18."""
    lam, ok = power_iterate(diagonal([-45.0, -4.0, -1.0, -0.1]), tol_pi=1e-4, max_it=2000,
                            seed=0)
    assert ok and abs(lam) == pytest.approx(45.0, rel=1e-2)


def test_power_iteration_repeatable():
    """test_spectrum.py:21-25: same seed, same (lambda, converged)."""
    op = diagonal([-9.0, -3.0, -1.5])
    assert power_iterate(op, seed=7) == power_iterate(op, seed=7)


def test_power_iteration_zero_operator():
    """test_spectrum.py:28-31."""
    lam, ok = power_iterate(MatrixFreeOperator(lambda v: 0.0 * v, 6))
    assert lam == 0.0 and ok


def test_estimate_fields_and_gamma_floor():
    """test_spectrum.py:34-45."""
    est = make_estimate(-8.0, safety=1.25)
    assert (est.alpha, est.beta, est.c, est.gamma, est.age_steps) == \
        (pytest.approx(-10.0), 0.0, pytest.approx(-5.0), pytest.approx(2.5), 0)
    assert make_estimate(0.0).gamma == GAMMA_MIN


def test_refresh_policy_ages_recomputes_and_forces():
    """test_spectrum.py:48-80: a fresh estimate ages by one step; a stale,
    forced or missing one is recomputed from the operator."""
    op = diagonal([-60.0, -2.0])
    est = make_estimate(-6.0)
    aged = maybe_refresh(est, op, RefreshPolicy(n_recompute=50))
    assert aged.age_steps == 1 and aged.alpha == est.alpha
    stale = SpectrumEstimate(alpha=-2.0, beta=0.0, c=-1.0, gamma=0.5, safety=1.1,
                             age_steps=50)
    out = maybe_refresh(stale, op, RefreshPolicy(n_recompute=50))
    assert out.age_steps == 0 and abs(out.alpha) == pytest.approx(66.0, rel=5e-2)
    forced = maybe_refresh(est, op, RefreshPolicy(), force=True)
    assert forced.age_steps == 0 and abs(forced.alpha) > 60.0
    fresh = maybe_refresh(None, op, RefreshPolicy())
    assert fresh.age_steps == 0 and fresh.alpha < -60.0


# -------------------------------------------------------------- integrators

def two_dof_rhs():
    """A smooth nonlinear 2-dof ODE (not the reference's; same role)."""
    return CountingRhs(lambda u: np.array([-1.5 * u[0] + u[0] * u[1],
                                           -0.5 * u[1] - u[0] * u[0]]))


def engine_ctx(lam=-4.0):
    return EngineContext(est=make_estimate(lam), xi=ek.get_leja_points(400))


def test_order_tables():
    """test_integrators.py:30-36."""
    assert set(INTEGRATOR_ORDER) == set(INTEGRATORS) == set(EMBEDDED_ORDER)
    assert INTEGRATOR_ORDER["epirk5p1"] == 5 and INTEGRATOR_ORDER["exprb53s3"] == 5
    assert all(EMBEDDED_ORDER[k] < INTEGRATOR_ORDER[k] for k in INTEGRATORS)
    assert LEKRY_INTEGRATORS <= set(INTEGRATORS)


def test_remainder_properties():
    """test_integrators.py:39-59: zero at the linearisation point, ~0 for a
    linear RHS with its exact Jacobian, wrong length is ValueError."""
    rhs = two_dof_rhs()
    u = np.array([0.3, 0.8])
    sys = ek.make_linearized(rhs, u)
    assert np.array_equal(ek.remainder(sys, u), np.zeros(2))
    with pytest.raises(ValueError):
        ek.remainder(sys, np.ones(4))
    A = np.array([[-2.0, 0.5], [0.1, -1.0]])
    lin = ek.make_linearized(CountingRhs(lambda w: A @ w), np.array([0.5, -1.0]),
                             jac_factory=lambda w: (lambda v: A @ v))
    assert np.linalg.norm(ek.remainder(lin, np.array([2.0, 0.25]))) < 1e-13


@pytest.mark.parametrize("scheme", ["leja", "kiops"])
@pytest.mark.parametrize("name", INTEGRATORS)
def test_observed_order(name, scheme):
    """test_integrators.py:62-82: halving dt divides the global error by
    about 2^p."""
    rhs = two_dof_rhs()
    u0 = np.array([0.8, 0.6])
    T = 0.5
    ref = solve_ivp(lambda t, y: rhs.fn(y), (0.0, T), u0, method="DOP853", rtol=1e-13,
                    atol=1e-14).y[:, -1]
    errs = []
    for steps in (2, 4, 8):
        u = u0.copy()
        for _ in range(steps):
            u = ek.take_step(name, ek.make_linearized(rhs, u), T / steps, scheme, 1e-12,
                             engine_ctx()).u_high
        errs.append(np.linalg.norm(u - ref))
    rate = np.mean(np.log2(np.array(errs[:-1]) / np.array(errs[1:])))
    assert rate > INTEGRATOR_ORDER[name] - 0.7


@pytest.mark.parametrize("name", sorted(LEKRY_INTEGRATORS))
def test_all_routings_same_step(name):
    """test_integrators.py:85-98: leja, kiops and lekry agree on one step
    and on its error estimate."""
    u0 = np.array([0.7, -0.4])
    out = {s: ek.take_step(name, ek.make_linearized(two_dof_rhs(), u0), 0.04, s, 1e-13,
                           engine_ctx()) for s in SCHEMES}
    for s in ("leja", "lekry"):
        assert np.linalg.norm(out[s].u_high - out["kiops"].u_high) < 1e-10
        assert out[s].err_est == pytest.approx(out["kiops"].err_est, rel=1e-4, abs=1e-13)


def test_error_estimate_range():
    """test_integrators.py:101-105."""
    res = ek.take_step("exprb43", ek.make_linearized(two_dof_rhs(), np.array([0.8, 0.6])),
                       0.1, "kiops", 1e-12, engine_ctx(-30.0))
    assert 0.0 < res.err_est < 1e-4


@pytest.mark.parametrize("name,dt,scheme", [("rk45", 0.1, "leja"), ("exprb43", 0.1, "krylov"),
                                            ("exprb43", -0.1, "leja"),
                                            ("epirk5p1", 0.1, "lekry"),
                                            ("exprb43", 0.1, "lekry")])
def test_step_argument_errors(name, dt, scheme):
    """test_integrators.py:108-125: unknown integrator / scheme, negative
    dt, and LeKry outside its integrators are ValueError."""
    sys = ek.make_linearized(two_dof_rhs(), np.ones(2))
    with pytest.raises(ValueError):
        ek.take_step(name, sys, dt, scheme, 1e-8, engine_ctx())


@pytest.mark.parametrize("scheme", ["leja", "kiops"])
def test_group_charges_sum_to_counter(scheme):
    """test_integrators.py:128-150: per-group RHS charges add up to the
    counter; Leja internal-stage iterations never exceed the total."""
    rhs = two_dof_rhs()
    sys = ek.make_linearized(rhs, np.array([0.8, 0.6]))
    before = rhs.counter.count
    res = ek.take_step("epirk4s3", sys, 0.05, scheme, 1e-10, engine_ctx())
    assert sum(res.stats.group_rhs_evals.values()) == rhs.counter.count - before
    if scheme == "leja":
        assert 0 < res.stats.internal_stage_iters <= res.stats.leja_iters
    else:
        assert res.stats.krylov_matvecs > 0 and res.stats.substeps >= 1


# ------------------------------------------- the same contract, fused kernels

@pytest.mark.parametrize("mk", [lambda: ext.brusselator_periodic_problem(n=96),
                                lambda: ext.allen_cahn_periodic_problem(n=80)],
                         ids=["brusselator", "allen_cahn"])
def test_fused_vertical_equals_separate_calls(xi, mk):
    """test_leja.py:128-139 on the fused FD stencil path: the group's
    vectors equal the single calls within the FD tier (1e-7)
    and freeze in coefficient order."""
    prob = mk()
    rhs = ek.CountingRhs(prob.rhs)
    sys = ek.make_linearized(rhs, prob.u0)
    est = make_estimate(power_iterate(sys.J, seed=0)[0])
    coeffs = [1 / 3, 2 / 3, 1.0]
    b = sys.f_n
    res = leja_interpolate_vertical(sys.J, b, 1, coeffs, 2e-3, est, 1e-9, xi=xi)
    for ci, vec in zip(coeffs, res.vectors):
        single, _ = leja_interpolate(sys.J, b, 1, ci * 2e-3, est, 1e-9, xi=xi)
        assert relerr(vec, single) <= 1e-7
    assert res.freeze_iters == sorted(res.freeze_iters)


def test_fused_kiops_matvecs_equal_charges():
    """test_kiops.py:150-157 on the fused Arnoldi path. FD charges one RHS
    per matvec, except that a zero direction returns 0
    without an RHS call (integrators.py:88-91): with v_0 = 0 the first
    Krylov vector's state part is zero, so one matvec goes uncharged."""
    prob = ext.allen_cahn_periodic_problem(n=64)
    fu = prob.rhs(prob.u0)
    for v0, uncharged in ((1e-2 * prob.u0, 0), (np.zeros_like(fu), 1)):
        rhs = ek.CountingRhs(prob.rhs)
        sys = ek.make_linearized(rhs, prob.u0)
        before = rhs.counter.count
        _, stats = kiops_eval(sys.J, [v0, fu], 1e-3, tol=1e-9)
        assert stats.matvecs > 0
        assert rhs.counter.count - before == stats.matvecs - uncharged
