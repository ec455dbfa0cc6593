"""Pin the CPU oracle against the golden vectors of the real reference.

CPU-only. The golden fixtures (tests/golden/golden.npz) were produced by
tests/golden/make_golden.py importing the reference package; the oracle is a
restatement with the same op order, so every comparison here is BIT-EXACT:
vectors with np.array_equal, discrete counts with ==.
"""

import numpy as np
import pytest

from oracle import np_fields as F
from oracle import np_integrate as I
from oracle import np_phi as P

from conftest import cases

REF_PROBLEMS = {
    "adr": lambda: F.make("adr", alpha=0.1, n=16),
    "allen_cahn": lambda: F.make("allen_cahn", alpha=1e-2, n=16),
    "bruss_printed": lambda: F.brusselator(1e-3, 12, form="printed"),
    "bruss_standard": lambda: F.brusselator(0.02, 12, form="standard"),
    "gray_scott": lambda: F.make("gray_scott", alpha=1e-3, n=16),
    "semilinear": lambda: F.semilinear(20),
}

EXT_PROBLEMS = {
    "advdiff2d": lambda: F.advdiff2d(n=16, peclet=10.0),
    "allen_cahn_periodic": lambda: F.allen_cahn_periodic(n=16),
    "burgers2d": lambda: F.burgers2d(n=16),
    "brusselator_periodic": lambda: F.brusselator_periodic(n=16),
    "advdiff3d": lambda: F.advdiff3d(n=8),
}


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    assert a.shape == b.shape, (a.shape, b.shape)
    assert np.array_equal(a, b), float(np.max(np.abs(a - b)))


def test_leja_points_bitexact(golden):
    same(P.leja_points(400), golden["leja_points/xi"])


@pytest.mark.parametrize("name", list(REF_PROBLEMS))
def test_rhs_and_fd_jv_bitexact(golden, name):
    g = lambda k: golden[f"rhs/{name}/{k}"]  # noqa: E731
    p = REF_PROBLEMS[name]()
    same(p.u0, g("u0"))
    same(p.rhs(p.u0), g("f0"))
    same(p.rhs(g("u")), g("fu"))
    same(F.fd_jv(p.rhs, g("u"), g("v"), fu=g("fu")), g("jv"))
    if p.jac_factory is not None:
        same(p.jac_factory(g("u"))(g("v")), g("jac"))


def test_divided_differences_bitexact(golden, xi):
    for c in cases(golden, "dd"):
        g = lambda k: golden[f"dd/{c}/{k}"]  # noqa: E731
        est = P.estimate(float(g("lam")))
        same(P.newton_coeffs(int(g("l")), float(g("h")), est, xi, int(g("m"))),
             g("d"))


def test_leja_dense_bitexact(golden, xi):
    for c in cases(golden, "leja_dense"):
        g = lambda k: golden[f"leja_dense/{c}/{k}"]  # noqa: E731
        op = P.Operator.dense(g("A"))
        est = P.estimate(float(g("lam")))
        r = P.leja_vertical(op, g("b"), int(g("l")), list(g("coeffs")),
                            float(g("h")), est, float(g("tol")), xi)
        same(np.array(r.vectors), g("vectors"))
        assert r.iters == int(g("iters"))
        assert r.freeze_iters == list(g("freeze_iters"))
        assert op.counter.count == int(g("charges"))


def test_leja_stall_payload(golden, xi):
    A = golden["leja_stall/A"]
    op = P.Operator.dense(A)
    est = P.estimate(np.linalg.eigvals(A).real.min())
    with pytest.raises(P.NonConvergence) as exc:
        P.leja_vertical(op, np.ones(16), 1, [0.5, 1.0], 1.0, est, 1e-12, xi,
                        max_points=12)
    assert exc.value.iters == int(golden["leja_stall/iters"])
    assert exc.value.detail["stalled_coefficients"] == \
        list(golden["leja_stall/stalled"])


@pytest.mark.parametrize("name", ["allen_cahn", "bruss_standard",
                                  "gray_scott", "adr"])
def test_fd_engines_bitexact(golden, xi, name):
    g = lambda k: golden[f"fd/{name}/{k}"]  # noqa: E731
    p = REF_PROBLEMS[name]()
    rhs = P.CountedRhs(p.rhs)
    sys_ = I.linearize(rhs, p.u0)
    same(sys_.f_n, g("fu"))
    c0 = rhs.counter.count
    lam, conv = P.power_iterate(sys_.J)
    assert lam == float(g("lam")) and conv == bool(g("conv"))
    assert rhs.counter.count - c0 == int(g("pi_charges"))
    est = P.estimate(lam)
    dt = 20.0 / abs(est.alpha)
    assert dt == float(g("dt"))
    b = sys_.f_n * dt
    c1 = rhs.counter.count
    r = P.leja_vertical(sys_.J, b, 1, [0.25, 0.5, 1.0], dt, est, 1e-10, xi)
    same(np.array(r.vectors), g("leja"))
    assert r.iters == int(g("leja_iters"))
    assert r.freeze_iters == list(g("leja_freeze"))
    assert rhs.counter.count - c1 == int(g("leja_charges"))
    c2 = rhs.counter.count
    w, st = P.kiops_eval(sys_.J, [np.zeros_like(b), b, 0.1 * b], dt, 1e-10)
    same(w, g("kiops"))
    assert [st.substeps, st.rejections, st.matvecs, st.expms, st.m_last] == \
        list(g("kiops_stats"))
    assert st.err_sum == float(g("kiops_err_sum"))
    assert rhs.counter.count - c2 == int(g("kiops_charges"))
    ws, st2 = P.kiops(sys_.J.scaled(dt), [np.zeros_like(b), b],
                      tau_out=[0.25, 0.5, 1.0], tol=1e-10)
    same(np.array(ws), g("kvert"))
    assert [st2.substeps, st2.rejections, st2.matvecs, st2.expms,
            st2.m_last] == list(g("kvert_stats"))


def test_kiops_dense_bitexact(golden):
    for c in cases(golden, "kiops_dense"):
        g = lambda k: golden[f"kiops_dense/{c}/{k}"]  # noqa: E731
        op = P.Operator.dense(g("A"))
        vecs = list(g("vecs"))
        taus = tuple(g("taus"))
        if taus == (-1.0,):
            w, st = P.kiops_eval(op, vecs, float(g("dt")), float(g("tol")))
            ws = [w]
        else:
            ws, st = P.kiops(op, vecs, tau_out=taus, tol=float(g("tol")))
        same(np.array(ws), g("out"))
        assert [st.substeps, st.rejections, st.matvecs, st.expms,
                st.m_last] == list(g("stats"))
        assert op.counter.count == int(g("charges"))


STEP_CASES = [k[len("step/"):-len("/u_high")] for k in
              np.load(__import__("conftest").GOLDEN_PATH).files
              if k.startswith("step/") and k.endswith("/u_high")]


@pytest.mark.parametrize("case", STEP_CASES)
def test_take_step_bitexact(golden, xi, case):
    pname, integ, scheme = case.split("/")
    g = lambda k: golden[f"step/{case}/{k}"]  # noqa: E731
    p = REF_PROBLEMS[pname]()
    rhs = P.CountedRhs(p.rhs)
    sys_ = I.linearize(rhs, p.u0, jac_factory=p.jac_factory)
    lam, _ = P.power_iterate(sys_.J)
    assert lam == float(g("lam"))
    ctx = I.Ctx(est=P.estimate(lam), xi=xi)
    c0 = rhs.counter.count
    res = I.step(integ, sys_, float(g("dt")), scheme, 1e-8, ctx)
    same(res.u_high, g("u_high"))
    assert res.err_est == float(g("err"))
    st = res.stats
    assert [st.leja_iters, st.krylov_matvecs, st.substeps,
            st.internal_stage_iters] == list(g("counts"))
    assert rhs.counter.count - c0 == int(g("charges"))
    assert [f"{k}={v}" for k, v in sorted(st.group_rhs_evals.items())] == \
        list(g("groups"))


TRAJ_CASES = [k[len("traj/"):-len("/u")] for k in
              np.load(__import__("conftest").GOLDEN_PATH).files
              if k.startswith("traj/") and k.endswith("/u")]


@pytest.mark.parametrize("case", TRAJ_CASES)
def test_adaptive_trajectory_bitexact(golden, xi, case):
    pname, integ, scheme = case.split("/")
    g = lambda k: golden[f"traj/{case}/{k}"]  # noqa: E731
    p = REF_PROBLEMS[pname]()
    tr = I.adaptive(p.rhs, p.u0, p.t_final, integ, scheme, float(g("tol")),
                    jac_factory=p.jac_factory, ctx=I.Ctx(xi=xi),
                    max_steps=int(g("max_steps")))
    same(tr.u, g("u"))
    assert tr.t == float(g("t"))
    assert [tr.steps_accepted, tr.steps_rejected, tr.rhs_evals,
            tr.leja_iters, tr.krylov_matvecs, tr.substeps] == list(g("counts"))
    same(np.array(tr.dts), g("dts"))


@pytest.mark.parametrize("integ", ["epirk4s3", "epirk4s3a", "epirk5p1",
                                   "exprb43", "exprb53s3"])
def test_fixed_step_bitexact(golden, integ):
    p = REF_PROBLEMS["semilinear"]()
    u = I.fixed(p.rhs, p.u0, 1.0, 4, integ, "kiops", 1e-13,
                jac_factory=p.jac_factory)
    same(u, golden[f"fixed/semilinear/{integ}/u"])


@pytest.mark.parametrize("name", list(EXT_PROBLEMS))
def test_ext_problems_vs_reference_engines(golden, xi, name):
    """BASELINE plugins: the oracle's own engines/steppers reproduce the
    reference engines driven by the same NumPy RHS, bit for bit."""
    g = lambda k: golden[f"ext/{name}/{k}"]  # noqa: E731
    p = EXT_PROBLEMS[name]()
    same(p.u0, g("u0"))
    rhs = P.CountedRhs(p.rhs)
    sys_ = I.linearize(rhs, p.u0, jac_factory=p.jac_factory)
    same(sys_.f_n, g("f0"))
    lam, _ = P.power_iterate(sys_.J)
    assert lam == float(g("lam"))
    est = P.estimate(lam)
    dt = float(g("dt"))
    ctx = I.Ctx(est=est, xi=xi, engine_tol_factor=1.0)
    r2 = I.step("exprb2", sys_, dt, "leja", 1e-10, ctx)
    same(r2.u_high, g("exprb2"))
    assert r2.stats.leja_iters == int(g("iters"))
    r3 = I.step("exprb32", sys_, dt, "leja", 1e-10, ctx)
    same(r3.u_high, g("exprb32"))
    assert r3.err_est == float(g("exprb32_err"))


EXTTRAJ = [k[len("exttraj/"):-len("/u")] for k in
           np.load(__import__("conftest").GOLDEN_PATH).files
           if k.startswith("exttraj/") and k.endswith("/u")]


@pytest.mark.parametrize("case", EXTTRAJ)
def test_ext_trajectories_bitexact(golden, xi, case):
    name, integ, scheme = case.split("/")
    g = lambda k: golden[f"exttraj/{case}/{k}"]  # noqa: E731
    p = EXT_PROBLEMS[name]()
    tr = I.adaptive(p.rhs, p.u0, 1.0, integ, scheme, 1e-8,
                    jac_factory=p.jac_factory, ctx=I.Ctx(xi=xi), max_steps=10)
    same(tr.u, g("u"))
    assert [tr.steps_accepted, tr.steps_rejected, tr.rhs_evals,
            tr.leja_iters, tr.krylov_matvecs, tr.substeps] == list(g("counts"))
    same(np.array(tr.dts), g("dts"))
