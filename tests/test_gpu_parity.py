"""GPU parity of the B200 path against the golden vectors of the reference
and against the CPU oracle run live on the same inputs.

Tiers:
  * discrete outputs (iters, freeze_iters, KIOPS stats, RHS charges,
    accepted-step counts) must be IDENTICAL;
  * stencil RHS values: bit-exact (1 ulp allowed where NumPy's pow(x, 3) is
    involved) — tolerance 1e-14 relative;
  * vectors through an FD Jacobian: <= 1e-7 relative (the FD quotient
    amplifies last-ulp norm differences by 1/eps ~ 1e8; intrinsic);
  * vectors through analytic / dense operators: <= 1e-12 relative.
"""

import numpy as np
import pytest
import torch

import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import ext, problems as P
from paper_2211_08948_b200 import _device as D, _native as N

from conftest import cases
from oracle import np_fields as OF, np_integrate as OI

pytestmark = pytest.mark.gpu

REF = {
    "adr": lambda: ek.make_problem("adr", alpha=0.1, n=16),
    "allen_cahn": lambda: ek.make_problem("allen_cahn", alpha=1e-2, n=16),
    "bruss_printed": lambda: P.brusselator_problem(1e-3, 12, form="printed"),
    "bruss_standard": lambda: P.brusselator_problem(0.02, 12, form="standard"),
    "gray_scott": lambda: ek.make_problem("gray_scott", alpha=1e-3, n=16),
    "semilinear": lambda: P.semilinear_problem(20),
}
EXT = {
    "advdiff2d": lambda: ext.advdiff2d_problem(n=16, peclet=10.0),
    "allen_cahn_periodic": lambda: ext.allen_cahn_periodic_problem(n=16),
    "burgers2d": lambda: ext.burgers2d_problem(n=16),
    "brusselator_periodic": lambda: ext.brusselator_periodic_problem(n=16),
    "advdiff3d": lambda: ext.advdiff3d_problem(n=8),
}


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    d = np.linalg.norm(a - b)
    s = np.linalg.norm(b)
    return d / s if s > 0 else d


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    N.lib()


# ----------------------------------------------------------------- stencils

@pytest.mark.parametrize("name", list(REF))
def test_rhs_matches_reference(golden, name):
    g = lambda k: golden[f"rhs/{name}/{k}"]  # noqa: E731
    p = REF[name]()
    assert rel(p.rhs(g("u0")), g("f0")) <= 1e-14
    assert rel(p.rhs(g("u")), g("fu")) <= 1e-14
    if name not in ("allen_cahn", "semilinear"):
        assert np.array_equal(p.rhs(g("u")), g("fu"))


@pytest.mark.parametrize("name", list(REF))
def test_fd_jv_kernel_same_eps_bitexact(golden, name):
    """The FD stencil kernel with the reference's own eps reproduces
    (f(u+eps v) - fu)/eps; bit-exact where no pow(x,3) is involved."""
    import math
    g = lambda k: golden[f"rhs/{name}/{k}"]  # noqa: E731
    p = REF[name]()
    u, v, fu = g("u"), g("v"), g("fu")
    eps = math.sqrt(ek.linalg.EPS) * (1.0 + np.linalg.norm(u)) / np.linalg.norm(v)
    ud, vd, fd = D.to_dev(u), D.to_dev(v), D.to_dev(fu)
    out = D.empty(len(u))
    N.check(N.lib().ek_jv(N.C.byref(p.rhs.grid), N.JAC_FD, N.C.c_void_p(ud.data_ptr()),
                          N.C.c_void_p(fd.data_ptr()), N.C.c_void_p(vd.data_ptr()), eps,
                          N.C.c_void_p(out.data_ptr()), None, None, None, D.stream()))
    got = out.cpu().numpy()
    if name in ("allen_cahn", "semilinear"):
        assert rel(got, g("jv")) <= 1e-7
    else:
        assert np.array_equal(got, g("jv"))


@pytest.mark.parametrize("name", list(REF))
def test_fd_jacobian_apply_public(golden, name):
    g = lambda k: golden[f"rhs/{name}/{k}"]  # noqa: E731
    p = REF[name]()
    rhs = ek.CountingRhs(p.rhs)
    out = ek.fd_jacobian_apply(rhs, g("u"), g("v"), fu=g("fu"))
    assert rhs.counter.count == 1
    assert isinstance(out, np.ndarray)
    assert rel(out, g("jv")) <= 1e-7


def test_semilinear_analytic_jacobian(golden):
    g = lambda k: golden[f"rhs/semilinear/{k}"]  # noqa: E731
    p = REF["semilinear"]()
    assert rel(p.jac_factory(g("u"))(g("v")), g("jac")) <= 1e-14


# -------------------------------------------------------------------- Leja

def test_divided_differences_host_bitexact(golden, xi):
    for c in cases(golden, "dd"):
        g = lambda k: golden[f"dd/{c}/{k}"]  # noqa: E731
        est = ek.make_estimate(float(g("lam")))
        d = ek.divided_differences(int(g("l")), float(g("h")), est, xi, int(g("m"))).d
        assert np.array_equal(d, g("d"))


def test_leja_dense_operator(golden, xi):
    for c in cases(golden, "leja_dense"):
        g = lambda k: golden[f"leja_dense/{c}/{k}"]  # noqa: E731
        op = ek.MatrixFreeOperator.from_matrix(g("A"))
        est = ek.make_estimate(float(g("lam")))
        r = ek.leja_interpolate_vertical(op, g("b"), int(g("l")), list(g("coeffs")),
                                         float(g("h")), est, float(g("tol")), xi=xi)
        assert r.iters == int(g("iters"))
        assert r.freeze_iters == list(g("freeze_iters"))
        assert op.counter.count == int(g("charges"))
        assert rel(np.array(r.vectors), g("vectors")) <= 1e-12


def test_leja_nonconvergence_payload(golden, xi):
    A = golden["leja_stall/A"]
    op = ek.MatrixFreeOperator.from_matrix(A)
    est = ek.make_estimate(np.linalg.eigvals(A).real.min())
    with pytest.raises(ek.NonConvergence) as exc:
        ek.leja_interpolate_vertical(op, np.ones(16), 1, [0.5, 1.0], 1.0, est, 1e-12,
                                     xi=xi, max_points=12)
    assert exc.value.iters == int(golden["leja_stall/iters"])
    assert exc.value.detail["stalled_coefficients"] == list(golden["leja_stall/stalled"])


@pytest.mark.parametrize("name", ["allen_cahn", "bruss_standard", "gray_scott", "adr"])
def test_fd_engines_fused(golden, xi, name):
    """Power iteration, vertical Leja and KIOPS on a native FD Jacobian:
    identical counts and charges, vectors within the FD tier."""
    g = lambda k: golden[f"fd/{name}/{k}"]  # noqa: E731
    p = REF[name]()
    rhs = ek.CountingRhs(p.rhs)
    sys_ = ek.make_linearized(rhs, p.u0)
    assert rel(sys_.f_n, g("fu")) <= 1e-14
    c0 = rhs.counter.count
    lam, conv = ek.power_iterate(sys_.J)
    assert conv == bool(g("conv"))
    assert rhs.counter.count - c0 == int(g("pi_charges"))
    assert abs(lam - float(g("lam"))) <= 1e-7 * abs(float(g("lam")))
    # drive the engines with the reference's own estimate and dt
    est = ek.make_estimate(float(g("lam")))
    dt = float(g("dt"))
    b = g("fu") * dt
    c1 = rhs.counter.count
    r = ek.leja_interpolate_vertical(sys_.J, b, 1, [0.25, 0.5, 1.0], dt, est, 1e-10, xi=xi)
    assert r.iters == int(g("leja_iters"))
    assert r.freeze_iters == list(g("leja_freeze"))
    assert rhs.counter.count - c1 == int(g("leja_charges"))
    assert rel(np.array(r.vectors), g("leja")) <= 1e-7
    c2 = rhs.counter.count
    w, st = ek.kiops_eval(sys_.J, [np.zeros_like(b), b, 0.1 * b], dt, 1e-10)
    assert [st.substeps, st.rejections, st.matvecs, st.expms, st.m_last] == \
        list(g("kiops_stats"))
    assert rhs.counter.count - c2 == int(g("kiops_charges"))
    assert rel(w, g("kiops")) <= 1e-7
    ws, st2 = ek.kiops(sys_.J.scaled(dt), [np.zeros_like(b), b], tau_out=[0.25, 0.5, 1.0],
                       tol=1e-10)
    assert [st2.substeps, st2.rejections, st2.matvecs, st2.expms, st2.m_last] == \
        list(g("kvert_stats"))
    assert rel(np.array(ws), g("kvert")) <= 1e-7


def test_kiops_dense(golden):
    for c in cases(golden, "kiops_dense"):
        g = lambda k: golden[f"kiops_dense/{c}/{k}"]  # noqa: E731
        op = ek.MatrixFreeOperator.from_matrix(g("A"))
        vecs = list(g("vecs"))
        taus = tuple(g("taus"))
        if taus == (-1.0,):
            w, st = ek.kiops_eval(op, vecs, float(g("dt")), float(g("tol")))
            ws = [w]
        else:
            ws, st = ek.kiops(op, vecs, tau_out=taus, tol=float(g("tol")))
        assert [st.substeps, st.rejections, st.matvecs, st.expms, st.m_last] == \
            list(g("stats")), c
        assert op.counter.count == int(g("charges"))
        assert rel(np.array(ws), g("out")) <= 1e-11


# ------------------------------------------------------------------ steppers

STEP_CASES = [k[len("step/"):-len("/u_high")] for k in
              np.load(__import__("conftest").GOLDEN_PATH).files
              if k.startswith("step/") and k.endswith("/u_high")]


@pytest.mark.parametrize("case", STEP_CASES)
def test_take_step(golden, xi, case):
    pname, integ, scheme = case.split("/")
    g = lambda k: golden[f"step/{case}/{k}"]  # noqa: E731
    p = REF[pname]()
    rhs = ek.CountingRhs(p.rhs)
    sys_ = ek.make_linearized(rhs, p.u0, jac_factory=p.jac_factory)
    ctx = ek.EngineContext(est=ek.make_estimate(float(g("lam"))), xi=xi)
    c0 = rhs.counter.count
    res = ek.take_step(integ, sys_, float(g("dt")), scheme, 1e-8, ctx)
    st = res.stats
    assert [st.leja_iters, st.krylov_matvecs, st.substeps, st.internal_stage_iters] == \
        list(g("counts"))
    assert rhs.counter.count - c0 == int(g("charges"))
    assert [f"{k}={v}" for k, v in sorted(st.group_rhs_evals.items())] == list(g("groups"))
    tolv = 1e-13 if pname == "semilinear" else 1e-9
    assert rel(res.u_high, g("u_high")) <= tolv
    assert res.err_est == pytest.approx(float(g("err")), rel=1e-3, abs=1e-14)


TRAJ = [k[len("traj/"):-len("/u")] for k in
        np.load(__import__("conftest").GOLDEN_PATH).files
        if k.startswith("traj/") and k.endswith("/u")]


@pytest.mark.parametrize("case", TRAJ)
def test_adaptive_trajectory(golden, xi, case):
    pname, integ, scheme = case.split("/")
    g = lambda k: golden[f"traj/{case}/{k}"]  # noqa: E731
    p = REF[pname]()
    tr = ek.adaptive_loop(p.rhs, p.u0, p.t_final, integ, scheme, float(g("tol")),
                          jac_factory=p.jac_factory, ctx=ek.EngineContext(xi=xi),
                          max_steps=int(g("max_steps")))
    counts = [tr.steps_accepted, tr.steps_rejected, tr.rhs_evals, tr.leja_iters,
              tr.krylov_matvecs, tr.substeps]
    same = counts == list(g("counts")) and len(tr.dts) == len(g("dts"))
    if same:
        d_dts = rel(np.array(tr.dts), g("dts"))
        d_u = rel(tr.u, g("u"))
        if d_dts <= 1e-8 and d_u <= 1e-10:
            return  # tier T3: identical decisions, <= 1e-10 solution
    assert "kiops" in scheme or scheme == "lekry", "Leja runs must meet tier T3"
    # KIOPS adaptivity (ceil/log decisions, kiops.py:212-252) amplifies ulp
    # differences; the contract is then the oracle's own sensitivity
    # envelope: rerun the oracle with its norms perturbed by one ulp.
    env = _oracle_envelope(pname, integ, scheme, float(g("tol")), int(g("max_steps")), xi)
    base = list(g("counts"))
    for i, c in enumerate(counts):
        lo = min([base[i]] + [e[0][i] for e in env])
        hi = max([base[i]] + [e[0][i] for e in env])
        assert lo <= c <= hi, (i, c, lo, hi)
    env_u = max(rel(e[1], g("u")) for e in env)
    assert rel(tr.u, g("u")) <= max(10.0 * env_u, 1e-10), (rel(tr.u, g("u")), env_u)


ORACLE = {
    "adr": lambda: OF.make("adr", alpha=0.1, n=16),
    "allen_cahn": lambda: OF.make("allen_cahn", alpha=1e-2, n=16),
    "bruss_printed": lambda: OF.brusselator(1e-3, 12, form="printed"),
    "bruss_standard": lambda: OF.brusselator(0.02, 12, form="standard"),
    "gray_scott": lambda: OF.make("gray_scott", alpha=1e-3, n=16),
    "semilinear": lambda: OF.semilinear(20),
}


def _oracle_envelope(pname, integ, scheme, tol, max_steps, xi):
    """Oracle runs with every np.linalg.norm scaled by 1 +- 1 ulp
    (SURVEY.md Appendix B): [(counts, u), ...]."""
    def run():
        p = ORACLE[pname]()
        r = OI.adaptive(p.rhs, p.u0, p.t_final, integ, scheme, tol,
                        jac_factory=p.jac_factory, ctx=OI.Ctx(xi=xi),
                        max_steps=max_steps)
        return ([r.steps_accepted, r.steps_rejected, r.rhs_evals, r.leja_iters,
                 r.krylov_matvecs, r.substeps], r.u)
    out = []
    real = np.linalg.norm
    for f in (1.0 + 2.0**-52, 1.0 - 2.0**-53, 1.0 + 2.0**-51, 1.0 - 2.0**-52):
        np.linalg.norm = lambda *a, f=f, **k: real(*a, **k) * f
        try:
            out.append(run())
        finally:
            np.linalg.norm = real
    return out


@pytest.mark.parametrize("name", list(EXT))
def test_ext_problem_steps(golden, xi, name):
    g = lambda k: golden[f"ext/{name}/{k}"]  # noqa: E731
    p = EXT[name]()
    assert np.array_equal(p.u0, g("u0"))
    rhs = ek.CountingRhs(p.rhs)
    sys_ = ek.make_linearized(rhs, p.u0, jac_factory=p.jac_factory)
    assert rel(sys_.f_n, g("f0")) <= 1e-14
    est = ek.make_estimate(float(g("lam")))
    ctx = ek.EngineContext(est=est, xi=xi, engine_tol_factor=1.0)
    dt = float(g("dt"))
    r2 = ext.take_step_ext("exprb2", sys_, dt, "leja", 1e-10, ctx)
    assert r2.stats.leja_iters == int(g("iters"))
    tolv = 1e-7 if p.jac_factory is None else 1e-12
    assert rel(r2.u_high, g("exprb2")) <= tolv
    r3 = ext.take_step_ext("exprb32", sys_, dt, "leja", 1e-10, ctx)
    assert rel(r3.u_high, g("exprb32")) <= tolv


@pytest.mark.parametrize("integ", ["epirk5p1", "exprb43"])
@pytest.mark.parametrize("name,state", [("brusselator_periodic", (1.0, 3.0)),
                                        ("allen_cahn_periodic", (1.0,))])
def test_zero_direction_stage_remainders(xi, integ, name, state):
    """Steps from an exact steady state (f(u_n) = 0): every stage equals u_n,
    so each fused remainder takes the k == u_n branch (R = 0, no RHS charge,
    integrators.py:104-105) — decided on the device by
    ek_remainder_combo_dev and charged at the next host sync. Counts, groups
    and the result must match the oracle's step exactly."""
    n = 16
    p = getattr(ext, f"{name}_problem")(n=n)
    q = getattr(OF, name)(n=n)
    u = np.concatenate([np.full(n * n, v) for v in state])
    rhs = ek.CountingRhs(p.rhs)
    sys_ = ek.make_linearized(rhs, u)
    assert not np.any(sys_.f_n)
    from oracle import np_phi as OP
    orhs = OP.CountedRhs(q.rhs)
    osys = OI.linearize(orhs, u)
    lam, _ = ek.power_iterate(ek.make_linearized(ek.CountingRhs(p.rhs), p.u0).J)
    est = ek.make_estimate(lam)
    dt = 10.0 / abs(est.alpha)
    c0, o0 = rhs.counter.count, orhs.counter.count
    st = ek.take_step(integ, sys_, dt, "leja", 1e-8, ek.EngineContext(est=est, xi=xi))
    ost = OI.step(integ, osys, dt, "leja", 1e-8, OI.Ctx(est=est, xi=xi))
    assert rhs.counter.count - c0 == orhs.counter.count - o0
    assert st.stats.leja_iters == ost.stats.leja_iters
    assert dict(st.stats.group_rhs_evals) == dict(ost.stats.group_rhs_evals)
    assert np.array_equal(st.u_high, ost.u_high)
    assert st.err_est == ost.err_est
