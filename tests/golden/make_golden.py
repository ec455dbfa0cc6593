"""Generate the golden fixtures that pin the oracle (and the GPU path).

Run ONLY in the build container, where the read-only reference exists:

    PYTHONPATH=/root/reference/pkg/src OPENBLAS_NUM_THREADS=1 \
        python tests/golden/make_golden.py

It imports the reference package `expkit` (arXiv 2211.08948 reference,
`/root/reference/pkg/src/expkit`) and records, for small seeded cases, the
outputs of the reference's own functions:

  * problem RHS / FD Jacobian action / analytic Jacobian (problems.py,
    linalg.py:111-129)
  * Leja points (leja.py:32-50), divided differences (leja.py:88-111)
  * vertical Leja interpolation incl. iters / freeze_iters / RHS charges
    (leja.py:133-189)
  * KIOPS outputs and KiopsStats (kiops.py:106-303)
  * power iteration (spectrum.py:43-63)
  * one take_step per integrator x scheme (integrators.py:258-433)
  * short adaptive_loop trajectories (timestep.py:84-164)
  * BASELINE plugin problems (not in the reference): the REFERENCE engines
    driven by the oracle's NumPy right-hand sides (oracle/np_fields.py).

Output: tests/golden/golden.npz (keys "<case>/<field>").
"""

import os
import sys
import tempfile
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REPO = HERE.parents[1]
sys.path.insert(0, str(REPO))
os.environ.setdefault("XDG_CACHE_HOME", tempfile.mkdtemp())

import expkit  # noqa: E402  (the reference; PYTHONPATH must point at it)
from expkit import integrators as R_int  # noqa: E402
R_kiops = sys.modules["expkit.kiops"]  # the module, not the function
from expkit import leja as R_leja  # noqa: E402
from expkit import linalg as R_lin  # noqa: E402
from expkit import problems as R_prob  # noqa: E402
from expkit import spectrum as R_spec  # noqa: E402
from expkit import timestep as R_ts  # noqa: E402

from oracle import np_fields as O_f  # noqa: E402

assert "reference" in expkit.__file__, expkit.__file__

OUT = {}


def put(case, **fields):
    for k, v in fields.items():
        OUT[f"{case}/{k}"] = np.asarray(v)


def stable(n, seed, radius):
    rng = np.random.default_rng(seed)
    A = -np.diag(np.linspace(0.2, radius, n))
    A += 0.05 * radius / n * rng.standard_normal((n, n))
    return A


def main():
    xi = R_leja.generate_leja_points(400)
    put("leja_points", xi=xi)

    # ------------------------------------------------------------ stencils
    rng = np.random.default_rng(1234)
    probs = {
        "adr": R_prob.make_problem("adr", alpha=0.1, n=16),
        "allen_cahn": R_prob.make_problem("allen_cahn", alpha=1e-2, n=16),
        "bruss_printed": R_prob.brusselator_problem(1e-3, 12, form="printed"),
        "bruss_standard": R_prob.brusselator_problem(0.02, 12, form="standard"),
        "gray_scott": R_prob.make_problem("gray_scott", alpha=1e-3, n=16),
        "semilinear": R_prob.semilinear_problem(20),
    }
    for name, p in probs.items():
        u = p.u0 + 0.05 * rng.standard_normal(p.u0.shape)
        v = rng.standard_normal(p.u0.shape)
        fu = p.rhs(u)
        jv = R_lin.fd_jacobian_apply(p.rhs, u, v, fu=fu)
        put(f"rhs/{name}", u0=p.u0, f0=p.rhs(p.u0), u=u, v=v, fu=fu, jv=jv)
        if p.jac_factory is not None:
            put(f"rhs/{name}", jac=p.jac_factory(u)(v))

    # ------------------------------------------------ divided differences
    for i, (l, h, lam, m) in enumerate([(0, 1.0, -4.0, 32), (1, 0.9, -8.0, 32),
                                        (3, 2.5, -30.0, 64), (4, 0.1, -300.0, 96),
                                        (1, 50.0, -1.0, 128), (2, 7.0, -11.0, 32)]):
        est = R_spec.make_estimate(lam)
        d = R_leja.divided_differences(l, h, est, xi, m).d
        put(f"dd/{i}", l=l, h=h, lam=lam, m=m, d=d)

    # ------------------------------------------------------- Leja (dense)
    cases = [(30, 7, 20.0, 0, [1.0], 0.4, 1e-12),
             (30, 7, 20.0, 1, [1.0], 0.4, 1e-12),
             (24, 11, 20.0, 1, [1.0 / 9.0, 1.0 / 8.0, 1.0], 0.5, 1e-12),
             (30, 7, 20.0, 3, [0.5, 1.0], 0.4, 1e-10),
             (30, 7, 200.0, 4, [1.0], 0.7, 1e-11)]
    for i, (n, seed, rad, l, coeffs, h, tol) in enumerate(cases):
        A = stable(n, seed, rad)
        b = np.random.default_rng(seed + 1).standard_normal(n)
        op = R_lin.MatrixFreeOperator.from_matrix(A)
        est = R_spec.make_estimate(np.linalg.eigvals(A).real.min())
        res = R_leja.leja_interpolate_vertical(op, b, l, coeffs, h, est, tol,
                                               xi=xi)
        put(f"leja_dense/{i}", A=A, b=b, l=l, coeffs=coeffs, h=h, tol=tol,
            lam=np.linalg.eigvals(A).real.min(), vectors=np.array(res.vectors),
            iters=res.iters, freeze_iters=res.freeze_iters,
            charges=op.counter.count)

    # non-convergence payload (test_leja.py:155-165 style)
    A = stable(16, 5, 400.0)
    op = R_lin.MatrixFreeOperator.from_matrix(A)
    est = R_spec.make_estimate(np.linalg.eigvals(A).real.min())
    try:
        R_leja.leja_interpolate_vertical(op, np.ones(16), 1, [0.5, 1.0], 1.0,
                                         est, 1e-12, xi=xi, max_points=12)
        raise SystemExit("expected NonConvergence")
    except expkit.NonConvergence as exc:
        put("leja_stall", A=A, iters=exc.iters,
            stalled=exc.detail["stalled_coefficients"])

    # ------------------------------------------------ Leja / KIOPS on FD J
    for name in ("allen_cahn", "bruss_standard", "gray_scott", "adr"):
        p = probs[name]
        rhs = R_lin.CountingRhs(p.rhs)
        sys_ = R_int.make_linearized(rhs, p.u0)
        c0 = rhs.counter.count
        lam, conv = R_spec.power_iterate(sys_.J)
        c1 = rhs.counter.count
        est = R_spec.make_estimate(lam)
        dt = 20.0 / abs(est.alpha)
        b = sys_.f_n * dt
        res = R_leja.leja_interpolate_vertical(sys_.J, b, 1, [0.25, 0.5, 1.0],
                                               dt, est, 1e-10, xi=xi)
        c2 = rhs.counter.count
        w, st = R_kiops.kiops_eval(sys_.J, [np.zeros_like(b), b, 0.1 * b], dt,
                                   1e-10)
        c3 = rhs.counter.count
        ws, st2 = R_kiops.kiops(sys_.J.scaled(dt), [np.zeros_like(b), b],
                                tau_out=[0.25, 0.5, 1.0], tol=1e-10)
        put(f"fd/{name}", u=p.u0, fu=sys_.f_n, lam=lam, conv=conv,
            pi_charges=c1 - c0, dt=dt, leja=np.array(res.vectors),
            leja_iters=res.iters, leja_freeze=res.freeze_iters,
            leja_charges=c2 - c1, kiops=w,
            kiops_stats=[st.substeps, st.rejections, st.matvecs, st.expms,
                         st.m_last], kiops_err_sum=st.err_sum,
            kiops_charges=c3 - c2, kvert=np.array(ws),
            kvert_stats=[st2.substeps, st2.rejections, st2.matvecs,
                         st2.expms, st2.m_last])

    # ------------------------------------------------------ KIOPS (dense)
    kcases = [(25, 5, 30.0, 4, 0.7, 1e-10, None),
              (18, 7, 12.0, 3, 1.0, 1e-10, (0.25, 0.5, 1.0)),
              (4, 9, 2.0, 2, 1.0, 1e-10, None),
              (12, 12, 40.0, 2, 0.5, 1e-9, None),
              (40, 3, 400.0, 5, 1.0, 1e-12, None)]
    for i, (n, seed, rad, nv, dt, tol, taus) in enumerate(kcases):
        rng = np.random.default_rng(seed)
        A = -np.diag(np.linspace(0.3, rad, n)) + 0.1 * rng.standard_normal((n, n))
        vecs = [rng.standard_normal(n) for _ in range(nv)]
        op = R_lin.MatrixFreeOperator.from_matrix(A)
        if taus is None:
            w, st = R_kiops.kiops_eval(op, vecs, dt, tol)
            ws = [w]
        else:
            ws, st = R_kiops.kiops(op, vecs, tau_out=taus, tol=tol)
        put(f"kiops_dense/{i}", A=A, vecs=np.array(vecs), dt=dt, tol=tol,
            taus=(-1.0,) if taus is None else taus, out=np.array(ws),
            stats=[st.substeps, st.rejections, st.matvecs, st.expms, st.m_last],
            err_sum=st.err_sum, charges=op.counter.count)

    # ------------------------------------------------ one step per scheme
    for pname in ("bruss_standard", "semilinear", "allen_cahn"):
        p = probs[pname]
        for integ in R_int.INTEGRATORS:
            for scheme in R_int.SCHEMES:
                if scheme == "lekry" and integ not in R_int.LEKRY_INTEGRATORS:
                    continue
                rhs = R_lin.CountingRhs(p.rhs)
                sys_ = R_int.make_linearized(rhs, p.u0,
                                             jac_factory=p.jac_factory)
                lam, _ = R_spec.power_iterate(sys_.J)
                ctx = R_int.EngineContext(est=R_spec.make_estimate(lam), xi=xi)
                dt = 5.0 / abs(ctx.est.alpha) if pname != "semilinear" else 0.05
                c0 = rhs.counter.count
                res = R_int.take_step(integ, sys_, dt, scheme, 1e-8, ctx)
                st = res.stats
                put(f"step/{pname}/{integ}/{scheme}", u=p.u0, dt=dt,
                    lam=lam, u_high=res.u_high, err=res.err_est,
                    counts=[st.leja_iters, st.krylov_matvecs, st.substeps,
                            st.internal_stage_iters],
                    charges=rhs.counter.count - c0,
                    groups=sorted(st.group_rhs_evals.items()) and
                    [f"{k}={v}" for k, v in sorted(st.group_rhs_evals.items())])

    # ------------------------------------------------ adaptive trajectories
    runs = [("allen_cahn", "exprb43", "leja", 1e-6, 25),
            ("allen_cahn", "exprb43", "kiops", 1e-6, 25),
            ("bruss_standard", "epirk5p1", "leja", 1e-6, 15),
            ("bruss_standard", "epirk4s3", "lekry", 1e-6, 15),
            ("semilinear", "exprb43", "kiops", 1e-6, 400),
            ("semilinear", "epirk4s3", "lekry", 1e-6, 400),
            ("gray_scott", "exprb53s3", "leja", 1e-5, 12)]
    for pname, integ, scheme, tol, nmax in runs:
        p = probs[pname]
        ctx = R_int.EngineContext(xi=xi)
        tr = R_ts.adaptive_loop(p.rhs, p.u0, p.t_final, integ, scheme, tol,
                                jac_factory=p.jac_factory, ctx=ctx,
                                max_steps=nmax)
        put(f"traj/{pname}/{integ}/{scheme}", tol=tol, max_steps=nmax,
            u=tr.u, t=tr.t,
            counts=[tr.steps_accepted, tr.steps_rejected, tr.rhs_evals,
                    tr.leja_iters, tr.krylov_matvecs, tr.substeps],
            dts=tr.dts)

    # fixed-step loop (criterion 4 style)
    p = probs["semilinear"]
    for integ in R_int.INTEGRATORS:
        u = R_ts.fixed_step_loop(p.rhs, p.u0, 1.0, 4, integ, "kiops", 1e-13,
                                 jac_factory=p.jac_factory)
        put(f"fixed/semilinear/{integ}", u=u)

    # ------------------------- BASELINE plugins: reference engines + NumPy RHS
    ext = {
        "advdiff2d": O_f.advdiff2d(n=16, peclet=10.0),
        "allen_cahn_periodic": O_f.allen_cahn_periodic(n=16),
        "burgers2d": O_f.burgers2d(n=16),
        "brusselator_periodic": O_f.brusselator_periodic(n=16),
        "advdiff3d": O_f.advdiff3d(n=8),
    }
    for name, p in ext.items():
        rhs = R_lin.CountingRhs(p.rhs)
        sys_ = R_int.make_linearized(rhs, p.u0, jac_factory=p.jac_factory)
        lam, conv = R_spec.power_iterate(sys_.J)
        est = R_spec.make_estimate(lam)
        dt = p.params["dt_cfl"] * 50.0 if "dt_cfl" in p.params else \
            10.0 / abs(est.alpha)
        b = sys_.f_n * dt
        phi1, iters = R_leja.leja_interpolate(sys_.J, b, 1, dt, est, 1e-10,
                                              xi=xi)
        put(f"ext/{name}", u0=p.u0, f0=sys_.f_n, lam=lam, dt=dt,
            exprb2=p.u0 + phi1, iters=iters, charges=rhs.counter.count)
        # EXPRB32 one step from reference pieces
        a = p.u0 + phi1
        Ra = R_int.remainder(sys_, a)
        t3, it3 = R_leja.leja_interpolate(sys_.J, (2.0 * Ra) * dt, 3, dt, est,
                                          1e-10, xi=xi)
        put(f"ext/{name}", exprb32=a + t3,
            exprb32_err=np.linalg.norm((a + t3) - a), iters3=it3)
    for name, integ, scheme in (("allen_cahn_periodic", "exprb43", "leja"),
                                ("allen_cahn_periodic", "exprb43", "kiops"),
                                ("burgers2d", "epirk4s3", "lekry"),
                                ("brusselator_periodic", "epirk5p1", "leja")):
        p = ext[name]
        tr = R_ts.adaptive_loop(p.rhs, p.u0, 1.0, integ, scheme, 1e-8,
                                jac_factory=p.jac_factory,
                                ctx=R_int.EngineContext(xi=xi), max_steps=10)
        put(f"exttraj/{name}/{integ}/{scheme}", u=tr.u, t=tr.t,
            counts=[tr.steps_accepted, tr.steps_rejected, tr.rhs_evals,
                    tr.leja_iters, tr.krylov_matvecs, tr.substeps],
            dts=tr.dts)

    out = HERE / "golden.npz"
    np.savez_compressed(out, **OUT)
    print(f"wrote {len(OUT)} arrays to {out} ({out.stat().st_size} bytes)")


if __name__ == "__main__":
    main()
