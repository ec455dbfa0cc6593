#!/usr/bin/env python
"""All five BASELINE configs on one B200 (plus the CPU oracle where it
finishes in reasonable time): ms per step, Jacobian actions per second and
the discrete counts, one JSON line per run.

    python tools/configs_bench.py [--oracle] [--only c1,c2,...] > configs.jsonl

Timing: device-resident state, `torch.cuda.synchronize()` around each run,
wall clock of the public API (the adaptive / fixed-step loops are host
driven). Jv counts = Leja iterations + Krylov matvecs + RHS charges of
FD power iterations and remainders, as `bench.py` counts them.
"""

import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--oracle", action="store_true", help="also time the CPU oracle (configs 1-3)")
    ap.add_argument("--only", default="")
    args = ap.parse_args()
    only = set(filter(None, args.only.split(",")))

    import numpy as np
    import torch
    import paper_2211_08948_b200 as ek
    from paper_2211_08948_b200 import ext
    xi = ek.get_leja_points(400)

    def emit(d):
        print(json.dumps(d), flush=True)

    def sync():
        torch.cuda.synchronize()

    def oracle_adaptive(name, n, integ, scheme, tol, ms, jac):
        from oracle import np_fields as OF, np_integrate as OI, np_phi as OP
        q = getattr(OF, name)(n=n)
        t0 = time.perf_counter()
        tr = OI.adaptive(q.rhs, q.u0, 1.0, integ, scheme, tol,
                         jac_factory=q.jac_factory if jac else None,
                         ctx=OI.Ctx(xi=OP.leja_points(400)), max_steps=ms)
        return time.perf_counter() - t0, tr

    # ---- config 1: adv-diff 64^2, one EXPRB2 step, dt = 50 dt_CFL, Pe 1 / 10
    if not only or "c1" in only:
        for pe in (1.0, 10.0):
            p = ext.advdiff2d_problem(n=64, peclet=pe)
            dt = 50.0 * p.params["dt_cfl"]
            run = lambda: ek.fixed_step_loop(p.rhs, p.u0, dt, 1, "exprb2", "leja", 1e-10,
                                             jac_factory=p.jac_factory,
                                             ctx=ek.EngineContext(xi=xi),
                                             stepper=ext.take_step_ext)
            for _ in range(3):
                run()
            sync()
            reps = 20
            t0 = time.perf_counter()
            for _ in range(reps):
                run()
            sync()
            t = (time.perf_counter() - t0) / reps
            d = {"config": 1, "problem": "advdiff2d 64^2", "peclet": pe, "integrator": "exprb2",
                 "scheme": "leja", "ms_per_step_gpu": t * 1e3,
                 "note": "latency-bound (32 KB per vector): includes linearisation, power "
                         "iteration and divided differences on the host"}
            if args.oracle:
                from oracle import np_fields as OF, np_integrate as OI, np_phi as OP
                q = OF.advdiff2d(n=64, peclet=pe)
                t0 = time.perf_counter()
                rhs = OP.CountedRhs(q.rhs)
                sys_ = OI.linearize(rhs, q.u0, jac_factory=q.jac_factory)
                ctx = OI.Ctx(xi=OP.leja_points(400))
                ctx.est = OP.refresh(None, sys_.J, OP.Policy())
                OI.step("exprb2", sys_, dt, "leja", 1e-10, ctx)
                d["ms_per_step_oracle_1core"] = (time.perf_counter() - t0) * 1e3
            emit(d)

    # ---- config 2: Allen-Cahn 256^2, EXPRB43, 100 adaptive steps, leja / kiops
    if not only or "c2" in only:
        p = ext.allen_cahn_periodic_problem(n=256)
        for scheme in ("leja", "kiops"):
            run = lambda: ek.adaptive_loop(p.rhs, p.u0, 1.0, "exprb43", scheme, 1e-10,
                                           ctx=ek.EngineContext(xi=xi), max_steps=100)
            run()
            sync()
            t0 = time.perf_counter()
            tr = run()
            sync()
            t = time.perf_counter() - t0
            jv = tr.leja_iters + tr.krylov_matvecs
            d = {"config": 2, "problem": "allen_cahn_periodic 256^2", "integrator": "exprb43",
                 "scheme": scheme, "steps": tr.steps_accepted + tr.steps_rejected,
                 "accepted": tr.steps_accepted, "t_reached": tr.t, "rhs_evals": tr.rhs_evals,
                 "leja_iters": tr.leja_iters, "krylov_matvecs": tr.krylov_matvecs,
                 "s_gpu": t, "ms_per_step_gpu": t / max(1, tr.steps_accepted + tr.steps_rejected) * 1e3,
                 "jv_per_s_gpu": jv / t}
            if args.oracle:
                to, otr = oracle_adaptive("allen_cahn_periodic", 256, "exprb43", scheme, 1e-10,
                                          100, False)
                d["s_oracle_1core"] = to
                d["speedup_vs_oracle"] = to / t
                d["counts_match_oracle"] = [tr.steps_accepted, tr.rhs_evals, tr.leja_iters,
                                            tr.krylov_matvecs] == \
                    [otr.steps_accepted, otr.rhs_evals, otr.leja_iters, otr.krylov_matvecs]
            emit(d)

    # ---- config 3: Burgers 1024^2, EPIRK4s3, 20 adaptive steps, analytic Jv
    if not only or "c3" in only:
        p = ext.burgers2d_problem(n=1024)
        for scheme in ("leja", "lekry", "kiops"):
            run = lambda: ek.adaptive_loop(p.rhs, p.u0, 1.0, "epirk4s3", scheme, 1e-8,
                                           jac_factory=p.jac_factory,
                                           ctx=ek.EngineContext(xi=xi), max_steps=20)
            run()
            sync()
            t0 = time.perf_counter()
            tr = run()
            sync()
            t = time.perf_counter() - t0
            jv = tr.leja_iters + tr.krylov_matvecs
            d = {"config": 3, "problem": "burgers2d 1024^2", "integrator": "epirk4s3",
                 "scheme": scheme, "steps": tr.steps_accepted + tr.steps_rejected,
                 "t_reached": tr.t, "leja_iters": tr.leja_iters,
                 "krylov_matvecs": tr.krylov_matvecs, "s_gpu": t,
                 "ms_per_step_gpu": t / max(1, tr.steps_accepted + tr.steps_rejected) * 1e3,
                 "jv_per_s_gpu": jv / t}
            if args.oracle and scheme != "kiops":
                to, otr = oracle_adaptive("burgers2d", 1024, "epirk4s3", scheme, 1e-8, 20, True)
                d["s_oracle_1core"] = to
                d["speedup_vs_oracle"] = to / t
                d["counts_match_oracle"] = [tr.steps_accepted, tr.leja_iters,
                                            tr.krylov_matvecs] == \
                    [otr.steps_accepted, otr.leja_iters, otr.krylov_matvecs]
            emit(d)

    # ---- config 4: Brusselator 4096^2 x 2, EPIRK5P1 fixed dt = 50/|alpha|, leja / kiops
    if not only or "c4" in only:
        p = ext.brusselator_periodic_problem(n=4096)
        u0 = torch.from_numpy(p.u0).cuda()
        rhs0 = ek.CountingRhs(p.rhs)
        lam, _ = ek.power_iterate(ek.make_linearized(rhs0, u0).J)
        dt = 50.0 / abs(ek.make_estimate(lam).alpha)
        for scheme in ("leja", "kiops"):
            steps = 5
            run = lambda: ek.fixed_step_loop(p.rhs, u0, steps * dt, steps, "epirk5p1", scheme,
                                             1e-8, ctx=ek.EngineContext(xi=xi))
            run()
            sync()
            t0 = time.perf_counter()
            run()
            sync()
            t = time.perf_counter() - t0
            emit({"config": 4, "problem": "brusselator_periodic 4096^2 x 2",
                  "integrator": "epirk5p1", "scheme": scheme, "dt_alpha": 50.0,
                  "steps": steps, "ms_per_step_gpu": t / steps * 1e3,
                  "note": "includes the first step's power iteration (maybe_refresh)"})

        # window (ii) of SURVEY.md §8(d) d8b: 20 adaptive steps from the
        # reference's dt_init = 1e-5 t_final (t_final = 1), tol 1e-8
        for scheme in ("leja", "kiops"):
            run = lambda: ek.adaptive_loop(p.rhs, u0, 1.0, "epirk5p1", scheme, 1e-8,
                                           ctx=ek.EngineContext(xi=xi), max_steps=20)
            run()
            sync()
            t0 = time.perf_counter()
            tr = run()
            sync()
            t = time.perf_counter() - t0
            nst = tr.steps_accepted + tr.steps_rejected
            emit({"config": 4, "problem": "brusselator_periodic 4096^2 x 2",
                  "integrator": "epirk5p1", "scheme": scheme, "window": "adaptive",
                  "steps": nst, "accepted": tr.steps_accepted, "t_reached": tr.t,
                  "rhs_evals": tr.rhs_evals, "leja_iters": tr.leja_iters,
                  "krylov_matvecs": tr.krylov_matvecs, "ms_per_step_gpu": t / max(1, nst) * 1e3,
                  "note": "adaptive from dt_init = 1e-5 (tiny first steps: few Leja iterations "
                          "each); includes the spectrum estimate"})

    # ---- config 5: adv-diff 512^3, EXPRB32 Leja, fixed dt = 50 dt_CFL
    if not only or "c5" in only:
        p = ext.advdiff3d_problem(n=512)
        u0 = torch.from_numpy(p.u0).cuda()
        dt = 50.0 * p.params["dt_cfl"]
        steps = 3
        run = lambda: ek.fixed_step_loop(p.rhs, u0, steps * dt, steps, "exprb32", "leja", 1e-10,
                                         jac_factory=p.jac_factory,
                                         ctx=ek.EngineContext(xi=xi),
                                         stepper=ext.take_step_ext)
        run()
        sync()
        t0 = time.perf_counter()
        run()
        sync()
        t = time.perf_counter() - t0
        emit({"config": 5, "problem": "advdiff3d 512^3", "integrator": "exprb32",
              "scheme": "leja", "dt_cfl_mult": 50.0, "steps": steps,
              "ms_per_step_gpu": t / steps * 1e3,
              "note": "includes the first step's power iteration (maybe_refresh)"})
        # window (ii): 20 adaptive steps from dt_init = 1e-5 t_final, tol 1e-10
        run = lambda: ek.adaptive_loop(p.rhs, u0, 1.0, "exprb32", "leja", 1e-10,
                                       jac_factory=p.jac_factory,
                                       ctx=ek.EngineContext(xi=xi), max_steps=20,
                                       stepper=ext.take_step_ext,
                                       order=ext.EXT_ORDER["exprb32"])
        run()
        sync()
        t0 = time.perf_counter()
        tr = run()
        sync()
        t = time.perf_counter() - t0
        nst = tr.steps_accepted + tr.steps_rejected
        emit({"config": 5, "problem": "advdiff3d 512^3", "integrator": "exprb32",
              "scheme": "leja", "window": "adaptive", "steps": nst,
              "accepted": tr.steps_accepted, "t_reached": tr.t, "leja_iters": tr.leja_iters,
              "ms_per_step_gpu": t / max(1, nst) * 1e3,
              "note": "adaptive from dt_init = 1e-5; includes the spectrum estimate"})


if __name__ == "__main__":
    main()
