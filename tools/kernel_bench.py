#!/usr/bin/env python
"""Steady-state microbenchmark of the fused Leja iteration kernel.

Runs `--iters` Leja iterations that never freeze (tol = 1e-300) on the
periodic Brusselator (config 4 geometry) with the FD Jacobian, for k
accumulators, and reports per-launch time and achieved algorithmic HBM
bandwidth 8N(4+2k)/t. Used for ncu captures:

  ncu --set full -k regex:k_stencil2d -s 3 -c 2 python tools/kernel_bench.py --k 1
"""

import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=4096)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--problem", default="brusselator_periodic")
    ap.add_argument("--no-tma", action="store_true")
    ap.add_argument("--tma-mode", type=int, default=None,
                    help="2 row march (default), 1 32x8 chunks, 0 register-staged")
    ap.add_argument("--kiops", action="store_true")
    ap.add_argument("--reps", type=int, default=5, help="timed repetitions (median)")
    ap.add_argument("--defer", type=int, default=None,
                    help="1 / 0: force deferred accumulation on / off (default: the "
                         "library's own choice by size and group)")
    ap.add_argument("--repro", action="store_true",
                    help="order-independent sums (ek_set_repro): the RP = 1 kernel instances")
    args = ap.parse_args()

    import torch
    import paper_2211_08948_b200 as ek
    from paper_2211_08948_b200 import ext, leja as L, _native as NAT
    if args.repro:
        NAT.lib().ek_set_repro(1)
    if args.no_tma:
        NAT.lib().ek_set_tma(0)
    if args.tma_mode is not None:
        NAT.lib().ek_set_tma(args.tma_mode)

    if args.defer is not None:
        L._DEFER[0] = bool(args.defer)
        L._DEFER[1], L._DEFER[2], L._DEFER[4] = 0, 1, 1
    prob = ext.make_ext_problem(args.problem, n=args.n)
    rhs = ek.CountingRhs(prob.rhs)
    sys_ = ek.make_linearized(rhs, prob.u0, jac_factory=prob.jac_factory)
    lam, _ = ek.power_iterate(sys_.J)
    est = ek.make_estimate(lam)
    dt = 50.0 / abs(est.alpha)
    b = ek.linalg.D.ev(ek.linalg.D.V(sys_._f) * dt)
    coeffs = [1.0, 0.5, 0.25, 0.125][:args.k]
    xi = ek.get_leja_points(400)

    def run(iters):
        L.PROFILE = []
        try:
            ek.leja_interpolate_vertical(sys_.J, b, 1, coeffs, dt, est, 1e-300, xi=xi,
                                         max_points=iters + 1)
        except ek.NonConvergence:
            pass
        torch.cuda.synchronize()
        prof, L.PROFILE = L.PROFILE, None
        return prof

    for _ in range(3):  # warm-up: clocks up, tensor maps and DD tables cached
        run(args.iters)
    ts = []
    for _ in range(max(1, args.reps)):
        prof = run(args.iters)
        ts.append(sum(s.elapsed_time(e) for s, e in prof[0]["events"]) / 1e3)
    t = sorted(ts)[len(ts) // 2]
    n = sys_._u.numel()
    fd = prof[0]["fd"]
    lin = args.problem in ("advdiff2d", "advdiff3d")
    # algorithmic bytes: FD reads u, f(u_n), y; linear y;
    # state-dependent analytic (Burgers) u, y; + k accumulators read and
    # written, y' written. The FD pass itself re-evaluates f(u_n) (one vector less).
    base = 4 if fd else (2 if lin else 3)
    deferred = bool(prof[0].get("deferred"))
    # deferred accumulation: the iteration moves no accumulator (the call ends
    # by max_points here, so the combine pass is not part of this timing)
    per = 8 * n * (base + (0 if deferred else 2 * args.k))
    per_pass = per - (8 * n if fd else 0)
    out = {"problem": args.problem, "tma_mode": args.tma_mode, "repro": bool(args.repro),
           "n": args.n, "dofs": n, "k": args.k, "iters": args.iters, "deferred": deferred,
           "ms_per_launch": t / args.iters * 1e3, "bytes_per_launch": per,
           "GBps": per * args.iters / t / 1e9, "GBps_pass": per_pass * args.iters / t / 1e9,
           "ms_per_launch_reps": [round(x / args.iters * 1e3, 4) for x in ts]}
    print(json.dumps(out))
    if args.kiops:
        # KIOPS Arnoldi steps on the same operator: one substep of m steps
        K = ek
        vecs = [None, b]
        try:
            K.kiops(sys_.J.scaled(dt), vecs, tol=1e-300, m_init=4, m_min=4, m_max=4,
                    tau_min_frac=0.5)
        except ek.NonConvergence:
            pass
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        try:
            _, st = K.kiops(sys_.J.scaled(dt), vecs, tol=1e-300, m_init=args.iters,
                            m_min=args.iters, m_max=args.iters, tau_min_frac=0.5)
        except ek.NonConvergence as exc:
            st = None
            del exc
        e1.record()
        torch.cuda.synchronize()
        tk = e0.elapsed_time(e1) / 1e3
        # per Arnoldi step (FD, p_nz = 1): pass A 8N(5+1), B 8N*4, C 8N*2 (n+p ~ n)
        perk = 8 * n * ((3 if fd else (2 if lin else 3)) + 1 + 1 + 1 + 4 + 2)
        print(json.dumps({"kiops_steps": args.iters, "ms_per_arnoldi_step_incl_host":
                          tk / args.iters * 1e3, "bytes_per_step": perk,
                          "GBps_incl_host": perk * args.iters / tk / 1e9}))


if __name__ == "__main__":
    main()
