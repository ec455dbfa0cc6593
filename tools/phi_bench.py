#!/usr/bin/env python
"""Throughput window of SURVEY.md §8(d) d8b(i): long phi-calls at a
representative stiffness, dt |alpha| in {50, 300}, on the config-4 geometry
(FD Brusselator 4096^2 x 2) and the config-5 geometry (linear 3-D adv-diff
512^3), through the public API with device-resident vectors.

Per call: Leja phi_1 (k = 1) and a vertical group of k = 3 coefficients,
and KIOPS phi_1 (2-D only: its basis at 512^3 would hold ~100 GB). Reports
iterations / matvecs, ms per call, Jacobian actions per second and, for
Leja, the fused kernel's algorithmic GB/s and fraction of the measured HBM
peak over the call (SURVEY's bytes 8N(4 + 2 k_active) FD, 8N(2 + 2k) linear;
CUDA events around the launch batches, host waits excluded).

    python tools/phi_bench.py [--only 2d,3d] > profiles/r1c_phi_window.jsonl
"""

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="2d,3d")
    args = ap.parse_args()
    only = set(args.only.split(","))

    import torch
    import paper_2211_08948_b200 as ek
    from paper_2211_08948_b200 import ext, leja as L
    import bench as B

    peak, _ = B.peaks()
    xi = ek.get_leja_points(400)
    cases = []
    if "2d" in only:
        cases.append(("config4 brusselator_periodic 4096^2x2 FD", ext.brusselator_periodic_problem(n=4096)))
    if "3d" in only:
        cases.append(("config5 advdiff3d 512^3 linear", ext.advdiff3d_problem(n=512)))

    for name, prob in cases:
        rhs = ek.CountingRhs(prob.rhs)
        sys_ = ek.make_linearized(rhs, prob.u0, jac_factory=prob.jac_factory)
        lam, _ = ek.power_iterate(sys_.J)
        est = ek.make_estimate(lam)
        for da in (50.0, 300.0):
            dt = da / abs(est.alpha)
            b = ek.linalg.D.ev(ek.linalg.D.V(sys_._f) * dt)
            for coeffs in ([1.0], [1.0 / 3.0, 2.0 / 3.0, 1.0]):
                def call():
                    return ek.leja_interpolate_vertical(sys_.J, b, 1, coeffs, dt, est, 1e-10,
                                                        xi=xi)
                # warm-up: divided-difference tables, iterate buffers (deferred
                # accumulation allocates one per iteration) and the profiled path
                for _ in range(2):
                    call()
                L.PROFILE = []
                call()
                torch.cuda.synchronize()
                walls = []
                for _ in range(3):  # median of three timed calls
                    L.PROFILE = []
                    t0 = time.perf_counter()
                    r = call()
                    torch.cuda.synchronize()
                    walls.append(time.perf_counter() - t0)
                    prof, L.PROFILE = L.PROFILE, None
                wall = sorted(walls)[1]
                alg, _, launches = B.leja_bytes(prof[0])
                kt = sum(s.elapsed_time(e) for s, e in prof[0]["events"]) / 1e3
                print(json.dumps({
                    "case": name, "engine": "leja", "dt_alpha": da, "k": len(coeffs),
                    "iters": r.iters, "freeze_iters": r.freeze_iters,
                    "deferred": bool(prof[0].get("deferred")),
                    "ms_per_call": wall * 1e3, "jv_per_s": r.iters / wall,
                    "ms_per_call_reps": [round(w * 1e3, 3) for w in walls],
                    "kernel_ms": kt * 1e3, "alg_GBps": alg / kt / 1e9 if kt else None,
                    "frac_of_peak": alg / kt / 1e9 / peak if kt else None,
                    "peak_GBps": peak}), flush=True)
            if "brusselator" in name:
                def kcall():
                    return ek.kiops_eval(sys_.J, [None, b], dt, 1e-10)
                kcall()
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                _, st = kcall()
                torch.cuda.synchronize()
                wall = time.perf_counter() - t0
                print(json.dumps({
                    "case": name, "engine": "kiops", "dt_alpha": da, "matvecs": st.matvecs,
                    "substeps": st.substeps, "rejections": st.rejections,
                    "ms_per_call": wall * 1e3, "jv_per_s": st.matvecs / wall}), flush=True)
        del sys_, rhs, b
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
