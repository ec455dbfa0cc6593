#!/usr/bin/env python
"""One KIOPS call (kiops_eval, FD Jacobian) on config-4 geometry; used for
launch lists: ncu --metrics gpu__time_duration.sum python tools/kiops_bench.py"""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2211_08948_b200 as ek
    from paper_2211_08948_b200 import ext
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    prob = ext.brusselator_periodic_problem(n=n)
    rhs = ek.CountingRhs(prob.rhs)
    sys_ = ek.make_linearized(rhs, prob.u0)
    lam, _ = ek.power_iterate(sys_.J)
    est = ek.make_estimate(lam)
    dt = 50.0 / abs(est.alpha)
    b = ek.linalg.D.ev(ek.linalg.D.V(sys_._f) * dt)
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        w, st = ek.kiops_eval(sys_.J, [None, b], dt, 1e-10)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    print(json.dumps({"n": n, "ms": t * 1e3, "matvecs": st.matvecs, "substeps": st.substeps,
                      "rejections": st.rejections, "ms_per_matvec": t * 1e3 / max(1, st.matvecs)}))


if __name__ == "__main__":
    main()
