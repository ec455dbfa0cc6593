#!/usr/bin/env python
"""Light-weight wall-clock attribution of a small-grid adaptive run (cProfile
inflates cheap calls): wraps the main host entry points with perf_counter
timers (inclusive times) and prints ms per step for each.

    python tools/host_timers.py c3_leja
"""

import sys
import time
from collections import defaultdict
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c3_leja"
    import torch
    import paper_2211_08948_b200 as ek
    from paper_2211_08948_b200 import ext, leja as L, integrators as I, _device as D
    from paper_2211_08948_b200 import timestep as T, _dense, spectrum as S
    acc = defaultdict(float)
    cnt = defaultdict(int)

    def wrap(mod, name, label=None):
        f = getattr(mod, name)
        label = label or f"{mod.__name__.split('.')[-1]}.{name}"

        def g(*a, **k):
            t0 = time.perf_counter()
            try:
                return f(*a, **k)
            finally:
                acc[label] += time.perf_counter() - t0
                cnt[label] += 1
        setattr(mod, name, g)

    wrap(L, "leja_interpolate_vertical")
    wrap(L, "_dd_group")
    wrap(I, "_remainder_dev")
    wrap(D, "evaluate")
    wrap(D, "flush_checks")
    wrap(I, "make_linearized")
    wrap(T, "make_linearized", "timestep.make_linearized")
    wrap(T, "maybe_refresh", "timestep.maybe_refresh")
    wrap(T, "take_step", "timestep.take_step")
    xi = ek.get_leja_points(400)
    cfg, scheme = which.split("_")
    if cfg == "c2":
        p = ext.allen_cahn_periodic_problem(n=256)
        run = lambda: ek.adaptive_loop(p.rhs, p.u0, 1.0, "exprb43", scheme, 1e-10,
                                       ctx=ek.EngineContext(xi=xi), max_steps=100)
    else:
        p = ext.burgers2d_problem(n=1024)
        run = lambda: ek.adaptive_loop(p.rhs, p.u0, 1.0, "epirk4s3", scheme, 1e-8,
                                       jac_factory=p.jac_factory,
                                       ctx=ek.EngineContext(xi=xi), max_steps=20)
    run()
    L._DD_CACHE.clear()
    run()
    torch.cuda.synchronize()
    L._DD_CACHE.clear()
    acc.clear()
    cnt.clear()
    t0 = time.perf_counter()
    tr = run()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    nst = tr.steps_accepted + tr.steps_rejected
    print(f"{which}: {el / nst * 1e3:.3f} ms/step over {nst} steps")
    for k, v in sorted(acc.items(), key=lambda kv: -kv[1]):
        print(f"  {v / nst * 1e3:8.3f} ms/step  {cnt[k] / nst:6.2f} calls/step  "
              f"{v / max(1, cnt[k]) * 1e6:8.1f} us/call  {k}")


if __name__ == "__main__":
    main()
