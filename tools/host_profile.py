#!/usr/bin/env python
"""Host-side profile of a small-grid adaptive run (where the per-step time
goes when the device work is microseconds): cProfile of one run after a
warm-up, top functions by internal and cumulative time.

    python tools/host_profile.py c3_leja > hp.txt
"""

import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    which = sys.argv[1] if len(sys.argv) > 1 else "c3_leja"
    import torch
    import paper_2211_08948_b200 as ek
    from paper_2211_08948_b200 import ext
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
    from paper_2211_08948_b200 import leja as L
    run()
    torch.cuda.synchronize()
    L._DD_CACHE.clear()
    t0 = time.perf_counter()
    tr = run()
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    nst = tr.steps_accepted + tr.steps_rejected
    print(f"{which}: {nst} steps in {el:.4f} s ({el / nst * 1e3:.3f} ms/step), "
          f"leja {tr.leja_iters}, krylov {tr.krylov_matvecs}")
    L._DD_CACHE.clear()
    pr = cProfile.Profile()
    pr.enable()
    run()
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr, stream=sys.stdout)
    st.sort_stats("tottime").print_stats(35)
    st.sort_stats("cumulative").print_stats(45)


if __name__ == "__main__":
    main()
