#!/usr/bin/env python
"""cProfile of a small-grid adaptive run (host-overhead analysis).

    python tools/host_profile.py [problem n integrator scheme steps]
"""
import cProfile, pstats, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import ext

a = sys.argv[1:]
name = a[0] if a else "allen_cahn_periodic"
n = int(a[1]) if len(a) > 1 else 256
integ = a[2] if len(a) > 2 else "exprb43"
scheme = a[3] if len(a) > 3 else "leja"
steps = int(a[4]) if len(a) > 4 else 100
p = ext.make_ext_problem(name, n=n)
xi = ek.get_leja_points(400)


def run():
    return ek.adaptive_loop(p.rhs, p.u0, 1.0, integ, scheme, 1e-10 if name != "burgers2d" else 1e-8,
                            jac_factory=p.jac_factory, ctx=ek.EngineContext(xi=xi),
                            max_steps=steps)


run()
t0 = time.perf_counter()
tr = run()
t1 = time.perf_counter()
print(f"{name} {n} {integ} {scheme}: {steps} steps in {t1 - t0:.3f} s "
      f"({(t1 - t0) / steps * 1e3:.2f} ms/step), rhs {tr.rhs_evals}, leja {tr.leja_iters}, "
      f"krylov {tr.krylov_matvecs}")
pr = cProfile.Profile()
pr.enable()
run()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
st.sort_stats("cumulative").print_stats(40)
