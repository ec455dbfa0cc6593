#!/usr/bin/env python
"""cProfile of the host side of the bench step (config 4, EPIRK5P1 Leja,
fixed dt): where the Python time of a step goes while the device works.

    python tools/step_profile.py [n] [steps]
"""
import cProfile
import pstats
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import ext, _device as D
import bench as B

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
prob = ext.brusselator_periodic_problem(n=n)
xi = ek.get_leja_points(400)
rhs = ek.CountingRhs(prob.rhs)
u = D.to_dev(prob.u0, copy=True)
sys0 = ek.make_linearized(rhs, u)
lam, _ = ek.power_iterate(sys0.J)
dt = B.DT_ALPHA / abs(ek.make_estimate(lam).alpha)
policy = ek.RefreshPolicy()
ctx = ek.EngineContext(xi=xi)


def step(u):
    s = ek.make_linearized(rhs, u, _as_numpy=False)
    ctx.est = ek.maybe_refresh(ctx.est, s.J, policy)
    return ek.take_step(B.INTEGRATOR, s, dt, "leja", B.TOL, ctx)._u


for _ in range(4):
    u = step(u)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(steps):
    u = step(u)
torch.cuda.synchronize()
print(f"{(time.perf_counter() - t0) / steps * 1e3:.3f} ms per step (wall)")
pr = cProfile.Profile()
pr.enable()
for _ in range(steps):
    u = step(u)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats(40)
