#!/usr/bin/env python
"""Device idle time inside the bench step (config 4, EPIRK5P1 Leja).

Runs the bench workload under torch.profiler (CUPTI kernel records) and
reports, over K steps: wall time, summed kernel time, the union of kernel
intervals (device busy) and the idle gaps between kernels, by size.
"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch
from torch.profiler import profile, ProfilerActivity
import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import ext, _device as D
import bench as B

prob = ext.brusselator_periodic_problem(n=4096)
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


for _ in range(3):
    u = step(u)
torch.cuda.synchronize()
if len(sys.argv) > 2 and sys.argv[2] == "cprof":
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(10):
        u = step(u)
    torch.cuda.synchronize()
    pr.disable()
    st = pstats.Stats(pr)
    st.sort_stats("tottime").print_stats(25)
    st.print_callers("read|synchronize|item|tolist")
    sys.exit(0)
K = int(sys.argv[1]) if len(sys.argv) > 1 else 5
if len(sys.argv) > 2 and sys.argv[2] == "nogc":
    import gc
    gc.disable()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(K):
        u = step(u)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
iv = sorted((e.time_range.start, e.time_range.end, e.name) for e in ev)
busy, gaps, cur_s, cur_e, prev = 0.0, [], None, None, ""
for s, e, name in iv:
    if cur_e is None:
        cur_s, cur_e = s, e
    elif s > cur_e:
        busy += cur_e - cur_s
        gaps.append((s - cur_e, name[:60] + "  after  " + prev[:60]))
        cur_s, cur_e = s, e
    else:
        cur_e = max(cur_e, e)
    prev = name
busy += cur_e - cur_s
span = iv[-1][1] - iv[0][0]
ktot = sum(e - s for s, e, _ in iv)
print(f"steps {K}: span {span/1e3:.3f} ms, busy {busy/1e3:.3f} ms ({busy/span:.1%}), "
      f"kernel sum {ktot/1e3:.3f} ms, {len(iv)} records, {len(gaps)} gaps")
gaps.sort(reverse=True)
tot = sum(g for g, _ in gaps)
print(f"idle {tot/1e3:.3f} ms = {tot/span:.1%} of span; per step {tot/K/1e3:.3f} ms")
for lim in (5, 20, 50, 100, 1000):
    sel = [g for g, _ in gaps if g >= lim]
    print(f"  gaps >= {lim:5d} us: {len(sel):4d}, {sum(sel)/1e3:.3f} ms")
for g, name in gaps[:12]:
    print(f"  {g:9.1f} us before {name[:90]}")
by = {}
for s, e, name in iv:
    key = name[:70]
    c, t = by.get(key, (0, 0.0))
    by[key] = (c + 1, t + (e - s))
print("device time by kernel (per step):")
for key, (c, t) in sorted(by.items(), key=lambda kv: -kv[1][1])[:16]:
    print(f"  {t / K / 1e3:8.3f} ms  {c / K:6.1f} x  {key}")
