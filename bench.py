#!/usr/bin/env python
"""Benchmark of the phi-action hot path on B200 (BASELINE.json config 4).

Workload (N=1): the two-species periodic Brusselator on a 4096^2 grid per
species (N = 33,554,432 dofs, 268 MB per vector — every input is larger
than the 126 MB L2), FD Jacobian, EPIRK5P1 integrator with real-Leja
phi-actions at a fixed step dt = 50/|alpha| (dt |alpha| = 50, SURVEY.md
§8(d) d8b window (i)). One "step" = one fixed-step integrator step exactly
as `fixed_step_loop` runs it: linearise (1 RHS), `maybe_refresh` of the
spectrum estimate (power iteration every 50 steps), `take_step`
("epirk5p1", "leja"). EPIRK5P1 + LeKry is undefined in the reference
(integrators.py:247-251), so the Leja routing is used (deviation noted in
`config`).

metric: Jacobian actions (matvec-equivalents) per second = (Leja iterations
+ remainder FD Jvs + power-iteration Jvs) / wall time of the K timed steps,
timed with CUDA events on the launching stream; `ms_per_step` alongside.

Extra keys: `roofline` (fused Leja iteration kernel, algorithmic bytes
8N(4+2k_active) per launch over its CUDA-event time in the timed region),
`e2e` (same metric through the public API with host NumPy buffers, H2D of u
and D2H of u_high inside the timed region), `cpu_baseline` (the oracle on
this host's cores, bounded sample), `gpu_launches`, `clocks`.

`--impl reference` times the reference algorithm on the host CPU (the
NumPy oracle restatement in oracle/, pinned bit-exact to the reference), on
the same config and metric, one Leja iteration per step.
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_GRID = 4096
DT_ALPHA = 50.0
TOL = 1e-8
INTEGRATOR = "epirk5p1"
METRIC = ("Jv matvec-equivalents/s (EPIRK5P1 Leja step, periodic Brusselator "
          "4096^2 x 2 species, FD Jv)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--grid", type=int, default=N_GRID)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the other BASELINE configs (the 'configs' key)")
    ap.add_argument("--configs-budget", type=float, default=120.0)
    return ap.parse_args()


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def config_dict(n, dt, extra=None):
    d = {"workload": f"config4: brusselator_periodic {n}x{n}x2, EPIRK5P1 leja, FD Jv, "
                     f"fixed dt = {DT_ALPHA:g}/|alpha|, tol {TOL:g}",
         "grid": n, "species": 2, "dofs": 2 * n * n, "dt": dt, "dt_alpha": DT_ALPHA,
         "integrator": INTEGRATOR, "scheme": "leja", "jacobian": "fd", "tol": TOL,
         "l2": "inputs larger than L2 (268 MB per vector at 4096^2)",
         "deviation": "EPIRK5P1+LeKry is undefined in the reference "
                      "(integrators.py:247-251); the Leja routing is timed"}
    if extra:
        d.update(extra)
    return d


# ------------------------------------------------------------------ clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.path or not os.path.exists(self.path):
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                 "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


# -------------------------------------------------------------- our arm

def leja_bytes(prof):
    """Bytes of every fused Leja launch of one call, two models.

    algorithmic (the roofline contract): iteration m
    reads u, f(u_n), y and the k_active accumulators and writes y' and them,
    8 N (4 + 2 k_active(m)) with FD (8 N (2 + 2k) for a linear Jacobian);
    pass: what this implementation moves, 8 N (3 + 2 k_active(m)) with FD --
    the kernel re-evaluates f(u_n) from the u neighbourhood it reads anyway
    instead of streaming it."""
    n = prof["n"]
    per_vec = 8 * n
    alg, pas, launches = 0, 0, 0
    freeze = prof.get("freeze", [])
    for m in range(1, prof.get("iters", 0) + 1):
        # deferred accumulation (ek_leja_run_seq): the iteration moves no
        # accumulator; ek_leja_combine forms them afterwards (combine_bytes)
        k_act = 0 if prof.get("deferred") else sum(1 for f in freeze if f >= m)
        alg += per_vec * ((4 if prof["fd"] else 2) + 2 * k_act)
        # (the K = 0 FD iteration streams the stored f(u_n): it moves all 4)
        pas += per_vec * ((4 if prof.get("deferred") else 3) if prof["fd"] else 2) \
            + per_vec * 2 * k_act
        launches += 1
    return alg, pas, launches


def combine_bytes(prof):
    """Bytes of the deferred-accumulation pass of one call: it reads the
    iterates y_0 .. y_M once (M = the last iteration any accumulator took a
    term from) and writes the k accumulators."""
    if not prof.get("deferred") or not prof.get("iters"):
        return 0
    freeze = prof.get("freeze", [])
    last = max(freeze) if freeze else prof["iters"]
    return 8 * prof["n"] * (last + 1 + prof["k"])


def run_ours(args, rank, world, local):
    import torch
    import paper_2211_08948_b200 as ek
    from paper_2211_08948_b200 import ext, _native as N, _device as D
    from paper_2211_08948_b200 import leja as L

    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    n = args.grid
    prob = ext.brusselator_periodic_problem(n=n)
    if world > 1:
        # strong scaling: the global 4096^2 x 2 grid in row slabs, NCCL halos
        # and rank-ordered reductions (paper_2211_08948_b200/slab.py).
        # EK_BENCH_BACKEND=gloo exercises the same path host-staged (tests).
        import torch.distributed as dist
        from paper_2211_08948_b200 import slab as SL
        backend = os.environ.get("EK_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
        prob = SL.distribute(prob, SL.SlabComm())
    xi = ek.get_leja_points(400)
    rhs = ek.CountingRhs(prob.rhs)
    u0 = D.to_dev(prob.u0, copy=True)
    sys0 = ek.make_linearized(rhs, u0)
    lam, _ = ek.power_iterate(sys0.J)
    alpha = ek.make_estimate(lam).alpha
    dt = DT_ALPHA / abs(alpha)
    policy = ek.RefreshPolicy()
    ctx = ek.EngineContext(xi=xi)

    counts = {"jv": 0}

    def step(u):
        c0 = rhs.counter.count
        sys_ = ek.make_linearized(rhs, u, _as_numpy=False)
        c1 = rhs.counter.count
        ctx.est = ek.maybe_refresh(ctx.est, sys_.J, policy)
        c2 = rhs.counter.count
        res = ek.take_step(INTEGRATOR, sys_, dt, "leja", TOL, ctx)
        rem = res.stats.group_rhs_evals.get("remainder", 0)
        counts["jv"] += res.stats.leja_iters + (c2 - c1) + rem // 2
        counts["leja"] = counts.get("leja", 0) + res.stats.leja_iters
        del c0
        return res._u

    u = u0
    for _ in range(args.warmup):
        u = step(u)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    counts["jv"] = 0
    counts["leja"] = 0
    L.PROFILE = []
    from paper_2211_08948_b200 import integrators as I
    spec0 = dict(I.SPEC_STATS)
    launches0 = N.lib().ek_launch_count()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        e0.record()
        for _ in range(args.steps):
            u = step(u)
        e1.record()
        torch.cuda.synchronize()
    launches = N.lib().ek_launch_count() - launches0
    prof, L.PROFILE = L.PROFILE, None
    # graph mode: the library counts one launch per Leja graph; the kernels
    # its device-side loop ran are the call's iterations (calls with deferred
    # accumulation run sized launch batches, which the library counts itself)
    launches += sum(int(p.get("iters") or 0) for p in prof if p.get("graph"))
    elapsed = e0.elapsed_time(e1) / 1e3
    if world > 1:
        t = torch.tensor([elapsed], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed = float(t.item())
    # every Jacobian action is one global operation over all slabs (all ranks
    # count the same iterations), so the job total is rank 0's count
    total_jv = float(counts["jv"])

    # roofline of the fused Leja iteration kernel, live from the timed region
    kb, kp, kl, kt = 0, 0, 0, 0.0
    cb, cl, ct = 0, 0, 0.0  # the deferred-accumulation passes
    d3b = 0  # SURVEY d3's bytes of the same iterations with per-iteration accumulation
    deferred = any(p.get("deferred") for p in prof)
    for p in prof:
        d3b += leja_bytes({**p, "deferred": False})[0]
        b, bp, l_ = leja_bytes(p)
        kb += b
        kp += bp
        kl += l_
        kt += sum(s.elapsed_time(e) for s, e in p["events"]) / 1e3
        cev = p.get("combine_events") or []
        if cev and p.get("iters"):
            cb += combine_bytes(p)
            cl += len(cev)
            ct += sum(s.elapsed_time(e) for s, e in cev) / 1e3
    peak, peak_kind = peaks()
    achieved = kb / kt / 1e9 if kt > 0 else None
    traffic = None
    tp = ROOT / "profiles" / "leja_kernel_traffic.json"
    if tp.exists():
        try:
            traffic = json.loads(tp.read_text()).get("bytes_per_launch")
        except (ValueError, KeyError):
            traffic = None
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak if achieved else None, "traffic": traffic,
            "kernel": ("k_march2d<PBruss<true>, EV_FD, EP_LEJA, K = 0, S> (bulk-copy row march "
                       "with a producer warp): fused FD Jv + Leja recurrence + ||y||^2 + device "
                       "freeze test; the k accumulators are formed once per call by "
                       "k_leja_combine (deferred accumulation, see `combine`)") if deferred else
                      ("k_march2d<PBruss<true>, EV_FD, EP_LEJA, K, S> (bulk-copy row march "
                       "with a producer warp): fused FD Jv + Leja recurrence + k accumulators "
                       "+ ||y||^2 + device freeze test"),
            "bytes_model": ("algorithmic, SURVEY.md §8(d) d3 with k = 0: 8*N*4 per launch (reads "
                            "u, f(u_n), y; writes y'), N = 2*n^2 — the accumulator traffic "
                            "8*N*2*k_active per iteration of d3 is replaced by one pass per "
                            "call (`combine`)") if deferred else
                           ("algorithmic, SURVEY.md §8(d) d3: 8*N*(4+2*k_active) per launch "
                            "(reads u, f(u_n), y, p_1..k; writes y', p_1..k), N = 2*n^2"),
            "achieved_pass_bytes": kp / kt / 1e9 if kt > 0 else None,
            "frac_pass_bytes": kp / kt / 1e9 / peak if kt > 0 else None,
            "frac_note": ("deferred accumulation: the K = 0 iteration streams the stored f(u_n), "
                          "so the bytes it moves are SURVEY's algorithmic bytes with k = 0 and "
                          "frac_pass_bytes = frac") if deferred else
                         ("frac uses SURVEY's algorithmic bytes, which count a read of f(u_n) "
                          "that the fused pass replaces by re-evaluating f from the u "
                          "neighbourhood it reads anyway, so frac can exceed 1; "
                          "frac_pass_bytes is the fraction on the bytes the pass moves"),
            "pass_bytes_model": ("8*N*4: u, f(u_n), y read, y' written") if deferred else
                                ("8*N*(3+2*k_active): the bytes this kernel moves (f(u_n) is "
                                 "re-evaluated from the u neighbourhood instead of read)"),
            "launches": kl, "avg_launch_ms": kt / kl * 1e3 if kl else None,
            "share_of_step": kt / elapsed if elapsed else None,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"}
    if deferred:
        roof["deferred_accumulation"] = True
        roof["combine"] = {
            "kernel": "k_leja_combine: p_i = sum_m d_i[m] y_m per element in registers, "
                      "the reference's order and roundings",
            "bytes_model": "8*N*(M+1+k) per call: reads y_0..y_M, writes p_1..k",
            "launches": cl, "avg_launch_ms": ct / cl * 1e3 if cl else None,
            "achieved": cb / ct / 1e9 if ct > 0 else None,
            "frac": cb / ct / 1e9 / peak if ct > 0 else None,
            "share_of_step": ct / elapsed if elapsed else None}
        # the whole Leja work of the timed region (iterations + combine passes)
        # against the bytes SURVEY d3 assigns to the same iterations when every
        # iteration reads and writes its live accumulators (the reference's
        # formulation): > 1 means the path runs faster than that formulation's
        # HBM roofline
        roof["vs_d3_per_iteration_model"] = {
            "bytes": d3b, "ms": (kt + ct) * 1e3,
            "GBps": d3b / (kt + ct) / 1e9 if kt + ct > 0 else None,
            "frac": d3b / (kt + ct) / 1e9 / peak if kt + ct > 0 else None}

    out = {"metric": METRIC, "value": total_jv / elapsed, "unit": "Jv/s",
           "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": elapsed / args.steps * 1e3, "higher_is_better": True,
           "scaling": "strong", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic: seeded smooth perturbation of the Brusselator steady state",
           "config": config_dict(n, dt, {"parallelism": (
               f"slab{world} (row slabs; Leja passes store halo rows + partial sums into "
               "the peers' windows over NVLink (CUDA IPC), device-side pass flags and "
               "decisions, no NCCL per iteration; NCCL for once-per-call halos / sums)")
               if world > 1 else "single GPU"}),
           "roofline": roof, "gpu_launches": int(launches),
           "clocks": clk.summary(),
           "jv_per_step": total_jv / args.steps,
           "speculation": {"steps": I.SPEC_STATS["steps"] - spec0["steps"],
                           "misses": I.SPEC_STATS["misses"] - spec0["misses"],
                           "what": "phi-calls enqueued without a host sync, one sync per "
                                   "step; a miss recomputes the step synchronously"}}

    if not args.no_e2e:
        out["e2e"] = e2e(args, ek, prob, dt, xi, world)
    if world == 1 and not args.no_configs:
        del prob, u
        torch.cuda.empty_cache()
        out["configs"] = secondary_configs(ek, xi, budget_s=args.configs_budget)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(n, lam)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return out


def e2e(args, ek, prob, dt, xi, world=1):
    """Same metric through the public API with host buffers: each step takes
    the state from pinned host memory (H2D inside make_linearized) and
    returns u_high as a NumPy array (D2H). With N ranks every rank moves its
    own slab; the time is the max over ranks and the byte counts are the
    whole job's."""
    import numpy as np
    import torch
    rhs = ek.CountingRhs(prob.rhs)
    ctx = ek.EngineContext(xi=xi)
    policy = ek.RefreshPolicy()
    n_el = prob.u0.size
    pinned = torch.empty(n_el, dtype=torch.float64, pin_memory=True)
    u_host = pinned.numpy()
    u_host[:] = prob.u0
    jv = 0

    def step(u):
        nonlocal jv
        sys_ = ek.make_linearized(rhs, u)        # NumPy state in: host -> device
        c1 = rhs.counter.count
        ctx.est = ek.maybe_refresh(ctx.est, sys_.J, policy)
        c2 = rhs.counter.count
        res = ek.take_step(INTEGRATOR, sys_, dt, "leja", TOL, ctx)
        jv += res.stats.leja_iters + (c2 - c1) + res.stats.group_rhs_evals.get("remainder", 0) // 2
        return res.u_high                         # NumPy state out: device -> host

    u = u_host
    for _ in range(min(args.warmup, 2)):
        u = step(u)
    jv = 0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        u = step(u)
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([el], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        el = float(t.item())
    return {"value": jv / el, "unit": "Jv/s", "h2d_bytes_per_step": 8 * n_el * world,
            "d2h_bytes_per_step": 8 * n_el * world, "ms_per_step": el / args.steps * 1e3,
            "api": "make_linearized(rhs, numpy u) + maybe_refresh + take_step -> "
                   "StepResult.u_high (numpy)"}


# ------------------------------------------------- the other BASELINE configs

def secondary_configs(ek, xi, budget_s=120.0):
    """The other BASELINE.json configs, each timed on the device after one
    untimed run (wall clock around a synchronised run of the public API —
    small grids are host-latency bound, so the host time is the number),
    with the discrete counts. Config 5 also reports the fused 3-D Leja
    kernel's roofline fraction (linear Jv: 8N(2+2k_active) per launch,
    CUDA events). Skipped configs (budget) say so."""
    import torch
    from paper_2211_08948_b200 import ext
    from paper_2211_08948_b200 import leja as L
    t_start = time.perf_counter()
    out = {}

    def timed(run, reps=1):
        # two warm-up runs (the second one with cold divided-difference
        # tables, so the worker pool for tables beyond the first 32-point
        # chunk is up, a one-time process start), then the timed runs, again
        # with cold tables: the warm-up runs' tables (same dt sequence) must
        # not serve the timed window
        run()
        L._DD_CACHE.clear()
        run()
        torch.cuda.synchronize()
        L._DD_CACHE.clear()
        t0 = time.perf_counter()
        for _ in range(reps):
            r = run()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps, r

    def left():
        return budget_s - (time.perf_counter() - t_start)

    # config 1: adv-diff 64^2, one EXPRB2 Leja step at dt = 50 dt_CFL, Pe 1 and 10
    for pe in (1.0, 10.0):
        p = ext.advdiff2d_problem(n=64, peclet=pe)
        dt = 50.0 * p.params["dt_cfl"]
        t, _ = timed(lambda: ek.fixed_step_loop(p.rhs, p.u0, dt, 1, "exprb2", "leja", 1e-10,
                                                jac_factory=p.jac_factory,
                                                ctx=ek.EngineContext(xi=xi),
                                                stepper=ext.take_step_ext), reps=20)
        out[f"config1_pe{pe:g}"] = {
            "workload": "advdiff2d 64^2, one EXPRB2 Leja step, dt = 50 dt_CFL, tol 1e-10 "
                        "(NumPy in/out, includes linearisation + power iteration)",
            "us_per_call": t * 1e6}
    # config 2: Allen-Cahn 256^2 EXPRB43, 100 adaptive steps, Leja / KIOPS
    p = ext.allen_cahn_periodic_problem(n=256)
    for scheme in ("leja", "kiops"):
        t, tr = timed(lambda: ek.adaptive_loop(p.rhs, p.u0, 1.0, "exprb43", scheme, 1e-10,
                                               ctx=ek.EngineContext(xi=xi), max_steps=100))
        nst = tr.steps_accepted + tr.steps_rejected
        out[f"config2_{scheme}"] = {
            "workload": "allen_cahn_periodic 256^2, EXPRB43, FD Jv, tol 1e-10, 100 adaptive "
                        "steps from dt_init = 1e-5",
            "ms_per_step": t / nst * 1e3, "steps": nst, "t_reached": tr.t,
            "rhs_evals": tr.rhs_evals, "leja_iters": tr.leja_iters,
            "krylov_matvecs": tr.krylov_matvecs,
            "jv_per_s": (tr.leja_iters + tr.krylov_matvecs) / t}
    # config 3: Burgers 1024^2 EPIRK4s3, 20 adaptive steps, Leja / LeKry / KIOPS
    p = ext.burgers2d_problem(n=1024)
    for scheme in ("leja", "lekry", "kiops"):
        t, tr = timed(lambda: ek.adaptive_loop(p.rhs, p.u0, 1.0, "epirk4s3", scheme, 1e-8,
                                               jac_factory=p.jac_factory,
                                               ctx=ek.EngineContext(xi=xi), max_steps=20))
        nst = tr.steps_accepted + tr.steps_rejected
        out[f"config3_{scheme}"] = {
            "workload": "burgers2d 1024^2, EPIRK4s3, analytic Jv, tol 1e-8, 20 adaptive steps",
            "ms_per_step": t / nst * 1e3, "steps": nst, "t_reached": tr.t,
            "leja_iters": tr.leja_iters, "krylov_matvecs": tr.krylov_matvecs,
            "jv_per_s": (tr.leja_iters + tr.krylov_matvecs) / t}
    del p
    # config 4, window (ii) of SURVEY.md §8(d) d8b: 20 adaptive EPIRK5P1 Leja
    # steps from the reference's dt_init = 1e-5 t_final, tol 1e-8
    if left() > 30.0:
        p = ext.brusselator_periodic_problem(n=4096)
        u0 = torch.from_numpy(p.u0).cuda()
        t, tr = timed(lambda: ek.adaptive_loop(p.rhs, u0, 1.0, "epirk5p1", "leja", 1e-8,
                                               ctx=ek.EngineContext(xi=xi), max_steps=20))
        nst = tr.steps_accepted + tr.steps_rejected
        out["config4_adaptive_leja"] = {
            "workload": "brusselator_periodic 4096^2 x 2, EPIRK5P1 Leja, FD Jv, tol 1e-8, 20 "
                        "adaptive steps from dt_init = 1e-5 (window (ii); includes the "
                        "spectrum estimate and every divided-difference table)",
            "ms_per_step": t / nst * 1e3, "steps": nst, "t_reached": tr.t,
            "rhs_evals": tr.rhs_evals, "leja_iters": tr.leja_iters}
        del p, u0
        torch.cuda.empty_cache()
    # config 5: adv-diff 512^3, EXPRB32 Leja at fixed dt = 50 dt_CFL (3 steps)
    if left() < 20.0:
        out["config5"] = {"skipped": "bench configs time budget"}
        return out
    p = ext.advdiff3d_problem(n=512)
    u0 = torch.from_numpy(p.u0).cuda()
    dt = 50.0 * p.params["dt_cfl"]
    steps = 3
    rhs = ek.CountingRhs(p.rhs)
    sys0 = ek.make_linearized(rhs, u0, jac_factory=p.jac_factory, _as_numpy=False)
    est = ek.make_estimate(ek.power_iterate(sys0.J)[0])
    del sys0

    def run5():
        ctx = ek.EngineContext(xi=xi, est=est)
        u, it = u0, 0
        for _ in range(steps):
            s_ = ek.make_linearized(rhs, u, jac_factory=p.jac_factory, _as_numpy=False)
            ctx.est = ek.maybe_refresh(ctx.est, s_.J, ek.RefreshPolicy())
            r = ext.take_step_ext("exprb32", s_, dt, "leja", 1e-10, ctx)
            u, it = r._u, it + r.stats.leja_iters
        return it

    run5()
    torch.cuda.synchronize()
    L.PROFILE = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    iters = run5()
    e1.record()
    torch.cuda.synchronize()
    prof, L.PROFILE = L.PROFILE, None
    el = e0.elapsed_time(e1) / 1e3
    kb, kt = 0, 0.0
    for q in prof:
        kb += leja_bytes(q)[0]
        kt += sum(a.elapsed_time(b) for a, b in q["events"]) / 1e3
    peak, _ = peaks()
    out["config5"] = {
        "workload": "advdiff3d 512^3 (1.07 GB per vector), EXPRB32 Leja, linear analytic Jv, "
                    "fixed dt = 50 dt_CFL, tol 1e-10, 3 steps (estimate precomputed)",
        "ms_per_step": el / steps * 1e3, "leja_iters": iters,
        "jv_per_s": (iters + steps) / el,
        "leja_kernel": {"achieved_gbs": kb / kt / 1e9 if kt else None, "peak_gbs": peak,
                        "frac": kb / kt / 1e9 / peak if kt else None,
                        "bytes_model": "8*N*(2+2*k_active) per launch (linear Jv)",
                        "share_of_step": kt / el}}
    return out


# ------------------------------------------------------------ CPU side

def reference_engines():
    """The reference's own engines for the CPU legs: the unmodified
    reference package installed under baseline/_ref (pure Python; it
    travels with the repo snapshot, git-ignored) when present, else the
    NumPy restatement in oracle/ (pinned bit-exact to it). Returns
    (kind, namespace) with the engine calls the CPU legs need."""
    ref = ROOT / "baseline" / "_ref"
    if (ref / "expkit" / "integrators.py").exists():
        if str(ref) not in sys.path:
            sys.path.insert(0, str(ref))
        try:
            from expkit import integrators as RI, linalg as RL, spectrum as RS, leja as RLJ

            class NS:
                kind = "reference"
                source = "baseline/_ref (the unmodified reference package expkit)"
                CountingRhs = RL.CountingRhs
                make_estimate = RS.make_estimate
                leja_points = staticmethod(lambda: RLJ.get_leja_points(400))

                @staticmethod
                def linearize(rhs, u, jac_factory=None):
                    return RI.make_linearized(rhs, u, jac_factory=jac_factory)

                @staticmethod
                def step(name, sys_, dt, scheme, tol, est, xi):
                    return RI.take_step(name, sys_, dt, scheme, tol,
                                        RI.EngineContext(est=est, xi=xi))
            return NS
        except ImportError:
            pass
    from oracle import np_integrate as OI, np_phi as OP

    class NSP:
        kind = "port"
        source = "oracle/ (NumPy restatement of the reference, pinned bit-exact)"
        CountingRhs = OP.CountedRhs
        make_estimate = staticmethod(OP.estimate)
        leja_points = staticmethod(lambda: OP.leja_points(400))

        @staticmethod
        def linearize(rhs, u, jac_factory=None):
            return OI.linearize(rhs, u, jac_factory=jac_factory)

        @staticmethod
        def step(name, sys_, dt, scheme, tol, est, xi):
            return OI.step(name, sys_, dt, scheme, tol, OI.Ctx(est=est, xi=xi))
    return NSP


def _limit_threads(k):
    os.environ["OPENBLAS_NUM_THREADS"] = str(k)
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=k)
    except ImportError:
        import contextlib
        return contextlib.nullcontext()


def cpu_epirk5p1_steps(n, lam, steps, budget_s=None):
    """Full EPIRK5P1 Leja steps of config 4 by the reference engines on one
    host core (1 BLAS thread; numpy elementwise is single-threaded): the
    same problem (oracle/np_fields' restatement of the periodic Brusselator
    plugin, which the reference lacks), the same estimate and dt as the GPU
    arm (lam = its power-iteration |lambda|), the same tolerance. Returns
    (Jv, seconds, steps, kind, source). Linearisation of each step is timed
    (it is part of the step, as in fixed_step_loop)."""
    from oracle import np_fields as OF
    R = reference_engines()
    with _limit_threads(1):
        q = OF.brusselator_periodic(n=n)
        xi = R.leja_points()
        est = R.make_estimate(lam)
        dt = DT_ALPHA / abs(est.alpha)
        rhs = R.CountingRhs(q.rhs)
        u = q.u0
        jv, el, done = 0, 0.0, 0
        for _ in range(steps):
            t0 = time.perf_counter()
            sys_ = R.linearize(rhs, u)
            res = R.step(INTEGRATOR, sys_, dt, "leja", TOL, est, xi)
            el += time.perf_counter() - t0
            u = res.u_high
            jv += res.stats.leja_iters + res.stats.group_rhs_evals.get("remainder", 0) // 2
            done += 1
            if budget_s is not None and el > budget_s:
                break
    return jv, el, done, R.kind, R.source


def cpu_config5_jv(budget=1):
    """Per-Jv rate of config 5 (512^3 linear analytic Jacobian) by the
    oracle's plugin RHS on one core (per-Jv rate only)."""
    from oracle import np_fields as OF
    with _limit_threads(1):
        q = OF.advdiff3d(n=512)
        v = q.u0
        t0 = time.perf_counter()
        for _ in range(budget):
            v = q.rhs(v)
        el = time.perf_counter() - t0
    return budget / el


def cpu_baseline(n, lam, with_c5=True):
    """cpu_baseline of our arm: one full EPIRK5P1 step of the same workload
    by the reference engines on one host core (~20-30 s)."""
    jv, el, done, kind, source = cpu_epirk5p1_steps(n, lam, 1)
    out = {"value": jv / el, "unit": "Jv/s", "cores": 1, "kind": kind,
           "sample": f"{done} full EPIRK5P1 Leja step(s) of config 4 ({n}x{n}x2, dt|alpha| "
                     f"= {DT_ALPHA:g}, tol {TOL:g}; {jv} Jacobian actions) by {source}, "
                     "1 BLAS thread",
           "ms_per_step": el / done * 1e3, "seconds": el, "host": _host_info()}
    if with_c5:
        out["config5_jv_per_s"] = cpu_config5_jv()
    return out


def _host_info():
    info = {"nproc": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                info["lscpu_model"] = line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    import numpy
    import scipy
    info["numpy"] = numpy.__version__
    info["scipy"] = scipy.__version__
    try:
        from threadpoolctl import threadpool_info
        info["blas"] = [f"{d.get('internal_api')} {d.get('version')} "
                        f"({d.get('threading_layer')})" for d in threadpool_info()
                        if d.get("user_api") == "blas"]
    except ImportError:
        pass
    return info


def run_reference(args, rank, world):
    """Reference arm: the reference's engines (baseline/_ref, else the
    pinned port) on the host CPU, one core (1 BLAS thread),
    timing min(steps, 2) full EPIRK5P1 Leja steps of config 4 — the same
    step, metric and dt rule as our arm. dt comes from the reference's own
    power iteration of the same linearisation (untimed setup, as in our
    arm). Under torchrun only rank 0 runs."""
    if rank != 0:
        return None
    from oracle import np_fields as OF
    n = args.grid
    R = reference_engines()
    with _limit_threads(1):
        q = OF.brusselator_periodic(n=n)
        if R.kind == "reference":
            from expkit import spectrum as RS
            lam, _ = RS.power_iterate(R.linearize(R.CountingRhs(q.rhs), q.u0).J)
        else:
            from oracle import np_phi as OP
            lam, _ = OP.power_iterate(R.linearize(R.CountingRhs(q.rhs), q.u0).J)
        del q
    steps = max(1, min(args.steps, 2))
    jv, el, done, kind, source = cpu_epirk5p1_steps(n, lam, steps)
    val = jv / el
    dt = DT_ALPHA / abs(R.make_estimate(lam).alpha)
    return {"impl": "reference", "metric": METRIC, "value": val, "unit": "Jv/s",
            "n_gpus": world, "steps": done, "warmup": 0,
            "ms_per_step": el / done * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded smooth perturbation of the Brusselator steady state",
            "config": config_dict(n, dt, {
                "step": "one full EPIRK5P1 Leja step (linearise + take_step), as our arm",
                "timed_steps": f"min(--steps, 2) = {done} (CPU steps take ~20-30 s each); "
                               "no warm-up (NumPy has nothing to warm)"}),
            "cpu_baseline": {"value": val, "unit": "Jv/s", "cores": 1, "kind": kind,
                             "sample": f"{done} EPIRK5P1 steps ({jv} Jacobian actions) by "
                                       f"{source}; plugin RHS from oracle/np_fields; "
                                       "1 BLAS thread (numpy elementwise is single-threaded)",
                             "host": _host_info()},
            "e2e": {"value": val, "unit": "Jv/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def spawn(n):
    """`bench.py --gpus N` without a launcher: re-exec under
    torch.distributed.run with N ranks on this node (127.0.0.1), the same
    command form the driver uses; rank 0 prints the JSON line."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={n}", "--master-addr=127.0.0.1", f"--master-port={port}",
           str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn(args.gpus))
    rank, world, local = dist_env()
    if world != args.gpus and rank == 0:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; using {world} ranks",
              file=sys.stderr)
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        out = run_ours(args, rank, world, local)
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
