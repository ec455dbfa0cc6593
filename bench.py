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
        k_act = sum(1 for f in freeze if f >= m)
        alg += per_vec * ((4 if prof["fd"] else 2) + 2 * k_act)
        pas += per_vec * ((3 if prof["fd"] else 2) + 2 * k_act)
        launches += 1
    return alg, pas, launches


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
        del c0
        return res._u

    u = u0
    for _ in range(args.warmup):
        u = step(u)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    counts["jv"] = 0
    L.PROFILE = []
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
    for p in prof:
        b, bp, l_ = leja_bytes(p)
        kb += b
        kp += bp
        kl += l_
        kt += sum(s.elapsed_time(e) for s, e in p["events"]) / 1e3
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
            "kernel": "k_march2d<PBruss<true>, EV_FD, EP_LEJA, K, S> for k >= 3 accumulators "
                      "(bulk-copy row march), k_tma2d<.., K, 4> (TMA 32x8 chunks) for k <= 2: "
                      "fused FD Jv + Leja recurrence + k accumulators + ||y||^2 + device "
                      "freeze test",
            "bytes_model": "algorithmic, SURVEY.md §8(d) d3: 8*N*(4+2*k_active) per launch "
                           "(reads u, f(u_n), y, p_1..k; writes y', p_1..k), N = 2*n^2",
            "achieved_pass_bytes": kp / kt / 1e9 if kt > 0 else None,
            "pass_bytes_model": "8*N*(3+2*k_active): the bytes this kernel moves (f(u_n) is "
                                "re-evaluated from the u neighbourhood instead of read)",
            "launches": kl, "avg_launch_ms": kt / kl * 1e3 if kl else None,
            "share_of_step": kt / elapsed if elapsed else None,
            "peak_source": f"MEASURED_PEAKS.json hbm_gbs ({peak_kind})"}

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
           "jv_per_step": total_jv / args.steps}

    if not args.no_e2e:
        out["e2e"] = e2e(args, ek, prob, dt, xi, world)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(n, dt)
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


# ------------------------------------------------------------ CPU side

def _oracle_setup(n):
    from oracle import np_fields as OF, np_integrate as OI, np_phi as OP
    q = OF.brusselator_periodic(n=n)
    rhs = OP.CountedRhs(q.rhs)
    sys_ = OI.linearize(rhs, q.u0)
    return OP, sys_, rhs


def _limit_threads(k):
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=k)
    except ImportError:
        import contextlib
        return contextlib.nullcontext()


def cpu_baseline(n, dt, iters=8):
    """The oracle (NumPy restatement of the reference, pinned bit-exact) on
    this host, 1 core: `iters` FD Leja iterations of the same workload."""
    with _limit_threads(1):
        OP, sys_, rhs = _oracle_setup(n)
        xi = OP.leja_points(400)
        # the GPU run's stiffness window: alpha = -50/dt
        est = OP.estimate(DT_ALPHA / dt / 1.1)
        b = sys_.f_n * dt
        c0 = rhs.counter.count
        t0 = time.perf_counter()
        try:
            OP.leja_vertical(sys_.J, b, 1, [1.0], dt, est, 1e-300, xi, max_points=iters + 1)
        except OP.NonConvergence:
            pass
        el = time.perf_counter() - t0
        jvs = rhs.counter.count - c0
    return {"value": jvs / el, "unit": "Jv/s", "cores": 1, "kind": "port",
            "sample": f"{jvs} FD Leja iterations (phi_1, k=1) of config 4 "
                      f"({n}x{n}x2) by oracle/np_phi.leja_vertical, 1 BLAS thread",
            "seconds": el, "host": _host_info()}


def _host_info():
    info = {"nproc": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu"] = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    import numpy
    import scipy
    info["numpy"] = numpy.__version__
    info["scipy"] = scipy.__version__
    return info


def run_reference(args, rank, world):
    """Reference arm: the reference's algorithm on the host CPU (oracle
    restatement), one FD Leja iteration per step, same config / metric."""
    if rank != 0:
        return None
    n = args.grid
    OP, sys_, rhs = _oracle_setup(n)
    xi = OP.leja_points(400)
    # the same stiffness window as our arm: dt |alpha| = 50 with alpha from a
    # short power iteration of the oracle
    lam, _ = OP.power_iterate(sys_.J, max_it=8)
    est = OP.estimate(lam)
    dt = DT_ALPHA / abs(est.alpha)
    b = sys_.f_n * dt
    if args.warmup > 0:
        try:
            OP.leja_vertical(sys_.J, b, 1, [1.0], dt, est, 1e-300, xi, max_points=2)
        except OP.NonConvergence:
            pass
    c0 = rhs.counter.count
    t0 = time.perf_counter()
    try:
        OP.leja_vertical(sys_.J, b, 1, [1.0], dt, est, 1e-300, xi,
                         max_points=args.steps + 1)
    except OP.NonConvergence:
        pass
    el = time.perf_counter() - t0
    jvs = rhs.counter.count - c0
    threads = int(os.environ.get("OPENBLAS_NUM_THREADS", os.cpu_count() or 1))
    val = jvs / el
    return {"impl": "reference", "metric": METRIC, "value": val, "unit": "Jv/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": el / max(jvs, 1) * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic: seeded smooth perturbation of the Brusselator steady state",
            "config": config_dict(n, dt, {"step": "one FD Leja iteration (bounded sample)"}),
            "cpu_baseline": {"value": val, "unit": "Jv/s", "cores": 1, "kind": "port",
                             "sample": f"{jvs} FD Leja iterations of config 4 by the "
                                       "NumPy oracle (numpy elementwise is single-"
                                       f"threaded; BLAS threads {threads})",
                             "host": _host_info()},
            "e2e": {"value": val, "unit": "Jv/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.impl == "reference":
        out = run_reference(args, rank, world)
    else:
        out = run_ours(args, rank, world, local)
    if rank == 0 and out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
