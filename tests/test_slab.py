"""Slab decomposition (multi-GPU path).

CPU (gloo, world size 2): halo exchange for periodic and Neumann grids,
rank-ordered sums, scatter / gather — the host logic of the N > 1 path.
GPU: the slab code path at P = 1 reproduces the single-GPU path bit for bit,
and two ranks sharing one GPU through host-staged gloo exchanges (no kernel
waits on another rank's kernel) reproduce the single-GPU Leja / power
iteration / EPIRK5P1 results with identical decisions.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2211_08948_b200 import _native as N
from paper_2211_08948_b200 import slab as S
from paper_2211_08948_b200.problems import make_grid


@pytest.fixture(autouse=True)
def _restore_repro():
    """`slab.distribute` switches the order-independent sums on for the
    process; leave the default for the other test modules."""
    yield
    try:
        N.lib().ek_set_repro(0)
    except RuntimeError:
        pass


def _repro(on):
    from paper_2211_08948_b200 import _device as D
    return D.set_reproducible(on)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _cpu_worker(rank, world, port, q):
    _init(rank, world, port)
    try:
        comm = S.SlabComm()
        out = {}
        for bc in (N.BC_PERIODIC, N.BC_NEUMANN):
            for ncomp in (1, 2):
                n = 8
                g = make_grid(N.P_BRUSS_STANDARD if ncomp == 2 else N.P_ALLEN_CAHN, bc, 2,
                              ncomp, n, 1.0 / n)
                glob = np.arange(ncomp * n * n, dtype=np.float64) * 1.5 + 7.0
                loc = torch.from_numpy(comm.scatter(glob, g))
                gl = S.slab_grid(g, comm)
                halo = torch.zeros(2 * ncomp * n, dtype=torch.float64)
                comm.exchange(loc, gl, halo)
                out[(bc, ncomp)] = (int(gl.row0), int(gl.rows), halo.numpy().copy(),
                                    comm.gather(loc.numpy(), g))
        out["sum"] = comm.allsum([0.1 * (rank + 1), 1e-17 * rank])
        part = torch.tensor([1.0 + rank, 2.0 * rank], dtype=torch.float64)
        out["pairs"] = comm.allgather_pairs(part).numpy().copy()
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_gloo_halo_exchange_and_sums():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_cpu_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 8
    for bc in (N.BC_PERIODIC, N.BC_NEUMANN):
        for ncomp in (1, 2):
            glob = (np.arange(ncomp * n * n, dtype=np.float64) * 1.5 + 7.0).reshape(ncomp, n, n)
            for r in range(world):
                row0, rows, halo, gathered = res[r][(bc, ncomp)]
                assert rows == n // world and row0 == r * rows
                assert np.array_equal(gathered, glob.reshape(-1))
                lo = halo[:ncomp * n].reshape(ncomp, n)
                hi = halo[ncomp * n:].reshape(ncomp, n)
                up, down = row0 - 1, row0 + rows
                if bc == N.BC_PERIODIC:
                    up, down = up % n, down % n
                else:  # np.pad 'reflect'
                    up = 1 if up < 0 else up
                    down = n - 2 if down >= n else down
                assert np.array_equal(lo, glob[:, up, :])
                assert np.array_equal(hi, glob[:, down, :])
    for r in range(world):
        assert res[r]["sum"] == [0.1 + 0.2, 0.0 + 1e-17]
        assert np.array_equal(res[r]["pairs"], np.array([[1.0, 0.0], [2.0, 2.0]]))


# ----------------------------------------------------------------- GPU

def _gpu_run(local, n, comm=None, dim=2, name=None):
    """Power iteration + vertical Leja + one EPIRK5P1 step on the periodic
    Brusselator (dim 2) or the 3-D advection-diffusion problem (dim 3), on
    the full grid (comm None) or this rank's slab."""
    import paper_2211_08948_b200 as ek
    from paper_2211_08948_b200 import ext
    if name == "allen_cahn":  # Neumann (reflect) edges, FD Jacobian
        prob = ek.make_problem("allen_cahn", n=n)
    else:
        prob = (ext.brusselator_periodic_problem(n=n) if dim == 2
                else ext.advdiff3d_problem(n=n))
    if comm is not None:
        prob = S.distribute(prob, comm)
    xi = ek.get_leja_points(400)
    rhs = ek.CountingRhs(prob.rhs)
    sys_ = ek.make_linearized(rhs, prob.u0)
    lam, conv = ek.power_iterate(sys_.J)
    est = ek.make_estimate(lam)
    dt = 40.0 / abs(est.alpha)
    r = ek.leja_interpolate_vertical(sys_.J, sys_.f_n * dt, 1, [0.4, 1.0], dt, est, 1e-10, xi=xi)
    st = ek.take_step("epirk5p1", sys_, dt, "leja", 1e-8, ek.EngineContext(est=est, xi=xi))
    vecs = [sys_.f_n, *r.vectors, st.u_high]
    if comm is not None:
        g = prob.rhs.global_grid
        vecs = [comm.gather(v, g) for v in vecs]
    return {"lam": lam, "conv": conv, "iters": r.iters, "freeze": r.freeze_iters,
            "step_iters": st.stats.leja_iters, "err": st.err_est,
            "charges": rhs.counter.count, "vecs": vecs}


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n", [(2, 96), (3, 34)])
def test_slab_path_p1_bit_identical(dim, n):
    from paper_2211_08948_b200 import _device as D
    _repro(True)  # as the slab path: order-independent sums (same bits for every P)
    a = _gpu_run(0, n, dim=dim)
    b = _gpu_run(0, n, comm=S.SlabComm(), dim=dim)
    D.COMM = None
    assert (a["iters"], a["freeze"], a["step_iters"], a["charges"]) == \
        (b["iters"], b["freeze"], b["step_iters"], b["charges"])
    assert a["lam"] == b["lam"] and a["err"] == b["err"]
    for x, y in zip(a["vecs"], b["vecs"]):
        assert np.array_equal(x, y)


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n,name", [(2, 96, None), (2, 600, None), (2, 64, "allen_cahn"),
                                        (3, 34, None)])
def test_peer_mode_p1_bit_identical(dim, n, name):
    """The fused compute + exchange path (boundary rows stored into the
    window halo slots by the Leja kernel, pass flags + device decide, no
    NCCL per iteration), run by one process on its own window (periodic: the
    rank is its own neighbour; reflect: it writes its own mirror ghosts):
    bit-identical to the whole-grid path, counts included."""
    from paper_2211_08948_b200 import _device as D
    _repro(True)
    a = _gpu_run(0, n, dim=dim, name=name)
    comm = S.SlabComm(peer=True)
    assert comm.peer
    b = _gpu_run(0, n, comm=comm, dim=dim, name=name)
    D.COMM = None
    assert comm._windows and next(iter(comm._windows.values())).epoch > 0  # peer path ran
    assert (a["iters"], a["freeze"], a["step_iters"], a["charges"]) == \
        (b["iters"], b["freeze"], b["step_iters"], b["charges"])
    assert a["lam"] == b["lam"] and a["err"] == b["err"]
    for x, y in zip(a["vecs"], b["vecs"]):
        assert np.array_equal(x, y)


def _gpu_worker(rank, world, port, n, q, dim=2):
    _init(rank, world, port)
    try:
        torch.cuda.set_device(0)
        out = _gpu_run(0, n, comm=S.SlabComm(), dim=dim)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n", [(2, 128), (3, 34)])
def test_two_ranks_match_single_gpu(dim, n):
    ref = _gpu_run(0, n, dim=dim)
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, n, q, dim))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        got = res[r]
        assert (got["iters"], got["freeze"], got["step_iters"], got["charges"]) == \
            (ref["iters"], ref["freeze"], ref["step_iters"], ref["charges"])
        assert got["lam"] == pytest.approx(ref["lam"], rel=1e-13)
        assert np.array_equal(got["vecs"][0], ref["vecs"][0])   # RHS: bit-exact
        for x, y in zip(got["vecs"][1:], ref["vecs"][1:]):
            assert np.linalg.norm(x - y) <= 1e-7 * np.linalg.norm(y)
    # both ranks hold the same gathered results
    for x, y in zip(res[0]["vecs"], res[1]["vecs"]):
        assert np.array_equal(x, y)


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n", [(2, 128), (3, 34)])
def test_two_ranks_bitwise_equal_whole_grid_with_repro_sums(dim, n):
    """with the order-independent sums the two-rank run
    (power iteration, vertical Leja call, one EPIRK5P1 step with its FD
    remainders and error norm) equals the whole-grid run bit for bit."""
    _repro(True)
    ref = _gpu_run(0, n, dim=dim)
    _repro(False)
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_worker, args=(r, world, port, n, q, dim))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        got = res[r]
        assert (got["iters"], got["freeze"], got["step_iters"], got["charges"]) == \
            (ref["iters"], ref["freeze"], ref["step_iters"], ref["charges"])
        assert got["lam"] == ref["lam"] and got["conv"] == ref["conv"]
        assert got["err"] == ref["err"]
        for x, y in zip(got["vecs"], ref["vecs"]):
            assert np.array_equal(x, y)


def _gpu_kiops_run(n, comm=None, dim=2):
    """KIOPS on the full grid (fused Arnoldi passes) or this rank's slab
    (`kiops._SlabArnoldi`: local device passes + rank-ordered global dots
    and norms): kiops_eval of phi_1 and one EXPRB43 KIOPS step."""
    import paper_2211_08948_b200 as ek
    from paper_2211_08948_b200 import ext
    prob = ext.brusselator_periodic_problem(n=n) if dim == 2 else ext.advdiff3d_problem(n=n)
    if comm is not None:
        prob = S.distribute(prob, comm)
    rhs = ek.CountingRhs(prob.rhs)
    sys_ = ek.make_linearized(rhs, prob.u0, jac_factory=prob.jac_factory)
    lam, _ = ek.power_iterate(sys_.J)
    dt = 30.0 / abs(lam)
    f = np.asarray(sys_.f_n)
    w, ks = ek.kiops_eval(sys_.J, [np.zeros_like(f), f * dt], dt, 1e-9)
    st = ek.take_step("exprb43", sys_, dt, "kiops", 1e-8, ek.EngineContext())
    vecs = [np.asarray(w), np.asarray(st.u_high)]
    if comm is not None:
        g = prob.rhs.global_grid
        vecs = [comm.gather(v, g) for v in vecs]
    return {"counts": (ks.matvecs, ks.substeps, ks.rejections, st.stats.krylov_matvecs,
                       st.stats.substeps, rhs.counter.count),
            "vecs": vecs}


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n", [(2, 96), (3, 34)])
def test_kiops_slab_p1_matches_fused(dim, n):
    """The slab KIOPS path at P = 1 against the fused
    whole-grid Arnoldi: identical counts, vectors within the FD tier."""
    from paper_2211_08948_b200 import _device as D
    a = _gpu_kiops_run(n, dim=dim)
    try:
        b = _gpu_kiops_run(n, comm=S.SlabComm(), dim=dim)
    finally:
        D.COMM = None
    assert a["counts"] == b["counts"]
    for x, y in zip(a["vecs"], b["vecs"]):
        assert np.linalg.norm(x - y) <= 1e-7 * np.linalg.norm(y)


def _gpu_kiops_worker(rank, world, port, n, q, dim):
    _init(rank, world, port)
    try:
        torch.cuda.set_device(0)
        q.put((rank, _gpu_kiops_run(n, comm=S.SlabComm(), dim=dim)))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n", [(2, 128), (3, 34)])
def test_kiops_two_ranks_match_single_gpu(dim, n):
    """Two slab ranks (host-staged gloo sums and halos, one GPU) take the
    single-GPU run's KIOPS decisions: same matvecs / substeps / rejections,
    vectors within the FD tier, identical on both ranks."""
    ref = _gpu_kiops_run(n, dim=dim)
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_kiops_worker, args=(r, world, port, n, q, dim))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r]["counts"] == ref["counts"]
        for x, y in zip(res[r]["vecs"], ref["vecs"]):
            assert np.linalg.norm(x - y) <= 1e-7 * np.linalg.norm(y)
    for x, y in zip(res[0]["vecs"], res[1]["vecs"]):
        assert np.array_equal(x, y)


@pytest.mark.gpu
@pytest.mark.parametrize("dim,n", [(2, 128), (3, 34)])
def test_kiops_two_ranks_bitwise_equal_one_rank_slab_path(dim, n):
    """SURVEY.md §8(e) e4 for KIOPS: with the order-independent sums (window
    dots, ||w||, ||V[j,:n]||, beta) the slab path gives the same bits on one
    rank and on two — Hessenberg entries, adaptive decisions, outputs."""
    from paper_2211_08948_b200 import _device as D
    try:
        ref = _gpu_kiops_run(n, comm=S.SlabComm(), dim=dim)
    finally:
        D.COMM = None
    # ... and the whole-grid fused Arnoldi passes in repro mode form the same
    # sums (n-part as an integer accumulator, then the tail terms)
    _repro(True)
    whole = _gpu_kiops_run(n, dim=dim)
    _repro(False)
    assert whole["counts"] == ref["counts"]
    for x, y in zip(whole["vecs"], ref["vecs"]):
        assert np.array_equal(x, y)
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_gpu_kiops_worker, args=(r, world, port, n, q, dim))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for r in range(world):
        assert res[r]["counts"] == ref["counts"]
        for x, y in zip(res[r]["vecs"], ref["vecs"]):
            assert np.array_equal(x, y)
