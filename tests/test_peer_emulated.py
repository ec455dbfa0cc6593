"""The multi-GPU Leja path (the fused compute + halo
exchange over peer memory, `ek_leja_run_peer`) with P = 2 and 4 ranks,
emulated on ONE GPU in ONE process.

Ranks whose kernels wait on one another must not run as separate launches
on one GPU (B200_PROFILING.md: Xid 109), so this test drives the ranks in
lockstep on a single stream with the phase-split entry point
`ek_leja_run_peer_phase`: for every iteration m, first every rank's fused
pass (which stores its boundary rows of y' into the neighbours' halo slots
and its partial sums plus a pass flag into every rank's window), then every
rank's decide kernel (which finds all flags already raised). The windows
are real `ek_ipc_alloc` allocations and every rank sees every window
through its `ek_peer` map, exactly as after `PeerWindow`'s IPC exchange; the
kernels, slot layout, epochs and decisions are those of the multi-process
run. Result: the same iterations and freeze points as the whole-grid fused
call, and the same vectors (analytic Jacobian: 1e-13; FD Jacobian: the
1e-7 tier — the rank-ordered partial sums change ||y|| in the last ulp).
The IPC handle exchange itself between two processes is covered by
tests/test_peer_ipc.py."""

import ctypes as C

import numpy as np
import pytest
import torch

import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import _device as D, _native as N, ext, leja as L

pytestmark = pytest.mark.gpu


def _halo(xg, ncomp, n, rowlen, P, r, periodic):
    """[2][ncomp][rowlen] ghost rows -1 / rows of rank r's slab (host)."""
    rows = n // P
    x = xg.reshape(ncomp, n, rowlen)
    lo, hi = r * rows - 1, (r + 1) * rows
    if periodic:
        lo, hi = lo % n, hi % n
    else:  # np.pad 'reflect' at the global edges
        lo = 1 if lo < 0 else lo
        hi = n - 2 if hi >= n else hi
    return np.concatenate([x[:, lo, :].ravel(), x[:, hi, :].ravel()])


def _emulated_peer_leja(grid, jac, u, fu, b, coeffs, l, h, est, tol, xi, P):
    lib = N.lib()
    n, ncomp = int(grid.n), int(grid.ncomp)
    rowlen = n if grid.dim == 2 else n * n
    rows = n // P
    periodic = grid.bc == N.BC_PERIODIC
    k = len(coeffs)
    dds = L._dd_group(l, [c * h for c in coeffs], est, xi, 32)
    table = L._CoefTable(k)
    table.load(0, 32, dds, est.c, est.gamma, xi)
    ug, fg, bg = (np.asarray(v).reshape(ncomp, n, rowlen) for v in (u, fu, b))
    ranks = []
    for r in range(P):
        g = N.Grid()
        C.pointer(g)[0] = grid
        g.rows, g.row0, g.slab = rows, r * rows, 1
        sl = lambda x: D.to_dev(np.ascontiguousarray(x[:, r * rows:(r + 1) * rows, :]).ravel())
        rk = {"g": g, "u": sl(ug), "fu": sl(fg), "b": sl(bg),
              "uh": D.to_dev(_halo(ug, ncomp, n, rowlen, P, r, periodic)),
              "bh": D.to_dev(_halo(bg, ncomp, n, rowlen, P, r, periodic))}
        rk["p"] = [D.empty(rk["b"].numel()) for _ in range(k)]
        rk["y"] = [D.empty(rk["b"].numel()), D.empty(rk["b"].numel())]
        nbytes = lib.ek_peer_window_bytes(C.byref(g))
        ptr, handle = C.c_void_p(), (C.c_char * 64)()
        N.check(lib.ek_ipc_alloc(nbytes, C.byref(ptr), handle), "ek_ipc_alloc")
        rk["win"] = ptr.value
        ranks.append(rk)
    # ||u|| of the global field as the slab path forms it: rank-ordered sum
    # of the ranks' sums of squares; in repro mode the exact merge of the
    # ranks' integer accumulators (ek_xsum_host is the kernels' per-term code)
    if lib.ek_set_repro(-1):
        slots = (C.c_int64 * (N.XSLOTS * P))()
        for r, rk in enumerate(ranks):
            ur = np.ascontiguousarray(rk["u"].cpu().numpy())
            lib.ek_xsum_host(ur.ctypes.data_as(C.c_void_p), ur.size, 1,
                             C.cast(C.byref(slots, 8 * N.XSLOTS * r), C.POINTER(C.c_int64)))
        nu = lib.ek_xsum_value(slots, P)
    else:
        nu = 0.0
        for rk in ranks:
            nu = nu + float(torch.sum(rk["u"] * rk["u"]))
    nu = float(np.sqrt(nu)) if jac == N.JAC_FD else 0.0
    for r, rk in enumerate(ranks):
        up = r - 1 if r > 0 else (P - 1 if periodic else -1)
        down = r + 1 if r < P - 1 else (0 if periodic else -1)
        host = N.Peer(world=P, rank=r, up=up, down=down, rowlen=rowlen, ncomp=ncomp)
        for q, other in enumerate(ranks):
            host.win[q] = other["win"]
        rk["peer"] = torch.frombuffer(bytearray(bytes(host)), dtype=torch.uint8).to(D.device())
        rk["st"] = D.DevState(N.LejaState, tol=float(tol), nu=nu, k=k, defer=1, p_init=0)
    ws = D.work_ptr(lib.ek_workspace_bytes(C.byref(ranks[0]["g"])))
    s = D.stream()
    # m = 0: local partials, then every rank decides on the rank-ordered sums
    for rk in ranks:
        N.check(lib.ek_leja_begin_len(rk["b"].numel(), C.c_void_p(rk["b"].data_ptr()),
                                      N.ptrs(rk["p"]), k, C.c_void_p(table.dev.data_ptr()),
                                      rk["st"].ptr, ws, s), "begin")
    gathered = torch.stack([L._part_view(rk["st"]) for rk in ranks])
    for rk in ranks:
        N.check(lib.ek_leja_decide(rk["st"].ptr, C.c_void_p(gathered.data_ptr()), P,
                                   C.c_void_p(table.dev.data_ptr()), 0, 0, k,
                                   1 if jac == N.JAC_FD else 0, 1, s), "begin decide")
    for m in range(1, 32):
        for phase in (1, 2):
            for rk in ranks:
                halo = N.ptrs([rk["uh"], rk["bh"], None])
                N.check(lib.ek_leja_run_peer_phase(
                    C.byref(rk["g"]), jac, C.c_void_p(rk["u"].data_ptr()),
                    C.c_void_p(rk["fu"].data_ptr()), C.c_void_p(rk["b"].data_ptr()),
                    N.ptrs(rk["y"]), N.ptrs(rk["p"]), k, C.c_void_p(table.dev.data_ptr()), 0,
                    m, m + 1, float(est.gamma), rk["st"].ptr, ws, halo,
                    C.c_void_p(rk["peer"].data_ptr()), C.c_void_p(rk["win"]), m - 1, phase,
                    s), "peer phase")
    torch.cuda.synchronize()
    states = [rk["st"].read() for rk in ranks]
    out = [np.concatenate([rk["p"][i].cpu().numpy().reshape(ncomp, rows, rowlen)
                           for rk in ranks], axis=1).ravel() for i in range(k)]
    for rk in ranks:
        N.check(lib.ek_ipc_free(C.c_void_p(rk["win"])), "ek_ipc_free")
    return states, out


CASES = [("advdiff2d", 64, N.JAC_ANALYTIC, 2), ("advdiff2d", 64, N.JAC_ANALYTIC, 4),
         ("brusselator_periodic", 64, N.JAC_FD, 2), ("brusselator_periodic", 64, N.JAC_FD, 4),
         ("allen_cahn", 64, N.JAC_FD, 2), ("advdiff3d", 32, N.JAC_ANALYTIC, 4)]


@pytest.mark.parametrize("name,n,jac,P", CASES)
def test_peer_leja_emulated_ranks_match_whole_grid(name, n, jac, P):
    xi = ek.get_leja_points(400)
    if name == "allen_cahn":  # the reference's Neumann problem: reflect ghosts
        p = ek.make_problem("allen_cahn", n=n)
    else:
        p = ext.make_ext_problem(name, n=n)
    jf = p.jac_factory if jac == N.JAC_ANALYTIC else None
    rhs = ek.CountingRhs(p.rhs)
    sys_ = ek.make_linearized(rhs, p.u0, jac_factory=jf)
    est = ek.make_estimate(ek.power_iterate(sys_.J)[0])
    dt = 20.0 / abs(est.alpha)
    b = sys_.f_n * dt
    coeffs = [0.5, 1.0]
    ref = ek.leja_interpolate_vertical(sys_.J, b, 1, coeffs, dt, est, 1e-10, xi=xi)
    assert 3 < ref.iters < 31
    states, got = _emulated_peer_leja(p.rhs.grid, jac, p.u0, sys_.f_n, b, coeffs, 1, dt, est,
                                      1e-10, xi, P)
    for h in states:
        assert h.status == N.ST_OK and h.done
        assert int(h.iters) == ref.iters
        assert [int(h.freeze[i]) for i in range(2)] == ref.freeze_iters
    tol = 1e-13 if jac == N.JAC_ANALYTIC else 1e-7
    for g, r in zip(got, ref.vectors):
        assert np.linalg.norm(g - r) <= tol * np.linalg.norm(r)


REPRO_CASES = [("advdiff2d", 64, N.JAC_ANALYTIC), ("brusselator_periodic", 64, N.JAC_FD),
               ("allen_cahn", 64, N.JAC_FD), ("advdiff3d", 32, N.JAC_ANALYTIC)]


@pytest.mark.parametrize("name,n,jac", REPRO_CASES)
def test_repro_sums_make_the_leja_call_bitwise_identical_for_every_P(name, n, jac):
    """with the order-independent sums (ek_set_repro) the
    whole-grid fused call and the peer path at P = 1, 2, 4 give the same
    bits — vectors, iterations and freeze points — for analytic and FD
    Jacobians (through the FD increment every ulp of ||y|| would show)."""
    xi = ek.get_leja_points(400)
    old = D.set_reproducible(True)
    try:
        if name == "allen_cahn":
            p = ek.make_problem("allen_cahn", n=n)
        else:
            p = ext.make_ext_problem(name, n=n)
        jf = p.jac_factory if jac == N.JAC_ANALYTIC else None
        rhs = ek.CountingRhs(p.rhs)
        sys_ = ek.make_linearized(rhs, p.u0, jac_factory=jf)
        est = ek.make_estimate(ek.power_iterate(sys_.J)[0])
        dt = 20.0 / abs(est.alpha)
        b = sys_.f_n * dt
        coeffs = [0.5, 1.0]
        ref = ek.leja_interpolate_vertical(sys_.J, b, 1, coeffs, dt, est, 1e-10, xi=xi)
        assert 3 < ref.iters < 31
        periodic = p.rhs.grid.bc == N.BC_PERIODIC
        for P in ((1, 2, 4) if periodic else (2, 4)):
            states, got = _emulated_peer_leja(p.rhs.grid, jac, p.u0, sys_.f_n, b, coeffs, 1, dt,
                                              est, 1e-10, xi, P)
            for h in states:
                assert h.status == N.ST_OK and h.done
                assert int(h.iters) == ref.iters
                assert [int(h.freeze[i]) for i in range(2)] == ref.freeze_iters
                assert h.ny == states[0].ny and h.eps == states[0].eps
            for g, r in zip(got, ref.vectors):
                assert np.array_equal(g, r), (P, np.abs(g - r).max())
    finally:
        D.set_reproducible(old)
