"""Row-slab domain decomposition over GPUs.

One process per GPU (torch.distributed; NCCL over NVLink on a multi-GPU box,
gloo for host-staged CPU tests). Every state vector is split along axis 0
(rows in 2-D, planes in 3-D) into equal slabs, component by component, so a
rank's local vector is itself component-major:
[comp0 rows row0..row0+rows-1, comp1 ...]. The stencil kernels read the
ghost rows -1 / rows from a halo buffer ([2][ncomp][row length]) that
`SlabComm.exchange` fills before every stencil pass:

  * interior ranks: row -1 = last row of rank-1, row `rows` = first row of
    rank+1 (two grouped send/recv pairs per component);
  * periodic: rank 0 and rank P-1 are neighbours;
  * Neumann (reflect): the global edges mirror locally (rows 1 / rows-2).

Reductions are split: the kernels leave their local sums in the state
block (`defer`), the ranks all-gather them, and the device decision sums
them in rank order — identical on every rank, so all ranks take the same
branch every iteration without any host round trip.

Peer mode (`SlabComm(peer=True)`, the default over NCCL): the Leja
recurrence — the hot loop — exchanges nothing through NCCL. Every rank maps
every rank's device window (CUDA IPC over NVLink, `PeerWindow`); the fused
Leja kernel stores its boundary rows of y' straight into the neighbours'
halo slots and its partial sums plus a pass flag into every window, and a
one-warp decide kernel waits for the flags and applies the freeze test
(`ek_leja_run_peer`). A launch batch of iterations is enqueued like the
single-GPU one, with no host round trip or NCCL call per iteration.

Activate with `distribute(problem)`; the returned Problem carries a local
`StencilRhs` and the rank's slice of the initial condition.
"""

import ctypes as C
import os

import numpy as np
import torch
import torch.distributed as dist

from . import _device as D
from . import _native as N
from .problems import NativeJacFactory, Problem, StencilRhs


class SlabComm:
    """Neighbour exchange and rank-ordered sums for one slab decomposition.

    peer: None = on over NCCL (device ranks), off over gloo / single process;
    True forces it (a single process then maps its own window: the test of
    the fused path on one GPU), False disables it."""

    def __init__(self, group=None, peer=None):
        if dist.is_available() and dist.is_initialized():
            self.group = group
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
            self.backend = dist.get_backend(group)
        else:
            self.group, self.rank, self.world, self.backend = None, 0, 1, None
        if peer is None:
            peer = self.backend == "nccl" and self.world > 1
        self.peer = bool(peer) and not self.host_staged
        self._windows = {}

    def window(self, grid):
        """The PeerWindow of a local slab grid (created collectively on first
        use; every rank reaches it in the same order)."""
        key = (int(grid.dim), int(grid.ncomp), int(grid.n), int(grid.rows))
        w = self._windows.get(key)
        if w is None:
            w = self._windows[key] = PeerWindow(self, grid)
        return w

    @property
    def host_staged(self):
        return self.backend == "gloo"

    def rows_of(self, n):
        if n % self.world:
            raise ValueError(f"grid extent {n} is not divisible by {self.world} ranks")
        rows = n // self.world
        return self.rank * rows, rows

    # ------------------------------------------------------------ halos
    def exchange(self, x, grid, halo):
        """Fill `halo` (flat tensor, 2 * ncomp * rowlen) with the ghost rows
        -1 and `rows` of the local field x."""
        ncomp, rows = int(grid.ncomp), int(grid.rows)
        rowlen = int(grid.n) if grid.dim == 2 else int(grid.n) * int(grid.n)
        npts = rows * rowlen
        periodic = grid.bc == N.BC_PERIODIC
        first = [x[c * npts: c * npts + rowlen] for c in range(ncomp)]
        last = [x[c * npts + (rows - 1) * rowlen: c * npts + rows * rowlen]
                for c in range(ncomp)]
        lo = [halo[c * rowlen:(c + 1) * rowlen] for c in range(ncomp)]
        hi = [halo[(ncomp + c) * rowlen:(ncomp + c + 1) * rowlen] for c in range(ncomp)]
        up = self.rank - 1 if self.rank > 0 else (self.world - 1 if periodic else None)
        down = self.rank + 1 if self.rank < self.world - 1 else (0 if periodic else None)
        if not periodic:
            # reflect ghosts at the global edges (np.pad 'reflect')
            if up is None:
                for c in range(ncomp):
                    src = x[c * npts + rowlen: c * npts + 2 * rowlen] if rows > 1 else first[c]
                    lo[c].copy_(src)
            if down is None:
                for c in range(ncomp):
                    src = (x[c * npts + (rows - 2) * rowlen: c * npts + (rows - 1) * rowlen]
                           if rows > 1 else last[c])
                    hi[c].copy_(src)
        if self.world == 1:
            if periodic:
                for c in range(ncomp):
                    lo[c].copy_(last[c])
                    hi[c].copy_(first[c])
            return halo
        # Messages between one pair of ranks match in posting order, and with
        # two periodic ranks `up` and `down` are the same peer: post the
        # downward flow (my last row -> down's row -1) before the upward one
        # on both the sending and the receiving side.
        ops = []
        if down is not None:
            ops += [("send", last[c], down, None) for c in range(ncomp)]
        if up is not None:
            ops += [("send", first[c], up, None) for c in range(ncomp)]
        if up is not None:
            ops += [("recv", None, up, lo[c]) for c in range(ncomp)]
        if down is not None:
            ops += [("recv", None, down, hi[c]) for c in range(ncomp)]
        self._p2p(ops)
        return halo

    def _p2p(self, ops):
        p2p = []
        back = []
        for kind, src, peer, dst in ops:
            if kind == "send":
                t = src.cpu() if self.host_staged else src.contiguous()
                p2p.append(dist.P2POp(dist.isend, t, peer, self.group))
            else:
                t = torch.empty(dst.numel(), dtype=dst.dtype,
                                device="cpu" if self.host_staged else dst.device)
                p2p.append(dist.P2POp(dist.irecv, t, peer, self.group))
                back.append((t, dst))
        for req in dist.batch_isend_irecv(p2p):
            req.wait()
        for t, dst in back:
            dst.copy_(t)

    # ------------------------------------------------------- reductions
    def allgather_pairs(self, part):
        """[world, k] device tensor of every rank's k-slot `part` view (the
        EK_PART_SLOTS block of a control state: fp64 values, or in repro
        mode the bit patterns of the integer accumulator — the gather only
        moves bytes)."""
        k = part.numel()
        if self.world == 1:
            return part.reshape(1, k)
        if self.host_staged:
            bufs = [torch.empty(k, dtype=torch.float64) for _ in range(self.world)]
            dist.all_gather(bufs, part.cpu(), group=self.group)
            return torch.stack(bufs).to(part.device)
        out = torch.empty(self.world * k, dtype=torch.float64, device=part.device)
        dist.all_gather_into_tensor(out, part.contiguous(), group=self.group)
        return out.reshape(self.world, k)

    def allgather_vals(self, part):
        """[world * k] device tensor of every rank's k-double device view
        (rank-major), stream-ordered over NCCL (no host sync); host-staged
        over gloo."""
        k = part.numel()
        if self.world == 1:
            return part.reshape(-1)
        if self.host_staged:
            bufs = [torch.empty(k, dtype=torch.float64) for _ in range(self.world)]
            dist.all_gather(bufs, part.cpu(), group=self.group)
            return torch.cat(bufs).to(part.device)
        out = torch.empty(self.world * k, dtype=torch.float64, device=part.device)
        dist.all_gather_into_tensor(out, part.contiguous(), group=self.group)
        return out

    def allsum(self, values):
        """Rank-ordered sums of a list of host floats (identical on all ranks)."""
        if self.world == 1:
            return list(values)
        t = torch.tensor(values, dtype=torch.float64)
        if not self.host_staged:
            t = t.cuda()
        bufs = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(bufs, t, group=self.group)
        rows = [b.cpu().tolist() for b in bufs]
        out = []
        for i in range(len(values)):
            s = rows[0][i]
            for r in range(1, self.world):
                s = s + rows[r][i]
            out.append(s)
        return out

    def allgather_ints(self, values):
        """[world][len(values)] host ints of every rank (int64 payload: the
        slots of an order-independent accumulator, ek_xsum.cuh)."""
        if self.world == 1:
            return [list(values)]
        t = torch.tensor(values, dtype=torch.int64)
        if not self.host_staged:
            t = t.cuda()
        bufs = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(bufs, t, group=self.group)
        return [b.cpu().tolist() for b in bufs]

    # --------------------------------------------------- data movement
    def scatter(self, u_global, grid_global):
        """This rank's slab of a global component-major vector (host)."""
        ncomp = int(grid_global.ncomp)
        n = int(grid_global.n)
        rowlen = n if grid_global.dim == 2 else n * n
        row0, rows = self.rows_of(n)
        u = np.asarray(u_global).reshape(ncomp, n, rowlen)
        return np.ascontiguousarray(u[:, row0:row0 + rows, :]).reshape(-1)

    def gather(self, u_local, grid_global):
        """Global vector on every rank (tests / output)."""
        ncomp = int(grid_global.ncomp)
        n = int(grid_global.n)
        rowlen = n if grid_global.dim == 2 else n * n
        loc = torch.as_tensor(np.asarray(D.to_host(u_local))).reshape(-1)
        if self.world == 1:
            return loc.numpy()
        if not self.host_staged:
            loc = loc.cuda()
        bufs = [torch.empty_like(loc) for _ in range(self.world)]
        dist.all_gather(bufs, loc, group=self.group)
        parts = [b.cpu().numpy().reshape(ncomp, -1, rowlen) for b in bufs]
        return np.concatenate(parts, axis=1).reshape(-1)


class PeerWindow:
    """This rank's device window and the map of every rank's window
    (ek_peer, include/expkit_sm100.h): flags, partial sums, halo slots."""

    def __init__(self, comm, grid):
        lib = N.lib()
        rows = int(grid.rows)
        if rows < 2:
            raise ValueError("peer mode needs slabs of at least two rows")
        nbytes = lib.ek_peer_window_bytes(C.byref(grid))
        ptr = C.c_void_p()
        handle = (C.c_char * 64)()
        N.check(lib.ek_ipc_alloc(nbytes, C.byref(ptr), handle), "ek_ipc_alloc")
        self.local = ptr.value
        mine = bytes(handle)
        if comm.world > 1:
            handles = [None] * comm.world
            dist.all_gather_object(handles, mine, group=comm.group)
        else:
            handles = [mine]
        self._opened = []
        wins = []
        for r, h in enumerate(handles):
            if r == comm.rank:
                wins.append(self.local)
            else:
                p = C.c_void_p()
                N.check(lib.ek_ipc_open(h, C.byref(p)), "ek_ipc_open")
                self._opened.append(p.value)
                wins.append(p.value)
        periodic = grid.bc == N.BC_PERIODIC
        up = comm.rank - 1 if comm.rank > 0 else (comm.world - 1 if periodic else -1)
        down = comm.rank + 1 if comm.rank < comm.world - 1 else (0 if periodic else -1)
        host = N.Peer(world=comm.world, rank=comm.rank, up=up, down=down,
                      rowlen=int(grid.n) if grid.dim == 2 else int(grid.n) ** 2,
                      ncomp=int(grid.ncomp))
        for r, w in enumerate(wins):
            host.win[r] = w
        raw = bytes(host)
        self.dev = torch.frombuffer(bytearray(raw), dtype=torch.uint8).to(D.device())
        self.epoch = 0  # passes issued so far (identical on every rank)
        if comm.world > 1:
            dist.barrier(group=comm.group)

    @property
    def ptr(self):
        return C.c_void_p(self.dev.data_ptr())

    def take(self, passes):
        """Epoch of the first of `passes` consecutive fused passes."""
        e = self.epoch
        self.epoch += passes
        return e


def slab_grid(grid, comm):
    """Local ek_grid of this rank's slab."""
    g = N.Grid()
    C.pointer(g)[0] = grid
    row0, rows = comm.rows_of(int(grid.n))
    g.rows, g.row0, g.slab = rows, row0, 1
    return g


def distribute(problem, comm=None):
    """Problem restricted to this rank's slab: local StencilRhs (halo
    exchange + stencil), local slice of u0. Also registers `comm` as the
    process's reduction communicator (one slab decomposition per process)."""
    comm = comm or SlabComm()
    st = problem.rhs
    if not isinstance(st, StencilRhs) or st.grid.dim < 2:
        raise ValueError("only 2-D / 3-D native stencil problems can be distributed")
    g = slab_grid(st.grid, comm)
    rhs = StencilRhs(st.name, g, analytic=st.analytic)
    rhs.comm = comm
    rhs.global_grid = st.grid
    D.COMM = comm if comm.world > 1 else None
    # every norm on the path is an order-independent
    # sum, so results are bitwise identical for every decomposition (and for
    # the whole-grid run under `_device.set_reproducible()`); EK_REPRO=0
    # keeps the rank-ordered fp64 sums
    if os.environ.get("EK_REPRO", "1") != "0":
        D.set_reproducible(True)
    jf = NativeJacFactory(rhs) if isinstance(problem.jac_factory, NativeJacFactory) else None
    u0 = comm.scatter(problem.u0, st.grid)
    out = Problem(problem.name, rhs, u0, problem.t_final, n=problem.n,
                  n_components=problem.n_components, params=problem.params,
                  jac_factory=jf)
    out.comm = comm
    return out


def halo_buffer(grid):
    rowlen = int(grid.n) if grid.dim == 2 else int(grid.n) ** 2
    return D.empty(2 * int(grid.ncomp) * rowlen)
