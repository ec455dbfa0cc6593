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

Activate with `distribute(problem)`; the returned Problem carries a local
`StencilRhs` and the rank's slice of the initial condition.
"""

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from . import _device as D
from . import _native as N
from .problems import NativeJacFactory, Problem, StencilRhs


class SlabComm:
    """Neighbour exchange and rank-ordered sums for one slab decomposition."""

    def __init__(self, group=None):
        if dist.is_available() and dist.is_initialized():
            self.group = group
            self.rank = dist.get_rank(group)
            self.world = dist.get_world_size(group)
            self.backend = dist.get_backend(group)
        else:
            self.group, self.rank, self.world, self.backend = None, 0, 1, None

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
        """[world, 2] device tensor of every rank's 2-double `part` view."""
        if self.world == 1:
            return part.reshape(1, 2)
        if self.host_staged:
            bufs = [torch.empty(2, dtype=torch.float64) for _ in range(self.world)]
            dist.all_gather(bufs, part.cpu(), group=self.group)
            return torch.stack(bufs).to(part.device)
        out = torch.empty(self.world * 2, dtype=torch.float64, device=part.device)
        dist.all_gather_into_tensor(out, part.contiguous(), group=self.group)
        return out.reshape(self.world, 2)

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
