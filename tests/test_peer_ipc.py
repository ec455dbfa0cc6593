"""The CUDA-IPC window exchange of the peer-mode slab path, with two real
processes (`slab.PeerWindow` -> ek_ipc_alloc /
ek_ipc_open / ek_ipc_close / ek_ipc_free).

Two gloo ranks on the one GPU of the box each build the `PeerWindow` of
their slab collectively (all-gather of the 64-byte IPC handles, then
`ek_ipc_open` of the other rank's window), write a marker into their own
window's halo slots and read the other rank's marker through the mapped
pointer. No kernel waits for another process here (the waiting kernels of
the fused path are exercised with emulated ranks in
tests/test_peer_emulated.py), so sharing one GPU is safe."""

import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, errq):
    try:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        from paper_2211_08948_b200 import _native as N, ext, slab as SL
        p = ext.brusselator_periodic_problem(n=64)
        comm = SL.SlabComm(peer=False)
        g = SL.slab_grid(p.rhs.grid, comm)
        win = SL.PeerWindow(comm, g)
        host = N.Peer.from_buffer_copy(bytes(win.dev.cpu().numpy()))
        assert host.world == world and host.rank == rank
        assert host.win[rank] == win.local and len(win._opened) == world - 1
        marker = np.full(16, 1000.0 + rank)
        lib = N.lib()
        N.check(lib.ek_copy(C.c_void_p(win.local + N.PEER_HALO_OFFSET),
                            marker.ctypes.data_as(C.c_void_p), marker.nbytes, 1, None), "put")
        torch.cuda.synchronize()
        dist.barrier()
        other = (rank + 1) % world
        got = np.zeros(16)
        N.check(lib.ek_copy(got.ctypes.data_as(C.c_void_p),
                            C.c_void_p(host.win[other] + N.PEER_HALO_OFFSET), got.nbytes, 2,
                            None), "get")
        assert np.all(got == 1000.0 + other), got
        # and write into the other rank's window: it reads its own slot back
        N.check(lib.ek_copy(C.c_void_p(host.win[other] + N.PEER_HALO_OFFSET + 128),
                            marker.ctypes.data_as(C.c_void_p), marker.nbytes, 1, None), "put2")
        torch.cuda.synchronize()
        dist.barrier()
        mine = np.zeros(16)
        N.check(lib.ek_copy(mine.ctypes.data_as(C.c_void_p),
                            C.c_void_p(win.local + N.PEER_HALO_OFFSET + 128), mine.nbytes, 2,
                            None), "get2")
        assert np.all(mine == 1000.0 + other), mine
        dist.barrier()
        for ptr in win._opened:
            N.check(lib.ek_ipc_close(C.c_void_p(ptr)), "ek_ipc_close")
        dist.barrier()
        N.check(lib.ek_ipc_free(C.c_void_p(win.local)), "ek_ipc_free")
        dist.destroy_process_group()
    except BaseException as exc:  # noqa: BLE001 - reported to the parent
        errq.put(f"rank {rank}: {type(exc).__name__}: {exc}")
        raise


def test_peer_windows_across_two_processes():
    import torch.multiprocessing as mp
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    ctx = mp.get_context("spawn")
    errq = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, errq)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    errs = []
    while not errq.empty():
        errs.append(errq.get())
    for p in procs:
        if p.is_alive():
            p.kill()
            errs.append("timeout")
    assert not errs, errs
    assert all(p.exitcode == 0 for p in procs)
