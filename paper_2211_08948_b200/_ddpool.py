"""Divided-difference worker processes.

The Leja divided differences of a 32-point chunk are the first column of
phi_l of an (m + l)-sized bidiagonal matrix, computed on the host by scipy's
`expm` exactly as the reference does (leja.py:88-111, 168-171). At large m
that is the dominant host cost of a long phi-call (m = 384: ~75 ms per
coefficient, while the 32 fused Leja iterations of a chunk take ~30 ms at
512^3), and scipy's `expm` holds the GIL, so a thread cannot overlap it.

This pool runs the same torch-free code (`_dense.phi_divided_differences`)
in separate Python processes: the Leja loop submits the tables of the
chunks it will need ahead of time and collects them at the chunk boundary,
so the host work runs in parallel across cores and overlaps the device
work. Results are bit-identical to the in-process computation (same
function, same libraries, same inputs; checked by tests/test_host.py).
Any pool failure falls back to computing in-process.
"""

import atexit
import os
import pickle
import select
import struct
import subprocess
import sys

_HDR = struct.Struct("<I")


class _Worker:
    def __init__(self):
        env = dict(os.environ)
        env.setdefault("OPENBLAS_NUM_THREADS", "1")  # one core per worker
        # run the worker file as a script: it imports `_dense` directly, not
        # the package (whose __init__ would import torch)
        here = os.path.dirname(os.path.abspath(__file__))
        self.proc = subprocess.Popen(
            [sys.executable, os.path.join(here, "_ddworker.py")],
            stdin=subprocess.PIPE, stdout=subprocess.PIPE, env=env, cwd=here, bufsize=0)
        self.fifo = []  # request keys in submission order

    def send(self, key, args):
        blob = pickle.dumps((key, args), protocol=pickle.HIGHEST_PROTOCOL)
        self.proc.stdin.write(_HDR.pack(len(blob)) + blob)
        self.proc.stdin.flush()
        self.fifo.append(key)

    def _read(self, n):
        buf = b""
        while len(buf) < n:
            chunk = self.proc.stdout.read(n - len(buf))
            if not chunk:
                raise RuntimeError("divided-difference worker exited")
            buf += chunk
        return buf

    def ready(self):
        """A result frame is waiting (unbuffered pipe: select is exact)."""
        return bool(self.fifo) and bool(select.select([self.proc.stdout], [], [], 0)[0])

    def recv(self):
        (size,) = _HDR.unpack(self._read(_HDR.size))
        key, ok, val = pickle.loads(self._read(size))
        self.fifo.pop(0)
        return key, ok, val

    def close(self):
        try:
            self.proc.stdin.close()
            self.proc.wait(timeout=2)
        except Exception:  # noqa: BLE001 - best-effort shutdown
            self.proc.kill()


class DDPool:
    """Submit / collect divided-difference tables keyed like leja._dd_cached."""

    def __init__(self, nworkers=None):
        n = nworkers or min(4, max(1, (os.cpu_count() or 2) - 2))
        self.workers = [_Worker() for _ in range(n)]
        self.owner = {}    # key -> worker of a pending request
        self.done = {}     # key -> (ok, value) received but not collected

    def pending(self, key):
        return key in self.owner or key in self.done

    def _drain(self):
        """Move finished results out of the pipes, so a worker whose tables
        nobody collected (a call that ended early) never blocks on a full
        pipe; keep the newest uncollected ones."""
        for w in self.workers:
            while w.ready():
                k, ok, val = w.recv()
                self.owner.pop(k, None)
                self.done[k] = (ok, val)
        while len(self.done) > 256:
            self.done.pop(next(iter(self.done)))

    def submit(self, key, args):
        self._drain()
        if self.pending(key):
            return
        w = min(self.workers, key=lambda x: len(x.fifo))  # least loaded
        w.send(key, args)
        self.owner[key] = w

    def collect(self, key):
        """(ok, value) of a submitted key; blocks until its worker answers."""
        if key in self.done:
            return self.done.pop(key)
        w = self.owner.get(key)
        if w is None:
            raise KeyError(key)
        while True:
            k, ok, val = w.recv()
            self.owner.pop(k, None)
            if k == key:
                return ok, val
            self.done[k] = (ok, val)

    def close(self):
        for w in self.workers:
            w.close()
        self.workers = []


_POOL = None
_DISABLED = os.environ.get("EK_DD_POOL", "1") == "0"


def existing():
    """The pool if it has been started (never starts it)."""
    return None if _DISABLED else _POOL


def pool():
    """The process-wide pool (started on first use), or None if disabled or
    it could not start. The Leja loop starts it at the first chunk crossing
    it meets, so runs whose phi-calls stay within one chunk never pay for the
    worker start-up (~0.3 s of numpy / scipy imports per worker)."""
    global _POOL, _DISABLED
    if _DISABLED:
        return None
    if _POOL is None:
        try:
            _POOL = DDPool()
            atexit.register(_POOL.close)
        except Exception:  # noqa: BLE001 - host helper: compute in-process instead
            _DISABLED = True
            return None
    return _POOL


def disable():
    """Stop using the pool (after a worker failure)."""
    global _POOL, _DISABLED
    _DISABLED = True
    if _POOL is not None:
        _POOL.close()
        _POOL = None
