"""Device plumbing: fp64 CUDA tensors (torch = allocator + streams only),
device state blocks, workspaces, and the elementwise-expression builder that
lowers NumPy-style stage algebra to one `ek_vexpr` launch.

Every computation below runs in libexpkit_sm100.so on the current CUDA
device; torch is used for memory, streams and host<->device copies.
"""

import ctypes as C
import math

import numpy as np
import torch

from . import _native as N

F64 = torch.float64


# ---------------------------------------------------------------- device

_READY = False
_DEVICES = {}
# current device index without torch.cuda.current_device()'s lazy-init checks
# (the host path asks ~100 times per integrator step); valid once _READY
_GET_DEVICE = getattr(torch._C, "_cuda_getDevice", None)


def _index():
    return _GET_DEVICE() if _GET_DEVICE is not None else torch.cuda.current_device()


def device():
    global _READY
    if not _READY:
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2211_08948_b200 needs a CUDA device (B200); "
                               "there is no CPU fallback")
        N.lib()
        torch.cuda.init()
        _READY = True
    i = _index()
    d = _DEVICES.get(i)
    if d is None:
        d = _DEVICES[i] = torch.device("cuda", i)
    return d


_RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def stream():
    """torch's current stream on the current device (raw handle; the fast
    accessor avoids building a torch.cuda.Stream object per call)."""
    if _RAW_STREAM is not None and _READY:
        return C.c_void_p(_RAW_STREAM(_index()))
    if _RAW_STREAM is not None:
        return C.c_void_p(_RAW_STREAM(torch.cuda.current_device()))
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def is_dev(x):
    return isinstance(x, torch.Tensor)


def to_dev(x, copy=False):
    """fp64 contiguous 1-D CUDA tensor view/copy of x (numpy or torch)."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=device(), dtype=F64)
        t = t.contiguous().reshape(-1)
        if copy and t.data_ptr() == x.data_ptr():
            t = t.clone()
        return t
    arr = np.ascontiguousarray(np.asarray(x, dtype=np.float64)).reshape(-1)
    return torch.from_numpy(arr).to(device=device())


_PIN_MIN = 1 << 20  # bytes; larger results come back through pinned memory


def like_input(t, ref):
    """Return t in the kind of `ref`: numpy in -> numpy out, tensor -> tensor."""
    if isinstance(ref, torch.Tensor):
        return t
    return to_host(t)


def to_host(t):
    """Device -> NumPy. Large vectors are copied into page-locked memory
    (torch's caching host allocator), a direct DMA at full PCIe rate; the
    array keeps its pinned buffer alive and a later H2D of it is direct too."""
    if not isinstance(t, torch.Tensor):
        return np.asarray(t)
    if t.is_cuda and t.numel() * t.element_size() >= _PIN_MIN:
        host = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        host.copy_(t)
        return host.numpy()
    return t.cpu().numpy()


def empty(n):
    return torch.empty(int(n), dtype=F64, device=device())


def zeros(n):
    return torch.zeros(int(n), dtype=F64, device=device())


# ------------------------------------------------------------- workspace

_WORK = {}


def work(nbytes=None):
    """Per-device scratch for block partials (grows monotonically)."""
    dev = device().index
    need = max(int(nbytes or 0), 148 * 16 * 8 * 8)
    buf = _WORK.get(dev)
    if buf is None or buf.numel() * 8 < need:
        buf = torch.empty((need + 7) // 8, dtype=F64, device=device())
        _WORK[dev] = buf
    return buf


def work_ptr(nbytes=None):
    return C.c_void_p(work(nbytes).data_ptr())


# ---------------------------------------------------------- state blocks

class DevState:
    """A ctypes Structure mirrored in device memory."""

    def __init__(self, ctype, upload=True, **init):
        self.ctype = ctype
        self.size = C.sizeof(ctype)
        # fully initialised by the upload below (no fill kernel), or by a
        # device init kernel of the caller (upload=False)
        self.buf = torch.empty(self.size, dtype=torch.uint8, device=device())
        self.host = ctype()
        for k, v in init.items():
            setattr(self.host, k, v)
        if upload:
            self.upload()

    @property
    def ptr(self):
        return C.c_void_p(self.buf.data_ptr())

    def upload(self):
        N.check(N.lib().ek_copy(self.ptr, C.byref(self.host), self.size, 1, stream()),
                "state upload")

    def _pull(self):
        N.check(N.lib().ek_copy(C.byref(self.host), self.ptr, self.size, 2, stream()),
                "state read")
        return self.host

    def read(self):
        """Stream-ordered D2H copy into pageable memory: returns once the
        stream has reached this point (the host sync of a chunk). Deferred
        checks of earlier passes are resolved first (program order)."""
        self._pull()
        if _PENDING:
            flush_checks()
        return self.host


# Deferred error checks (single GPU): a pass whose state carries only an
# error flag (the remainder's non-finite test, integrators.py:107-108) is
# not synchronised on by itself; its flag is checked at the stream's next
# host sync, before that sync's own result is interpreted (so the
# reference's exception, and no later work's counter charges, wins), and at
# the end of the step. The host keeps enqueueing while the pass runs.
# Deferred counter charges (defer_fn callbacks) add what they charge to
# ADJ[0], so that per-group counter windows opened before a flush can leave
# them out (integrators._Engines._charge).
_PENDING = []
ADJ = [0]


def defer_check(state, mask, make_exc):
    _PENDING.append((state, mask, make_exc))


def defer_fn(state, fn):
    """fn(host_state) at the next flush (in program order with the checks)."""
    _PENDING.append((state, None, fn))


def clear_checks():
    _PENDING.clear()


_PIN = [None]


def _pull_all(states):
    """Read several state blocks with ONE stream synchronisation: async
    copies into a pinned staging buffer, one sync, then host copies."""
    sizes = [(s.size + 15) // 16 * 16 for s in states]
    total = sum(sizes)
    buf = _PIN[0]
    if buf is None or buf.numel() < total:
        buf = torch.empty(max(total, 1 << 16), dtype=torch.uint8, pin_memory=True)
        _PIN[0] = buf
    base, off, strm = buf.data_ptr(), 0, stream()
    for st, sz in zip(states, sizes):
        N.check(N.lib().ek_copy(C.c_void_p(base + off), st.ptr, st.size, 2, strm),
                "state read")
        off += sz
    N.check(N.lib().ek_sync(strm), "state sync")
    off = 0
    for st, sz in zip(states, sizes):
        C.memmove(C.addressof(st.host), base + off, st.size)
        off += sz


def flush_checks():
    if len(_PENDING) > 1:
        uniq = list({id(st): st for st, _, _ in _PENDING}.values())
        _pull_all(uniq)
        fresh = {id(st) for st in uniq}
    else:
        fresh = ()
    while _PENDING:
        st, mask, fn = _PENDING.pop(0)
        h = st.host if id(st) in fresh else st._pull()
        if mask is None:
            fn(h)
        elif h.flag & mask:
            _PENDING.clear()
            raise fn()


def scalar_state():
    return DevState(N.ScalarState)


# Slab communicator of this process (set by slab.distribute): reductions of
# distributed vectors become rank-ordered global sums. One decomposition
# per process (one process per GPU).
COMM = None


def global_norm(h):
    """(||x||, flags) from a reduced ek_scalar_state, global in slab mode:
    the exact merge of the ranks' integer accumulators in repro mode
    (identical for every decomposition), else the
    rank-ordered fp64 sum."""
    if COMM is None:
        return float(h.val[1]), int(h.flag)
    flags = [int(h.flag & 1), int((h.flag >> 1) & 1), int((h.flag >> 2) & 1)]
    if h.repro:
        rows = COMM.allgather_ints([int(v) for v in h.xs] + flags)
        slots = (C.c_int64 * (N.XSLOTS * len(rows)))()
        for r, row in enumerate(rows):
            for i in range(N.XSLOTS):
                slots[r * N.XSLOTS + i] = row[i]
        s = N.lib().ek_xsum_value(slots, len(rows))
        nz, nf, nj = (sum(row[N.XSLOTS + i] for row in rows) for i in range(3))
    else:
        s, nz, nf, nj = COMM.allsum([float(h.val[0])] + [float(f) for f in flags])
    return math.sqrt(s), (1 if nz > 0 else 0) | (2 if nf > 0 else 0) | (4 if nj > 0 else 0)


def set_reproducible(on=True):
    """Order-independent sums on the Leja / power-iteration / integrator-norm
    path (csrc/ek_xsum.cuh): norms, and with them every decision and FD
    increment, are bitwise identical for whole-grid runs and for any slab
    decomposition. Slab decompositions switch it on (`slab.distribute`).
    Returns the previous setting."""
    return bool(N.lib().ek_set_repro(1 if on else 0))


def global_sum(v):
    return v if COMM is None else COMM.allsum([float(v)])[0]


def global_sum_state(h):
    """val[0] of a reduced ek_scalar_state (a sum: a dot product), global in
    slab mode — the exact merge of the ranks' integer accumulators in repro
    mode, as `global_norm`."""
    if COMM is None:
        return float(h.val[0])
    if h.repro:
        rows = COMM.allgather_ints([int(v) for v in h.xs])
        slots = (C.c_int64 * (N.XSLOTS * len(rows)))()
        for r, row in enumerate(rows):
            for i in range(N.XSLOTS):
                slots[r * N.XSLOTS + i] = row[i]
        return N.lib().ek_xsum_value(slots, len(rows))
    return COMM.allsum([float(h.val[0])])[0]


def norm2(x, st=None):
    """(||x||, flags) of a device vector; synchronises. flags bit0: any
    nonzero, bit1: any non-finite."""
    st = st or scalar_state()
    N.check(N.lib().ek_norm2(x.numel(), C.c_void_p(x.data_ptr()), st.ptr, 0,
                             work_ptr(), stream()), "ek_norm2")
    return global_norm(st.read())


def l1(x):
    return l1_many([x])[0]


def l1_many(xs):
    """L1 norms of up to 8 device vectors: one reduction kernel each into
    the slots of one state block, one host synchronisation."""
    st = scalar_state()
    wp = work_ptr()
    for i, x in enumerate(xs):
        N.check(N.lib().ek_l1(x.numel(), C.c_void_p(x.data_ptr()), st.ptr, i,
                              wp, stream()), "ek_l1")
    h = st.read()
    return [global_sum(float(h.val[i])) for i in range(len(xs))]


# ------------------------------------------------------- vexpr builder

class Expr:
    """Tiny expression tree mirroring NumPy elementwise evaluation order.

    Python builds `w3a * Ra + w3b * Rb` with the same associativity for Expr
    leaves as it does for numpy arrays, so compiling the tree to the stack
    program gives the reference's rounding sequence exactly."""

    __slots__ = ("op", "a", "b")
    __array_priority__ = 1000

    def __init__(self, op, a=None, b=None):
        self.op, self.a, self.b = op, a, b

    @staticmethod
    def wrap(x):
        if isinstance(x, Expr):
            return x
        if isinstance(x, torch.Tensor):
            return Expr("vec", x)
        if isinstance(x, (float, int, np.floating, np.integer)):
            return Expr("const", float(x))
        raise TypeError(f"unsupported operand {type(x)}")

    def __add__(self, o): return Expr("add", self, Expr.wrap(o))
    def __radd__(self, o): return Expr("add", Expr.wrap(o), self)
    def __sub__(self, o): return Expr("sub", self, Expr.wrap(o))
    def __rsub__(self, o): return Expr("sub", Expr.wrap(o), self)
    def __mul__(self, o): return Expr("mul", self, Expr.wrap(o))
    def __rmul__(self, o): return Expr("mul", Expr.wrap(o), self)
    def __truediv__(self, o): return Expr("div", self, Expr.wrap(o))
    def __rtruediv__(self, o): return Expr("div", Expr.wrap(o), self)
    def __neg__(self): return Expr("neg", self)


def V(t):
    """Leaf for a device vector (an Expr passes through: lazy engine results)."""
    return t if isinstance(t, Expr) else Expr("vec", t)


_OPC = {"add": N.VX_ADD, "sub": N.VX_SUB, "mul": N.VX_MUL, "div": N.VX_DIV}


class _Prog:
    def __init__(self):
        self.code, self.scal, self.ins = [], [], []

    def emit(self, op, arg=0):
        self.code.append(op | (arg << 8))

    def vec(self, t):
        for i, x in enumerate(self.ins):
            if x.data_ptr() == t.data_ptr() and x.numel() == t.numel():
                return i
        self.ins.append(t)
        return len(self.ins) - 1

    def const(self, v):
        self.scal.append(float(v))
        return len(self.scal) - 1

    def lower(self, e):
        if e.op == "vec":
            self.emit(N.VX_LOAD, self.vec(e.a))
        elif e.op == "const":
            self.emit(N.VX_CONST, self.const(e.a))
        elif e.op == "neg":
            self.lower(e.a)
            self.emit(N.VX_NEG)
        else:
            self.lower(e.a)
            self.lower(e.b)
            self.emit(_OPC[e.op])


LT_X, LT_MUL, LT_DIV, LT_MUL2 = 0, 1, 2, 3
LC_IN, LC_OUT, LC_TERMS = 8, 3, 6


def _scaled_vec(e):
    """(tensor, c) for c*x / x*c, else None."""
    if e.op == "mul":
        if e.a.op == "const" and e.b.op == "vec":
            return e.b.a, e.a.a
        if e.b.op == "const" and e.a.op == "vec":
            return e.a.a, e.b.a
    return None


def _term(e):
    """(tensor, mode, coef[, coef2]) for x, c*x, x*c, x/c, c1*(c2*x), -x,
    -(c*x); else None."""
    if e.op == "vec":
        return (e.a, LT_X, 1.0)
    if e.op == "mul":
        sv = _scaled_vec(e)
        if sv is not None:
            return (sv[0], LT_MUL, sv[1])
        # c1 * (c2 * x): a lazy m = 0 Leja result d0*b scaled by a stage weight
        if e.a.op == "const" and _scaled_vec(e.b) is not None:
            x, c2 = _scaled_vec(e.b)
            return (x, LT_MUL2, e.a.a, c2)
        if e.b.op == "const" and _scaled_vec(e.a) is not None:
            x, c2 = _scaled_vec(e.a)
            return (x, LT_MUL2, e.b.a, c2)
    if e.op == "div" and e.a.op == "vec" and e.b.op == "const":
        return (e.a.a, LT_DIV, e.b.a)
    if e.op == "neg":
        t = _term(e.a)
        if t is not None:
            return _negate(t)
    return None


def _negate(t):
    # a - x == a + (-1)*x, a - c*x == a + (-c)*x, a - x/c == a + x/(-c),
    # a - c1*(c2*x) == a + (-c1)*(c2*x): each is bit-identical in IEEE
    # arithmetic (negation is exact)
    v, m, c = t[:3]
    if m == LT_X:
        return (v, LT_MUL, -1.0)
    return (v, m, -c) + tuple(t[3:])


def _chain(e):
    """Left-deep +/- chain of terms -> list of terms, else None."""
    t = _term(e)
    if t is not None:
        return [t]
    if e.op in ("add", "sub"):
        left = _chain(e.a)
        right = _term(e.b)
        if left is None or right is None:
            return None
        return left + [right if e.op == "add" else _negate(right)]
    return None


def _fold(e):
    """(terms, fin_mode, fin_value) for fin(chain) or None."""
    terms = _chain(e)
    if terms is not None:
        return terms, 0, 0.0
    if e.op == "mul":
        if e.b.op == "const":
            inner = _chain(e.a)
            if inner is not None:
                return inner, 1, e.b.a
        if e.a.op == "const":
            inner = _chain(e.b)
            if inner is not None:
                return inner, 1, e.a.a
    if e.op == "div" and e.b.op == "const":
        inner = _chain(e.a)
        if inner is not None:
            return inner, 2, e.b.a
    return None


def _lincomb(outputs, length, rmode):
    """Lower to one ek_lincomb launch; False when the expressions do not fit."""
    folds = [_fold(Expr.wrap(ex)) for ex, _ in outputs]
    if len(outputs) > LC_OUT or any(f is None or len(f[0]) > LC_TERMS for f in folds):
        return False
    ins = []

    def idx(t):
        for i, x in enumerate(ins):
            if x.data_ptr() == t.data_ptr() and x.numel() == t.numel():
                return i
        ins.append(t)
        return len(ins) - 1

    nout = len(outputs)
    nterm = (C.c_int32 * nout)()
    src = (C.c_int32 * (nout * LC_TERMS))()
    mode = (C.c_int32 * (nout * LC_TERMS))()
    coef = (C.c_double * (nout * LC_TERMS))()
    coef2 = (C.c_double * (nout * LC_TERMS))()
    fin = (C.c_int32 * nout)()
    fval = (C.c_double * nout)()
    for o, (terms, fm, fv) in enumerate(folds):
        nterm[o] = len(terms)
        for t, term in enumerate(terms):
            v, m, c = term[:3]
            src[o * LC_TERMS + t] = idx(v)
            mode[o * LC_TERMS + t] = m
            coef[o * LC_TERMS + t] = float(c)
            coef2[o * LC_TERMS + t] = float(term[3]) if len(term) > 3 else 0.0
        fin[o] = fm
        fval[o] = float(fv)
    if len(ins) > LC_IN:
        return False
    return ins, nterm, src, mode, coef, coef2, fin, fval


def evaluate(outputs, length, norm=False, check=False, norm_diff=False, lazy=False):
    """Run one fused elementwise pass.

    outputs: list of (Expr, out_tensor_or_None). norm/check apply to the
    first expression (norm_diff: to the difference of the first two):
    returns (||value||, flags) after a sync when requested, else None.
    lazy (single GPU): return the unread state block of the reducing pass
    instead (linear combinations only; other expressions sync as usual).
    Linear combinations go to `ek_lincomb`; anything else to the general
    elementwise program `ek_vexpr`."""
    rmode = 2 if norm_diff else (1 if (norm or check) else 0)
    low = _lincomb(outputs, length, rmode)
    if low:
        ins, nterm, src, mode, coef, coef2, fin, fval = low
        outs = [o for _, o in outputs]
        st = scalar_state() if rmode else None
        N.check(N.lib().ek_lincomb(
            int(length), N.ptrs(ins), len(ins), N.ptrs(outs), len(outs), nterm, src, mode,
            coef, coef2, fin, fval, rmode, st.ptr if st else None, work_ptr() if st else None,
            stream()), "ek_lincomb")
        if st is None:
            return None
        if lazy and COMM is None:
            return st
        return global_norm(st.read())
    if norm_diff:
        a, b = outputs[0][0], outputs[1][0]
        evaluate(outputs, length)
        return evaluate([(Expr.wrap(a) - Expr.wrap(b), None)], length, norm=True)
    pr = _Prog()
    outs = []
    for i, (ex, out) in enumerate(outputs):
        pr.lower(Expr.wrap(ex))
        if out is not None:
            outs.append(out)
            pr.emit(N.VX_STORE, len(outs) - 1)
        if i == 0 and norm:
            pr.emit(N.VX_NORM, 0)
        if i == 0 and check:
            pr.emit(N.VX_CHECK)
        pr.emit(N.VX_POP)
    if len(pr.ins) > 8 or len(pr.scal) > 16 or len(pr.code) > 48:
        raise ValueError("elementwise program too large")
    code = (C.c_int32 * len(pr.code))(*pr.code)
    scal = (C.c_double * max(1, len(pr.scal)))(*pr.scal)
    st = scalar_state() if (norm or check) else None
    N.check(N.lib().ek_vexpr(
        int(length), code, len(pr.code), scal, len(pr.scal), N.ptrs(pr.ins),
        len(pr.ins), N.ptrs(outs), len(outs), st.ptr if st else None,
        work_ptr() if st else None, stream()), "ek_vexpr")
    if st is None:
        return None
    return global_norm(st.read())


def ev(expr, length=None, out=None):
    """Evaluate one expression into a new (or given) device vector."""
    if length is None:
        length = _length(Expr.wrap(expr))
    out = out if out is not None else empty(length)
    evaluate([(expr, out)], length)
    return out


def _length(e):
    if e.op == "vec":
        return e.a.numel()
    if e.op == "const":
        return None
    for c in (e.a, e.b):
        if isinstance(c, Expr):
            n = _length(c)
            if n is not None:
                return n
    return None


def copy(x):
    out = empty(x.numel())
    N.check(N.lib().ek_copy(C.c_void_p(out.data_ptr()), C.c_void_p(x.data_ptr()),
                            x.numel() * 8, 3, stream()), "ek_copy")
    return out


def sqrt_eps():
    return math.sqrt(float(np.finfo(np.float64).eps))
