"""ctypes binding of libexpkit_sm100.so (C ABI: include/expkit_sm100.h).

The product path has no fallback: if the library or a CUDA device is
missing, `lib()` raises RuntimeError and nothing computes.
"""

import ctypes as C
import os
from pathlib import Path

_HERE = Path(__file__).resolve().parent
LIB_NAME = "libexpkit_sm100.so"

EK_OK, EK_ERR_INVALID, EK_ERR_CUDA, EK_ERR_UNSUPPORTED, EK_ERR_NONFINITE = 0, 1, 2, 3, 4
ST_OK, ST_JV_NONFINITE, ST_NORM_NONFINITE, ST_REM_NONFINITE, ST_PEER_TIMEOUT = 0, 1, 2, 3, 4

# enum ek_problem
P_ADR, P_ALLEN_CAHN, P_BRUSS_PRINTED, P_BRUSS_STANDARD, P_GRAY_SCOTT, \
    P_SEMILINEAR, P_ADVDIFF2D, P_BURGERS2D, P_ADVDIFF3D = range(1, 10)
BC_NEUMANN, BC_PERIODIC, BC_DIRICHLET = 0, 1, 2
JAC_FD, JAC_ANALYTIC = 0, 1

# vexpr opcodes
VX_LOAD, VX_CONST, VX_ADD, VX_SUB, VX_MUL, VX_DIV, VX_NEG, VX_STORE, VX_POP, \
    VX_NORM, VX_CHECK, VX_ACC = range(1, 13)


class Grid(C.Structure):
    _fields_ = [("problem", C.c_int32), ("bc", C.c_int32), ("dim", C.c_int32),
                ("ncomp", C.c_int32), ("n", C.c_int64), ("rows", C.c_int64),
                ("row0", C.c_int64), ("slab", C.c_int32), ("pad_", C.c_int32),
                ("h", C.c_double), ("h2", C.c_double), ("two_h", C.c_double),
                ("prm", C.c_double * 8)]


class LejaState(C.Structure):
    _fields_ = [("ny", C.c_double), ("eps", C.c_double), ("nu", C.c_double),
                ("tol", C.c_double), ("m", C.c_int32), ("done", C.c_int32),
                ("status", C.c_int32), ("k", C.c_int32), ("active", C.c_uint32),
                ("fd_evals", C.c_int32), ("ticket", C.c_uint32),
                ("iters", C.c_int32), ("freeze", C.c_int32 * 8), ("defer", C.c_int32),
                ("p_init", C.c_int32), ("part", C.c_double * 8), ("lazy0", C.c_int32),
                ("pad_", C.c_int32)]


class Peer(C.Structure):
    """ek_peer: the window map of a slab decomposition in peer mode."""
    _fields_ = [("world", C.c_int32), ("rank", C.c_int32), ("up", C.c_int32),
                ("down", C.c_int32), ("rowlen", C.c_int64), ("ncomp", C.c_int32),
                ("pad_", C.c_int32), ("win", C.c_void_p * 8)]


PEER_HALO_OFFSET = 2048
XSLOTS, PART_SLOTS, PART_COUNT, PART_TAG = 5, 8, 5, 6


class ScalarState(C.Structure):
    _fields_ = [("val", C.c_double * 8), ("flag", C.c_int32),
                ("ticket", C.c_uint32), ("count", C.c_int32),
                ("status", C.c_int32), ("xs", C.c_int64 * 5), ("repro", C.c_int32),
                ("pad_", C.c_int32)]


class PowerState(C.Structure):
    _fields_ = [("lam", C.c_double), ("nw", C.c_double), ("nv", C.c_double),
                ("nu", C.c_double), ("tol_pi", C.c_double), ("it", C.c_int32),
                ("max_it", C.c_int32), ("done", C.c_int32),
                ("converged", C.c_int32), ("fd_evals", C.c_int32),
                ("ticket", C.c_uint32), ("status", C.c_int32),
                ("defer", C.c_int32), ("part", C.c_double * 8)]


class ArnoldiState(C.Structure):
    _fields_ = [("nrm", C.c_double), ("nvn", C.c_double), ("nu", C.c_double),
                ("tol", C.c_double), ("beta", C.c_double), ("j", C.c_int32),
                ("happy", C.c_int32), ("status", C.c_int32),
                ("fd_evals", C.c_int32), ("ticket", C.c_uint32),
                ("defer", C.c_int32), ("part", C.c_double * 24)]


_P = C.c_void_p
_D = C.c_double
_I = C.c_int
_L = C.c_int64
_PP = C.POINTER(C.c_void_p)

_SIGS = {
    "ek_last_error": (C.c_char_p, []),
    "ek_version": (_I, []),
    "ek_launch_count": (C.c_longlong, []),
    "ek_set_tma": (_I, [_I]),
    "ek_set_march": (_I, [_I]),
    "ek_set_repro": (_I, [_I]),
    "ek_xsum_value": (_D, [C.POINTER(C.c_int64), _I]),
    "ek_xsum_host": (None, [_P, _L, _I, C.POINTER(C.c_int64)]),
    "ek_selftest_xsum": (_I, [_L, _P, _I, _I, _P, _P, _P]),
    "ek_grid_len": (_L, [C.POINTER(Grid)]),
    "ek_workspace_bytes": (_L, [C.POINTER(Grid)]),
    "ek_copy": (_I, [_P, _P, _L, _I, _P]),
    "ek_sync": (_I, [_P]),
    "ek_rhs": (_I, [C.POINTER(Grid), _P, _P, _PP, _P]),
    "ek_rhs_norm": (_I, [C.POINTER(Grid), _P, _P, _P, _P, _PP, _P]),
    "ek_jv": (_I, [C.POINTER(Grid), _I, _P, _P, _P, _D, _P, _P, _P, _PP, _P]),
    "ek_remainder": (_I, [C.POINTER(Grid), _I, _P, _P, _P, _D, _P, _P, _P, _PP, _P]),
    "ek_remainder_combo": (_I, [C.POINTER(Grid), _I, _P, _P, _P, _D, _P, _I, _PP, _P,
                                C.POINTER(_D), C.POINTER(_D), C.POINTER(_D), _P, _P, _PP, _P]),
    "ek_remainder_combo_dev": (_I, [C.POINTER(Grid), _I, _P, _P, _P, _P, _P, _P, _I, _PP, _P,
                                    C.POINTER(_D), C.POINTER(_D), C.POINTER(_D), _P, _P, _PP,
                                    _P]),
    "ek_leja_begin_len": (_I, [_L, _P, _PP, _I, _P, _P, _P, _P]),
    "ek_leja_call": (_I, [C.POINTER(Grid), _I, _P, _P, _P, _PP, _PP, _I, _P, _P, _D, _D, _P,
                          _I, _I, _I, _D, _P, _P, _P]),
    "ek_leja_run": (_I, [C.POINTER(Grid), _I, _P, _P, _P, _PP, _PP, _I, _P, _I,
                         _I, _I, _D, _P, _P, _PP, _P]),
    "ek_leja_run_graph": (_I, [C.POINTER(Grid), _I, _P, _P, _P, _PP, _PP, _I, _P, _I,
                               _I, _I, _D, _P, _P, _P]),
    "ek_leja_run_seq": (_I, [C.POINTER(Grid), _I, _P, _P, _PP, _PP, _I, _P, _I, _I, _D, _P, _P,
                             _P]),
    "ek_leja_combine": (_I, [_L, _PP, _I, _PP, _I, _P, _I, _I, _P, _P]),
    "ek_leja_call_seq": (_I, [C.POINTER(Grid), _I, _P, _P, _P, _PP, _PP, _I, _PP, _I, _P, _P,
                              _D, _D, _P, _I, _D, _P, _P, _P]),
    "ek_leja_update": (_I, [_L, _P, _P, _P, _PP, _I, _P, _I, _I, _D, _I, _P,
                            _P, _P]),
    "ek_power_run": (_I, [C.POINTER(Grid), _I, _P, _P, _P, _PP, _I, _I, _P, _P,
                          _PP, _P]),
    "ek_power_norm": (_I, [_L, _P, _I, _P, _P, _P]),
    "ek_leja_decide": (_I, [_P, _P, _I, _P, _I, _I, _I, _I, _I, _P]),
    "ek_power_decide": (_I, [_P, _P, _I, _I, _I, _P]),
    "ek_peer_window_bytes": (_L, [C.POINTER(Grid)]),
    "ek_ipc_alloc": (_I, [_L, C.POINTER(_P), _P]),
    "ek_ipc_open": (_I, [_P, C.POINTER(_P)]),
    "ek_ipc_close": (_I, [_P]),
    "ek_ipc_free": (_I, [_P]),
    "ek_leja_run_peer": (_I, [C.POINTER(Grid), _I, _P, _P, _P, _PP, _PP, _I, _P, _I,
                              _I, _I, _D, _P, _P, _PP, _P, _P, _L, _P]),
    "ek_leja_run_peer_phase": (_I, [C.POINTER(Grid), _I, _P, _P, _P, _PP, _PP, _I, _P, _I,
                                    _I, _I, _D, _P, _P, _PP, _P, _P, _L, _I, _P]),
    "ek_arnoldi_init": (_I, [_L, _I, _P, C.POINTER(_D), _P, _P, _P, _P]),
    "ek_arnoldi_slab_init": (_I, [_L, _I, _P, C.POINTER(_D), _P, _P, _P, _P]),
    "ek_arnoldi_slab_pass": (_I, [C.POINTER(Grid), _I, _P, _P, _PP, _PP, C.POINTER(_I), _I,
                                  _D, _I, _I, _P, _P, _I, _I, _I, _D, _P, _PP, _P]),
    "ek_arnoldi_slab_decide": (_I, [_PP, _L, _I, _I, _I, _P, _I, _P, _P, _I, _I, _P]),
    "ek_arnoldi_run": (_I, [C.POINTER(Grid), _I, _P, _P, _PP, _PP,
                            C.POINTER(_I), _I, _D, _I, _I, _P, _P, _I, _I, _I,
                            _D, _P, _P]),
    "ek_arnoldi_augment": (_I, [_L, _I, _P, _PP, _I, _I, _PP, C.POINTER(_I),
                                _I, _D, _P, _I, _P, _P, _P]),
    "ek_arnoldi_orth": (_I, [_L, _I, _PP, _I, _I, _P, _I, _P, _P, _P]),
    "ek_basis_combine": (_I, [_L, _PP, C.POINTER(_D), _I, _P, _P]),
    "ek_vexpr": (_I, [_L, C.POINTER(C.c_int32), _I, C.POINTER(_D), _I, _PP, _I,
                      _PP, _I, _P, _P, _P]),
    "ek_norm2": (_I, [_L, _P, _P, _I, _P, _P]),
    "ek_l1": (_I, [_L, _P, _P, _I, _P, _P]),
    "ek_selftest_div": (_I, [_L, _P, _P, _P, _P, _P]),
    "ek_lincomb": (_I, [_L, _PP, _I, _PP, _I, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                        C.POINTER(C.c_int32), C.POINTER(_D), C.POINTER(_D),
                        C.POINTER(C.c_int32), C.POINTER(_D), _I, _P, _P, _P]),
    "ek_dense_gemv": (_I, [_L, _P, _P, _P, _P]),
    "ek_ctx_create": (_P, [_I, _P]),
    "ek_ctx_destroy": (None, [_P]),
    "ek_op_create": (_P, [_P, C.POINTER(Grid), _I]),
    "ek_op_destroy": (None, [_P]),
    "ek_op_linearize": (_I, [_P, _P, _P, C.POINTER(_D)]),
    "ek_op_rhs": (_I, [_P, _P, _P]),
    "ek_op_jv": (_I, [_P, _P, _P]),
    "ek_power_step": (_I, [_P, _P, _P, C.POINTER(_D)]),
    "ek_axpby": (_I, [_L, _D, _P, _D, _P, _P, _P]),
    "ek_dot_multi": (_I, [_L, _P, _PP, _I, _P, C.POINTER(_D), _P, _P]),
}

_lib = None


def lib_path():
    # EK_LIB_PATH: an alternative build of the same library (tools/ A/B runs)
    return Path(os.environ["EK_LIB_PATH"]) if os.environ.get("EK_LIB_PATH") else _HERE / LIB_NAME


def lib():
    """Load the native library (once). Raises RuntimeError when it is absent:
    there is deliberately no CPU fallback."""
    global _lib
    if _lib is not None:
        return _lib
    path = lib_path()
    if not path.exists():
        raise RuntimeError(
            f"{LIB_NAME} not built ({path}); run `python __graft_entry__.py` "
            "or paper_2211_08948_b200._build.build_native()")
    handle = C.CDLL(str(path), mode=os.RTLD_GLOBAL if hasattr(os, "RTLD_GLOBAL") else 0)
    for name, (res, args) in _SIGS.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    if os.environ.get("EK_TMA_MODE"):  # A/B runs of the stencil staging (tools/)
        handle.ek_set_tma(int(os.environ["EK_TMA_MODE"]))
    if os.environ.get("EK_MARCH_MASK"):
        handle.ek_set_march(int(os.environ["EK_MARCH_MASK"]))
    _lib = handle
    return _lib


def exported_symbols():
    return list(_SIGS)


class NativeError(RuntimeError):
    pass


def check(rc, what=""):
    if rc == EK_OK:
        return
    msg = lib().ek_last_error().decode(errors="replace")
    if rc == EK_ERR_INVALID:
        raise ValueError(f"{what}: {msg}")
    if rc == EK_ERR_NONFINITE:
        raise FloatingPointError(f"{what}: {msg}")
    raise NativeError(f"{what}: {msg} (status {rc})")


def ptrs(tensors):
    """C array of device pointers (None -> NULL)."""
    arr = (C.c_void_p * max(1, len(tensors)))()
    for i, t in enumerate(tensors):
        arr[i] = None if t is None else t.data_ptr()
    return arr
