"""CPU-side checks of the product package (no GPU needed):

  * the C-ABI library loads and exports every symbol include/expkit_sm100.h
    declares, and the ctypes structs match the header's layouts;
  * the public API mirrors the reference's 40 exports and registries;
  * host-side logic (controllers, ICs, Leja points / divided differences,
    the elementwise-program compiler) matches the oracle bit for bit.
"""

import ctypes as C
import math
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2211_08948_b200 as ek
from paper_2211_08948_b200 import _device as D, _native as N, ext
from paper_2211_08948_b200 import problems as P
from paper_2211_08948_b200 import timestep as T
from oracle import np_fields as OF, np_integrate as OI, np_phi as OP

REPO = Path(__file__).resolve().parents[1]
HEADER = REPO / "include" / "expkit_sm100.h"


def header_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ek_[a-z0-9_]+)\s*\(", text)))


def test_library_built_and_exports_header_symbols():
    path = N.lib_path()
    assert path.exists(), "run __graft_entry__.build() first"
    lib = C.CDLL(str(path))
    for name in header_functions():
        assert hasattr(lib, name), name
    assert set(header_functions()) == set(N.exported_symbols())


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", str(N.lib_path())],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def _header_struct_fields(name):
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    body = re.search(r"typedef struct %s \{(.*?)\} %s;" % (name, name), text, re.S).group(1)
    fields = []
    for line in body.split(";"):
        m = re.search(r"(\w+)\s+(\w+)(\[\d+\])?\s*$", line.strip())
        if m:
            fields.append(m.group(2))
    return fields


@pytest.mark.parametrize("cname,py", [("ek_grid", N.Grid), ("ek_leja_state", N.LejaState),
                                      ("ek_scalar_state", N.ScalarState),
                                      ("ek_power_state", N.PowerState),
                                      ("ek_arnoldi_state", N.ArnoldiState)])
def test_ctypes_structs_match_header(cname, py):
    assert _header_struct_fields(cname) == [f[0] for f in py._fields_]
    assert C.sizeof(py) % 8 == 0


def test_grid_len_on_host():
    g = P.make_grid(N.P_BRUSS_STANDARD, N.BC_PERIODIC, 2, 2, 64, 1 / 64)
    assert N.lib().ek_grid_len(C.byref(g)) == 2 * 64 * 64
    g3 = P.make_grid(N.P_ADVDIFF3D, N.BC_PERIODIC, 3, 1, 16, 1 / 16)
    assert N.lib().ek_grid_len(C.byref(g3)) == 16 ** 3
    gs = P.make_grid(N.P_SEMILINEAR, N.BC_DIRICHLET, 1, 1, 20, 1 / 21)
    assert N.lib().ek_grid_len(C.byref(gs)) == 21


def test_public_api_surface():
    assert len(ek.__all__) == 40  # the reference list, incl. __version__
    for name in ek.__all__:
        assert hasattr(ek, name), name
    assert ek.PROBLEMS == ("adr", "allen_cahn", "brusselator", "gray_scott", "semilinear")
    assert ek.INTEGRATORS == ("epirk4s3", "epirk4s3a", "epirk5p1", "exprb43", "exprb53s3")
    assert ek.SCHEMES == ("leja", "kiops", "lekry")
    assert ek.LEKRY_INTEGRATORS == frozenset({"epirk4s3", "epirk4s3a", "exprb53s3"})
    with pytest.raises(ValueError):
        ek.make_problem("heat")
    import importlib
    K = importlib.import_module("paper_2211_08948_b200.kiops")
    L = importlib.import_module("paper_2211_08948_b200.leja")
    S = importlib.import_module("paper_2211_08948_b200.spectrum")
    for mod, names in ((K, ["AugmentedSystem", "KiopsStats", "arnoldi_iop", "augmented_apply"]),
                       (L, ["DEFAULT_NUM_POINTS", "generate_leja_points", "_cached_points"]),
                       (S, ["GAMMA_MIN"]),
                       (T, ["COST_ALPHA", "COST_BETA", "COST_DELTA", "COST_LAMBDA"]),
                       (P, ["brusselator_problem", "semilinear_forcing", "semilinear_problem"])):
        for n in names:
            assert hasattr(mod, n), (mod.__name__, n)


# ---------------------------------------------------------- host numerics

@pytest.mark.parametrize("args", [(0.1, 1e-4, 1e-6, 4), (0.2, 0.0, 1e-6, 4),
                                  (0.2, 1e6, 1e-6, 3), (1e-5, 3.3e-9, 1e-8, 5)])
def test_traditional_dt_same_as_oracle(args):
    assert ek.traditional_dt(*args) == OI.traditional_dt(*args)


@pytest.mark.parametrize("args", [(0.3, 0.2, 7.0, 7.0), (1.0, 1.0 - 1e-12, 1e30, 1.0),
                                  (2.0, 1.0, 17.0, 10.0), (0.4, 0.4, 9.0, 5.0),
                                  (1e-4, 3e-5, 12.0, 9.0)])
def test_cost_dt_same_as_oracle(args):
    assert ek.cost_dt(*args) == OI.cost_dt(*args)


def test_controller_validation():
    with pytest.raises(ValueError):
        ek.traditional_dt(0.0, 1.0, 1.0, 4)
    for args in ((0.0, 0.1, 1, 1), (0.1, 0.1, 0, 1), (0.1, -0.1, 1, 1)):
        with pytest.raises(ValueError):
            ek.cost_dt(*args)


def test_leja_points_and_dd_bitexact(golden):
    xi = ek.generate_leja_points(400)
    assert np.array_equal(xi, golden["leja_points/xi"])
    for l, h, lam, m in [(0, 1.0, -4.0, 32), (3, 2.5, -30.0, 64), (4, 0.1, -300.0, 96)]:
        est = ek.make_estimate(lam)
        assert np.array_equal(ek.divided_differences(l, h, est, xi, m).d,
                              OP.newton_coeffs(l, h, OP.estimate(lam), xi, m))


def test_make_estimate_same_as_oracle():
    for lam in (-20.0, 0.0, 3.3e5, -1e-20):
        a, b = ek.make_estimate(lam, 1.1), OP.estimate(lam, 1.1)
        assert (a.alpha, a.beta, a.c, a.gamma) == (b.alpha, b.beta, b.c, b.gamma)


@pytest.mark.parametrize("mk,ok", [
    (lambda: ek.make_problem("adr", alpha=0.1, n=17), lambda: OF.make("adr", alpha=0.1, n=17)),
    (lambda: ek.make_problem("allen_cahn", n=33), lambda: OF.make("allen_cahn", n=33)),
    (lambda: ek.make_problem("brusselator", n=12), lambda: OF.make("brusselator", n=12)),
    (lambda: ek.make_problem("gray_scott", n=16), lambda: OF.make("gray_scott", n=16)),
    (lambda: ek.make_problem("semilinear", n=20), lambda: OF.make("semilinear", n=20)),
    (lambda: ext.advdiff2d_problem(n=64, peclet=10.0), lambda: OF.advdiff2d(n=64, peclet=10.0)),
    (lambda: ext.allen_cahn_periodic_problem(n=64), lambda: OF.allen_cahn_periodic(n=64)),
    (lambda: ext.burgers2d_problem(n=64), lambda: OF.burgers2d(n=64)),
    (lambda: ext.brusselator_periodic_problem(n=64), lambda: OF.brusselator_periodic(n=64)),
    (lambda: ext.advdiff3d_problem(n=16), lambda: OF.advdiff3d(n=16)),
])
def test_initial_conditions_bitexact(mk, ok):
    a, b = mk(), ok()
    assert np.array_equal(a.u0, b.u0)
    assert a.t_final == b.t_final


def test_grid_scalars_follow_python_evaluation():
    p = ek.make_problem("allen_cahn", alpha=1e-2, n=33)
    h = 2.0 / 32
    assert p.rhs.grid.h == h and p.rhs.grid.h2 == h**2 and p.rhs.grid.two_h == 2.0 * h
    q = ext.advdiff2d_problem(n=64, peclet=10.0)
    assert q.params["dt_cfl"] == OF.advdiff2d(n=64, peclet=10.0).params["dt_cfl"]


# ------------------------------------------------------ expression compiler

def _fake(ptr, n=4):
    class T:
        def __init__(self, p):
            self.p = p

        def data_ptr(self):
            return self.p

        def numel(self):
            return n
    return T(ptr)


def test_expression_lowering_keeps_numpy_order():
    import torch
    u, ra, rb = (torch.empty(0) for _ in range(3))
    pr = D._Prog()
    pr.lower(D.Expr.wrap((32.0 * D.V(ra) + -13.5 * D.V(rb)) * 0.25))
    ops = [w & 0xFF for w in pr.code]
    assert ops == [N.VX_CONST, N.VX_LOAD, N.VX_MUL, N.VX_CONST, N.VX_LOAD, N.VX_MUL,
                   N.VX_ADD, N.VX_CONST, N.VX_MUL]
    assert pr.scal == [32.0, -13.5, 0.25]
    pr2 = D._Prog()
    pr2.lower(D.Expr.wrap(1.0 - D.V(u) / 3.0))
    assert [w & 0xFF for w in pr2.code] == [N.VX_CONST, N.VX_LOAD, N.VX_CONST, N.VX_DIV,
                                            N.VX_SUB]


def test_cpu_has_no_silent_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError):
        ek.norm_l2(np.ones(3))
    p = ek.make_problem("allen_cahn", n=8)
    with pytest.raises(RuntimeError):
        p.rhs(p.u0)


def test_monkeypatch_contract_globals():
    # adaptive_loop resolves the controllers through module globals
    code = T.adaptive_loop.__code__
    assert "traditional_dt" in code.co_names and "cost_dt" in code.co_names
    from paper_2211_08948_b200 import leja as L
    assert "generate_leja_points" in L.get_leja_points.__code__.co_names
    assert math.isclose(T.COST_LAMBDA, OI.COST_LAMBDA)


def test_batched_divided_differences_bit_identical():
    """The batched exponential of a vertical group's tables gives every
    table the bits of its own scipy expm call (leja.py:88-111)."""
    from paper_2211_08948_b200._dense import (phi_divided_differences,
                                               phi_divided_differences_many)
    xi = ek.get_leja_points(400)
    rng = np.random.default_rng(3)
    for _ in range(200):
        c = -rng.uniform(1.0, 1e6)
        g = abs(c) / 2.0
        dt = 10.0 ** rng.uniform(-12, -1)
        l = int(rng.integers(0, 5))
        m = int(rng.choice([4, 16, 32]))
        hs = [ci * dt for ci in sorted(rng.uniform(0.05, 1.0, int(rng.integers(1, 4))))]
        for h, d in zip(hs, phi_divided_differences_many(l, hs, c, g, xi, m)):
            assert np.array_equal(d, phi_divided_differences(l, h, c, g, xi, m))


def test_bench_byte_models_of_the_leja_call():
    """bench.py's roofline bytes: per-iteration accumulation counts the live
    accumulators of every iteration; the deferred form
    counts k = 0 iterations plus one combine pass of M + 1 + k vectors."""
    import importlib.util
    from pathlib import Path
    spec = importlib.util.spec_from_file_location(
        "bench_root", Path(__file__).resolve().parents[1] / "bench.py")
    B = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(B)
    n = 1000
    prof = {"n": n, "fd": True, "k": 3, "iters": 4, "freeze": [2, 4, 4]}
    alg, pas, launches = B.leja_bytes(prof)
    # live accumulators per iteration: 3, 3, 2, 2
    assert launches == 4
    assert alg == 8 * n * (4 * 4 + 2 * (3 + 3 + 2 + 2))
    assert pas == 8 * n * (3 * 4 + 2 * (3 + 3 + 2 + 2))
    assert B.combine_bytes(prof) == 0
    prof["deferred"] = True
    alg, pas, launches = B.leja_bytes(prof)
    assert alg == pas == 8 * n * 4 * 4 and launches == 4
    assert B.combine_bytes(prof) == 8 * n * (4 + 1 + 3)
    lin = {"n": n, "fd": False, "k": 2, "iters": 3, "freeze": [3, 3], "deferred": True}
    assert B.leja_bytes(lin)[0] == 8 * n * 2 * 3
