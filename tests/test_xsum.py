"""Order-independent sums (csrc/ek_xsum.cuh): the integer
accumulator behind the repro mode of the reducing kernels.

CPU: the host restatement the library exports (`ek_xsum_host`, the same
code the kernels run per term) gives the correctly rounded exact sum
(`math.fsum`) and the same accumulator value for every permutation and
partition of the terms. GPU: the kernels' reduction path reproduces those
bits for any grid size, and the norm kernels / fused stencil passes in repro
mode agree with it."""

import ctypes as C
import math

import numpy as np
import pytest

from paper_2211_08948_b200 import _native as N


def _lib():
    try:
        return N.lib()
    except RuntimeError:
        pytest.skip("native library not built")


def _host(x, sq):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = (C.c_int64 * N.XSLOTS)()
    _lib().ek_xsum_host(x.ctypes.data_as(C.c_void_p), len(x), sq, out)
    return list(out)


def _value(slot_lists):
    flat = (C.c_int64 * (N.XSLOTS * len(slot_lists)))()
    for r, sl in enumerate(slot_lists):
        for i, v in enumerate(sl):
            flat[r * N.XSLOTS + i] = v
    return _lib().ek_xsum_value(flat, len(slot_lists))


def _vectors():
    rng = np.random.default_rng(7)
    for trial in range(60):
        n = int(rng.integers(1, 4000))
        kind = trial % 6
        if kind == 0:
            yield rng.standard_normal(n)
        elif kind == 1:  # wide dynamic range
            yield rng.standard_normal(n) * 10.0 ** rng.integers(-12, 12, size=n)
        elif kind == 2:  # near the bottom of the exponent range
            yield rng.standard_normal(n) * 1e-290
        elif kind == 3:  # heavy cancellation
            a = rng.standard_normal(n) * 1e8
            yield np.concatenate([a, -a, rng.standard_normal(5)])
        elif kind == 4:
            yield rng.uniform(-1, 1, n) * 2.0 ** int(rng.integers(-200, 200))
        else:
            yield np.zeros(n)


def test_host_accumulator_is_the_correctly_rounded_exact_sum():
    for x in _vectors():
        assert _value([_host(x, 0)]) == math.fsum(x.tolist())
        assert _value([_host(x, 1)]) == math.fsum((x * x).tolist())


def test_host_accumulator_is_order_and_partition_independent():
    rng = np.random.default_rng(3)
    for x in _vectors():
        want = _value([_host(x, 0)])
        xp = x[rng.permutation(len(x))]
        assert _value([_host(xp, 0)]) == want
        cuts = sorted(int(c) for c in rng.integers(0, len(x) + 1, size=7))
        parts = np.split(xp, cuts)
        assert _value([_host(p, 0) for p in parts]) == want


def test_non_finite_terms_give_a_non_finite_sum():
    x = np.array([1.0, np.inf, 2.0])
    assert not math.isfinite(_value([_host(x, 0)]))
    x = np.array([1.0, np.nan])
    assert not math.isfinite(_value([_host(x, 1)]))
    assert _value([_host(np.zeros(0), 0)]) == 0.0


@pytest.mark.gpu
def test_device_reduction_path_matches_host_bits_for_any_grid():
    import torch
    from paper_2211_08948_b200 import _device as D
    lib = _lib()
    rng = np.random.default_rng(11)
    for n in (1, 255, 4097, 1 << 20):
        x = rng.standard_normal(n) * 10.0 ** rng.integers(-6, 6, size=n)
        xd = D.to_dev(x)
        for sq in (0, 1):
            want = _host(x, sq)
            for blocks in (1, 3, 148, 2368):
                st = D.scalar_state()
                slots = torch.zeros(N.XSLOTS, dtype=torch.int64, device=xd.device)
                N.check(lib.ek_selftest_xsum(n, C.c_void_p(xd.data_ptr()), sq, blocks, st.ptr,
                                             C.c_void_p(slots.data_ptr()), D.stream()), "xsum")
                got = slots.cpu().tolist()
                assert _value([got]) == _value([want])
                assert float(st.read().val[0]) == _value([want])


@pytest.mark.gpu
def test_norm_kernels_in_repro_mode_equal_the_exact_sum():
    import torch
    from paper_2211_08948_b200 import _device as D
    rng = np.random.default_rng(5)
    x = rng.standard_normal(300001)
    xd = D.to_dev(x)
    exact = math.sqrt(math.fsum((x * x).tolist()))
    old = D.set_reproducible(True)
    try:
        nrm, _ = D.norm2(xd)
        assert nrm == exact
        # a stage expression with a fused norm (k_lincomb), and a general
        # elementwise program (k_vexpr)
        y = rng.standard_normal(300001)
        yd = D.to_dev(y)
        z = x + (-0.25) * y
        got, _ = D.evaluate([(D.V(xd) - 0.25 * D.V(yd), None)], xd.numel(), norm=True)
        assert got == math.sqrt(math.fsum((z * z).tolist()))
        w = x * y
        got, _ = D.evaluate([(D.V(xd) * D.V(yd), None)], xd.numel(), norm=True)
        assert got == math.sqrt(math.fsum((w * w).tolist()))
    finally:
        D.set_reproducible(old)
    nrm2, _ = D.norm2(xd)  # default mode: same value within an ulp or two
    assert abs(nrm2 - exact) <= 4e-16 * exact
    # the general elementwise program's reductions in the default mode
    # (linalg.dot: VX_ACC; an expression norm: VX_NORM)
    from paper_2211_08948_b200 import linalg as LA
    got = LA.dot(xd, yd)
    want = math.fsum((x * y).tolist())
    assert abs(got - want) <= 1e-12 * math.sqrt(len(x))
    got, _ = D.evaluate([(D.V(xd) * D.V(yd), None)], xd.numel(), norm=True)
    assert abs(got - math.sqrt(math.fsum((w * w).tolist()))) <= 1e-13 * got
    old = D.set_reproducible(True)
    try:
        assert LA.dot(xd, yd) == want
    finally:
        D.set_reproducible(old)


@pytest.mark.gpu
@pytest.mark.parametrize("name,n,fd", [("brusselator_periodic", 96, True),
                                       ("allen_cahn", 65, True), ("advdiff2d", 128, False)])
def test_repro_mode_is_independent_of_the_kernel_staging(name, n, fd):
    """The stagings of the 2-D stencil passes (register-staged, 32 x 8 TMA
    chunks, row march) give bit-identical pointwise results and differ only in
    how the norms' partial sums are grouped (ek_set_tma). With the
    order-independent sums nothing is left to differ: a whole vertical Leja
    call — FD increments and freeze decisions included — has the same bits
    under every staging (n = 65: odd rows, the register-staged fallback)."""
    import paper_2211_08948_b200 as ek
    from paper_2211_08948_b200 import _device as D, ext
    lib = _lib()
    p = ek.make_problem(name, n=n) if name in ek.PROBLEMS else ext.make_ext_problem(name, n=n)
    xi = ek.get_leja_points(400)
    old_r = D.set_reproducible(True)
    old_t = lib.ek_set_tma(-1)
    try:
        outs = []
        for mode in (0, 1, 2, 3):
            lib.ek_set_tma(mode)
            rhs = ek.CountingRhs(p.rhs)
            sys_ = ek.make_linearized(rhs, p.u0, jac_factory=None if fd else p.jac_factory)
            lam, _ = ek.power_iterate(sys_.J)
            est = ek.make_estimate(lam)
            dt = 25.0 / abs(est.alpha)
            r = ek.leja_interpolate_vertical(sys_.J, sys_.f_n * dt, 1, [0.5, 1.0], dt, est,
                                             1e-10, xi=xi)
            outs.append((lam, r))
        lam0, r0 = outs[0]
        assert r0.iters > 3
        for lam, r in outs[1:]:
            assert lam == lam0
            assert r.iters == r0.iters and r.freeze_iters == r0.freeze_iters
            for x, y in zip(r.vectors, r0.vectors):
                assert np.array_equal(x, y)
    finally:
        lib.ek_set_tma(old_t)
        D.set_reproducible(old_r)
