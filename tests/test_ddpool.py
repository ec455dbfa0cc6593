"""Divided-difference worker pool (`_ddpool`): host-only.

The pool computes the Leja tables beyond the first chunk in worker
processes. Its tables must be the bits `leja.divided_differences` produces
with one BLAS thread (the reference's own setting), it must not deadlock
when prefetched tables are never collected, and `_dd_cached` must give the
same tables with and without it.
"""

import numpy as np
import pytest

from paper_2211_08948_b200 import _ddpool, _dense, leja
from paper_2211_08948_b200.spectrum import make_estimate


@pytest.fixture(scope="module")
def xi():
    return leja.generate_leja_points(400)


def _one_thread():
    from threadpoolctl import threadpool_limits
    return threadpool_limits(limits=1, user_api="blas")


def test_pool_tables_bit_identical(xi):
    pool = _ddpool.DDPool(3)
    try:
        args = [(l, h, -1234.5, 617.25, xi, m) for l in (1, 4) for h in (1e-4, 3e-3)
                for m in (64, 160, 400)]
        for i, a in enumerate(args):
            pool.submit(i, a)
        got = [pool.collect(i) for i in reversed(range(len(args)))][::-1]
        with _one_thread():
            ref = [_dense.phi_divided_differences(*a) for a in args]
        for (ok, d), r in zip(got, ref):
            assert ok and np.array_equal(d, r)
    finally:
        pool.close()


def test_uncollected_results_do_not_block(xi):
    pool = _ddpool.DDPool(1)
    try:
        for i in range(60):  # ~3.3 KB per answer: more than a pipe buffer
            pool.submit(("x", i), (1, 1e-3 * (i + 1), -10.0, 5.0, xi, 400))
        pool.submit("last", (2, 1e-3, -10.0, 5.0, xi, 64))
        ok, d = pool.collect("last")
        assert ok and d.shape == (64,)
        assert len(pool.done) <= 256
    finally:
        pool.close()


def test_worker_error_is_reported(xi):
    pool = _ddpool.DDPool(1)
    try:
        pool.submit("bad", (1, 1e-3, -10.0, 5.0, "not an array", 64))
        ok, msg = pool.collect("bad")
        assert not ok and isinstance(msg, str)
    finally:
        pool.close()


def test_dd_cached_same_with_and_without_pool(xi, monkeypatch):
    est = make_estimate(2.5e4)
    cases = [(1, 2e-3, 96), (3, 4e-3, 128), (1, 2e-3, 32)]
    leja._DD_CACHE.clear()
    assert _ddpool.pool() is not None
    for l, h, m in cases:  # submitted ahead, collected below
        leja._dd_prefetch(l, h, est, xi, m)
    with_pool = [leja._dd_cached(l, h, est, xi, m).copy() for l, h, m in cases]
    leja._DD_CACHE.clear()
    monkeypatch.setattr(_ddpool, "_DISABLED", True)
    without = [leja._dd_cached(l, h, est, xi, m).copy() for l, h, m in cases]
    leja._DD_CACHE.clear()
    for a, b in zip(with_pool, without):
        assert np.array_equal(a, b)
    # and both are the reference's divided differences (one BLAS thread)
    with _one_thread():
        for (l, h, m), a in zip(cases, with_pool):
            assert np.array_equal(a, leja.divided_differences(l, h, est, xi, m).d)
