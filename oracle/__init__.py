"""CPU oracle for the phi-action hot path — TEST INFRASTRUCTURE ONLY.

This package is a plain NumPy/SciPy restatement of the reference `expkit`
algorithms on the north-star path (arXiv 2211.08948; reference tree
`/root/reference/pkg/src/expkit`). Every function cites the reference
`file:line` it restates, and keeps the reference's elementwise evaluation
order so that, on the same host with the same numpy/scipy, its outputs are
bit-identical to the reference's.

Who may import this package: `tests/`, `__graft_entry__.smoke()` and the
`cpu_baseline` / `--impl reference` legs of `bench.py` — and there only as
the checker or the timed CPU baseline. The product package
`paper_2211_08948_b200` never imports it; the product path runs on the GPU
through `libexpkit_sm100.so` and fails loudly if that library is missing.

Pinning: `tests/golden/make_golden.py` imports the real reference (only
possible in the build container, where `/root/reference` exists) and writes
golden fixtures under `tests/golden/`; `tests/test_oracle_golden.py`
checks this oracle against them bit-for-bit. For the BASELINE problems the
reference does not define (see `np_fields.py`), the golden vectors are the
*reference engines* driven by this oracle's NumPy right-hand sides.

Modules:
  np_fields    — PDE right-hand sides, FD Jacobian action, analytic Jv
  np_phi       — Leja points, divided differences, Leja interpolation,
                 KIOPS, power iteration / spectrum estimate
  np_integrate — embedded exponential integrators and the time loops
"""

from . import np_fields, np_phi, np_integrate  # noqa: F401
