"""Shared pytest configuration.

Markers:
  gpu  — needs a B200 (CUDA) and the built libexpkit_sm100.so; run on the GPU
         box with `pytest -m gpu`. Everything else runs on the CPU here.
"""

import os
import sys
from pathlib import Path

import numpy as np
import pytest

REPO = Path(__file__).resolve().parents[1]
if str(REPO) not in sys.path:
    sys.path.insert(0, str(REPO))

# The CPU oracle must run single-threaded BLAS (threaded
# OpenBLAS norms are pathologically slow on small vectors).
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")

GOLDEN_PATH = REPO / "tests" / "golden" / "golden.npz"


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: requires a CUDA device (B200) and the native library")


@pytest.fixture(scope="session")
def golden():
    """Golden fixtures written by tests/golden/make_golden.py from the real
    reference. Returned as a dict-like of arrays keyed "<case>/<field>"."""
    with np.load(GOLDEN_PATH, allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def xi(golden):
    return golden["leja_points/xi"]


def cases(golden, prefix):
    """Distinct case names under `prefix/` in the golden store."""
    out = []
    for k in golden:
        if k.startswith(prefix + "/"):
            name = k[len(prefix) + 1:].rsplit("/", 1)[0]
            if name not in out:
                out.append(name)
    return out
