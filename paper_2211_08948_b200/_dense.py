"""Small dense host math (torch-free): the matrix exponential and the phi
functions of small matrices, and the divided differences of the Leja
interpolation built on them.

Kept free of torch / CUDA imports so the divided-difference worker
processes (`_ddpool`) import exactly this code: the tables they return are
the bits the in-process computation produces (same function, same
libraries, same inputs).
"""

import math

import numpy as np
import scipy.linalg

try:  # the compiled routine behind scipy.linalg.expm (same bits, batched)
    from scipy.linalg._matfuncs import matrix_exponential as _matrix_exponential
except ImportError:  # pragma: no cover - other scipy layouts
    _matrix_exponential = None

def dense_expm(M):
    """exp(M) of a small dense matrix by scipy's Pade scaling-and-squaring
    (linalg.py:132-139) — the same function the reference calls."""
    M = np.asarray(M, dtype=float)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("dense_expm expects a square matrix")
    if not np.isfinite(M).all():
        raise FloatingPointError("non-finite entries in dense_expm input")
    return scipy.linalg.expm(M)


def _phi_taylor(l, M, terms=20):
    """sum_k M^k / (k+l)!  for tiny ||M|| (linalg.py:142-150)."""
    acc = np.zeros_like(M)
    power = np.eye(M.shape[0])
    for k in range(terms):
        acc += power / math.factorial(k + l)
        power = power @ M
    return acc


def dense_phi(l, M):
    """phi_l(M) via the block upper-bidiagonal embedding (linalg.py:153-175)."""
    M = np.asarray(M, dtype=float)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("dense_phi expects a square matrix")
    if l < 0:
        raise ValueError("phi order must be >= 0")
    if l == 0:
        return dense_expm(M)
    if np.linalg.norm(M) < 1e-8:
        return _phi_taylor(l, M)
    n = M.shape[0]
    big = np.zeros(((l + 1) * n, (l + 1) * n))
    big[:n, :n] = M
    eye = np.eye(n)
    for k in range(l):
        big[k * n:(k + 1) * n, (k + 1) * n:(k + 2) * n] = eye
    return dense_expm(big)[:n, -n:]


def dense_phi_action(l, M, b):
    """phi_l(M) b from one (n+l)-dimensional exponential (linalg.py:178-199)."""
    M = np.asarray(M, dtype=float)
    n = M.shape[0]
    if b.shape != (n,):
        raise ValueError("vector length mismatch in dense_phi_action")
    if l == 0:
        return dense_expm(M) @ b
    if np.linalg.norm(M) < 1e-8:
        return _phi_taylor(l, M) @ b
    aug = np.zeros((n + l, n + l))
    aug[:n, :n] = M
    aug[:n, n] = b
    idx = np.arange(l - 1)
    aug[n + idx, n + idx + 1] = 1.0
    last = np.zeros(n + l)
    last[-1] = 1.0
    return (dense_expm(aug) @ last)[:n]


def phi_divided_differences(l, h, c, gamma, xi, m):
    """Newton divided differences of z -> phi_l(h (c + gamma z)) at xi[:m]:
    the first column of phi_l of the lower bidiagonal matrix
    diag(h (c + gamma xi)) + h gamma * subdiag (leja.py:88-111)."""
    L = np.diag(h * (c + gamma * np.asarray(xi[:m], dtype=np.float64)))
    r = np.arange(m - 1)
    L[r + 1, r] = h * gamma
    e1 = np.zeros(m)
    e1[0] = 1.0
    return dense_phi_action(l, L, e1)


def phi_divided_differences_many(l, hs, c, gamma, xi, m):
    """phi_divided_differences for several scales h sharing l, c, gamma and
    xi (one vertical Leja group): the augmented matrices of
    `dense_phi_action` are stacked and exponentiated in ONE call of the
    routine scipy.linalg.expm runs (it treats a stack slice by slice, so
    every table has the bits of its own call — checked in
    tests/test_host.py). Tables whose matrix takes another branch of
    `dense_phi_action` (tiny norm: Taylor series; non-finite entries: the
    error path) are computed one by one as before."""
    hs = [float(h) for h in hs]
    if _matrix_exponential is None or not hs or l < 0:
        return [phi_divided_differences(l, h, c, gamma, xi, m) for h in hs]
    x = np.asarray(xi[:m], dtype=np.float64)
    r = np.arange(m - 1)
    n = m + l if l > 0 else m
    stack = np.zeros((len(hs), n, n))
    batch, out = [], [None] * len(hs)
    for i, h in enumerate(hs):
        L = np.diag(h * (c + gamma * x))
        L[r + 1, r] = h * gamma
        if not np.isfinite(L).all() or (l > 0 and np.linalg.norm(L) < 1e-8):
            out[i] = phi_divided_differences(l, h, c, gamma, xi, m)
            continue
        a = stack[len(batch)]
        a[:m, :m] = L
        if l > 0:
            a[0, m] = 1.0                     # aug[:n, n] = b = e_1
            idx = np.arange(l - 1)
            a[m + idx, m + idx + 1] = 1.0
        batch.append(i)
    if batch:
        E, info = _matrix_exponential(stack[:len(batch)])
        if info != 0:
            return [phi_divided_differences(l, h, c, gamma, xi, m) for h in hs]
        for j, i in enumerate(batch):
            # dense_phi_action: (expm(aug) @ e_last)[:m]; l = 0: expm(L) @ e_1
            out[i] = E[j][:m, -1].copy() if l > 0 else E[j][:m, 0].copy()
    return out
