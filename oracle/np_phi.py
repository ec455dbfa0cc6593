"""NumPy/SciPy restatement of the phi-action engines.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Restates, with the reference's operation order:
  * dense phi / expm helpers        linalg.py:132-199
  * Leja point sequence              leja.py:32-50
  * divided differences              leja.py:88-111
  * vertical Leja interpolation      leja.py:121-189
  * KIOPS                            kiops.py:106-303
  * power iteration + estimate       spectrum.py:43-96

Operators are plain Python objects with `.apply(v)`, `.dim` and a shared
`Tally` (the reference's EvalCounter, linalg.py:21-32), so RHS-evaluation
accounting can be compared against the device implementation.
"""

import math
from dataclasses import dataclass, replace

import numpy as np
import scipy.linalg


class NonConvergence(RuntimeError):
    """errors.py:4-14."""

    def __init__(self, message, iters=0, detail=None):
        super().__init__(message)
        self.iters = iters
        self.detail = detail


class StepFailure(RuntimeError):
    """errors.py:17-22."""

    def __init__(self, message, cause=None):
        super().__init__(message)
        self.cause = cause


# ------------------------------------------------------------ accounting


class Tally:
    """linalg.py:21-32."""

    def __init__(self):
        self.count = 0

    def charge(self, k=1):
        if k < 0:
            raise ValueError("counter cannot decrease")
        self.count += k


class CountedRhs:
    """linalg.py:35-48."""

    def __init__(self, fn, tally=None):
        self.fn = fn
        self.counter = tally if tally is not None else Tally()

    def __call__(self, u):
        self.counter.charge()
        return self.fn(u)


class Operator:
    """linalg.py:51-90: v -> A v with a charge per application."""

    def __init__(self, fn, dim, counter=None, charge=1):
        self.fn = fn
        self.dim = int(dim)
        if self.dim < 1:
            raise ValueError("operator dimension must be positive")
        self.counter = counter if counter is not None else Tally()
        self.charge = charge

    def apply(self, v):
        if v.shape != (self.dim,):
            raise ValueError("shape mismatch")
        if self.charge:
            self.counter.charge(self.charge)
        return self.fn(v)

    def scaled(self, s):
        return Operator(lambda v: s * self.apply(v), self.dim,
                        counter=self.counter, charge=0)

    @classmethod
    def dense(cls, A, counter=None):
        A = np.asarray(A, dtype=float)
        return cls(lambda v: A @ v, A.shape[0], counter=counter)


# ------------------------------------------------------------ dense phi


def expm_checked(M):
    """linalg.py:132-139."""
    M = np.asarray(M, dtype=float)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("square matrix expected")
    if not np.all(np.isfinite(M)):
        raise FloatingPointError("non-finite entries in dense_expm input")
    return scipy.linalg.expm(M)


def phi_series(l, M, terms=20):
    """linalg.py:142-150."""
    acc = np.zeros_like(M)
    t = np.eye(M.shape[0])
    for k in range(terms):
        acc += t / math.factorial(k + l)
        t = t @ M
    return acc


def phi_matrix(l, M):
    """linalg.py:153-175."""
    M = np.asarray(M, dtype=float)
    if M.ndim != 2 or M.shape[0] != M.shape[1]:
        raise ValueError("square matrix expected")
    if l < 0:
        raise ValueError("phi order must be >= 0")
    if l == 0:
        return expm_checked(M)
    if np.linalg.norm(M) < 1e-8:
        return phi_series(l, M)
    n = M.shape[0]
    W = np.zeros(((l + 1) * n, (l + 1) * n))
    W[:n, :n] = M
    for k in range(l):
        W[k * n:(k + 1) * n, (k + 1) * n:(k + 2) * n] = np.eye(n)
    return expm_checked(W)[:n, -n:]


def phi_apply(l, M, b):
    """linalg.py:178-199: phi_l(M) b from one (n+l)-dim exponential."""
    M = np.asarray(M, dtype=float)
    n = M.shape[0]
    if b.shape != (n,):
        raise ValueError("vector length mismatch")
    if l == 0:
        return expm_checked(M) @ b
    if np.linalg.norm(M) < 1e-8:
        return phi_series(l, M) @ b
    big = np.zeros((n + l, n + l))
    big[:n, :n] = M
    big[:n, n] = b
    for k in range(l - 1):
        big[n + k, n + k + 1] = 1.0
    e = np.zeros(n + l)
    e[-1] = 1.0
    return (expm_checked(big) @ e)[:n]


# ----------------------------------------------------------------- Leja

CHUNK = 32          # leja.py:27
NUM_POINTS = 400    # leja.py:25


def leja_points(m=NUM_POINTS, n_candidates=100_000):
    """leja.py:32-50: greedy log-product maximiser on a uniform grid,
    xi_0 = 2, argmax ties toward the smaller candidate."""
    grid = np.linspace(-2.0, 2.0, n_candidates)
    pts = np.empty(m)
    pts[0] = 2.0
    with np.errstate(divide="ignore"):
        score = np.log(np.abs(grid - pts[0]))
        for k in range(1, m):
            pts[k] = grid[int(np.argmax(score))]
            score += np.log(np.abs(grid - pts[k]))
    return pts


@dataclass(frozen=True)
class Estimate:
    """spectrum.py:19-31."""
    alpha: float
    beta: float
    c: float
    gamma: float
    safety: float
    age_steps: int = 0

    def aged(self):
        return replace(self, age_steps=self.age_steps + 1)


def newton_coeffs(l, h, est, xi, m_max):
    """leja.py:88-111: first column of phi_l(h*(c I + gamma * bidiag(xi)))."""
    if not 0 <= l <= 4:
        raise ValueError("phi order must be in 0..4")
    if h < 0:
        raise ValueError("scale h must be >= 0")
    m_max = min(m_max, len(xi))
    L = np.diag(h * (est.c + est.gamma * xi[:m_max]))
    sub = h * est.gamma
    for j in range(m_max - 1):
        L[j + 1, j] = sub
    e1 = np.zeros(m_max)
    e1[0] = 1.0
    d = phi_apply(l, L, e1)
    if not np.all(np.isfinite(d)):
        raise NonConvergence("non-finite divided differences")
    return d


@dataclass
class LejaOut:
    vectors: list
    iters: int
    freeze_iters: list


def leja_vertical(J, b, l, coeffs, h, est, tol, xi, max_points=NUM_POINTS):
    """leja.py:133-189: shared Newton basis, one accumulator per scale."""
    if tol <= 0:
        raise ValueError("tolerance must be positive")
    if len(coeffs) < 1:
        raise ValueError("need at least one coefficient")
    if any(not 0.0 < ci <= 1.0 for ci in coeffs):
        raise ValueError("coefficients must lie in (0, 1]")
    k = len(coeffs)
    c, gamma = est.c, est.gamma
    avail = min(CHUNK, max_points)
    d = [newton_coeffs(l, ci * h, est, xi, avail) for ci in coeffs]
    y = b.astype(float, copy=True)
    ny = float(np.linalg.norm(y))
    acc = [d[i][0] * y for i in range(k)]
    done = [abs(d[i][0]) * ny < tol for i in range(k)]
    at = [0] * k
    if all(done):
        return LejaOut(acc, 0, at)
    for m in range(1, max_points):
        if m >= avail:
            avail = min(avail + CHUNK, max_points)
            d = [newton_coeffs(l, ci * h, est, xi, avail) for ci in coeffs]
        y = J.apply(y) / gamma - (c / gamma + xi[m - 1]) * y
        ny = float(np.linalg.norm(y))
        if not np.isfinite(ny):
            raise NonConvergence("polynomial iteration diverged", iters=m)
        for i in range(k):
            if done[i]:
                continue
            acc[i] = acc[i] + d[i][m] * y
            if abs(d[i][m]) * ny < tol:
                done[i] = True
                at[i] = m
        if all(done):
            return LejaOut(acc, m, at)
    raise NonConvergence(
        f"no convergence in {max_points} Leja points", iters=max_points,
        detail={"stalled_coefficients":
                [coeffs[i] for i in range(k) if not done[i]]})


def leja_single(J, b, l, h, est, tol, xi, max_points=NUM_POINTS):
    """leja.py:121-130."""
    r = leja_vertical(J, b, l, [1.0], h, est, tol, xi, max_points)
    return r.vectors[0], r.iters


# ---------------------------------------------------------------- KIOPS


@dataclass
class KStats:
    """kiops.py:96-103."""
    substeps: int = 0
    rejections: int = 0
    matvecs: int = 0
    expms: int = 0
    m_last: int = 0
    err_sum: float = 0.0


def kiops(op, vectors, tau_out=(1.0,), tol=1e-7, m_init=10, m_min=10,
          m_max=128, iop_len=2, tau_min_frac=1e-8):
    """kiops.py:106-289: adaptive-substep incomplete-orthogonalisation
    Krylov evaluation of sum_j tau^j phi_j(tau A) v_j."""
    U = np.array([np.asarray(v, dtype=float) for v in vectors])
    nvec, n = U.shape
    p = nvec - 1
    if p == 0:
        p = 1
        U = np.vstack([U, np.zeros((1, n))])
    tau_out = np.asarray(tau_out, dtype=float)
    if np.any(tau_out <= 0) or np.any(np.diff(tau_out) < 0):
        raise ValueError("tau_out must be positive and ascending")
    n_out = len(tau_out)
    m = max(m_min, min(m_init, m_max))
    V = np.zeros((m_max + 1, n + p))
    H = np.zeros((m_max + 1, m_max + 1))
    st = KStats()
    t_now, t_end = 0.0, float(tau_out[-1])
    happy = False
    j = 0
    W = np.zeros((n_out, n))
    W[0] = U[0]
    nxt = 0
    scale = np.max(np.sum(np.abs(U[1:]), axis=1)) if nvec > 1 else 0.0
    if scale > 0:
        e = math.ceil(math.log2(scale))
        nu, mu = 2.0 ** (-e), 2.0 ** e
    else:
        nu, mu = 1.0, 1.0
    flip = nu * np.flipud(U[1:])
    tau = t_end
    g, g_mmax = (0.2, 0.1) if t_end > 1 else (0.9, 0.6)
    delta = 1.4
    old_m, old_tau, omega = -1, math.nan, math.nan
    order_old, kest_old = True, True
    order, kest = 1.0, 2.0
    beta = 0.0
    nrej = 0
    while t_now < t_end * (1.0 - 1e-12):
        if j == 0:
            H[:, :] = 0.0
            V[0, :n] = W[nxt]
            for k in range(p - 1):
                i = p - 1 - k
                V[0, n + k] = (t_now ** i) / math.factorial(i) * mu
            V[0, n + p - 1] = mu
            beta = float(np.linalg.norm(V[0]))
            V[0] /= beta
        while j < m:
            j += 1
            V[j, :n] = op.apply(V[j - 1, :n]) + V[j - 1, n:] @ flip
            V[j, n:n + p - 1] = V[j - 1, n + 1:n + p]
            V[j, -1] = 0.0
            st.matvecs += 1
            lo = max(0, j - iop_len)
            H[lo:j, j - 1] = V[lo:j] @ V[j]
            V[j] -= V[lo:j].T @ H[lo:j, j - 1]
            nrm = float(np.linalg.norm(V[j]))
            if nrm < tol:
                happy = True
                break
            H[j, j - 1] = nrm
            V[j] /= nrm
        H[0, j] = 1.0
        nrm = H[j, j - 1]
        H[j, j - 1] = 0.0
        F = scipy.linalg.expm(tau * H[:j + 1, :j + 1])
        st.expms += 1
        H[j, j - 1] = nrm
        if happy:
            omega = 0.0
            err = 0.0
            tau_new = min(t_end - (t_now + tau), tau)
            m_new = m
            happy = False
        else:
            err = abs(beta * nrm * F[j - 1, j])
            prev_omega = omega
            omega = t_end * err / (tau * tol)
            if m == old_m and tau != old_tau and nrej >= 1:
                order = max(1.0, math.log(omega / prev_omega)
                            / math.log(tau / old_tau))
                order_old = False
            elif order_old or nrej == 0:
                order_old = True
                order = j / 4.0
            else:
                order_old = True
            if m != old_m and tau == old_tau and nrej >= 1:
                kest = max(1.1, (omega / prev_omega) ** (1.0 / (old_m - m)))
                kest_old = False
            elif kest_old or nrej == 0:
                kest_old = True
                kest = 2.0
            else:
                kest_old = True
            remaining = (t_end - t_now if omega > delta
                         else t_end - (t_now + tau))
            same_tau = min(remaining, tau)
            tau_opt = tau * (g / omega) ** (1.0 / order)
            tau_opt = min(remaining, max(tau / 5.0, min(5.0 * tau, tau_opt)))
            m_opt = math.ceil(j + math.log(omega / g) / math.log(kest))
            m_opt = max(m_min, min(m_max, max(math.floor(3 * m / 4),
                                              min(m_opt, math.ceil(4 * m / 3)))))
            if j == m_max:
                if omega > delta:
                    m_new = j
                    tau_new = tau * (g_mmax / omega) ** (1.0 / order)
                    tau_new = min(t_end - t_now, max(tau / 5.0, tau_new))
                else:
                    tau_new = tau_opt
                    m_new = m
            else:
                m_new = m_opt
                tau_new = same_tau
        if omega <= delta:
            st.substeps += 1
            t_next = t_now + tau
            blown = 0
            for k in range(nxt, n_out):
                if tau_out[k] < t_next - 1e-14 * t_end:
                    blown += 1
            if blown:
                W[nxt + blown] = W[nxt]
                for k in range(blown):
                    F2 = scipy.linalg.expm((tau_out[nxt + k] - t_now) * H[:j, :j])
                    W[nxt + k] = beta * F2[:j, 0] @ V[:j, :n]
                    st.expms += 1
                nxt += blown
            W[nxt] = beta * F[:j, 0] @ V[:j, :n]
            t_now += tau
            j = 0
            nrej = 0
            st.err_sum += err
        else:
            st.rejections += 1
            nrej += 1
            H[0, j] = 0.0
        old_tau, tau = tau, tau_new
        old_m, m = m, m_new
        if tau < tau_min_frac * t_end and t_now < t_end:
            raise NonConvergence(
                f"KIOPS substep shrank below {tau_min_frac} of the interval",
                iters=st.matvecs)
    st.m_last = old_m
    return [W[k].copy() for k in range(n_out)], st


def kiops_eval(A, vectors, dt, tol, **kw):
    """kiops.py:292-303."""
    if len(vectors) - 1 > 4:
        raise ValueError("phi orders above 4 are not supported")
    if dt == 0.0:
        return np.asarray(vectors[0], dtype=float).copy(), KStats()
    ws, st = kiops(A.scaled(dt), vectors, tau_out=(1.0,), tol=tol, **kw)
    return ws[0], st


# ------------------------------------------------------------- spectrum

GAMMA_MIN = 1e-13  # spectrum.py:16


@dataclass(frozen=True)
class Policy:
    """spectrum.py:34-40."""
    n_recompute: int = 50
    safety: float = 1.1
    tol_pi: float = 1e-2
    max_it: int = 1000
    seed: int = 0


def power_iterate(J, tol_pi=1e-2, max_it=1000, seed=0):
    """spectrum.py:43-63."""
    v = np.random.default_rng(seed).standard_normal(J.dim)
    v /= np.linalg.norm(v)
    lam = 0.0
    for _ in range(max_it):
        w = J.apply(v)
        nw = np.linalg.norm(w)
        if nw == 0.0:
            return 0.0, True
        v = w / nw
        if abs(nw - lam) <= tol_pi * nw:
            return float(nw), True
        lam = nw
    return float(lam), False


def estimate(lam, safety=1.1):
    """spectrum.py:66-78."""
    if not np.isfinite(lam):
        raise ValueError("non-finite eigenvalue estimate")
    alpha = -safety * abs(lam)
    beta = 0.0
    return Estimate(alpha=alpha, beta=beta, c=(alpha + beta) / 2.0,
                    gamma=max(abs(beta - alpha) / 4.0, GAMMA_MIN),
                    safety=safety, age_steps=0)


def refresh(est, J, policy, force=False):
    """spectrum.py:81-96."""
    if force or est is None or est.age_steps >= policy.n_recompute:
        lam, ok = power_iterate(J, tol_pi=policy.tol_pi, max_it=policy.max_it,
                                seed=policy.seed)
        base = est.safety if est is not None else policy.safety
        return estimate(lam, safety=base if ok else base * 1.5)
    return est.aged()
