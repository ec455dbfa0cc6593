// ek_decide.cuh — the algorithmic decisions taken on the device after a
// reduction: Leja freeze test (leja.py:159-184), power-iteration convergence
// (spectrum.py:56-63). Called by the last block of a reducing kernel with
// the block-partial totals, or — in slab (multi-GPU) mode, where the kernel
// only leaves its local sums in `part[]` — by a one-thread decide kernel
// with the rank-ordered sums of every rank's `part[]`.
#pragma once

#include "ek_common.cuh"

namespace ek {

// m = 0 (leja.py:159-165): freeze test on ||b||, FD increment for m = 1.
__device__ inline void leja_begin_decide(ek_leja_state* st, const double* coef, int nk,
                                         double ssq) {
    const double ny = sqrt(ssq);
    uint32_t act = 0u;
    for (int q = 0; q < nk; ++q) {
        const double d0 = coef[(1 + q) * 32];
        if (!(fabs(d0) * ny < st->tol)) act |= 1u << q;
        st->freeze[q] = 0;
    }
    st->active = act;
    st->ny = ny;
    st->m = 0;
    st->status = EK_ST_OK;
    st->eps = (SQRT_EPS * (1.0 + st->nu)) / ny;
    st->done = act == 0u ? 1 : 0;
    st->iters = 0;
}

// iteration m (leja.py:172-184) given ||y_m||^2 and the non-finite count of
// the Jacobian action (FD only).
__device__ inline void leja_decide(ek_leja_state* st, const double* coef, int mi, int m, int nk,
                                   double ssq, double bad, bool fd) {
    const double ny = sqrt(ssq);  // np.linalg.norm(y)   leja.py:173
    if (fd && st->ny != 0.0) st->fd_evals += 1;
    if (fd && bad > 0.0) {
        st->status = EK_ST_JV_NONFINITE;  // linalg.py:127-128
        st->done = 1;
        st->iters = m;
        return;
    }
    if (!isfinite(ny)) {
        st->status = EK_ST_NORM_NONFINITE;  // leja.py:174-175
        st->done = 1;
        st->iters = m;
        return;
    }
    uint32_t act = st->active;
    for (int q = 0; q < nk; ++q) {
        if ((act >> q) & 1u) {
            const double dq = coef[(1 + q) * 32 + mi];
            if (fabs(dq) * ny < st->tol) {  // leja.py:180
                act &= ~(1u << q);
                st->freeze[q] = m;
            }
        }
    }
    st->active = act;
    st->ny = ny;
    st->m = m;
    st->eps = (SQRT_EPS * (1.0 + st->nu)) / ny;  // linalg.py:123
    if (act == 0u) {
        st->done = 1;
        st->iters = m;
    }
}

// one power iteration (spectrum.py:56-63) given ||J v||^2
__device__ inline void power_decide(ek_power_state* st, double ssq, double bad, bool fd) {
    const double nw = sqrt(ssq);  // spectrum.py:58
    if (fd) st->fd_evals += 1;
    if (fd && bad > 0.0) {
        st->status = EK_ST_JV_NONFINITE;
        st->done = 1;
        return;
    }
    st->it += 1;
    if (nw == 0.0) {  // spectrum.py:59-60
        st->lam = 0.0;
        st->converged = 1;
        st->done = 1;
    } else if (fabs(nw - st->lam) <= st->tol_pi * nw) {  // spectrum.py:63
        st->lam = nw;
        st->converged = 1;
        st->done = 1;
    } else {
        st->lam = nw;
        if (st->it >= st->max_it) st->done = 1;
    }
    st->nw = nw;
}

// Slab mode: global sums of the gathered part[] blocks (EK_PART_SLOTS
// slots per rank, see EK_PART_*): the sum channel as the exact merge of the
// ranks' integer accumulators (repro mode: any P gives the same bits), else
// as the rank-ordered fp64 sum; the count channel in rank order.
__device__ inline void gathered_sums(const double* g, int nranks, double& s0, double& s1) {
    s0 = 0.0;
    s1 = 0.0;
    const bool xs = g[EK_PART_TAG] != 0.0;
    XAcc tot;
    xzero(tot);
    for (int r = 0; r < nranks; ++r) {
        const double* p = g + (long)r * EK_PART_SLOTS;
        if (xs) xmerge(tot, xload(reinterpret_cast<const long long*>(p)));
        else s0 = r == 0 ? p[0] : s0 + p[0];
        s1 += p[EK_PART_COUNT];
    }
    if (xs) s0 = xvalue(tot);
}

}  // namespace ek
