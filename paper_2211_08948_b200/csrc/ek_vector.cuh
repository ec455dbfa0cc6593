// ek_vector.cuh — non-stencil fp64 vector kernels (grid-stride, fixed grid
// per length so reductions are deterministic).
#pragma once

#include "ek_common.cuh"
#include "ek_decide.cuh"

namespace ek {

constexpr int VGRID_MAX = 148 * 16;  // 16 resident 256-thread blocks per SM

__host__ __forceinline__ int vgrid(int64_t len) {
    int64_t b = (len + TPB - 1) / TPB;
    if (b < 1) b = 1;
    return (int)(b < VGRID_MAX ? b : VGRID_MAX);
}
// Streaming kernels take 4 consecutive elements per thread and iteration
// (two 16-byte loads per operand, all issued before use): 4x the bytes in
// flight of one element per thread, which a grid-stride loop needs to get
// near the HBM bandwidth (one 8-byte load per thread is latency bound).
__host__ __forceinline__ int vgrid4(int64_t len) { return vgrid((len + 3) / 4); }

__device__ __forceinline__ bool al16d(const void* p) { return ((uintptr_t)p & 15) == 0; }
// x[e0 .. e0+3] (zeros past len); `full`: whole group and x 16-byte aligned
__device__ __forceinline__ void ld4(const double* __restrict__ x, int64_t e0, int64_t len,
                                    bool full, double (&v)[4]) {
    if (full) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(x + e0));
        const double2 b = __ldg(reinterpret_cast<const double2*>(x + e0) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    } else {
#pragma unroll
        for (int w = 0; w < 4; ++w) v[w] = e0 + w < len ? __ldg(x + e0 + w) : 0.0;
    }
}
// plain (coherent) loads: for buffers this kernel also writes
__device__ __forceinline__ void ld4c(const double* x, int64_t e0, int64_t len, bool full,
                                     double (&v)[4]) {
    if (full) {
        const double2 a = reinterpret_cast<const double2*>(x + e0)[0];
        const double2 b = reinterpret_cast<const double2*>(x + e0)[1];
        v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    } else {
#pragma unroll
        for (int w = 0; w < 4; ++w) v[w] = e0 + w < len ? x[e0 + w] : 0.0;
    }
}
__device__ __forceinline__ void st4(double* x, int64_t e0, int64_t len, bool full,
                                    const double (&v)[4]) {
    if (full) {
        reinterpret_cast<double2*>(x + e0)[0] = make_double2(v[0], v[1]);
        reinterpret_cast<double2*>(x + e0)[1] = make_double2(v[2], v[3]);
    } else {
#pragma unroll
        for (int w = 0; w < 4; ++w)
            if (e0 + w < len) x[e0 + w] = v[w];
    }
}
#define EK_FOR4(e0, len)                                                                  \
    for (int64_t e0 = ((int64_t)blockIdx.x * TPB + threadIdx.x) * 4; e0 < (len);         \
         e0 += (int64_t)gridDim.x * TPB * 4)

// ---------------------------------------------------------------- norms
// ||x||^2 (+ flags: bit0 any nonzero, bit1 any non-finite) -> st->val[slot]
// = ssq, st->val[slot+1] = sqrt(ssq). `div` (nullable) scales on read.
__global__ void __launch_bounds__(TPB) k_norm2(int64_t len, const double* __restrict__ x,
                                               const double* div, ek_scalar_state* st,
                                               int slot, double* work, int repro) {
    double acc[3] = {0.0, 0.0, 0.0};
    XAcc xs[1];
    xzero(xs[0]);
    const double d = div ? *div : 1.0;
    const bool has_div = div != nullptr, vec = al16d(x);
    EK_FOR4(e0, len) {
        double v[4];
        ld4(x, e0, len, vec && e0 + 4 <= len, v);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            if (e0 + w >= len) break;
            if (has_div) v[w] = v[w] / d;
            if (repro) xadd<false>(xs[0], v[w] * v[w]);
            else acc[0] += v[w] * v[w];
            acc[1] += (v[w] != 0.0) ? 1.0 : 0.0;
            acc[2] += isfinite(v[w]) ? 0.0 : 1.0;
        }
    }
    double tot[3];
    XAcc xt[1];
    if (reduce_grid<3, 1>(acc, xs, repro != 0, work, &st->ticket, false, tot, xt)) {
        if (threadIdx.x == 0) {
            if (slot == 0) {
                if (repro) xstore((long long*)st->xs, xt[0]);
                st->repro = repro;
            }
            st->val[slot] = tot[0];
            st->val[slot + 1] = sqrt(tot[0]);
            st->flag |= (tot[1] > 0.0 ? 1 : 0) | (tot[2] > 0.0 ? 2 : 0);
        }
    }
}

// sum |x_e| -> st->val[slot]  (kiops.py:146 L1 norms of the augmentation)
__global__ void __launch_bounds__(TPB) k_l1(int64_t len, const double* __restrict__ x,
                                            ek_scalar_state* st, int slot, double* work) {
    double acc[1] = {0.0};
    const bool vec = al16d(x);
    EK_FOR4(e0, len) {
        double v[4];
        ld4(x, e0, len, vec && e0 + 4 <= len, v);
#pragma unroll
        for (int w = 0; w < 4; ++w) acc[0] += fabs(v[w]);  // zeros past len
    }
    block_sum<1>(acc);
    if (publish_and_arrive<1>(acc, work, &st->ticket)) {
        double tot[1];
        gather_partials<1>(work, gridDim.x, tot);
        if (threadIdx.x == 0) st->val[slot] = tot[0];
    }
}

// ------------------------------------------------------------------ Leja
struct LejaVArgs {
    int64_t len;
    const double* b;      // begin: start vector; update: Jacobian action
    const double* y;      // update: previous iterate
    double* ynext;
    double* p[8];
    int nk;
    const double* coef;
    int mi;
    int m;
    double gamma;
    ek_leja_state* st;
    double* work;
    int repro;            // order-independent ||.||^2 (ek_xsum.cuh)
};

// Slab mode: a vector pass leaves its local sum in part[] (EK_PART_*).
__device__ __forceinline__ void part_store_v(double* part, int repro, double ssq, const XAcc& xt) {
    if (repro) xstore(reinterpret_cast<long long*>(part), xt);
    else part[0] = ssq;
    part[EK_PART_COUNT] = 0.0;
    part[EK_PART_TAG] = repro ? 1.0 : 0.0;
}

// Initialise a Leja state block on the device (ek_leja_call): the host
// values travel as kernel arguments, ||u|| optionally from a device slot.
__global__ void k_leja_init(ek_leja_state* st, double tol, double nu, const double* nu_dev,
                            int k, int p_init, int lazy0) {
    if (threadIdx.x == 0) {
        ek_leja_state z{};
        z.tol = tol;
        z.nu = nu_dev ? *nu_dev : nu;
        z.k = k;
        z.p_init = p_init;
        z.lazy0 = lazy0;
        *st = z;
    }
}

// m = 0 of the Newton-Leja sum (leja.py:159-165).
__global__ void __launch_bounds__(TPB) k_leja_begin(const LejaVArgs a) {
    // fold request (host set p_init = -1): leave p to the first iteration.
    // Every block reads the flag before the last one rewrites it.
    const bool fold = a.st->p_init < 0;
    double acc[1] = {0.0};
    XAcc xs[1];
    xzero(xs[0]);
    double d[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) d[q] = q < a.nk ? a.coef[(1 + q) * 32 + a.mi] : 0.0;
    bool vec = al16d(a.b);
#pragma unroll
    for (int q = 0; q < 8; ++q)
        if (q < a.nk) vec = vec && al16d(a.p[q]);
    if (fold) {
        // read-only pass (||b||^2): 4 groups of 4 elements per thread and
        // iteration, all 8 loads issued before use (128 B in flight per
        // thread instead of 32 B: a lone streaming read needs the depth)
        const int64_t stride = (int64_t)gridDim.x * TPB * 4;
        for (int64_t e0 = ((int64_t)blockIdx.x * TPB + threadIdx.x) * 4; e0 < a.len;
             e0 += 4 * stride) {
            double y[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int64_t e = e0 + u * stride;
                ld4(a.b, e, a.len, vec && e + 4 <= a.len, y[u]);  // zeros past len
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int w = 0; w < 4; ++w) {
                    if (a.repro) xadd<false>(xs[0], y[u][w] * y[u][w]);
                    else acc[0] += y[u][w] * y[u][w];
                }
        }
    } else EK_FOR4(e0, a.len) {
        const bool full = vec && e0 + 4 <= a.len;
        double y[4];
        ld4(a.b, e0, a.len, full, y);
#pragma unroll
        for (int w = 0; w < 4; ++w) {  // zeros past len
            if (a.repro) xadd<false>(xs[0], y[w] * y[w]);
            else acc[0] += y[w] * y[w];
        }
        {
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < a.nk) {
                    double pv[4];
#pragma unroll
                    for (int w = 0; w < 4; ++w) pv[w] = d[q] * y[w];  // dds[i][0] * y
                    st4(a.p[q], e0, a.len, full, pv);
                }
        }
    }
    double tot[1];
    XAcc xt[1];
    if (reduce_grid<1, 1>(acc, xs, a.repro != 0, a.work, &a.st->ticket, false, tot, xt)) {
        if (threadIdx.x == 0) {
            a.st->p_init = fold ? 0 : 1;
            if (a.st->defer) {
                part_store_v(a.st->part, a.repro, tot[0], xt[0]);
            } else {
                leja_begin_decide(a.st, a.coef, a.nk, tot[0]);
            }
        }
    }
}

// Folded begin: if every accumulator froze at m = 0 no iteration will write
// the accumulators, so write p_i = d_i[0] b here (a no-op otherwise).
__global__ void __launch_bounds__(TPB) k_leja_fold_done(const LejaVArgs a) {
    if (!a.st->done || a.st->p_init != 0 || a.st->lazy0) return;
    double d[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) d[q] = q < a.nk ? a.coef[(1 + q) * 32] : 0.0;
    bool vec = al16d(a.b);
#pragma unroll
    for (int q = 0; q < 8; ++q)
        if (q < a.nk) vec = vec && al16d(a.p[q]);
    EK_FOR4(e0, a.len) {
        const bool full = vec && e0 + 4 <= a.len;
        double y[4];
        ld4(a.b, e0, a.len, full, y);
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (q < a.nk) {
                double pv[4];
#pragma unroll
                for (int w = 0; w < 4; ++w) pv[w] = d[q] * y[w];  // dds[i][0] * y
                st4(a.p[q], e0, a.len, full, pv);
            }
    }
}

// Deferred accumulation (ek_leja_run_seq + ek_leja_combine): the iterations
// of a chunk keep every iterate y_m in its own buffer and leave the
// accumulators alone; this pass then forms, per element and in registers,
//     p_i = ((d_i[0] y_0 + d_i[1] y_1) + d_i[2] y_2) + ...   (leja.py:161, 179)
// term by term in the reference's order with the same two roundings per term
// (product, sum; the library is built without FMA contraction), up to the
// iteration at which accumulator i froze (state block: freeze[i], or m while
// it is still active). A call of M iterations and k accumulators then moves
// M + 1 + k vectors once instead of 2 k per iteration.
struct LejaCombineArgs {
    int64_t len;
    const double* y[33];  // y[j]: the iterate of table column j (first chunk: y[0] = b)
    int ny;
    double* p[8];
    int nk;
    const double* coef;   // this chunk's table: row 1 + i = d_i, 32 columns
    int chunk_base;       // iteration of column 0
    int cont;             // 1: p already holds the sum over the earlier chunks
    const ek_leja_state* st;
};

template <int NK>
__global__ void __launch_bounds__(TPB) k_leja_combine(const LejaCombineArgs a) {
    __shared__ double d[NK][32];
    __shared__ int last[NK];  // last column of accumulator i in this chunk (-1: none)
    // m = 0 result of a folded begin is written by k_leja_fold_done (or stays lazy)
    if (!a.cont && a.st->done && a.st->iters == 0 && a.st->status == EK_ST_OK) return;
    for (int t = threadIdx.x; t < NK * 32; t += TPB) {
        const int q = t >> 5, j = t & 31;
        d[q][j] = q < a.nk ? a.coef[(1 + q) * 32 + j] : 0.0;
    }
    if (threadIdx.x < NK) {
        const int q = threadIdx.x;
        int l = -1;
        if (q < a.nk) {
            const int ml = ((a.st->active >> q) & 1u) ? a.st->m : a.st->freeze[q];
            l = ml - a.chunk_base;
            if (l > a.ny - 1) l = a.ny - 1;
            if (l < 0) l = -1;
        }
        last[q] = l;
    }
    __syncthreads();
    int lq[NK], maxl = -1;
#pragma unroll
    for (int q = 0; q < NK; ++q) {
        lq[q] = last[q];
        maxl = lq[q] > maxl ? lq[q] : maxl;
    }
    if (maxl < 0) return;
    bool vec = true;
    for (int j = 0; j <= maxl; ++j) vec = vec && al16d(a.y[j]);
#pragma unroll
    for (int q = 0; q < NK; ++q)
        if (q < a.nk) vec = vec && al16d(a.p[q]);
    const bool cont = a.cont != 0;
    EK_FOR4(e0, a.len) {
        const bool full = vec && e0 + 4 <= a.len;
        double acc[NK][4];
#pragma unroll
        for (int q = 0; q < NK; ++q) {
            if (cont && lq[q] >= 0) ld4(a.p[q], e0, a.len, full, acc[q]);
            else {
#pragma unroll
                for (int w = 0; w < 4; ++w) acc[q][w] = 0.0;
            }
        }
        // four iterates per turn: their loads are all issued before the
        // first one is used (128 B in flight per thread)
        for (int j0 = 0; j0 <= maxl; j0 += 4) {
            double yv[4][4];
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (j0 + u <= maxl) ld4(a.y[j0 + u], e0, a.len, full, yv[u]);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int j = j0 + u;
                if (j <= maxl) {
                    const bool first = j == 0 && !cont;
#pragma unroll
                    for (int q = 0; q < NK; ++q)
                        if (j <= lq[q]) {
                            const double dq = d[q][j];
#pragma unroll
                            for (int w = 0; w < 4; ++w) {
                                const double t = dq * yv[u][w];
                                acc[q][w] = first ? t : acc[q][w] + t;
                            }
                        }
                }
            }
        }
#pragma unroll
        for (int q = 0; q < NK; ++q)
            if (lq[q] >= 0) st4(a.p[q], e0, a.len, full, acc[q]);
    }
}

// out = (a*x) + (b*y)
__global__ void __launch_bounds__(TPB) k_axpby(int64_t n, double a, const double* __restrict__ x,
                                               double b, const double* __restrict__ y,
                                               double* __restrict__ out) {
    const bool vec = al16d(x) && al16d(y) && al16d(out);
    EK_FOR4(e0, n) {
        const bool full = vec && e0 + 4 <= n;
        double xv[4], yv[4], o[4];
        ld4(x, e0, n, full, xv);
        ld4(y, e0, n, full, yv);
#pragma unroll
        for (int w = 0; w < 4; ++w) o[w] = (a * xv[w]) + (b * yv[w]);
        st4(out, e0, n, full, o);
    }
}

struct DotArgs {
    int64_t n;
    const double* x;
    const double* y[8];
    int k;
    ek_scalar_state* st;
    double* work;
};

// st->val[q] = x . y_q, q < k, one pass over x
__global__ void __launch_bounds__(TPB) k_dot_multi(const DotArgs a) {
    double acc[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) acc[q] = 0.0;
    bool vec = al16d(a.x);
#pragma unroll
    for (int q = 0; q < 8; ++q)
        if (q < a.k) vec = vec && al16d(a.y[q]);
    EK_FOR4(e0, a.n) {
        const bool full = vec && e0 + 4 <= a.n;
        double xv[4];
        ld4(a.x, e0, a.n, full, xv);
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (q < a.k) {
                double yv[4];
                ld4(a.y[q], e0, a.n, full, yv);
#pragma unroll
                for (int w = 0; w < 4; ++w) acc[q] += xv[w] * yv[w];  // zeros past n
            }
    }
    block_sum<8>(acc);
    if (publish_and_arrive<8>(acc, a.work, &a.st->ticket)) {
        double tot[8];
        gather_partials<8>(a.work, gridDim.x, tot);
        if (threadIdx.x == 0) {
#pragma unroll
            for (int q = 0; q < 8; ++q) a.st->val[q] = q < a.k ? tot[q] : 0.0;
        }
    }
}

// Slab mode: apply a deferred Leja decision to the gathered per-rank sums
// (`g` = [nranks][EK_PART_SLOTS] part[] blocks, see gathered_sums).
__global__ void k_leja_decide(ek_leja_state* st, const double* g, int nranks, const double* coef,
                              int mi, int m, int nk, int fd, int begin) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (!begin && st->done) return;
    double s0, s1;
    gathered_sums(g, nranks, s0, s1);
    if (begin) leja_begin_decide(st, coef, nk, s0);
    else leja_decide(st, coef, mi, m, nk, s0, s1, fd != 0);
}

// Peer mode: wait until every rank raised its flag for pass `epoch`
// (ld.acquire.sys on the own window), then the rank-ordered sums of the
// partials the ranks wrote into red[epoch & 1] and the freeze test. A flag
// that never comes (a dead peer) ends in EK_ST_PEER_TIMEOUT, not a hang.
__global__ void k_peer_decide(ek_leja_state* st, const ek_peer* P, long epoch, const double* coef,
                              int mi, int m, int nk, int fd) {
    if (st->done) return;
    const int lane = threadIdx.x;
    const double* win = P->win[P->rank];
    bool ok = true;
    if (lane < P->world) {
        const unsigned long long* f = (const unsigned long long*)win + lane;
        const unsigned long long want = (unsigned long long)epoch + 1;
        unsigned long long got = 0, t0, t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
        for (;;) {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(got) : "l"(f) : "memory");
            if (got >= want) break;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            if (t - t0 > 60ull * 1000000000ull) {  // 60 s: give up instead of hanging
                ok = false;
                break;
            }
            __nanosleep(32);
        }
    }
    ok = __all_sync(0xffffffffu, ok);
    if (lane != 0) return;
    if (!ok) {
        st->status = EK_ST_PEER_TIMEOUT;
        st->done = 1;
        st->iters = m;
        return;
    }
    double s0, s1;
    gathered_sums((const double*)((const char*)win + 64) + (epoch & 1) * 8 * EK_PART_SLOTS,
                  P->world, s0, s1);
    leja_decide(st, coef, mi, m, nk, s0, s1, fd != 0);
}

// Slab mode: deferred power-iteration decision; which = 0 iteration,
// 1 = ||v0|| (first divisor), 2 = ||v|| (FD increment).
__global__ void k_power_decide(ek_power_state* st, const double* g, int nranks, int fd,
                               int which) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    if (which == 0 && (st->done || st->status)) return;
    if (which == 2 && (st->done || st->status)) return;
    double s0, s1;
    gathered_sums(g, nranks, s0, s1);
    if (which == 0) power_decide(st, s0, s1, fd != 0);
    else if (which == 1) st->nw = sqrt(s0);
    else st->nv = sqrt(s0);
}

// One recurrence step for a Jacobian action computed elsewhere
// (dense / callable / 1-D operators).
__global__ void __launch_bounds__(TPB) k_leja_update(const LejaVArgs a) {
    const ek_leja_state* cst = a.st;
    if (cst->done) return;
    const double shift = a.coef[a.mi];
    const Dv gam = mkdv(a.gamma);
    const uint32_t act = cst->active;
    double d[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) d[q] = q < a.nk ? a.coef[(1 + q) * 32 + a.mi] : 0.0;
    double acc[1] = {0.0};
    XAcc xs[1];
    xzero(xs[0]);
    for (int64_t e = (int64_t)blockIdx.x * TPB + threadIdx.x; e < a.len;
         e += (int64_t)gridDim.x * TPB) {
        const double yn = dv(__ldg(a.b + e), gam) - (shift * __ldg(a.y + e));
        a.ynext[e] = yn;
        if (a.repro) xadd<false>(xs[0], yn * yn);
        else acc[0] += yn * yn;
#pragma unroll
        for (int q = 0; q < 8; ++q)
            if (q < a.nk && ((act >> q) & 1u)) a.p[q][e] = a.p[q][e] + (d[q] * yn);
    }
    double tot[1];
    XAcc xt[1];
    if (reduce_grid<1, 1>(acc, xs, a.repro != 0, a.work, &a.st->ticket, false, tot, xt)) {
        if (threadIdx.x == 0) {
            if (a.st->defer) {
                part_store_v(a.st->part, a.repro, tot[0], xt[0]);
            } else {
                // the Jacobian action was checked by its own operator
                leja_decide(a.st, a.coef, a.mi, a.m, a.nk, tot[0], 0.0, false);
            }
        }
    }
}

// ----------------------------------------------------------------- KIOPS
struct ArnVArgs {
    int64_t n;            // operator dimension (the n-part)
    int p;                // tail length
    const double* jv;     // generic augment: op.apply(V[j-1,:n]) (already scaled)
    const double* win[4]; // window rows V[lo..jj-1]
    int nwin;
    const double* aug[5];
    int aug_tail[5];
    int naug;
    double aug_scale;
    double* w;            // V[jj]
    double* H;
    int ldh;
    int jj;
    double tail0[5];      // init: tail values of V[0]
    const double* src;    // init: V[0][:n] source
    ek_arnoldi_state* st;
    double* work;
    int repro;            // order-independent sums (ek_xsum.cuh)
};

// Slab mode: channel 0 of part[] (EK_ARN_PART_*) from a vector pass.
__device__ __forceinline__ void arn_part_store(double* part, int repro, double ssq,
                                               const XAcc& xt) {
    if (repro) xstore(reinterpret_cast<long long*>(part), xt);
    else part[0] = ssq;
    part[EK_ARN_PART_COUNT] = 0.0;
    part[EK_ARN_PART_TAG] = repro ? 1.0 : 0.0;
}

// V[0] = [w_l ; tail], beta = ||V[0]||  (kiops.py:168-176)
__global__ void __launch_bounds__(TPB) k_arn_init(const ArnVArgs a) {
    double acc[1] = {0.0};
    XAcc xs[1];
    xzero(xs[0]);
    const bool rp = a.repro != 0;
    const bool vec = al16d(a.src) && al16d(a.w);
    EK_FOR4(e0, a.n) {
        const bool full = vec && e0 + 4 <= a.n;
        double v[4];
        ld4(a.src, e0, a.n, full, v);
        st4(a.w, e0, a.n, full, v);
#pragma unroll
        for (int w = 0; w < 4; ++w) {  // zeros past n
            if (rp) xadd<false>(xs[0], v[w] * v[w]);
            else acc[0] += v[w] * v[w];
        }
    }
    double tot[1];
    XAcc xt[1];
    if (reduce_grid<1, 1>(acc, xs, rp, a.work, &a.st->ticket, false, tot, xt)) {
        if (threadIdx.x == 0) {
            double ssq = tot[0];
            if (a.st->defer) {  // slab: beta from the gathered sums (which 3)
                for (int t = 0; t < a.p; ++t) a.w[a.n + t] = a.tail0[t];
                arn_part_store(a.st->part, rp, tot[0], xt[0]);
                a.st->happy = 0;
                a.st->status = EK_ST_OK;
                a.st->j = 0;
                return;
            }
            for (int t = 0; t < a.p; ++t) {
                a.w[a.n + t] = a.tail0[t];
                ssq += a.tail0[t] * a.tail0[t];
            }
            const double beta = sqrt(ssq);
            a.st->nrm = beta;
            a.st->beta = beta;
            a.st->happy = 0;
            a.st->status = EK_ST_OK;
            a.st->j = 0;
        }
    }
}

// generic pass A: w[:n] = jv + tail@uflip, tail shift, window dots
__global__ void __launch_bounds__(TPB) k_arn_augment(const ArnVArgs a) {
    const ek_arnoldi_state* cst = a.st;
    if (cst->happy || cst->status) return;
    double augc[5];  // tail * nu, exact because nu is a power of two
#pragma unroll
    for (int t = 0; t < 5; ++t)
        augc[t] = t < a.naug ? a.win[a.nwin - 1][a.n + a.aug_tail[t]] * a.aug_scale : 0.0;
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t e = (int64_t)blockIdx.x * TPB + threadIdx.x; e < a.n;
         e += (int64_t)gridDim.x * TPB) {
        double augv = 0.0;
#pragma unroll
        for (int t = 0; t < 5; ++t)
            if (t < a.naug) augv = augv + (augc[t] * __ldg(a.aug[t] + e));
        const double w = __ldg(a.jv + e) + augv;
        a.w[e] = w;
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q < a.nwin) acc[q] += __ldg(a.win[q] + e) * w;
    }
    block_sum<4>(acc);
    if (publish_and_arrive<4>(acc, a.work, &a.st->ticket)) {
        double tot[4];
        gather_partials<4>(a.work, gridDim.x, tot);
        if (threadIdx.x == 0) {
            const int64_t n = a.n;
            const double* prev = a.win[a.nwin - 1];
            for (int t = 0; t + 1 < a.p; ++t) a.w[n + t] = prev[n + t + 1];
            if (a.p > 0) a.w[n + a.p - 1] = 0.0;
            const int lo = a.jj - a.nwin;
            for (int q = 0; q < a.nwin; ++q) {
                double tl = 0.0;
                for (int t = 0; t < a.p; ++t) tl += a.win[q][n + t] * a.w[n + t];
                a.H[(long)(lo + q) * a.ldh + (a.jj - 1)] = tot[q] + tl;
            }
            a.H[(long)a.jj * a.ldh + (a.jj - 1)] = 0.0;
        }
    }
}

// pass B: V[j] -= V[lo:j].T @ H[lo:j, j-1]; nrm = ||V[j]||; happy test
// (kiops.py:188-193). Runs over the full n+p row.
__global__ void __launch_bounds__(TPB) k_arn_orth(const ArnVArgs a) {
    const ek_arnoldi_state* cst = a.st;
    if (cst->happy || cst->status) return;
    const int lo = a.jj - a.nwin;
    double h[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) h[q] = q < a.nwin ? a.H[(long)(lo + q) * a.ldh + (a.jj - 1)] : 0.0;
    const int64_t len = a.n + a.p;
    // slab: the tail is added once, in the decision; repro mode forms the
    // norm the same way on the whole grid (the n-part as an order-independent
    // sum, then the tail terms), so both give the same bits
    const bool rp = a.repro != 0;
    const bool nonly = cst->defer != 0 || rp;
    double acc[1] = {0.0};
    XAcc xs[1];
    xzero(xs[0]);
    bool vec = al16d(a.w);
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (q < a.nwin) vec = vec && al16d(a.win[q]);
    EK_FOR4(e0, len) {
        const bool full = vec && e0 + 4 <= len;
        double wv[4], t[4];
        ld4c(a.w, e0, len, full, wv);
        ld4(a.win[0], e0, len, full, t);
#pragma unroll
        for (int w = 0; w < 4; ++w) t[w] = t[w] * h[0];
#pragma unroll
        for (int q = 1; q < 4; ++q)
            if (q < a.nwin) {
                double x[4];
                ld4(a.win[q], e0, len, full, x);
#pragma unroll
                for (int w = 0; w < 4; ++w) t[w] = t[w] + (x[w] * h[q]);
            }
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            wv[w] = wv[w] - t[w];
            if (!nonly || e0 + w < a.n) {  // zeros past len
                if (rp) xadd<false>(xs[0], wv[w] * wv[w]);
                else acc[0] += wv[w] * wv[w];
            }
        }
        st4(a.w, e0, len, full, wv);
    }
    double tot[1];
    XAcc xt[1];
    if (reduce_grid<1, 1>(acc, xs, rp, a.work, &a.st->ticket, false, tot, xt)) {
        if (threadIdx.x == 0) {
            ek_arnoldi_state* st = a.st;
            if (st->defer) {
                arn_part_store(st->part, rp, tot[0], xt[0]);
                return;
            }
            double ssq = tot[0];
            if (rp)  // as k_arn_decide (which = 1): the tail, written by this pass
                for (int t = 0; t < a.p; ++t) {
                    const double tv = __ldcg(a.w + a.n + t);
                    ssq += tv * tv;
                }
            const double nrm = sqrt(ssq);
            st->nrm = nrm;
            if (nrm < st->tol) {  // happy breakdown, kiops.py:190-192
                st->happy = 1;
                st->j = a.jj;
            } else {
                a.H[(long)a.jj * a.ldh + (a.jj - 1)] = nrm;
            }
        }
    }
}

// pass C: V[j] /= nrm; ||V[j,:n]|| for the next FD increment (kiops.py:194).
__global__ void __launch_bounds__(TPB) k_arn_scale(const ArnVArgs a) {
    const ek_arnoldi_state* cst = a.st;
    if (cst->happy || cst->status) return;
    const Dv nrm = mkdv(cst->nrm);
    const int64_t len = a.n + a.p;
    const bool rp = a.repro != 0;
    double acc[1] = {0.0};
    XAcc xs[1];
    xzero(xs[0]);
    const bool vec = al16d(a.w);
    EK_FOR4(e0, len) {
        const bool full = vec && e0 + 4 <= len;
        double v[4];
        ld4c(a.w, e0, len, full, v);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            v[w] = dv(v[w], nrm);
            if (e0 + w < a.n) {
                if (rp) xadd<false>(xs[0], v[w] * v[w]);
                else acc[0] += v[w] * v[w];
            }
        }
        st4(a.w, e0, len, full, v);
    }
    double tot[1];
    XAcc xt[1];
    if (reduce_grid<1, 1>(acc, xs, rp, a.work, &a.st->ticket, false, tot, xt)) {
        if (threadIdx.x == 0) {
            if (a.st->defer) arn_part_store(a.st->part, rp, tot[0], xt[0]);
            else a.st->nvn = sqrt(tot[0]);
            a.st->j = a.jj;
        }
    }
}

// Slab mode: the decision of one Arnoldi pass from the gathered per-rank
// part[] blocks (EK_ARN_PART_*; tails, replicated on every rank, added once).
__global__ void k_arn_decide(const ArnVArgs a, const double* g, int nranks, int which) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    ek_arnoldi_state* st = a.st;
    // channel q of the gathered part[] blocks (EK_ARN_PART_*): the exact
    // merge of the ranks' integer accumulators (repro mode: the same bits
    // for every P), else the rank-ordered fp64 sum
    const bool xs = g[EK_ARN_PART_TAG] != 0.0;
    auto sum = [&](int q) {
        if (xs) {
            XAcc tot;
            xzero(tot);
            for (int r = 0; r < nranks; ++r)
                xmerge(tot, xload(reinterpret_cast<const long long*>(
                                g + (long)r * EK_ARN_PART_SLOTS + q * XSLOTS)));
            return xvalue(tot);
        }
        double s = g[q * XSLOTS];
        for (int r = 1; r < nranks; ++r) s = s + g[(long)r * EK_ARN_PART_SLOTS + q * XSLOTS];
        return s;
    };
    auto count = [&]() {
        double s = 0.0;
        for (int r = 0; r < nranks; ++r) s += g[(long)r * EK_ARN_PART_SLOTS + EK_ARN_PART_COUNT];
        return s;
    };
    const int64_t n = a.n;
    if (which == 3) {  // after init: beta = ||[w ; tail]||  (kiops.py:176)
        double ssq = sum(0);
        for (int t = 0; t < a.p; ++t) ssq += a.w[n + t] * a.w[n + t];
        st->nrm = sqrt(ssq);
        st->beta = st->nrm;
        return;
    }
    if (st->happy || st->status) return;
    if (which == 0) {  // after pass A: H column (kiops.py:187) + non-finite Jv
        if (count() > 0.0) {
            st->status = EK_ST_JV_NONFINITE;
            return;
        }
        const int lo = a.jj - a.nwin;
        for (int q = 0; q < a.nwin; ++q) {
            double tl = 0.0;
            for (int t = 0; t < a.p; ++t) tl += a.win[q][n + t] * a.w[n + t];
            a.H[(long)(lo + q) * a.ldh + (a.jj - 1)] = sum(q) + tl;
        }
        a.H[(long)a.jj * a.ldh + (a.jj - 1)] = 0.0;
    } else if (which == 1) {  // after pass B: ||w||, happy breakdown (kiops.py:188-193)
        double ssq = sum(0);
        for (int t = 0; t < a.p; ++t) ssq += a.w[n + t] * a.w[n + t];
        const double nrm = sqrt(ssq);
        st->nrm = nrm;
        if (nrm < st->tol) {
            st->happy = 1;
            st->j = a.jj;
        } else {
            a.H[(long)a.jj * a.ldh + (a.jj - 1)] = nrm;
        }
    } else {  // after pass C: ||V[jj,:n]|| for the next FD increment
        st->nvn = sqrt(sum(0));
    }
}

// out = sum_i coef[i] * V_i[:n]   (kiops.py:267, 270)
constexpr int MAXB = 136;
struct CombineArgs {
    int64_t n;
    int j;
    double* out;
    const double* rows[MAXB];
    double coef[MAXB];
};
__global__ void __launch_bounds__(TPB) k_basis_combine(const CombineArgs a) {
    bool vec = al16d(a.out);
    for (int i = 0; i < a.j; ++i) vec = vec && al16d(a.rows[i]);
    EK_FOR4(e0, a.n) {
        const bool full = vec && e0 + 4 <= a.n;
        double s[4], x[4];
        ld4(a.rows[0], e0, a.n, full, x);
#pragma unroll
        for (int w = 0; w < 4; ++w) s[w] = a.coef[0] * x[w];
        for (int i = 1; i < a.j; ++i) {
            ld4(a.rows[i], e0, a.n, full, x);
#pragma unroll
            for (int w = 0; w < 4; ++w) s[w] = s[w] + (a.coef[i] * x[w]);
        }
        st4(a.out, e0, a.n, full, s);
    }
}

// ------------------------------------------------------------- power init
// ||v0|| -> st->nw (the divisor of the first iterate), FD: ||v0/||v0|| || -> nv
__global__ void __launch_bounds__(TPB) k_power_norm(int64_t len, const double* __restrict__ x,
                                                    int scaled, ek_power_state* st,
                                                    double* work, int repro) {
    if (scaled && (st->done || st->status)) return;
    const Dv d = mkdv(st->nw);
    double acc[1] = {0.0};
    XAcc xs[1];
    xzero(xs[0]);
    const bool vec = al16d(x);
    EK_FOR4(e0, len) {
        double v[4];
        ld4(x, e0, len, vec && e0 + 4 <= len, v);
#pragma unroll
        for (int w = 0; w < 4; ++w) {
            if (e0 + w >= len) break;
            if (scaled) v[w] = dv(v[w], d);
            if (repro) xadd<false>(xs[0], v[w] * v[w]);
            else acc[0] += v[w] * v[w];
        }
    }
    double tot[1];
    XAcc xt[1];
    if (reduce_grid<1, 1>(acc, xs, repro != 0, work, &st->ticket, false, tot, xt)) {
        if (threadIdx.x == 0) {
            if (st->defer) {
                part_store_v(st->part, repro, tot[0], xt[0]);
            } else if (scaled) {
                st->nv = sqrt(tot[0]);
            } else {
                st->nw = sqrt(tot[0]);
            }
        }
    }
}

// ----------------------------------------------------------------- vexpr
// Elementwise stack program, NumPy order. Opcode word: op | (arg << 8).
enum {
    VX_LOAD = 1,   // push in[arg][e]
    VX_CONST = 2,  // push scal[arg]
    VX_ADD = 3, VX_SUB = 4, VX_MUL = 5, VX_DIV = 6, VX_NEG = 7,
    VX_STORE = 8,  // out[arg][e] = top (keeps it)
    VX_POP = 9,
    VX_NORM = 10,  // acc[arg] += top*top
    VX_CHECK = 11, // flags: bit0 nonzero, bit1 non-finite (of top)
    VX_ACC = 12    // acc[arg] += top   (dot products)
};
constexpr int VX_MAXPROG = 48;
struct VexprArgs {
    int64_t len;
    int nprog;
    int32_t prog[VX_MAXPROG];
    double scal[16];
    const double* in[8];
    double* out[4];
    ek_scalar_state* st;
    double* work;
    int reduce;  // 1 if the program has NORM/CHECK ops
    int repro;   // order-independent NORM / ACC channels (ek_xsum.cuh)
};
__global__ void __launch_bounds__(TPB) k_vexpr(const VexprArgs a) {
    double acc[4] = {0.0, 0.0, 0.0, 0.0};  // 0,1: norms ; 2: nonzero ; 3: non-finite
    XAcc xs[2];
    xzero(xs[0]);
    xzero(xs[1]);
    for (int64_t e = (int64_t)blockIdx.x * TPB + threadIdx.x; e < a.len;
         e += (int64_t)gridDim.x * TPB) {
        double s0 = 0, s1 = 0, s2 = 0, s3 = 0, s4 = 0, s5 = 0;  // register stack
        int sp = 0;
#define VX_PUSH(v)                                  \
    do {                                            \
        const double v_ = (v);                      \
        switch (sp) {                               \
            case 0: s0 = v_; break;                 \
            case 1: s1 = v_; break;                 \
            case 2: s2 = v_; break;                 \
            case 3: s3 = v_; break;                 \
            case 4: s4 = v_; break;                 \
            default: s5 = v_; break;                \
        }                                           \
        ++sp;                                       \
    } while (0)
#define VX_AT(i) ((i) == 0 ? s0 : (i) == 1 ? s1 : (i) == 2 ? s2 : (i) == 3 ? s3 : (i) == 4 ? s4 : s5)
        for (int pc = 0; pc < a.nprog; ++pc) {
            const int w = a.prog[pc];
            const int op = w & 0xff, arg = w >> 8;
            switch (op) {
                case VX_LOAD: VX_PUSH(__ldg(a.in[arg] + e)); break;
                case VX_CONST: VX_PUSH(a.scal[arg]); break;
                case VX_NEG: {
                    const double t = VX_AT(sp - 1);
                    --sp;
                    VX_PUSH(-t);
                } break;
                case VX_STORE: a.out[arg][e] = VX_AT(sp - 1); break;
                case VX_POP: --sp; break;
                case VX_NORM: {  // channel 0 or 1 (static indices: registers)
                    const double t = VX_AT(sp - 1);
                    const double tt = t * t;
                    if (a.repro) {
                        if (arg == 0) xadd<false>(xs[0], tt);
                        else xadd<false>(xs[1], tt);
                    } else if (arg == 0) acc[0] += tt;
                    else acc[1] += tt;
                } break;
                case VX_ACC: {
                    const double t = VX_AT(sp - 1);
                    if (a.repro) {
                        if (arg == 0) xadd<true>(xs[0], t);
                        else xadd<true>(xs[1], t);
                    } else if (arg == 0) acc[0] += t;
                    else acc[1] += t;
                } break;
                case VX_CHECK: {
                    const double t = VX_AT(sp - 1);
                    acc[2] += t != 0.0 ? 1.0 : 0.0;
                    acc[3] += isfinite(t) ? 0.0 : 1.0;
                } break;
                default: {
                    const double b = VX_AT(sp - 1);
                    const double x = VX_AT(sp - 2);
                    sp -= 2;
                    double r;
                    if (op == VX_ADD) r = x + b;
                    else if (op == VX_SUB) r = x - b;
                    else if (op == VX_MUL) r = x * b;
                    else r = x / b;
                    VX_PUSH(r);
                } break;
            }
        }
#undef VX_PUSH
#undef VX_AT
    }
    if (a.reduce) {
        double tot[4];
        XAcc xt[2];
        if (reduce_grid<4, 2>(acc, xs, a.repro != 0, a.work, &a.st->ticket, false, tot, xt)) {
            if (threadIdx.x == 0) {
                if (a.repro) xstore((long long*)a.st->xs, xt[0]);
                a.st->repro = a.repro;
                a.st->val[0] = tot[0];
                a.st->val[1] = sqrt(tot[0]);
                a.st->val[2] = tot[1];
                a.st->val[3] = sqrt(tot[1]);
                a.st->flag |= (tot[2] > 0.0 ? 1 : 0) | (tot[3] > 0.0 ? 2 : 0);
            }
        }
    }
}

// ------------------------------------------------------------- lincomb
// Up to LC_OUT outputs, each a left fold over up to LC_TERMS terms of up to
// LC_IN shared inputs: out = fin(((t0 + t1) + t2) + ...), term = x, c*x or
// x/c, fin = identity, *s or /s. This covers every stage expression of the
// steppers in NumPy's exact rounding order (a - c*b is folded as
// a + (-c)*b, which is bit-identical). Output 0 may be "virtual" (not
// stored) and is the one reduced: ||out0||^2 and nonzero / non-finite flags.
constexpr int LC_IN = 8, LC_OUT = 3, LC_TERMS = 6;
enum { LT_X = 0, LT_MUL = 1, LT_DIV = 2, LT_MUL2 = 3 };
struct LincombArgs {
    int64_t len;
    const double* in[LC_IN];
    double* out[LC_OUT];
    int nout;
    int nterm[LC_OUT];
    int src[LC_OUT][LC_TERMS];
    int mode[LC_OUT][LC_TERMS];
    Dv coef[LC_OUT][LC_TERMS];   // c (LT_MUL: c.d is the factor; LT_MUL2: c.d * (c.r * x)) or divisor
    int fin[LC_OUT];             // 0 none, 1 multiply, 2 divide
    Dv fval[LC_OUT];
    int reduce;
    ek_scalar_state* st;
    double* work;
    int repro;  // order-independent ||out0||^2 (ek_xsum.cuh)
};

__device__ __forceinline__ double lc_term(const LincombArgs& a, int o, int t, double x) {
    const int m = a.mode[o][t];
    if (m == LT_MUL) return a.coef[o][t].d * x;
    if (m == LT_DIV) return dv(x, a.coef[o][t]);
    if (m == LT_MUL2) return a.coef[o][t].d * (a.coef[o][t].r * x);
    return x;
}

// 4 consecutive elements per thread and iteration (two 16-byte loads per
// term), all term loads issued before the fold.
template <int NOUT, bool ALIGNED>
__global__ void __launch_bounds__(TPB) k_lincomb(const LincombArgs a) {
    constexpr int W = 4;
    double red[3] = {0.0, 0.0, 0.0};
    XAcc xs[1];
    xzero(xs[0]);
    const int64_t ngroups = (a.len + W - 1) / W;
    for (int64_t gi = (int64_t)blockIdx.x * TPB + threadIdx.x; gi < ngroups;
         gi += (int64_t)gridDim.x * TPB) {
        const int64_t e0 = gi * W;
        const bool full = ALIGNED && e0 + W <= a.len;
        double r[W];
#pragma unroll
        for (int o = 0; o < NOUT; ++o) {
            double x[LC_TERMS][W];
#pragma unroll
            for (int t = 0; t < LC_TERMS; ++t) {
                if (t < a.nterm[o]) {
                    const double* p = a.in[a.src[o][t]] + e0;
                    if (full) {
                        const double2 v0 = __ldg(reinterpret_cast<const double2*>(p));
                        const double2 v1 = __ldg(reinterpret_cast<const double2*>(p) + 1);
                        x[t][0] = v0.x; x[t][1] = v0.y; x[t][2] = v1.x; x[t][3] = v1.y;
                    } else {
#pragma unroll
                        for (int w = 0; w < W; ++w) x[t][w] = e0 + w < a.len ? __ldg(p + w) : 0.0;
                    }
                }
            }
            double s[W];
#pragma unroll
            for (int t = 0; t < LC_TERMS; ++t) {
                if (t < a.nterm[o]) {
#pragma unroll
                    for (int w = 0; w < W; ++w) {
                        const double v = lc_term(a, o, t, x[t][w]);
                        s[w] = t == 0 ? v : s[w] + v;
                    }
                }
            }
#pragma unroll
            for (int w = 0; w < W; ++w) {
                if (a.fin[o] == 1) s[w] = s[w] * a.fval[o].d;
                else if (a.fin[o] == 2) s[w] = dv(s[w], a.fval[o]);
            }
            double* q = a.out[o];
            if (q) {
                if (full) {
                    reinterpret_cast<double2*>(q + e0)[0] = make_double2(s[0], s[1]);
                    reinterpret_cast<double2*>(q + e0)[1] = make_double2(s[2], s[3]);
                } else {
#pragma unroll
                    for (int w = 0; w < W; ++w)
                        if (e0 + w < a.len) q[e0 + w] = s[w];
                }
            }
#pragma unroll
            for (int w = 0; w < W; ++w) {
                if (o == 0) r[w] = s[w];
                else if (o == 1 && a.reduce == 2) r[w] = r[w] - s[w];  // ||out0 - out1||
            }
        }
        if (a.reduce) {
#pragma unroll
            for (int w = 0; w < W; ++w) {
                if (e0 + w < a.len) {
                    if (a.repro) xadd<false>(xs[0], r[w] * r[w]);
                    else red[0] += r[w] * r[w];
                    red[1] += r[w] != 0.0 ? 1.0 : 0.0;
                    red[2] += isfinite(r[w]) ? 0.0 : 1.0;
                }
            }
        }
    }
    if (a.reduce) {
        double tot[3];
        XAcc xt[1];
        if (reduce_grid<3, 1>(red, xs, a.repro != 0, a.work, &a.st->ticket, false, tot, xt)) {
            if (threadIdx.x == 0) {
                if (a.repro) xstore((long long*)a.st->xs, xt[0]);
                a.st->repro = a.repro;
                a.st->val[0] = tot[0];
                a.st->val[1] = sqrt(tot[0]);
                a.st->flag |= (tot[1] > 0.0 ? 1 : 0) | (tot[2] > 0.0 ? 2 : 0);
            }
        }
    }
}

// --------------------------------------------------------- self test
// fast[i] = dv(x[i], mkdv(d[i])), exact[i] = x[i] / d[i] (division
// instruction): proves the reciprocal-correction quotient is bit-identical.
__global__ void __launch_bounds__(TPB) k_selftest_div(int64_t n, const double* __restrict__ x,
                                                      const double* __restrict__ d,
                                                      double* __restrict__ fast,
                                                      double* __restrict__ exact) {
    for (int64_t e = (int64_t)blockIdx.x * TPB + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * TPB) {
        const double xv = x[e], dd = d[e];
        fast[e] = dv(xv, mkdv(dd));
        exact[e] = xv / dd;
    }
}

// ------------------------------------------------------------ dense GEMV
// y = A x, one warp per row, fixed lane order (linalg.py:87-90).
__global__ void __launch_bounds__(TPB) k_dense_gemv(int64_t n, const double* __restrict__ A,
                                                    const double* __restrict__ x,
                                                    double* __restrict__ y) {
    const int lane = threadIdx.x & 31;
    const int64_t row = ((int64_t)blockIdx.x * TPB + threadIdx.x) >> 5;
    if (row >= n) return;
    double s = 0.0;
    for (int64_t c = lane; c < n; c += 32) s += __ldg(A + row * n + c) * __ldg(x + c);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
    if (lane == 0) y[row] = s;
}

}  // namespace ek
