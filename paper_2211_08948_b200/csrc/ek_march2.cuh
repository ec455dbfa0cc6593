// ek_march2.cuh — row-marching TMA 2-D stencil kernel (sm_100a).
//
// Same value / epilogue algebra as k_tma2d / k_stencil2d, with a different
// data movement: a block owns a contiguous, balanced range of rows of one
// (or two) column strips and marches down it one grid row at a time.
//
// Strip = W2 = 256 columns (one per thread); one pipeline stage holds ONE
// row of the strip. Each field row segment is ONE 1-D bulk copy
// (`cp.async.bulk`, byte count on the stage mbarrier): for the raw
// neighbourhood fields (u, y / k, u) the 2080 B from column j0-2 to j0+257,
// i.e. the strip plus the neighbour strips' edge columns; for the centre
// fields (f(u), Leja accumulators, Arnoldi window / augmentation rows) the
// 2 KB of the strip. At the domain edge the segment is clipped to the row
// and one extra 16-B copy brings the ghost column pair (columns n-2, n-1 /
// 0, 1 for periodic; 0, 1 / n-2, n-1 for np.pad 'reflect'). Row i is
// computed from the stages of rows i-1, i, i+1, so every raw row is fetched
// once per item (plus one ghost row at each end): no halo row or column is
// re-read beyond 2 x 16 B per row, and a row costs one copy per field.
// Ghost rows outside the domain are copied from the wrapped / reflected row
// or the slab halo buffer.
// Work split: see Item2. Pipeline as in k_tma3d: full[s] counts the bytes of the row in
// stage s, a shared counter the warps that released it; the last warp to
// release a stage refills it with the row S sequence numbers ahead.
#pragma once

#include "ek_stream.cuh"

namespace ek {

constexpr int W2 = 256;    // columns per strip
constexpr int T2 = 256;    // compute threads: one column each
constexpr int NW2 = T2 / 32;
#ifndef EK_TIGHT2
#define EK_TIGHT2 1  // 1: K = 0 Leja instance: row loop without per-row divisions
#endif
#ifndef EK_WAIT2_NS
#define EK_WAIT2_NS 0  // > 0: suspend-time hint (ns) of the row waits' try_wait (measured: none is best)
#endif
#ifndef EK_PROD2
#define EK_PROD2 1  // 1: one extra producer warp issues the row copies
#endif
constexpr int NT2 = T2 + (EK_PROD2 ? 32 : 0);  // threads per block
// Resident blocks per SM the register budget is sized for. The Leja
// iteration without accumulators (K = 0, deferred accumulation) moves so few
// bytes per point that it is bound by its fp64 dependency chains, not by
// DRAM: a third block per SM gives the schedulers the warps to hide them.
#ifndef EK_MARCH_LB0
#define EK_MARCH_LB0 3
#endif
template <int EP, int K>
__host__ __device__ constexpr int march2_lb() {
    return (EP == EP_LEJA && K == 0) ? EK_MARCH_LB0 : 2;
}
constexpr int RAW2 = 272;  // doubles per raw row slot: element e <-> column j0 - 2 + e
constexpr int CTR2 = 256;  // doubles per centre row slot

// The FD passes re-evaluate f(u_n) from the u neighbourhood they stage anyway
// instead of streaming it (one vector less to move). The Leja iteration
// without accumulators (K = 0) is bound by its fp64 work, not by DRAM, so
// that instance streams the stored f(u_n) as a centre field instead and
// evaluates f once per point.
#ifndef EK_FD_READFU
#define EK_FD_READFU 2  // 0 re-evaluate, 1 staged: 0.1955 ms, 2 direct loads: 0.1935 ms (config 4)
#endif
template <int EV, int EP, int K>
__host__ __device__ constexpr bool march_rfu() {
    return EK_FD_READFU && EV == EV_FD && EP == EP_LEJA && K == 0;
}
// EK_FD_READFU = 1: f(u_n) staged as a centre field of the row ring; 2: loaded
// by the thread that uses it straight from global memory one row ahead (the
// ring keeps its smaller stage, so more rows are in flight per block).
__host__ __device__ constexpr bool march_rfu_direct_on() {
    return EK_FD_READFU == 2 && EK_PROD2 && EK_TIGHT2;
}
template <int EV, int EP, int K>
__host__ __device__ constexpr bool march_rfu_staged() {
    return march_rfu<EV, EP, K>() && !march_rfu_direct_on();
}
template <int EV, int EP, int K>
__host__ __device__ constexpr bool march_rfu_direct() {
    return march_rfu<EV, EP, K>() && EK_FD_READFU == 2 && EK_PROD2 && EK_TIGHT2;
}
template <int EV, int EP, int K>
__host__ __device__ constexpr bool march_fu() {
    return needs_fu<EV>() || march_rfu_staged<EV, EP, K>();
}
template <int EV, int EP, int K>
__host__ __device__ constexpr int nctr2() {
    return nctr_maps<EV, EP, K>() + (march_rfu_staged<EV, EP, K>() ? 1 : 0);
}

template <int EV, int EP, int NC, int K>
__host__ __device__ constexpr int stage2_doubles() {
    return nraw<EV>() * NC * RAW2 + nctr2<EV, EP, K>() * NC * CTR2;
}

// Work items: strip s (columns s*W2 ..) x row segment g (rows
// [g rows / NG, (g+1) rows / NG)), numbered t = g * NS + s. The host sizes
// the grid to NS * NG blocks, so block b owns exactly one item and, at any
// moment, the blocks of a segment read the same few rows across the whole
// width: the concurrently open DRAM pages are whole contiguous rows, not
// one 2 KB piece per block. (Grids wider than the persistent grid has
// blocks fall back to NG = 1 and a strided item loop.)
struct Item2 {
    long t;
    int j0, r0, L;
};
__device__ __forceinline__ Item2 item2(long t, int ns, int ng, int rows) {
    Item2 it;
    it.t = t;
    const long s = t % ns, g = t / ns;
    it.j0 = (int)s * W2;
    it.r0 = (int)(g * rows / ng);
    it.L = (int)((g + 1) * rows / ng) - it.r0;
    return it;
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
        ::"r"(smem_u32(dst)), "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, uint32_t bytes,
                                              uint64_t* bar, uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1], %2, [%3], %4;"
        ::"r"(smem_u32(dst)), "l"((uint64_t)src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
        : "memory");
}

// Centre field g of a stage: f(u_n) first (if used), then the Leja
// accumulators / Arnoldi slots.
template <int EV, int EP>
__device__ __forceinline__ const double* ctr_field(const KArgs& a, int g) {
    constexpr int FU = needs_fu<EV>() ? 1 : 0;
    if (g < FU) return a.fu;
    if constexpr (EP == EP_ARN) return arn_slot(a, g - FU);
    if constexpr (EP == EP_REM) return a.xin;
    return a.p[g - FU];
}

// Issue position `pos` (row r0 - 1 + pos) of item `it` into stage `buf`.
template <int EV, int EP, int NC, int K>
__device__ __forceinline__ void issue_row(const KArgs& a, double* buf, uint64_t* bar,
                                          const Item2& it, int pos, int rows, uint32_t active) {
    constexpr int NR = nraw<EV>(), NCM = nctr2<EV, EP, K>();
    constexpr int FU = march_fu<EV, EP, K>() ? 1 : 0;
    const int i = it.r0 - 1 + pos;
    const bool centre = pos >= 1 && pos <= it.L;
    const long cols = a.g.n;
    const bool per = a.g.bc == EK_BC_PERIODIC;
    // raw segment [c0, c1) of the row, ghost column pairs at the domain edge
    const bool le = it.j0 == 0, re = it.j0 + W2 >= cols;
    const long c0 = le ? 0 : it.j0 - 2, c1 = re ? cols : it.j0 + W2 + 2;
    const uint32_t seg = (uint32_t)(c1 - c0) * 8;
    const uint32_t cbytes = (uint32_t)((re ? cols - it.j0 : W2) * 8);
    uint32_t bytes = NR * NC * (seg + (le ? 16 : 0) + (re ? 16 : 0));
    if (centre) {
#pragma unroll
        for (int g = 0; g < NCM; ++g)
            if (g < FU || ((active >> (g - FU)) & 1u)) bytes += NC * cbytes;
    }
    mbar_arrive_expect(bar, bytes);
    const double* rb[2];
    const double* rh[2];
    raw_fields<EV>(a, rb, rh);
    const bool in = i >= 0 && i < rows;
    const long wi = in ? i : wrap_idx(i, rows, a.g.bc);
#pragma unroll
    for (int f = 0; f < NR; ++f)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            double* dst = buf + (f * NC + c) * RAW2;
            const double* row = (!in && a.g.slab)
                                    ? rh[f] + ((i < 0 ? 0 : 1) * (long)NC + c) * cols  // halo [2][ncomp][n]
                                    : rb[f] + c * a.npts + wi * cols;
            bulk_g2s(dst + (c0 - (it.j0 - 2)), row + c0, seg, bar);
            if (le) bulk_g2s(dst, row + (per ? cols - 2 : 0), 16, bar);
            if (re) bulk_g2s(dst + (cols - it.j0 + 2), row + (per ? 0 : cols - 2), 16, bar);
        }
    if (centre) {
        double* ctr = buf + NR * NC * RAW2;
        const uint64_t pol = policy_evict_first();
#pragma unroll
        for (int g = 0; g < NCM; ++g)
            if (g < FU || ((active >> (g - FU)) & 1u)) {
                const double* fb = (march_rfu_staged<EV, EP, K>() && g == 0) ? a.fu
                                                                      : ctr_field<EV, EP>(a, g);
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    bulk_g2s_hint(ctr + (g * NC + c) * CTR2, fb + c * a.npts + (long)i * cols + it.j0,
                                  cbytes, bar, pol);
            }
    }
}

// Point (i, j) from the row stages pm (i-1), pc (i), pp (i+1); t = column
// offset inside the strip; raw slot element t + 2 is column j.
template <class P, int EV, int EP, int K, class XS>
__device__ __forceinline__ void march2_point(const KArgs& a, const Ctl& ctl, const double* pm,
                                             const double* pc, const double* pp, long i, int j,
                                             int t, int cols, double* acc, XS xs,
                                             const double* fug = nullptr) {
    constexpr int NC = P::NC, NCH = ev_nch(EV), NR = nraw<EV>();
    constexpr int FU = march_fu<EV, EP, K>() ? 1 : 0;
    Nb nb[NC][NCH];
    double yc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        double rc[NR], rxm[NR], rxp[NR], rym[NR], ryp[NR];
#pragma unroll
        for (int f = 0; f < NR; ++f) {
            const int o = (f * NC + c) * RAW2 + t + 2;
            rc[f] = pc[o];
            rxm[f] = pm[o];
            rxp[f] = pp[o];
            rym[f] = pc[o - 1];
            ryp[f] = pc[o + 1];
        }
        yc[c] = rc[yraw<EV>() < NR ? yraw<EV>() : 0];
        double hc[NCH], hxm[NCH], hxp[NCH], hym[NCH], hyp[NCH];
        make_ch<EV, NCH, NR>(ctl, rc, hc);
        make_ch<EV, NCH, NR>(ctl, rxm, hxm);
        make_ch<EV, NCH, NR>(ctl, rxp, hxp);
        make_ch<EV, NCH, NR>(ctl, rym, hym);
        make_ch<EV, NCH, NR>(ctl, ryp, hyp);
#pragma unroll
        for (int h = 0; h < NCH; ++h) nb[c][h] = Nb{hc[h], hxm[h], hxp[h], hym[h], hyp[h], 0.0, 0.0};
    }
    Centre<EV, EP, NC, K> z;
    const double* ctr = pc + NR * NC * RAW2;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if constexpr (march_rfu_direct<EV, EP, K>()) z.fu[c] = fug[c];
        else z.fu[c] = FU ? ctr[c * CTR2 + t] : 0.0;
        if constexpr (EP == EP_RHSN) z.y[c] = yc[c];  // u at the centre
        if constexpr (EP == EP_LEJA || EP == EP_ARN) {
            z.y[c] = yc[c];
#pragma unroll
            for (int q = 0; q < K; ++q)
                z.p[q][c] = (EP == EP_ARN && q == a.nwin - 1)
                                ? yc[c] : ctr[((FU + q) * NC + c) * CTR2 + t];
        }
        if constexpr (EP == EP_REM && K > 0) z.p[0][c] = ctr[(FU * NC + c) * CTR2 + t];
    }
    double val[NC];
    evaluate<P, EV, NCH, march_rfu<EV, EP, K>()>(a, ctl, nb, z.fu, val, z.jbad);
    epilogue<EV, EP, NC, K>(a, ctl, i * cols + j, val, z, acc, xs);
}

// Strips across the row length; segments per strip for a grid of G blocks.
__host__ __device__ __forceinline__ int march2_strips(long cols) { return (int)((cols + W2 - 1) / W2); }
__host__ __device__ __forceinline__ int march2_segs(long G, int ns) {
    return G >= ns ? (int)(G / ns) : 1;
}

template <class P, int EV, int EP, int K, int S, int RP>
__global__ void __launch_bounds__(NT2, (march2_lb<EP, K>())) k_march2d(const KArgs a) {
    static_assert(S >= 4, "row ring needs i-1, i, i+1 and one in flight");
    constexpr int NC = P::NC, NQ = nq_of<EV, EP>();
    constexpr int NR = nraw<EV>();
    constexpr int SD = stage2_doubles<EV, EP, NC, K>();
    extern __shared__ __align__(1024) double smem[];
    __shared__ __align__(8) uint64_t full[S];
#if EK_PROD2
    __shared__ __align__(8) uint64_t empty[S];  // the NW2 compute warps released stage s
#else
    __shared__ int released[S];  // warps that released stage s, cumulative
#endif

    Ctl ctl;
    if (!load_ctl<EV, EP>(a, ctl)) return;
    const int lane = threadIdx.x & 31, t = threadIdx.x;
    const int cols = (int)a.g.n, rows = (int)a.g.rows;
    const long G = gridDim.x;
    const int ns = march2_strips(cols), ng = march2_segs(G, ns);
    const long nitems = (long)ns * ng;

    // Issue the row S sequence numbers after position `pos` of item `it`
    // (if the block has one) into stage s.
    auto issue_ahead = [&](Item2 it, int pos, int s) {
        pos += S;
        while (pos >= it.L + 2) {
            pos -= it.L + 2;
            const long nx = it.t + G;
            if (nx >= nitems) return;
            it = item2(nx, ns, ng, rows);
        }
        issue_row<EV, EP, NC, K>(a, smem + s * SD, &full[s], it, pos, rows, ctr_mask(ctl));
    };

    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
#if EK_PROD2
            mbar_init(&empty[s], NW2);
#else
            released[s] = 0;
#endif
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#if !EK_PROD2
        if (blockIdx.x < nitems) {
            const Item2 it0 = item2(blockIdx.x, ns, ng, rows);
            for (int s = 0; s < S; ++s) issue_ahead(it0, s - S, s);
        }
#endif
    }
    __syncthreads();

    double acc[NQ];
    XAcc xsa[ep_nx(EP)];  // repro mode (RP = 1): the sum channels (ek_xsum.cuh)
#pragma unroll
    for (int q = 0; q < ep_nx(EP); ++q) xzero(xsa[q]);
    const XsT<RP> xs{xsa};
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;

#if EK_PROD2
    // Producer warp (the last one): issues every row of this block's items
    // in sequence order into its ring stage as soon as the NW2 compute warps
    // have released the stage's previous row (as in k_tma3d).
    if ((int)(threadIdx.x >> 5) == NW2) {
        if (lane == 0) {
            long q = 0;
            for (long tt = blockIdx.x; tt < nitems; tt += G) {
                const Item2 it = item2(tt, ns, ng, rows);
                for (int pos = 0; pos < it.L + 2; ++pos, ++q) {
                    const int s = (int)(q % S);
                    if (q >= S) mbar_wait(&empty[s], (uint32_t)(((q / S) - 1) & 1));
                    issue_row<EV, EP, NC, K>(a, smem + s * SD, &full[s], it, pos, rows,
                                             ctr_mask(ctl));
                }
            }
        }
        __syncwarp();
        reduce_and_finalize<EV, EP, NQ, NT2, RP>(a, acc, xsa);
        return;
    }
#endif

    // (the K = 0 Leja instance only: measured neutral for the DRAM-bound ones)
#if EK_PROD2
    if constexpr (EK_TIGHT2 && EP == EP_LEJA && K == 0) {
        // Tight row loop (producer-warp build): the ring position is a stage
        // index plus one phase bit per stage — every sequence number is waited
        // for exactly once by each warp, in order — so the loop carries no
        // division; a warp whose row has not landed sleeps in the barrier unit
        // (try_wait with a suspend-time hint) instead of spinning.
        int sn = 0;         // stage of the next sequence number this warp waits for
        uint32_t ph = 0;    // bit s: parity of that wait on stage s
        auto wait_next = [&]() {
            const int s = sn;
            mbar_wait_ns<EK_WAIT2_NS>(&full[s], (ph >> s) & 1u);
            ph ^= 1u << s;
            sn = s + 1 == S ? 0 : s + 1;
            return s;
        };
        auto release_s = [&](int s) {
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[s]);
        };
        for (long tt = blockIdx.x; tt < nitems; tt += G) {
            const Item2 it = item2(tt, ns, ng, rows);
            const int j = it.j0 + t;
            const bool live = j < cols;
            int sm = wait_next(), sc = wait_next();
            const double* pm = smem + sm * SD;
            const double* pc = smem + sc * SD;
            long i = it.r0;
            for (int p = 1; p <= it.L; ++p, ++i) {
                double fug[NC];
                if constexpr (march_rfu_direct<EV, EP, K>()) {
                    // f(u_n) at this thread's point, in flight while the warp
                    // waits for row i + 1 and evaluates f(u_n + eps y)
#pragma unroll
                    for (int c = 0; c < NC; ++c)
                        fug[c] = live ? __ldg(a.fu + c * a.npts + i * cols + j) : 0.0;
                }
                const int sp = wait_next();
                const double* pp = smem + sp * SD;
                if (live)
                    march2_point<P, EV, EP, K>(a, ctl, pm, pc, pp, i, j, t, cols, acc, xs, fug);
                release_s(sm);
                sm = sc; sc = sp; pm = pc; pc = pp;
            }
            release_s(sm);
            release_s(sc);
        }
    } else
#endif
    {
        auto wait_full = [&](int q) { mbar_wait(&full[q % S], (uint32_t)((q / S) & 1)); };
        auto release = [&](int q, const Item2& it, int pos) {
            __syncwarp();
            if (lane == 0) {
                const int s = q % S;
#if EK_PROD2
                (void)it; (void)pos;
                mbar_arrive(&empty[s]);
#else
                if ((atomicAdd(&released[s], 1) + 1) % NW2 == 0) issue_ahead(it, pos, s);
#endif
            }
        };

        int q0 = 0;  // sequence number of position 0 of the current item
        for (long tt = blockIdx.x; tt < nitems; tt += G) {
            const Item2 it = item2(tt, ns, ng, rows);
            const int j = it.j0 + t;
            const bool live = j < cols;
            wait_full(q0);
            wait_full(q0 + 1);
            int sm = q0 % S, sc = (q0 + 1) % S;
            for (int p = 1; p <= it.L; ++p) {
                wait_full(q0 + p + 1);
                const int sp = sc + 1 == S ? 0 : sc + 1;
                const double* pm = smem + sm * SD;
                const double* pc = smem + sc * SD;
                const double* pp = smem + sp * SD;
                const long i = it.r0 + p - 1;
                if (live) march2_point<P, EV, EP, K>(a, ctl, pm, pc, pp, i, j, t, cols, acc, xs);
                release(q0 + p - 1, it, p - 1);
                sm = sc;
                sc = sp;
            }
            release(q0 + it.L, it, it.L);
            release(q0 + it.L + 1, it, it.L + 1);
            q0 += it.L + 2;
        }
    }
    reduce_and_finalize<EV, EP, NQ, NT2, RP>(a, acc, xsa);
}

}  // namespace ek
