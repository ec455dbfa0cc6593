// ek_stream3.cuh — TMA-pipelined 3-D stencil kernel (sm_100a).
//
// Same value / epilogue algebra as ek_stencil.cuh (k_stencil3d), staged by
// 3-D tensor copies (`cp.async.bulk.tensor.3d`). Layout: flat index
// i*n*n + jy*n + kx, axis 0 (i, the slab axis) outermost; a tensor map views
// a field as (ncomp*rows) x n x n, so component c starts at plane c*rows.
//
// Work item = 64 (kx) x 16 (jy) columns x SEG3 consecutive planes of axis 0.
// A block marches the planes of an item in order; one pipeline stage holds
// one plane of the item: per raw field an 18 x 68 box (jy0-1..jy0+16,
// kx0-2..kx0+65) and per centre field (f(u), accumulators, Arnoldi slots) a
// 16 x 64 box (IY x 64 with IY = 8 when many centre streams are staged);
// 16 warps, each thread computes IY / 8 points of the plane. Plane i is computed from stages i-1, i, i+1, so every raw
// plane is fetched once per item (plus the two ghost planes at its ends)
// and the axis-0 neighbours cost no extra traffic. Ghost planes outside the
// domain are fetched by the copy engine too: the wrapped / reflected plane
// for a whole domain, the halo buffer (its own tensor map) for a slab.
// Ghost rows / columns of axes 1 and 2 (x-y boundary of the item) are read
// from global memory by the lanes that need them (EDGE items only).
//
// Pipeline: full[s] counts the bytes of the plane in stage s; a shared
// counter the warps that released it. The last warp to release a stage
// refills it with the plane S sequence numbers ahead, so copies are issued
// the moment a stage frees up and no warp ever waits for another one.
#pragma once

#include <type_traits>

#include "ek_stream.cuh"

namespace ek {

constexpr int SEG3 = 32;  // planes per work item

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x, int y, int z,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_hint(void* dst, const CUtensorMap* map, int x, int y,
                                                 int z, uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}

// Item geometry: I3X columns (kx) x IY rows (jy); raw boxes carry one
// ghost row above/below and two columns left/right (16-byte multiples).
// IY = 16 where two blocks per SM still hold >= 6 plane stages, else 8
// (many centre streams: Leja k >= 2, Arnoldi windows).
// Thread t computes the plane points t, t + T3, ... of the item (row-major,
// 64 per row): IY * 64 / T3 points per thread and plane.
#ifndef EK_T3
#define EK_T3 512
#endif
#ifndef EK_LB3
#define EK_LB3 2  // resident blocks per SM the register budget is sized for
#endif
#ifndef EK_MAP3_FLAT
#define EK_MAP3_FLAT 0
#endif
#ifndef EK_PROD3
#define EK_PROD3 1  // 1: one extra producer warp issues the plane copies
#endif
#ifndef EK_TIGHT3
#define EK_TIGHT3 1  // 1: the plane loop with hoisted per-thread geometry (producer-warp build)
#endif
#ifndef EK_WAIT3_NS
#define EK_WAIT3_NS 1000  // > 0: suspend-time hint (ns) of the plane waits' try_wait
#endif
#ifndef EK_T3_IY8
#define EK_T3_IY8 256  // compute threads of the IY = 8 items (two points per thread, as IY = 16)
#endif
#ifndef EK_CARRY3
#define EK_CARRY3 0  // 1: single-field instances carry planes i-1 / i in registers (measured slower)
#endif
#ifndef EK_I3X
#define EK_I3X 64  // item width along the contiguous axis (A/B: 128)
#endif
constexpr int I3X = EK_I3X;
constexpr int TBW3 = I3X + 4;
__host__ __device__ constexpr int raw3(int iy) { return (TBW3 * (iy + 2) + 15) / 16 * 16; }
__host__ __device__ constexpr int ctr3(int iy) { return I3X * iy; }
// Ghost side slots of a raw field (boundary items only): the wrapped /
// reflected row above (j = -1) and below (j = n), TBW3 wide, and the ghost
// column pair left (k = -1) and right (k = n), IY + 2 rows; 128-B multiples.
constexpr int GROW3 = (TBW3 + 15) / 16 * 16;  // >= TBW3, a 128-B multiple
__host__ __device__ constexpr int gcol3(int iy) { return (2 * (iy + 2) + 15) / 16 * 16; }
__host__ __device__ constexpr int side3(int iy) { return 2 * GROW3 + 2 * gcol3(iy); }
template <int EV, int EP, int NC, int K>
__host__ __device__ constexpr int stage3_doubles_iy(int iy) {
    return nraw<EV>() * NC * (raw3(iy) + side3(iy)) + nctr_maps<EV, EP, K>() * NC * ctr3(iy);
}
template <int EV, int EP, int NC, int K>
__host__ __device__ constexpr int iy3() {
#ifdef EK_IY3
    if (EK_IY3 == 8 || stage3_doubles_iy<EV, EP, NC, K>(16) * 8 * 5 <= 220 * 1024) return EK_IY3;
#endif
    return (220 * 1024 / EK_LB3) / (stage3_doubles_iy<EV, EP, NC, K>(16) * 8) >= 5 ? 16 : 8;
}
template <int EV, int EP, int NC, int K>
__host__ __device__ constexpr int stage3_doubles() {
    return stage3_doubles_iy<EV, EP, NC, K>(iy3<EV, EP, NC, K>());
}

// Compute threads / threads per block of an instantiation (the producer warp
// is one more warp).
template <int EV, int EP, int NC, int K>
__host__ __device__ constexpr int t3_of() {
    return iy3<EV, EP, NC, K>() == 16 ? EK_T3 : EK_T3_IY8;
}
template <int EV, int EP, int NC, int K>
__host__ __device__ constexpr int nt3_of() {
    return t3_of<EV, EP, NC, K>() + (EK_PROD3 ? 32 : 0);
}

struct Item3 {
    int k0, j0, i0, L;
};
template <int IY>
__device__ __forceinline__ Item3 item3(long t, int n, int rows) {
    const int tk = (n + I3X - 1) / I3X, tj = (n + IY - 1) / IY;
    Item3 it;
    it.k0 = (int)(t % tk) * I3X;
    it.j0 = (int)((t / tk) % tj) * IY;
    it.i0 = (int)(t / ((long)tk * tj)) * SEG3;
    it.L = rows - it.i0 < SEG3 ? rows - it.i0 : SEG3;
    return it;
}

// Thread 0: issue position `pos` (plane i0 - 1 + pos) of item `it`.
template <int EV, int EP, int NC, int K>
__device__ __forceinline__ void issue_plane(const KArgs& a, const TmaMaps& maps, double* buf,
                                            uint64_t* bar, const Item3& it, int pos, int rows,
                                            uint32_t active) {
    constexpr int NR = nraw<EV>(), NCM = nctr_maps<EV, EP, K>();
    constexpr int FU = needs_fu<EV>() ? 1 : 0;
    constexpr int IY = iy3<EV, EP, NC, K>(), RAW3 = raw3(IY), CTR3 = ctr3(IY);
    const int i = it.i0 - 1 + pos;
    const bool centre = pos >= 1 && pos <= it.L;
    const int n = (int)a.g.n;
    // ghost sides needed by this item's points (centre planes only)
    const bool gym = centre && it.j0 == 0, gyp = centre && it.j0 + IY >= n;
    const bool gzm = centre && it.k0 == 0, gzp = centre && it.k0 + I3X >= n;
    uint32_t bytes = NR * NC * (TBW3 * (IY + 2) * 8);
    bytes += NR * NC * (((gym ? 1 : 0) + (gyp ? 1 : 0)) * TBW3 * 8 +
                        ((gzm ? 1 : 0) + (gzp ? 1 : 0)) * 2 * (IY + 2) * 8);
    if (centre) {
#pragma unroll
        for (int g = 0; g < NCM; ++g)
            if (g < FU || ((active >> (g - FU)) & 1u)) bytes += NC * (CTR3 * 8);
    }
    mbar_arrive_expect(bar, bytes);
    const bool in = i >= 0 && i < rows;
#pragma unroll
    for (int f = 0; f < NR; ++f)
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            double* dst = buf + (f * NC + c) * RAW3;
            if (in) {
                tma_load_3d(dst, &maps.m[f], it.k0 - 2, it.j0 - 1, c * rows + i, bar);
            } else if (a.g.slab) {  // halo buffer [2][ncomp][plane]
                tma_load_3d(dst, &maps.h[f], it.k0 - 2, it.j0 - 1, (i < 0 ? 0 : NC) + c, bar);
            } else {
                const int w = (int)wrap_idx(i, rows, a.g.bc);
                tma_load_3d(dst, &maps.m[f], it.k0 - 2, it.j0 - 1, c * rows + w, bar);
            }
            double* sd = buf + NR * NC * RAW3 + NCM * NC * CTR3 + (f * NC + c) * side3(IY);
            const int z = c * rows + i;
            if (gym) tma_load_3d(sd, &maps.gr[f], it.k0 - 2, (int)wrap_idx(-1, n, a.g.bc), z, bar);
            if (gyp) tma_load_3d(sd + GROW3, &maps.gr[f], it.k0 - 2, (int)wrap_idx(n, n, a.g.bc), z, bar);
            // column pair boxes start on an even column (16-byte aligned box
            // origin); the ghost is element (column & 1) of each box row
            if (gzm) tma_load_3d(sd + 2 * GROW3, &maps.gc[f], (int)wrap_idx(-1, n, a.g.bc) & ~1,
                                 it.j0 - 1, z, bar);
            if (gzp) tma_load_3d(sd + 2 * GROW3 + gcol3(IY), &maps.gc[f],
                                 (int)wrap_idx(n, n, a.g.bc) & ~1, it.j0 - 1, z, bar);
        }
    if (centre) {
        double* ctr = buf + NR * NC * RAW3;
        const uint64_t pol = policy_evict_first();
#pragma unroll
        for (int g = 0; g < NCM; ++g)
            if (g < FU || ((active >> (g - FU)) & 1u)) {
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    tma_load_3d_hint(ctr + (g * NC + c) * CTR3, &maps.m[NR + g], it.k0, it.j0,
                                     c * rows + i, bar, pol);
            }
    }
}

// One point (i, jy, kx) from the stages of planes i-1 (pm), i (pc), i+1 (pp);
// ro / co: its offset inside a raw / centre slot.
// EDGE: bit 0 = the item touches a y edge (j = 0 / n-1), bit 1 = a z edge
// (k = 0 / n-1); only those ghost selects are compiled in. zpar: the
// column parity of the wrapped ghost columns -1 / n (launch constants).
// CARRY (one raw field, one component): cv[0] / cv[1] hold the point's
// values in planes i-1 / i from the two previous plane steps, so only plane
// i+1's value is read from its stage (pm is not touched) and the values move
// down one plane afterwards.
template <class P, int EV, int EP, int K, int IY, int EDGE, class XS, bool CARRY = false>
__device__ __forceinline__ void tma3_point(const KArgs& a, const Ctl& ctl, const double* pm,
                                           const double* pc, const double* pp,
                                           int ly, int lx, int jy, int kx, int ro, int co, int n,
                                           long off, double* acc, XS xs, int zpm, int zpp,
                                           double* cv = nullptr) {
    constexpr int NC = P::NC, NCH = ev_nch(EV), NR = nraw<EV>();
    constexpr int FU = needs_fu<EV>() ? 1 : 0;
    constexpr int RAW3 = raw3(IY), CTR3 = ctr3(IY);
    constexpr int SIDE = NR * NC * RAW3 + nctr_maps<EV, EP, K>() * NC * CTR3;
    constexpr bool EY = (EDGE & 1) != 0, EZ = (EDGE & 2) != 0;
    const bool gy_m = EY && jy == 0, gy_p = EY && jy == n - 1;
    const bool gz_m = EZ && kx == 0, gz_p = EZ && kx == n - 1;
    Nb nb[NC][NCH];
    double yc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        double rc[NR], rxm[NR], rxp[NR], rym[NR], ryp[NR], rzm[NR], rzp[NR];
#pragma unroll
        for (int f = 0; f < NR; ++f) {
            const int o = (f * NC + c) * RAW3 + ro;
            const double* bx = pc + o;
            rxp[f] = pp[o];
            if constexpr (CARRY) {
                rxm[f] = cv[0];
                rc[f] = cv[1];
                cv[0] = rc[f];
                cv[1] = rxp[f];
            } else {
                rc[f] = bx[0];
                rxm[f] = pm[o];
            }
            // ghost rows / columns from the side slots the copy engine filled
            const double* sd = pc + SIDE + (f * NC + c) * side3(IY);
            if constexpr (EY) {
                rym[f] = gy_m ? sd[2 + lx] : bx[-TBW3];
                ryp[f] = gy_p ? sd[GROW3 + 2 + lx] : bx[TBW3];
            } else {
                rym[f] = bx[-TBW3];
                ryp[f] = bx[TBW3];
            }
            if constexpr (EZ) {
                rzm[f] = gz_m ? sd[2 * GROW3 + (1 + ly) * 2 + zpm] : bx[-1];
                rzp[f] = gz_p ? sd[2 * GROW3 + gcol3(IY) + (1 + ly) * 2 + zpp] : bx[1];
            } else {
                rzm[f] = bx[-1];
                rzp[f] = bx[1];
            }
        }
        yc[c] = rc[yraw<EV>() < NR ? yraw<EV>() : 0];
        double hc[NCH], hxm[NCH], hxp[NCH], hym[NCH], hyp[NCH], hzm[NCH], hzp[NCH];
        make_ch<EV, NCH, NR>(ctl, rc, hc);
        make_ch<EV, NCH, NR>(ctl, rxm, hxm);
        make_ch<EV, NCH, NR>(ctl, rxp, hxp);
        make_ch<EV, NCH, NR>(ctl, rym, hym);
        make_ch<EV, NCH, NR>(ctl, ryp, hyp);
        make_ch<EV, NCH, NR>(ctl, rzm, hzm);
        make_ch<EV, NCH, NR>(ctl, rzp, hzp);
#pragma unroll
        for (int h = 0; h < NCH; ++h)
            nb[c][h] = Nb{hc[h], hxm[h], hxp[h], hym[h], hyp[h], hzm[h], hzp[h]};
    }
    Centre<EV, EP, NC, K> z;
    const double* ctr = pc + NR * NC * RAW3;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        z.fu[c] = FU ? ctr[c * CTR3 + co] : 0.0;
        if constexpr (EP == EP_RHSN) z.y[c] = yc[c];  // u at the centre
        if constexpr (EP == EP_LEJA || EP == EP_ARN) {
            z.y[c] = yc[c];
#pragma unroll
            for (int q = 0; q < K; ++q)
                z.p[q][c] = (EP == EP_ARN && q == a.nwin - 1)
                                ? yc[c] : ctr[((FU + q) * NC + c) * CTR3 + co];
        }
        if constexpr (EP == EP_REM && K > 0) z.p[0][c] = ctr[(FU * NC + c) * CTR3 + co];
    }
    double val[NC];
    evaluate<P, EV, NCH>(a, ctl, nb, z.fu, val, z.jbad);
    epilogue<EV, EP, NC, K>(a, ctl, off, val, z, acc, xs);
}


template <class P, int EV, int EP, int K, int S, int RP>
__global__ void __launch_bounds__((nt3_of<EV, EP, P::NC, K>()), EK_LB3)
k_tma3d(const KArgs a, const __grid_constant__ TmaMaps maps) {
    static_assert(S >= 4, "plane ring needs i-1, i, i+1 and one in flight");
    constexpr int NC = P::NC, NQ = nq_of<EV, EP>();
    constexpr int NR = nraw<EV>();
    constexpr int SD = stage3_doubles<EV, EP, NC, K>();
    constexpr int T3 = t3_of<EV, EP, NC, K>(), NW3 = T3 / 32, NT3 = nt3_of<EV, EP, NC, K>();
    constexpr int IY = iy3<EV, EP, NC, K>(), PPT = IY * I3X / T3;
    static_assert(PPT >= 1 && PPT * T3 == IY * I3X, "item points must split evenly");
    extern __shared__ __align__(1024) double smem[];
    __shared__ __align__(8) uint64_t full[S];
#if EK_PROD3
    __shared__ __align__(8) uint64_t empty[S];  // the NW3 compute warps released stage s
#else
    __shared__ int released[S];  // warps that released stage s, cumulative
#endif

    Ctl ctl;
    if (!load_ctl<EV, EP>(a, ctl)) return;
    const int lane = threadIdx.x & 31;
    const int n = (int)a.g.n, rows = (int)a.g.rows;
    const long nitems = (long)((n + I3X - 1) / I3X) * ((n + IY - 1) / IY) *
                        ((rows + SEG3 - 1) / SEG3);
    const long G = gridDim.x;

    // Issue the plane S sequence numbers after position `pos` of item t
    // (if any) into stage s.
    auto issue_ahead = [&](long t, Item3 it, int pos, int s) {
        pos += S;
        while (pos >= it.L + 2) {
            pos -= it.L + 2;
            t += G;
            if (t >= nitems) return;
            it = item3<IY>(t, n, rows);
        }
        issue_plane<EV, EP, NC, K>(a, maps, smem + s * SD, &full[s], it, pos, rows, ctr_mask(ctl));
    };

    if (threadIdx.x == 0) {
#pragma unroll
        for (int t = 0; t < NR + nctr_maps<EV, EP, K>(); ++t)
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&maps.m[t]) : "memory");
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
#if EK_PROD3
            mbar_init(&empty[s], NW3);
#else
            released[s] = 0;
#endif
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#if !EK_PROD3
        // fill the ring: sequence numbers 0 .. S-1
        if (blockIdx.x < nitems) {
            const Item3 it0 = item3<IY>(blockIdx.x, n, rows);
            for (int s = 0; s < S; ++s) issue_ahead(blockIdx.x, it0, s - S, s);
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

#if EK_PROD3
    // Producer warp (the last one): issues every plane of this block's items
    // in sequence order, each into its ring stage as soon as the NW3 compute
    // warps have released the stage's previous plane. The compute warps only
    // wait for the copies they consume and arrive on empty[] when done.
    if ((int)(threadIdx.x >> 5) == NW3) {
        if (lane == 0) {
            long q = 0;
            for (long t = blockIdx.x; t < nitems; t += G) {
                const Item3 it = item3<IY>(t, n, rows);
                for (int pos = 0; pos < it.L + 2; ++pos, ++q) {
                    const int s = (int)(q % S);
                    if (q >= S) mbar_wait(&empty[s], (uint32_t)(((q / S) - 1) & 1));
                    issue_plane<EV, EP, NC, K>(a, maps, smem + s * SD, &full[s], it, pos, rows,
                                               ctr_mask(ctl));
                }
            }
        }
        __syncwarp();
        reduce_and_finalize<EV, EP, NQ, NT3, RP>(a, acc, xsa);
        return;
    }
#endif

    const int zpm = (int)(wrap_idx(-1, n, a.g.bc) & 1), zpp = (int)(wrap_idx(n, n, a.g.bc) & 1);
#if EK_PROD3 && EK_TIGHT3
    // Tight plane loop (producer-warp build). Everything that depends only
    // on the thread is formed once: its points' (row, column) in the item,
    // their offsets inside a raw / centre slot. The ring position is a stage
    // index plus one phase bit per stage (every sequence number is waited
    // for exactly once by each warp, in order), so the loop carries no
    // division, and the item's edge class is decided outside the plane loop.
    constexpr bool CARRY = EK_CARRY3 && NR * NC == 1;
    int lyv[PPT], lxv[PPT], rov[PPT], cov[PPT];
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
        if constexpr (IY == NW3 && PPT == 2 && !EK_MAP3_FLAT) {
            lyv[r] = threadIdx.x >> 5;
            lxv[r] = lane + 32 * r;
        } else {
            const int idx = threadIdx.x + r * T3;
            lyv[r] = idx / I3X;
            lxv[r] = idx % I3X;
        }
        rov[r] = (1 + lyv[r]) * TBW3 + 2 + lxv[r];
        cov[r] = lyv[r] * I3X + lxv[r];
    }
    int sn = 0;         // stage of the next sequence number this warp waits for
    uint32_t ph = 0;    // bit s: parity of that wait on stage s
    auto wait_next = [&]() {
        const int s = sn;
        mbar_wait_ns<EK_WAIT3_NS>(&full[s], (ph >> s) & 1u);
        ph ^= 1u << s;
        sn = s + 1 == S ? 0 : s + 1;
        return s;
    };
    auto release_s = [&](int s) {
        // the stage's shared-memory reads of this warp have completed (their
        // values were consumed), so no fence is needed before the copy
        // engine may overwrite it
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
    };
    const long plane = (long)n * n;
    for (long t = blockIdx.x; t < nitems; t += G) {
        const Item3 it = item3<IY>(t, n, rows);
#ifdef EK_NOEDGE3  // timing experiment only: wrong results on boundary items
        const int edge = 0;
#else
        const int edge = ((it.j0 < 1 || it.j0 + IY >= n) ? 1 : 0) |
                         ((it.k0 < 1 || it.k0 + I3X >= n) ? 2 : 0);
#endif
        int sm = wait_next(), sc = wait_next();
        long off[PPT];
#pragma unroll
        for (int r = 0; r < PPT; ++r)
            off[r] = ((long)it.i0 * n + it.j0 + lyv[r]) * n + it.k0 + lxv[r];
        const double* pm = smem + sm * SD;
        const double* pc = smem + sc * SD;
        // CARRY: planes i-1 / i of each point live in registers; the stage of
        // plane i-1 is released before the plane loop and every stage one
        // plane step earlier, so one more plane is in flight.
        double cv[CARRY ? PPT : 1][2];
        if constexpr (CARRY) {
#pragma unroll
            for (int r = 0; r < PPT; ++r) {
                cv[r][0] = pm[rov[r]];
                cv[r][1] = pc[rov[r]];
            }
            release_s(sm);
        }
        // one plane step of the item; E = -1: the edge class per point
        auto plane_step = [&](auto etag, const double* pp) {
            constexpr int E = decltype(etag)::value;
#pragma unroll
            for (int r = 0; r < PPT; ++r) {
                double* c = CARRY ? cv[CARRY ? r : 0] : nullptr;
                if constexpr (E == 0) {
                    tma3_point<P, EV, EP, K, IY, 0, decltype(xs), CARRY>(
                        a, ctl, pm, pc, pp, lyv[r], lxv[r], 0, 0, rov[r], cov[r], n, off[r], acc,
                        xs, zpm, zpp, c);
                } else {
                    const int jy = it.j0 + lyv[r], kx = it.k0 + lxv[r];
                    if (jy < n && kx < n) {
                        // y-edge items: only the rows j = 0 / n-1 need the selects
                        const int e = edge & ~((jy > 0 && jy < n - 1) ? 1 : 0);
                        if (e == 2)
                            tma3_point<P, EV, EP, K, IY, 2, decltype(xs), CARRY>(
                                a, ctl, pm, pc, pp, lyv[r], lxv[r], jy, kx, rov[r], cov[r], n,
                                off[r], acc, xs, zpm, zpp, c);
                        else if (e == 0)
                            tma3_point<P, EV, EP, K, IY, 0, decltype(xs), CARRY>(
                                a, ctl, pm, pc, pp, lyv[r], lxv[r], jy, kx, rov[r], cov[r], n,
                                off[r], acc, xs, zpm, zpp, c);
                        else
                            tma3_point<P, EV, EP, K, IY, 3, decltype(xs), CARRY>(
                                a, ctl, pm, pc, pp, lyv[r], lxv[r], jy, kx, rov[r], cov[r], n,
                                off[r], acc, xs, zpm, zpp, c);
                    } else if constexpr (CARRY) {  // keep the carried planes in step
                        c[0] = c[1];
                        c[1] = pp[rov[r]];
                    }
                }
                off[r] += plane;
            }
        };
        auto advance = [&](int sp, const double* pp) {
            if constexpr (CARRY) {
                release_s(sc);
            } else {
                release_s(sm);
                sm = sc;
                pm = pc;
            }
            sc = sp;
            pc = pp;
        };
        if (edge == 0) {
            for (int p = 1; p <= it.L; ++p) {
                const int sp = wait_next();
                const double* pp = smem + sp * SD;
                plane_step(std::integral_constant<int, 0>{}, pp);
                advance(sp, pp);
            }
        } else {
            for (int p = 1; p <= it.L; ++p) {
                const int sp = wait_next();
                const double* pp = smem + sp * SD;
                plane_step(std::integral_constant<int, -1>{}, pp);
                advance(sp, pp);
            }
        }
        if constexpr (!CARRY) release_s(sm);
        release_s(sc);
    }
#else
    auto wait_full = [&](int q) { mbar_wait(&full[q % S], (uint32_t)((q / S) & 1)); };
    // This warp is done with sequence number q (position pos of item t). The
    // last of the NW3 warps to release the stage refills it with the plane S
    // sequence numbers ahead, so no warp ever waits for another one.
    auto release = [&](int q, long t, const Item3& it, int pos) {
        __syncwarp();
        if (lane == 0) {
            // the stage's shared-memory reads of this warp have completed
            // (their values were consumed above), so no fence is needed
            // before the copy engine may overwrite it
            const int s = q % S;
#if EK_PROD3
            (void)t; (void)it; (void)pos;
            mbar_arrive(&empty[s]);
#else
            if ((atomicAdd(&released[s], 1) + 1) % NW3 == 0) issue_ahead(t, it, pos, s);
#endif
        }
    };

    // point r of this thread in the item plane: with one item row per warp
    // (IY == NW3) warp w owns row w, lanes columns lane + 32 r; otherwise
    // row-major over the block (IY * 64 / T3 points per thread).
    auto point_of = [&](int r, int& ly, int& lx) {
        if constexpr (IY == NW3 && PPT == 2 && !EK_MAP3_FLAT) {
            ly = threadIdx.x >> 5;
            lx = lane + 32 * r;
        } else {
            const int idx = threadIdx.x + r * T3;
            ly = idx / I3X;
            lx = idx % I3X;
        }
    };

    int q0 = 0;  // sequence number of position 0 of the current item
    for (long t = blockIdx.x; t < nitems; t += G) {
        const Item3 it = item3<IY>(t, n, rows);
#ifdef EK_NOEDGE3  // timing experiment only: wrong results on boundary items
        const int edge = 0;
#else
        const int edge = ((it.j0 < 1 || it.j0 + IY >= n) ? 1 : 0) |
                         ((it.k0 < 1 || it.k0 + I3X >= n) ? 2 : 0);
#endif
        wait_full(q0);
        wait_full(q0 + 1);
        int sm = q0 % S, sc = (q0 + 1) % S;
        // flat offsets of this thread's points in plane i0; + n^2 per plane
        long off[PPT];
#pragma unroll
        for (int r = 0; r < PPT; ++r) {
            int ly, lx;
            point_of(r, ly, lx);
            off[r] = ((long)it.i0 * n + it.j0 + ly) * n + it.k0 + lx;
        }
        const long plane = (long)n * n;
        for (int p = 1; p <= it.L; ++p) {
            wait_full(q0 + p + 1);
            const int sp = sc + 1 == S ? 0 : sc + 1;
            const double* pm = smem + sm * SD;
            const double* pc = smem + sc * SD;
            const double* pp = smem + sp * SD;
#pragma unroll
            for (int r = 0; r < PPT; ++r) {
                int ly, lx;
                point_of(r, ly, lx);
                const int jy = it.j0 + ly, kx = it.k0 + lx;
                const int ro = (1 + ly) * TBW3 + 2 + lx, co = ly * I3X + lx;
                if (edge == 0)
                    tma3_point<P, EV, EP, K, IY, 0>(a, ctl, pm, pc, pp, ly, lx, jy, kx, ro,
                                                    co, n, off[r], acc, xs, zpm, zpp);
                else if (jy < n && kx < n) {
                    // y-edge items: only the rows j = 0 / n-1 need the selects
                    const int e = edge & ~((jy > 0 && jy < n - 1) ? 1 : 0);
                    if (e == 2)
                        tma3_point<P, EV, EP, K, IY, 2>(a, ctl, pm, pc, pp, ly, lx, jy, kx,
                                                        ro, co, n, off[r], acc, xs, zpm, zpp);
                    else if (e == 0)
                        tma3_point<P, EV, EP, K, IY, 0>(a, ctl, pm, pc, pp, ly, lx, jy, kx,
                                                        ro, co, n, off[r], acc, xs, zpm, zpp);
                    else
                        tma3_point<P, EV, EP, K, IY, 3>(a, ctl, pm, pc, pp, ly, lx, jy, kx,
                                                        ro, co, n, off[r], acc, xs, zpm, zpp);
                }
                off[r] += plane;
            }
            release(q0 + p - 1, t, it, p - 1);
            sm = sc;
            sc = sp;
        }
        release(q0 + it.L, t, it, it.L);
        release(q0 + it.L + 1, t, it, it.L + 1);
        q0 += it.L + 2;
    }
#endif
    reduce_and_finalize<EV, EP, NQ, NT3, RP>(a, acc, xsa);
}

}  // namespace ek
