// ek_stream.cuh — TMA-pipelined 2-D stencil kernel (sm_100a).
//
// Same value / epilogue algebra as ek_stencil.cuh, but every input tile is
// moved by the Tensor Memory Accelerator with 2-D tensor copies
// (`cp.async.bulk.tensor.2d`, completion counted in bytes on an mbarrier),
// S stages deep. One thread issues a handful of box copies per chunk; the
// data in flight lives in shared memory, not registers, so a block keeps
// up to S chunks (~80-110 KB) of HBM reads outstanding. Stages are released
// per warp (mbarrier arrivals), so the warps of a block never wait for each
// other, and interior chunks take a branch-free path with no ghost logic.
//
// Chunk = 32 columns x 8 rows (one row per warp). Per stage:
//   raw[f][c]  box of 10 x 36 doubles: rows r0-1..r0+8, columns j0-2..j0+33
//              of raw neighbourhood field f (u, y or k, u), component c.
//              The tensor map views a field as a (ncomp*rows) x cols
//              matrix, so component c starts at row c*rows.
//   ctr[g]     box of 8 x 32: f(u_n) / Leja accumulators at the centres.
// Ghost rows/columns at the domain boundary (row -1 / rows, column -1 /
// cols: wrap, reflect, or slab halo rows) are not in the boxes (TMA fills
// them with zeros or they belong to another component); the lanes that need
// one read it from global memory directly, so boundary conditions never
// touch the copy engine. Requires 16-byte row pitch (even row length).
#pragma once

#include <cuda.h>

#include "ek_stencil.cuh"

namespace ek {

#ifndef EK_EXP_TBW               // (EK_EXP_*: traffic experiments only, wrong results)
#define EK_EXP_TBW 36
#define EK_EXP_TBR 10
#endif
constexpr int TBW = EK_EXP_TBW;  // raw box width
constexpr int TBR = EK_EXP_TBR;  // raw box rows
constexpr int RAW_SLOT = 368;    // doubles per raw box slot (2944 B, 128-B multiple)
constexpr int CTR_SLOT = 256;    // 8 x 32 doubles
constexpr int MAX_MAPS = 11;     // 2 raw + f(u) + 8 accumulators

struct TmaMaps {
    CUtensorMap m[MAX_MAPS];     // [0, nraw) raw fields, then f(u), then p_q
    CUtensorMap h[2];            // 3-D slab: halo buffers of the raw fields
    CUtensorMap gr[2];           // 3-D: one ghost row (box TBW3 x 1) of a raw field
    CUtensorMap gc[2];           // 3-D: one ghost column pair (box 2 x (IY+2)) of a raw field
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(x), "r"(y), "r"(smem_u32(bar))
        : "memory");
}
// Same with an L2 eviction-priority hint (createpolicy), for streams read once.
__device__ __forceinline__ void tma_load_2d_hint(void* dst, const CUtensorMap* map, int x, int y,
                                                 uint64_t* bar, uint64_t policy) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
// Blocking wait on an mbarrier phase: try_wait without a suspend-time hint
// (the hardware parks the warp for a bounded window and wakes it when the
// phase completes). With an explicit hint ptxas emits a NANOSLEEP retry
// loop, which quantises the wake-up and measured as the top stall of the
// row-marching kernel.
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "LAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra LAB_WAIT;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
// The same wait with a suspend-time hint of NS nanoseconds: a warp whose
// stage has not landed sleeps in the barrier unit instead of spinning
// through issue slots the other warps need (NS = 0: plain try_wait loop).
template <int NS>
__device__ __forceinline__ void mbar_wait_ns(uint64_t* bar, uint32_t parity) {
    if constexpr (NS > 0) {
        asm volatile(
            "{\n\t.reg .pred P1;\n"
            "LAB_WAITH:\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1, %2;\n\t"
            "@!P1 bra LAB_WAITH;\n}" ::"r"(smem_u32(bar)),
            "r"(parity), "r"(NS)
            : "memory");
    } else {
        mbar_wait(bar, parity);
    }
}

// raw neighbourhood fields per value kind
template <int EV>
__host__ __device__ constexpr int nraw() {
    return (EV == EV_RHS || EV == EV_LIN) ? 1 : 2;
}
// index (within the raw fields) of y, whose centre value the Leja update needs
template <int EV>
__host__ __device__ constexpr int yraw() {
    return EV == EV_LIN ? 0 : 1;
}

template <int EV, int NCH, int NR>
__device__ __forceinline__ void make_ch(const Ctl& ctl, const double (&r)[NR], double (&ch)[NCH]) {
    if constexpr (EV == EV_RHS) {
        ch[0] = r[0];
    } else if constexpr (EV == EV_FD) {
        const double yv = ctl.has_div ? dv(r[1], ctl.ydiv) : r[1];
        ch[0] = r[0] + ctl.eps * yv;  // u + eps*v   (linalg.py:126)
        ch[1] = r[0];                 // u: f(u_n) is re-evaluated, not streamed
    } else if constexpr (EV == EV_LIN) {
        ch[0] = ctl.has_div ? dv(r[0], ctl.ydiv) : r[0];
    } else if constexpr (EV == EV_BURGJ) {
        ch[0] = r[0];
        ch[1] = ctl.has_div ? dv(r[1], ctl.ydiv) : r[1];
    } else if constexpr (EV == EV_REMFD) {
        ch[0] = r[0];
        ch[1] = r[1] + ctl.eps * (r[0] - r[1]);  // u + eps*(k - u)
        ch[2] = r[1];
    } else if constexpr (EV == EV_REMLIN) {
        ch[0] = r[0];
        ch[1] = r[0] - r[1];
    } else {
        ch[0] = r[0];
        ch[1] = r[1];
        ch[2] = r[0] - r[1];
    }
}

// centre maps: f(u_n) (if used) then K more: the Leja accumulators, or the
// Arnoldi window rows followed by the augmentation vectors
template <int EV, int EP, int K>
__host__ __device__ constexpr int nctr_maps() {
    return (needs_fu<EV>() ? 1 : 0) + ((EP == EP_LEJA || EP == EP_ARN || EP == EP_REM) ? K : 0);
}
template <int EV, int EP, int NC, int K>
__host__ __device__ constexpr int stage_doubles() {
    return nraw<EV>() * NC * RAW_SLOT + nctr_maps<EV, EP, K>() * NC * CTR_SLOT;
}

// Raw field base pointers (field 0 / 1) and halo buffers per value kind.
template <int EV>
__device__ __forceinline__ void raw_fields(const KArgs& a, const double* (&b)[2],
                                           const double* (&h)[2]) {
    if constexpr (EV == EV_RHS) {
        b[0] = a.u; h[0] = a.hu; b[1] = nullptr; h[1] = nullptr;
    } else if constexpr (EV == EV_LIN) {
        b[0] = a.y; h[0] = a.hy; b[1] = nullptr; h[1] = nullptr;
    } else if constexpr (EV == EV_FD || EV == EV_BURGJ) {
        b[0] = a.u; h[0] = a.hu; b[1] = a.y; h[1] = a.hy;
    } else {
        b[0] = a.k; h[0] = a.hk; b[1] = a.u; h[1] = a.hu;
    }
}

// Thread 0: expect the bytes of chunk (j0, r0) and issue its box copies.
template <int EV, int EP, int NC, int K>
__device__ __forceinline__ void issue_chunk(const TmaMaps& maps, double* buf, uint64_t* bar,
                                            int j0, int r0, int rows, uint32_t active) {
    constexpr int NR = nraw<EV>(), NCM = nctr_maps<EV, EP, K>();
    constexpr int FU = needs_fu<EV>() ? 1 : 0;
    uint32_t bytes = NR * NC * (TBW * TBR * 8);
#pragma unroll
    for (int g = 0; g < NCM; ++g)
        if (g < FU || ((active >> (g - FU)) & 1u)) bytes += NC * (32 * 8 * 8);
    mbar_arrive_expect(bar, bytes);
#pragma unroll
    for (int f = 0; f < NR; ++f)
#pragma unroll
        for (int c = 0; c < NC; ++c)
            tma_load_2d(buf + (f * NC + c) * RAW_SLOT, &maps.m[f], j0 - (TBW - 32) / 2,
                            c * rows + r0 - (TBR - 8) / 2, bar);
    double* ctr = buf + NR * NC * RAW_SLOT;
#pragma unroll
    for (int g = 0; g < NCM; ++g) {
        if (g < FU || ((active >> (g - FU)) & 1u)) {
#pragma unroll
            for (int c = 0; c < NC; ++c)
                tma_load_2d_hint(ctr + (g * NC + c) * CTR_SLOT, &maps.m[NR + g], j0, c * rows + r0,
                                 bar, policy_evict_first());
        }
    }
}

// One grid point (i, j) of chunk stage `raw`/`ctr`. EDGE = the chunk touches
// the domain boundary, so ghost rows/columns may come from global memory;
// interior chunks (the vast majority) read everything from the stage.
template <class P, int EV, int EP, int K, bool EDGE, class XS>
__device__ __forceinline__ void tma_point(const KArgs& a, const Ctl& ctl, const double* raw,
                                          const double* ctr, const double* const (&rb)[2],
                                          const double* const (&rh)[2], int i, int j, int wid,
                                          int lane, int rows, int cols, double* acc, XS xs) {
    constexpr int NC = P::NC, NCH = ev_nch(EV), NR = nraw<EV>();
    constexpr int FU = needs_fu<EV>() ? 1 : 0;
    const bool gx_m = EDGE && i == 0, gx_p = EDGE && i == rows - 1;  // ghost rows (warp-uniform)
    const bool gy_m = EDGE && j == 0, gy_p = EDGE && j == cols - 1;  // ghost columns
    Nb nb[NC][NCH];
    double yc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        double rc[NR], rxm[NR], rxp[NR], rym[NR], ryp[NR];
#pragma unroll
        for (int f = 0; f < NR; ++f) {
            const double* bx = raw + (f * NC + c) * RAW_SLOT + (1 + wid) * TBW + 2 + lane;
            rc[f] = bx[0];
            if constexpr (EDGE) {
                rxm[f] = gx_m ? __ldg(slab_row(a, rb[f], rh[f], c, -1, cols) + j) : bx[-TBW];
                rxp[f] = gx_p ? __ldg(slab_row(a, rb[f], rh[f], c, rows, cols) + j) : bx[TBW];
                const double* rowg = rb[f] + c * a.npts + (long)i * cols;
                rym[f] = gy_m ? __ldg(rowg + wrap_idx(-1, cols, a.g.bc)) : bx[-1];
                ryp[f] = gy_p ? __ldg(rowg + wrap_idx(cols, cols, a.g.bc)) : bx[1];
            } else {
                rxm[f] = bx[-TBW];
                rxp[f] = bx[TBW];
                rym[f] = bx[-1];
                ryp[f] = bx[1];
            }
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
    const int co = wid * 32 + lane;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        z.fu[c] = FU ? ctr[c * CTR_SLOT + co] : 0.0;
        if constexpr (EP == EP_RHSN) z.y[c] = yc[c];  // u at the centre
        if constexpr (EP == EP_LEJA || EP == EP_ARN) {
            z.y[c] = yc[c];
#pragma unroll
            for (int q = 0; q < K; ++q)
                z.p[q][c] = (EP == EP_ARN && q == a.nwin - 1)
                                ? yc[c] : ctr[((FU + q) * NC + c) * CTR_SLOT + co];
        }
        if constexpr (EP == EP_REM && K > 0) z.p[0][c] = ctr[(FU * NC + c) * CTR_SLOT + co];
    }
    double val[NC];
    evaluate<P, EV, NCH>(a, ctl, nb, z.fu, val, z.jbad);
    epilogue<EV, EP, NC, K>(a, ctl, (long)i * cols + j, val, z, acc, xs);
}

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred P1;\n\t"
        "mbarrier.test_wait.parity.shared::cta.b64 P1, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, P1;\n}"
        : "=r"(ok)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    return ok != 0;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

// Pipeline: full[s] counts the bytes of the chunk in stage s; empty[s] the
// 8 warps that released it. Thread 0 is the producer: before consuming
// chunk k it makes sure chunk k has been issued (blocking on the release of
// chunk k-S only if that is the oldest one still missing) and then issues as
// many further chunks as have free stages, without waiting. Warps never
// synchronise with each other, only with the copies they consume.
template <class P, int EV, int EP, int K, int S, int RP>
__global__ void __launch_bounds__(TPB) k_tma2d(const KArgs a, const __grid_constant__ TmaMaps maps) {
    constexpr int NC = P::NC, NQ = nq_of<EV, EP>();
    constexpr int NR = nraw<EV>();
    constexpr int SD = stage_doubles<EV, EP, NC, K>();
    extern __shared__ __align__(1024) double smem[];
    __shared__ __align__(8) uint64_t full[S];
    __shared__ __align__(8) uint64_t empty[S];

    Ctl ctl;
    if (!load_ctl<EV, EP>(a, ctl)) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int cols = (int)a.g.n, rows = (int)a.g.rows;
    const int tiles_c = (cols + 31) / 32;
    const int nchunks = tiles_c * ((rows + 7) / 8);
    const int G = gridDim.x;
#ifndef EK_EXP_COLMAJOR
    const int my = nchunks > (int)blockIdx.x ? (nchunks - 1 - (int)blockIdx.x) / G + 1 : 0;
    auto chunk_pos = [&](int k, int& j0, int& r0) {
        const int t = (int)blockIdx.x + k * G;
        j0 = (t % tiles_c) * 32;
        r0 = (t / tiles_c) * 8;
    };
#else  // experiment: block b takes a contiguous run of chunks down the strips
    const int tiles_r = (rows + 7) / 8;
    const int cb = (int)((long)nchunks * blockIdx.x / G), ce = (int)((long)nchunks * (blockIdx.x + 1) / G);
    const int my = ce - cb;
    auto chunk_pos = [&](int k, int& j0, int& r0) {
        const int t = cb + k;
        j0 = (t / tiles_r) * 32;
        r0 = (t % tiles_r) * 8;
    };
#endif
    const double* rb[2];
    const double* rh[2];
    raw_fields<EV>(a, rb, rh);

    if (threadIdx.x == 0) {
#pragma unroll
        for (int t = 0; t < NR + nctr_maps<EV, EP, K>(); ++t)
            asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&maps.m[t]) : "memory");
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], NWARP);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    double acc[NQ];
    XAcc xsa[ep_nx(EP)];  // repro mode (RP = 1): the sum channels (ek_xsum.cuh)
#pragma unroll
    for (int q = 0; q < ep_nx(EP); ++q) xzero(xsa[q]);
    const XsT<RP> xs{xsa};
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;

    int issued = 0;  // producer (thread 0) only
    for (int k = 0; k < my; ++k) {
        if (threadIdx.x == 0) {
            while (issued < my && issued < k + S) {
                const int s = issued % S;
                if (issued >= S) {
                    const uint32_t par = (uint32_t)((issued / S - 1) & 1);
                    if (issued <= k) mbar_wait(&empty[s], par);
                    else if (!mbar_test(&empty[s], par)) break;
                }
                int jj, rr;
                chunk_pos(issued, jj, rr);
                issue_chunk<EV, EP, NC, K>(maps, smem + s * SD, &full[s], jj, rr, rows,
                                           ctr_mask(ctl));
                ++issued;
            }
        }
        const int s = k % S;
        int j0, r0;
        chunk_pos(k, j0, r0);
        const int i = r0 + wid, j = j0 + lane;
        const double* raw = smem + s * SD;
        const double* ctr = raw + NR * NC * RAW_SLOT;
        mbar_wait(&full[s], (uint32_t)((k / S) & 1));
        if (r0 >= 1 && r0 + 8 < rows && j0 >= 1 && j0 + 32 < cols)
            tma_point<P, EV, EP, K, false>(a, ctl, raw, ctr, rb, rh, i, j, wid, lane, rows, cols, acc, xs);
        else if (i < rows && j < cols)
            tma_point<P, EV, EP, K, true>(a, ctl, raw, ctr, rb, rh, i, j, wid, lane, rows, cols, acc, xs);
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);  // this warp is done with stage s
    }
    reduce_and_finalize<EV, EP, NQ, TPB, RP>(a, acc, xsa);
}

}  // namespace ek
