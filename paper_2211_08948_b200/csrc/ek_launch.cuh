// ek_launch.cuh — host-side stencil launchers shared by the per-problem
// translation units (stencil_inst.cu, compiled once per problem struct so
// the kernel instantiations build in parallel).
//
// Pick the kernel instance for (problem, value, epilogue), its staging
// (TMA row march / TMA chunks / register-staged) and size the persistent grid.
#pragma once

#include <cstring>
#include <type_traits>

#include <cudaTypedefs.h>

#include "ek_common.cuh"
#include "ek_stencil.cuh"
#include "ek_stream.cuh"
#include "ek_stream3.cuh"
#include "ek_march2.cuh"

namespace ek {

// Rows (2-D) / planes (3-D) marched per thread: keep the register footprint
// of the neighbourhood (RPT+2)*NC*NCH and the centre values moderate.
__host__ __device__ constexpr int rpt_for(int nc, int nch, int dim) {
    return dim == 3 ? 2 : (nc * nch >= 2 ? 2 : 4);
}

inline int sm_count() {
    static int n = 0;
    if (n == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n < 1)
            n = 148;
    }
    return n;
}

inline int64_t stencil_tiles(const ek_grid* g, int rpt) {
    if (g->dim == 3)
        return ((g->n + 31) / 32) * ((g->n + 7) / 8) * ((g->rows + rpt - 1) / rpt);
    return ((g->n + 31) / 32) * ((g->rows + 8 * rpt - 1) / (8 * rpt));
}

// Persistent grid: min(tiles, SMs x resident blocks of this kernel). The
// occupancy is cached per kernel instantiation by the caller.
template <typename Kern>
inline unsigned persistent_grid(Kern kern, int64_t tiles, int& occ_cache) {
    if (occ_cache == 0) {
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, TPB, 0) != cudaSuccess ||
            occ < 1)
            occ = 1;
        occ_cache = occ;
    }
    const int64_t cap = (int64_t)sm_count() * occ_cache;
    return (unsigned)(tiles < cap ? (tiles > 0 ? tiles : 1) : cap);
}

inline bool al16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

// The TMA-staged kernel needs 16-byte aligned row segments of every field.
inline bool tma_ok(const KArgs& a) {
    if ((a.g.dim != 2 && a.g.dim != 3) || (a.g.n & 1) || a.g.n < 2 || (a.npts & 1)) return false;
    if (a.g.rows < 1 || a.g.n * a.g.ncomp * a.g.rows >= (int64_t)1 << 31) return false;
    const void* ps[] = {a.u, a.y, a.k, a.fu, a.hu, a.hy, a.hk};
    for (const void* p : ps)
        if (p && !al16(p)) return false;
    for (int q = 0; q < 8; ++q)
        if (a.p[q] && !al16(a.p[q])) return false;
    return true;
}

// The row march copies 16-byte aligned row segments: even row length, every
// field (and slab halo buffer) 16-byte aligned, and components npts apart.
inline bool march_ok(const KArgs& a) {
    if (a.g.dim != 2 || !tma_ok(a)) return false;
    if (a.g.slab && ((a.hu && !al16(a.hu)) || (a.hy && !al16(a.hy)) || (a.hk && !al16(a.hk))))
        return false;
    return true;
}

// 2-D staging: 0 register-staged k_stencil2d, 1 TMA 32x8 chunks (k_tma2d),
// 2 TMA row march (k_march2d, default). 3-D: any nonzero mode = k_tma3d.
// Launch recorder (graph mode): when set, the launchers describe the kernel
// they would launch instead of launching it.
struct LaunchDesc {
    void* func;
    dim3 grid, block;
    size_t smem;
    KArgs args;
    TmaMaps maps;
    bool has_maps;
};
extern thread_local LaunchDesc* g_record;
template <typename Kern>
inline bool record_launch(Kern kern, unsigned grid, unsigned block, size_t smem, const KArgs& a,
                          const TmaMaps* maps) {
    if (!g_record) return false;
    LaunchDesc& d = *g_record;
    d.func = (void*)kern;
    d.grid = dim3(grid);
    d.block = dim3(block);
    d.smem = smem;
    d.args = a;
    d.has_maps = maps != nullptr;
    if (maps) d.maps = *maps;
    return true;
}

extern int g_tma_mode;
extern int g_march_mask;  // auto mode: passes (bit EP_*) staged by the row march

// TMA stage count: as deep as fits two resident blocks per SM.
template <int EV, int EP, int NC, int K>
constexpr int tma_stages() {
    constexpr int bytes = stage_doubles<EV, EP, NC, K>() * 8;
    return bytes * 4 <= 110 * 1024 ? 4 : (bytes * 3 <= 110 * 1024 ? 3 : 2);
}
// 2-D row ring: i-1, i, i+1 resident plus S-3 rows in flight, as deep as
// fits two resident blocks per SM (at most 12 stages).
template <int EV, int EP, int NC, int K>
constexpr int tma_stages2() {
    constexpr int bytes = stage2_doubles<EV, EP, NC, K>() * 8;
    // per-block budget: 220 KB of shared memory over the resident blocks
    constexpr int two = (220 * 1024 / march2_lb<EP, K>()) / bytes;
#ifdef EK_MARCH_S
    return EK_MARCH_S;
#else
    return two > 12 ? 12 : (two < 4 ? 4 : two);
#endif
}

// 3-D plane ring: i-1, i, i+1 resident plus S-3 planes in flight; two
// blocks per SM if 5 stages fit, else one (0: no TMA variant).
template <int EV, int EP, int NC, int K>
constexpr int tma_stages3() {
    constexpr int bytes = stage3_doubles<EV, EP, NC, K>() * 8;
    // per-block budget: 220 KB of shared memory over EK_LB3 resident blocks
    constexpr int two = (220 * 1024 / EK_LB3) / bytes, one = (220 * 1024) / bytes;
#ifdef EK_S3
    if (EK_S3 > 0 && EK_S3 * bytes <= 220 * 1024 / EK_LB3) return EK_S3;
#endif
    if (EK_LB3 == 1) return one >= 5 ? (one > 16 ? 16 : one) : 0;
    // 5 stages (i-1, i, i+1 resident, two planes in flight) measured best on
    // the B200 for k = 1..3 at 512^3 (1.04 / 1.45 / 1.77 ms vs 1.06 / 1.57 /
    // 1.97 ms with 6 and 1.43 / 1.71 / 1.89 ms with 4): a deeper ring leaves
    // less L1 for the boundary items' ghost loads and the spill slots.
    return two >= 5 ? 5 : (one >= 5 ? 5 : 0);
}

// ---- tensor maps (driver entry point through the runtime, cached)
inline PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

struct MapEntry {
    const void* p;
    int rank;
    int promo;
    int64_t d[3];
    uint32_t b[3];
    CUtensorMap map;
};

// (ptr, dims, box) -> encoded map of a dense row-major fp64 tensor; the Leja
// / Arnoldi loops reuse a handful of buffers, so the cache turns encoding
// into a lookup.
// L2 promotion: 256-B for boxes whose rows are 256-B aligned (centre
// fields); none for the neighbourhood boxes, whose rows start 16 B before a
// 256-B boundary and would otherwise pull three 256-B lines per row.
inline bool tensor_map_nd(CUtensorMap* out, const double* p, int rank, const int64_t* d,
                          const uint32_t* b, int promo = -1) {
    static MapEntry cache[96];
    static int next = 0;
    if (promo < 0) promo = (b[0] % 32 == 0) ? 1 : 0;
    for (auto& e : cache) {
        if (e.p != p || e.rank != rank || e.promo != promo) continue;
        bool same = true;
        for (int r = 0; r < rank; ++r) same = same && e.d[r] == d[r] && e.b[r] == b[r];
        if (same) {
            *out = e.map;
            return true;
        }
    }
    auto fn = encode_fn();
    if (!fn) return false;
    MapEntry& e = cache[next];
    next = (next + 1) % 96;
    cuuint64_t dims[3], strides[2];
    cuuint32_t box[3], es[3];
    cuuint64_t st = 8;
    for (int r = 0; r < rank; ++r) {
        dims[r] = (cuuint64_t)d[r];
        box[r] = b[r];
        es[r] = 1;
        if (r > 0) strides[r - 1] = st;
        st *= (cuuint64_t)d[r];
    }
    if (fn(&e.map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, (void*)p, dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
           promo == 1   ? CU_TENSOR_MAP_L2_PROMOTION_L2_256B
           : promo == 2 ? CU_TENSOR_MAP_L2_PROMOTION_L2_128B
                        : CU_TENSOR_MAP_L2_PROMOTION_NONE,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        e.p = nullptr;
        return false;
    }
    e.p = p;
    e.rank = rank;
    e.promo = promo;
    for (int r = 0; r < 3; ++r) {
        e.d[r] = r < rank ? d[r] : 0;
        e.b[r] = r < rank ? b[r] : 0;
    }
    *out = e.map;
    return true;
}
inline bool tensor_map(CUtensorMap* out, const double* p, int64_t cols, int64_t rows, uint32_t bw,
                       uint32_t bh, int promo = -1) {
    const int64_t d[2] = {cols, rows};
    const uint32_t b[2] = {bw, bh};
    return tensor_map_nd(out, p, 2, d, b, promo);
}
inline bool tensor_map3(CUtensorMap* out, const double* p, int64_t n, int64_t planes, uint32_t bw,
                        uint32_t bh) {
    const int64_t d[3] = {n, n, planes};
    const uint32_t b[3] = {bw, bh, 1};
    return tensor_map_nd(out, p, 3, d, b);
}

template <int EV, int EP, int NC, int K>
inline bool build_maps(const KArgs& a, TmaMaps& m) {
    memset(&m, 0, sizeof(m));
    const int64_t cols = a.g.n, rt = (int64_t)a.g.ncomp * a.g.rows;
    const bool d3 = a.g.dim == 3;
    // 2-D: (ncomp*rows) x n matrix; 3-D: (ncomp*rows) x n x n tensor
    constexpr int IY = iy3<EV, EP, NC, K>();
    const uint32_t rw = d3 ? TBW3 : TBW, rh = d3 ? IY + 2 : TBR;  // raw boxes
    const uint32_t cw = d3 ? I3X : 32, ch = d3 ? IY : 8;          // centre boxes
    auto mk = [&](CUtensorMap* out, const double* f, uint32_t bw, uint32_t bh) {
        return d3 ? tensor_map3(out, f, cols, rt, bw, bh)
                  : tensor_map(out, f, cols, rt, bw, bh);
    };
    const double* raw[2] = {nullptr, nullptr};
    const double* hal[2] = {nullptr, nullptr};
    if constexpr (EV == EV_RHS) { raw[0] = a.u; hal[0] = a.hu; }
    else if constexpr (EV == EV_LIN) { raw[0] = a.y; hal[0] = a.hy; }
    else if constexpr (EV == EV_FD || EV == EV_BURGJ) {
        raw[0] = a.u; raw[1] = a.y; hal[0] = a.hu; hal[1] = a.hy;
    } else { raw[0] = a.k; raw[1] = a.u; hal[0] = a.hk; hal[1] = a.hu; }
    int t = 0;
    for (int f = 0; f < nraw<EV>(); ++f) {
        if (!mk(&m.m[t++], raw[f], rw, rh)) return false;
        // 3-D ghost side slots (boundary items): one row, one column pair
        if (d3 && (!tensor_map3(&m.gr[f], raw[f], cols, rt, TBW3, 1) ||
                   !tensor_map3(&m.gc[f], raw[f], cols, rt, 2, IY + 2)))
            return false;
        if (d3 && a.g.slab &&
            (!hal[f] || !al16(hal[f]) ||
             !tensor_map3(&m.h[f], hal[f], cols, 2 * (int64_t)a.g.ncomp, rw, rh)))
            return false;
    }
    if constexpr (needs_fu<EV>())
        if (!mk(&m.m[t++], a.fu, cw, ch)) return false;
    if constexpr (EP == EP_LEJA)
        for (int q = 0; q < K && q < a.nk; ++q)
            if (!mk(&m.m[t++], a.p[q], cw, ch)) return false;
    if constexpr (EP == EP_REM)
        for (int q = 0; q < K; ++q)
            if (!mk(&m.m[t++], a.xin, cw, ch)) return false;
    if constexpr (EP == EP_ARN)
        for (int q = 0; q < K && q < a.nwin + a.naug; ++q) {
            const double* f = arn_slot(a, q);
            if (!al16(f) || !mk(&m.m[t++], f, cw, ch)) return false;
        }
    return true;
}

// RP = 1: the kernel instances that accumulate the sum channels in integers
// (repro mode, ek_xsum.cuh); RP = 0: the default instances (no trace of it).
template <class P, int EV, int EP, int K, int RP>
inline int launch_k_rp(const KArgs& a, cudaStream_t s);

template <class P, int EV, int EP, int K>
inline int launch_k(const KArgs& a, cudaStream_t s) {
    if constexpr (ep_xsum(EP))
        if (a.repro) return launch_k_rp<P, EV, EP, K, 1>(a, s);
    return launch_k_rp<P, EV, EP, K, 0>(a, s);
}

template <class P, int EV, int EP, int K, int RP>
inline int launch_k_rp(const KArgs& a, cudaStream_t s) {
    constexpr int RPT = rpt_for(P::NC, ev_nch(EV), P::DIM);
    static int occ = 0;  // one per template instantiation
    if constexpr (P::DIM == 2) {
        TmaMaps maps;
        // auto (3): the row march for every Leja pass — with its producer
        // warp it is the faster staging at every accumulator count on the
        // B200 (config 4: k = 1 0.265 vs 0.274 ms, k = 2 0.318 vs 0.342 ms,
        // k = 3 0.403 vs 0.499 ms for the 32 x 8 chunks); chunks for the
        // other passes. (Mode 4 keeps round 1's pairing for A/B runs: march
        // iff >= 3 accumulators are active, chunks iff <= 2, each launch of a
        // pair exiting at its first read of the state block unless it is
        // the one that runs.)
        const bool pair = g_tma_mode == 4 && EP == EP_LEJA && K >= 3 && march_ok(a);
        const bool march = g_tma_mode == 2 || pair ||
                           (g_tma_mode == 3 && ((g_march_mask >> EP) & 1));
        if (march && march_ok(a)) {
            constexpr int S = tma_stages2<EV, EP, P::NC, K>();
            constexpr int SMEM = S * stage2_doubles<EV, EP, P::NC, K>() * 8;
            static int tocc = 0;
            auto kern = k_march2d<P, EV, EP, K, S, RP>;
            if (tocc == 0) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
                // the ring is sized for two resident blocks: ask for the full
                // shared-memory carve-out explicitly (kernel nodes of a graph
                // do not get the direct launch's automatic choice)
                cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tocc, kern, NT2, SMEM) !=
                        cudaSuccess || tocc < 1)
                    tocc = 1;
            }
            // NS strips x NG row segments, one item per block; segments of >= 8
            // rows (a segment of r rows fetches r + 2)
            const int64_t ns = march2_strips(a.g.n), cap = (int64_t)sm_count() * tocc;
            int64_t ng = cap >= ns ? cap / ns : 1;
            if (ng > a.g.rows / 8) ng = a.g.rows / 8 > 0 ? a.g.rows / 8 : 1;
            const unsigned grid = (unsigned)(cap >= ns ? ns * ng : cap);
            KArgs am = a;
            if (pair) { am.act_lo = 3; am.act_hi = 8; }
            if (record_launch(kern, grid, NT2, SMEM, am, nullptr)) return EK_OK;
            kern<<<grid, NT2, SMEM, s>>>(am);
            EK_LAUNCH_CHECK("bulk-copy march stencil launch");
            if (!pair) return EK_OK;
        }
        if (g_tma_mode != 0 && tma_ok(a) && build_maps<EV, EP, P::NC, K>(a, maps)) {
            constexpr int S = tma_stages<EV, EP, P::NC, K>();
            constexpr int SMEM = S * stage_doubles<EV, EP, P::NC, K>() * 8;
            static int tocc = 0;
            auto kern = k_tma2d<P, EV, EP, K, S, RP>;
            if (tocc == 0) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
                // the ring is sized for two resident blocks: ask for the full
                // shared-memory carve-out explicitly (kernel nodes of a graph
                // do not get the direct launch's automatic choice)
                cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tocc, kern, TPB, SMEM) !=
                        cudaSuccess || tocc < 1)
                    tocc = 1;
            }
            const int64_t chunks = ((a.g.n + 31) / 32) * ((a.g.rows + 7) / 8);
            const int64_t cap = (int64_t)sm_count() * tocc;
            const unsigned grid = (unsigned)(chunks < cap ? chunks : cap);
            KArgs ac = a;
            if (pair) { ac.act_lo = 0; ac.act_hi = 2; }
            if (record_launch(kern, grid, TPB, SMEM, ac, &maps)) return EK_OK;
            kern<<<grid, TPB, SMEM, s>>>(ac, maps);
            EK_LAUNCH_CHECK("tma stencil launch");
            return EK_OK;
        }
    }
    if constexpr (P::DIM == 3) {
        TmaMaps maps;
        constexpr int S = tma_stages3<EV, EP, P::NC, K>();
        if constexpr (S >= 5) if (g_tma_mode != 0 && tma_ok(a) && build_maps<EV, EP, P::NC, K>(a, maps)) {
            constexpr int SMEM = S * stage3_doubles<EV, EP, P::NC, K>() * 8;
            constexpr int NT = nt3_of<EV, EP, P::NC, K>();  // threads per block
            static int tocc = 0;
            auto kern = k_tma3d<P, EV, EP, K, S, RP>;
            if (tocc == 0) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM);
                // the ring is sized for two resident blocks: ask for the full
                // shared-memory carve-out explicitly (kernel nodes of a graph
                // do not get the direct launch's automatic choice)
                cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&tocc, kern, NT, SMEM) !=
                        cudaSuccess || tocc < 1)
                    tocc = 1;
            }
            constexpr int IY = iy3<EV, EP, P::NC, K>();
            const int64_t items = ((a.g.n + I3X - 1) / I3X) * ((a.g.n + IY - 1) / IY) *
                                  ((a.g.rows + SEG3 - 1) / SEG3);
            const int64_t cap = (int64_t)sm_count() * tocc;
            const unsigned grid = (unsigned)(items < cap ? items : cap);
            if (record_launch(kern, grid, NT, SMEM, a, &maps)) return EK_OK;
            kern<<<grid, NT, SMEM, s>>>(a, maps);
            EK_LAUNCH_CHECK("tma3 stencil launch");
            return EK_OK;
        }
    }
    const int64_t tiles = stencil_tiles(&a.g, RPT);
    if constexpr (P::DIM == 3) {
        auto kern = k_stencil3d<P, EV, EP, RPT, K>;
        if (record_launch(kern, persistent_grid(kern, tiles, occ), TPB, 0, a, nullptr)) return EK_OK;
        kern<<<persistent_grid(kern, tiles, occ), TPB, 0, s>>>(a);
    } else {
        auto kern = k_stencil2d<P, EV, EP, RPT, K>;
        if (record_launch(kern, persistent_grid(kern, tiles, occ), TPB, 0, a, nullptr)) return EK_OK;
        kern<<<persistent_grid(kern, tiles, occ), TPB, 0, s>>>(a);
    }
    EK_LAUNCH_CHECK("stencil launch");
    return EK_OK;
}

template <class P, int EV, int EP>
inline int launch_p(const KArgs& a, cudaStream_t s) {
    if constexpr (EP == EP_LEJA) {
        switch (a.nk) {
            // deferred accumulation (ek_leja_run_seq): the iteration only
            // advances the recurrence, ek_leja_combine forms the sums
            case 0: return launch_k<P, EV, EP, 0>(a, s);
            case 1: return launch_k<P, EV, EP, 1>(a, s);
            case 2: return launch_k<P, EV, EP, 2>(a, s);
            case 3: return launch_k<P, EV, EP, 3>(a, s);
            default: return launch_k<P, EV, EP, 8>(a, s);
        }
    } else if constexpr (EP == EP_ARN) {
        // centre slots = window rows + nonzero augmentation vectors
        switch (a.nwin + a.naug) {
            case 1: return launch_k<P, EV, EP, 1>(a, s);
            case 2: return launch_k<P, EV, EP, 2>(a, s);
            case 3: return launch_k<P, EV, EP, 3>(a, s);
            default: return launch_k<P, EV, EP, 8>(a, s);
        }
    } else {
        if constexpr (EP == EP_REM)
            if (a.xin) return launch_k<P, EV, EP, 1>(a, s);  // centre slot: xin
        return launch_k<P, EV, EP, 0>(a, s);
    }
}

// Valid (problem, value) pairs; EV_LIN only for linear problems, EV_BURGJ /
// EV_REMBURG only for Burgers.
template <class P, int EP>
inline int launch_ev(int ev, const KArgs& a, cudaStream_t s) {
    switch (ev) {
        case EV_RHS:
            if constexpr (EP == EP_STORE || EP == EP_RHSN) return launch_p<P, EV_RHS, EP>(a, s);
            break;
        case EV_FD:
            if constexpr (EP != EP_REM) return launch_p<P, EV_FD, EP>(a, s);
            break;
        case EV_LIN:
            if constexpr (P::LINEAR && EP != EP_REM) return launch_p<P, EV_LIN, EP>(a, s);
            break;
        case EV_BURGJ:
            if constexpr (std::is_same<P, PBurgers>::value && EP != EP_REM)
                return launch_p<P, EV_BURGJ, EP>(a, s);
            break;
        case EV_REMFD:
            if constexpr (EP == EP_REM) return launch_p<P, EV_REMFD, EP>(a, s);
            break;
        case EV_REMLIN:
            if constexpr (P::LINEAR && EP == EP_REM) return launch_p<P, EV_REMLIN, EP>(a, s);
            break;
        case EV_REMBURG:
            if constexpr (std::is_same<P, PBurgers>::value && EP == EP_REM)
                return launch_p<P, EV_REMBURG, EP>(a, s);
            break;
    }
    set_error("unsupported stencil pass (problem %d, value %d, epilogue %d)", a.g.problem, ev, EP);
    return EK_ERR_UNSUPPORTED;
}

// One entry per problem struct (stencil_inst.cu): dispatch on the epilogue.
#define EK_PROBLEMS(X)                      \
    X(PAdr, adr)                            \
    X(PAllenCahn, allen_cahn)               \
    X(PBruss<false>, bruss_printed)         \
    X(PBruss<true>, bruss_standard)         \
    X(PGrayScott, gray_scott)               \
    X(PAdvDiff2, advdiff2d)                 \
    X(PBurgers, burgers2d)                  \
    X(PAdvDiff3, advdiff3d)
#define EK_DECL_LAUNCH(P, name) int launch_##name(int ep, int ev, const KArgs& a, cudaStream_t s);
EK_PROBLEMS(EK_DECL_LAUNCH)
#undef EK_DECL_LAUNCH

template <class P>
inline int launch_problem(int ep, int ev, const KArgs& a, cudaStream_t s) {
    switch (ep) {
        case EP_STORE: return launch_ev<P, EP_STORE>(ev, a, s);
        case EP_LEJA: return launch_ev<P, EP_LEJA>(ev, a, s);
        case EP_POWER: return launch_ev<P, EP_POWER>(ev, a, s);
        case EP_ARN: return launch_ev<P, EP_ARN>(ev, a, s);
        case EP_REM: return launch_ev<P, EP_REM>(ev, a, s);
        case EP_RHSN: return launch_ev<P, EP_RHSN>(ev, a, s);
    }
    set_error("unsupported epilogue %d", ep);
    return EK_ERR_UNSUPPORTED;
}

}  // namespace ek
