// ek_common.cuh — shared device helpers for libexpkit_sm100.so.
//
// Deterministic reductions: every reducing kernel writes ONE partial per
// block (slot b of `work`), then the last block to arrive (atomic ticket)
// sums the partials in a fixed order (thread t takes b = t, t+256, ...;
// then a fixed shuffle tree). The result is independent of block
// scheduling, so repeated runs are bit-identical.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <math.h>

#include "../../include/expkit_sm100.h"
#include "ek_xsum.cuh"

namespace ek {

constexpr int TPB = 256;               // threads per block, every kernel
constexpr int NWARP = TPB / 32;
constexpr double SQRT_EPS = 1.4901161193847656e-08;  // math.sqrt(2**-52), linalg.py:123

// ---------------------------------------------------------------- errors
void set_error(const char* fmt, ...);
int cuda_status(cudaError_t e, const char* where);
void count_launch();  // ek_launch_count(): kernels launched by this library
#define EK_LAUNCH_CHECK(where)                                                \
    do {                                                                      \
        ::ek::count_launch();                                                 \
        cudaError_t e_ = cudaGetLastError();                                  \
        if (e_ != cudaSuccess) return ::ek::cuda_status(e_, where);           \
    } while (0)

__device__ __forceinline__ int flat_tid() {
    return threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
}
__device__ __forceinline__ long flat_bid() {
    return blockIdx.x + (long)gridDim.x * (blockIdx.y + (long)gridDim.y * blockIdx.z);
}
__device__ __forceinline__ long nblocks() {
    return (long)gridDim.x * gridDim.y * gridDim.z;
}

// Sum NQ values over the block; the totals land in thread 0.
template <int NQ, int NW = NWARP>
__device__ __forceinline__ void block_sum(double (&v)[NQ]) {
    __shared__ double sh[NQ][NW];
    const int t = flat_tid(), lane = t & 31, w = t >> 5;
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v[q] += __shfl_down_sync(0xffffffffu, v[q], o);
    }
    __syncthreads();  // protect sh from a previous use
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) sh[q][w] = v[q];
    }
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            double x = lane < NW ? sh[q][lane] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
            v[q] = x;
        }
    }
}

// Publish this block's NQ partials to work[b*NQ + q] and return true in the
// last block to arrive (all threads of that block see true). The last block
// resets the ticket for the next launch.
template <int NQ>
__device__ __forceinline__ bool publish_and_arrive(const double (&v)[NQ], double* work,
                                                   uint32_t* ticket, bool sys = false) {
    __shared__ bool s_last;
    const int t = flat_tid();
    if (t == 0) {
        const long b = flat_bid();
#pragma unroll
        for (int q = 0; q < NQ; ++q) work[b * NQ + q] = v[q];
        if (sys) __threadfence_system();  // orders the block's peer stores too
        else __threadfence();
        const uint32_t got = atomicAdd(ticket, 1u);
        s_last = (got == (uint32_t)(nblocks() - 1));
        if (s_last) *ticket = 0u;
    }
    __syncthreads();
    return s_last;
}

// In the last block: totals of the NQ partial channels, fixed order.
// Result valid in thread 0.
template <int NQ, int NT = TPB>
__device__ __forceinline__ void gather_partials(const double* work, long nb, double (&tot)[NQ]) {
    const int t = flat_tid();
#pragma unroll
    for (int q = 0; q < NQ; ++q) tot[q] = 0.0;
    for (long b = t; b < nb; b += NT) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) tot[q] += __ldcg(work + b * NQ + q);
    }
    block_sum<NQ, NT / 32>(tot);
}

// Grid-wide reduction of NQ fp64 channels, of which the first NX are real
// sums: block partials -> ticket -> the last block totals them (tot[],
// valid in its thread 0; returns true in every thread of that block). In
// `repro` mode the first NX channels are taken from the integer
// accumulators xs[] instead (ek_xsum.cuh): their block partials follow the
// fp64 ones in `work` (nblocks * NQ doubles, then nblocks * NX * XSLOTS
// slots), the last block merges them (any order gives the same bits) and
// tot[q] = xvalue(xt[q]) for q < NX.
// The two repro-mode steps are out of line (called once per thread, after
// the kernel's main loop) and take copies of the accumulators, so the
// integer merge code does not raise the register count of the kernels.
template <int NX, int NT>
__device__ __noinline__ void xpublish(const XAcc* xs_in, long long* xwork) {
    XAcc xs[NX];
#pragma unroll
    for (int q = 0; q < NX; ++q) xs[q] = xs_in[q];
    block_xsum<NX, NT / 32>(xs);
    if (flat_tid() == 0) {
        const long b = flat_bid();
#pragma unroll
        for (int q = 0; q < NX; ++q) xstore(xwork + (b * NX + q) * XSLOTS, xs[q]);
    }
}
template <int NX, int NT>
__device__ __noinline__ void xgather(const long long* xwork, long nb, XAcc* xt_out, double* tot) {
    const int t = flat_tid();
    XAcc xt[NX];
#pragma unroll
    for (int q = 0; q < NX; ++q) xzero(xt[q]);
    for (long b = t; b < nb; b += NT) {
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            XAcc y;
            const long long* src = xwork + (b * NX + q) * XSLOTS;
#pragma unroll
            for (int i = 0; i < 4; ++i) y.a[i] = __ldcg(src + i);
            y.top = (int)__ldcg(src + 4);
            xmerge(xt[q], y);
        }
    }
    block_xsum<NX, NT / 32>(xt);
    if (t == 0) {
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            tot[q] = xvalue(xt[q]);
            xt_out[q] = xt[q];
        }
    }
}

template <int NQ, int NX, int NT = TPB>
__device__ __forceinline__ bool reduce_grid(double (&acc)[NQ], XAcc (&xs)[NX], bool repro,
                                            double* work, uint32_t* ticket, bool sys,
                                            double (&tot)[NQ], XAcc (&xt)[NX]) {
    block_sum<NQ, NT / 32>(acc);
    const long nb = nblocks();
    long long* xwork = reinterpret_cast<long long*>(work + nb * NQ);
    if (repro) {
        XAcc tmp[NX];
#pragma unroll
        for (int q = 0; q < NX; ++q) tmp[q] = xs[q];
        xpublish<NX, NT>(tmp, xwork);
    }
    if (!publish_and_arrive<NQ>(acc, work, ticket, sys)) return false;
    gather_partials<NQ, NT>(work, nb, tot);
    if (repro) {
        XAcc tmp[NX];
        double tv[NX];
        xgather<NX, NT>(xwork, nb, tmp, tv);
        if (flat_tid() == 0) {
#pragma unroll
            for (int q = 0; q < NX; ++q) {
                tot[q] = tv[q];
                xt[q] = tmp[q];
            }
        }
    }
    return true;
}

// Division by a launch-uniform divisor: reciprocal r = RN(1/d) plus one
// exact-residual correction, q = x r; q += (x - q d) r. Returns the
// correctly rounded IEEE quotient (checked against the division
// instruction on the device by tests/test_gpu_kernels.py).
struct Dv {
    double d, r;  // divisor and RN(1/d)
};
__host__ __device__ __forceinline__ Dv mkdv(double d) { return Dv{d, 1.0 / d}; }
__device__ __forceinline__ double dv(double x, const Dv& c) {
    const double q = __dmul_rn(x, c.r);
    const double e = fma(-q, c.d, x);
    return fma(e, c.r, q);
}

// x^3 with a double-double intermediate: the correctly rounded cube in all
// but vanishingly rare cases, which is what NumPy's pow(x, 3) returns
// (problems.py:94 `f**3`).
__device__ __forceinline__ double cube_cr(double x) {
    const double p = __dmul_rn(x, x);
    const double pe = fma(x, x, -p);        // exact: x*x = p + pe
    const double q = __dmul_rn(p, x);
    const double qe = fma(p, x, -q);        // exact: p*x = q + qe
    const double lo = fma(pe, x, qe);       // tiny correction
    return __dadd_rn(q, lo);
}

}  // namespace ek
