// ek_xsum.cuh — order-independent (reproducible) summation of fp64 terms.
//
// SURVEY.md §8(e) e4 asks for norms and dots that are bitwise identical for
// P = 1/2/4/8 slabs. Instead of tying every kernel's partial sums to a fixed
// global block grid, the "repro" mode of the reducing kernels accumulates
// each term in integers, so the result does not depend on which thread,
// block, kernel staging or rank saw which term:
//
//   * an fp64 term is a 53-bit integer times a power of two; seen as a bit
//     string on an absolute grid (bit 0 = the subnormal LSB 2^-1074) it is
//     cut into slices at fixed 32-bit bin boundaries;
//   * an accumulator (XAcc) keeps the integer sums of the slices of the FOUR
//     highest bins any of its terms reached (`top` and the three below), one
//     int64 per bin, with NO carry between bins until the very end; a term
//     reaching a higher bin moves the window up and drops the lowest bins
//     wholesale;
//   * merging two accumulators aligns them to the higher window and adds
//     bin by bin.
//
// Whatever the order, the final accumulator holds, for the four bins below
// the highest bit of the largest |term|, the exact sums of all terms' slices
// in those bins: every term's slice in a bin depends on the term alone, a
// partial accumulator never drops a bin the final window keeps (its window
// is never higher), and integer addition is associative. The value is then
// rounded to fp64 once (round to nearest even). What is lost lies below
// 2^-96 of the largest term per term: the result is the correctly rounded
// exact sum for any vector whose useful dynamic range fits 96 bits, and
// identical for every P, grid and staging in all cases.
//
// Capacity: slices are < 2^32, so one bin takes 2^30 terms of one sign
// before an int64 could overflow (the largest grid here is 2^27 points).
#pragma once

#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>
#include <string.h>

namespace ek {

struct XAcc {
    long long a[4];  // a[i]: sum of the slices in bin top - i
    int top;         // highest bin reached; XTOP_NONE = empty, XTOP_BAD = non-finite term
};
constexpr int XTOP_NONE = -8;
constexpr int XTOP_BAD = 1 << 20;
constexpr int XSLOTS = 5;  // 8-byte slots of a stored XAcc: a[0..3], top

__host__ __device__ __forceinline__ void xzero(XAcc& x) {
    x.a[0] = x.a[1] = x.a[2] = x.a[3] = 0;
    x.top = XTOP_NONE;
}

// Move the window up to bin `nt` (> x.top): the bins that fall below it are
// dropped whole (never carried).
__host__ __device__ __forceinline__ void xraise(XAcc& x, int nt) {
    const int d = nt - x.top;
    if (d == 1) {
        x.a[3] = x.a[2]; x.a[2] = x.a[1]; x.a[1] = x.a[0]; x.a[0] = 0;
    } else if (d == 2) {
        x.a[3] = x.a[1]; x.a[2] = x.a[0]; x.a[1] = 0; x.a[0] = 0;
    } else if (d == 3) {
        x.a[3] = x.a[0]; x.a[2] = 0; x.a[1] = 0; x.a[0] = 0;
    } else {
        x.a[0] = x.a[1] = x.a[2] = x.a[3] = 0;
    }
    x.top = nt;
}

// x += t (SIGNED = false: the caller guarantees t >= 0, e.g. squares).
template <bool SIGNED>
__host__ __device__ __forceinline__ void xadd(XAcc& x, double t) {
#ifdef __CUDA_ARCH__
    const long long u = __double_as_longlong(t);
#else
    long long u;
    memcpy(&u, &t, 8);
#endif
    int e = (int)((u >> 52) & 0x7ff);
    unsigned long long m = (unsigned long long)u & 0xfffffffffffffull;
    if (e == 0x7ff) {  // inf / nan: the sum is non-finite
        x.top = XTOP_BAD;
        return;
    }
    if (e) m |= 1ull << 52;
    else e = 1;  // subnormal (or zero)
    const int L = e - 1;               // absolute position of the mantissa LSB
    const int bt = (L + 52) >> 5;      // bin of the leading bit
    if (bt > x.top) xraise(x, bt);
    if (x.top == XTOP_BAD) return;
    const int sh = L - 32 * (x.top - 3);  // LSB position above the window bottom (< 76)
    unsigned long long lo, hi;
    if (sh >= 64) {
        lo = 0;
        hi = m << (sh - 64);
    } else if (sh > 0) {
        lo = m << sh;
        hi = m >> (64 - sh);
    } else if (sh > -64) {
        lo = m >> (-sh);  // the part of the term below the window is not kept
        hi = 0;
    } else {
        lo = 0;
        hi = 0;
    }
    const long long s3 = (long long)(lo & 0xffffffffull), s2 = (long long)(lo >> 32);
    const long long s1 = (long long)(hi & 0xffffffffull), s0 = (long long)(hi >> 32);
    if (SIGNED && u < 0) {
        x.a[3] -= s3; x.a[2] -= s2; x.a[1] -= s1; x.a[0] -= s0;
    } else {
        x.a[3] += s3; x.a[2] += s2; x.a[1] += s1; x.a[0] += s0;
    }
}

// x += y (accumulators).
__host__ __device__ __forceinline__ void xmerge(XAcc& x, const XAcc& y) {
    if (y.top == XTOP_NONE) return;
    if (x.top == XTOP_BAD || y.top == XTOP_BAD) {
        x.top = XTOP_BAD;
        return;
    }
    XAcc z = y;
    if (z.top > x.top) xraise(x, z.top);
    else if (x.top > z.top) xraise(z, x.top);
    x.a[0] += z.a[0]; x.a[1] += z.a[1]; x.a[2] += z.a[2]; x.a[3] += z.a[3];
}

// The accumulated value, rounded once to fp64 (round to nearest even).
__host__ __device__ inline double xvalue(const XAcc& x) {
    if (x.top == XTOP_NONE) return 0.0;
    if (x.top == XTOP_BAD) {
#ifdef __CUDA_ARCH__
        return __longlong_as_double(0x7ff8000000000000ll);
#else
        return NAN;
#endif
    }
    // carry-normalise upwards: bins 1..3 into [0, 2^32), bin 0 keeps the sign
    long long b3 = x.a[3], b2 = x.a[2], b1 = x.a[1], b0 = x.a[0];
    b2 += b3 >> 32; b3 &= 0xffffffffll;
    b1 += b2 >> 32; b2 &= 0xffffffffll;
    b0 += b1 >> 32; b1 &= 0xffffffffll;
    bool neg = b0 < 0;
    if (neg) {  // negate the 160-bit two's complement number (b0 : b1 : b2 : b3)
        b3 = (~b3 & 0xffffffffll) + 1;
        b2 = (~b2 & 0xffffffffll) + (b3 >> 32); b3 &= 0xffffffffll;
        b1 = (~b1 & 0xffffffffll) + (b2 >> 32); b2 &= 0xffffffffll;
        b0 = ~b0 + (b1 >> 32); b1 &= 0xffffffffll;
    }
    // limbs of 32 bits, most significant first: l[0] = b0 >> 32 ... l[4] = b3
    unsigned long long l[5] = {(unsigned long long)b0 >> 32, (unsigned long long)b0 & 0xffffffffull,
                               (unsigned long long)b1, (unsigned long long)b2,
                               (unsigned long long)b3};
    int h = 0;
    while (h < 5 && l[h] == 0) ++h;
    if (h == 5) return 0.0;
    // 96 bits from the highest nonzero limb, plus a sticky bit for the rest
    const unsigned long long w0 = l[h], w1 = h + 1 < 5 ? l[h + 1] : 0, w2 = h + 2 < 5 ? l[h + 2] : 0;
    bool sticky = false;
    for (int i = h + 3; i < 5; ++i) sticky = sticky || l[i] != 0;
    unsigned long long M = (w0 << 32) | w1;  // w0 != 0: at most 31 leading zeros
    int lz = 0;
    while (!((M << lz) >> 63)) ++lz;
    unsigned long long top64 = lz ? (M << lz) | (w2 >> (32 - lz)) : M;
    const unsigned long long rest = lz ? (w2 << lz) & 0xffffffffull : w2;
    sticky = sticky || rest != 0;
    unsigned long long mant = top64 >> 11;
    const unsigned long long rem = top64 & 0x7ffull;
    if (rem > 0x400ull || (rem == 0x400ull && (sticky || (mant & 1ull)))) ++mant;
    // Relative to the window bottom (absolute bit 32*(top-3)) limb h has
    // weight 2^(32*(4-h)), so M = (limb h : limb h+1) has its LSB at bit
    // 32*(3-h), top64 = M * 2^lz (plus bits of limb h+2) at 32*(3-h) - lz, and
    // mant = top64 >> 11 eleven bits above that; bit 0 is 2^-1074.
    const int ex = 32 * (x.top - 3) + 32 * (3 - h) - lz + 11 - 1074;
    double v = (double)(long long)mant;  // <= 2^53: exact
#ifdef __CUDA_ARCH__
    v = scalbn(v, ex);
#else
    v = ldexp(v, ex);
#endif
    return neg ? -v : v;
}

// 8-byte slot storage (part[] arrays, work buffer, peer windows)
__host__ __device__ __forceinline__ void xstore(long long* s, const XAcc& x) {
    s[0] = x.a[0]; s[1] = x.a[1]; s[2] = x.a[2]; s[3] = x.a[3]; s[4] = x.top;
}
__host__ __device__ __forceinline__ XAcc xload(const long long* s) {
    XAcc x;
    x.a[0] = s[0]; x.a[1] = s[1]; x.a[2] = s[2]; x.a[3] = s[3]; x.top = (int)s[4];
    return x;
}

// ------------------------------------------------------ block / grid level
#ifdef __CUDACC__
__device__ __forceinline__ XAcc xshfl_down(const XAcc& x, int o) {
    XAcc y;
#pragma unroll
    for (int i = 0; i < 4; ++i) y.a[i] = __shfl_down_sync(0xffffffffu, x.a[i], o);
    y.top = __shfl_down_sync(0xffffffffu, x.top, o);
    return y;
}

// Merge NX accumulators over the block (NW warps); totals land in thread 0.
template <int NX, int NW>
__device__ __forceinline__ void block_xsum(XAcc (&x)[NX]) {
    __shared__ long long shx[NX][NW][XSLOTS];
    const int t = threadIdx.x + blockDim.x * (threadIdx.y + blockDim.y * threadIdx.z);
    const int lane = t & 31, w = t >> 5;
#pragma unroll
    for (int q = 0; q < NX; ++q) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) xmerge(x[q], xshfl_down(x[q], o));
    }
    __syncthreads();  // protect shx from a previous use
    if (lane == 0) {
#pragma unroll
        for (int q = 0; q < NX; ++q) xstore(shx[q][w], x[q]);
    }
    __syncthreads();
    if (w == 0) {
#pragma unroll
        for (int q = 0; q < NX; ++q) {
            XAcc y;
            if (lane < NW) y = xload(shx[q][lane]);
            else xzero(y);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) xmerge(y, xshfl_down(y, o));
            x[q] = y;
        }
    }
}
#endif

}  // namespace ek
