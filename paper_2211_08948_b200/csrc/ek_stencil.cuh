// ek_stencil.cuh — fp64 2-D / 3-D stencil kernels of the phi-action path.
//
// One kernel template covers every fused pass that touches a stencil:
//
//   value  (EV_*)   : what is evaluated at each grid point
//     EV_RHS     f(u)                                   problems.py rhs closures
//     EV_FD      (f(u + eps*y) - fu) / eps              linalg.py:111-129
//     EV_LIN     f(y)              (linear problems: exact Jacobian = f)
//     EV_BURGJ   eta Lap y + d_x(u y) + d_y(u y)        Burgers analytic Jv
//     EV_REMFD   (f(k) - fn) - (f(u + eps*(k-u)) - fn)/eps   integrators.py:99-109
//     EV_REMLIN  (f(k) - fn) - f(k-u)
//     EV_REMBURG (f(k) - fn) - J(u)(k-u)
//   epilogue (EP_*)  : what is done with the value
//     EP_STORE   out = value
//     EP_LEJA    y' = value/gamma - shift*y ; p_i += d_i y' ; ||y'||^2 ;
//                device-side freeze test (leja.py:172-184)
//     EP_POWER   w = value ; ||w||^2 ; convergence test (spectrum.py:56-63)
//     EP_ARN     w = dt*value + tail@uflip ; window dots (kiops.py:182-187)
//     EP_REM     out = value ; non-finite flag (integrators.py:107-108)
//     EP_RHSN    out = f(u) ; ||u||^2 and nonzero / non-finite flags of u
//                (the RHS pass of a linearisation also yields linalg.py:123's
//                ||u||, one vector pass less)
//
// Geometry: a warp owns 32 consecutive columns of the contiguous axis (one
// lane per column, coalesced 256-B segments) and marches RPT consecutive
// rows of axis 0 (the slab axis) held in registers, so vertical neighbours
// are reused. Horizontal neighbours come from warp shuffles; lanes 0 and 1
// load the two halo columns of the warp. In 3-D the middle axis comes from
// the neighbouring warps through L1. Every input of a tile (neighbourhood
// rows, centre values, accumulators) is loaded before the first store, so a
// thread keeps ~(RPT+2)*NC*NCH + RPT*NC*(K+2) independent loads in flight.
// Blocks are persistent (grid = SMs x occupancy) and walk the tiles.
// Ghost rows follow the boundary condition: reflect (np.pad 'reflect',
// Neumann), wrap (periodic), or the halo buffers of a slab (multi-GPU).
//
// Arithmetic: every expression follows NumPy's evaluation order and the
// library is compiled with -fmad=false. Divisions by launch-uniform values
// (h**2, 2h, h, eps, gamma, ||w||) use the reciprocal r = RN(1/d) with one
// exact-residual correction, q = x r; q += (x - q d) r (two FMAs), which
// returns the correctly rounded IEEE quotient x/d (verified on the device
// against the division instruction, tests/test_gpu_kernels.py), at a third
// of the cost of a division call.
#pragma once

#include "ek_common.cuh"
#include "ek_decide.cuh"

namespace ek {

enum { EV_RHS = 0, EV_FD, EV_LIN, EV_BURGJ, EV_REMFD, EV_REMLIN, EV_REMBURG };
enum { EP_STORE = 0, EP_LEJA, EP_POWER, EP_ARN, EP_REM, EP_RHSN };

// Channels per point. EV_FD / EV_REMFD carry u itself as the last channel:
// f(u_n) is re-evaluated from the u neighbourhood the pass reads anyway
// (same code and order as the RHS pass that produced f_n, so the same bits)
// instead of streaming f_n from HBM — one vector less per pass.
__host__ __device__ constexpr int ev_nch(int ev) {
    return ev == EV_FD ? 2 : ev == EV_BURGJ ? 2 : ev == EV_REMFD ? 3 : ev == EV_REMLIN ? 2
         : ev == EV_REMBURG ? 3 : 1;
}
__host__ __device__ constexpr int ep_nq(int ep) {
    return ep == EP_LEJA ? 2 : ep == EP_POWER ? 2 : ep == EP_ARN ? 5 : ep == EP_REM ? 1
         : ep == EP_RHSN ? 3 : 0;
}
// accumulators of a pass; the FD remainder also counts non-finite FD
// Jacobian actions (the reference raises 'non-finite Jacobian action' from
// fd_jacobian_apply before the remainder check, linalg.py:127-128)
// Sum channels (the first ones of the epilogue's reduction) that repro mode
// accumulates in integers (ek_xsum.cuh): ||y||^2 of the Leja / power / RHS
// norm passes, the four window dots of the Arnoldi pass.
__host__ __device__ constexpr int ep_nx(int ep) { return ep == EP_ARN ? 4 : 1; }
__host__ __device__ constexpr bool ep_xsum(int ep) {
    return ep == EP_LEJA || ep == EP_POWER || ep == EP_RHSN || ep == EP_ARN;
}

template <int EV, int EP>
__host__ __device__ constexpr int nq_of() {
    return (EP == EP_REM && EV == EV_REMFD) ? 2 : (ep_nq(EP) > 0 ? ep_nq(EP) : 1);
}

struct Nb {
    double c, xm, xp, ym, yp, zm, zp;  // centre, axis0 -/+, axis1 -/+, axis2 -/+
};

// Problem constants of one launch.
struct PC {
    Dv h2, two_h, h;
    double prm[8];
};

// ------------------------------------------------------------------ physics

__device__ __forceinline__ double lap2(const Nb& s, const PC& g) {
    return dv((((s.xm + s.xp) + s.ym) + s.yp) - 4.0 * s.c, g.h2);  // problems.py:28-29
}
__device__ __forceinline__ double lap3(const Nb& s, const PC& g) {
    return dv(((((s.xm + s.xp) + s.ym) + s.yp) + s.zm) + s.zp - 6.0 * s.c, g.h2);
}
// one-sided difference following the sign of +v.grad u (forward for v >= 0).
// The operands are selected first and ONE quotient is formed: the same
// subtraction and division as `v >= 0 ? (xp - c) / h : (c - xm) / h`, but
// the compiler cannot predicate both divisions (12 fp64 issues per 3-D point).
__device__ __forceinline__ double upw(double m, double c, double p, double v, const PC& g) {
    const bool fwd = v >= 0.0;
    return dv((fwd ? p : c) - (fwd ? c : m), g.h);
}
__device__ __forceinline__ double upw_x(const Nb& s, double v, const PC& g) {
    return upw(s.xm, s.c, s.xp, v, g);
}
__device__ __forceinline__ double upw_y(const Nb& s, double v, const PC& g) {
    return upw(s.ym, s.c, s.yp, v, g);
}
__device__ __forceinline__ double upw_z(const Nb& s, double v, const PC& g) {
    return upw(s.zm, s.c, s.zp, v, g);
}

// problems.py:69-83. prm: alpha, beta, gamma
struct PAdr {
    static constexpr int NC = 1, DIM = 2;
    static constexpr bool LINEAR = false;
    __device__ static void f(const Nb (&s)[1], double (&o)[1], const PC& g) {
        const Nb& q = s[0];
        const double lap = lap2(q, g);
        const double gx = dv(q.xp - q.xm, g.two_h);
        const double gy = dv(q.yp - q.ym, g.two_h);
        const double grad = gx + gy;
        const double c = q.c;
        o[0] = ((g.prm[0] * lap) + (g.prm[1] * grad)) + (((g.prm[2] * c) * (1.0 - c)) * (c - 0.5));
    }
};

// problems.py:86-97 (and the periodic BASELINE variant). prm: alpha
struct PAllenCahn {
    static constexpr int NC = 1, DIM = 2;
    static constexpr bool LINEAR = false;
    __device__ static void f(const Nb (&s)[1], double (&o)[1], const PC& g) {
        o[0] = ((g.prm[0] * lap2(s[0], g)) + s[0].c) - cube_cr(s[0].c);
    }
};

// problems.py:100-124. prm: alpha. STD selects form="standard" (u^2 v).
template <bool STD>
struct PBruss {
    static constexpr int NC = 2, DIM = 2;
    static constexpr bool LINEAR = false;
    __device__ static void f(const Nb (&s)[2], double (&o)[2], const PC& g) {
        const double u = s[0].c, v = s[1].c;
        const double uu_v = (u * u) * v;
        const double react = STD ? uu_v : u * (v * v);
        o[0] = (((g.prm[0] * lap2(s[0], g)) + react) - (4.0 * u)) + 1.0;
        o[1] = ((g.prm[0] * lap2(s[1], g)) - uu_v) + (3.0 * u);
    }
};

// problems.py:127-145. prm: alpha, a, a+b
struct PGrayScott {
    static constexpr int NC = 2, DIM = 2;
    static constexpr bool LINEAR = false;
    __device__ static void f(const Nb (&s)[2], double (&o)[2], const PC& g) {
        const double u = s[0].c, v = s[1].c;
        const double uvv = u * (v * v);
        o[0] = ((g.prm[0] * lap2(s[0], g)) - uvv) + (g.prm[1] * (1.0 - u));
        o[1] = ((g.prm[0] * lap2(s[1], g)) + uvv) - (g.prm[2] * v);
    }
};

// BASELINE config 1. prm: D, vx, vy. Linear: J = f.
struct PAdvDiff2 {
    static constexpr int NC = 1, DIM = 2;
    static constexpr bool LINEAR = true;
    __device__ static void f(const Nb (&s)[1], double (&o)[1], const PC& g) {
        const Nb& q = s[0];
        o[0] = ((g.prm[0] * lap2(q, g)) + (g.prm[1] * upw_x(q, g.prm[1], g)))
               + (g.prm[2] * upw_y(q, g.prm[2], g));
    }
};

// BASELINE config 3. prm: eta.
struct PBurgers {
    static constexpr int NC = 1, DIM = 2;
    static constexpr bool LINEAR = false;
    __device__ static void f(const Nb (&s)[1], double (&o)[1], const PC& g) {
        const Nb& q = s[0];
        const double gx = dv((q.xp * q.xp) - (q.xm * q.xm), g.two_h);
        const double gy = dv((q.yp * q.yp) - (q.ym * q.ym), g.two_h);
        o[0] = ((g.prm[0] * lap2(q, g)) + (0.5 * gx)) + (0.5 * gy);
    }
    // J(u) v = eta Lap v + d_x(u v) + d_y(u v)
    __device__ static double jac(const Nb& u, const Nb& v, const PC& g) {
        const double gx = dv((u.xp * v.xp) - (u.xm * v.xm), g.two_h);
        const double gy = dv((u.yp * v.yp) - (u.ym * v.ym), g.two_h);
        return ((g.prm[0] * lap2(v, g)) + gx) + gy;
    }
};

// BASELINE config 5. prm: D, vx, vy, vz. Linear.
// FWD: instantiation for velocities >= 0 on every axis (the launcher picks
// it from the parameters): the forward differences without the operand
// selects (12 FSEL per point), the same subtraction and quotient.
template <bool FWD>
struct PAdvDiff3T {
    static constexpr int NC = 1, DIM = 3;
    static constexpr bool LINEAR = true;
    __device__ static void f(const Nb (&s)[1], double (&o)[1], const PC& g) {
        const Nb& q = s[0];
        if constexpr (FWD) {
            o[0] = (((g.prm[0] * lap3(q, g)) + (g.prm[1] * dv(q.xp - q.c, g.h)))
                    + (g.prm[2] * dv(q.yp - q.c, g.h)))
                   + (g.prm[3] * dv(q.zp - q.c, g.h));
        } else {
            o[0] = (((g.prm[0] * lap3(q, g)) + (g.prm[1] * upw_x(q, g.prm[1], g)))
                    + (g.prm[2] * upw_y(q, g.prm[2], g)))
                   + (g.prm[3] * upw_z(q, g.prm[3], g));
        }
    }
};
using PAdvDiff3 = PAdvDiff3T<false>;

// ------------------------------------------------------------- launch args

struct KArgs {
    ek_grid g;
    PC pc;
    long npts;            // points per component (local)
    long n_aug;           // length of the tail (KIOPS p), 0 otherwise
    // raw fields, component-major
    const double* u;
    const double* y;
    const double* k;
    const double* fu;
    // slab halos: [2 sides][ncomp][row length]
    const double* hu;
    const double* hy;
    const double* hk;
    double* out;          // store target / next iterate
    double* p[8];         // Leja accumulators
    int nk;
    int mi;               // column of the coefficient table
    int m;                // iteration index
    int jj;               // Arnoldi: index of the vector being built
    const double* coef;   // Leja table: row 0 shift, rows 1..k d_i (32 wide)
    Dv gamma;
    double eps;           // host-provided FD increment (EP_STORE / EP_REM)
    double dt;            // Arnoldi: operator scale (A.scaled(dt))
    void* st;             // state block (type depends on the epilogue)
    double* work;         // block partials
    // Arnoldi
    const double* win[4]; // window rows V[lo..jj-1] (n+p long), oldest first
    int nwin;
    const double* aug[5]; // nonzero augmentation vectors (u_flip rows / nu)
    int aug_tail[5];      // tail index each of them multiplies
    int naug;
    double aug_scale;     // nu (power of two)
    double* H;
    int ldh;
    // slab mode over peer memory (ek_leja_run_peer): window map and pass
    // number; null off that mode
    const ek_peer* peer;
    long epoch;
    // Leja pair launches (ek_launch.cuh): run only if act_lo <= #active <=
    // act_hi and iteration m-1 is the last finalised one; 0 / 0 = always
    int act_lo, act_hi;
    // EP_REM secondary outputs (ek_remainder_combo): xo[q] = ((xa[q] * xin)
    // + (xr[q] * R)) * xf[q], or (xr[q] * R) * xf[q] without xin
    double* xo[3];
    const double* xin;
    double xa[3], xr[3], xf[3];
    int nxo;
    // EP_REM with the direction norm on the device (ek_remainder_combo_dev):
    // pre->val[1] = ||k - u_n||, pre->flag bit0 = k != u_n; *nu = ||u_n||
    const ek_scalar_state* pre;
    const double* nu;
    // reproducible sums (ek_set_repro, ek_xsum.cuh): the norm channel of the
    // reducing epilogues is accumulated in integers, independent of order
    int repro;
    // Leja iterations as nodes of a CUDA graph WHILE loop (ek_leja_run_graph):
    // m < 0 = take the iteration index from the state block (m = st->m + 1;
    // -1: this node runs the odd iterations, -2: the even ones), column
    // m - chunk_base of the coefficient table, stop before m_limit; the
    // finalising block sets the loop condition `cond`
    int chunk_base, m_limit, cond_on;
    cudaGraphConditionalHandle cond;
};

// ----------------------------------------------------------------- geometry

__device__ __forceinline__ long wrap_idx(long i, long n, int bc) {
    if (i >= 0 && i < n) return i;
    if (bc == EK_BC_PERIODIC) return i < 0 ? i + n : i - n;
    if (n == 1) return 0;
    return i < 0 ? 1 : n - 2;  // np.pad 'reflect': mirror without repeating the edge
}

// Offset of row (2-D) / plane (3-D) `i` of component c inside a field, or of
// its copy in the halo buffer; i in [-1, rows].
__device__ __forceinline__ const double* slab_row(const KArgs& a, const double* base,
                                                  const double* halo, int c, long i,
                                                  long rowlen) {
    const long rows = a.g.rows;
    if (i >= 0 && i < rows) return base + c * a.npts + i * rowlen;
    if (a.g.slab) return halo + ((i < 0 ? 0 : 1) * (long)a.g.ncomp + c) * rowlen;
    return base + c * a.npts + wrap_idx(i, rows, a.g.bc) * rowlen;
}

// Scalars a kernel reads from its state block before the sweep.
struct Ctl {
    double eps;
    Dv eps_d;
    Dv ydiv;              // power iteration: v = w / ||w||
    bool has_div;
    uint32_t active;
    double shift;
    double d[8];
    bool y_zero;          // FD closure shortcut: J 0 = 0 (integrators.py:89-90)
    bool pinit;           // Leja: accumulators already hold d_i[0] b
    uint64_t wpol;        // L2 policy of the streamed outputs (evict first)
    double d0[8];         // Leja, first iteration: d_i[0]
    double augc[5];       // Arnoldi: tail[aug_tail[t]] * nu (exact: nu = 2^-e)
    // peer mode: where this pass's boundary rows of y' go ([ncomp][rowlen]
    // halo slots in a window): row 0 -> up's row `rows` ghost, row rows-1 ->
    // down's row -1 ghost; at a reflect edge rows 1 / rows-2 -> own ghosts
    double* h_first;
    double* h_second;
    double* h_penult;
    double* h_last;
    long rowlen;
    bool repro;           // order-independent sum channel (ek_xsum.cuh)
};

// Halo slot [ncomp][rowlen] of (rank r, parity, side) in the peer windows.
__device__ __forceinline__ double* peer_halo(const ek_peer* P, int r, int parity, int side) {
    return (double*)((char*)P->win[r] + EK_PEER_HALO_OFFSET) +
           (long)((parity * 2 + side) * P->ncomp) * P->rowlen;
}

// Channel values of one grid point.
template <int EV, int NCH>
__device__ __forceinline__ void fetch(const Ctl& ctl, const double* pu, const double* py,
                                      const double* pk, long e, double (&ch)[NCH]) {
    if constexpr (EV == EV_RHS) {
        ch[0] = __ldg(pu + e);
    } else if constexpr (EV == EV_FD) {
        double yv = __ldg(py + e);
        if (ctl.has_div) yv = dv(yv, ctl.ydiv);
        const double uv = __ldg(pu + e);
        ch[0] = uv + ctl.eps * yv;  // u + eps*v   (linalg.py:126)
        ch[1] = uv;
    } else if constexpr (EV == EV_LIN) {
        double yv = __ldg(py + e);
        if (ctl.has_div) yv = dv(yv, ctl.ydiv);
        ch[0] = yv;
    } else if constexpr (EV == EV_BURGJ) {
        double yv = __ldg(py + e);
        if (ctl.has_div) yv = dv(yv, ctl.ydiv);
        ch[0] = __ldg(pu + e);
        ch[1] = yv;
    } else if constexpr (EV == EV_REMFD) {
        const double kv = __ldg(pk + e), uv = __ldg(pu + e);
        const double dk = kv - uv;               // dk = k - u_n (integrators.py:103)
        ch[0] = kv;
        ch[1] = uv + ctl.eps * dk;
        ch[2] = uv;
    } else if constexpr (EV == EV_REMLIN) {
        const double kv = __ldg(pk + e), uv = __ldg(pu + e);
        ch[0] = kv;
        ch[1] = kv - uv;
    } else {  // EV_REMBURG
        const double kv = __ldg(pk + e), uv = __ldg(pu + e);
        ch[0] = kv;
        ch[1] = uv;
        ch[2] = kv - uv;
    }
}

// Value at the centre from the channel neighbourhoods; fuc = f(u_n) there.
// RFU (EV_FD only): take f(u_n) from fuc — the stored RHS vector, the same
// bits — instead of evaluating it again from the u neighbourhood.
template <class P, int EV, int NCH, bool RFU = false>
__device__ __forceinline__ void evaluate(const KArgs& a, const Ctl& ctl,
                                         const Nb (&nb)[P::NC][NCH],
                                         const double (&fuc)[P::NC], double (&val)[P::NC],
                                         double& jbad) {
    constexpr int NC = P::NC;
    if constexpr (EV == EV_RHS || EV == EV_LIN) {
        Nb s[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) s[c] = nb[c][0];
        P::f(s, val, a.pc);
    } else if constexpr (EV == EV_FD) {
        Nb s[NC], su[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) { s[c] = nb[c][0]; su[c] = nb[c][1]; }
        double fw[NC], fu[NC];
        P::f(s, fw, a.pc);
        if constexpr (RFU) {
#pragma unroll
            for (int c = 0; c < NC; ++c) fu[c] = fuc[c];
        } else {
            P::f(su, fu, a.pc);  // f(u_n), bit-identical to the RHS pass
        }
#pragma unroll
        for (int c = 0; c < NC; ++c)
            val[c] = ctl.y_zero ? 0.0 : dv(fw[c] - fu[c], ctl.eps_d);  // linalg.py:126
    } else if constexpr (EV == EV_BURGJ) {
        if constexpr (NC == 1 && NCH == 2) val[0] = PBurgers::jac(nb[0][0], nb[0][1], a.pc);
    } else if constexpr (EV == EV_REMFD) {
        Nb s0[NC], s1[NC], s2[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) { s0[c] = nb[c][0]; s1[c] = nb[c][1]; s2[c] = nb[c][2]; }
        double fk[NC], fw[NC], fu[NC];
        P::f(s0, fk, a.pc);
        P::f(s1, fw, a.pc);
        P::f(s2, fu, a.pc);  // f(u_n)
        jbad = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const double jd = dv(fw[c] - fu[c], ctl.eps_d);  // J(u_n)(k - u_n), linalg.py:126
            jbad += isfinite(jd) ? 0.0 : 1.0;
            val[c] = (fk[c] - fu[c]) - jd;  // integrators.py:106
        }
    } else if constexpr (EV == EV_REMLIN) {
        Nb s0[NC], s1[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) { s0[c] = nb[c][0]; s1[c] = nb[c][1]; }
        double fk[NC], jd[NC];
        P::f(s0, fk, a.pc);
        P::f(s1, jd, a.pc);
#pragma unroll
        for (int c = 0; c < NC; ++c) val[c] = (fk[c] - fuc[c]) - jd[c];
    } else {  // EV_REMBURG
        if constexpr (NC == 1 && NCH == 3) {
            Nb s0[1] = {nb[0][0]}, s1[1] = {nb[0][1]};
            double fk[1], fu[1];
            P::f(s0, fk, a.pc);
            P::f(s1, fu, a.pc);  // f(u_n) from the u channel
            val[0] = (fk[0] - fu[0]) - PBurgers::jac(nb[0][1], nb[0][2], a.pc);
        }
    }
}

template <int EV>
__host__ __device__ constexpr bool needs_fu() {
    return EV == EV_REMLIN;
}

// Read the state scalars; false = the iteration has already terminated.
template <int EV, int EP>
__device__ __forceinline__ bool load_ctl(const KArgs& a, Ctl& ctl) {
    ctl.eps = a.eps;
    ctl.has_div = false;
    ctl.ydiv = Dv{1.0, 1.0};
    ctl.active = 0u;
    ctl.shift = 0.0;
    ctl.y_zero = false;
    ctl.pinit = true;
    ctl.repro = a.repro != 0;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(ctl.wpol));
    if constexpr (EP == EP_LEJA) {
        const ek_leja_state* st = (const ek_leja_state*)a.st;
        if (st->done) return false;
        int mi = a.mi;
        if (a.m < 0) {  // graph loop node: the next iteration, if it is this node's turn
            const int m = st->m + 1;
            if ((m & 1) != (a.m & 1) || m >= a.m_limit || m - a.chunk_base >= 32) return false;
            mi = m - a.chunk_base;
        }
        if (a.act_hi > 0) {
            const int na = __popc(st->active);
            if (na < a.act_lo || na > a.act_hi || st->m != a.m - 1) return false;
        }
        ctl.eps = st->eps;
        ctl.active = st->active;
        ctl.y_zero = (EV == EV_FD) && (st->ny == 0.0);
        ctl.shift = a.coef[mi];
        ctl.pinit = st->p_init != 0;  // 0 only before the first iteration (m = 1, chunk 0)
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            ctl.d[q] = q < a.nk ? a.coef[(1 + q) * 32 + mi] : 0.0;
            ctl.d0[q] = q < a.nk ? a.coef[(1 + q) * 32] : 0.0;
        }
    } else if constexpr (EP == EP_POWER) {
        const ek_power_state* st = (const ek_power_state*)a.st;
        if (st->done || st->status) return false;
        ctl.ydiv = mkdv(st->nw);  // v = w / ||w|| of the previous iterate
        ctl.has_div = true;
        ctl.eps = (SQRT_EPS * (1.0 + st->nu)) / st->nv;
    } else if constexpr (EP == EP_ARN) {
        const ek_arnoldi_state* st = (const ek_arnoldi_state*)a.st;
        if (st->happy || st->status) return false;
        ctl.eps = (SQRT_EPS * (1.0 + st->nu)) / st->nvn;
        ctl.y_zero = (EV == EV_FD) && (st->nvn == 0.0);
        const long n = (long)a.g.ncomp * a.npts;
#pragma unroll
        for (int t = 0; t < 5; ++t)
            ctl.augc[t] = t < a.naug ? a.win[a.nwin - 1][n + a.aug_tail[t]] * a.aug_scale : 0.0;
        // centre slots: window rows, then augmentation vectors; d[q] holds
        // the tail coefficient of augmentation slot q
        // (bits = slots fetched from memory; slot nwin-1 is V[j-1] = y itself,
        // whose centre value the streaming kernel already holds)
        ctl.active = ((1u << (a.nwin + a.naug)) - 1u) & ~(1u << (a.nwin - 1));
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int t = q - a.nwin;
            ctl.d[q] = (t >= 0 && t < a.naug)
                           ? a.win[a.nwin - 1][n + a.aug_tail[t]] * a.aug_scale : 0.0;
        }
    }
    if constexpr (EP == EP_REM) {
        ctl.active = a.xin ? 1u : 0u;  // centre slot 0 = xin
        if (a.pre) {
            // `if not np.any(dk)`: R = 0 (integrators.py:104-105)
            ctl.y_zero = (a.pre->flag & 1) == 0;
            // eps = sqrt(EPS) * (1 + ||u||) / ||dk||, Python's order (linalg.py:123)
            if (EV == EV_REMFD) ctl.eps = (SQRT_EPS * (1.0 + *a.nu)) / a.pre->val[1];
        }
    }
    ctl.h_first = ctl.h_second = ctl.h_penult = ctl.h_last = nullptr;
    ctl.rowlen = 0;
    if constexpr (EP == EP_LEJA) {
        if (a.peer) {
            const ek_peer* P = a.peer;
            const int par = (int)((a.epoch + 1) & 1);  // read by pass epoch + 1
            ctl.rowlen = P->rowlen;
            if (P->up >= 0) ctl.h_first = peer_halo(P, P->up, par, 1);
            else ctl.h_second = peer_halo(P, P->rank, par, 0);
            if (P->down >= 0) ctl.h_last = peer_halo(P, P->down, par, 0);
            else ctl.h_penult = peer_halo(P, P->rank, par, 1);
        }
    }
    ctl.eps_d = mkdv(ctl.eps);
    return true;
}

// Peer mode: copy y'(off) of component c into the halo slots it feeds.
__device__ __forceinline__ void peer_halo_store(const KArgs& a, const Ctl& ctl, long off, int c,
                                                double v) {
    const long rl = ctl.rowlen, lo2 = (a.g.rows - 2) * rl, co = c * rl;
    if (off < 2 * rl) {
        if (off < rl) {
            if (ctl.h_first) ctl.h_first[co + off] = v;
        } else if (ctl.h_second) {
            ctl.h_second[co + off - rl] = v;
        }
    }
    if (off >= lo2) {
        if (off >= lo2 + rl) {
            if (ctl.h_last) ctl.h_last[co + off - lo2 - rl] = v;
        } else if (ctl.h_penult) {
            ctl.h_penult[co + off - lo2] = v;
        }
    }
}

// Centre slots a streaming kernel has to fetch (bit q: accumulator /
// Arnoldi slot q); none of the Leja accumulators before they exist.
__device__ __forceinline__ uint32_t ctr_mask(const Ctl& ctl) {
    return ctl.pinit ? ctl.active : 0u;
}

// EP_ARN centre slot q: window row q (q < nwin), else augmentation q - nwin
__host__ __device__ __forceinline__ const double* arn_slot(const KArgs& a, int q) {
    return q < a.nwin ? a.win[q] : a.aug[q - a.nwin];
}

// Centre values loaded with the neighbourhood, before any store.
template <int EV, int EP, int NC, int K>
struct Centre {
    double fu[NC];
    double y[NC];
    double p[K > 0 ? K : 1][NC];
    double jbad;  // EV_REMFD: non-finite FD Jacobian actions at this point
};

template <int EV, int EP, int NC, int K>
__device__ __forceinline__ void load_centre(const KArgs& a, const Ctl& ctl, long off,
                                            Centre<EV, EP, NC, K>& z) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const long e = c * a.npts + off;
        if constexpr (needs_fu<EV>()) z.fu[c] = __ldg(a.fu + e);
        else z.fu[c] = 0.0;
        if constexpr (EP == EP_RHSN) z.y[c] = __ldg(a.u + e);
        if constexpr (EP == EP_LEJA) {
            z.y[c] = __ldg(a.y + e);
#pragma unroll
            for (int q = 0; q < K; ++q)
                z.p[q][c] = (ctl.pinit && ((ctl.active >> q) & 1u)) ? a.p[q][e] : 0.0;
        } else if constexpr (EP == EP_ARN) {
#pragma unroll
            for (int q = 0; q < K; ++q)
                z.p[q][c] = q < a.nwin + a.naug ? __ldg(arn_slot(a, q) + e) : 0.0;
        } else if constexpr (EP == EP_REM && K > 0) {
            z.p[0][c] = __ldg(a.xin + e);  // input of the secondary outputs
        }
    }
}

// Store of a streamed output (read again only by the next pass, long after
// it has left L2): evict-first, so the re-read halo rows stay resident.
__device__ __forceinline__ void st_stream(double* p, double v, uint64_t pol) {
    asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;" ::"l"(p), "d"(v), "l"(pol)
                 : "memory");
}

// The repro-mode accumulators of a thread, with the mode in the type: RP = 0
// the kernel instance never uses them (the default, fp64 partial sums: no
// branch and no registers), 1 always (the instance launched in repro mode),
// 2 decided at run time by ctl.repro (the register-staged fallback kernels).
template <int RP>
struct XsT {
    static constexpr int mode = RP;
    XAcc* p;
};
template <class XS>
__device__ __forceinline__ bool xs_on(const XS&, const Ctl& ctl) {
    if constexpr (XS::mode == 0) return false;
    else if constexpr (XS::mode == 1) return true;
    else return ctl.repro;
}

// Per-point epilogue; acc[] collects this thread's partial reductions.
template <int EV, int EP, int NC, int K, class XS>
__device__ __forceinline__ void epilogue(const KArgs& a, const Ctl& ctl, long off,
                                         const double (&val)[NC],
                                         const Centre<EV, EP, NC, K>& z, double* acc, XS xs) {
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const long e = c * a.npts + off;
        const double v = val[c];
        if constexpr (EP == EP_STORE) {
            st_stream(a.out + e, v, ctl.wpol);
        } else if constexpr (EP == EP_RHSN) {
            st_stream(a.out + e, v, ctl.wpol);
            const double uc = z.y[c];
            if (xs_on(xs, ctl)) xadd<false>(xs.p[0], uc * uc);
            else acc[0] += uc * uc;
            acc[1] += uc != 0.0 ? 1.0 : 0.0;
            acc[2] += isfinite(uc) ? 0.0 : 1.0;
        } else if constexpr (EP == EP_LEJA) {
            // y = J.apply(y)/gamma - (c/gamma + xi[m-1]) * y      leja.py:172
            const double yn = dv(v, a.gamma) - (ctl.shift * z.y[c]);
            st_stream(a.out + e, yn, ctl.wpol);
            if (ctl.rowlen) peer_halo_store(a, ctl, off, c, yn);
            if (xs_on(xs, ctl)) xadd<false>(xs.p[0], yn * yn);
            else acc[0] += yn * yn;
            if constexpr (EV == EV_FD) acc[1] += isfinite(v) ? 0.0 : 1.0;
#pragma unroll
            for (int q = 0; q < K; ++q) {
                if (ctl.pinit) {
                    if ((ctl.active >> q) & 1u)  // ps[i] + dds[i][m]*y  leja.py:179
                        st_stream(a.p[q] + e, z.p[q][c] + (ctl.d[q] * yn), ctl.wpol);
                } else if (q < a.nk) {
                    // first iteration with the m = 0 term folded in: ps[i] = dds[i][0]*b
                    // (leja.py:161), then ps[i] + dds[i][1]*y -- same two roundings
                    const double p0 = ctl.d0[q] * z.y[c];
                    st_stream(a.p[q] + e, ((ctl.active >> q) & 1u) ? p0 + (ctl.d[q] * yn) : p0,
                              ctl.wpol);
                }
            }
        } else if constexpr (EP == EP_POWER) {
            st_stream(a.out + e, v, ctl.wpol);
            if (xs_on(xs, ctl)) xadd<false>(xs.p[0], v * v);
            else acc[0] += v * v;
            if constexpr (EV == EV_FD) acc[1] += isfinite(v) ? 0.0 : 1.0;
        } else if constexpr (EP == EP_ARN) {
            // V[j,:n] = op.apply(V[j-1,:n]) + V[j-1,n:] @ u_flip    kiops.py:182
            // centre slots (z.p): window rows [0, nwin), augmentation [nwin, nwin+naug)
            double augv = 0.0;
#pragma unroll
            for (int q = 0; q < K; ++q)
                if (q >= a.nwin && q < a.nwin + a.naug) augv = augv + (ctl.d[q] * z.p[q][c]);
            const double w = (a.dt * v) + augv;
            st_stream(a.out + e, w, ctl.wpol);
#pragma unroll
            for (int q = 0; q < (K < 4 ? K : 4); ++q)
                if (q < a.nwin) {
                    if (xs_on(xs, ctl)) xadd<true>(xs.p[q], z.p[q][c] * w);
                    else acc[q] += z.p[q][c] * w;
                }
            if constexpr (EV == EV_FD) acc[4] += isfinite(v) ? 0.0 : 1.0;
        } else {  // EP_REM
            const double r = ctl.y_zero ? 0.0 : v;  // zero direction (device-side test)
            if (a.out) st_stream(a.out + e, r, ctl.wpol);
            if (a.nxo) {  // the stage algebra that consumes R, in registers
                const double xin = K > 0 ? z.p[0][c] : 0.0;  // staged with the pass
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    if (q < a.nxo) {
                        const double rv = a.xr[q] * r;
                        const double t = K > 0 ? (a.xa[q] * xin) + rv : rv;
                        st_stream(a.xo[q] + e, t * a.xf[q], ctl.wpol);
                    }
                }
            }
            acc[0] += isfinite(r) ? 0.0 : 1.0;
            if constexpr (EV == EV_REMFD) acc[1] += ctl.y_zero ? 0.0 : z.jbad;
        }
    }
}

// Last-block bookkeeping of one fused pass. `xt`: the order-independent
// total of the sum channel (repro mode; tot[0] already holds its value).
template <int EV, int EP>
__device__ void finalize(const KArgs& a, const double* tot, const XAcc* xt);

template <int EP>
__device__ __forceinline__ uint32_t* ticket_of(const KArgs& a) {
    if constexpr (EP == EP_LEJA) return &((ek_leja_state*)a.st)->ticket;
    else if constexpr (EP == EP_POWER) return &((ek_power_state*)a.st)->ticket;
    else if constexpr (EP == EP_ARN) return &((ek_arnoldi_state*)a.st)->ticket;
    else return &((ek_scalar_state*)a.st)->ticket;
}

template <int EV, int EP, int NQ, int NT = TPB, int RP = 2>
__device__ __forceinline__ void reduce_and_finalize(const KArgs& a, double (&acc)[NQ],
                                                    XAcc (&xs)[ep_nx(EP)]) {
    if constexpr (ep_nq(EP) > 0) {
        // peer mode: this block's halo stores must reach the peers before
        // the last block raises the pass flag (system-scope fence)
        double tot[NQ];
        constexpr int NX = ep_nx(EP);
        XAcc xt[NX];
        const bool repro = RP == 1 || (RP == 2 && ep_xsum(EP) && a.repro != 0);
        if (reduce_grid<NQ, NX, NT>(acc, xs, repro, a.work, ticket_of<EP>(a),
                                    a.peer != nullptr, tot, xt)) {
            if (flat_tid() == 0) finalize<EV, EP>(a, tot, xt);
        }
    }
}

// ------------------------------------------------------------ 2-D kernel
// Tile = 32 columns x (8 warps * RPT rows); 1-D blocks of 256 threads.

template <class P, int EV, int EP, int RPT, int K>
__global__ void __launch_bounds__(TPB) k_stencil2d(const KArgs a) {
    constexpr int NC = P::NC, NCH = ev_nch(EV), NQ = nq_of<EV, EP>();
    Ctl ctl;
    if (!load_ctl<EV, EP>(a, ctl)) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long cols = a.g.n, rows = a.g.rows;
    const long tiles_c = (cols + 31) / 32;
    const long tile_rows = 8L * RPT;
    const long ntiles = tiles_c * ((rows + tile_rows - 1) / tile_rows);
    double acc[NQ];
    XAcc xsa[ep_nx(EP)];  // repro mode: the sum channels, order-independent (ek_xsum.cuh)
#pragma unroll
    for (int q = 0; q < ep_nx(EP); ++q) xzero(xsa[q]);
    const XsT<2> xs{xsa};
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;

    for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const long j0 = (t % tiles_c) * 32;
        const long i0 = (t / tiles_c) * tile_rows + (long)wid * RPT;
        const long j = j0 + lane;
        const long jc = j < cols ? j : cols - 1;
        const int elane = (int)(cols - 1 - j0 < 31 ? cols - 1 - j0 : 31);
        // lane 0 holds the west halo column of the warp, lane 1 the east one
        const long hcol = lane == 0 ? wrap_idx(j0 - 1, cols, a.g.bc)
                                    : wrap_idx(j0 + elane + 1, cols, a.g.bc);
        double cv[RPT + 2][NC][NCH];
        double hv[RPT][NC][NCH];
        Centre<EV, EP, NC, K> zc[RPT];
#pragma unroll
        for (int r = 0; r < RPT + 2; ++r) {
            long i = i0 - 1 + r;
            if (i > rows) i = rows;  // beyond the ghost row: clamp (unused)
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const double* pu = slab_row(a, a.u, a.hu, c, i, cols);
                const double* py = slab_row(a, a.y, a.hy, c, i, cols);
                const double* pk = slab_row(a, a.k, a.hk, c, i, cols);
                fetch<EV, NCH>(ctl, pu, py, pk, jc, cv[r][c]);
                if (r >= 1 && r <= RPT) {
                    if (lane < 2) fetch<EV, NCH>(ctl, pu, py, pk, hcol, hv[r - 1][c]);
                    else {
#pragma unroll
                        for (int h = 0; h < NCH; ++h) hv[r - 1][c][h] = 0.0;
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            long i = i0 + r;
            if (i >= rows) i = rows - 1;
            load_centre<EV, EP, NC, K>(a, ctl, i * cols + jc, zc[r]);
        }
#pragma unroll
        for (int r = 1; r <= RPT; ++r) {
            const long i = i0 + r - 1;
            Nb nb[NC][NCH];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
#pragma unroll
                for (int h = 0; h < NCH; ++h) {
                    const double cc = cv[r][c][h];
                    double w = __shfl_up_sync(0xffffffffu, cc, 1);
                    double e = __shfl_down_sync(0xffffffffu, cc, 1);
                    const double hw = __shfl_sync(0xffffffffu, hv[r - 1][c][h], 0);
                    const double he = __shfl_sync(0xffffffffu, hv[r - 1][c][h], 1);
                    if (lane == 0) w = hw;
                    if (lane == elane) e = he;
                    nb[c][h].c = cc;
                    nb[c][h].xm = cv[r - 1][c][h];
                    nb[c][h].xp = cv[r + 1][c][h];
                    nb[c][h].ym = w;
                    nb[c][h].yp = e;
                    nb[c][h].zm = 0.0;
                    nb[c][h].zp = 0.0;
                }
            }
            if (i < rows && j < cols) {
                double val[NC];
                evaluate<P, EV, NCH>(a, ctl, nb, zc[r - 1].fu, val, zc[r - 1].jbad);
                epilogue<EV, EP, NC, K>(a, ctl, i * cols + j, val, zc[r - 1], acc, xs);
            }
        }
    }
    reduce_and_finalize<EV, EP, NQ>(a, acc, xsa);
}

// ------------------------------------------------------------ 3-D kernel
// Tile = 32 (k, contiguous) x 8 (j, one per warp) x RPT planes (i).

template <class P, int EV, int EP, int RPT, int K>
__global__ void __launch_bounds__(TPB) k_stencil3d(const KArgs a) {
    constexpr int NC = P::NC, NCH = ev_nch(EV), NQ = nq_of<EV, EP>();
    Ctl ctl;
    if (!load_ctl<EV, EP>(a, ctl)) return;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const long n = a.g.n, rows = a.g.rows, plane = n * n;
    const long tk = (n + 31) / 32, tj = (n + 7) / 8, ti = (rows + RPT - 1) / RPT;
    const long ntiles = tk * tj * ti;
    double acc[NQ];
    XAcc xsa[ep_nx(EP)];  // repro mode: the sum channels, order-independent (ek_xsum.cuh)
#pragma unroll
    for (int q = 0; q < ep_nx(EP); ++q) xzero(xsa[q]);
    const XsT<2> xs{xsa};
#pragma unroll
    for (int q = 0; q < NQ; ++q) acc[q] = 0.0;

    for (long t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const long k0 = (t % tk) * 32;
        const long jy = ((t / tk) % tj) * 8 + wid;
        const long i0 = (t / (tk * tj)) * RPT;
        const long kx = k0 + lane;
        const long kc = kx < n ? kx : n - 1;
        const long jc = jy < n ? jy : n - 1;
        const int elane = (int)(n - 1 - k0 < 31 ? n - 1 - k0 : 31);
        const long hcol = lane == 0 ? wrap_idx(k0 - 1, n, a.g.bc)
                                    : wrap_idx(k0 + elane + 1, n, a.g.bc);
        const long jm = wrap_idx(jc - 1, n, a.g.bc), jp = wrap_idx(jc + 1, n, a.g.bc);
        double cv[RPT + 2][NC][NCH];
        double cjm[RPT][NC][NCH], cjp[RPT][NC][NCH];
        double hv[RPT][NC][NCH];
        Centre<EV, EP, NC, K> zc[RPT];
#pragma unroll
        for (int r = 0; r < RPT + 2; ++r) {
            long i = i0 - 1 + r;
            if (i > rows) i = rows;
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                const double* pu = slab_row(a, a.u, a.hu, c, i, plane);
                const double* py = slab_row(a, a.y, a.hy, c, i, plane);
                const double* pk = slab_row(a, a.k, a.hk, c, i, plane);
                fetch<EV, NCH>(ctl, pu, py, pk, jc * n + kc, cv[r][c]);
                if (r >= 1 && r <= RPT) {
                    fetch<EV, NCH>(ctl, pu, py, pk, jm * n + kc, cjm[r - 1][c]);
                    fetch<EV, NCH>(ctl, pu, py, pk, jp * n + kc, cjp[r - 1][c]);
                    if (lane < 2) fetch<EV, NCH>(ctl, pu, py, pk, jc * n + hcol, hv[r - 1][c]);
                    else {
#pragma unroll
                        for (int h = 0; h < NCH; ++h) hv[r - 1][c][h] = 0.0;
                    }
                }
            }
        }
#pragma unroll
        for (int r = 0; r < RPT; ++r) {
            long i = i0 + r;
            if (i >= rows) i = rows - 1;
            load_centre<EV, EP, NC, K>(a, ctl, i * plane + jc * n + kc, zc[r]);
        }
#pragma unroll
        for (int r = 1; r <= RPT; ++r) {
            const long i = i0 + r - 1;
            Nb nb[NC][NCH];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
#pragma unroll
                for (int h = 0; h < NCH; ++h) {
                    const double cc = cv[r][c][h];
                    double w = __shfl_up_sync(0xffffffffu, cc, 1);
                    double e = __shfl_down_sync(0xffffffffu, cc, 1);
                    const double hw = __shfl_sync(0xffffffffu, hv[r - 1][c][h], 0);
                    const double he = __shfl_sync(0xffffffffu, hv[r - 1][c][h], 1);
                    if (lane == 0) w = hw;
                    if (lane == elane) e = he;
                    nb[c][h].c = cc;
                    nb[c][h].xm = cv[r - 1][c][h];
                    nb[c][h].xp = cv[r + 1][c][h];
                    nb[c][h].ym = cjm[r - 1][c][h];
                    nb[c][h].yp = cjp[r - 1][c][h];
                    nb[c][h].zm = w;
                    nb[c][h].zp = e;
                }
            }
            if (i < rows && kx < n && jy < n) {
                double val[NC];
                evaluate<P, EV, NCH>(a, ctl, nb, zc[r - 1].fu, val, zc[r - 1].jbad);
                epilogue<EV, EP, NC, K>(a, ctl, i * plane + jy * n + kx, val, zc[r - 1], acc, xs);
            }
        }
    }
    reduce_and_finalize<EV, EP, NQ>(a, acc, xsa);
}

// --------------------------------------------------------------- finalize

// Slab mode: leave a pass's local sums in part[] (EK_PART_*): the sum
// channel as one double, or in repro mode as the integer accumulator.
__device__ __forceinline__ void part_store(double* part, const KArgs& a, double ssq,
                                           const XAcc& xt, double count) {
    if (a.repro) xstore(reinterpret_cast<long long*>(part), xt);
    else part[0] = ssq;
    part[EK_PART_COUNT] = count;
    part[EK_PART_TAG] = a.repro ? 1.0 : 0.0;
}

template <int EV, int EP>
__device__ void finalize(const KArgs& a, const double* tot, const XAcc* xt) {
    if constexpr (EP == EP_RHSN) {
        ek_scalar_state* st = (ek_scalar_state*)a.st;
        if (a.repro) xstore((long long*)st->xs, xt[0]);
        st->repro = a.repro;
        st->val[0] = tot[0];
        st->val[1] = sqrt(tot[0]);
        st->flag |= (tot[1] > 0.0 ? 1 : 0) | (tot[2] > 0.0 ? 2 : 0);
        return;
    }
    if constexpr (EP == EP_LEJA) {
        ek_leja_state* st = (ek_leja_state*)a.st;
        st->p_init = 1;
        if (a.peer) {  // peer mode: partials into every window, then the flag
            const ek_peer* P = a.peer;
            const int par = (int)(a.epoch & 1);
            for (int r = 0; r < P->world; ++r) {
                double* red = (double*)((char*)P->win[r] + 64) +
                              (par * 8 + P->rank) * EK_PART_SLOTS;
                part_store(red, a, tot[0], xt[0], tot[1]);
            }
            __threadfence_system();
            for (int r = 0; r < P->world; ++r) {
                unsigned long long* f = (unsigned long long*)P->win[r] + P->rank;
                asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(f),
                             "l"((unsigned long long)(a.epoch + 1))
                             : "memory");
            }
            return;
        }
        if (st->defer) {  // slab mode: ek_leja_decide finishes with global sums
            part_store(st->part, a, tot[0], xt[0], tot[1]);
            return;
        }
        const int m = a.m < 0 ? st->m + 1 : a.m;
        const int mi = a.m < 0 ? m - a.chunk_base : a.mi;
        leja_decide(st, a.coef, mi, m, a.nk > 0 ? a.nk : st->k, tot[0], tot[1], EV == EV_FD);
        if (a.cond_on)  // another turn of the graph loop?
            cudaGraphSetConditional(a.cond, (!st->done && m + 1 < a.m_limit &&
                                             m + 1 - a.chunk_base < 32) ? 1u : 0u);
    } else if constexpr (EP == EP_POWER) {
        ek_power_state* st = (ek_power_state*)a.st;
        if (st->defer) {
            part_store(st->part, a, tot[0], xt[0], tot[1]);
            return;
        }
        power_decide(st, tot[0], tot[1], EV == EV_FD);
    } else if constexpr (EP == EP_ARN) {
        ek_arnoldi_state* st = (ek_arnoldi_state*)a.st;
        if (EV == EV_FD && st->nvn != 0.0) st->fd_evals += 1;
        if (st->defer) {  // slab mode: local sums; ek_arnoldi_slab_decide finishes
            // window dots (EK_ARN_PART_*): fp64 values, or in repro mode the
            // integer accumulators; then the non-finite count and the tag
            for (int q = 0; q < 4; ++q) {
                if (a.repro) xstore(reinterpret_cast<long long*>(st->part) + q * XSLOTS, xt[q]);
                else st->part[q * XSLOTS] = tot[q];
            }
            st->part[EK_ARN_PART_COUNT] = tot[4];
            st->part[EK_ARN_PART_TAG] = a.repro ? 1.0 : 0.0;
            const long n = a.g.ncomp * a.npts;
            const int p = (int)a.n_aug;
            const double* prev = a.win[a.nwin - 1];
            double* cur = a.out;
            for (int t = 0; t + 1 < p; ++t) cur[n + t] = prev[n + t + 1];
            if (p > 0) cur[n + p - 1] = 0.0;
            return;
        }
        if (EV == EV_FD && tot[4] > 0.0) {
            st->status = EK_ST_JV_NONFINITE;
            return;
        }
        // tail of V[j]: shift of the previous tail, last entry 0 (kiops.py:183-184)
        const long n = a.g.ncomp * a.npts;
        const int p = (int)a.n_aug;
        const double* prev = a.win[a.nwin - 1];
        double* cur = a.out;
        for (int t = 0; t + 1 < p; ++t) cur[n + t] = prev[n + t + 1];
        if (p > 0) cur[n + p - 1] = 0.0;
        const int jj = a.jj;
        const int lo = jj - a.nwin;
        for (int q = 0; q < a.nwin; ++q) {
            double tail = 0.0;
            for (int t = 0; t < p; ++t) tail += a.win[q][n + t] * cur[n + t];
            a.H[(long)(lo + q) * a.ldh + (jj - 1)] = tot[q] + tail;  // kiops.py:187
        }
        a.H[(long)jj * a.ldh + (jj - 1)] = 0.0;
    } else if constexpr (EP == EP_REM) {
        ek_scalar_state* st = (ek_scalar_state*)a.st;
        if (tot[0] > 0.0) {
            st->flag |= 2;
            st->status = EK_ST_REM_NONFINITE;
        }
        if constexpr (EV == EV_REMFD) {
            if (tot[1] > 0.0) {  // checked first by the host, as fd_jacobian_apply raises first
                st->flag |= 4;
                st->status = EK_ST_JV_NONFINITE;
            }
        }
    }
}

}  // namespace ek
