/*
 * expkit_sm100.h — C ABI of libexpkit_sm100.so, the B200 (sm_100a) engine for
 * the phi-action hot path of arXiv 2211.08948 (reference: /root/reference,
 * package `expkit`).
 *
 * Plain C: pointers, sizes, POD structs. No torch types. All `double*`
 * vector arguments are DEVICE pointers (fp64, contiguous) unless the name
 * ends in `_host`. Every entry point takes the CUDA stream it must run on
 * (`void* stream`, a cudaStream_t; NULL = legacy default stream) and returns
 * an int status (EK_OK = 0); `ek_last_error()` gives the text of the last
 * failure on the calling thread.
 *
 * Each function names the reference interface it replaces (file:line under
 * /root/reference/pkg/src/expkit/). INTEGRATION.md shows the ctypes binding a
 * reference maintainer would add.
 *
 * Numerics: compiled with -fmad=false (no FMA contraction) and IEEE division,
 * so elementwise arithmetic follows NumPy's operation order bit-for-bit
 * (SURVEY.md §8(a)). Reductions are deterministic: fixed block partials,
 * reduced in a fixed order by the last block to finish (run-to-run and
 * scheduling invariant).
 */
#ifndef EXPKIT_SM100_H
#define EXPKIT_SM100_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
#define EK_OK 0
#define EK_ERR_INVALID 1      /* bad argument (-> ValueError)                */
#define EK_ERR_CUDA 2         /* CUDA runtime failure                        */
#define EK_ERR_UNSUPPORTED 3  /* combination not implemented                 */
#define EK_ERR_NONFINITE 4    /* non-finite result (-> FloatingPointError)   */

/* device-side numerical status codes (ek_*_state.status) */
#define EK_ST_OK 0
#define EK_ST_JV_NONFINITE 1   /* non-finite FD Jacobian action: linalg.py:127-128 -> FloatingPointError */
#define EK_ST_NORM_NONFINITE 2 /* non-finite ||y||: leja.py:173-175 -> NonConvergence               */
#define EK_ST_REM_NONFINITE 3  /* non-finite remainder: integrators.py:107-108 -> FloatingPointError */
#define EK_ST_PEER_TIMEOUT 4   /* peer mode: a rank's pass flag never arrived (no hang: error)     */

/* ------------------------------------------------------------------ grids */
enum ek_problem {
    EK_P_ADR = 1,             /* problems.py:69-83                         */
    EK_P_ALLEN_CAHN = 2,      /* problems.py:86-97 (+ periodic variant)    */
    EK_P_BRUSS_PRINTED = 3,   /* problems.py:100-124, form="printed"       */
    EK_P_BRUSS_STANDARD = 4,  /* problems.py:100-124, form="standard"      */
    EK_P_GRAY_SCOTT = 5,      /* problems.py:127-145                       */
    EK_P_SEMILINEAR = 6,      /* problems.py:154-196 (1-D, nonlocal term)  */
    EK_P_ADVDIFF2D = 7,       /* BASELINE config 1 (not in the reference)  */
    EK_P_BURGERS2D = 8,       /* BASELINE config 3 (not in the reference)  */
    EK_P_ADVDIFF3D = 9        /* BASELINE config 5 (not in the reference)  */
};
enum ek_bc { EK_BC_NEUMANN = 0, EK_BC_PERIODIC = 1, EK_BC_DIRICHLET = 2 };
enum ek_jac { EK_JAC_FD = 0, EK_JAC_ANALYTIC = 1 };

/* Uniform grid of one problem, component-major vectors with flat index
 * i*n + j (2-D, i = x slowest, problems.py meshgrid indexing="ij") or
 * (i*n + j)*n + k (3-D). For slab decomposition (multi-GPU) the local vector
 * holds rows [row0, row0+rows) of axis 0 and the rows just outside come from
 * halo buffers; single-GPU: rows == n, row0 == 0, slab == 0. */
typedef struct ek_grid {
    int32_t problem;   /* enum ek_problem                                  */
    int32_t bc;        /* enum ek_bc                                       */
    int32_t dim;       /* 1, 2 or 3                                        */
    int32_t ncomp;     /* 1 or 2 components                                */
    int64_t n;         /* points per axis                                  */
    int64_t rows;      /* local extent of axis 0                           */
    int64_t row0;      /* global index of local row 0                      */
    int32_t slab;      /* 1: rows -1 and `rows` come from halo buffers     */
    int32_t pad_;
    double h;          /* grid spacing                                     */
    double h2;         /* h**2 exactly as Python evaluates it              */
    double two_h;      /* 2.0*h                                            */
    double prm[8];     /* problem parameters            */
} ek_grid;

/* Length of one state vector (ncomp * points, +1 for the semilinear time). */
int64_t ek_grid_len(const ek_grid* g);

/* ------------------------------------------------- reproducible sums */
/* norms (and with them every decision and every FD
 * increment) that are bitwise identical for P = 1/2/4/8 slabs. In repro
 * mode (ek_set_repro(1); slab decompositions switch it on) the sum channel
 * of every reducing pass on the Leja / power-iteration / integrator-norm
 * path is accumulated in integers, independent of the order of the terms
 * (csrc/ek_xsum.cuh): a local sum is EK_XSLOTS 8-byte integer slots (four
 * 32-bit-bin sums and the index of the highest bin), merged exactly across
 * blocks, kernels and ranks and rounded to fp64 once. Whole-grid runs in
 * repro mode give the same bits as any slab decomposition. Replaces the
 * reference's np.linalg.norm (leja.py:173, spectrum.py:58, linalg.py:122,
 * timestep.py:46-52), which has no decomposition to be invariant to. */
#define EK_XSLOTS 5
/* part[] of the control blocks (slab mode), red[][] of the peer windows:
 * slots 0..4 the sum channel (slot 0 an fp64 value, or in repro mode the
 * EK_XSLOTS integers), slot 5 the non-finite count, slot 6 the format tag
 * (1.0 = integers). */
#define EK_PART_SLOTS 8
#define EK_PART_COUNT 5
#define EK_PART_TAG 6
/* part[] of the Arnoldi control block: four channels of EK_XSLOTS slots (the
 * window dots of pass A; channel 0 alone for the sums of squares of passes B
 * and C and of the init pass), then the non-finite count and the tag. */
#define EK_ARN_PART_SLOTS 24
#define EK_ARN_PART_COUNT 20
#define EK_ARN_PART_TAG 21
/* Returns the previous setting; negative only queries. */
int ek_set_repro(int on);
/* The fp64 value of a merged accumulator: `slots` = [n][EK_XSLOTS] integer
 * slots (host memory) of n local sums. */
double ek_xsum_value(const int64_t* slots, int n);
/* Host-side accumulation of n fp64 terms (sq = 1: their squares) into
 * slots_out[EK_XSLOTS]: the restatement the tests check the kernels with. */
void ek_xsum_host(const double* x, int64_t n, int sq, int64_t* slots_out);

/* -------------------------------------------------------- device states */
/* Leja iteration control block, lives in device memory (leja.py:159-184).
 * The host initialises tol, nu, k (and zeroes the rest) before
 * ek_leja_begin_len. */
typedef struct ek_leja_state {
    double ny;          /* ||y_m|| of the last finalised iterate            */
    double eps;         /* FD increment for the next Jacobian action        */
    double nu;          /* ||u|| at the linearisation point                 */
    double tol;         /* absolute termination tolerance                   */
    int32_t m;          /* index of the last finalised iterate              */
    int32_t done;       /* 1: all accumulators frozen, or an error          */
    int32_t status;     /* EK_ST_*                                          */
    int32_t k;          /* number of accumulators (<= 8)                    */
    uint32_t active;    /* bit i: accumulator i still accumulating          */
    int32_t fd_evals;   /* FD Jacobian actions performed (RHS charges)      */
    uint32_t ticket;    /* internal: last-block counter (keep 0)            */
    int32_t iters;      /* iteration count at termination                   */
    int32_t freeze[8];  /* freeze_iters                                     */
    int32_t defer;      /* slab mode: kernels leave their local sums in
                           part[] and ek_leja_decide applies the decision
                           to the rank-ordered global sums                  */
    int32_t p_init;     /* host: -1 requests folding m = 0 into the first
                           iteration (see ek_leja_begin_len). Device: 1 when
                           p_i holds d_i[0] b, 0 while the first fused
                           iteration (m = 1) still has to write it       */
    double part[8];     /* EK_PART_SLOTS: local ||y||^2 and non-finite count
                           (layout: EK_PART_*)                               */
    int32_t lazy0;      /* host: 1 = if everything freezes at m = 0, do not
                           write p_i = d_i[0] b (the caller uses d_i[0]*b as
                           an expression, ek_lincomb mode 3)                 */
    int32_t pad_;
} ek_leja_state;

/* Scalar reduction slot (norms, dots, flags), device memory. */
typedef struct ek_scalar_state {
    double val[8];      /* reduced values                                   */
    int32_t flag;       /* bit0: any nonzero, bit1: any non-finite, bit2:
                           non-finite FD Jacobian action (FD remainder)    */
    uint32_t ticket;    /* internal (keep 0)                                */
    int32_t count;
    int32_t status;     /* EK_ST_*                                          */
    int64_t xs[5];      /* EK_XSLOTS; repro mode: the integer accumulator of
                           val[0] (a sum of squares), merged exactly across
                           ranks                                             */
    int32_t repro;      /* 1: xs is valid                                   */
    int32_t pad_;
} ek_scalar_state;

/* Power iteration control block (spectrum.py:43-63). Host initialises
 * lam = 0, nu, tol_pi, max_it. */
typedef struct ek_power_state {
    double lam;         /* last estimate                                    */
    double nw;          /* ||J v|| of the last iteration (next divisor)     */
    double nv;          /* ||v|| of the current iterate (FD increment)      */
    double nu;          /* ||u||                                            */
    double tol_pi;
    int32_t it;         /* iterations done                                  */
    int32_t max_it;
    int32_t done;
    int32_t converged;
    int32_t fd_evals;
    uint32_t ticket;    /* internal (keep 0)                                */
    int32_t status;     /* EK_ST_*                                          */
    int32_t defer;      /* slab mode, see ek_leja_state                     */
    double part[8];     /* EK_PART_SLOTS: local sums of the last pass        */
} ek_power_state;

/* KIOPS Arnoldi control block (kiops.py:168-194). Host initialises nu, tol. */
typedef struct ek_arnoldi_state {
    double nrm;         /* last ||w|| (and the current normaliser)          */
    double nvn;         /* ||V[j,:n]|| (FD increment of the next Jv)        */
    double nu;          /* ||u||                                            */
    double tol;         /* happy-breakdown threshold                        */
    double beta;        /* ||V[0]|| of the current substep                  */
    int32_t j;          /* current basis size                               */
    int32_t happy;      /* 1 = happy breakdown                              */
    int32_t status;     /* EK_ST_*                                          */
    int32_t fd_evals;   /* FD Jacobian actions performed                    */
    uint32_t ticket;    /* internal (keep 0)                                */
    int32_t defer;      /* slab mode: passes leave local sums in part[] and
                           ek_arnoldi_slab_decide applies the gathered ones  */
    double part[24];    /* EK_ARN_PART_SLOTS: local window dots / sums of
                           squares (slab mode)                               */
} ek_arnoldi_state;

/* ------------------------------------------------------------ utilities */
const char* ek_last_error(void);
int ek_version(void);
/* Number of kernels this library has launched (process-wide). */
long long ek_launch_count(void);
/* Select the stencil staging of 2-D grids: 3 (default) = auto (bulk-copy
 * row march k_march2d for every Leja pass, TMA 32 x 8 chunks k_tma2d for
 * the other passes), 4 = round 1's auto (march only while >= 3 Leja
 * accumulators are active), 2 = row march everywhere, 1 = TMA chunks
 * everywhere, 0 = register-staged; 3-D grids use the TMA plane march for
 * any nonzero mode. A negative mode only queries. Returns the previous
 * setting. All give bit-identical pointwise results (block partial sums of
 * norms / dots are grouped differently). */
int ek_set_tma(int mode);
/* Auto mode: the passes (bit 1 << EP, EP_STORE = 0, LEJA, POWER, ARN, REM,
 * RHSN) staged by the row march; default 1 << 1 (Leja). Negative: query. */
int ek_set_march(int mask);
/* Bytes of device workspace (block partials) any call on this grid needs. */
int64_t ek_workspace_bytes(const ek_grid* g);
/* Stream-ordered copies (kind: 1 = host->device, 2 = device->host; a copy
 * to pageable host memory returns after the stream reached it). */
int ek_copy(void* dst, const void* src, int64_t bytes, int kind, void* stream);
int ek_sync(void* stream);

/* ------------------------------------------------ stencils (problems.py) */
/* out = f(u). Replaces Problem.rhs closures, problems.py:76-80, 92-95,
 * 115-121, 136-142, 170-175 (+ BASELINE plugins). halo: NULL, or
 * {u_halo, y_halo, k_halo} for a slab. */
int ek_rhs(const ek_grid* g, const double* u, double* out,
           const double* const* halo, void* stream);
/* f(u) as ek_rhs, plus ||u||^2 -> st->val[0], ||u|| -> st->val[1], flag
 * bit0 any nonzero, bit1 any non-finite (the ||u|| of linalg.py:123 that
 * an FD linearisation needs, from the same pass). 2-D / 3-D grids. */
int ek_rhs_norm(const ek_grid* g, const double* u, double* out, ek_scalar_state* st,
                double* work, const double* const* halo, void* stream);

/* out = J(u) v.  jac = EK_JAC_FD: (f(u+eps v) - fu)/eps with the caller's
 * eps = (sqrt(eps_mach)*(1+||u||))/||v|| (linalg.py:111-129); when `st` is
 * given, st->flag bit1 reports a non-finite result (linalg.py:127-128).
 * jac = EK_JAC_ANALYTIC: the problem's exact Jacobian stencil
 * (problems.py:177-189 / BASELINE plugins). */
int ek_jv(const ek_grid* g, int jac, const double* u, const double* fu,
          const double* v, double eps, double* out, ek_scalar_state* st,
          double* work, const double* const* halo, void* stream);

/* Fused nonlinear remainder R(k) = (f(k) - f_n) - J(k-u), one HBM pass over
 * both stencils (integrators.py:99-109). FD: J(dk) = (f(u+eps dk)-f_n)/eps
 * with the caller's eps from ||k-u||. st->flag bit1: non-finite output. */
int ek_remainder(const ek_grid* g, int jac, const double* u, const double* fu,
                 const double* k, double eps, double* out, ek_scalar_state* st,
                 double* work, const double* const* halo, void* stream);
/* The remainder pass fused with the stage algebra that consumes R: besides
 * (or instead of, out = NULL) R it stores nx <= 3 vectors
 *   xo[q] = ((xa[q] * xin) + (xr[q] * R)) * xf[q]     (xin != NULL)
 *   xo[q] = (xr[q] * R) * xf[q]                       (xin == NULL)
 * in NumPy's rounding order, e.g. R(a)*dt or ((-2 R(a)) + R(b))*dt of
 * EPIRK5P1 (integrators.py:318-341), without writing R and re-reading it. */
int ek_remainder_combo(const ek_grid* g, int jac, const double* u, const double* fu,
                       const double* k, double eps, double* out, int nx, double* const* xo,
                       const double* xin, const double* xa, const double* xr,
                       const double* xf, ek_scalar_state* st, double* work,
                       const double* const* halo, void* stream);
/* ek_remainder_combo with the direction test on the device: pre is the
 * state of the pass that formed k (val[1] = ||k - u_n||, flag bit0 =
 * k != u_n), nu points at ||u_n|| (FD only). The FD increment
 * eps = (sqrt(EPS) * (1 + ||u_n||)) / ||k - u_n|| (linalg.py:123) is formed by
 * the kernel in Python's order; if k == u_n the outputs take R = 0
 * (integrators.py:104-105). No host round trip between the two passes. */
int ek_remainder_combo_dev(const ek_grid* g, int jac, const double* u, const double* fu,
                           const double* k, const ek_scalar_state* pre, const double* nu,
                           double* out, int nx, double* const* xo, const double* xin,
                           const double* xa, const double* xr, const double* xf,
                           ek_scalar_state* st, double* work, const double* const* halo,
                           void* stream);

/* ------------------------------------------------------- Leja (leja.py) */
/* Coefficient table coef_dev: (k+1) rows x 32 columns, row 0 the shifts
 * c/gamma + xi[m-1], row 1+i the divided differences d_i[m], column
 * m - chunk_base. */

/* m = 0 of leja_interpolate_vertical (leja.py:159-165): p_i = d_i[0]*b,
 * ||b||, freeze test, FD increment for m = 1. If the host set
 * st->p_init = -1 (fold request; not in slab mode), this pass only takes
 * the norm and the decisions: the first ek_leja_run iteration writes
 * p_i = d_i[0]*b + d_i[1]*y_1 in its own pass (same two roundings), and if
 * every accumulator froze at m = 0 a follow-up pass on the device writes
 * p_i = d_i[0]*b. */
int ek_leja_begin_len(int64_t len, const double* b, double* const* p, int k,
                      const double* coef_dev, ek_leja_state* st, double* work,
                      void* stream);

/* Iterations m in [m_begin, m_end) of the Newton-Leja recurrence
 * (leja.py:167-184), each ONE fused HBM pass: Jacobian stencil (FD or
 * analytic) + y' = Jy/gamma - shift*y + p_i += d_i[m] y' + deterministic
 * ||y'||^2 + device-side freeze test. y ping-pongs between ybuf[0]/ybuf[1];
 * iterate m-1 is read from `b` when m == 1. Launches early-exit once
 * st->done is set, so the host syncs only per chunk. */
int ek_leja_run(const ek_grid* g, int jac, const double* u, const double* fu,
                const double* b, double* const* ybuf, double* const* p, int k,
                const double* coef_dev, int chunk_base, int m_begin, int m_end,
                double gamma, ek_leja_state* st, double* work,
                const double* const* halo, void* stream);

/* The same iterations as ONE launch of a CUDA graph whose WHILE node loops
 * on the device (whole-grid path): from m_begin (1, or
 * the even first iteration of a later 32-point chunk) until the call is done,
 * m reaches m_limit, or the chunk's last column has been used. Every node
 * takes its iteration index from the state block and the finalising block
 * of an iteration sets the loop condition, so no launch ever finds the call
 * finished and the host does nothing per iteration. Graphs are cached per
 * kernel instance; a call rewrites the nodes' arguments. Results are those
 * of ek_leja_run bit for bit. */
int ek_leja_run_graph(const ek_grid* g, int jac, const double* u, const double* fu,
                      const double* b, double* const* ybuf, double* const* p, int k,
                      const double* coef_dev, int chunk_base, int m_begin, int m_limit,
                      double gamma, ek_leja_state* st, double* work, void* stream);

/* One whole-grid fused Leja call up to its first host check, in ONE
 * call (the single-GPU fast path of leja_interpolate_vertical,
 * leja.py:133-184): upload the first 32-point coefficient chunk from
 * `coef_host` ((k+1) x 32, as for ek_leja_run) into `coef_dev`, initialise
 * the state block (tol; ||u|| = nu, or *nu_dev when given; fold: the m = 0
 * accumulators are folded into the first iteration; lazy0 as in
 * ek_leja_state), run the begin pass, then iterations 1 .. m_end-1
 * (m_end < 0: as one graph launch, ek_leja_run_graph with m_limit = -m_end). */
int ek_leja_call(const ek_grid* g, int jac, const double* u, const double* fu,
                 const double* b, double* const* ybuf, double* const* p, int k,
                 const double* coef_host, double* coef_dev, double tol, double nu,
                 const double* nu_dev, int fold, int lazy0, int m_end, double gamma,
                 ek_leja_state* st, double* work, void* stream);

/* Deferred accumulation (whole-grid path, large grids). The reference adds
 * the term d_i[m] y_m to every live accumulator inside the iteration
 * (leja.py:179), which costs 2k vector transfers per iteration. Here the
 * iterations m_begin .. m_begin + count - 1 read y_{m-1} from yin[i], write
 * y_m to yout[i] (one buffer per iterate) and leave the accumulators alone;
 * the freeze decisions are taken over the state block's k as in
 * ek_leja_run. ek_leja_combine then forms
 *     p_i = ((d_i[0] y_0 + d_i[1] y_1) + d_i[2] y_2) + ...
 * per element in registers, in the reference's order and with its two
 * roundings per term, up to the iteration at which accumulator i froze
 * (read from the state block on the device): bit for bit the accumulators of
 * ek_leja_run, with M + 1 + k vector transfers per call instead of 2kM.
 * y[j] is the iterate of table column j of the chunk starting at iteration
 * chunk_base (first chunk: y[0] = b); cont = 1 continues sums that already
 * hold the earlier chunks. ek_leja_call_seq = ek_leja_call with a folded
 * begin pass followed by ek_leja_run_seq(count) from m = 1. */
int ek_leja_run_seq(const ek_grid* g, int jac, const double* u, const double* fu,
                    const double* const* yin, double* const* yout, int count,
                    const double* coef_dev, int chunk_base, int m_begin, double gamma,
                    ek_leja_state* st, double* work, void* stream);
int ek_leja_combine(int64_t len, const double* const* y, int ny, double* const* p, int k,
                    const double* coef_dev, int chunk_base, int cont,
                    const ek_leja_state* st, void* stream);
int ek_leja_call_seq(const ek_grid* g, int jac, const double* u, const double* fu,
                     const double* b, const double* const* yin, double* const* yout,
                     int count, double* const* p, int k, const double* coef_host,
                     double* coef_dev, double tol, double nu, const double* nu_dev,
                     int lazy0, double gamma, ek_leja_state* st, double* work,
                     void* stream);

/* One recurrence step for a Jacobian action computed elsewhere (dense,
 * callable or 1-D operators): y' = jv/gamma - shift*y, accumulators, norm,
 * freeze test (leja.py:172-184). */
int ek_leja_update(int64_t len, const double* jv, const double* y,
                   double* ynext, double* const* p, int k,
                   const double* coef_dev, int chunk_base, int m,
                   double gamma, int check_jv, ek_leja_state* st,
                   double* work, void* stream);

/* ------------------------------------------------ spectrum (spectrum.py) */
/* Power iterations it in [it_begin, it_end) (spectrum.py:43-63) on a native
 * stencil Jacobian, no host sync: it_begin == 0 first normalises v0
 * (spectrum.py:50-51); the iterate is read as w/||w|| (scaled on read, bit-
 * identical to the reference's v = w / nw). Output ping-pongs in wbuf. */
int ek_power_run(const ek_grid* g, int jac, const double* u, const double* fu,
                 const double* v0, double* const* wbuf, int it_begin,
                 int it_end, ek_power_state* st, double* work,
                 const double* const* halo, void* stream);
/* ||x||^2 (scaled = 0: divisor of the start vector; 1: ||x/nw|| for the FD
 * increment) into the power state (part[] in slab mode). */
int ek_power_norm(int64_t len, const double* x, int scaled, ek_power_state* st,
                  double* work, void* stream);

/* ----------------------------------------------- slab (multi-GPU) mode */
/* With state->defer = 1 the reducing kernels leave their local sums in
 * state->part[EK_PART_SLOTS]; the caller all-gathers the part[] blocks of
 * every rank (`gathered` = nranks x EK_PART_SLOTS slots, device) and applies
 * the decision with the global sums: the exact merge of the ranks' integer
 * accumulators in repro mode (identical for every P), else the rank-ordered
 * fp64 sums: */
int ek_leja_decide(ek_leja_state* st, const double* gathered, int nranks,
                   const double* coef_dev, int chunk_base, int m, int k, int fd,
                   int begin, void* stream);
/* which: 0 = power iteration step, 1 = ||v0||, 2 = ||v|| (FD increment). */
int ek_power_decide(ek_power_state* st, const double* gathered, int nranks,
                    int fd, int which, void* stream);

/* ------------------------------- slab mode over NVLink peer memory */
/* Fused compute + exchange for the Leja recurrence: every
 * rank owns one device "window" that all ranks map (CUDA IPC):
 *   uint64 flag[8]            flag[r] = e+1 once rank r finished pass e
 *   double red[2][8][EK_PART_SLOTS]  [e & 1][r]: rank r's local sums of pass e (EK_PART_*)
 *   double halo[2][2][ncomp][rowlen]  [parity][0: row -1, 1: row `rows`]
 * The fused Leja kernel of pass e stores its boundary rows of y' straight
 * into the neighbours' halo[(e+1) & 1] (reflect ghosts into its own), and
 * its last block writes its partial sums into every window's red[e & 1]
 * and then flag[rank] = e+1 (system-scope fences). A one-warp decide kernel
 * waits for every rank's flag, sums the partials in rank order and applies
 * the freeze test: no host round trip, no NCCL call per iteration. */
typedef struct ek_peer {
    int32_t world;      /* ranks (<= 8)                                    */
    int32_t rank;
    int32_t up;         /* rank owning row -1 of this slab, -1: reflect    */
    int32_t down;       /* rank owning row `rows`, -1: reflect             */
    int64_t rowlen;     /* points per row (2-D) / plane (3-D)              */
    int32_t ncomp;
    int32_t pad_;
    double* win[8];     /* every rank's window as mapped in this process   */
} ek_peer;
#define EK_PEER_HALO_OFFSET 2048 /* bytes: flags (64) + red[2][8][EK_PART_SLOTS] (1024), aligned */
/* Window size for a slab grid. */
int64_t ek_peer_window_bytes(const ek_grid* g);
/* Device allocation (zeroed) plus its CUDA IPC handle (64 bytes out). */
int ek_ipc_alloc(int64_t bytes, void** dptr, void* handle64);
/* Map another process's window; ek_ipc_close unmaps, ek_ipc_free frees. */
int ek_ipc_open(const void* handle64, void** dptr);
int ek_ipc_close(void* dptr);
int ek_ipc_free(void* dptr);
/* Leja iterations m in [m_begin, m_end) in peer mode: pass e = epoch0 +
 * (m - m_begin) reads the ghost rows of y_{m-1} from `halo_b` ([u, y, k]
 * halo pointers as for ek_leja_run, y entry used only when m == 1) or from
 * the own window halo[e & 1], and is followed by the decide kernel. `peer`
 * is a device copy of the ek_peer struct, `win_local` this rank's window.
 * st->defer must be 1. */
int ek_leja_run_peer(const ek_grid* g, int jac, const double* u, const double* fu,
                     const double* b, double* const* ybuf, double* const* p, int k,
                     const double* coef_dev, int chunk_base, int m_begin, int m_end,
                     double gamma, ek_leja_state* st, double* work,
                     const double* const* halo_b, const ek_peer* peer, double* win_local,
                     int64_t epoch0, void* stream);

/* ek_leja_run_peer split by phase: 1 = the fused passes only (halo rows
 * and partial sums stored into the peers' windows, pass flags raised),
 * 2 = the decide kernels only, 3 = both (= ek_leja_run_peer). With fewer
 * GPUs than ranks, a test drives every rank's pass of iteration m before
 * any rank's decide kernel, all on one stream, so no kernel ever waits for
 * one that has not been launched (tests/test_peer_emulated.py). */
int ek_leja_run_peer_phase(const ek_grid* g, int jac, const double* u, const double* fu,
                           const double* b, double* const* ybuf, double* const* p, int k,
                           const double* coef_dev, int chunk_base, int m_begin, int m_end,
                           double gamma, ek_leja_state* st, double* work,
                           const double* const* halo_b, const ek_peer* peer,
                           double* win_local, int64_t epoch0, int phase, void* stream);

/* --------------------------------------------------- KIOPS (kiops.py) */
/* V[0] = [src ; tail], beta = ||V[0]||, V[0] /= beta, ||V[0,:n]||
 * (kiops.py:168-177). Rows of V are device pointers of length n+p. */
int ek_arnoldi_init(int64_t n, int p, const double* src, const double* tail_host,
                    double* V0, ek_arnoldi_state* st, double* work, void* stream);

/* Arnoldi steps j_begin+1 .. j_end (kiops.py:180-194) on a native stencil
 * operator A = dt*J: pass A fuses Jv + augmentation tail@u_flip (the
 * nonzero rows of u_flip are passed as aug[t] = u_flip row / aug_scale with
 * the tail index aug_tail[t] they multiply) + window dots; pass B the CGS subtraction +
 * norm + happy test; pass C the normalisation + ||V[j,:n]||. H is a device
 * row-major ldh x ldh matrix. Stops (early-exit) at a happy breakdown. */
int ek_arnoldi_run(const ek_grid* g, int jac, const double* u,
                   const double* fu, double* const* V, const double* const* aug,
                   const int* aug_tail, int naug, double aug_scale,
                   int j_begin, int j_end,
                   double* H, ek_arnoldi_state* st, int p, int iop, int ldh,
                   double dt, double* work, void* stream);

/* Slab-decomposed Arnoldi with device-side decisions (kiops.py:168-194 on
 * a row slab). Basis rows are the rank's n-part
 * followed by the p tail values, replicated on every rank. The state block
 * has defer = 1: every pass leaves its LOCAL sums in st->part (n-part only:
 * tails are added once, in the decision) and ek_arnoldi_slab_decide applies
 * the global sums of the gathered [nranks][EK_ARN_PART_SLOTS] part blocks:
 *   which 3 after ek_arnoldi_slab_init: beta = ||V[0]||;
 *   which 0 after pass A (phase 0: Jv of V[jj-1] with the halo rows in
 *           `halo`, augmentation, window dots): H[lo.., jj-1] (+ tail dots),
 *           non-finite Jacobian action -> status;
 *   which 1 after pass B (phase 1: CGS subtraction): ||w||, happy test,
 *           H[jj, jj-1];
 *   which 2 after pass C (phase 2: V[jj] /= ||w||): ||V[jj,:n]|| (the next
 *           FD increment).
 * Every rank takes the same decisions; no host synchronisation between the
 * passes (the all-gathers are stream-ordered NCCL collectives). */
int ek_arnoldi_slab_init(int64_t n, int p, const double* src, const double* tail_host,
                         double* V0, ek_arnoldi_state* st, double* work, void* stream);
int ek_arnoldi_slab_pass(const ek_grid* g, int jac, const double* u, const double* fu,
                         double* const* V, const double* const* aug, const int* aug_tail,
                         int naug, double aug_scale, int jj, int phase, double* H,
                         ek_arnoldi_state* st, int p, int iop, int ldh, double dt,
                         double* work, const double* const* halo, void* stream);
int ek_arnoldi_slab_decide(double* const* V, int64_t n, int p, int jj, int iop, double* H,
                           int ldh, ek_arnoldi_state* st, const double* gathered, int nranks,
                           int which, void* stream);

/* Generic-operator Arnoldi: pass A with the (already scaled) action jv. */
int ek_arnoldi_augment(int64_t n, int p, const double* jv, double* const* V,
                       int jj, int iop, const double* const* aug,
                       const int* aug_tail, int naug, double aug_scale,
                       double* H, int ldh,
                       ek_arnoldi_state* st, double* work, void* stream);
/* Passes B and C for basis vector jj. */
int ek_arnoldi_orth(int64_t n, int p, double* const* V, int jj, int iop,
                    double* H, int ldh, ek_arnoldi_state* st, double* work,
                    void* stream);

/* out = sum_i coef_host[i] * V[i][:n], i < j  (kiops.py:267, 270). */
int ek_basis_combine(int64_t n, double* const* V, const double* coef_host,
                     int j, double* out, void* stream);

/* ------------------------------------------------------------ vectors */
/* Elementwise stack program over up to 8 inputs / 4 outputs, NumPy
 * operation order (stage algebra of integrators.py:258-416). Opcodes:
 * 1 LOAD i, 2 CONST s, 3 ADD, 4 SUB, 5 MUL, 6 DIV, 7 NEG, 8 STORE o, 9 POP,
 * 10 NORM slot (st->val[0|2] = ssq, val[1|3] = sqrt), 11 CHECK (flags);
 * word = op | arg << 8. */
int ek_vexpr(int64_t len, const int32_t* prog, int nprog,
             const double* scal, int nscal, const double* const* in, int nin,
             double* const* out, int nout, ek_scalar_state* st, double* work,
             void* stream);
/* Fused linear combinations (the stage algebra's fast path): output o is
 * fin_o(((t_0 + t_1) + t_2) + ...) with t = in[src] (mode 0), coef*in[src]
 * (mode 1), in[src]/coef (mode 2) or coef*(coef2*in[src]) (mode 3: a Leja
 * result that froze at m = 0, d_0*b, consumed without being stored); fin:
 * 0 none, 1 multiply by fval, 2 divide by fval. src / mode / coef / coef2
 * are nout x 6 row-major (coef2 may be NULL without mode 3). out[o] may be
 * NULL (not stored). rmode 1 reduces output 0, rmode 2 the difference
 * out0 - out1 (err = ||u5 - u4||): st->val[0] = ||.||^2, val[1] = ||.||,
 * flag bit0 any nonzero, bit1 any non-finite. */
int ek_lincomb(int64_t len, const double* const* in, int nin,
               double* const* out, int nout, const int32_t* nterm,
               const int32_t* src, const int32_t* mode, const double* coef,
               const double* coef2, const int32_t* fin, const double* fval, int rmode,
               ek_scalar_state* st, double* work, void* stream);
/* ||x||^2 -> st->val[slot], ||x|| -> st->val[slot+1]; st->flag bit0 any
 * nonzero, bit1 any non-finite. */
int ek_norm2(int64_t len, const double* x, ek_scalar_state* st, int slot,
             double* work, void* stream);
/* sum |x| -> st->val[slot]  (kiops.py:146). */
int ek_l1(int64_t len, const double* x, ek_scalar_state* st, int slot,
          double* work, void* stream);
/* Self test of the division used by the kernels: fast[i] = reciprocal-
 * correction quotient, exact[i] = x[i]/d[i] by the division instruction. */
int ek_selftest_div(int64_t n, const double* x, const double* d, double* fast,
                    double* exact, void* stream);
/* Self test of the order-independent sums: sum of x[0..n) (sq = 1: of the
 * squares) by a grid of `blocks` blocks through the kernels' reduction path;
 * out_slots[EK_XSLOTS] (device) = the merged accumulator, st->val[0] = its
 * fp64 value. Synchronises the stream. */
int ek_selftest_xsum(int64_t n, const double* x, int sq, int blocks, ek_scalar_state* st,
                     int64_t* out_slots, void* stream);
/* y = A x, A dense row-major (linalg.py:87-90 from_matrix). */
int ek_dense_gemv(int64_t n, const double* A, const double* x, double* y,
                  void* stream);

/* -------------------------------------------------------- handle layer */
/* Context / operator handles over the grid-level entry points, for hosts
 * that prefer an object API. The library owns the
 * handles' workspaces and state blocks; vectors stay caller-owned. */
typedef struct ek_ctx ek_ctx;
typedef struct ek_op ek_op;

/* Bind a device and the stream every call on this context runs on. NULL on
 * failure (ek_last_error). Multi-GPU: one context per process/GPU; the
 * slab exchange itself is the host framework's (torch.distributed / NCCL). */
ek_ctx* ek_ctx_create(int device, void* stream);
void ek_ctx_destroy(ek_ctx* ctx);

/* Operator of one problem on one grid (problem id, dims, components, bc,
 * parameters: all in `g`) with the Jacobian kind jac (EK_JAC_FD /
 * EK_JAC_ANALYTIC) -- the native counterpart of MatrixFreeOperator over a
 * Problem's rhs / jac_factory (linalg.py:67-85, problems.py:46-60). */
ek_op* ek_op_create(ek_ctx* ctx, const ek_grid* g, int jac);
void ek_op_destroy(ek_op* op);

/* make_linearized (integrators.py:80-96): fu = f(u), *out_norm_u_host =
 * ||u||; (u, fu) become the operator's linearisation point. Syncs. */
int ek_op_linearize(ek_op* op, const double* u, double* fu, double* out_norm_u_host);
/* out = f(u) */
int ek_op_rhs(ek_op* op, const double* u, double* out);
/* out = J v at the linearisation point. FD (fd_jacobian_apply,
 * linalg.py:111-129): eps = (sqrt(eps_mach)*(1+||u||))/||v||; ||v|| = 0 ->
 * EK_ERR_INVALID, non-finite result -> EK_ERR_NONFINITE. Syncs (FD). */
int ek_op_jv(ek_op* op, const double* v, double* out);
/* One power-iteration step (spectrum.py:56-58): w = J v, *norm_out_host =
 * ||w||. Syncs. */
int ek_power_step(ek_op* op, const double* v, double* w, double* norm_out_host);

/* out = (a*x) + (b*y), NumPy order. */
int ek_axpby(int64_t n, double a, const double* x, double b, const double* y,
             double* out, void* stream);
/* st->val[i] = x . ys[i] for i < k <= 8, one pass, deterministic block
 * partials (the window dots of kiops.py:188-190). out_host (nullable):
 * the k results copied to the host (syncs). work: ek_workspace_bytes. */
int ek_dot_multi(int64_t n, const double* x, const double* const* ys, int k,
                 ek_scalar_state* st, double* out_host, double* work, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* EXPKIT_SM100_H */
