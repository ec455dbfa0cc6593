// expkit_sm100.cu — C ABI of libexpkit_sm100.so (see include/expkit_sm100.h).
//
// Host-side launchers: pick the kernel instance for (problem, value,
// epilogue), size the grid, and loop over iterations on the stream without
// host synchronisation (the iteration state lives in device memory).
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <map>
#include <mutex>
#include <tuple>
#include <type_traits>

#include <cudaTypedefs.h>

#include "ek_common.cuh"
#include "ek_launch.cuh"
#include "ek_vector.cuh"

namespace ek {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int cuda_status(cudaError_t e, const char* where) {
    set_error("%s: CUDA error %d (%s)", where, (int)e, cudaGetErrorString(e));
    return EK_ERR_CUDA;
}

static std::atomic<long long> g_launches{0};
int g_tma_mode = 3;  // see ek_set_tma
int g_march_mask = 1 << EP_LEJA;  // see ek_set_march
int g_repro = 0;  // see ek_set_repro: order-independent sums (ek_xsum.cuh)
thread_local LaunchDesc* g_record = nullptr;  // see ek_launch.cuh
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// ------------------------------------------------------------- 1-D problem
// problems.py:154-196: semilinear, Dirichlet, nonlocal trapezoid integral.
// One block; thread 0 reproduces NumPy's pairwise summation order
// (loops_utils.h pairwise_sum) for np.sum(u).

struct SemiArgs {
    int64_t n;         // interior points; the vector has n+1 entries
    double h, h2, h24; // h, h**2, h/24.0
    int mode;          // 0: f(u)  1: (f(u+eps y)-fu)/eps  2: J(t_n) y
    const double* u;
    const double* y;
    const double* fu;
    double eps;
    double* out;
    ek_scalar_state* st;  // optional: non-finite flag (mode 1)
};

__device__ __forceinline__ double semi_in(const SemiArgs& a, int64_t i) {
    if (a.mode == 0) return a.u[i];
    if (a.mode == 1) return a.u[i] + a.eps * a.y[i];
    return a.y[i];
}

__device__ double semi_pairwise(const SemiArgs& a, int64_t lo, int64_t n) {
    if (n < 8) {
        double r = -0.0;
        for (int64_t i = 0; i < n; ++i) r += semi_in(a, lo + i);
        return r;
    }
    if (n <= 128) {
        double r[8];
        for (int q = 0; q < 8; ++q) r[q] = semi_in(a, lo + q);
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int q = 0; q < 8; ++q) r[q] += semi_in(a, lo + i + q);
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += semi_in(a, lo + i);
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return semi_pairwise(a, lo, n2) + semi_pairwise(a, lo + n2, n - n2);
}

__device__ __forceinline__ double semi_forcing(double x, double t) {
    return exp(t) * (((x * (1.0 - x)) + 2.0) - (1.0 / 6.0));  // problems.py:148-151
}

__global__ void __launch_bounds__(TPB) k_semilinear(const SemiArgs a) {
    __shared__ double s_q;
    __shared__ int s_bad;
    const int64_t n = a.n;
    if (threadIdx.x == 0) {
        s_bad = 0;
        const double S = semi_pairwise(a, 0, n);
        const double w0 = semi_in(a, 0), w1 = n > 1 ? semi_in(a, 1) : 0.0;
        const double wl = semi_in(a, n - 1), wl2 = n > 1 ? semi_in(a, n - 2) : 0.0;
        const double corr = a.h24 * ((((4.0 * w0) - w1) + (4.0 * wl)) - wl2);  // problems.py:167
        s_q = (a.h * S) + corr;
    }
    __syncthreads();
    const double q = s_q;
    const double t = semi_in(a, n);  // time component
    const double tn = a.u[n];         // linearisation time (mode 2)
    int bad = 0;
    for (int64_t i = threadIdx.x; i <= n; i += TPB) {
        double r;
        if (i == n) {
            r = a.mode == 0 ? 1.0 : a.mode == 1 ? (1.0 - a.fu[n]) / a.eps : 0.0;
        } else {
            const double wm = i > 0 ? semi_in(a, i - 1) : 0.0;
            const double wp = i + 1 < n ? semi_in(a, i + 1) : 0.0;
            const double wi = semi_in(a, i);
            const double d2 = ((wm - (2.0 * wi)) + wp) / a.h2;  // problems.py:172-173
            const double x = a.h * (double)(i + 1);
            if (a.mode == 2) {
                r = (d2 + q) + (semi_forcing(x, tn) * t);  // problems.py:186
            } else {
                r = (d2 + q) + semi_forcing(x, t);  // problems.py:174
                if (a.mode == 1) r = (r - a.fu[i]) / a.eps;
            }
        }
        a.out[i] = r;
        bad |= isfinite(r) ? 0 : 1;
    }
    if (a.st && bad) atomicOr(&s_bad, 1);
    __syncthreads();
    if (a.st && threadIdx.x == 0 && s_bad) a.st->flag |= 2;
}

// --------------------------------------------------------------- dispatch

static int64_t grid_points(const ek_grid* g) {
    if (g->dim == 1) return g->n;
    if (g->dim == 2) return g->rows * g->n;
    return g->rows * g->n * g->n;
}

static bool grid_ok(const ek_grid* g) {
    if (!g) {
        set_error("null grid");
        return false;
    }
    if (g->n < 1 || g->rows < 1 || g->ncomp < 1 || g->ncomp > 2 || g->dim < 1 || g->dim > 3) {
        set_error("invalid grid (n=%lld rows=%lld ncomp=%d dim=%d)", (long long)g->n,
                  (long long)g->rows, g->ncomp, g->dim);
        return false;
    }
    return true;
}


template <int EP>
static int launch_stencil(int ev, const KArgs& a, cudaStream_t s) {
    switch (a.g.problem) {
        case EK_P_ADR: return launch_adr(EP, ev, a, s);
        case EK_P_ALLEN_CAHN: return launch_allen_cahn(EP, ev, a, s);
        case EK_P_BRUSS_PRINTED: return launch_bruss_printed(EP, ev, a, s);
        case EK_P_BRUSS_STANDARD: return launch_bruss_standard(EP, ev, a, s);
        case EK_P_GRAY_SCOTT: return launch_gray_scott(EP, ev, a, s);
        case EK_P_ADVDIFF2D: return launch_advdiff2d(EP, ev, a, s);
        case EK_P_BURGERS2D: return launch_burgers2d(EP, ev, a, s);
        case EK_P_ADVDIFF3D: return launch_advdiff3d(EP, ev, a, s);
    }
    set_error("problem %d has no 2-D/3-D stencil", a.g.problem);
    return EK_ERR_UNSUPPORTED;
}

static void base_args(KArgs& a, const ek_grid* g, const double* const* halo) {
    memset(&a, 0, sizeof(a));
    a.g = *g;
    a.npts = grid_points(g);
    a.pc.h2 = mkdv(g->h2);
    a.pc.two_h = mkdv(g->two_h);
    a.pc.h = mkdv(g->h);
    for (int i = 0; i < 8; ++i) a.pc.prm[i] = g->prm[i];
    a.gamma = mkdv(1.0);
    a.repro = g_repro;
    if (halo) {
        a.hu = halo[0];
        a.hy = halo[1];
        a.hk = halo[2];
    }
}

// analytic Jacobian value kind of a problem
static int analytic_ev(const ek_grid* g) {
    if (g->problem == EK_P_ADVDIFF2D || g->problem == EK_P_ADVDIFF3D) return EV_LIN;
    if (g->problem == EK_P_BURGERS2D) return EV_BURGJ;
    return -1;
}

static int jv_ev(const ek_grid* g, int jac) {
    if (jac == EK_JAC_FD) return EV_FD;
    const int ev = analytic_ev(g);
    if (ev < 0) set_error("problem %d has no analytic Jacobian stencil", g->problem);
    return ev;
}

}  // namespace ek

using namespace ek;

// =============================================================== C ABI
extern "C" {

const char* ek_last_error(void) { return g_err; }
int ek_version(void) { return 1; }
long long ek_launch_count(void) { return g_launches.load(); }
int ek_set_tma(int mode) {
    const int old = g_tma_mode;
    if (mode >= 0) g_tma_mode = mode > 4 ? 3 : mode;
    return old;
}

int ek_set_repro(int on) {
    const int old = g_repro;
    if (on >= 0) g_repro = on ? 1 : 0;
    return old;
}

double ek_xsum_value(const int64_t* slots, int n) {
    XAcc tot;
    xzero(tot);
    for (int r = 0; r < n; ++r) xmerge(tot, xload((const long long*)slots + (long)r * XSLOTS));
    return xvalue(tot);
}

void ek_xsum_host(const double* x, int64_t n, int sq, int64_t* slots_out) {
    XAcc acc;
    xzero(acc);
    for (int64_t i = 0; i < n; ++i) {
        if (sq) xadd<false>(acc, x[i] * x[i]);
        else xadd<true>(acc, x[i]);
    }
    xstore((long long*)slots_out, acc);
}

int ek_set_march(int mask) {
    const int old = g_march_mask;
    if (mask >= 0) g_march_mask = mask;
    return old;
}

int ek_copy(void* dst, const void* src, int64_t bytes, int kind, void* stream) {
    const cudaMemcpyKind k = kind == 1 ? cudaMemcpyHostToDevice
                           : kind == 2 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    cudaError_t e = cudaMemcpyAsync(dst, src, (size_t)bytes, k, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e, "ek_copy");
    return EK_OK;
}

int ek_sync(void* stream) {
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_status(e, "ek_sync");
    return EK_OK;
}

int64_t ek_grid_len(const ek_grid* g) {
    if (!g) return 0;
    if (g->problem == EK_P_SEMILINEAR) return g->n + 1;
    return (int64_t)g->ncomp * grid_points(g);
}

int64_t ek_workspace_bytes(const ek_grid* g) {
    int64_t nb = VGRID_MAX;
    if (g && g->dim >= 2) {
        const int64_t sb = (int64_t)sm_count() * 8;  // persistent stencil grids
        if (sb > nb) nb = sb;
    }
    // per block: up to 8 fp64 partials, and in repro mode up to 8 integer
    // accumulators of XSLOTS slots behind them
    return nb * (8 + 8 * XSLOTS) * (int64_t)sizeof(double);
}

int ek_rhs(const ek_grid* g, const double* u, double* out, const double* const* halo,
           void* stream) {
    if (!grid_ok(g)) return EK_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    if (g->problem == EK_P_SEMILINEAR) {
        SemiArgs a{};
        a.n = g->n; a.h = g->h; a.h2 = g->h2; a.h24 = g->prm[0];
        a.mode = 0; a.u = u; a.out = out;
        k_semilinear<<<1, TPB, 0, s>>>(a);
        EK_LAUNCH_CHECK("k_semilinear");
        return EK_OK;
    }
    KArgs a;
    base_args(a, g, halo);
    a.u = u;
    a.out = out;
    return launch_stencil<EP_STORE>(EV_RHS, a, s);
}

int ek_rhs_norm(const ek_grid* g, const double* u, double* out, ek_scalar_state* st,
                double* work, const double* const* halo, void* stream) {
    if (!grid_ok(g)) return EK_ERR_INVALID;
    if (g->dim < 2 || !st || !work) {
        set_error("ek_rhs_norm: 2-D / 3-D stencil grids with a state block and workspace");
        return EK_ERR_INVALID;
    }
    KArgs a;
    base_args(a, g, halo);
    a.u = u;
    a.out = out;
    a.st = st;
    a.work = work;
    return launch_stencil<EP_RHSN>(EV_RHS, a, (cudaStream_t)stream);
}

int ek_jv(const ek_grid* g, int jac, const double* u, const double* fu, const double* v,
          double eps, double* out, ek_scalar_state* st, double* work,
          const double* const* halo, void* stream) {
    (void)work;
    if (!grid_ok(g)) return EK_ERR_INVALID;
    cudaStream_t s = (cudaStream_t)stream;
    if (g->problem == EK_P_SEMILINEAR) {
        SemiArgs a{};
        a.n = g->n; a.h = g->h; a.h2 = g->h2; a.h24 = g->prm[0];
        a.mode = jac == EK_JAC_FD ? 1 : 2;
        a.u = u; a.y = v; a.fu = fu; a.eps = eps; a.out = out; a.st = st;
        k_semilinear<<<1, TPB, 0, s>>>(a);
        EK_LAUNCH_CHECK("k_semilinear");
        return EK_OK;
    }
    const int ev = jv_ev(g, jac);
    if (ev < 0) return EK_ERR_UNSUPPORTED;
    KArgs a;
    base_args(a, g, halo);
    a.u = u; a.fu = fu; a.y = v; a.eps = eps; a.out = out;
    int rc = launch_stencil<EP_STORE>(ev, a, s);
    if (rc != EK_OK || jac != EK_JAC_FD || !st) return rc;
    // non-finite check of the FD result (linalg.py:127-128)
    k_norm2<<<vgrid4(ek_grid_len(g)), TPB, 0, s>>>(ek_grid_len(g), out, nullptr, st, 6, work, 0);
    EK_LAUNCH_CHECK("k_norm2");
    return EK_OK;
}

int ek_remainder(const ek_grid* g, int jac, const double* u, const double* fu, const double* k,
                 double eps, double* out, ek_scalar_state* st, double* work,
                 const double* const* halo, void* stream) {
    if (!grid_ok(g)) return EK_ERR_INVALID;
    if (g->problem == EK_P_SEMILINEAR) {
        set_error("semilinear remainder runs through the generic path");
        return EK_ERR_UNSUPPORTED;
    }
    int ev;
    if (jac == EK_JAC_FD) ev = EV_REMFD;
    else if (analytic_ev(g) == EV_LIN) ev = EV_REMLIN;
    else if (analytic_ev(g) == EV_BURGJ) ev = EV_REMBURG;
    else {
        set_error("problem %d has no analytic Jacobian stencil", g->problem);
        return EK_ERR_UNSUPPORTED;
    }
    KArgs a;
    base_args(a, g, halo);
    a.u = u; a.fu = fu; a.k = k; a.eps = eps; a.out = out; a.st = st; a.work = work;
    return launch_stencil<EP_REM>(ev, a, (cudaStream_t)stream);
}

static int remainder_combo(const ek_grid* g, int jac, const double* u, const double* fu,
                           const double* k, double eps, const ek_scalar_state* pre,
                           const double* nu, double* out, int nx, double* const* xo,
                           const double* xin, const double* xa, const double* xr,
                           const double* xf, ek_scalar_state* st, double* work,
                           const double* const* halo, void* stream) {
    if (!grid_ok(g)) return EK_ERR_INVALID;
    if (pre && jac == EK_JAC_FD && !nu) {
        set_error("ek_remainder_combo_dev: FD needs the device ||u_n||");
        return EK_ERR_INVALID;
    }
    if (nx < 0 || nx > 3 || (nx > 0 && (!xo || !xr || !xf || (xin && !xa))) || (!out && nx == 0)) {
        set_error("ek_remainder_combo: bad outputs (nx=%d)", nx);
        return EK_ERR_INVALID;
    }
    if (g->problem == EK_P_SEMILINEAR) {
        set_error("semilinear remainder runs through the generic path");
        return EK_ERR_UNSUPPORTED;
    }
    int ev;
    if (jac == EK_JAC_FD) ev = EV_REMFD;
    else if (analytic_ev(g) == EV_LIN) ev = EV_REMLIN;
    else if (analytic_ev(g) == EV_BURGJ) ev = EV_REMBURG;
    else {
        set_error("problem %d has no analytic Jacobian stencil", g->problem);
        return EK_ERR_UNSUPPORTED;
    }
    KArgs a;
    base_args(a, g, halo);
    a.u = u; a.fu = fu; a.k = k; a.eps = eps; a.out = out; a.st = st; a.work = work;
    a.pre = pre; a.nu = nu;
    a.nxo = nx;
    a.xin = xin;
    for (int q = 0; q < nx; ++q) {
        a.xo[q] = xo[q];
        a.xa[q] = xin ? xa[q] : 0.0;
        a.xr[q] = xr[q];
        a.xf[q] = xf[q];
    }
    return launch_stencil<EP_REM>(ev, a, (cudaStream_t)stream);
}

int ek_remainder_combo(const ek_grid* g, int jac, const double* u, const double* fu,
                       const double* k, double eps, double* out, int nx, double* const* xo,
                       const double* xin, const double* xa, const double* xr, const double* xf,
                       ek_scalar_state* st, double* work, const double* const* halo,
                       void* stream) {
    return remainder_combo(g, jac, u, fu, k, eps, nullptr, nullptr, out, nx, xo, xin, xa, xr,
                           xf, st, work, halo, stream);
}

int ek_remainder_combo_dev(const ek_grid* g, int jac, const double* u, const double* fu,
                           const double* k, const ek_scalar_state* pre, const double* nu,
                           double* out, int nx, double* const* xo, const double* xin,
                           const double* xa, const double* xr, const double* xf,
                           ek_scalar_state* st, double* work, const double* const* halo,
                           void* stream) {
    if (!pre) {
        set_error("ek_remainder_combo_dev: pre is required");
        return EK_ERR_INVALID;
    }
    return remainder_combo(g, jac, u, fu, k, 0.0, pre, nu, out, nx, xo, xin, xa, xr, xf, st,
                           work, halo, stream);
}

// ------------------------------------------------------------------- Leja
// m = 0 over a flat vector of length len (the state block must hold tol,
// nu and k; see ek_leja_state).
int ek_leja_begin_len(int64_t len, const double* b, double* const* p, int k,
                      const double* coef_dev, ek_leja_state* st, double* work, void* stream) {
    if (k < 1 || k > 8 || len < 1) {
        set_error("ek_leja_begin_len: bad k=%d len=%lld", k, (long long)len);
        return EK_ERR_INVALID;
    }
    LejaVArgs a{};
    a.len = len; a.b = b; a.nk = k; a.coef = coef_dev; a.mi = 0; a.m = 0; a.st = st; a.work = work;
    a.repro = g_repro;
    for (int q = 0; q < k; ++q) a.p[q] = p[q];
    k_leja_begin<<<vgrid4(len), TPB, 0, (cudaStream_t)stream>>>(a);
    EK_LAUNCH_CHECK("k_leja_begin");
    // folded begin that froze everything at m = 0: write d_i[0] b (early
    // exit in every other case)
    k_leja_fold_done<<<vgrid4(len), TPB, 0, (cudaStream_t)stream>>>(a);
    EK_LAUNCH_CHECK("k_leja_fold_done");
    return EK_OK;
}

int ek_leja_run(const ek_grid* g, int jac, const double* u, const double* fu, const double* b,
                double* const* ybuf, double* const* p, int k, const double* coef_dev,
                int chunk_base, int m_begin, int m_end, double gamma, ek_leja_state* st,
                double* work, const double* const* halo, void* stream) {
    if (!grid_ok(g)) return EK_ERR_INVALID;
    if (k < 1 || k > 8) {
        set_error("ek_leja_run: k=%d out of range", k);
        return EK_ERR_INVALID;
    }
    const int ev = jv_ev(g, jac);
    if (ev < 0) return EK_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    KArgs a;
    base_args(a, g, halo);
    a.u = u; a.fu = fu; a.nk = k; a.coef = coef_dev; a.gamma = mkdv(gamma); a.st = st; a.work = work;
    for (int q = 0; q < k; ++q) a.p[q] = p[q];
    for (int m = m_begin; m < m_end; ++m) {
        a.m = m;
        a.mi = m - chunk_base;
        a.y = (m == 1) ? b : ybuf[(m - 1) & 1];
        a.out = ybuf[m & 1];
        const int rc = launch_stencil<EP_LEJA>(ev, a, s);
        if (rc != EK_OK) return rc;
    }
    return EK_OK;
}

// ------------------------------------------------- Leja loop as a CUDA graph
// the iterations of a phi-call as a device-side loop. The
// graph holds iteration 1 (kind A only) and a conditional WHILE node whose
// body is two kernel nodes, the even and the odd iterations (the iterate
// ping-pongs between two buffers, so each node's pointers are fixed); every
// node takes its iteration index from the state block and the block that
// finalises an iteration sets the loop condition (leja_decide: not done, and
// the next column is still in this 32-point chunk). One graph launch runs
// the call to its end or to the chunk boundary: no launch batch to size, no
// launches that find the call finished, no host work per iteration.
// Executable graphs are cached per kernel instance and launch geometry; a
// call only rewrites the three nodes' arguments.
namespace {
struct LejaGraph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaGraphNode_t first = nullptr, even = nullptr, odd = nullptr;
    cudaGraphConditionalHandle cond = 0;
};
using LejaGraphKey = std::tuple<void*, void*, void*, unsigned, unsigned, size_t, int, int, int>;
std::map<LejaGraphKey, LejaGraph> g_leja_graphs;
std::mutex g_leja_graphs_mu;

void kernel_params(const LaunchDesc& d, void** kp, cudaKernelNodeParams& p) {
    kp[0] = (void*)&d.args;
    kp[1] = (void*)&d.maps;
    p = cudaKernelNodeParams{};
    p.func = d.func;
    p.gridDim = d.grid;
    p.blockDim = d.block;
    p.sharedMemBytes = (unsigned)d.smem;
    p.kernelParams = kp;
}

int build_leja_graph(LejaGraph& lg, LaunchDesc* d, bool with_first) {
    cudaError_t e = cudaGraphCreate(&lg.graph, 0);
    if (e != cudaSuccess) return cuda_status(e, "leja graph: create");
    // kind A: iteration 1 decides whether the loop runs at all (default 0);
    // kind B (a later chunk, launched only while the call is unfinished): 1
    e = cudaGraphConditionalHandleCreate(&lg.cond, lg.graph, with_first ? 0u : 1u,
                                         cudaGraphCondAssignDefault);
    if (e != cudaSuccess) return cuda_status(e, "leja graph: conditional handle");
    for (int i = 0; i < 3; ++i) {
        d[i].args.cond = lg.cond;
        d[i].args.cond_on = 1;
    }
    void* kp[2];
    cudaKernelNodeParams p;
    if (with_first) {
        kernel_params(d[0], kp, p);
        e = cudaGraphAddKernelNode(&lg.first, lg.graph, nullptr, 0, &p);
        if (e != cudaSuccess) return cuda_status(e, "leja graph: first node");
    }
    cudaGraphNodeParams cp = {cudaGraphNodeTypeConditional};
    cp.conditional.handle = lg.cond;
    cp.conditional.type = cudaGraphCondTypeWhile;
    cp.conditional.size = 1;
    cudaGraphNode_t loop;
    e = cudaGraphAddNode(&loop, lg.graph, with_first ? &lg.first : nullptr, with_first ? 1 : 0,
                         &cp);
    if (e != cudaSuccess) return cuda_status(e, "leja graph: while node");
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    kernel_params(d[1], kp, p);
    e = cudaGraphAddKernelNode(&lg.even, body, nullptr, 0, &p);
    if (e != cudaSuccess) return cuda_status(e, "leja graph: even node");
    kernel_params(d[2], kp, p);
    e = cudaGraphAddKernelNode(&lg.odd, body, &lg.even, 1, &p);
    if (e != cudaSuccess) return cuda_status(e, "leja graph: odd node");
    e = cudaGraphInstantiate(&lg.exec, lg.graph, 0);
    if (e != cudaSuccess) return cuda_status(e, "leja graph: instantiate");
    return EK_OK;
}

// Iterations m_begin .. of one chunk (until done, m_limit or the chunk end)
// as one graph launch. m_begin == 1: the first chunk; otherwise m_begin must
// be even (chunk boundaries are multiples of 32).
int leja_graph_run(int ev, const KArgs& base, const double* b, double* const* ybuf,
                   int chunk_base, int m_begin, int m_limit, cudaStream_t s) {
    const bool with_first = m_begin == 1;
    if (!with_first && (m_begin & 1)) {
        set_error("leja graph: a later chunk must start at an even iteration (m=%d)", m_begin);
        return EK_ERR_INVALID;
    }
    LaunchDesc d[3];
    for (int i = 0; i < 3; ++i) {
        KArgs a = base;
        a.chunk_base = chunk_base;
        a.m_limit = m_limit;
        if (i == 0) {  // iteration 1: y_0 = b
            a.m = 1; a.mi = 1 - chunk_base; a.y = b; a.out = ybuf[1];
        } else if (i == 1) {  // even iterations: y_{m-1} in ybuf[1]
            a.m = -2; a.y = ybuf[1]; a.out = ybuf[0];
        } else {  // odd iterations > 1
            a.m = -1; a.y = ybuf[0]; a.out = ybuf[1];
        }
        if (i == 0 && !with_first) continue;
        g_record = &d[i];
        const int rc = launch_stencil<EP_LEJA>(ev, a, s);
        const bool recorded = g_record->func != nullptr;
        g_record = nullptr;
        if (rc != EK_OK) return rc;
        if (!recorded) {
            set_error("leja graph: launch not recorded");
            return EK_ERR_UNSUPPORTED;
        }
    }
    int dev = 0;
    cudaGetDevice(&dev);  // executable graphs belong to one device
    const LejaGraphKey key{with_first ? d[0].func : nullptr, d[1].func, d[2].func, d[1].grid.x,
                           d[1].block.x, d[1].smem, with_first ? (int)d[0].grid.x : 0,
                           d[1].has_maps ? 1 : 0, dev};
    std::lock_guard<std::mutex> lock(g_leja_graphs_mu);
    auto it = g_leja_graphs.find(key);
    if (it == g_leja_graphs.end()) {
        LejaGraph lg;
        const int rc = build_leja_graph(lg, d, with_first);
        if (rc != EK_OK) return rc;
        it = g_leja_graphs.emplace(key, lg).first;
    }
    LejaGraph& lg = it->second;
    void* kp[2];
    cudaKernelNodeParams p;
    for (int i = with_first ? 0 : 1; i < 3; ++i) {
        d[i].args.cond = lg.cond;
        d[i].args.cond_on = 1;
        kernel_params(d[i], kp, p);
        cudaGraphNode_t node = i == 0 ? lg.first : (i == 1 ? lg.even : lg.odd);
        cudaError_t e = cudaGraphExecKernelNodeSetParams(lg.exec, node, &p);
        if (e != cudaSuccess) return cuda_status(e, "leja graph: node arguments");
    }
    cudaError_t e = cudaGraphLaunch(lg.exec, s);
    if (e != cudaSuccess) return cuda_status(e, "leja graph: launch");
    count_launch();
    return EK_OK;
}
}  // namespace

int ek_leja_run_graph(const ek_grid* g, int jac, const double* u, const double* fu,
                      const double* b, double* const* ybuf, double* const* p, int k,
                      const double* coef_dev, int chunk_base, int m_begin, int m_limit,
                      double gamma, ek_leja_state* st, double* work, void* stream) {
    if (!grid_ok(g)) return EK_ERR_INVALID;
    if (k < 1 || k > 8) {
        set_error("ek_leja_run_graph: k=%d out of range", k);
        return EK_ERR_INVALID;
    }
    const int ev = jv_ev(g, jac);
    if (ev < 0) return EK_ERR_UNSUPPORTED;
    KArgs a;
    base_args(a, g, nullptr);
    a.u = u; a.fu = fu; a.nk = k; a.coef = coef_dev; a.gamma = mkdv(gamma); a.st = st; a.work = work;
    for (int q = 0; q < k; ++q) a.p[q] = p[q];
    return leja_graph_run(ev, a, b, ybuf, chunk_base, m_begin, m_limit, (cudaStream_t)stream);
}

int ek_leja_call(const ek_grid* g, int jac, const double* u, const double* fu, const double* b,
                 double* const* ybuf, double* const* p, int k, const double* coef_host,
                 double* coef_dev, double tol, double nu, const double* nu_dev, int fold,
                 int lazy0, int m_end, double gamma, ek_leja_state* st, double* work,
                 void* stream) {
    if (!grid_ok(g)) return EK_ERR_INVALID;
    if (k < 1 || k > 8 || !coef_host || !coef_dev || !st) {
        set_error("ek_leja_call: bad arguments (k=%d)", k);
        return EK_ERR_INVALID;
    }
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyAsync(coef_dev, coef_host, (size_t)(k + 1) * 32 * sizeof(double),
                                    cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "ek_leja_call");
    k_leja_init<<<1, 32, 0, s>>>(st, tol, nu, nu_dev, k, fold ? -1 : 0, lazy0);
    EK_LAUNCH_CHECK("k_leja_init");
    int rc = ek_leja_begin_len(ek_grid_len(g), b, p, k, coef_dev, st, work, stream);
    if (rc != EK_OK || (m_end >= 0 && m_end <= 1)) return rc;
    if (m_end < 0)  // graph mode: the whole first chunk as one device-side loop, up to -m_end
        return ek_leja_run_graph(g, jac, u, fu, b, ybuf, p, k, coef_dev, 0, 1, -m_end, gamma, st,
                                 work, stream);
    return ek_leja_run(g, jac, u, fu, b, ybuf, p, k, coef_dev, 0, 1, m_end, gamma, st, work,
                       nullptr, stream);
}

// Deferred accumulation: iterations m_begin .. m_begin + count - 1 with
// explicit iterate buffers (y_{m-1} in yin[i], y_m into yout[i]) and no
// accumulator traffic (kernel instances with K = 0); the freeze decisions
// run over the state block's k as usual.
int ek_leja_run_seq(const ek_grid* g, int jac, const double* u, const double* fu,
                    const double* const* yin, double* const* yout, int count,
                    const double* coef_dev, int chunk_base, int m_begin, double gamma,
                    ek_leja_state* st, double* work, void* stream) {
    if (!grid_ok(g)) return EK_ERR_INVALID;
    if (count < 0 || !yin || !yout || !st) {
        set_error("ek_leja_run_seq: bad arguments (count=%d)", count);
        return EK_ERR_INVALID;
    }
    const int ev = jv_ev(g, jac);
    if (ev < 0) return EK_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    KArgs a;
    base_args(a, g, nullptr);
    a.u = u; a.fu = fu; a.nk = 0; a.coef = coef_dev; a.gamma = mkdv(gamma); a.st = st; a.work = work;
    for (int i = 0; i < count; ++i) {
        a.m = m_begin + i;
        a.mi = a.m - chunk_base;
        a.y = yin[i];
        a.out = yout[i];
        const int rc = launch_stencil<EP_LEJA>(ev, a, s);
        if (rc != EK_OK) return rc;
    }
    return EK_OK;
}

int ek_leja_combine(int64_t len, const double* const* y, int ny, double* const* p, int k,
                    const double* coef_dev, int chunk_base, int cont, const ek_leja_state* st,
                    void* stream) {
    if (len < 1 || k < 1 || k > 8 || ny < 1 || ny > 33 || !y || !p || !coef_dev || !st) {
        set_error("ek_leja_combine: bad arguments (k=%d ny=%d)", k, ny);
        return EK_ERR_INVALID;
    }
    LejaCombineArgs a{};
    a.len = len; a.ny = ny; a.nk = k; a.coef = coef_dev; a.chunk_base = chunk_base;
    a.cont = cont; a.st = st;
    for (int j = 0; j < ny; ++j) a.y[j] = y[j];
    for (int q = 0; q < k; ++q) a.p[q] = p[q];
    const dim3 grid = vgrid4(len);
    cudaStream_t s = (cudaStream_t)stream;
    switch (k) {
        case 1: k_leja_combine<1><<<grid, TPB, 0, s>>>(a); break;
        case 2: k_leja_combine<2><<<grid, TPB, 0, s>>>(a); break;
        case 3: k_leja_combine<3><<<grid, TPB, 0, s>>>(a); break;
        case 4: k_leja_combine<4><<<grid, TPB, 0, s>>>(a); break;
        default: k_leja_combine<8><<<grid, TPB, 0, s>>>(a); break;
    }
    EK_LAUNCH_CHECK("k_leja_combine");
    return EK_OK;
}

// ek_leja_call with deferred accumulation: table upload, state init, folded
// begin pass and the first `count` iterations (ek_leja_run_seq).
int ek_leja_call_seq(const ek_grid* g, int jac, const double* u, const double* fu,
                     const double* b, const double* const* yin, double* const* yout, int count,
                     double* const* p, int k, const double* coef_host, double* coef_dev,
                     double tol, double nu, const double* nu_dev, int lazy0, double gamma,
                     ek_leja_state* st, double* work, void* stream) {
    if (!grid_ok(g)) return EK_ERR_INVALID;
    if (k < 1 || k > 8 || !coef_host || !coef_dev || !st) {
        set_error("ek_leja_call_seq: bad arguments (k=%d)", k);
        return EK_ERR_INVALID;
    }
    cudaStream_t s = (cudaStream_t)stream;
    cudaError_t e = cudaMemcpyAsync(coef_dev, coef_host, (size_t)(k + 1) * 32 * sizeof(double),
                                    cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_status(e, "ek_leja_call_seq");
    k_leja_init<<<1, 32, 0, s>>>(st, tol, nu, nu_dev, k, -1, lazy0);
    EK_LAUNCH_CHECK("k_leja_init");
    const int rc = ek_leja_begin_len(ek_grid_len(g), b, p, k, coef_dev, st, work, stream);
    if (rc != EK_OK || count < 1) return rc;
    return ek_leja_run_seq(g, jac, u, fu, yin, yout, count, coef_dev, 0, 1, gamma, st, work,
                           stream);
}

int ek_leja_update(int64_t len, const double* jv, const double* y, double* ynext,
                   double* const* p, int k, const double* coef_dev, int chunk_base, int m,
                   double gamma, int check_jv, ek_leja_state* st, double* work, void* stream) {
    (void)check_jv;
    if (k < 1 || k > 8) {
        set_error("ek_leja_update: k=%d out of range", k);
        return EK_ERR_INVALID;
    }
    LejaVArgs a{};
    a.len = len; a.b = jv; a.y = y; a.ynext = ynext; a.nk = k; a.coef = coef_dev;
    a.mi = m - chunk_base; a.m = m; a.gamma = gamma; a.st = st; a.work = work;
    a.repro = g_repro;
    for (int q = 0; q < k; ++q) a.p[q] = p[q];
    k_leja_update<<<vgrid(len), TPB, 0, (cudaStream_t)stream>>>(a);
    EK_LAUNCH_CHECK("k_leja_update");
    return EK_OK;
}

// ------------------------------------------------------------------ power
int ek_power_run(const ek_grid* g, int jac, const double* u, const double* fu, const double* v0,
                 double* const* wbuf, int it_begin, int it_end, ek_power_state* st,
                 double* work, const double* const* halo, void* stream) {
    if (!grid_ok(g)) return EK_ERR_INVALID;
    const int ev = jv_ev(g, jac);
    if (ev < 0) return EK_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t len = ek_grid_len(g);
    // slab mode (halo given): only the stencil passes; the caller runs the
    // norms (ek_power_norm) and the decisions (ek_power_decide) between them
    const bool slab = halo != nullptr;
    if (it_begin == 0 && !slab) {
        // v = v0 / ||v0||   (spectrum.py:49-51): divisor and, for FD, ||v||
        k_power_norm<<<vgrid4(len), TPB, 0, s>>>(len, v0, 0, st, work, g_repro);
        EK_LAUNCH_CHECK("k_power_norm");
        if (jac == EK_JAC_FD) {
            k_power_norm<<<vgrid4(len), TPB, 0, s>>>(len, v0, 1, st, work, g_repro);
            EK_LAUNCH_CHECK("k_power_norm");
        }
    }
    KArgs a;
    base_args(a, g, halo);
    a.u = u; a.fu = fu; a.st = st; a.work = work;
    for (int it = it_begin; it < it_end; ++it) {
        a.y = it == 0 ? v0 : wbuf[(it - 1) & 1];
        a.out = wbuf[it & 1];
        const int rc = launch_stencil<EP_POWER>(ev, a, s);
        if (rc != EK_OK) return rc;
        if (jac == EK_JAC_FD && !slab) {
            k_power_norm<<<vgrid4(len), TPB, 0, s>>>(len, a.out, 1, st, work, g_repro);
            EK_LAUNCH_CHECK("k_power_norm");
        }
    }
    return EK_OK;
}

int ek_power_norm(int64_t len, const double* x, int scaled, ek_power_state* st, double* work,
                  void* stream) {
    k_power_norm<<<vgrid4(len), TPB, 0, (cudaStream_t)stream>>>(len, x, scaled, st, work, g_repro);
    EK_LAUNCH_CHECK("k_power_norm");
    return EK_OK;
}

// ------------------------------------------------------- slab decisions
int ek_leja_decide(ek_leja_state* st, const double* gathered, int nranks, const double* coef_dev,
                   int chunk_base, int m, int k, int fd, int begin, void* stream) {
    k_leja_decide<<<1, 32, 0, (cudaStream_t)stream>>>(st, gathered, nranks, coef_dev,
                                                       m - chunk_base, m, k, fd, begin);
    EK_LAUNCH_CHECK("k_leja_decide");
    return EK_OK;
}

int ek_power_decide(ek_power_state* st, const double* gathered, int nranks, int fd, int which,
                    void* stream) {
    k_power_decide<<<1, 32, 0, (cudaStream_t)stream>>>(st, gathered, nranks, fd, which);
    EK_LAUNCH_CHECK("k_power_decide");
    return EK_OK;
}

// --------------------------------------- slab mode over NVLink peer memory
int ek_leja_run_peer_phase(const ek_grid* g, int jac, const double* u, const double* fu,
                           const double* b, double* const* ybuf, double* const* p, int k,
                           const double* coef_dev, int chunk_base, int m_begin, int m_end,
                           double gamma, ek_leja_state* st, double* work,
                           const double* const* halo_b, const ek_peer* peer,
                           double* win_local, int64_t epoch0, int phase, void* stream);
int64_t ek_peer_window_bytes(const ek_grid* g) {
    if (!grid_ok(g) || g->dim < 2) return 0;
    const int64_t rowlen = g->dim == 2 ? g->n : g->n * g->n;
    return EK_PEER_HALO_OFFSET + 2 * 2 * (int64_t)g->ncomp * rowlen * (int64_t)sizeof(double);
}

int ek_ipc_alloc(int64_t bytes, void** dptr, void* handle64) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    if (bytes <= 0 || !dptr || !handle64) {
        set_error("ek_ipc_alloc: bad arguments");
        return EK_ERR_INVALID;
    }
    cudaError_t e = cudaMalloc(dptr, (size_t)bytes);
    if (e == cudaSuccess) e = cudaMemset(*dptr, 0, (size_t)bytes);
    if (e == cudaSuccess) e = cudaIpcGetMemHandle((cudaIpcMemHandle_t*)handle64, *dptr);
    if (e != cudaSuccess) return cuda_status(e, "ek_ipc_alloc");
    return EK_OK;
}

int ek_ipc_open(const void* handle64, void** dptr) {
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cuda_status(e, "ek_ipc_open");
    return EK_OK;
}

int ek_ipc_close(void* dptr) {
    cudaError_t e = cudaIpcCloseMemHandle(dptr);
    if (e != cudaSuccess) return cuda_status(e, "ek_ipc_close");
    return EK_OK;
}

int ek_ipc_free(void* dptr) {
    cudaError_t e = cudaFree(dptr);
    if (e != cudaSuccess) return cuda_status(e, "ek_ipc_free");
    return EK_OK;
}

int ek_leja_run_peer(const ek_grid* g, int jac, const double* u, const double* fu,
                     const double* b, double* const* ybuf, double* const* p, int k,
                     const double* coef_dev, int chunk_base, int m_begin, int m_end,
                     double gamma, ek_leja_state* st, double* work,
                     const double* const* halo_b, const ek_peer* peer, double* win_local,
                     int64_t epoch0, void* stream) {
    return ek_leja_run_peer_phase(g, jac, u, fu, b, ybuf, p, k, coef_dev, chunk_base, m_begin,
                                  m_end, gamma, st, work, halo_b, peer, win_local, epoch0, 3,
                                  stream);
}

int ek_leja_run_peer_phase(const ek_grid* g, int jac, const double* u, const double* fu,
                           const double* b, double* const* ybuf, double* const* p, int k,
                           const double* coef_dev, int chunk_base, int m_begin, int m_end,
                           double gamma, ek_leja_state* st, double* work,
                           const double* const* halo_b, const ek_peer* peer,
                           double* win_local, int64_t epoch0, int phase, void* stream) {
    if (phase < 1 || phase > 3) {
        set_error("ek_leja_run_peer_phase: phase must be 1 (pass), 2 (decide) or 3");
        return EK_ERR_INVALID;
    }
    if (!grid_ok(g)) return EK_ERR_INVALID;
    if (k < 1 || k > 8 || !peer || !win_local || !halo_b || !g->slab || g->rows < 2 ||
        g->dim < 2) {
        set_error("ek_leja_run_peer: needs a slab grid (rows >= 2), halos, a peer map, 1 <= k <= 8");
        return EK_ERR_INVALID;
    }
    const int ev = jv_ev(g, jac);
    if (ev < 0) return EK_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t rowlen = g->dim == 2 ? g->n : g->n * g->n;
    KArgs a;
    base_args(a, g, halo_b);
    a.u = u; a.fu = fu; a.nk = k; a.coef = coef_dev; a.gamma = mkdv(gamma); a.st = st; a.work = work;
    a.peer = peer;
    for (int q = 0; q < k; ++q) a.p[q] = p[q];
    for (int m = m_begin; m < m_end; ++m) {
        const int64_t e = epoch0 + (m - m_begin);
        a.m = m;
        a.mi = m - chunk_base;
        a.epoch = (long)e;
        a.y = (m == 1) ? b : ybuf[(m - 1) & 1];
        a.out = ybuf[m & 1];
        // ghost rows of y_{m-1}: exchanged once for b, else written into the
        // own window by the neighbours' previous pass
        a.hy = (m == 1) ? halo_b[1]
                        : (const double*)((const char*)win_local + EK_PEER_HALO_OFFSET) +
                              (e & 1) * 2 * (int64_t)g->ncomp * rowlen;
        if (phase & 1) {
            const int rc = launch_stencil<EP_LEJA>(ev, a, s);
            if (rc != EK_OK) return rc;
        }
        if (phase & 2) {
            k_peer_decide<<<1, 32, 0, s>>>(st, peer, (long)e, coef_dev, m - chunk_base, m, k,
                                           jac == EK_JAC_FD ? 1 : 0);
            EK_LAUNCH_CHECK("k_peer_decide");
        }
    }
    return EK_OK;
}

// ------------------------------------------------------------------ KIOPS
int ek_arnoldi_init(int64_t n, int p, const double* src, const double* tail_host, double* V0,
                    ek_arnoldi_state* st, double* work, void* stream) {
    if (p < 0 || p > 5) {
        set_error("ek_arnoldi_init: p=%d out of range", p);
        return EK_ERR_INVALID;
    }
    ArnVArgs a{};
    a.repro = g_repro;
    a.n = n; a.p = p; a.src = src; a.w = V0; a.st = st; a.work = work;
    for (int t = 0; t < p; ++t) a.tail0[t] = tail_host[t];
    cudaStream_t s = (cudaStream_t)stream;
    k_arn_init<<<vgrid4(n), TPB, 0, s>>>(a);
    EK_LAUNCH_CHECK("k_arn_init");
    a.jj = 0;
    k_arn_scale<<<vgrid4(n + p), TPB, 0, s>>>(a);
    EK_LAUNCH_CHECK("k_arn_scale");
    return EK_OK;
}

static void arn_window(ArnVArgs& a, double* const* V, int jj, int iop) {
    const int lo = jj - iop > 0 ? jj - iop : 0;
    a.nwin = jj - lo;
    for (int q = 0; q < a.nwin; ++q) a.win[q] = V[lo + q];
}

int ek_arnoldi_run(const ek_grid* g, int jac, const double* u, const double* fu,
                   double* const* V, const double* const* aug, const int* aug_tail, int naug,
                   double aug_scale, int j_begin, int j_end, double* H, ek_arnoldi_state* st, int p, int iop,
                   int ldh, double dt, double* work, void* stream) {
    if (!grid_ok(g)) return EK_ERR_INVALID;
    if (iop < 1 || iop > 4 || p < 1 || p > 5 || naug > 5 || iop + naug > 8) {
        set_error("ek_arnoldi_run: iop=%d p=%d naug=%d out of range", iop, p, naug);
        return EK_ERR_INVALID;
    }
    const int ev = jv_ev(g, jac);
    if (ev < 0) return EK_ERR_UNSUPPORTED;
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = ek_grid_len(g);
    KArgs a;
    base_args(a, g, nullptr);
    a.u = u; a.fu = fu; a.st = st; a.work = work; a.H = H; a.ldh = ldh; a.dt = dt;
    a.n_aug = p; a.naug = naug; a.aug_scale = aug_scale;
    for (int t = 0; t < naug; ++t) {
        a.aug[t] = aug[t];
        a.aug_tail[t] = aug_tail[t];
    }
    ArnVArgs b{};
    b.repro = g_repro;
    b.n = n; b.p = p; b.H = H; b.ldh = ldh; b.st = st; b.work = work;
    for (int jj = j_begin + 1; jj <= j_end; ++jj) {
        ArnVArgs w{};
        arn_window(w, V, jj, iop);
        a.nwin = w.nwin;
        for (int q = 0; q < 4; ++q) a.win[q] = w.win[q];
        a.jj = jj;
        a.y = V[jj - 1];
        a.out = V[jj];
        int rc = launch_stencil<EP_ARN>(ev, a, s);
        if (rc != EK_OK) return rc;
        b.nwin = w.nwin;
        for (int q = 0; q < 4; ++q) b.win[q] = w.win[q];
        b.jj = jj;
        b.w = V[jj];
        k_arn_orth<<<vgrid4(n + p), TPB, 0, s>>>(b);
        EK_LAUNCH_CHECK("k_arn_orth");
        k_arn_scale<<<vgrid4(n + p), TPB, 0, s>>>(b);
        EK_LAUNCH_CHECK("k_arn_scale");
    }
    return EK_OK;
}

int ek_arnoldi_slab_init(int64_t n, int p, const double* src, const double* tail_host,
                         double* V0, ek_arnoldi_state* st, double* work, void* stream) {
    if (p < 0 || p > 5) {
        set_error("ek_arnoldi_slab_init: p=%d out of range", p);
        return EK_ERR_INVALID;
    }
    ArnVArgs a{};
    a.repro = g_repro;
    a.n = n; a.p = p; a.src = src; a.w = V0; a.st = st; a.work = work;
    for (int t = 0; t < p; ++t) a.tail0[t] = tail_host[t];
    k_arn_init<<<vgrid4(n), TPB, 0, (cudaStream_t)stream>>>(a);
    EK_LAUNCH_CHECK("k_arn_init");
    return EK_OK;
}

int ek_arnoldi_slab_pass(const ek_grid* g, int jac, const double* u, const double* fu,
                         double* const* V, const double* const* aug, const int* aug_tail,
                         int naug, double aug_scale, int jj, int phase, double* H,
                         ek_arnoldi_state* st, int p, int iop, int ldh, double dt,
                         double* work, const double* const* halo, void* stream) {
    if (!grid_ok(g)) return EK_ERR_INVALID;
    if (iop < 1 || iop > 4 || p < 1 || p > 5 || naug > 5 || iop + naug > 8 || phase < 0 ||
        phase > 2 || jj < 0 || (phase < 2 && jj < 1)) {
        set_error("ek_arnoldi_slab_pass: iop=%d p=%d naug=%d phase=%d jj=%d out of range", iop,
                  p, naug, phase, jj);
        return EK_ERR_INVALID;
    }
    cudaStream_t s = (cudaStream_t)stream;
    const int64_t n = ek_grid_len(g);
    ArnVArgs b{};
    b.repro = g_repro;
    b.n = n; b.p = p; b.H = H; b.ldh = ldh; b.st = st; b.work = work; b.jj = jj;
    if (jj > 0) arn_window(b, V, jj, iop);
    b.w = V[jj];
    if (phase == 0) {
        const int ev = jv_ev(g, jac);
        if (ev < 0) return EK_ERR_UNSUPPORTED;
        KArgs a;
        base_args(a, g, halo);
        a.u = u; a.fu = fu; a.st = st; a.work = work; a.H = H; a.ldh = ldh; a.dt = dt;
        a.n_aug = p; a.naug = naug; a.aug_scale = aug_scale;
        for (int t = 0; t < naug; ++t) {
            a.aug[t] = aug[t];
            a.aug_tail[t] = aug_tail[t];
        }
        a.nwin = b.nwin;
        for (int q = 0; q < 4; ++q) a.win[q] = b.win[q];
        a.jj = jj;
        a.y = V[jj - 1];
        a.out = V[jj];
        return launch_stencil<EP_ARN>(ev, a, s);
    }
    if (phase == 1) {
        k_arn_orth<<<vgrid4(n + p), TPB, 0, s>>>(b);
        EK_LAUNCH_CHECK("k_arn_orth");
    } else {
        k_arn_scale<<<vgrid4(n + p), TPB, 0, s>>>(b);
        EK_LAUNCH_CHECK("k_arn_scale");
    }
    return EK_OK;
}

int ek_arnoldi_slab_decide(double* const* V, int64_t n, int p, int jj, int iop, double* H,
                           int ldh, ek_arnoldi_state* st, const double* gathered, int nranks,
                           int which, void* stream) {
    if (which < 0 || which > 3 || nranks < 1 || p < 0 || p > 5) {
        set_error("ek_arnoldi_slab_decide: which=%d nranks=%d p=%d", which, nranks, p);
        return EK_ERR_INVALID;
    }
    ArnVArgs b{};
    b.repro = g_repro;
    b.n = n; b.p = p; b.H = H; b.ldh = ldh; b.st = st; b.jj = jj;
    if (jj > 0) arn_window(b, V, jj, iop);
    b.w = V[jj];
    k_arn_decide<<<1, 32, 0, (cudaStream_t)stream>>>(b, gathered, nranks, which);
    EK_LAUNCH_CHECK("k_arn_decide");
    return EK_OK;
}

int ek_arnoldi_augment(int64_t n, int p, const double* jv, double* const* V, int jj, int iop,
                       const double* const* aug, const int* aug_tail, int naug, double aug_scale,
                       double* H, int ldh,
                       ek_arnoldi_state* st, double* work, void* stream) {
    if (iop < 1 || iop > 4 || p < 1 || p > 5 || naug > 5) {
        set_error("ek_arnoldi_augment: iop=%d p=%d naug=%d out of range", iop, p, naug);
        return EK_ERR_INVALID;
    }
    ArnVArgs a{};
    a.repro = g_repro;
    a.n = n; a.p = p; a.jv = jv; a.H = H; a.ldh = ldh; a.st = st; a.work = work; a.jj = jj;
    a.naug = naug; a.aug_scale = aug_scale;
    for (int t = 0; t < naug; ++t) {
        a.aug[t] = aug[t];
        a.aug_tail[t] = aug_tail[t];
    }
    arn_window(a, V, jj, iop);
    a.w = V[jj];
    k_arn_augment<<<vgrid(n), TPB, 0, (cudaStream_t)stream>>>(a);
    EK_LAUNCH_CHECK("k_arn_augment");
    return EK_OK;
}

int ek_arnoldi_orth(int64_t n, int p, double* const* V, int jj, int iop, double* H, int ldh,
                    ek_arnoldi_state* st, double* work, void* stream) {
    ArnVArgs a{};
    a.repro = g_repro;
    a.n = n; a.p = p; a.H = H; a.ldh = ldh; a.st = st; a.work = work; a.jj = jj;
    arn_window(a, V, jj, iop);
    a.w = V[jj];
    cudaStream_t s = (cudaStream_t)stream;
    k_arn_orth<<<vgrid4(n + p), TPB, 0, s>>>(a);
    EK_LAUNCH_CHECK("k_arn_orth");
    k_arn_scale<<<vgrid4(n + p), TPB, 0, s>>>(a);
    EK_LAUNCH_CHECK("k_arn_scale");
    return EK_OK;
}

int ek_basis_combine(int64_t n, double* const* V, const double* coef_host, int j, double* out,
                     void* stream) {
    if (j < 1 || j > MAXB) {
        set_error("ek_basis_combine: j=%d out of range", j);
        return EK_ERR_INVALID;
    }
    CombineArgs a;
    memset(&a, 0, sizeof(a));
    a.n = n; a.j = j; a.out = out;
    for (int i = 0; i < j; ++i) {
        a.rows[i] = V[i];
        a.coef[i] = coef_host[i];
    }
    k_basis_combine<<<vgrid4(n), TPB, 0, (cudaStream_t)stream>>>(a);
    EK_LAUNCH_CHECK("k_basis_combine");
    return EK_OK;
}

// ---------------------------------------------------------------- vectors
int ek_vexpr(int64_t len, const int32_t* prog, int nprog, const double* scal, int nscal,
             const double* const* in, int nin, double* const* out, int nout,
             ek_scalar_state* st, double* work, void* stream) {
    if (nprog < 1 || nprog > VX_MAXPROG || nscal > 16 || nin > 8 || nout > 4) {
        set_error("ek_vexpr: program too large (nprog=%d nscal=%d nin=%d nout=%d)", nprog,
                  nscal, nin, nout);
        return EK_ERR_INVALID;
    }
    VexprArgs a;
    memset(&a, 0, sizeof(a));
    a.len = len; a.nprog = nprog; a.st = st; a.work = work;
    a.repro = g_repro;
    int reduce = 0;
    for (int i = 0; i < nprog; ++i) {
        a.prog[i] = prog[i];
        const int op = prog[i] & 0xff;
        if (op == VX_NORM || op == VX_CHECK || op == VX_ACC) reduce = 1;
    }
    if (reduce && (!st || !work)) {
        set_error("ek_vexpr: reducing program needs a state block and workspace");
        return EK_ERR_INVALID;
    }
    a.reduce = reduce;
    for (int i = 0; i < nscal; ++i) a.scal[i] = scal[i];
    for (int i = 0; i < nin; ++i) a.in[i] = in[i];
    for (int i = 0; i < nout; ++i) a.out[i] = out[i];
    k_vexpr<<<vgrid(len), TPB, 0, (cudaStream_t)stream>>>(a);
    EK_LAUNCH_CHECK("k_vexpr");
    return EK_OK;
}

int ek_norm2(int64_t len, const double* x, ek_scalar_state* st, int slot, double* work,
             void* stream) {
    if (slot < 0 || slot > 6) {
        set_error("ek_norm2: slot %d", slot);
        return EK_ERR_INVALID;
    }
    k_norm2<<<vgrid4(len), TPB, 0, (cudaStream_t)stream>>>(len, x, nullptr, st, slot, work, g_repro);
    EK_LAUNCH_CHECK("k_norm2");
    return EK_OK;
}

int ek_l1(int64_t len, const double* x, ek_scalar_state* st, int slot, double* work,
          void* stream) {
    k_l1<<<vgrid4(len), TPB, 0, (cudaStream_t)stream>>>(len, x, st, slot, work);
    EK_LAUNCH_CHECK("k_l1");
    return EK_OK;
}

int ek_lincomb(int64_t len, const double* const* in, int nin, double* const* out, int nout,
               const int32_t* nterm, const int32_t* src, const int32_t* mode, const double* coef,
               const double* coef2, const int32_t* fin, const double* fval, int rmode,
               ek_scalar_state* st, double* work, void* stream) {
    if (nin < 1 || nin > LC_IN || nout < 1 || nout > LC_OUT) {
        set_error("ek_lincomb: nin=%d nout=%d out of range", nin, nout);
        return EK_ERR_INVALID;
    }
    LincombArgs a;
    memset(&a, 0, sizeof(a));
    a.len = len;
    a.nout = nout;
    a.repro = g_repro;
    for (int i = 0; i < nin; ++i) a.in[i] = in[i];
    for (int o = 0; o < nout; ++o) {
        a.out[o] = out[o];
        a.nterm[o] = nterm[o];
        if (nterm[o] < 1 || nterm[o] > LC_TERMS) {
            set_error("ek_lincomb: %d terms", nterm[o]);
            return EK_ERR_INVALID;
        }
        for (int t = 0; t < nterm[o]; ++t) {
            const int k = o * LC_TERMS + t;
            if (src[k] < 0 || src[k] >= nin) {
                set_error("ek_lincomb: bad source %d", src[k]);
                return EK_ERR_INVALID;
            }
            a.src[o][t] = src[k];
            a.mode[o][t] = mode[k];
            if (mode[k] == LT_MUL2 && !coef2) {
                set_error("ek_lincomb: mode 3 needs coef2");
                return EK_ERR_INVALID;
            }
            a.coef[o][t] = mode[k] == LT_DIV    ? mkdv(coef[k])
                         : mode[k] == LT_MUL2 ? Dv{coef[k], coef2[k]}
                                              : Dv{coef[k], 0.0};
        }
        a.fin[o] = fin[o];
        a.fval[o] = fin[o] == 2 ? mkdv(fval[o]) : Dv{fval[o], 0.0};
    }
    if (rmode && (!st || !work || (rmode == 2 && nout < 2))) {
        set_error("ek_lincomb: reduction mode %d needs a state block, workspace (and 2 outputs)",
                  rmode);
        return EK_ERR_INVALID;
    }
    a.reduce = rmode;
    a.st = st;
    a.work = work;
    cudaStream_t s = (cudaStream_t)stream;
    const int g = vgrid((len + 3) / 4);  // 4 elements per thread and iteration
    bool aligned = true;
    for (int i = 0; i < nin; ++i) aligned = aligned && al16(in[i]);
    for (int o = 0; o < nout; ++o) aligned = aligned && (!out[o] || al16(out[o]));
    if (aligned) {
        if (nout == 1) k_lincomb<1, true><<<g, TPB, 0, s>>>(a);
        else if (nout == 2) k_lincomb<2, true><<<g, TPB, 0, s>>>(a);
        else k_lincomb<3, true><<<g, TPB, 0, s>>>(a);
    } else {
        if (nout == 1) k_lincomb<1, false><<<g, TPB, 0, s>>>(a);
        else if (nout == 2) k_lincomb<2, false><<<g, TPB, 0, s>>>(a);
        else k_lincomb<3, false><<<g, TPB, 0, s>>>(a);
    }
    EK_LAUNCH_CHECK("k_lincomb");
    return EK_OK;
}

int ek_selftest_div(int64_t n, const double* x, const double* d, double* fast, double* exact,
                    void* stream) {
    k_selftest_div<<<vgrid(n), TPB, 0, (cudaStream_t)stream>>>(n, x, d, fast, exact);
    EK_LAUNCH_CHECK("k_selftest_div");
    return EK_OK;
}

// Order-independent sum self-test: the sum of x (sq = 1: of its squares) by
// a grid of `blocks` blocks, through the kernels' own reduce_grid path.
// out_slots[EK_XSLOTS] (device) receives the merged accumulator, st->val[0]
// its value.
__global__ void __launch_bounds__(TPB) k_selftest_xsum(int64_t n, const double* __restrict__ x,
                                                       int sq, ek_scalar_state* st,
                                                       long long* out_slots, double* work) {
    double acc[1] = {0.0};
    XAcc xs[1];
    xzero(xs[0]);
    for (int64_t e = (int64_t)blockIdx.x * TPB + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * TPB) {
        if (sq) xadd<false>(xs[0], x[e] * x[e]);
        else xadd<true>(xs[0], x[e]);
    }
    double tot[1];
    XAcc xt[1];
    if (reduce_grid<1, 1>(acc, xs, true, work, &st->ticket, false, tot, xt)) {
        if (threadIdx.x == 0) {
            st->val[0] = tot[0];
            xstore(out_slots, xt[0]);
        }
    }
}

int ek_selftest_xsum(int64_t n, const double* x, int sq, int blocks, ek_scalar_state* st,
                     int64_t* out_slots, void* stream) {
    if (n < 0 || blocks < 1 || blocks > VGRID_MAX || !st || !out_slots) {
        set_error("ek_selftest_xsum: bad arguments");
        return EK_ERR_INVALID;
    }
    double* work = nullptr;
    if (cudaMalloc(&work, (size_t)blocks * (1 + XSLOTS) * sizeof(double)) != cudaSuccess)
        return cuda_status(cudaGetLastError(), "ek_selftest_xsum");
    k_selftest_xsum<<<blocks, TPB, 0, (cudaStream_t)stream>>>(n, x, sq, st, (long long*)out_slots,
                                                              work);
    cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
    cudaFree(work);
    if (e != cudaSuccess) return cuda_status(e, "ek_selftest_xsum");
    return EK_OK;
}

int ek_dense_gemv(int64_t n, const double* A, const double* x, double* y, void* stream) {
    const int64_t warps = n;
    const int64_t blocks = (warps * 32 + TPB - 1) / TPB;
    k_dense_gemv<<<(unsigned)blocks, TPB, 0, (cudaStream_t)stream>>>(n, A, x, y);
    EK_LAUNCH_CHECK("k_dense_gemv");
    return EK_OK;
}


// ------------------------------------------------------------ handle layer

struct ek_ctx {
    int device;
    cudaStream_t stream;
};

struct ek_op {
    ek_ctx* ctx;
    ek_grid g;
    int jac;
    double* work;            // device workspace (block partials)
    ek_scalar_state* st;     // device scalar state
    const double* u;         // linearisation point (caller-owned)
    const double* fu;
    double nu;               // ||u||
};

ek_ctx* ek_ctx_create(int device, void* stream) {
    if (cudaSetDevice(device) != cudaSuccess) {
        set_error("ek_ctx_create: cudaSetDevice(%d) failed", device);
        return nullptr;
    }
    ek_ctx* c = new ek_ctx;
    c->device = device;
    c->stream = (cudaStream_t)stream;
    return c;
}

void ek_ctx_destroy(ek_ctx* ctx) { delete ctx; }

ek_op* ek_op_create(ek_ctx* ctx, const ek_grid* g, int jac) {
    if (!ctx || !grid_ok(g) || (jac != EK_JAC_FD && jac != EK_JAC_ANALYTIC)) {
        if (ctx && grid_ok(g)) set_error("ek_op_create: jac=%d", jac);
        return nullptr;
    }
    if (jac == EK_JAC_ANALYTIC && jv_ev(g, jac) < 0) {
        set_error("ek_op_create: problem %d has no analytic Jacobian", g->problem);
        return nullptr;
    }
    ek_op* op = new ek_op{};
    op->ctx = ctx;
    op->g = *g;
    op->jac = jac;
    if (cudaMalloc(&op->work, ek_workspace_bytes(g)) != cudaSuccess ||
        cudaMalloc(&op->st, sizeof(ek_scalar_state)) != cudaSuccess ||
        cudaMemsetAsync(op->st, 0, sizeof(ek_scalar_state), ctx->stream) != cudaSuccess) {
        set_error("ek_op_create: device allocation failed");
        cudaFree(op->work);
        cudaFree(op->st);
        delete op;
        return nullptr;
    }
    return op;
}

void ek_op_destroy(ek_op* op) {
    if (!op) return;
    cudaStreamSynchronize(op->ctx->stream);
    cudaFree(op->work);
    cudaFree(op->st);
    delete op;
}

// read the scalar state block back (syncs the operator's stream)
static int read_state(ek_op* op, ek_scalar_state* h) {
    if (cudaMemcpyAsync(h, op->st, sizeof(*h), cudaMemcpyDeviceToHost, op->ctx->stream) !=
            cudaSuccess ||
        cudaStreamSynchronize(op->ctx->stream) != cudaSuccess) {
        set_error("ek_op: state read failed: %s", cudaGetErrorString(cudaGetLastError()));
        return EK_ERR_CUDA;
    }
    return EK_OK;
}

int ek_op_linearize(ek_op* op, const double* u, double* fu, double* out_norm_u_host) {
    if (!op || !u || !fu) return EK_ERR_INVALID;
    const int64_t n = ek_grid_len(&op->g);
    int rc = ek_rhs(&op->g, u, fu, nullptr, op->ctx->stream);
    if (rc != EK_OK) return rc;
    rc = ek_norm2(n, u, op->st, 0, op->work, op->ctx->stream);
    if (rc != EK_OK) return rc;
    ek_scalar_state h;
    if ((rc = read_state(op, &h)) != EK_OK) return rc;
    op->u = u;
    op->fu = fu;
    op->nu = h.val[1];
    if (out_norm_u_host) *out_norm_u_host = op->nu;
    return EK_OK;
}

int ek_op_rhs(ek_op* op, const double* u, double* out) {
    if (!op) return EK_ERR_INVALID;
    return ek_rhs(&op->g, u, out, nullptr, op->ctx->stream);
}

int ek_op_jv(ek_op* op, const double* v, double* out) {
    if (!op || !op->u) {
        set_error("ek_op_jv: operator not linearised");
        return EK_ERR_INVALID;
    }
    cudaStream_t s = op->ctx->stream;
    if (op->jac == EK_JAC_ANALYTIC)
        return ek_jv(&op->g, op->jac, op->u, op->fu, v, 0.0, out, nullptr, op->work, nullptr, s);
    const int64_t n = ek_grid_len(&op->g);
    int rc = ek_norm2(n, v, op->st, 0, op->work, s);
    if (rc != EK_OK) return rc;
    ek_scalar_state h;
    if ((rc = read_state(op, &h)) != EK_OK) return rc;
    const double nv = h.val[1];
    if (nv == 0.0) {  // linalg.py:121-122
        set_error("ek_op_jv: cannot form a finite-difference step for a zero vector");
        return EK_ERR_INVALID;
    }
    const double eps = (SQRT_EPS * (1.0 + op->nu)) / nv;  // linalg.py:123-124
    if (cudaMemsetAsync(&op->st->flag, 0, sizeof(int32_t), s) != cudaSuccess) return EK_ERR_CUDA;
    rc = ek_jv(&op->g, op->jac, op->u, op->fu, v, eps, out, op->st, op->work, nullptr, s);
    if (rc != EK_OK) return rc;
    if ((rc = read_state(op, &h)) != EK_OK) return rc;
    if (h.flag & 2) {  // linalg.py:127-128
        set_error("ek_op_jv: non-finite Jacobian action");
        return EK_ERR_NONFINITE;
    }
    return EK_OK;
}

int ek_power_step(ek_op* op, const double* v, double* w, double* norm_out_host) {
    int rc = ek_op_jv(op, v, w);
    if (rc != EK_OK) return rc;
    rc = ek_norm2(ek_grid_len(&op->g), w, op->st, 0, op->work, op->ctx->stream);
    if (rc != EK_OK) return rc;
    ek_scalar_state h;
    if ((rc = read_state(op, &h)) != EK_OK) return rc;
    if (norm_out_host) *norm_out_host = h.val[1];
    return EK_OK;
}

int ek_axpby(int64_t n, double a, const double* x, double b, const double* y, double* out,
             void* stream) {
    if (n < 0 || !x || !y || !out) return EK_ERR_INVALID;
    if (n == 0) return EK_OK;
    k_axpby<<<vgrid4(n), TPB, 0, (cudaStream_t)stream>>>(n, a, x, b, y, out);
    EK_LAUNCH_CHECK("k_axpby");
    return EK_OK;
}

int ek_dot_multi(int64_t n, const double* x, const double* const* ys, int k, ek_scalar_state* st,
                 double* out_host, double* work, void* stream) {
    if (n < 1 || k < 1 || k > 8 || !x || !ys || !st || !work) {
        set_error("ek_dot_multi: bad arguments (n=%lld, k=%d)", (long long)n, k);
        return EK_ERR_INVALID;
    }
    DotArgs a{};
    a.n = n; a.x = x; a.k = k; a.st = st; a.work = work;
    for (int q = 0; q < k; ++q) a.y[q] = ys[q];
    cudaStream_t s = (cudaStream_t)stream;
    k_dot_multi<<<vgrid4(n), TPB, 0, s>>>(a);
    EK_LAUNCH_CHECK("k_dot_multi");
    if (out_host) {
        ek_scalar_state h;
        if (cudaMemcpyAsync(&h, st, sizeof(h), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
            cudaStreamSynchronize(s) != cudaSuccess) {
            set_error("ek_dot_multi: read back failed");
            return EK_ERR_CUDA;
        }
        for (int q = 0; q < k; ++q) out_host[q] = h.val[q];
    }
    return EK_OK;
}

}  // extern "C"
