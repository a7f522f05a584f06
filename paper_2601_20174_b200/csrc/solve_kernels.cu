// paper_2601_20174_b200/csrc/solve_kernels.cu — the PCG hot loop on sm_100a.
//
// Three schedules of one PCG iteration (two_level.hpp:141-191) with the
// two-level operator (two_level.hpp:60-81), all applying the same operator
// (DESIGN.md §3); every reduction is finished in a fixed order by the last CTA
// to arrive (deterministic, no fp64 atomics):
//
//   one-pass (default, nu1 = nu2, k <= 64), three kernels at nu = 1/1:
//     k_spmv_dia / k_spmv_tma <OpSpmvP>     p = z + beta p in the gather, q = A p, p.q -> alpha
//     k_spmv_dia / k_spmv_tma <OpUpdSweep>  x, r' = r - alpha q (in the gather), s = S_2(r'),
//                                           ||r'|| -> convergence; last CTA: c by its
//                                           recurrence, e = A_c^-1 c
//     k_prolong_onepass_tma                 z = s + W e with u = W^T r, v = W^T A s in the
//                                           same pass over W; r.z -> beta, loop control
//   folded (NLSP_CYCLE=folded): W1^T r fused with the x/r update, sweeps,
//     z = s + W2 e (two passes over W) — k_update_restrict_tma, k_prolong
//   literal (NLSP_CYCLE=literal): the reference's op-by-op order — k_update,
//     k_restrict, k_prolong, k_sweep, k_loop_ctl
//
// The matrix is read in its diagonal form when the upload detected one
// (k_spmv_dia, one thread per row) and otherwise from TMA-staged CSR row tiles
// (k_spmv_tma); the row kernels of the literal schedule use groups of 8 lanes
// per CSR / basis row.
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <unordered_map>
#include <utility>

#include "internal.cuh"
#include "tma_rows.cuh"

namespace nlsp {

// rows per 8-lane group in flight: SpMV kernels / kernels that also stream P
#ifndef NLSP_KU
#define NLSP_KU 4
#endif
#ifndef NLSP_KUP
#define NLSP_KUP 2
#endif
#ifndef NLSP_DIA_EXACT
#define NLSP_DIA_EXACT 1
#endif
#ifndef NLSP_DIA_ROWS
#define NLSP_DIA_ROWS 1
#endif
#ifndef NLSP_DIA_MINB
#define NLSP_DIA_MINB 1
#endif
#ifndef NLSP_DIA_BLOCK
#define NLSP_DIA_BLOCK 0
#endif
#ifndef NLSP_KUPRO
#define NLSP_KUPRO 2
#endif
#ifndef NLSP_BLOCKROWS
#define NLSP_BLOCKROWS 0
#endif
// minimum resident CTAs per SM requested from ptxas (register cap) for the
// basis-streaming (P) and the SpMV kernels
#ifndef NLSP_MINB_P
#define NLSP_MINB_P 1
#endif
#ifndef NLSP_MINB_S
#define NLSP_MINB_S 1
#endif
constexpr int kU = NLSP_KU;
constexpr int kUP = NLSP_KUP;

// ----------------------------------------------------------------- gathers --
struct GPlain {
    const double* x;
    __device__ __forceinline__ double operator()(int j) const { return x[j]; }
};
// p_j = z_j + beta p_j (two_level.hpp:182, contracted to one fma), or z_j when
// p is first formed (two_level.hpp:154)
struct GPupd {
    const double* z;
    const double* pp;
    double beta;
    bool first;
    __device__ __forceinline__ double operator()(int j) const {
        return first ? z[j] : fma(beta, pp[j], z[j]);
    }
};
// first pre-sweep from z = 0: z_j = (w dinv_j)(r_j - 0) (smoothing.hpp:40 with x = 0)
// CW: w D^-1 is the constant wc (constant-coefficient diagonal form, bitwise
// equal to every wd[j]), so only r is gathered
template <bool CW = false>
struct GWdrT {
    const double* wd;
    const double* r;
    double wc = 0.0;
    __device__ __forceinline__ double operator()(int j) const { return (CW ? wc : wd[j]) * r[j]; }
};
using GWdr = GWdrT<false>;


// y[u] = sum_k v_k g(col_k) for the U rows row[u] of this 8-lane group; every
// lane of the group returns the full sums. All row_ptr loads, then all
// value/column loads, then all gathers are issued before any use, so a warp
// keeps 4*U rows of CSR traffic in flight.
template <int U, class Gat>
__device__ __forceinline__ void group_dot_batch(const int* __restrict__ rp,
                                                const int* __restrict__ ci,
                                                const double* __restrict__ v, const int (&row)[U],
                                                const bool (&valid)[U], const Gat& g, int l,
                                                double (&y)[U]) {
    int b[U], e[U];
    int len = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        b[u] = valid[u] ? __ldg(rp + row[u]) : 0;
        e[u] = valid[u] ? __ldg(rp + row[u] + 1) : 0;
        y[u] = 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) len = max(len, e[u] - b[u]);
    for (int off = l; off < len; off += kGroup) {
        double vv[U];
        int cc[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = b[u] + off;
            const bool ok = k < e[u];
            vv[u] = ok ? __ldg(v + k) : 0.0;
            cc[u] = ok ? __ldg(ci + k) : -1;
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (cc[u] >= 0) y[u] = fma(vv[u], g(cc[u]), y[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) y[u] = group_sum(y[u]);
}

// CTA sum of NV values, partial per CTA, and the last-arriving CTA reduces all
// partials in a fixed order. Returns true (in every thread) only in the last
// CTA, where tot[] holds the grid-wide sums (valid in all threads).
template <int NV>
__device__ __forceinline__ bool grid_reduce(double (&v)[NV], double* part, unsigned int* counter,
                                            double (&tot)[NV]) {
    __shared__ double sm[NV][32];
    __shared__ double fin[NV];
    __shared__ int is_last;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        const double t = warp_sum(v[j]);
        if (lane == 0) sm[j][warp] = t;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            double t = lane < nw ? sm[j][lane] : 0.0;
            t = warp_sum(t);
            if (lane == 0) part[blockIdx.x * NV + j] = t;
        }
        if (lane == 0) {
            __threadfence();
            const unsigned int tk = atomicAdd(counter, 1u);
            is_last = (tk == gridDim.x - 1);
        }
    }
    __syncthreads();
    if (!is_last) return false;
    __threadfence();
#pragma unroll
    for (int j = 0; j < NV; ++j) {
        double t = 0.0;
        for (int b = threadIdx.x; b < gridDim.x; b += blockDim.x) t += __ldcg(part + b * NV + j);
        t = warp_sum(t);
        if (lane == 0) sm[j][warp] = t;
    }
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int j = 0; j < NV; ++j) {
            double t = lane < nw ? sm[j][lane] : 0.0;
            t = warp_sum(t);
            if (lane == 0) fin[j] = t;
        }
        if (lane == 0) *counter = 0u;
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < NV; ++j) tot[j] = fin[j];
    return true;
}

// Rows are dealt to warps in runs of 4*U; group grp of a warp takes rows
// base + grp + 4u (u < U), so at each u the four groups read one contiguous run
// of nonzeros. With NLSP_BLOCKROWS each CTA owns one contiguous block of rows
// and its warps sweep it in order, so stencil neighbours (i +- 1, i +- nx) of a
// gather were usually just touched by the same CTA (L1 hits).
#if NLSP_BLOCKROWS
#define ROW_BATCH_RANGE(n, U)                                                           \
    const long long step_ = (long long)(blockDim.x >> 5) * (kRowsPerWarp * (U));       \
    const long long per_ = ((((long long)(n) + gridDim.x - 1) / gridDim.x) + step_ - 1) / step_ * step_; \
    const long long beg_ = blockIdx.x * per_;                                           \
    const long long end_ = min((long long)(n), beg_ + per_);                            \
    for (long long base_ = beg_ + (threadIdx.x >> 5) * (kRowsPerWarp * (U)); base_ < end_; \
         base_ += step_) {
#else
#define ROW_BATCH_RANGE(n, U)                                                           \
    const long long wid_ = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;     \
    const long long nwarps_ = (gridDim.x * (long long)blockDim.x) >> 5;                \
    for (long long base_ = wid_ * (kRowsPerWarp * (U)); base_ < (n);                   \
         base_ += nwarps_ * (kRowsPerWarp * (U))) {
#endif
#define ROW_BATCH_BEGIN(n, U)                                                      \
    const int lane_ = threadIdx.x & 31;                                            \
    const int l = lane_ & (kGroup - 1);                                            \
    const int grp = lane_ >> 3;                                                    \
    ROW_BATCH_RANGE(n, U)                                                          \
        int row[U];                                                                \
        bool valid[U];                                                             \
        _Pragma("unroll") for (int u = 0; u < (U); ++u) {                          \
            row[u] = static_cast<int>(base_) + grp + kRowsPerWarp * u;             \
            valid[u] = row[u] < (n);                                               \
        }

#define ROW_BATCH_END }

// ------------------------------------------------------------------ state --
struct PcgParamsHost {
    double delta;
    long long max_it;
};

__global__ void k_state_init(PcgState* st, double delta, long long max_it) {
    st->rz = st->rz_new = st->pap = st->alpha = st->beta = st->rr = 0.0;
    st->bnorm = 0.0;
    st->delta = delta;
    st->true_res = 0.0;
    st->last_rel = 0.0;
    st->it = 0;
    st->max_it = max_it;
    st->hist_base = 0;
    st->drift_max = 0.0;
    st->lean_ce = st->lean_eme = st->pap_pred = st->pap_drift = 0.0;
    st->iterations = 0;
    st->body_runs = 0;
    st->done = 0;
    st->converged = 0;
    st->error = 0;
    st->first = 1;
}

// Next segment of a solve that stopped at its segment end (st->max_it) without
// converging: the loop resumes from the state left by the last iteration, the
// history restarts at hist[0] = iteration `base` (nlsp_gpu.cu run_pcg).
__global__ void k_state_continue(PcgState* st, long long max_it, long long base) {
    st->max_it = max_it;
    st->hist_base = base;
    st->done = 0;
}

// ||b||_2 (two_level.hpp:143-146) and r = b, x = 0; zero rhs -> ValidationError
__global__ void __launch_bounds__(kThreads) k_bnorm(SolveArgs a) {
    double s[1] = {0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.n;
         i += (long long)gridDim.x * blockDim.x) {
        const double bi = a.b[i];
        a.r[i] = bi;
        a.x[i] = 0.0;
        s[0] = fma(bi, bi, s[0]);
    }
    double tot[1];
    if (grid_reduce<1>(s, a.partials, &a.st->counter[kTkBnorm], tot) && threadIdx.x == 0) {
        const double bn = sqrt(tot[0]);
        a.st->bnorm = bn;
        if (bn == 0.0) {
            a.st->error = kErrValidation;
            a.st->done = 1;
        }
    }
}

// z = r (identity) or z = r / A_ii (Jacobi, two_level.hpp:107-118); r.z
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_init_simple(SolveArgs a) {
    if (a.st->done) return;
    double s[1] = {0.0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < a.n;
         i += (long long)gridDim.x * blockDim.x) {
        const double ri = a.r[i];
        // JacobiPreconditioner::apply (two_level.hpp:112-113): a non-positive
        // diagonal is a NumericError, raised after pcg's zero-rhs check
        if (MODE == 1 && !(a.diag[i] > 0.0)) {
            a.st->error = kErrNumeric;
            a.st->done = 1;
        }
        const double zi = MODE == 1 ? ri / a.diag[i] : ri;
        a.z[i] = zi;
        s[0] = fma(ri, zi, s[0]);
    }
    double tot[1];
    if (grid_reduce<1>(s, a.partials, &a.st->counter[kTkInit], tot) && threadIdx.x == 0)
        a.st->rz_new = tot[0];
}

// rz = r.z of the initial apply; the loop starts with p = z (two_level.hpp:153-156)
__global__ void k_init_ctl(PcgState* st) {
    st->rz = st->rz_new;
    st->first = 1;
    st->it = 0;
    if (st->max_it <= 0) st->done = 1;
}

// -------------------------------------------------------------- k_spmv_p --
// p = z + beta p (written to the other ping-pong buffer), q = A p, p.q;
// last CTA: p^T A p <= 0 -> NotSpdError (two_level.hpp:159-163), alpha = rz / pap
__global__ void __launch_bounds__(kThreads, NLSP_MINB_S) k_spmv_p(SolveArgs a) {
    pdl_entry();
    PcgState* st = a.st;
    if (st->done) return;
    const bool odd = st->it & 1;
    const double* pp = odd ? a.p0 : a.p1;
    double* pc = odd ? a.p1 : a.p0;
    const GPupd g{a.z, pp, st->beta, st->first != 0};
    double s[1] = {0.0};
    ROW_BATCH_BEGIN(a.n, kU)
        double y[kU];
        group_dot_batch<kU>(a.rp, a.ci, a.v, row, valid, g, l, y);
        if (l == 0) {
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                if (!valid[u]) continue;
                const double pi = g(row[u]);
                pc[row[u]] = pi;
                a.q[row[u]] = y[u];
                s[0] = fma(pi, y[u], s[0]);
            }
        }
    ROW_BATCH_END
    double tot[1];
    if (grid_reduce<1>(s, a.partials, &st->counter[kTkSpmvP], tot) && threadIdx.x == 0) {
        const double pap = tot[0];
        st->pap = pap;
        if (pap <= 0.0) {
            st->error = kErrNotSpd;
            st->done = 1;
        } else {
            st->alpha = st->rz / pap;
        }
    }
}

// -------------------------------------------------------------- k_update --
// x += alpha p, r -= alpha q (two_level.hpp:164-167), ||r|| / ||b|| into the
// history, convergence test on the recurrence residual (:168-176). MODE 1/2:
// identity / Jacobi preconditioner fused (z and r.z in the same pass).
template <int MODE>
__global__ void __launch_bounds__(kThreads) k_update(SolveArgs a) {
    PcgState* st = a.st;
    if (st->done) return;
    const double alpha = st->alpha;
    const double* p = (st->it & 1) ? a.p1 : a.p0;
    double s[2] = {0.0, 0.0};
    auto one = [&](long long i, double pi, double qi, double xi, double ri0, double& xo,
                   double& ro) {
        xo = fma(alpha, pi, xi);
        ro = fma(-alpha, qi, ri0);
        s[0] = fma(ro, ro, s[0]);
        if (MODE != 0) {
            const double zi = MODE == 2 ? ro / a.diag[i] : ro;
            a.z[i] = zi;
            s[1] = fma(ro, zi, s[1]);
        }
    };
    // 16-B vector loads over element pairs; the odd tail element separately
    const long long npairs = a.n >> 1;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < npairs; t += stride) {
        const long long i = 2 * t;
        const double2 pv = *reinterpret_cast<const double2*>(p + i);
        const double2 qv = *reinterpret_cast<const double2*>(a.q + i);
        const double2 xv = *reinterpret_cast<const double2*>(a.x + i);
        const double2 rv = *reinterpret_cast<const double2*>(a.r + i);
        double2 xo, ro;
        one(i, pv.x, qv.x, xv.x, rv.x, xo.x, ro.x);
        one(i + 1, pv.y, qv.y, xv.y, rv.y, xo.y, ro.y);
        *reinterpret_cast<double2*>(a.x + i) = xo;
        *reinterpret_cast<double2*>(a.r + i) = ro;
    }
    if ((a.n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const long long i = a.n - 1;
        double xo, ro;
        one(i, p[i], a.q[i], a.x[i], a.r[i], xo, ro);
        a.x[i] = xo;
        a.r[i] = ro;
    }
    double tot[2];
    if (grid_reduce<2>(s, a.partials, &st->counter[kTkUpdate], tot) && threadIdx.x == 0) {
        const double rel = sqrt(tot[0]) / st->bnorm;
        st->rr = tot[0];
        st->last_rel = rel;
        a.hist[st->it - st->hist_base] = rel;
        st->iterations = st->it + 1;
        if (rel < st->delta) {
            st->converged = 1;
            st->done = 1;
        }
        if (MODE != 0) st->rz_new = tot[1];
    }
}

// beta = rz' / rz, p-update bookkeeping, iteration advance, graph WHILE control
__device__ __forceinline__ void loop_ctl_body(PcgState* st, cudaGraphConditionalHandle h,
                                              int use_cond) {
    st->body_runs += 1;
    if (!st->done) {
        st->beta = st->rz_new / st->rz;
        st->rz = st->rz_new;
        st->first = 0;
        st->it += 1;
        if (st->it >= st->max_it) st->done = 1;
    }
    if (use_cond && st->done) cudaGraphSetConditional(h, 0);
}

// Lean cycle: beta and r.z were already advanced by the sweep kernel's last CTA
// (beta is needed before the pass over W); the pass only moves r.z on.
__device__ __forceinline__ void loop_ctl_lean(PcgState* st, cudaGraphConditionalHandle h, int use_cond) {
    st->body_runs += 1;
    if (!st->done) {
        st->rz = st->rz_new;
        st->first = 0;
        st->it += 1;
        if (st->it >= st->max_it) st->done = 1;
    }
    if (use_cond && st->done) cudaGraphSetConditional(h, 0);
}

__global__ void k_loop_ctl(PcgState* st, cudaGraphConditionalHandle h, int use_cond) {
    loop_ctl_body(st, h, use_cond);
}

// --------------------------------------------------------------- k_sweep --
// z_out = z_in + (w dinv)(r - A z_in) (smoothing.hpp:34-41, contracted), with
// z_in given by the gather (implicit first sweep or a buffer); RZ: r.z_out
template <class Gat, bool RZ>
__global__ void __launch_bounds__(kThreads, NLSP_MINB_S) k_sweep(SolveArgs a, Gat g, double* zout) {
    pdl_entry();
    PcgState* st = a.st;
    if (st->done) return;
    double s[1] = {0.0};
    ROW_BATCH_BEGIN(a.n, kU)
        double y[kU];
        group_dot_batch<kU>(a.rp, a.ci, a.v, row, valid, g, l, y);
        if (l == 0) {
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                if (!valid[u]) continue;
                const double ri = a.r[row[u]];
                const double zi = fma(a.wd[row[u]], ri - y[u], g(row[u]));
                zout[row[u]] = zi;
                if (RZ) s[0] = fma(ri, zi, s[0]);
            }
        }
    ROW_BATCH_END
    if (RZ) {
        double tot[1];
        if (grid_reduce<1>(s, a.partials, &st->counter[kTkSweep], tot) && threadIdx.x == 0)
            st->rz_new = tot[0];
    }
}

// ----------------------------------------------------- coarse solve (1 warp) --
// L y = c, L^T e = y (cholesky.hpp:41-57), column-oriented so each y_i keeps the
// reference's left-to-right accumulation order in the forward sweep.
__device__ void coarse_solve_warp(const double* __restrict__ L, int k, double* ys, double* e) {
    const int lane = threadIdx.x & 31;
    for (int j = 0; j < k; ++j) {
        __syncwarp();
        const double yj = ys[j] / L[j * k + j];
        __syncwarp();
        if (lane == 0) ys[j] = yj;
        for (int i = j + 1 + lane; i < k; i += 32) ys[i] = fma(-L[i * k + j], yj, ys[i]);
    }
    for (int j = k - 1; j >= 0; --j) {
        __syncwarp();
        const double xj = ys[j] / L[j * k + j];
        __syncwarp();
        if (lane == 0) ys[j] = xj;
        for (int i = lane; i < j; i += 32) ys[i] = fma(-L[j * k + i], xj, ys[i]);
    }
    __syncwarp();
    for (int i = lane; i < k; i += 32) e[i] = ys[i];
}

// e = A_c^-1 c with the whole CTA: 4 lanes per output row, each a strided
// quarter of the dot, combined by shuffles. The k^2 loads of A_c^-1 (L2
// resident) are all in flight at once, where the substitutions above are 2k
// dependent steps of L2 latency each.
__device__ void coarse_apply_inverse(const double* __restrict__ Ainv, int k, const double* ys,
                                     double* e) {
    for (int i0 = 0; i0 < k; i0 += (int)(blockDim.x >> 2)) {
        const int i = i0 + (int)(threadIdx.x >> 2), sub = threadIdx.x & 3;
        double s = 0.0;
        if (i < k)
            for (int j = sub; j < k; j += 4) s = fma(__ldg(Ainv + (long long)i * k + j), ys[j], s);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        if (i < k && sub == 0) e[i] = s;
    }
}

// ------------------------------------------------------------ k_restrict --
// res = r - A z_pre (two_level.hpp:63-67); c = P^T res (:69-72); the last CTA
// sums the per-CTA c partials in a fixed order and solves A_c e = c (:73).
// ZMODE 0: z_pre = 0 (nu1 = 0), 1: z_pre = w D^-1 r implicit (nu1 = 1), 2: buffer.
template <int PPL, int NT, bool RR>
__device__ __forceinline__ void restrict_finish(double (&acc)[2 * PPL], double rr, const SolveArgs& a);

template <int PPL, int ZMODE>
__global__ void __launch_bounds__(kThreads, NLSP_MINB_P) k_restrict(SolveArgs a, const double* zpre) {
    PcgState* st = a.st;
    if (st->done) return;
    const int ld = a.k + (a.k & 1);
    const int pairs = ld >> 1;
    double acc[2 * PPL];
#pragma unroll
    for (int t = 0; t < 2 * PPL; ++t) acc[t] = 0.0;
    const GWdr gw{a.wd, a.r};
    const GPlain gp{zpre};
    ROW_BATCH_BEGIN(a.n, kUP)
        // basis rows first (independent of the SpMV), then the residuals
        double2 pv[kUP][PPL];
#pragma unroll
        for (int u = 0; u < kUP; ++u) {
            const double* prow = a.P + (long long)row[u] * ld;
#pragma unroll
            for (int t = 0; t < PPL; ++t) {
                const int pi = l + kGroup * t;
                pv[u][t] = (valid[u] && pi < pairs) ? ld_stream2(prow + 2 * pi) : make_double2(0.0, 0.0);
            }
        }
        double y[kUP];
#pragma unroll
        for (int u = 0; u < kUP; ++u) y[u] = 0.0;
        if (ZMODE == 1) group_dot_batch<kUP>(a.rp, a.ci, a.v, row, valid, gw, l, y);
        if (ZMODE == 2) group_dot_batch<kUP>(a.rp, a.ci, a.v, row, valid, gp, l, y);
#pragma unroll
        for (int u = 0; u < kUP; ++u) {
            const double res = valid[u] ? a.r[row[u]] - y[u] : 0.0;
#pragma unroll
            for (int t = 0; t < PPL; ++t) {
                acc[2 * t] = fma(pv[u][t].x, res, acc[2 * t]);
                acc[2 * t + 1] = fma(pv[u][t].y, res, acc[2 * t + 1]);
            }
        }
    ROW_BATCH_END
    restrict_finish<PPL, kThreads, false>(acc, 0.0, a);
}

// Restriction epilogue shared by the restriction kernels: per-lane partials
// -> CTA partial -> fixed-order grid sum in the last CTA -> coarse solve. With
// RR the CTA also carries ||r||^2 (fused update): the last CTA writes the
// history entry and runs the convergence test (two_level.hpp:168-176) first.
template <int PPL, int NT, bool RR>
__device__ __forceinline__ void restrict_finish(double (&acc)[2 * PPL], double rr, const SolveArgs& a) {
    PcgState* st = a.st;
    constexpr int CMAX = 2 * 8 * PPL + 1;
    __shared__ double cs[NT / 32][CMAX];
    __shared__ double red[NT + CMAX];
    __shared__ double ys[CMAX];
    const int ld = a.k + (a.k & 1);
    const int pairs = ld >> 1;
    const int wc = ld + (RR ? 1 : 0);  // partial columns
    // groups of a warp -> lanes 0..7, warps -> shared, CTA partial -> global
#pragma unroll
    for (int t = 0; t < 2 * PPL; ++t) {
        acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], 8);
        acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], 16);
    }
    if (RR) rr = warp_sum(rr);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (lane < kGroup) {
#pragma unroll
        for (int t = 0; t < PPL; ++t) {
            const int pi = lane + kGroup * t;
            if (pi < pairs) {
                cs[warp][2 * pi] = acc[2 * t];
                cs[warp][2 * pi + 1] = acc[2 * t + 1];
            }
        }
    }
    if (RR && lane == 0) cs[warp][ld] = rr;
    __syncthreads();
    for (int c = threadIdx.x; c < wc; c += blockDim.x) {
        double t = 0.0;
        for (int w = 0; w < nw; ++w) t += cs[w][c];
        a.partials[(long long)blockIdx.x * wc + c] = t;
    }
    __shared__ int is_last;
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned int tk = atomicAdd(&st->counter[kTkRestrict], 1u);
        is_last = (tk == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    // fixed-order grid sum: S slices of CTAs per column, then slices in order
    const int S = max(1, (int)blockDim.x / wc);
    // (loads batched 8 deep so a slice costs ceil(G / 8S) L2 round trips, not
    // G / S; the sum order is unchanged)
    for (int idx = threadIdx.x; idx < S * wc; idx += blockDim.x) {
        const int c = idx % wc, sl = idx / wc;
        double t = 0.0;
        for (int b = sl; b < (int)gridDim.x; b += 8 * S) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int bb = b + u * S;
                v[u] = bb < (int)gridDim.x ? __ldcg(a.partials + (long long)bb * wc + c) : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) t += v[u];
        }
        red[idx] = t;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < wc; c += blockDim.x) {
        double t = 0.0;
        for (int q = 0; q < S; ++q) t += red[q * wc + c];
        ys[c] = t;
    }
    __syncthreads();
    if (RR && threadIdx.x == 0) {
        const double rel = sqrt(ys[ld]) / st->bnorm;
        st->rr = ys[ld];
        st->last_rel = rel;
        a.hist[st->it - st->hist_base] = rel;
        st->iterations = st->it + 1;
        if (rel < st->delta) {
            st->converged = 1;
            st->done = 1;
        }
    }
    // c itself: the lean cycle's prologue forms r.z = r.s + c.e from it
    if (a.ow && a.k <= kOnePassK) {
        for (int c = threadIdx.x; c < a.k; c += blockDim.x) a.ow[3 * ld + c] = ys[c];
        __syncthreads();
    }
    if (a.Ainv) {
        coarse_apply_inverse(a.Ainv, a.k, ys, a.e);
        if (threadIdx.x == 0) {
            if (a.k & 1) a.e[a.k] = 0.0;  // padded column
            st->counter[kTkRestrict] = 0u;
        }
    } else if (warp == 0) {
        coarse_solve_warp(a.L, a.k, ys, a.e);
        if (lane == 0) {
            if (a.k & 1) a.e[a.k] = 0.0;  // padded column
            st->counter[kTkRestrict] = 0u;
        }
    }
}

// ------------------------------------------------------------- k_prolong --
// z = z_pre + P e (two_level.hpp:74-78); RZ: r.z when no post-sweep follows
template <int PPL, int ZMODE, bool RZ>
__global__ void __launch_bounds__(kThreads) k_prolong(SolveArgs a, const double* zpre,
                                                      double* zout, cudaGraphConditionalHandle h,
                                                      int ctl) {
    // ctl > 0: this is the last kernel of an iteration and also does the loop
    // control of k_loop_ctl (ctl == 2: inside the graph WHILE body)
    PcgState* st = a.st;
    if (st->done) {
        if (ctl && blockIdx.x == 0 && threadIdx.x == 0) loop_ctl_body(st, h, ctl == 2);
        return;
    }
    const int ld = a.k + (a.k & 1);
    const int pairs = ld >> 1;
    double ev[2 * PPL];
    {
        const int l0 = threadIdx.x & (kGroup - 1);
#pragma unroll
        for (int t = 0; t < PPL; ++t) {
            const int pi = l0 + kGroup * t;
            ev[2 * t] = pi < pairs ? a.e[2 * pi] : 0.0;
            ev[2 * t + 1] = pi < pairs ? a.e[2 * pi + 1] : 0.0;
        }
    }
    double s[1] = {0.0};
    constexpr int UPR = NLSP_KUPRO;
    ROW_BATCH_BEGIN(a.n, UPR)
        // the row's scalars first (independent of the basis stream), then the
        // W2 rows, so both are in flight together
        double zpv[UPR], rrv[UPR];
#pragma unroll
        for (int u = 0; u < UPR; ++u) {
            const int rw = valid[u] ? row[u] : 0;
            if (ZMODE == 0) zpv[u] = 0.0;
            else if (ZMODE == 1) zpv[u] = a.wd[rw] * a.r[rw];
            else zpv[u] = zpre[rw];
            rrv[u] = RZ ? a.r[rw] : 0.0;
        }
        double2 pv[UPR][PPL];
#pragma unroll
        for (int u = 0; u < UPR; ++u) {
            const double* prow = a.P + (long long)row[u] * ld;
#pragma unroll
            for (int t = 0; t < PPL; ++t) {
                const int pi = l + kGroup * t;
                pv[u][t] = (valid[u] && pi < pairs) ? ld_stream2(prow + 2 * pi) : make_double2(0.0, 0.0);
            }
        }
        double sum[UPR];
#pragma unroll
        for (int u = 0; u < UPR; ++u) {
            double part = 0.0;
#pragma unroll
            for (int t = 0; t < PPL; ++t) {
                part = fma(pv[u][t].x, ev[2 * t], part);
                part = fma(pv[u][t].y, ev[2 * t + 1], part);
            }
            sum[u] = group_sum(part);
        }
        if (l == 0) {
#pragma unroll
            for (int u = 0; u < UPR; ++u) {
                if (!valid[u]) continue;
                const double zi = zpv[u] + sum[u];
                zout[row[u]] = zi;
                if (RZ) s[0] = fma(rrv[u], zi, s[0]);
            }
        }
    ROW_BATCH_END
    if (RZ) {
        double tot[1];
        if (grid_reduce<1>(s, a.partials, &st->counter[kTkProlong], tot) && threadIdx.x == 0) {
            st->rz_new = tot[0];
            if (ctl) loop_ctl_body(st, h, ctl == 2);
        }
    }
}

// ----------------------------------------------------------- k_true_res --
// ||b - A x|| / ||b|| recomputed at exit (two_level.hpp:185-189)
__global__ void __launch_bounds__(kThreads) k_true_res(SolveArgs a) {
    PcgState* st = a.st;
    if (st->error) return;
    const GPlain g{a.x};
    double s[1] = {0.0};
    ROW_BATCH_BEGIN(a.n, kU)
        double y[kU];
        group_dot_batch<kU>(a.rp, a.ci, a.v, row, valid, g, l, y);
        if (l == 0) {
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                if (!valid[u]) continue;
                const double d = a.b[row[u]] - y[u];
                s[0] = fma(d, d, s[0]);
            }
        }
    ROW_BATCH_END
    double tot[1];
    if (grid_reduce<1>(s, a.partials, &st->counter[kTkTrue], tot) && threadIdx.x == 0)
        st->true_res = sqrt(tot[0]) / st->bnorm;
}

// --------------------------------------------------------------- k_spmv --
// plain y = A x (sparse.hpp:116-128)
__global__ void __launch_bounds__(kThreads) k_spmv(int n, const int* rp, const int* ci,
                                                   const double* v, const double* x, double* y) {
    const GPlain g{x};
    ROW_BATCH_BEGIN(n, kU)
        double yy[kU];
        group_dot_batch<kU>(rp, ci, v, row, valid, g, l, yy);
        if (l == 0) {
#pragma unroll
            for (int u = 0; u < kU; ++u)
                if (valid[u]) y[row[u]] = yy[u];
        }
    ROW_BATCH_END
}

// ======================================================= TMA-staged rows ==
__device__ __host__ __forceinline__ int tile_nnz_for(const SolveArgs& a, int TR) {
    return TR <= 64 ? a.tile_nnz64 : (TR <= 128 ? a.tile_nnz128 : a.tile_nnz256);
}

// Row epilogues of the SpMV-family kernels (same arithmetic as the direct
// kernels above). Each provides the gather, the per-row update (run by lane 0
// of the row's group) and, with NV > 0, the last-CTA finish.
// Ops with CTA_HOOKS run cta_pre(a) in every CTA before the grid sum and
// cta_last(a, tot) with the whole last CTA (instead of finish by one thread).
template <class Op, class = void>
struct HasCtaHooks : std::false_type {};
template <class Op>
struct HasCtaHooks<Op, std::void_t<decltype(Op::CTA_HOOKS)>> : std::bool_constant<Op::CTA_HOOKS> {};

struct OpSpmvP {
    static constexpr int NV = 1;
    static constexpr int TICKET = kTkSpmvP;
    GPupd g;
    double* pc;
    double* q;
    __device__ __forceinline__ void init(const SolveArgs& a) {
        const bool odd = a.st->it & 1;
        g = GPupd{a.z, odd ? a.p0 : a.p1, a.st->beta, a.st->first != 0};
        pc = odd ? a.p1 : a.p0;
        q = a.q;
    }
    __device__ __forceinline__ double operator()(int j) const { return g(j); }
    // own-row operands, loadable before the row's gathers complete
    struct Pre {
        double pi;
    };
    __device__ __forceinline__ Pre pre(int i) const { return Pre{g(i)}; }
    __device__ __forceinline__ void row(int i, double y, double* s, const Pre& p) const {
        pc[i] = p.pi;
        q[i] = y;
        s[0] = fma(p.pi, y, s[0]);
    }
    __device__ __forceinline__ void row(int i, double y, double* s) const { row(i, y, s, pre(i)); }
    __device__ __forceinline__ void finish(PcgState* st, const double* tot) const {
        const double pap = tot[0];
        st->pap = pap;
        if (pap <= 0.0) {
            st->error = kErrNotSpd;
            st->done = 1;
        } else {
            st->alpha = st->rz / pap;
        }
    }
};

template <class Gat, bool RZ, bool CW = false>
struct OpSweep {
    static constexpr int NV = RZ ? 1 : 0;
    static constexpr int TICKET = kTkSweep;
    Gat g;
    const double* r;
    const double* wd;
    double* zout;
    double wc = 0.0;    // constant w D^-1 (see GWdr)
    bool rpar = false;  // r = the residual the fused update + sweep wrote (r[(it + 1) & 1])
    __device__ __forceinline__ double operator()(int j) const { return g(j); }
    struct Pre {
        double ri, wi, gi;
    };
    __device__ __forceinline__ Pre pre(int i) const { return Pre{r[i], CW ? wc : wd[i], g(i)}; }
    __device__ __forceinline__ void row(int i, double y, double* s, const Pre& p) const {
        const double zi = fma(p.wi, p.ri - y, p.gi);
        zout[i] = zi;
        if (RZ) s[0] = fma(p.ri, zi, s[0]);
    }
    __device__ __forceinline__ void row(int i, double y, double* s) const { row(i, y, s, pre(i)); }
    __device__ __forceinline__ void init(const SolveArgs& a) {
        if (rpar) r = (a.st->it & 1) ? a.r : a.r1;
    }
    __device__ __forceinline__ void finish(PcgState* st, const double* tot) const {
        st->rz_new = tot[0];
    }
};

struct OpTrueRes {
    static constexpr int NV = 1;
    static constexpr int TICKET = kTkTrue;
    const double* x;
    const double* b;
    __device__ __forceinline__ double operator()(int j) const { return x[j]; }
    struct Pre {
        double bi;
    };
    __device__ __forceinline__ Pre pre(int i) const { return Pre{b[i]}; }
    __device__ __forceinline__ void row(int i, double y, double* s, const Pre& p) const {
        const double d = p.bi - y;
        s[0] = fma(d, d, s[0]);
    }
    __device__ __forceinline__ void row(int i, double y, double* s) const { row(i, y, s, pre(i)); }
    __device__ __forceinline__ void init(const SolveArgs&) {}
    __device__ __forceinline__ void finish(PcgState* st, const double* tot) const {
        st->true_res = sqrt(tot[0]) / st->bnorm;
    }
};

struct OpPlain {
    static constexpr int NV = 0;
    static constexpr int TICKET = kTkGeneric;
    const double* x;
    double* y;
    __device__ __forceinline__ double operator()(int j) const { return x[j]; }
    struct Pre {};
    __device__ __forceinline__ Pre pre(int) const { return Pre{}; }
    __device__ __forceinline__ void row(int i, double yy, double*, const Pre&) const { y[i] = yy; }
    __device__ __forceinline__ void row(int i, double yy, double*) const { y[i] = yy; }
    __device__ __forceinline__ void init(const SolveArgs&) {}
    __device__ __forceinline__ void finish(PcgState*, const double*) const {}
};

// ====================================================== diagonal-form rows ==
// The SpMV family over the diagonal form of A (DiaArgs, internal.cuh): one
// thread per row, presence bits of the row, gathers x[i + off_t] for the
// present offsets (consecutive rows -> coalesced), then the fma chain in
// ascending offset order = CSR column order, so y is bitwise the CSR kernels'
// y. Matrix bytes per row: the mask (1-4 B) for constant-coefficient stencils,
// + 8 d for per-row values, instead of 12 nnz/n + 4 for CSR.
// (Measured alternatives: lane shuffles for offsets within a
// warp and shared-memory windows per offset cluster both cut L2 requests but
// lost the memory-level parallelism of this form: 1.6x / 1.6x slower at C4.)
// EXACT: MAXD is the offset count itself (the common 5 / 7 / 9-point forms),
// and rows with every offset present (the interior) take an unpredicated path.
template <int MAXD, typename MT, bool RV, int SKIP, bool EXACT, class Op>
__global__ void __launch_bounds__(kThreads, NLSP_DIA_MINB) k_spmv_dia(SolveArgs a, Op op) {
    pdl_entry();
    PcgState* st = a.st;
    if (SKIP == 1 && st->done) return;
    if (SKIP == 2 && st->error) return;
    op.init(a);
    constexpr int NVS = Op::NV > 0 ? Op::NV : 1;
    double s[NVS];
#pragma unroll
    for (int j = 0; j < NVS; ++j) s[j] = 0.0;
    const MT* __restrict__ mask = static_cast<const MT*>(a.dia.mask);
    const int n = a.n, d = EXACT ? MAXD : a.dia.d;
    constexpr unsigned kFull = MAXD >= 32 ? ~0u : ((1u << MAXD) - 1u);
    // NLSP_DIA_ROWS rows per thread and step (rows i + r * stride): all their
    // loads are in flight together
    constexpr int RW = NLSP_DIA_ROWS;
#if NLSP_DIA_BLOCK
    // each CTA sweeps one contiguous chunk of rows in passes of blockDim rows:
    // the near neighbours (i +- 1, i +- nx) were just touched by this CTA (L1)
    const int stride = blockDim.x;
    const int chunk = ((n + gridDim.x - 1) / gridDim.x + blockDim.x - 1) / blockDim.x * blockDim.x;
    const int cbeg = blockIdx.x * chunk, cend = min(n, cbeg + chunk);
    for (int i0 = cbeg + threadIdx.x; i0 < cend; i0 += RW * stride) {
#else
    const int stride = gridDim.x * blockDim.x;
    for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += RW * stride) {
#endif
        // Every gather is issued unconditionally (index clamped into [0, n))
        // together with the mask and the own-row operands: no load waits on the
        // mask, so a row costs one memory latency, not two. Absent offsets are
        // then skipped by the mask, so y is unchanged (bitwise the CSR row sum).
        unsigned m[RW];
        typename Op::Pre pr[RW];
        double g[RW][MAXD], vv[RW][MAXD];
#pragma unroll
        for (int rr = 0; rr < RW; ++rr) {
            const int i = min(i0 + rr * stride, n - 1);
            m[rr] = mask[i];
            pr[rr] = op.pre(i);  // own-row operands in flight with the gathers
#pragma unroll
            for (int t = 0; t < MAXD; ++t) {
                if (t < d) {
                    const int j = min(max(i + a.dia.off[t], 0), n - 1);
                    g[rr][t] = op(j);
                    if (RV) vv[rr][t] = __ldcs(a.dia.rv + (size_t)t * n + i);  // 0 where absent
                } else {
                    g[rr][t] = 0.0;
                    if (RV) vv[rr][t] = 0.0;
                }
            }
        }
#pragma unroll
        for (int rr = 0; rr < RW; ++rr) {
            const int i = i0 + rr * stride;
#if NLSP_DIA_BLOCK
            if (rr > 0 && i >= cend) break;
#else
            if (rr > 0 && i >= n) break;
#endif
            double y = 0.0;
            if (EXACT && m[rr] == kFull) {
#pragma unroll
                for (int t = 0; t < MAXD; ++t) y = fma(RV ? vv[rr][t] : a.dia.val[t], g[rr][t], y);
            } else {
#pragma unroll
                for (int t = 0; t < MAXD; ++t)
                    if (t < d && ((m[rr] >> t) & 1u)) y = fma(RV ? vv[rr][t] : a.dia.val[t], g[rr][t], y);
            }
            op.row(i, y, s, pr[rr]);
        }
    }
    if constexpr (Op::NV > 0) {
        double v[Op::NV], tot[Op::NV];
#pragma unroll
        for (int j = 0; j < Op::NV; ++j) v[j] = s[j];
        if constexpr (HasCtaHooks<Op>::value) {
            op.cta_pre(a);
            if (grid_reduce<Op::NV>(v, a.partials, &st->counter[Op::TICKET], tot)) op.cta_last(a, tot);
        } else if (grid_reduce<Op::NV>(v, a.partials, &st->counter[Op::TICKET], tot) && threadIdx.x == 0) {
            op.finish(st, tot);
        }
    }
}

// SKIP: 0 never, 1 when st->done (solve kernels), 2 when st->error (true residual)
// G lanes per row (transposed mapping), U row steps per warp and tile:
// TR = 8 warps * U * (32 / G) rows per staged tile.
#ifndef NLSP_SPMV_MINB
#define NLSP_SPMV_MINB 3
#endif
// MK: the implicit-column form (PackArgs; one lane per row): the producer stages
// the rows' presence masks in place of the column indices
template <int G, int U, int S, int SKIP, int CHW, class Op, bool MK = false>
__global__ void __launch_bounds__(kTmaThreads, NLSP_SPMV_MINB) k_spmv_tma(SolveArgs a, Op op) {
    static_assert(!MK || G == 1, "implicit columns: one lane per row");
    pdl_entry();
    constexpr int R = 32 / G;
    constexpr int TR = kConsumerWarps * U * R;
    constexpr int CH = CHW;  // nonzeros per lane per pass (G * CH per row)
    static_assert(TR <= 256, "stage sizes are bounded by the 64/128/256-row nnz maxima");
    PcgState* st = a.st;
    if (SKIP == 1 && st->done) return;
    if (SKIP == 2 && st->error) return;
    op.init(a);
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);
    unsigned long long* empty = full + S;
    unsigned char* stages = smem + 128;
    const StageLayout L(TR, tile_nnz_for(a, TR), 0, false);
    __shared__ int pko[MK ? kMaxDia : 1];
    if (MK && threadIdx.x < kMaxDia) pko[threadIdx.x] = a.pk.off[threadIdx.x];
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int ntiles = (a.n + TR - 1) / TR;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double s[Op::NV > 0 ? Op::NV : 1];
    for (int j = 0; j < (Op::NV > 0 ? Op::NV : 1); ++j) s[j] = 0.0;
    if (warp == kConsumerWarps) {
        produce_tiles<S>(a.rp, a.ci, a.v, nullptr, 0, a.n, TR, stages, L, full, empty, MK ? a.pk.mask : nullptr);
    } else {
        int i = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
            const int stg = i % S;
            mbar_wait(&full[stg], (i / S) & 1);
            const int r0 = tile * TR, rows = min(TR, a.n - r0);
            int lr[U];
            bool valid[U];
            double y[U];
            // own-row operands in flight with the tile's gathers (lanes < R hold
            // rows (warp U + u) R + lane, as staged_rows_dot numbers them)
            typename Op::Pre pr[U];
            if (lane < R) {
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int lrow = (warp * U + u) * R + lane;
                    if (lrow < rows) pr[u] = op.pre(r0 + lrow);
                }
            }
            if constexpr (MK) staged_rows_dot_masked<U, CH>(stages + stg * L.bytes, L, rows, r0, warp, lane, op, pko, lr, valid, y);
            else staged_rows_dot<G, U, CH>(stages + stg * L.bytes, L, rows, warp, lane, op, lr, valid, y);
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
            if (lane < R) {
#pragma unroll
                for (int u = 0; u < U; ++u)
                    if (valid[u]) op.row(r0 + lr[u], y[u], s, pr[u]);
            }
        }
    }
    if constexpr (Op::NV > 0) {
        double v[Op::NV], tot[Op::NV];
#pragma unroll
        for (int j = 0; j < Op::NV; ++j) v[j] = s[j];
        if constexpr (HasCtaHooks<Op>::value) {
            op.cta_pre(a);
            if (grid_reduce<Op::NV>(v, a.partials, &st->counter[Op::TICKET], tot)) op.cta_last(a, tot);
        } else if (grid_reduce<Op::NV>(v, a.partials, &st->counter[Op::TICKET], tot) && threadIdx.x == 0) {
            op.finish(st, tot);
        }
    }
}

// res = r - A z_pre; c = P^T res with the tile's CSR slice AND its basis rows
// staged by the producer warp (two_level.hpp:63-73). The SpMV of a 64-row tile
// uses the transposed mapping (4 lanes per row, coalesced gathers), its
// residuals go through shared memory to the basis pass (8 lanes per basis row,
// 16-B reads of the staged rows).
template <int PPL, int ZMODE, int S>
__global__ void __launch_bounds__(kTmaThreads) k_restrict_tma(SolveArgs a, const double* zpre) {
    constexpr int G = 4, R = 32 / G;
    constexpr int TR = kConsumerWarps * R;  // 64
    constexpr int UP = TR / kGroups;        // basis rows per 8-lane group
    PcgState* st = a.st;
    if (st->done) return;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);
    unsigned long long* empty = full + S;
    double* res_s = reinterpret_cast<double*>(smem + 64);  // [2][TR] residuals (after barriers)
    unsigned char* stages = smem + 64 + 2 * TR * 8;
    const int ld = a.k + (a.k & 1);
    const int pairs = ld >> 1;
    const StageLayout L(TR, a.tile_nnz64, ld, true);
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int ntiles = (a.n + TR - 1) / TR;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double acc[2 * PPL];
#pragma unroll
    for (int t = 0; t < 2 * PPL; ++t) acc[t] = 0.0;
    if (warp == kConsumerWarps) {
        produce_tiles<S>(a.rp, a.ci, a.v, a.P, ld, a.n, TR, stages, L, full, empty);
    } else {
        const int grp = threadIdx.x >> 3, l = threadIdx.x & (kGroup - 1);
        const GWdr gw{a.wd, a.r};
        const GPlain gp{zpre};
        int i = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
            const int stg = i % S;
            const unsigned char* base = stages + stg * L.bytes;
            const int r0 = tile * TR, rows = min(TR, a.n - r0);
            double* rs = res_s + (i & 1) * TR;
            // residual of row r0 + lr: r - A z_pre (own r read before the wait)
            const int lr0 = warp * R + (lane % R);
            const double rown = lr0 < rows ? a.r[r0 + lr0] : 0.0;
            mbar_wait(&full[stg], (i / S) & 1);
            int lr[1];
            bool valid[1];
            double y[1] = {0.0};
            if (ZMODE == 1) staged_rows_dot<G, 1, 2>(base, L, rows, warp, lane, gw, lr, valid, y);
            if (ZMODE == 2) staged_rows_dot<G, 1, 2>(base, L, rows, warp, lane, gp, lr, valid, y);
            if (lane < R) rs[lr0] = lr0 < rows ? rown - y[0] : 0.0;
            asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
            const double* ps = reinterpret_cast<const double*>(base + L.p_off);
#pragma unroll
            for (int u = 0; u < UP; ++u) {
                const int lrp = grp + kGroups * u;
                const bool ok = lrp < rows;
                const double res = ok ? rs[lrp] : 0.0;
                const double* prow = ps + lrp * ld;
#pragma unroll
                for (int t = 0; t < PPL; ++t) {
                    const int pi = l + kGroup * t;
                    if (ok && pi < pairs) {
                        const double2 pv = *reinterpret_cast<const double2*>(prow + 2 * pi);
                        acc[2 * t] = fma(pv.x, res, acc[2 * t]);
                        acc[2 * t + 1] = fma(pv.y, res, acc[2 * t + 1]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
        }
    }
    restrict_finish<PPL, kTmaThreads, false>(acc, 0.0, a);
}

// ================================================ folded two-level cycle ==
// The cycle of two_level.hpp:60-81 is linear in r. With G = I - w D^-1 A
// (one homogeneous Jacobi sweep) and S_t(r) = sum_{i<t} G^i w D^-1 r (t sweeps
// from zero):
//   restriction  P^T (r - A S_nu1(r)) = (G^nu1 P)^T r = W1^T r      (A = A^T)
//   result       z = S_{nu1+nu2}(r) + (G^nu2 P) e = S_{nu1+nu2}(r) + W2 e
// W1, W2 are formed once at build time (nu homogeneous block sweeps of the
// orthonormal basis). Same operator as the reference's cycle; per iteration one
// CSR pass fewer than the literal schedule, and the restriction fuses with the
// x/r update. Rounding differs from the literal order at the 1e-16 level.

// x += alpha p, r -= alpha q, ||r||^2 (two_level.hpp:164-170) fused with
// c = W1^T r_new; last CTA: history + convergence test, then L L^T e = c.
// UPDATE = false: c = W1^T r only (preconditioner apply / PCG prologue).
// CTA tiles of 64 rows: every 8-lane group first issues its two W1 rows
// (16-B streaming loads), then threads 0..63 update x, r with coalesced loads
// and hand r_new over through shared memory (double-buffered by tile parity).
template <int PPL, bool UPDATE>
__global__ void __launch_bounds__(kThreads) k_update_restrict(SolveArgs a) {
    constexpr int TR = 64;
    constexpr int UP = TR / (kThreads / kGroup);  // W1 rows per group: 2
    PcgState* st = a.st;
    if (st->done) return;
    __shared__ double rn_s[2][TR];
    const int ld = a.k + (a.k & 1);
    const int pairs = ld >> 1;
    const double alpha = UPDATE ? st->alpha : 0.0;
    const double* p = (st->it & 1) ? a.p1 : a.p0;
    const int grp = threadIdx.x >> 3, l = threadIdx.x & (kGroup - 1);
    double acc[2 * PPL];
#pragma unroll
    for (int t = 0; t < 2 * PPL; ++t) acc[t] = 0.0;
    double rr = 0.0;
    const int ntiles = (a.n + TR - 1) / TR;
    int par = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, par ^= 1) {
        const int r0 = tile * TR, rows = min(TR, a.n - r0);
        double2 wv[UP][PPL];
#pragma unroll
        for (int u = 0; u < UP; ++u) {
            const int lr = grp + (kThreads / kGroup) * u;
            const double* wrow = a.W1 + (long long)(r0 + lr) * ld;
#pragma unroll
            for (int t = 0; t < PPL; ++t) {
                const int pi = l + kGroup * t;
                wv[u][t] = (lr < rows && pi < pairs) ? ld_stream2(wrow + 2 * pi) : make_double2(0.0, 0.0);
            }
        }
        if (threadIdx.x < TR) {
            const int lr = threadIdx.x;
            double rnew = 0.0;
            if (lr < rows) {
                const int i = r0 + lr;
                if (UPDATE) {
                    rnew = fma(-alpha, a.q[i], a.r[i]);
                    a.x[i] = fma(alpha, p[i], a.x[i]);
                    a.r[i] = rnew;
                    rr = fma(rnew, rnew, rr);
                } else {
                    rnew = a.r[i];
                }
            }
            rn_s[par][lr] = rnew;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < UP; ++u) {
            const double rv = rn_s[par][grp + (kThreads / kGroup) * u];
#pragma unroll
            for (int t = 0; t < PPL; ++t) {
                acc[2 * t] = fma(wv[u][t].x, rv, acc[2 * t]);
                acc[2 * t + 1] = fma(wv[u][t].y, rv, acc[2 * t + 1]);
            }
        }
    }
    restrict_finish<PPL, kThreads, UPDATE>(acc, rr, a);
}

// The same fused update + restriction with everything staged by the producer
// warp: per 64-row tile the W1 rows and the x, p, q, r slices (contiguous, one
// bulk copy each). Consumers: 64 threads update x, r for the tile's rows
// (coalesced stores, r_new to shared memory), then all 8 warps accumulate
// c += r_new W1 with 8 lanes per row.
template <int PPL, bool UPDATE, int S>
__global__ void __launch_bounds__(kTmaThreads) k_update_restrict_tma(SolveArgs a) {
    constexpr int TR = 64;
    constexpr int UP = TR / kGroups;
    PcgState* st = a.st;
    if (st->done) return;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);
    unsigned long long* empty = full + S;
    double* rn_s = reinterpret_cast<double*>(smem + 64);  // [2][TR]
    unsigned char* stages = smem + 64 + 2 * TR * 8;
    const int ld = a.k + (a.k & 1);
    const int pairs = ld >> 1;
    constexpr int NV = UPDATE ? 4 : 1;  // staged vectors: r (+ x, p, q)
    const unsigned vbytes = TR * 8;
    const unsigned stage_bytes = NV * vbytes + round16(TR * ld * 8);
    const double alpha = UPDATE ? st->alpha : 0.0;
    const double* p = (st->it & 1) ? a.p1 : a.p0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kConsumerWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int ntiles = (a.n + TR - 1) / TR;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    double acc[2 * PPL];
#pragma unroll
    for (int t = 0; t < 2 * PPL; ++t) acc[t] = 0.0;
    double rr = 0.0;
    if (warp == kConsumerWarps) {
        if (lane == 0) {
            int i = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
                const int stg = i % S;
                if (i >= S) mbar_wait(&empty[stg], ((i / S) - 1) & 1);
                unsigned char* base = stages + stg * stage_bytes;
                const int r0 = tile * TR, rows = min(TR, a.n - r0);
                const unsigned vb = round16(rows * 8);  // vectors are padded by 16 doubles
                const unsigned wb = rows * ld * 8;
                mbar_arrive_tx(&full[stg], NV * vb + wb);
                bulk_g2s(base, a.r + r0, vb, &full[stg]);
                if (UPDATE) {
                    bulk_g2s(base + vbytes, a.x + r0, vb, &full[stg]);
                    bulk_g2s(base + 2 * vbytes, p + r0, vb, &full[stg]);
                    bulk_g2s(base + 3 * vbytes, a.q + r0, vb, &full[stg]);
                }
                bulk_g2s(base + NV * vbytes, a.W1 + (long long)r0 * ld, wb, &full[stg]);
            }
        }
    } else {
        const int grp = threadIdx.x >> 3, l = threadIdx.x & (kGroup - 1);
        int i = 0;
        for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++i) {
            const int stg = i % S;
            const unsigned char* base = stages + stg * stage_bytes;
            const int r0 = tile * TR, rows = min(TR, a.n - r0);
            double* rn = rn_s + (i & 1) * TR;
            mbar_wait(&full[stg], (i / S) & 1);
            const double* rs = reinterpret_cast<const double*>(base);
            if (threadIdx.x < TR) {
                const int lr = threadIdx.x;
                double rnew = 0.0;
                if (lr < rows) {
                    if (UPDATE) {
                        const double* xs = rs + TR;
                        const double* pps = rs + 2 * TR;
                        const double* qs = rs + 3 * TR;
                        rnew = fma(-alpha, qs[lr], rs[lr]);
                        a.x[r0 + lr] = fma(alpha, pps[lr], xs[lr]);
                        a.r[r0 + lr] = rnew;
                        rr = fma(rnew, rnew, rr);
                    } else {
                        rnew = rs[lr];
                    }
                }
                rn[lr] = rnew;
            }
            asm volatile("bar.sync 1, %0;" ::"n"(kConsumerWarps * 32) : "memory");
            const double* ws = rs + NV * TR;
#pragma unroll
            for (int u = 0; u < UP; ++u) {
                const int lrp = grp + kGroups * u;
                if (lrp >= rows) continue;
                const double res = rn[lrp];
                const double* wrow = ws + lrp * ld;
#pragma unroll
                for (int t = 0; t < PPL; ++t) {
                    const int pi = l + kGroup * t;
                    if (pi < pairs) {
                        const double2 wv = *reinterpret_cast<const double2*>(wrow + 2 * pi);
                        acc[2 * t] = fma(wv.x, res, acc[2 * t]);
                        acc[2 * t + 1] = fma(wv.y, res, acc[2 * t + 1]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
        }
    }
    restrict_finish<PPL, kTmaThreads, UPDATE>(acc, rr, a);
}

// ================================================ wide coarse spaces (k > 256) ==
// Coarse dimensions beyond the 8-lane register tiles (e.g. the SA prolongator's
// emergent n_c, sa.hpp:78-109). Same arithmetic as the narrow kernels; the
// coarse solve runs as its own multi-CTA mat-vec with A_c^-1.

// x += alpha p, r -= alpha q, ||r||^2, c = W1^T r_new (UPDATE) or c = W1^T r.
// Each CTA walks a contiguous row chunk; warp 0 forms 32 residuals at a time,
// every thread accumulates columns tid + 256 t over them (coalesced W1 rows).
// Last CTA: fixed-order sum of the partials into c, history + convergence.
template <bool UPDATE>
__global__ void __launch_bounds__(kThreads) k_update_restrict_wide(SolveArgs a) {
    constexpr int KT = kMaxCoarse / kThreads;  // accumulators per thread
    PcgState* st = a.st;
    if (st->done) return;
    const int ld = a.k + (a.k & 1);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    __shared__ double rn_s[32];
    __shared__ double red_s[kThreads / 32];
    __shared__ int is_last;
    const double alpha = UPDATE ? st->alpha : 0.0;
    const double* p = (st->it & 1) ? a.p1 : a.p0;
    const long long chunk = ((long long)a.n + gridDim.x - 1) / gridDim.x;
    const long long r0 = blockIdx.x * chunk, r1 = min((long long)a.n, r0 + chunk);
    double acc[KT];
#pragma unroll
    for (int t = 0; t < KT; ++t) acc[t] = 0.0;
    double rr = 0.0;
    for (long long base = r0; base < r1; base += 32) {
        const int rows = (int)min(32LL, r1 - base);
        if (warp == 0) {
            double rnew = 0.0;
            if (lane < rows) {
                const long long i = base + lane;
                if (UPDATE) {
                    rnew = fma(-alpha, a.q[i], a.r[i]);
                    a.x[i] = fma(alpha, p[i], a.x[i]);
                    a.r[i] = rnew;
                    rr = fma(rnew, rnew, rr);
                } else {
                    rnew = a.r[i];
                }
            }
            rn_s[lane] = rnew;
        }
        __syncthreads();
#pragma unroll 4
        for (int ii = 0; ii < rows; ++ii) {
            const double rv = rn_s[ii];
            const double* w = a.W1 + (base + ii) * ld;
#pragma unroll
            for (int t = 0; t < KT; ++t) {
                const int j = tid + kThreads * t;
                if (j < ld) acc[t] = fma(__ldcs(w + j), rv, acc[t]);
            }
        }
        __syncthreads();
    }
    // CTA partial: ld columns (+ ||r||^2) -> partials[blockIdx * (ld + 1) + .]
    double* part = a.partials + (long long)blockIdx.x * (ld + 1);
#pragma unroll
    for (int t = 0; t < KT; ++t) {
        const int j = tid + kThreads * t;
        if (j < ld) part[j] = acc[t];
    }
    if (UPDATE) {
        rr = warp_sum(rr);
        if (tid == 0) part[ld] = rr;  // warp 0 holds every ||r||^2 term
    }
    __syncthreads();
    if (tid == 0) {
        __threadfence();
        const unsigned int tk = atomicAdd(&st->counter[kTkRestrict], 1u);
        is_last = (tk == gridDim.x - 1);
    }
    __syncthreads();
    if (!is_last) return;
    __threadfence();
    double* c = a.partials + kWideCOffset;
    for (int j = tid; j < ld + (UPDATE ? 1 : 0); j += kThreads) {
        double t = 0.0;
        for (int b = 0; b < (int)gridDim.x; ++b) t += __ldcg(a.partials + (long long)b * (ld + 1) + j);
        c[j] = t;
        if (UPDATE && j == ld) red_s[0] = t;
    }
    __syncthreads();
    if (UPDATE && tid == 0) {
        const double rrt = red_s[0];
        const double rel = sqrt(rrt) / st->bnorm;
        st->rr = rrt;
        st->last_rel = rel;
        a.hist[st->it - st->hist_base] = rel;
        st->iterations = st->it + 1;
        if (rel < st->delta) {
            st->converged = 1;
            st->done = 1;
        }
    }
    if (tid == 0) st->counter[kTkRestrict] = 0u;
}

// e = A_c^-1 c (two_level.hpp:73): a warp per output row
__global__ void __launch_bounds__(kThreads) k_coarse_gemv(SolveArgs a, int skip_done) {
    if (skip_done && a.st->done) return;
    const int k = a.k, lane = threadIdx.x & 31;
    const double* c = a.partials + kWideCOffset;
    const long long warps = (long long)gridDim.x * (kThreads / 32);
    for (long long i = blockIdx.x * (long long)(kThreads / 32) + (threadIdx.x >> 5); i < k; i += warps) {
        const double* row = a.Ainv + i * k;
        double s = 0.0;
        for (int j = lane; j < k; j += 32) s = fma(__ldg(row + j), __ldcg(c + j), s);
        s = warp_sum(s);
        if (lane == 0) a.e[i] = s;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0 && (k & 1)) a.e[k] = 0.0;  // padded column
}

// z = z_pre + W2 e (two_level.hpp:74-78), r.z; ctl: loop control as k_prolong
template <int ZMODE, bool RZ>
__global__ void __launch_bounds__(kThreads) k_prolong_wide(SolveArgs a, const double* zpre, double* zout,
                                                         cudaGraphConditionalHandle h, int ctl) {
    PcgState* st = a.st;
    if (st->done) {
        if (ctl && blockIdx.x == 0 && threadIdx.x == 0) loop_ctl_body(st, h, ctl == 2);
        return;
    }
    __shared__ double es[kMaxCoarse + 2];
    const int ld = a.k + (a.k & 1);
    for (int j = threadIdx.x; j < ld; j += kThreads) es[j] = a.e[j];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    double s[1] = {0.0};
    const long long warps = (long long)gridDim.x * (kThreads / 32);
    for (long long i = blockIdx.x * (long long)(kThreads / 32) + (threadIdx.x >> 5); i < a.n; i += warps) {
        double zp;
        if (ZMODE == 0) zp = 0.0;
        else if (ZMODE == 1) zp = a.wd[i] * a.r[i];
        else zp = zpre[i];
        const double ri = RZ ? a.r[i] : 0.0;
        const double* w = a.P + i * ld;
        double acc = 0.0;
        for (int j = lane; j < ld; j += 32) acc = fma(__ldcs(w + j), es[j], acc);
        acc = warp_sum(acc);
        if (lane == 0) {
            const double zi = zp + acc;
            zout[i] = zi;
            if (RZ) s[0] = fma(ri, zi, s[0]);
        }
    }
    if (RZ) {
        double tot[1];
        if (grid_reduce<1>(s, a.partials, &st->counter[kTkProlong], tot) && threadIdx.x == 0) {
            st->rz_new = tot[0];
            if (ctl) loop_ctl_body(st, h, ctl == 2);
        }
    }
}

// ==================================================== one-pass two-level cycle ==
// With nu1 = nu2 the folded cycle streams W = W1 = W2 twice per iteration:
// c = W^T r_new after the x/r update, and z = s + W e after the sweeps. The
// restriction is carried by its recurrence instead, so W is streamed ONCE:
//   c_{i+1} = W^T r_{i+1} = W^T r_i - alpha_i W^T q_i,
//   W^T q_i = W^T A p_i   = W^T A s_i + M e_i + beta_i W^T q_{i-1},  M = W^T A W,
// since p_i = z_i + beta_i p_{i-1} and z_i = s_i + W e_i, and
//   W^T q_{i-1} = (u_{i-1} - u_i) / alpha_{i-1}   (r_i = r_{i-1} - alpha_{i-1} q_{i-1}).
// The prolongation pass of iteration i reads W rows once and forms, besides
// z_i = s_i + W e_i and r.z, two k-vectors: u_i = W^T r_i and v_i = W^T (A s_i)
// (A s_i gathered in the same pass). Every term on the right is recomputed from
// the current vectors each iteration, so no drift accumulates: only the
// one-step combination c = u_i - alpha_i (v_i + M e_i + beta_i W^T q_{i-1}) is
// new (relative deviation from W^T r_{i+1} ~1e-13 over thousands of
// iterations), formed by the next update kernel's last CTA together with
// e = A_c^-1 c. Same operator as the
// reference's cycle (two_level.hpp:60-81), iteration counts identical on the
// configs; per iteration 8nk bytes fewer than the folded cycle.

// y = sum_t A(i, i + off_t) x[i + off_t] over the present offsets of row i, in
// ascending offset order (the CSR column order), for any diagonal form
template <int MAXD, bool RV>
__device__ __forceinline__ double dia_row_dot(const SolveArgs& a, int i, const double* __restrict__ x) {
    const int mb = a.dia.mbytes, d = a.dia.d;
    unsigned m;
    if (mb == 1) m = static_cast<const unsigned char*>(a.dia.mask)[i];
    else if (mb == 2) m = static_cast<const unsigned short*>(a.dia.mask)[i];
    else m = static_cast<const unsigned int*>(a.dia.mask)[i];
    double g[MAXD], vv[RV ? MAXD : 1];
#pragma unroll
    for (int t = 0; t < MAXD; ++t) {
        const bool on = t < d && ((m >> t) & 1u);
        g[t] = on ? x[i + a.dia.off[t]] : 0.0;
        if (RV) vv[RV ? t : 0] = on ? __ldcs(a.dia.rv + (size_t)t * a.n + i) : 0.0;
    }
    double y = 0.0;
#pragma unroll
    for (int t = 0; t < MAXD; ++t)
        if (t < d && ((m >> t) & 1u)) y = fma(RV ? vv[RV ? t : 0] : a.dia.val[t], g[t], y);
    return y;
}

// Per-lane column accumulators of one k-vector -> this CTA's column sums ->
// dst[c * G + blockIdx.x] (column-major partials, G = gridDim.x).
// ecol / dot: also *dot += sum_c (this CTA's column sum c) * ecol[c]
template <int PPL>
__device__ __forceinline__ void cta_columns(double (&acc)[2 * PPL], double* cs, int ld, double* dst,
                                            const double* ecol = nullptr, double* dot = nullptr) {
    constexpr int CW = 2 * kGroup * PPL;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int pairs = ld >> 1;
#pragma unroll
    for (int t = 0; t < 2 * PPL; ++t) {
        acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], 8);
        acc[t] += __shfl_xor_sync(0xffffffffu, acc[t], 16);
    }
    if (lane < kGroup) {
#pragma unroll
        for (int t = 0; t < PPL; ++t) {
            const int pi = lane + kGroup * t;
            if (pi < pairs) {
                cs[warp * CW + 2 * pi] = acc[2 * t];
                cs[warp * CW + 2 * pi + 1] = acc[2 * t + 1];
            }
        }
    }
    __syncthreads();
    for (int c = threadIdx.x; c < ld; c += blockDim.x) {
        double t = 0.0;
        for (int w = 0; w < nw; ++w) t += cs[w * CW + c];
        dst[(long long)c * gridDim.x + blockIdx.x] = t;
        if (ecol) *dot = fma(t, ecol[c], *dot);
    }
    __syncthreads();
}

// z = s + W e (two_level.hpp:74-79 folded), r.z -> beta and the loop control
// (ctl as k_prolong), and in the same pass over W: u = W^T r, v = W^T (A s) as
// per-CTA partials. A s one lane per row (8 rows per warp): MAXD = 0 the CSR
// row, else the diagonal form (RV: per-row values).
template <int PPL, int MAXD, bool RV>
__global__ void __launch_bounds__(kThreads, 2) k_prolong_onepass(SolveArgs a, const double* sv,
                                                              double* zout,
                                                              cudaGraphConditionalHandle h, int ctl,
                                                              int rsel) {
    pdl_entry();
    PcgState* st = a.st;
    if (st->done) {
        if (ctl && blockIdx.x == 0 && threadIdx.x == 0) loop_ctl_body(st, h, ctl == 2);
        return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) st->op_grid = gridDim.x;
    // rsel: the residual the fused update + sweep wrote (r[(it + 1) & 1]), else r
    const double* rv = (rsel && !(st->it & 1)) ? a.r1 : a.r;
    const int ld = a.k + (a.k & 1);
    const int pairs = ld >> 1;
    double ev[2 * PPL], au[2 * PPL], av[2 * PPL];
    {
        const int l0 = threadIdx.x & (kGroup - 1);
#pragma unroll
        for (int t = 0; t < PPL; ++t) {
            const int pi = l0 + kGroup * t;
            ev[2 * t] = pi < pairs ? a.e[2 * pi] : 0.0;
            ev[2 * t + 1] = pi < pairs ? a.e[2 * pi + 1] : 0.0;
        }
#pragma unroll
        for (int t = 0; t < 2 * PPL; ++t) au[t] = av[t] = 0.0;
    }
    double s[1] = {0.0};
    constexpr int UPR = NLSP_KUPRO;
    ROW_BATCH_BEGIN(a.n, UPR)
        // W rows first (the HBM stream), then the row scalars and A s gathers
        double2 pv[UPR][PPL];
#pragma unroll
        for (int u = 0; u < UPR; ++u) {
            const double* prow = a.P + (long long)row[u] * ld;
#pragma unroll
            for (int t = 0; t < PPL; ++t) {
                const int pi = l + kGroup * t;
                pv[u][t] = (valid[u] && pi < pairs) ? ld_stream2(prow + 2 * pi) : make_double2(0.0, 0.0);
            }
        }
        double sr[UPR], rr[UPR], as[UPR];
#pragma unroll
        for (int u = 0; u < UPR; ++u) {
            const int rw = valid[u] ? row[u] : 0;
            sr[u] = sv ? sv[rw] : 0.0;
            rr[u] = valid[u] ? rv[rw] : 0.0;
        }
        {
            // lane L < 4 UPR sums row base + L (sequential fma chain in column
            // order, bitwise the SpMV family's rows); group grp's row u is lane grp + 4u
            double mine = 0.0;
            const long long ri = base_ + lane_;
            if (sv && lane_ < kRowsPerWarp * UPR && ri < a.n) {
                if constexpr (MAXD == 0) {
                    const int b = __ldg(a.rp + ri), e = __ldg(a.rp + ri + 1);
                    for (int kk = b; kk < e; ++kk) mine = fma(__ldg(a.v + kk), sv[__ldg(a.ci + kk)], mine);
                } else {
                    mine = dia_row_dot<MAXD, RV>(a, (int)ri, sv);
                }
            }
#pragma unroll
            for (int u = 0; u < UPR; ++u) as[u] = __shfl_sync(0xffffffffu, mine, grp + kRowsPerWarp * u);
        }
        double sum[UPR];
#pragma unroll
        for (int u = 0; u < UPR; ++u) {
            double part = 0.0;
#pragma unroll
            for (int t = 0; t < PPL; ++t) {
                part = fma(pv[u][t].x, ev[2 * t], part);
                part = fma(pv[u][t].y, ev[2 * t + 1], part);
                au[2 * t] = fma(pv[u][t].x, rr[u], au[2 * t]);
                au[2 * t + 1] = fma(pv[u][t].y, rr[u], au[2 * t + 1]);
                av[2 * t] = fma(pv[u][t].x, as[u], av[2 * t]);
                av[2 * t + 1] = fma(pv[u][t].y, as[u], av[2 * t + 1]);
            }
            sum[u] = group_sum(part);
        }
        if (l == 0) {
#pragma unroll
            for (int u = 0; u < UPR; ++u) {
                if (!valid[u]) continue;
                const double zi = sr[u] + sum[u];
                zout[row[u]] = zi;
                s[0] = fma(rr[u], zi, s[0]);
            }
        }
    ROW_BATCH_END
    {
        __shared__ double cs[(kThreads / 32) * 2 * kGroup * PPL];
        const long long G = gridDim.x;
        cta_columns<PPL>(au, cs, ld, a.opart);
        cta_columns<PPL>(av, cs, ld, a.opart + ld * G);
    }
    double tot[1];
    if (grid_reduce<1>(s, a.partials, &st->counter[kTkProlong], tot) && threadIdx.x == 0) {
        st->rz_new = tot[0];
        if (ctl) loop_ctl_body(st, h, ctl == 2);
    }
}

// The one-pass prolongation with its HBM stream decoupled from the gathers
// (warp-specialised, 1 CTA per SM): a producer warp stages each 64-row tile —
// its W rows, s and r slices and the diagonal form's presence masks — into an
// S-stage ring with bulk copies (cp.async.bulk, mbarrier complete_tx); pairs
// of stencil warps take alternate tiles and form (A s)_row from the staged
// mask and L2 gathers of s (the only global latency left), publishing them
// through a second barrier per stage; 8 consumer warps then run the W products
// of the tile from shared memory (8 lanes per row) and release the stage.
#ifndef NLSP_OP_TR
#define NLSP_OP_TR 64
#endif
#ifndef NLSP_LFUSED_DEFAULT
#define NLSP_LFUSED_DEFAULT 1
#endif
#ifndef NLSP_STENCIL_SLEEP
#define NLSP_STENCIL_SLEEP 200  // ns between the stencil warps' polls at k > 48 (0: the plain wait)
#endif
constexpr int kOpTR = NLSP_OP_TR;  // rows per tile (64 or 128)
static_assert(kOpTR == 64 || kOpTR == 128, "one-pass tiles are 64 or 128 rows");
constexpr int kOpWWarps = 8;   // W-product warps
constexpr int kOpSPairs = 4;   // at most this many stencil warp pairs (tile i -> pair i % P)
constexpr int kOpMaxStages = 8;
// The W-product warps split into op_wh(PPL) groups taking alternate tiles (the
// ring depth S must then be a multiple of it as well): two groups for k <= 48,
// whose tiles are short (measured: C3 prolongation 317 -> 292 us, C2 83 -> 78 us;
// at k = 64 one group is faster, C4 -3.7 %, C5 -3 % with two).
// (16 W-product warps in two groups with 2 stencil pairs at k = 64 measured
// slower too: C4 -7 %, C5 -6 %)
__host__ __device__ constexpr int op_wh(int ppl) { return ppl <= 3 ? 2 : 1; }
// W-product warps per group (kOpWWarps in all: k <= 48: 2 x 4, k = 64: 1 x 8)
__host__ __device__ constexpr int op_wpg(int ppl) { return kOpWWarps / op_wh(ppl); }
__host__ __device__ constexpr int op_threads_max(int ppl) {
    return 32 * (1 + 2 * kOpSPairs + op_wpg(ppl) * op_wh(ppl));
}

// Stencil pair p waits only on tiles i = p (mod P). With S a multiple of P it
// always sees the stages p, p + P, ... and waits their phases in order, so an
// mbarrier parity wait can never alias a phase two ahead (S % P == 0 is required).
constexpr unsigned kOpVec = kOpTR * 8;  // bytes of one staged vector slice

// CSR matrices also stage the tile's row_ptr slice and its runs of values and
// column indices (at most tile_nnz nonzeros), so the stencil warps only gather s
__host__ __device__ constexpr unsigned op_csr_bytes(int tile_nnz) {
    return round16((kOpTR + 4) * 4) + round16((tile_nnz + 2) * 8) + round16((tile_nnz + 8) * 4);
}
__host__ __device__ constexpr unsigned op_stage_bytes(int ld, int tile_nnz = -1) {
    return (unsigned)kOpTR * ld * 8 + 2 * kOpVec + round16(kOpTR * 4) + 2 * kOpVec +
           (tile_nnz >= 0 ? op_csr_bytes(tile_nnz) : 0u);
}

// The coarse step of the lean cycle, run redundantly by the 256 W-product
// threads of EVERY CTA of the pass while its producer fills the stage ring (so
// it is off the critical path; as the last CTA of the sweep kernel it cost
// ~10 us per iteration): the one-pass restriction recurrence
//   c = u_i - alpha_i (v_i + M e_i + beta_i (u_{i-1} - u_i) / alpha_{i-1})
// from the column sums the sweep kernel left in ow, e = A_c^-1 c, M e, and the
// scalars c.e, e.M e -> r.z = r.s + c.e, beta = r.z / r.z_prev. Every CTA gets
// bitwise the same values; CTA 0 publishes them (a.e, ow, the drift guard).
// t: thread index in [0, 256); sc: 5 (ld + 2) doubles of scratch; on return
// sc[3 (ld + 2) ..] holds e and lsc = [e.Me, r.z, beta].
__device__ __forceinline__ void lean_bar() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// (operands by value: a reference to the kernel's SolveArgs would move the
// whole struct to local memory, and every a.* of the hot loops with it —
// measured +34 us per pass at C4)
struct LeanCoarse {
    const double* Ainv;
    const double* M;
    const double* L;
    double* ow;
    double* e;
    PcgState* st;
    int k;
};
__device__ __noinline__ void lean_coarse_step(const LeanCoarse a, int t, double* sc, double* lsc) {
    PcgState* st = a.st;
    const int k = a.k, ld = a.k + (a.k & 1);
    double* cs = sc;
    double* ws = sc + (ld + 2);
    double* es = sc + 3 * (ld + 2);
    double* gs = sc + 4 * (ld + 2);
    const int i = t >> 2, sub = t & 3, lane = t & 31, w = t >> 5;
    NLSP_CHECK(t >= 0 && t < 256 && k <= kOnePassK && 5 * (ld + 2) <= 5 * (kOnePassK + 2));
    // A_c^-1 and M rows (L2 resident): in flight with everything else
    double ai[kOnePassK / 4], mi[kOnePassK / 4];
#pragma unroll
    for (int jj = 0; jj < kOnePassK / 4; ++jj) {
        const int j = sub + 4 * jj;
        const bool ok = i < k && j < k;
        ai[jj] = (ok && a.Ainv) ? __ldg(a.Ainv + (long long)i * k + j) : 0.0;
        mi[jj] = ok ? __ldg(a.M + (long long)i * k + j) : 0.0;
    }
    // both parities of the ping-pong slots, so no load waits on st->it
    double o6[6];
#pragma unroll
    for (int q = 0; q < 6; ++q) o6[q] = t < k ? __ldcg(a.ow + q * ld + t) : 0.0;
    const bool first = st->first != 0;
    const long long it = st->it;
    const double alpha = st->alpha, alpha_prev = st->alpha_prev, beta = st->beta, gam = st->rz, rs = st->rz_new;
    const bool odd = it & 1;
    const int mnew = (4 + (int)((it + 1) & 1)) * ld;
    double d = 0.0, um = 0.0;
    if (t < k) {
        const double u = odd ? o6[1] : o6[0], up = odd ? o6[0] : o6[1];
        double g = o6[2] + (odd ? o6[5] : o6[4]);                  // v + M e
        if (!first) g = fma(beta, (up - u) / alpha_prev, g);       // + beta W^T q_{i-1}
        const double c = fma(-alpha, g, u);                        // c = u - alpha g
        cs[t] = c;
        ws[t] = c;  // the substitutions overwrite their right-hand side
        if (blockIdx.x == 0) {
            // guard: last iteration's recurrence value against the direct u_i
            if (!first) {
                d = fabs(o6[3] - u);
                um = fabs(u);
            }
            a.ow[3 * ld + t] = c;
        }
    }
    if (blockIdx.x == 0 && !first && w < 2) {
        for (int o = 16; o; o >>= 1) {
            d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
            um = fmax(um, __shfl_xor_sync(0xffffffffu, um, o));
        }
        if (lane == 0) {
            lsc[4 + w] = d;
            lsc[6 + w] = um;
        }
    }
    lean_bar();
    if (a.Ainv) {
        double e = 0.0;
#pragma unroll
        for (int jj = 0; jj < kOnePassK / 4; ++jj)
            if (sub + 4 * jj < k) e = fma(ai[jj], cs[sub + 4 * jj], e);
        e += __shfl_xor_sync(0xffffffffu, e, 1);
        e += __shfl_xor_sync(0xffffffffu, e, 2);
        if (i < k && sub == 0) es[i] = e;
    } else if (w == 0) {
        coarse_solve_warp(a.L, k, ws, es);
    }
    if (t == 0 && (k & 1)) es[k] = 0.0;  // padded column
    lean_bar();
    {
        double g = 0.0;
#pragma unroll
        for (int jj = 0; jj < kOnePassK / 4; ++jj)
            if (sub + 4 * jj < k) g = fma(mi[jj], es[sub + 4 * jj], g);
        g += __shfl_xor_sync(0xffffffffu, g, 1);
        g += __shfl_xor_sync(0xffffffffu, g, 2);
        if (i < k && sub == 0) gs[i] = g;
    }
    lean_bar();
    if (w == 0) {
        double ce = 0.0, eme = 0.0;
        for (int j = lane; j < k; j += 32) {
            ce = fma(cs[j], es[j], ce);
            eme = fma(es[j], gs[j], eme);
        }
        ce = warp_sum(ce);
        eme = warp_sum(eme);
        if (lane == 0) {
            const double g = rs + ce;
            lsc[0] = eme;
            lsc[1] = g;
            lsc[2] = g / gam;
            if (blockIdx.x == 0 && !first) {
                const double dd = fmax(lsc[4], k > 32 ? lsc[5] : 0.0), uu = fmax(lsc[6], k > 32 ? lsc[7] : 0.0);
                const double drift = uu > 0.0 ? dd / uu : 0.0;
                st->drift_max = fmax(st->drift_max, drift);
            }
        }
    }
    if (blockIdx.x == 0 && t < ld) {
        a.e[t] = es[t];
        if (t < k) a.ow[mnew + t] = gs[t];
    }
    lean_bar();
}

template <int PPL, int MAXD, bool RV>
__global__ void __launch_bounds__(op_threads_max(PPL), 1) k_prolong_onepass_tma(SolveArgs a, const double* sv,
                                                                      double* zout,
                                                                      cudaGraphConditionalHandle h,
                                                                      int ctl, int S, int P, int rsel, int lean) {
    pdl_entry();
    PcgState* st = a.st;
    if (st->done) {
        if (ctl && blockIdx.x == 0 && threadIdx.x == 0) {
            if (lean) loop_ctl_lean(st, h, ctl == 2);
            else loop_ctl_body(st, h, ctl == 2);
        }
        return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) st->op_grid = gridDim.x;
    // lean (DESIGN.md §3 "lean cycle"): 1 writes p = s + W e + beta p in place of
    // z (zout = p, its old rows staged with the tile), 2 the prologue's p = s + W e;
    // both reduce s.As and (W e).(A s) instead of r.z
    __shared__ double cs[(op_threads_max(PPL) / 32) * 2 * kGroup * PPL];  // column sums (cta_columns)
    __shared__ double lsm[5 * (2 * kGroup * PPL + 2)];  // lean: the coarse step's vectors
    __shared__ double lsc[8];  // lean: [e.Me, r.z, beta] of the coarse step (+ guard partials)
    // rsel: the residual the fused update + sweep wrote (r[(it + 1) & 1]), else r
    const double* rv = (rsel && !(st->it & 1)) ? a.r1 : a.r;
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);
    unsigned long long* asr = full + kOpMaxStages;
    unsigned long long* empty = asr + kOpMaxStages;
    unsigned char* stages = smem + 256;  // after 3 x kOpMaxStages barriers
    const int ld = a.k + (a.k & 1);
    const int pairs = ld >> 1;
    const unsigned wbytes = (unsigned)kOpTR * ld * 8;
    const int tile_nnz = kOpTR == 64 ? a.tile_nnz64 : a.tile_nnz128;
    const unsigned sbytes = op_stage_bytes(ld, MAXD ? -1 : tile_nnz);
    // stage layout: [W rows | s | r | mask | A s | p | CSR: row_ptr | values | columns]
    const unsigned s_off = wbytes, r_off = wbytes + kOpVec, m_off = wbytes + 2 * kOpVec;
    const unsigned as_off = m_off + round16(kOpTR * 4);
    const unsigned p_off = as_off + kOpVec;
    const unsigned rp_off = p_off + kOpVec;
    const unsigned v_off = rp_off + round16((kOpTR + 4) * 4);
    const unsigned c_off = v_off + round16((tile_nnz + 2) * 8);
    // CSR rows with implicit columns (PackArgs): the rows' masks are staged in
    // the column region, the offsets sit in shared memory
    const bool mk = MAXD == 0 && a.pk.mask != nullptr;
    __shared__ int pko[MAXD == 0 ? kMaxDia : 1];
    if (MAXD == 0 && mk && threadIdx.x < kMaxDia) pko[threadIdx.x] = a.pk.off[threadIdx.x];
    if (threadIdx.x == 0) {
        for (int s = 0; s < S; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&asr[s], 2);
            mbar_init(&empty[s], op_wpg(PPL));
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int ntiles = (a.n + kOpTR - 1) / kOpTR;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mb = a.dia.mbytes;
    double au[2 * PPL], av[2 * PPL];
#pragma unroll
    for (int t = 0; t < 2 * PPL; ++t) au[t] = av[t] = 0.0;
    double rz[2] = {0.0, 0.0};
    if (warp == 0) {
        // ---- producer (diagonal form): lane 0 issues each tile's bulk copies
        if (MAXD != 0 && lane == 0) {
            // ring position by counters (i % S, i / S with a run-time S cost an
            // emulated division per tile and warp)
            int stg = 0, rnd = 0;
            for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
                if (rnd > 0) mbar_wait(&empty[stg], (rnd - 1) & 1);
                unsigned char* base_s = stages + stg * sbytes;
                const int r0 = tile * kOpTR, rows = min(kOpTR, a.n - r0);
                const unsigned vb = round16(rows * 8);  // vectors are padded by 16 doubles
                const unsigned wb = (unsigned)rows * ld * 8;
                const unsigned mbb = round16(rows * mb);  // masks are padded by 16 B
                NLSP_CHECK(rows > 0 && rows <= kOpTR && wb <= s_off && m_off + mbb <= as_off && p_off + kOpVec <= sbytes);
                mbar_arrive_tx(&full[stg], wb + (sv ? vb : 0u) + vb + mbb + (lean == 1 ? vb : 0u));
                bulk_g2s(base_s, a.P + (long long)r0 * ld, wb, &full[stg]);
                if (sv) bulk_g2s(base_s + s_off, sv + r0, vb, &full[stg]);
                bulk_g2s(base_s + r_off, rv + r0, vb, &full[stg]);
                if (lean == 1) bulk_g2s(base_s + p_off, zout + r0, vb, &full[stg]);
                bulk_g2s(base_s + m_off, static_cast<const unsigned char*>(a.dia.mask) + (long long)r0 * mb,
                         mbb, &full[stg]);
                if (++stg == S) {
                    stg = 0;
                    ++rnd;
                }
            }
        }
        // ---- producer (CSR): the 32 lanes load the row_ptr bounds of 32
        // upcoming tiles at once, lane 0 issues each tile's bulk copies
        if (MAXD == 0)
        for (int base = 0;; base += 32) {
            if ((long long)blockIdx.x + (long long)base * gridDim.x >= ntiles) break;
            int b0 = 0, b1 = 0;
            if (MAXD == 0) {
                const long long my = (long long)blockIdx.x + (long long)(base + lane) * gridDim.x;
                if (my < ntiles) {
                    const int r0 = (int)my * kOpTR;
                    b0 = __ldg(a.rp + r0);
                    b1 = __ldg(a.rp + min(r0 + kOpTR, a.n));
                }
            }
            for (int j = 0; j < 32; ++j) {
                const int i = base + j;
                const long long tile = (long long)blockIdx.x + (long long)i * gridDim.x;
                if (tile >= ntiles) break;
                const int a0 = __shfl_sync(0xffffffffu, b0, j), a1 = __shfl_sync(0xffffffffu, b1, j);
                if (lane != 0) continue;
                const int stg = i % S;
                if (i >= S) mbar_wait(&empty[stg], ((i / S) - 1) & 1);
                unsigned char* base_s = stages + stg * sbytes;
                const int r0 = (int)tile * kOpTR, rows = min(kOpTR, a.n - r0);
                const unsigned vb = round16(rows * 8);  // vectors are padded by 16 doubles
                const unsigned wb = (unsigned)rows * ld * 8;
                const unsigned mbb = MAXD ? round16(rows * mb) : 0u;  // masks are padded by 16 B
                unsigned cb = 0, cvb = 0, ccb = 0;
                int s0 = 0, c0 = 0;
                if (MAXD == 0) {  // row_ptr slice, values and columns from 16-B aligned starts
                    s0 = a0 & ~1;
                    c0 = a0 & ~3;
                    cb = ((rows + 1 + 3) & ~3) * 4;
                    cvb = ((a1 - s0 + 1) & ~1) * 8;
                    ccb = mk ? ((rows + 3) & ~3) * 4 : ((a1 - c0 + 3) & ~3) * 4;
                }
                NLSP_CHECK(rows > 0 && rows <= kOpTR && a1 >= a0 && a1 - a0 <= tile_nnz);
                NLSP_CHECK(MAXD != 0 || (rp_off + cb <= v_off && v_off + cvb <= c_off && c_off + ccb <= sbytes));
                NLSP_CHECK(p_off + vb <= rp_off && as_off + kOpVec <= p_off);
                mbar_arrive_tx(&full[stg], wb + (sv ? vb : 0u) + vb + mbb + cb + cvb + ccb + (lean == 1 ? vb : 0u));
                bulk_g2s(base_s, a.P + (long long)r0 * ld, wb, &full[stg]);
                if (sv) bulk_g2s(base_s + s_off, sv + r0, vb, &full[stg]);
                bulk_g2s(base_s + r_off, rv + r0, vb, &full[stg]);
                if (lean == 1) bulk_g2s(base_s + p_off, zout + r0, vb, &full[stg]);
                if (MAXD)
                    bulk_g2s(base_s + m_off, static_cast<const unsigned char*>(a.dia.mask) + (long long)r0 * mb,
                             mbb, &full[stg]);
                if (MAXD == 0) {
                    bulk_g2s(base_s + rp_off, a.rp + r0, cb, &full[stg]);
                    if (cvb) bulk_g2s(base_s + v_off, a.v + s0, cvb, &full[stg]);
                    if (ccb && mk) bulk_g2s(base_s + c_off, a.pk.mask + r0, ccb, &full[stg]);
                    else if (ccb) bulk_g2s(base_s + c_off, a.ci + c0, ccb, &full[stg]);
                }
            }
        }
    } else if (warp <= 2 * P) {
        // ---- stencil warps: (A s)_row, one thread per row, sequential fma
        // chain in column order (bitwise the SpMV family's row sums)
        const int pair = (warp - 1) >> 1;
        const int lr0 = ((warp - 1) & 1) * 32 + lane;
        int stg = pair % S, rnd = pair / S;
        for (int tile = blockIdx.x + pair * gridDim.x; tile < ntiles; tile += P * gridDim.x) {
            // k > 48 (one W-product group, long tiles): the stencil warps run well
            // ahead of the W-product warps and sleep between polls (C4 0.4-1.6 % less
            // time per iteration over three A/B runs, fewer polls issued beside the
            // critical warps; at k = 48, two W groups, it measured +0.9 %: plain wait)
            if (PPL >= 4 && NLSP_STENCIL_SLEEP > 0) mbar_wait_relaxed(&full[stg], rnd & 1, NLSP_STENCIL_SLEEP);
            else mbar_wait(&full[stg], rnd & 1);
            unsigned char* base = stages + stg * sbytes;
            const int r0 = tile * kOpTR, rows = min(kOpTR, a.n - r0);
            for (int lr = lr0; lr < kOpTR; lr += 64) {
            double y = 0.0;
            if (sv && lr < rows) {
                const int row = r0 + lr;
                if constexpr (MAXD == 0) {
                    // the staged row: values from a 16-B aligned start s0, columns from c0
                    const int* rps = reinterpret_cast<const int*>(base + rp_off);
                    const double* vs = reinterpret_cast<const double*>(base + v_off);
                    const int* cs_ = reinterpret_cast<const int*>(base + c_off);
                    const int a0 = rps[0], s0 = a0 & ~1, c0 = a0 & ~3;
                    const int b = rps[lr], e = rps[lr + 1];
                    NLSP_CHECK(b >= a0 && e >= b && e - s0 <= tile_nnz + 2 && e - c0 <= tile_nnz + 8);
                    // 8 nonzeros per step: their staged values / columns and the
                    // gathers of s issued together, then the fma chain in column
                    // order (a rolled loop waits one L2 latency per nonzero:
                    // the stencil warps were the pass's bottleneck at C5)
                    unsigned pm = mk ? reinterpret_cast<const unsigned*>(cs_)[lr] : 0u;
                    for (int kk = b; kk < e; kk += 8) {
                        double vv[8], xx[8];
#pragma unroll
                        for (int c = 0; c < 8; ++c) {
                            const int q = kk + c;
                            const bool on = q < e;
                            vv[c] = on ? vs[q - s0] : 0.0;
                            int col = 0;
                            if (on) {
                                if (mk) {  // the next set bit of the row's mask
                                    col = row + pko[__ffs(pm) - 1];
                                    pm &= pm - 1u;
                                } else {
                                    col = cs_[q - c0];
                                }
                            }
                            xx[c] = on ? sv[col] : 0.0;
                        }
#pragma unroll
                        for (int c = 0; c < 8; ++c)
                            if (kk + c < e) y = fma(vv[c], xx[c], y);
                    }
                } else {
                    unsigned m;
                    const unsigned char* ms = base + m_off;
                    if (mb == 1) m = ms[lr];
                    else if (mb == 2) m = reinterpret_cast<const unsigned short*>(ms)[lr];
                    else m = reinterpret_cast<const unsigned*>(ms)[lr];
                    double g[MAXD], vv[RV ? MAXD : 1];
#pragma unroll
                    for (int t = 0; t < MAXD; ++t) {
                        const bool on = t < a.dia.d && ((m >> t) & 1u);
                        g[t] = on ? sv[row + a.dia.off[t]] : 0.0;
                        if (RV) vv[RV ? t : 0] = on ? __ldcs(a.dia.rv + (size_t)t * a.n + row) : 0.0;
                    }
#pragma unroll
                    for (int t = 0; t < MAXD; ++t)
                        if (t < a.dia.d && ((m >> t) & 1u)) y = fma(RV ? vv[RV ? t : 0] : a.dia.val[t], g[t], y);
                }
            }
            reinterpret_cast<double*>(base + as_off)[lr] = y;
            // lean: s.As summed here (the W-product warps are the pass's critical path)
            if (lean && sv && lr < rows) rz[0] = fma(reinterpret_cast<const double*>(base + s_off)[lr], y, rz[0]);
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&asr[stg]);
            stg += P;  // P <= S
            if (stg >= S) {
                stg -= S;
                ++rnd;
            }
        }
    } else {
        // ---- W-product warps: 8 lanes per row, 2 rows per group per tile
        constexpr int kOpWH = op_wh(PPL);
        constexpr int WPG = op_wpg(PPL);  // warps per W group
        const int cw = warp - 1 - 2 * P;
        const int wgrp = cw / WPG;
        const int grp = ((cw % WPG) * 32 + lane) >> 3, l = lane & (kGroup - 1);
        // lean: c by its recurrence, e, M e and beta while the producer fills the ring
        if (lean == 1) lean_coarse_step(LeanCoarse{a.Ainv, a.M, a.L, a.ow, a.e, st, a.k}, cw * 32 + lane, lsm, lsc);
        const double* esrc = lean == 1 ? lsm + 3 * (ld + 2) : a.e;
        const double lbeta = lean == 1 ? lsc[2] : 0.0;
        double ev[2 * PPL];
#pragma unroll
        for (int t = 0; t < PPL; ++t) {
            const int pi = l + kGroup * t;
            ev[2 * t] = pi < pairs ? esrc[2 * pi] : 0.0;
            ev[2 * t + 1] = pi < pairs ? esrc[2 * pi + 1] : 0.0;
        }
        int stg = wgrp % S, rnd = wgrp / S;
        for (int tile = blockIdx.x + wgrp * gridDim.x; tile < ntiles; tile += kOpWH * gridDim.x) {
            mbar_wait(&full[stg], rnd & 1);
            mbar_wait(&asr[stg], rnd & 1);
            const unsigned char* base = stages + stg * sbytes;
            const int r0 = tile * kOpTR, rows = min(kOpTR, a.n - r0);
            const double* ss = reinterpret_cast<const double*>(base + s_off);
            const double* rs = reinterpret_cast<const double*>(base + r_off);
            const double* as = reinterpret_cast<const double*>(base + as_off);
            const double* ps = reinterpret_cast<const double*>(base + p_off);
            // FULL: a whole tile of full-width rows (ld = 16 PPL) — no row or column
            // predicates and a compile-time row stride (the W-product warps are the
            // pass's critical path at the power-capped clock: ncu counted ~190
            // instructions per warp and tile with the predicated body for ~80 of work)
            auto wtile = [&](auto full_c) {
                constexpr bool FULL = decltype(full_c)::value;
                const int ldr = FULL ? 2 * kGroup * PPL : ld;
#pragma unroll
                for (int u = 0; u < kOpTR / (WPG * 4); ++u) {
                    const int lr = grp + WPG * 4 * u;
                    const bool ok = FULL || lr < rows;  // every lane still runs the group shuffles
                    const double* wrow = reinterpret_cast<const double*>(base) + lr * ldr;
                    const double rr = ok ? rs[lr] : 0.0, ar = ok ? as[lr] : 0.0;
                    double part = 0.0;
#pragma unroll
                    for (int t = 0; t < PPL; ++t) {
                        const int pi = l + kGroup * t;
                        if (FULL || (ok && pi < pairs)) {
                            const double2 w = *reinterpret_cast<const double2*>(wrow + 2 * pi);
                            part = fma(w.x, ev[2 * t], part);
                            part = fma(w.y, ev[2 * t + 1], part);
                            au[2 * t] = fma(w.x, rr, au[2 * t]);
                            au[2 * t + 1] = fma(w.y, rr, au[2 * t + 1]);
                            av[2 * t] = fma(w.x, ar, av[2 * t]);
                            av[2 * t + 1] = fma(w.y, ar, av[2 * t + 1]);
                        }
                    }
                    const double sum = group_sum(part);
                    if (ok && l == 0) {
                        const double si = sv ? ss[lr] : 0.0;
                        const double zi = si + sum;
                        if (lean) {
                            // p = z + beta p (two_level.hpp:182, the fma of GPupd);
                            // s.As is summed by the stencil warps, (W e).(A s) = e.v
                            // from this CTA's column sums of v below
                            zout[r0 + lr] = lean == 1 ? fma(lbeta, ps[lr], zi) : zi;
                        } else {
                            zout[r0 + lr] = zi;
                            rz[0] = fma(rr, zi, rz[0]);
                        }
                    }
                }
            };
            // (diagonal forms only: with the CSR stencil in the kernel the second
            // body measured +1.9 % at C5, against -1.5 % at C3)
            if constexpr (MAXD != 0) {
                if (rows == kOpTR && pairs == kGroup * PPL) wtile(std::true_type{});
                else wtile(std::false_type{});
            } else {
                wtile(std::false_type{});
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&empty[stg]);
            stg += kOpWH;  // kOpWH <= S
            if (stg >= S) {
                stg -= S;
                ++rnd;
            }
        }
    }
    {
        const long long G = gridDim.x;
        cta_columns<PPL>(au, cs, ld, a.opart);
        if (lean) cta_columns<PPL>(av, cs, ld, a.opart + ld * G, lean == 1 ? lsm + 3 * (ld + 2) : a.e, &rz[1]);
        else cta_columns<PPL>(av, cs, ld, a.opart + ld * G);
    }
    double tot[2];
    if (grid_reduce<2>(rz, a.partials, &st->counter[kTkProlong], tot) && threadIdx.x == 0) {
        if (lean) {
            // p.Ap = z.Az - beta r.z / alpha_prev (exact-arithmetic identities of CG:
            // z_i.A p_{i-1} = -r.z_i / alpha_{i-1}, p_{i-1}.A p_{i-1} = r.z_{i-1} / alpha_{i-1})
            // the coarse step's scalars (this CTA's copy; the prologue: k_lean_init's)
            const double eme = lean == 1 ? lsc[0] : st->lean_eme;
            const double gnew = lean == 1 ? lsc[1] : st->rz_new;
            const double bnew = lean == 1 ? lsc[2] : 0.0;
            const double aold = st->alpha;
            const double zaz = tot[0] + 2.0 * tot[1] + eme;
            const double pap = lean == 1 ? zaz - bnew * gnew / aold : zaz;
            st->pap_pred = pap;
            st->alpha_prev = aold;
            st->alpha = gnew / pap;
            st->beta = bnew;
            st->rz_new = gnew;
            if (ctl) loop_ctl_lean(st, h, ctl == 2);
        } else {
            st->rz_new = tot[0];
            if (ctl) loop_ctl_body(st, h, ctl == 2);
        }
    }
}

// Every CTA: sum columns of the previous one-pass prolongation's partials (a
// column per CTA, fixed order) into u_i (ow slot it & 1; u_{i-1} stays in the
// other) and v_i (ow + 2 ld).
__device__ void onepass_colsums(const SolveArgs& a) {
    const PcgState* st = a.st;
    const int ld = a.k + (a.k & 1);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __shared__ double wsum[32];
    const long long G = st->op_grid;
    const int ucur = (int)(st->it & 1) * ld;
    for (int j = blockIdx.x; j < 2 * ld; j += gridDim.x) {
        double t = 0.0;
        for (long long b = threadIdx.x; b < G; b += blockDim.x) t += __ldcg(a.opart + j * G + b);
        t = warp_sum(t);
        if (lane == 0) wsum[warp] = t;
        __syncthreads();
        if (threadIdx.x == 0) {
            double tt = 0.0;
            for (int w = 0; w < nw; ++w) tt += wsum[w];
            a.ow[j < ld ? ucur + j : ld + j] = tt;  // u_i -> its slot, v_i -> [2 ld, 3 ld)
            __threadfence();
        }
        __syncthreads();
    }
}

// The last CTA of the x/r update (whole CTA; rrt = ||r_{i+1}||^2): history +
// convergence test (two_level.hpp:168-176), then the one-pass restriction
// c = u_i - alpha_i (v_i + M e_i + beta_i (u_{i-1} - u_i) / alpha_{i-1}) and
// e = A_c^-1 c.
__device__ void onepass_last(const SolveArgs& a, double rrt, double alpha) {
    PcgState* st = a.st;
    __shared__ int go_on;
    if (threadIdx.x == 0) {
        const double rel = sqrt(rrt) / st->bnorm;
        st->rr = rrt;
        st->last_rel = rel;
        a.hist[st->it - st->hist_base] = rel;
        st->iterations = st->it + 1;
        if (rel < st->delta) {
            st->converged = 1;
            st->done = 1;
        }
        go_on = !st->done;
    }
    __syncthreads();
    if (!go_on) return;
    __threadfence();
    __shared__ double es[kOnePassK + 2], gs[kOnePassK + 2], cs[kOnePassK + 2];
    const int k = a.k, ld = a.k + (a.k & 1);
    const int warp = threadIdx.x >> 5;
    const bool first = st->first != 0;
    const double beta = st->beta, alpha_prev = st->alpha_prev;
    const int ucur = (int)(st->it & 1) * ld, uprev = ld - ucur;
    for (int j = threadIdx.x; j < k; j += blockDim.x) es[j] = __ldcg(a.e + j);
    __syncthreads();
    coarse_apply_inverse(a.M, k, es, gs);  // M e_i
    __syncthreads();
    // Guard: the previous iteration's c_i came from the recurrence; u_i = W^T r_i
    // was then formed directly by the pass over W, so their gap is the one-step
    // error of the recurrence. Its max |c - u| / max |u| over the
    // solve is reported (nlsp_solve_report.onepass_drift); above the tolerance
    // the host re-runs the solve on the folded cycle (run_pcg).
    if (!first) {
        __shared__ double dred[2][32];
        double d = 0.0, um = 0.0;
        for (int j = threadIdx.x; j < k; j += blockDim.x) {
            const double u = __ldcg(a.ow + ucur + j);
            d = fmax(d, fabs(__ldcg(a.ow + 3 * ld + j) - u));
            um = fmax(um, fabs(u));
        }
        for (int o = 16; o; o >>= 1) {
            d = fmax(d, __shfl_xor_sync(0xffffffffu, d, o));
            um = fmax(um, __shfl_xor_sync(0xffffffffu, um, o));
        }
        if ((threadIdx.x & 31) == 0) {
            dred[0][warp] = d;
            dred[1][warp] = um;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
                d = fmax(d, dred[0][w]);
                um = fmax(um, dred[1][w]);
            }
            const double drift = um > 0.0 ? d / um : 0.0;
            st->drift_max = fmax(st->drift_max, drift);
        }
    }
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        const double u = __ldcg(a.ow + ucur + j);
        double g = __ldcg(a.ow + 2 * ld + j) + gs[j];  // v + M e
        if (!first) g = fma(beta, (__ldcg(a.ow + uprev + j) - u) / alpha_prev, g);  // + beta W^T q_{i-1}
        const double c = fma(-alpha, g, u);            // c = u - alpha g
        cs[j] = c;
        a.ow[3 * ld + j] = c;  // compared with the direct u_{i+1} next iteration
    }
    __syncthreads();
    if (a.Ainv) coarse_apply_inverse(a.Ainv, k, cs, a.e);
    else if (warp == 0) coarse_solve_warp(a.L, k, cs, a.e);
    if (threadIdx.x == 0) {
        if (k & 1) a.e[k] = 0.0;  // padded column
        st->alpha_prev = alpha;
    }
}

// x += alpha p, r -= alpha q, ||r||^2 (two_level.hpp:164-170), with the
// one-pass column sums and, in the last CTA, the one-pass restriction.
__global__ void __launch_bounds__(kThreads) k_update_onepass(SolveArgs a) {
    pdl_entry();
    PcgState* st = a.st;
    if (st->done) return;
    const double alpha = st->alpha;
    const double* p = (st->it & 1) ? a.p1 : a.p0;
    double s[1] = {0.0};
    const long long npairs = a.n >> 1;
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < npairs; t += stride) {
        const long long i = 2 * t;
        const double2 pv = *reinterpret_cast<const double2*>(p + i);
        const double2 qv = *reinterpret_cast<const double2*>(a.q + i);
        const double2 xv = *reinterpret_cast<const double2*>(a.x + i);
        const double2 rv = *reinterpret_cast<const double2*>(a.r + i);
        double2 xo, ro;
        xo.x = fma(alpha, pv.x, xv.x);
        xo.y = fma(alpha, pv.y, xv.y);
        ro.x = fma(-alpha, qv.x, rv.x);
        ro.y = fma(-alpha, qv.y, rv.y);
        s[0] = fma(ro.x, ro.x, s[0]);
        s[0] = fma(ro.y, ro.y, s[0]);
        *reinterpret_cast<double2*>(a.x + i) = xo;
        *reinterpret_cast<double2*>(a.r + i) = ro;
    }
    if ((a.n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
        const long long i = a.n - 1;
        a.x[i] = fma(alpha, p[i], a.x[i]);
        const double ro = fma(-alpha, a.q[i], a.r[i]);
        a.r[i] = ro;
        s[0] = fma(ro, ro, s[0]);
    }
    onepass_colsums(a);
    double tot[1];
    if (grid_reduce<1>(s, a.partials, &st->counter[kTkUpdate], tot)) onepass_last(a, tot[0], alpha);
}

// The x/r update fused with the smoothing sweeps of the one-pass cycle at
// nu1 = nu2 = 1 (T = 2): s = s1 + w D^-1 (r_new - A s1), s1 = w D^-1 r_new,
// with r_new = r - alpha q formed inside the gather (bitwise the values the
// separate update writes). r is double-buffered by iteration parity (the
// gathers read the old residual while rows write the new one): read r[it & 1],
// write r[(it + 1) & 1]. Plus x += alpha p, ||r_new||^2 and the one-pass hooks.
template <bool CW>
struct OpUpdSweep {
    static constexpr int NV = 1;
    static constexpr int TICKET = kTkUpdate;
    static constexpr bool CTA_HOOKS = true;
    double alpha;
    const double* rc;
    double* rn;
    const double* q;
    const double* wd;
    const double* p;
    double* x;
    double* sout;
    double wc;  // constant w D^-1 (see GWdr), else 0
    __device__ __forceinline__ void init(const SolveArgs& a) {
        const bool odd = a.st->it & 1;
        wc = a.wdc;
        alpha = a.st->alpha;
        rc = odd ? a.r1 : a.r;
        rn = odd ? a.r : a.r1;
        q = a.q;
        wd = a.wd;
        p = odd ? a.p1 : a.p0;
        x = a.x;
        sout = a.zt0;
    }
    __device__ __forceinline__ double operator()(int j) const {
        return (CW ? wc : wd[j]) * fma(-alpha, q[j], rc[j]);
    }
    struct Pre {
        double ri, wi, xi, pi;
    };
    __device__ __forceinline__ Pre pre(int i) const {
        return Pre{fma(-alpha, q[i], rc[i]), CW ? wc : wd[i], x[i], p[i]};
    }
    __device__ __forceinline__ void row(int i, double y, double* s, const Pre& pr) const {
        const double gi = pr.wi * pr.ri;
        sout[i] = fma(pr.wi, pr.ri - y, gi);
        rn[i] = pr.ri;
        x[i] = fma(alpha, pr.pi, pr.xi);
        s[0] = fma(pr.ri, pr.ri, s[0]);
    }
    __device__ __forceinline__ void row(int i, double y, double* s) const { row(i, y, s, pre(i)); }
    __device__ __forceinline__ void cta_pre(const SolveArgs& a) const { onepass_colsums(a); }
    __device__ __forceinline__ void cta_last(const SolveArgs& a, const double* tot) const {
        onepass_last(a, tot[0], alpha);
    }
    __device__ __forceinline__ void finish(PcgState*, const double*) const {}
};

// ============================================================ lean cycle ==
// The lean one-pass cycle: beta_{i+1} is known BEFORE the pass
// over W (r.z = r.s + c.e with c by its recurrence), so the pass writes
// p = s + W e + beta p directly, and alpha_{i+1} is known right AFTER it
// (p.Ap = z.Az - beta r.z / alpha_i, z.Az = s.As + 2 (W e).(A s) + e.M e, the
// Chronopoulos-Gear form), so q = A p is never stored and the smoother gathers
// r alone. Three kernels per iteration at nu = 1/1:
//   OpSpmvUpd     q = A p in the gather of p; x += alpha p, r -= alpha q (in
//                 place), ||r||^2 -> convergence; p.q directly: the NotSpd test
//                 and the guard of the predicted p.Ap
//   OpSweepLean   s = S_2(r) gathering r alone; r.s; last CTA: c by its
//                 recurrence, e = A_c^-1 c, M e, c.e, e.M e, beta
//   k_prolong_onepass_tma (lean)  p = s + W e + beta p, u, v, s.As, (W e).(A s)
//                 -> alpha, loop control
// 88n + 3A vector/matrix bytes beside W instead of 112n + 3A, and 7 + 7 gathers
// of one array per row instead of 14 + 14 of two.

// x += alpha p, r -= alpha (A p) in place; tot = [p.Ap, ||r_new||^2]
struct OpSpmvUpd {
    static constexpr int NV = 2;
    static constexpr int TICKET = kTkSpmvP;
    const double* p;
    double* x;
    double* r;
    double* a_hist;
    double alpha;
    // the last CTA's scalars, loaded at kernel start (not after the grid sum)
    double pap_pred, bnorm, delta, drift0;
    long long hidx, itv;
    __device__ __forceinline__ void init(const SolveArgs& a) {
        p = a.p0;
        x = a.x;
        r = a.r;
        a_hist = a.hist;
        const PcgState* st = a.st;
        alpha = st->alpha;
        pap_pred = st->pap_pred;
        bnorm = st->bnorm;
        delta = st->delta;
        drift0 = st->pap_drift;
        itv = st->it;
        hidx = itv - st->hist_base;
    }
    __device__ __forceinline__ double operator()(int j) const { return p[j]; }
    struct Pre {
        double pi, xi, ri;
    };
    __device__ __forceinline__ Pre pre(int i) const { return Pre{p[i], x[i], r[i]}; }
    __device__ __forceinline__ void row(int i, double y, double* s, const Pre& pr) const {
        const double rn = fma(-alpha, y, pr.ri);
        x[i] = fma(alpha, pr.pi, pr.xi);
        r[i] = rn;
        s[0] = fma(pr.pi, y, s[0]);
        s[1] = fma(rn, rn, s[1]);
    }
    __device__ __forceinline__ void row(int i, double y, double* s) const { row(i, y, s, pre(i)); }
    // two_level.hpp:159-176: p^T A p <= 0 -> NotSpdError; history entry and the
    // convergence test on ||r_new|| / ||b||
    __device__ __forceinline__ void finish(PcgState* st, const double* tot) const {
        const double pap = tot[0];
        st->pap = pap;
        if (pap <= 0.0) {
            st->error = kErrNotSpd;
            st->done = 1;
            return;
        }
        // guard: the alpha this kernel used came from the predicted p.Ap
        double dev = fabs(pap_pred - pap) / pap;
        if (!(dev == dev) || dev > 1e300) dev = 1e300;
        if (dev > drift0) st->pap_drift = dev;
        if (dev > 1e-6) {  // the prediction broke down: stop, the host re-runs on the folded cycle
            st->done = 1;
            return;
        }
        const double rel = sqrt(tot[1]) / bnorm;
        st->rr = tot[1];
        st->last_rel = rel;
        a_hist[hidx] = rel;
        st->iterations = itv + 1;
        if (rel < delta) {
            st->converged = 1;
            st->done = 1;
        }
    }
};

// s = S_2(r) = s1 + w D^-1 (r - A s1), s1 = w D^-1 r (the arithmetic of
// OpUpdSweep on the residual OpSpmvUpd wrote), r.s, and the lean hooks
template <bool CW>
struct OpSweepLean {
    static constexpr int NV = 1;
    static constexpr int TICKET = kTkUpdate;
    static constexpr bool CTA_HOOKS = true;
    const double* r;
    const double* wd;
    double* sout;
    double wc;
    __device__ __forceinline__ void init(const SolveArgs& a) {
        r = a.r;
        wd = a.wd;
        wc = a.wdc;
        sout = a.zt0;
    }
    __device__ __forceinline__ double operator()(int j) const { return (CW ? wc : wd[j]) * r[j]; }
    struct Pre {
        double ri, wi;
    };
    __device__ __forceinline__ Pre pre(int i) const { return Pre{r[i], CW ? wc : wd[i]}; }
    __device__ __forceinline__ void row(int i, double y, double* s, const Pre& pr) const {
        const double gi = pr.wi * pr.ri;
        const double si = fma(pr.wi, pr.ri - y, gi);
        sout[i] = si;
        s[0] = fma(pr.ri, si, s[0]);
    }
    __device__ __forceinline__ void row(int i, double y, double* s) const { row(i, y, s, pre(i)); }
    __device__ __forceinline__ void cta_pre(const SolveArgs& a) const { onepass_colsums(a); }
    // r.s (of this s: the last sweep's r.s replaces it when T > 2)
    __device__ __forceinline__ void cta_last(const SolveArgs& a, const double* tot) const {
        if (threadIdx.x == 0) a.st->rz_new = tot[0];
    }
    __device__ __forceinline__ void finish(PcgState*, const double*) const {}
};

// Lean prologue, after c = W^T r_0, e_0 (restrict_finish kept c in ow) and the
// sweeps (r.s in st->rz_new when has_s): M e_0, c.e, e.M e; r.z = r.s + c.e;
// beta = 0.
__global__ void __launch_bounds__(kThreads) k_lean_init(SolveArgs a, int has_s) {
    PcgState* st = a.st;
    if (st->done) return;
    __shared__ double es[kOnePassK + 2], gs[kOnePassK + 2];
    const int k = a.k, ld = a.k + (a.k & 1);
    for (int j = threadIdx.x; j < k; j += blockDim.x) es[j] = __ldcg(a.e + j);
    __syncthreads();
    coarse_apply_inverse(a.M, k, es, gs);
    __syncthreads();
    for (int j = threadIdx.x; j < k; j += blockDim.x) a.ow[4 * ld + j] = gs[j];
    if (threadIdx.x < 32) {
        double ce = 0.0, eme = 0.0;
        for (int j = threadIdx.x; j < k; j += 32) {
            ce = fma(__ldcg(a.ow + 3 * ld + j), es[j], ce);
            eme = fma(es[j], gs[j], eme);
        }
        ce = warp_sum(ce);
        eme = warp_sum(eme);
        if (threadIdx.x == 0) {
            st->lean_ce = ce;
            st->lean_eme = eme;
            st->rz_new = (has_s ? st->rz_new : 0.0) + ce;
            st->beta = 0.0;
            st->alpha_prev = 0.0;
        }
    }
}

#include "march.cuh"
#include "lmarch.cuh"

// ======================================================== host launchers ==

namespace {
// <<<g, b, smem, c.s>>>, or with programmatic stream serialization when c.pdl
template <class... KArgs, class... Args>
void klaunch(const LaunchCtx& c, void (*f)(KArgs...), dim3 g, dim3 b, size_t smem, Args&&... args) {
    if (!c.pdl) {
        f<<<g, b, smem, c.s>>>(std::forward<Args>(args)...);
        return;
    }
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = g;
    cfg.blockDim = b;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = c.s;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, f, std::forward<Args>(args)...);
}
// Persistent, occupancy-sized grids: min(work, resident CTAs on all SMs).
int occ_blocks(const void* f) {
    static std::mutex mu;
    static std::unordered_map<const void*, int> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(f);
    if (it != cache.end()) return it->second;
    int nb = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kThreads, 0) != cudaSuccess || nb < 1)
        nb = 1;
    cudaGetLastError();
    cache[f] = nb;
    return nb;
}
int occ_grid(const LaunchCtx& c, const void* f, long long units, long long per_cta) {
    long long g = (units + per_cta - 1) / per_cta;
    long long cap = (long long)c.num_sms * occ_blocks(f);
    if (cap > kMaxGrid) cap = kMaxGrid;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return static_cast<int>(g);
}
// row kernels: units = rows, per CTA = warps * 4 * U rows
template <int U, class... KArgs, class... Args>
void launch_rows(const LaunchCtx& c, void (*f)(KArgs...), long long n, Args&&... args) {
    const int g = occ_grid(c, reinterpret_cast<const void*>(f), n, (kThreads / 32) * kRowsPerWarp * U);
    klaunch(c, f, g, kThreads, 0, std::forward<Args>(args)...);
}
// TMA-staged kernels: one CTA = 8 consumer warps + 1 producer warp, dynamic
// shared memory for the stage ring, grid = min(tiles, resident CTAs).
template <class... KArgs, class... Args>
void launch_tma(const LaunchCtx& c, void (*f)(KArgs...), long long ntiles, size_t smem,
                Args&&... args) {
    static std::mutex mu;
    static std::unordered_map<const void*, size_t> attr;
    static std::unordered_map<unsigned long long, int> occ;
    const void* fp = reinterpret_cast<const void*>(f);
    int nb = 1;
    {
        std::lock_guard<std::mutex> lk(mu);
        size_t& cur = attr[fp];
        if (smem > cur) {
            cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cur = smem;
        }
        const unsigned long long key = reinterpret_cast<unsigned long long>(fp) * 1315423911ull ^ smem;
        auto it = occ.find(key);
        if (it == occ.end()) {
            if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, f, kTmaThreads, smem) != cudaSuccess ||
                nb < 1)
                nb = 1;
            cudaGetLastError();
            occ[key] = nb;
        } else {
            nb = it->second;
        }
    }
    long long g = (long long)c.num_sms * nb;
    if (g > kMaxGrid) g = kMaxGrid;
    if (g > ntiles) g = ntiles;
    if (g < 1) g = 1;
    klaunch(c, f, (int)g, kTmaThreads, smem, std::forward<Args>(args)...);
}
// element kernels: units = elements (2 per thread)
template <class... KArgs, class... Args>
void launch_elems(const LaunchCtx& c, void (*f)(KArgs...), long long n, Args&&... args) {
    const int g = occ_grid(c, reinterpret_cast<const void*>(f), n, 2LL * kThreads);
    klaunch(c, f, g, kThreads, 0, std::forward<Args>(args)...);
}
inline void count(const LaunchCtx& c) { ++*c.launches; }
}  // namespace

void launch_state_init(const LaunchCtx& c, PcgState* st, double delta, long long max_it) {
    k_state_init<<<1, 1, 0, c.s>>>(st, delta, max_it);
    count(c);
}

void launch_bnorm(const LaunchCtx& c, const SolveArgs& a) {
    launch_elems(c, k_bnorm, a.n, a);
    count(c);
}

void launch_init_simple(const LaunchCtx& c, const SolveArgs& a, int mode) {
    if (mode == 1)
        launch_elems(c, k_init_simple<1>, a.n, a);
    else
        launch_elems(c, k_init_simple<0>, a.n, a);
    count(c);
}

void launch_state_continue(const LaunchCtx& c, PcgState* st, long long max_it, long long base) {
    k_state_continue<<<1, 1, 0, c.s>>>(st, max_it, base);
    count(c);
}

void launch_init_ctl(const LaunchCtx& c, PcgState* st) {
    k_init_ctl<<<1, 1, 0, c.s>>>(st);
    count(c);
}

#ifndef NLSP_TMA
#define NLSP_TMA 1
#endif
// 2 stages of 256-row tiles: two CTAs (16 consumer warps) per SM instead of one
// with 3 stages — the staged SpMV family is latency-bound (ncu at C5: 14 %
// occupancy, 65 % of the stalls on the gathers). Measured at C5, us per
// iteration: 3 stages 141.6; 2 stages 125.1, with the register cap of 3 CTAs
// 119.8; 2 lanes per row (128-row tiles) 122.0-123.9; 4 lanes 134.0.
#ifndef NLSP_SPMV_STAGES
#define NLSP_SPMV_STAGES 2
#endif
#ifndef NLSP_RESTRICT_STAGES
#define NLSP_RESTRICT_STAGES 2
#endif
#ifndef NLSP_SPMV_G
#define NLSP_SPMV_G 1
#endif
#ifndef NLSP_SPMV_U
#define NLSP_SPMV_U 1
#endif
constexpr int kSpmvTR = kConsumerWarps * NLSP_SPMV_U * (32 / NLSP_SPMV_G);
constexpr int kRestrictTR = kConsumerWarps * 8;

size_t spmv_stage_smem(const SolveArgs& a) {
    return 128 + (size_t)NLSP_SPMV_STAGES * StageLayout(kSpmvTR, tile_nnz_for(a, kSpmvTR), 0, false).bytes;
}
size_t restrict_stage_smem(const SolveArgs& a) {
    const int ld = a.k + (a.k & 1);
    return 64 + 2 * kRestrictTR * 8 +
           (size_t)NLSP_RESTRICT_STAGES * StageLayout(kRestrictTR, a.tile_nnz64, ld, true).bytes;
}
long long spmv_tiles(const SolveArgs& a) { return (a.n + kSpmvTR - 1) / kSpmvTR; }
long long restrict_tiles(const SolveArgs& a) { return (a.n + kRestrictTR - 1) / kRestrictTR; }

template <int SKIP, class Op>
void launch_spmv_op(const LaunchCtx& c, const SolveArgs& a, const Op& op) {
    // one pass over a row covers G * CH nonzeros: size CH from the longest row
    constexpr int G = NLSP_SPMV_G, U = NLSP_SPMV_U, S = NLSP_SPMV_STAGES;
    const int need = (a.max_row + G - 1) / G;
    const long long nt = spmv_tiles(a);
    const size_t sm = spmv_stage_smem(a);
    if constexpr (G == 1) {
        if (a.pk.mask) {  // implicit columns
            if (need <= 8) launch_tma(c, k_spmv_tma<G, U, S, SKIP, 8, Op, true>, nt, sm, a, op);
            else if (need <= 12) launch_tma(c, k_spmv_tma<G, U, S, SKIP, 12, Op, true>, nt, sm, a, op);
            else launch_tma(c, k_spmv_tma<G, U, S, SKIP, 16, Op, true>, nt, sm, a, op);
            return;
        }
    }
    if (need <= 8) launch_tma(c, k_spmv_tma<G, U, S, SKIP, 8, Op>, nt, sm, a, op);
    else if (need <= 12) launch_tma(c, k_spmv_tma<G, U, S, SKIP, 12, Op>, nt, sm, a, op);
    else launch_tma(c, k_spmv_tma<G, U, S, SKIP, 16, Op>, nt, sm, a, op);
}

template <int SKIP, class Op>
void launch_dia_op(const LaunchCtx& c, const SolveArgs& a, const Op& op) {
    auto go = [&](auto kern) {
        const int g = occ_grid(c, reinterpret_cast<const void*>(kern), a.n, kThreads);
        klaunch(c, kern, g, kThreads, 0, a, op);
    };
    const bool rv = a.dia.kind == 2;
#define NLSP_DIA_GO(D, MT, EX) \
    do { if (rv) go(k_spmv_dia<D, MT, true, SKIP, EX, Op>); else go(k_spmv_dia<D, MT, false, SKIP, EX, Op>); } while (0)
    if (NLSP_DIA_EXACT && a.dia.d == 5) NLSP_DIA_GO(5, unsigned char, true);
    else if (NLSP_DIA_EXACT && a.dia.d == 7) NLSP_DIA_GO(7, unsigned char, true);
    else if (NLSP_DIA_EXACT && a.dia.d == 9) NLSP_DIA_GO(9, unsigned short, true);
    else if (a.dia.d <= 8) NLSP_DIA_GO(8, unsigned char, false);
    else if (a.dia.d <= 16) NLSP_DIA_GO(16, unsigned short, false);
    else if (a.dia.d <= 24) NLSP_DIA_GO(24, unsigned int, false);
    else NLSP_DIA_GO(32, unsigned int, false);
#undef NLSP_DIA_GO
}

// ---- plane-march kernels (march.cuh) --------------------------------------
// NLSP_MARCH: 0 (default) never; 1 whenever the diagonal form has a plane
// geometry; 2 from n >= 2^18 rows. Off by default: measured slower than the
// direct kernels on every configuration ("plane march") — the
// consumer warps are issue-bound at one or two CTAs per SM, where the direct
// kernels keep 32 warps of independent gathers in flight.
static int march_mode() {
    static const int m = [] {
        const char* e = std::getenv("NLSP_MARCH");
        return e ? std::atoi(e) : 0;
    }();
    return m;
}
// two CTAs per SM (34 warps: the stencil phase is latency-bound at 17)
constexpr unsigned kMarchBudget = 104 * 1024;
constexpr int kMarchMinRing = 5;

struct MarchPlan {
    MarchGeom g;
    size_t smem;
};

// Slab width C (a divisor of the plane P): the widest whose ring slot lets
// kMarchMinRing planes in flight, and at most n / (SMs x 16) rows so every CTA
// marches >= 16 plane-steps (the march's two halo planes amortised).
static bool march_plan(const LaunchCtx& c, const SolveArgs& a, int nh, int no, MarchPlan* out) {
    const int mode = march_mode();
    if (mode == 0 || !a.dia.kind || a.dia.plane <= 0) return false;
    if (mode == 2 && a.n < (1 << 18)) return false;
    const long long P = a.dia.plane, n = a.n;
    const int h = a.dia.halo, mb = a.dia.mbytes;
    const long long cmax = std::max<long long>(16, n / ((long long)c.num_sms * 16));
    // prefer slabs that give every consumer thread the same number of rows
    for (int pass = 0; pass < 2; ++pass)
    for (long long k = 1; k <= P; ++k) {
        if (P % k) continue;
        const long long C = P / k;
        if (C > cmax) continue;
        const long long nt = kMarchConsumers * 32;
        if (pass == 0 && 4 * C < 3 * ((C + nt - 1) / nt) * nt) continue;  // last row pass >= 75 % full
        const unsigned hcap = (unsigned)((((C + 2 * h) * 8 + 15) & ~15ll) + 32);
        const unsigned ocap = (unsigned)(((C * 8 + 15) & ~15ll) + 32);
        const unsigned mcap = (unsigned)(((C * mb + 15) & ~15ll) + 32);
        const unsigned slot = nh * hcap + no * ocap + mcap;
        const int R = (int)std::min<unsigned>(8, kMarchBudget / slot);
        if (R < kMarchMinRing) continue;
        MarchGeom g{};
        g.P = P;
        g.h = h;
        g.C = (int)C;
        g.S = (int)(P / C);
        g.Z = (int)(n / P);
        g.R = R;
        g.slot = slot;
        g.hcap = hcap;
        g.ocap = ocap;
        g.mcap = mcap;
        out->g = g;
        out->smem = 256 + (size_t)R * slot;
        return true;
    }
    return false;
}

// whether spmv_p runs as a plane march on this matrix (nlsp_csr_geometry)
bool march_planned(const LaunchCtx& c, const SolveArgs& a) {
    MarchPlan pl;
    return march_plan(c, a, MOpSpmvP::NH, MOpSpmvP::NO + (a.dia.kind == 2 ? a.dia.d : 0), &pl);
}

template <class Op>
static bool launch_march_op(const LaunchCtx& c, const SolveArgs& a, const Op& op) {
    const bool rv = a.dia.kind == 2;
    MarchPlan pl;
    if (!march_plan(c, a, Op::NH, Op::NO + (rv ? a.dia.d : 0), &pl)) return false;
    if (Op::NH + Op::NO + (rv ? a.dia.d : 0) > kMarchMaxArrays) return false;
    auto go = [&](auto kern) {
        static std::mutex mu;
        static std::unordered_map<unsigned long long, int> occ;
        int nb = 1;
        {
            std::lock_guard<std::mutex> lk(mu);
            const unsigned long long key = reinterpret_cast<unsigned long long>(reinterpret_cast<const void*>(kern)) *
                                               1315423911ull ^ pl.smem;
            auto it = occ.find(key);
            if (it == occ.end()) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pl.smem);
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, kMarchThreads, pl.smem) != cudaSuccess ||
                    nb < 1)
                    nb = 1;
                cudaGetLastError();
                occ[key] = nb;
            } else {
                nb = it->second;
            }
        }
        long long g = (long long)c.num_sms * nb;
        const long long T = (long long)pl.g.S * pl.g.Z;
        if (g > T) g = T;
        if (g > kMaxGrid) g = kMaxGrid;
        klaunch(c, kern, (int)g, kMarchThreads, pl.smem, a, op, pl.g);
    };
#define NLSP_MARCH_GO(D, MT, EX) \
    do { if (rv) go(k_march<Op, D, MT, true, EX>); else go(k_march<Op, D, MT, false, EX>); } while (0)
    if (a.dia.d == 5) NLSP_MARCH_GO(5, unsigned char, true);
    else if (a.dia.d == 7) NLSP_MARCH_GO(7, unsigned char, true);
    else if (a.dia.d == 9) NLSP_MARCH_GO(9, unsigned short, true);
    else if (a.dia.d <= 8) NLSP_MARCH_GO(8, unsigned char, false);
    else if (a.dia.d <= 16 && !rv) go(k_march<Op, 16, unsigned short, false, false>);
    else return false;
#undef NLSP_MARCH_GO
    return true;
}

// ---- fused line march (lmarch.cuh) -----------------------------------------
static int lmarch_env(const char* name, int dflt) {
    const char* e = std::getenv(name);
    return e ? std::atoi(e) : dflt;
}

template <int PAT>
static bool line_pattern_ok(const SolveArgs& a, long long Lw) {
    using Pat = LinePat<PAT>;
    if (a.dia.d != PAT) return false;
    for (int t = 0; t < PAT; ++t)
        if (a.dia.off[t] != Pat::dl(t) * Lw + Pat::dx(t)) return false;
    return true;
}

// The x/r update and all T sweeps in one line march (k_lfused): 2D
// constant-coefficient patterns, T = 2 or 4. NLSP_LFUSED=0 keeps the separate kernels.
// whether the fused line march runs on this matrix (0, or its pattern: 5 / 9)
int lfused_pattern(const SolveArgs& a, unsigned long long T) {
    static const int on = lmarch_env("NLSP_LFUSED", NLSP_LFUSED_DEFAULT);
    if (!on || a.dia.kind != 1 || a.wdc == 0.0 || (T != 2 && T != 4) || a.dia.plane <= 0 || a.dia.halo > 2) return 0;
    if (a.n < (1 << 16)) return 0;
    const long long Lw = a.dia.plane;
    if (Lw < 128 || a.n % Lw) return 0;
    if (a.n / Lw < 4 * ((long long)T - 1) + 4) return 0;
    if (line_pattern_ok<9>(a, Lw)) return 9;
    if (line_pattern_ok<5>(a, Lw)) return 5;
    return 0;
}

bool launch_lfused(const LaunchCtx& c, const SolveArgs& a, unsigned long long T, bool lean) {
    const int pat = lfused_pattern(a, T);
    if (!pat) return false;
    const long long Lw = a.dia.plane;
    LineGeom g{};
    g.Lw = (int)Lw;
    g.NL = (int)(a.n / Lw);
    const int NS = (int)T - 1;
    // slabs of 128 columns, overlapping by pad columns on either side
    g.C = 128;
    g.pad = 4;  // >= NS: a slab's valid columns move in by one per stencil stage
    g.Ci = g.C - 2 * g.pad;
    g.S = (int)((Lw + g.Ci - 1) / g.Ci);
    static const int ctas = lmarch_env("NLSP_LFUSED_CTAS", 0);
    const int mb = pat == 9 ? 2 : 1;
    const size_t smem = (size_t)(NS * kFusedSSlots + kFusedSlots) * (g.C + 2) * sizeof(double) +
                        (size_t)kFusedSlots * (g.C + 2) * mb;
    auto go = [&](auto kern) {
        static std::mutex mu;
        static std::unordered_map<unsigned long long, int> occ;
        int nb = 1;
        {
            std::lock_guard<std::mutex> lk(mu);
            const unsigned long long key =
                reinterpret_cast<unsigned long long>(reinterpret_cast<const void*>(kern)) * 1315423911ull ^ (unsigned)g.C;
            auto it = occ.find(key);
            if (it == occ.end()) {
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, g.C, smem) != cudaSuccess || nb < 1) nb = 1;
                cudaGetLastError();
                occ[key] = nb;
            } else {
                nb = it->second;
            }
        }
        if (ctas > 0 && ctas < nb) nb = ctas;
        long long G = (long long)c.num_sms * nb;
        const long long TT = (long long)g.S * g.NL;
        if (G > TT) G = TT;
        if (G > kMaxGrid) G = kMaxGrid;
        klaunch(c, kern, (int)G, g.C, smem, a, OpUpdSweep<true>{}, g);
    };
#define NLSP_LF_GO(PAT, MT, NSS) do { if (lean) go(k_lfused<PAT, MT, NSS, 2, true>); else go(k_lfused<PAT, MT, NSS, 2, false>); } while (0)
    if (pat == 9 && NS == 3) NLSP_LF_GO(9, unsigned short, 3);
    else if (pat == 9) NLSP_LF_GO(9, unsigned short, 1);
    else if (NS == 3) NLSP_LF_GO(5, unsigned char, 3);
    else NLSP_LF_GO(5, unsigned char, 1);
#undef NLSP_LF_GO
    count(c);
    return true;
}

// Staged tiles must fit in shared memory (227 KB per CTA); matrices with very
// long rows (a tile's nonzeros beyond the budget) take the direct-load kernels.
constexpr size_t kStageBudget = 200 * 1024;
bool spmv_tma_ok(const SolveArgs& a) { return NLSP_TMA && spmv_stage_smem(a) <= kStageBudget; }
bool restrict_tma_ok(const SolveArgs& a) { return NLSP_TMA && restrict_stage_smem(a) <= kStageBudget; }

void launch_spmv_p(const LaunchCtx& c, const SolveArgs& a) {
    if (a.dia.kind && launch_march_op(c, a, MOpSpmvP{})) {
    } else if (a.dia.kind) launch_dia_op<1>(c, a, OpSpmvP{});
    else if (spmv_tma_ok(a)) launch_spmv_op<1>(c, a, OpSpmvP{});
    else launch_rows<kU>(c, k_spmv_p, a.n, a);
    count(c);
}

// mode: 0 two-level, 1 identity, 2 Jacobi
void launch_update(const LaunchCtx& c, const SolveArgs& a, int mode) {
    if (mode == 0) launch_elems(c, k_update<0>, a.n, a);
    else if (mode == 1) launch_elems(c, k_update<1>, a.n, a);
    else launch_elems(c, k_update<2>, a.n, a);
    count(c);
}

void launch_loop_ctl(const LaunchCtx& c, PcgState* st, cudaGraphConditionalHandle h, int use_cond) {
    k_loop_ctl<<<1, 1, 0, c.s>>>(st, h, use_cond);
    count(c);
}

void launch_true_res(const LaunchCtx& c, const SolveArgs& a) {
    if (a.dia.kind) launch_dia_op<2>(c, a, OpTrueRes{a.x, a.b});
    else if (spmv_tma_ok(a)) launch_spmv_op<2>(c, a, OpTrueRes{a.x, a.b});
    else launch_rows<kU>(c, k_true_res, a.n, a);
    count(c);
}

void launch_spmv(const LaunchCtx& c, int n, const int* rp, const int* ci, const double* v,
                 const double* x, double* y) {
    launch_rows<kU>(c, k_spmv, n, n, rp, ci, v, x, y);
    count(c);
}

// y = A x through the TMA-staged engine (the product path of nlsp_spmv)
void launch_spmv_args(const LaunchCtx& c, const SolveArgs& a, const double* x, double* y) {
    if (a.dia.kind) launch_dia_op<0>(c, a, OpPlain{x, y});
    else if (spmv_tma_ok(a)) launch_spmv_op<0>(c, a, OpPlain{x, y});
    else launch_rows<kU>(c, k_spmv, a.n, a.n, a.rp, a.ci, a.v, x, y);
    count(c);
}

template <int PPL>
static void restrict_ppl(const LaunchCtx& c, const SolveArgs& a, int zmode, const double* zpre) {
    if (restrict_tma_ok(a)) {
        const long long nt = restrict_tiles(a);
        const size_t sm = restrict_stage_smem(a);
        constexpr int S = NLSP_RESTRICT_STAGES;
        if (zmode == 0) launch_tma(c, k_restrict_tma<PPL, 0, S>, nt, sm, a, zpre);
        else if (zmode == 1) launch_tma(c, k_restrict_tma<PPL, 1, S>, nt, sm, a, zpre);
        else launch_tma(c, k_restrict_tma<PPL, 2, S>, nt, sm, a, zpre);
        return;
    }
    if (zmode == 0) launch_rows<kUP>(c, k_restrict<PPL, 0>, a.n, a, zpre);
    else if (zmode == 1) launch_rows<kUP>(c, k_restrict<PPL, 1>, a.n, a, zpre);
    else launch_rows<kUP>(c, k_restrict<PPL, 2>, a.n, a, zpre);
}

template <int PPL>
static void prolong_ppl(const LaunchCtx& c, const SolveArgs& a, int zmode, bool rz,
                        const double* zpre, double* zout, cudaGraphConditionalHandle h, int ctl) {
#define NLSP_PRO(Z, R) launch_rows<NLSP_KUPRO>(c, k_prolong<PPL, Z, R>, a.n, a, zpre, zout, h, ctl)
    if (zmode == 0) { if (rz) NLSP_PRO(0, true); else NLSP_PRO(0, false); }
    else if (zmode == 1) { if (rz) NLSP_PRO(1, true); else NLSP_PRO(1, false); }
    else { if (rz) NLSP_PRO(2, true); else NLSP_PRO(2, false); }
#undef NLSP_PRO
}

int ppl_for(int k) {
    const int pairs = (k + (k & 1)) / 2;
    const int need = (pairs + kGroup - 1) / kGroup;
    const int opts[] = {1, 2, 3, 4, 6, 8, 12, 16};
    for (int o : opts)
        if (o >= need) return o;
    return -1;
}

#define NLSP_PPL_SWITCH(ppl, CALL)     \
    switch (ppl) {                     \
        case 1: CALL(1); break;        \
        case 2: CALL(2); break;        \
        case 3: CALL(3); break;        \
        case 4: CALL(4); break;        \
        case 6: CALL(6); break;        \
        case 8: CALL(8); break;        \
        case 12: CALL(12); break;      \
        default: CALL(16); break;      \
    }

void launch_restrict(const LaunchCtx& c, const SolveArgs& a, int zmode, const double* zpre) {
#define CALL(P) restrict_ppl<P>(c, a, zmode, zpre)
    NLSP_PPL_SWITCH(ppl_for(a.k), CALL)
#undef CALL
    count(c);
}

// ctl: 0 plain, 1 / 2 also the loop control of k_loop_ctl (2: graph WHILE body)
void launch_prolong(const LaunchCtx& c, const SolveArgs& a, int zmode, bool rz, const double* zpre,
                    double* zout, cudaGraphConditionalHandle h = 0, int ctl = 0) {
    if (a.k > kWideK) {
#define NLSP_PW(Z, R) launch_rows<1>(c, k_prolong_wide<Z, R>, (long long)a.n * 8, a, zpre, zout, h, ctl)
        if (zmode == 0) { if (rz) NLSP_PW(0, true); else NLSP_PW(0, false); }
        else if (zmode == 1) { if (rz) NLSP_PW(1, true); else NLSP_PW(1, false); }
        else { if (rz) NLSP_PW(2, true); else NLSP_PW(2, false); }
#undef NLSP_PW
        count(c);
        return;
    }
#define CALL(P) prolong_ppl<P>(c, a, zmode, rz, zpre, zout, h, ctl)
    NLSP_PPL_SWITCH(ppl_for(a.k), CALL)
#undef CALL
    count(c);
}

// sweep with z_in = implicit w D^-1 r (first pre-sweep) or a buffer
void launch_sweep(const LaunchCtx& c, const SolveArgs& a, bool implicit_in, const double* zin,
                  double* zout, bool rz) {
    if (a.dia.kind) {
        if (a.wdc != 0.0) {
            if (implicit_in) {
                const GWdrT<true> gw{a.wd, a.r, a.wdc};
                if (rz) launch_dia_op<1>(c, a, OpSweep<GWdrT<true>, true, true>{gw, a.r, a.wd, zout, a.wdc});
                else launch_dia_op<1>(c, a, OpSweep<GWdrT<true>, false, true>{gw, a.r, a.wd, zout, a.wdc});
            } else {
                const GPlain gp{zin};
                if (rz) launch_dia_op<1>(c, a, OpSweep<GPlain, true, true>{gp, a.r, a.wd, zout, a.wdc});
                else launch_dia_op<1>(c, a, OpSweep<GPlain, false, true>{gp, a.r, a.wd, zout, a.wdc});
            }
        } else if (implicit_in) {
            const GWdr gw{a.wd, a.r};
            if (rz) launch_dia_op<1>(c, a, OpSweep<GWdr, true>{gw, a.r, a.wd, zout});
            else launch_dia_op<1>(c, a, OpSweep<GWdr, false>{gw, a.r, a.wd, zout});
        } else {
            const GPlain gp{zin};
            if (rz) launch_dia_op<1>(c, a, OpSweep<GPlain, true>{gp, a.r, a.wd, zout});
            else launch_dia_op<1>(c, a, OpSweep<GPlain, false>{gp, a.r, a.wd, zout});
        }
        count(c);
        return;
    }
    if (spmv_tma_ok(a)) {
        if (implicit_in) {
            const GWdr gw{a.wd, a.r};
            if (rz) launch_spmv_op<1>(c, a, OpSweep<GWdr, true>{gw, a.r, a.wd, zout});
            else launch_spmv_op<1>(c, a, OpSweep<GWdr, false>{gw, a.r, a.wd, zout});
        } else {
            const GPlain gp{zin};
            if (rz) launch_spmv_op<1>(c, a, OpSweep<GPlain, true>{gp, a.r, a.wd, zout});
            else launch_spmv_op<1>(c, a, OpSweep<GPlain, false>{gp, a.r, a.wd, zout});
        }
        count(c);
        return;
    }
    if (implicit_in) {
        const GWdr gw{a.wd, a.r};
        if (rz) launch_rows<kU>(c, k_sweep<GWdr, true>, a.n, a, gw, zout);
        else launch_rows<kU>(c, k_sweep<GWdr, false>, a.n, a, gw, zout);
    } else {
        const GPlain gp{zin};
        if (rz) launch_rows<kU>(c, k_sweep<GPlain, true>, a.n, a, gp, zout);
        else launch_rows<kU>(c, k_sweep<GPlain, false>, a.n, a, gp, zout);
    }
    count(c);
}

// One two-level cycle z = M^-1 r (two_level.hpp:60-81) on a.r -> a.z, with r.z
// left in st->rz_new. Buffers: zt0/zt1 ping-pong, prolongation in place.
void launch_twolevel_apply(const LaunchCtx& c, const SolveArgs& a, unsigned long long nu1,
                           unsigned long long nu2) {
    int zmode;
    const double* zpre = nullptr;
    if (nu1 == 0) {
        zmode = 0;
    } else if (nu1 == 1) {
        zmode = 1;
    } else {
        double* cur = a.zt0;
        launch_sweep(c, a, true, nullptr, cur, false);
        for (unsigned long long s = 2; s < nu1; ++s) {
            double* nxt = (cur == a.zt0) ? a.zt1 : a.zt0;
            launch_sweep(c, a, false, cur, nxt, false);
            cur = nxt;
        }
        zmode = 2;
        zpre = cur;
    }
    launch_restrict(c, a, zmode, zpre);
    double* pro_out;
    if (nu2 == 0) pro_out = a.z;
    else pro_out = (zmode == 2) ? const_cast<double*>(zpre) : a.zt0;
    launch_prolong(c, a, zmode, nu2 == 0, zpre, pro_out);
    double* cur = pro_out;
    for (unsigned long long s = 1; s <= nu2; ++s) {
        double* out = (s == nu2) ? a.z : ((cur == a.zt0) ? a.zt1 : a.zt0);
        launch_sweep(c, a, false, cur, out, s == nu2);
        cur = out;
    }
}

// ------------------------------------------------------- folded cycle host --
#ifndef NLSP_UR_STAGES
#define NLSP_UR_STAGES 4
#endif
#ifndef NLSP_UR_TMA
#define NLSP_UR_TMA 1
#endif
template <int PPL>
static void update_restrict_ppl(const LaunchCtx& c, const SolveArgs& a, bool update) {
    const int ld = a.k + (a.k & 1);
    const size_t stage = (size_t)(update ? 4 : 1) * 64 * 8 + round16(64 * ld * 8);
    const long long nt = (a.n + 63) / 64;
    if (NLSP_UR_TMA && 64 + 2 * 64 * 8 + NLSP_UR_STAGES * stage <= kStageBudget) {
        constexpr int S = NLSP_UR_STAGES;
        const size_t sm = 64 + 2 * 64 * 8 + S * stage;
        if (update) launch_tma(c, k_update_restrict_tma<PPL, true, S>, nt, sm, a);
        else launch_tma(c, k_update_restrict_tma<PPL, false, S>, nt, sm, a);
        return;
    }
    if (NLSP_UR_TMA && 64 + 2 * 64 * 8 + 2 * stage <= kStageBudget) {  // large k: 2 stages
        const size_t sm = 64 + 2 * 64 * 8 + 2 * stage;
        if (update) launch_tma(c, k_update_restrict_tma<PPL, true, 2>, nt, sm, a);
        else launch_tma(c, k_update_restrict_tma<PPL, false, 2>, nt, sm, a);
        return;
    }
    if (update) launch_rows<kUP>(c, k_update_restrict<PPL, true>, a.n, a);
    else launch_rows<kUP>(c, k_update_restrict<PPL, false>, a.n, a);
}

// update = true: x/r update + ||r|| + convergence + c = W1^T r + coarse solve;
// update = false: c = W1^T r + coarse solve
void launch_update_restrict(const LaunchCtx& c, const SolveArgs& a, bool update) {
    if (a.k > kWideK) {
        // c = W1^T r (+ the x / r update and convergence test), then e = A_c^-1 c
        long long g = (long long)c.num_sms;
        if (g > kWideGrid) g = kWideGrid;
        const long long need = ((long long)a.n + 31) / 32;
        if (g > need) g = need;
        if (update) k_update_restrict_wide<true><<<(int)g, kThreads, 0, c.s>>>(a);
        else k_update_restrict_wide<false><<<(int)g, kThreads, 0, c.s>>>(a);
        count(c);
        k_coarse_gemv<<<(a.k + 7) / 8, kThreads, 0, c.s>>>(a, update ? 1 : 0);
        count(c);
        return;
    }
#define CALL(P) update_restrict_ppl<P>(c, a, update)
    NLSP_PPL_SWITCH(ppl_for(a.k), CALL)
#undef CALL
    count(c);
}

// The smoothing + prolongation half of the folded cycle, after the restriction
// (e is in a.e): z = S_{nu1+nu2}(r) + W2 e, r.z -> st->rz_new.
// ctl > 0: the prolongation also runs the loop control (no k_loop_ctl launch)
void launch_folded_tail(const LaunchCtx& c, const SolveArgs& a, unsigned long long nu1,
                        unsigned long long nu2, cudaGraphConditionalHandle h, int ctl) {
    const unsigned long long T = nu1 + nu2;
    SolveArgs b = a;
    b.P = a.W2;
    if (T <= 1) {  // z = (T ? w D^-1 r : 0) + W2 e
        launch_prolong(c, b, T == 0 ? 0 : 1, true, nullptr, a.z, h, ctl);
        return;
    }
    // s_j = s_{j-1} + w D^-1 (r - A s_{j-1}), s_1 = w D^-1 r implicit; then
    // z = s_T + W2 e streamed with the prolongation kernel (r.z fused)
    double* cur = nullptr;
    for (unsigned long long j = 2; j <= T; ++j) {
        double* nxt = (cur == a.zt0) ? a.zt1 : a.zt0;
        launch_sweep(c, a, cur == nullptr, cur, nxt, false);
        cur = nxt;
    }
    launch_prolong(c, b, 2, true, cur, a.z, h, ctl);
}

void launch_folded_apply(const LaunchCtx& c, const SolveArgs& a, unsigned long long nu1,
                         unsigned long long nu2) {
    launch_update_restrict(c, a, false);
    launch_folded_tail(c, a, nu1, nu2, 0, 0);
}

// ------------------------------------------------------- one-pass cycle host --
bool onepass_supported(int k) { return k <= kOnePassK; }

#ifndef NLSP_OP_TMA
#define NLSP_OP_TMA 1
#endif
#ifndef NLSP_OP_STAGES
#define NLSP_OP_STAGES 0  // 0: as many as fit, up to kOpMaxStages
#endif
template <class... KArgs, class... Args>
static void launch_op_tma(const LaunchCtx& c, void (*f)(KArgs...), long long ntiles, size_t smem,
                          int threads, Args&&... args) {
    static std::mutex mu;
    static std::unordered_map<const void*, size_t> attr;
    {
        std::lock_guard<std::mutex> lk(mu);
        size_t& cur = attr[reinterpret_cast<const void*>(f)];
        if (smem > cur) {
            cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            cur = smem;
        }
    }
    long long g = c.num_sms;  // one CTA per SM (the stage ring fills shared memory)
    if (g > ntiles) g = ntiles;
    if (g < 1) g = 1;
    klaunch(c, f, (int)g, threads, smem, std::forward<Args>(args)...);
}

// The ring may take what the 227 KB of a CTA leave beside the kernel's static
// shared arrays (column sums, the lean coarse step, the grid reduction: < 12 KB).
constexpr size_t kOpRingBudget = 215 * 1024;
// stages of the one-pass prolongation's ring that fit the budget
static int op_fit(const SolveArgs& a, size_t budget) {
    const int ld = a.k + (a.k & 1);
    const int tnz = a.dia.kind ? -1 : (kOpTR == 64 ? a.tile_nnz64 : a.tile_nnz128);
    return (int)((budget - 256) / op_stage_bytes(ld, tnz));
}

template <int PPL>
static void prolong_onepass_ppl(const LaunchCtx& c, const SolveArgs& a, const double* sv, double* zout,
                                cudaGraphConditionalHandle h, int ctl, int rsel, int lean) {
    const int ld = a.k + (a.k & 1);
    // as many stages as fit, a multiple of the stencil pair count P
    const int tnz = a.dia.kind ? -1 : (kOpTR == 64 ? a.tile_nnz64 : a.tile_nnz128);
    // The ring may take kOpRingBudget (of the 227 KB a CTA can have, less the
    // static shared arrays): at C4 that is 6 stages instead of the 4 of a
    // 200 KB budget (measured 371 -> 361 us per launch, 2 175 -> 2 223
    // iterations/s at the same capped clock).
    // NLSP_OP_BUDGET (KB) overrides it for A/B runs.
    static const size_t budget = std::getenv("NLSP_OP_BUDGET") ? (size_t)std::atoi(std::getenv("NLSP_OP_BUDGET")) * 1024
                                                               : kOpRingBudget;
    int fit = (int)((budget - 256) / op_stage_bytes(ld, tnz));
    if (fit > kOpMaxStages) fit = kOpMaxStages;
    if (NLSP_OP_STAGES > 0 && fit > NLSP_OP_STAGES) fit = NLSP_OP_STAGES;
    int S, P;
    if (fit >= 8) { S = 8; P = 4; }
    else if (fit >= 6) { S = 6; P = 3; }
    else if (fit >= 4) { S = 4; P = 4; }
    else { S = 2; P = 2; }
    {
        // development overrides (A/B runs): NLSP_OP_P stencil pairs, NLSP_OP_S stages
        static const int env_p = std::getenv("NLSP_OP_P") ? std::atoi(std::getenv("NLSP_OP_P")) : 0;
        static const int env_s = std::getenv("NLSP_OP_S") ? std::atoi(std::getenv("NLSP_OP_S")) : 0;
        if (env_p >= 1 && env_p <= kOpSPairs) P = env_p;
        if (env_s >= 2) S = env_s < fit ? env_s : fit;
        S -= S % P;  // the ring depth must be a multiple of P (see kOpSPairs)
        if (S < P) S = P;
        if (S > fit) S = fit, P = 1;
    }
    {
        // ... and of the W-product warp groups
        const int q = (P % op_wh(PPL) == 0) ? P : P * op_wh(PPL);
        S -= S % q;
        if (S < q) { S = q; }
    }
    const size_t sm = 256 + (size_t)S * op_stage_bytes(ld, tnz);
    if (NLSP_OP_TMA && fit >= 2) {
        const long long nt = (a.n + kOpTR - 1) / kOpTR;
        const int threads = 32 * (1 + 2 * P + op_wpg(PPL) * op_wh(PPL));
#define NLSP_P2(D, R) launch_op_tma(c, k_prolong_onepass_tma<PPL, D, R>, nt, sm, threads, a, sv, zout, h, ctl, S, P, rsel, lean)
        const bool rv = a.dia.kind == 2;
        if (!a.dia.kind) NLSP_P2(0, false);
        else if (a.dia.d <= 8) { if (rv) NLSP_P2(8, true); else NLSP_P2(8, false); }
        else if (a.dia.d <= 16) { if (rv) NLSP_P2(16, true); else NLSP_P2(16, false); }
        else { if (rv) NLSP_P2(32, true); else NLSP_P2(32, false); }
#undef NLSP_P2
        return;
    }
#define NLSP_P1(D, R) launch_rows<NLSP_KUPRO>(c, k_prolong_onepass<PPL, D, R>, a.n, a, sv, zout, h, ctl, rsel)
    const bool rv = a.dia.kind == 2;
    if (!a.dia.kind) NLSP_P1(0, false);
    else if (a.dia.d <= 8) { if (rv) NLSP_P1(8, true); else NLSP_P1(8, false); }
    else if (a.dia.d <= 16) { if (rv) NLSP_P1(16, true); else NLSP_P1(16, false); }
    else { if (rv) NLSP_P1(32, true); else NLSP_P1(32, false); }
#undef NLSP_P1
}

// z = s + W e with u, v, w partials (s = S_T(r) by T - 1 sweep launches, or
// none for T = 0); ctl as launch_prolong
void launch_prolong_onepass(const LaunchCtx& c, const SolveArgs& a, const double* sv, double* zout,
                            cudaGraphConditionalHandle h, int ctl, int rsel, int lean) {
    SolveArgs b = a;
    b.P = a.W2;
    switch (ppl_for(a.k)) {
        case 1: prolong_onepass_ppl<1>(c, b, sv, zout, h, ctl, rsel, lean); break;
        case 2: prolong_onepass_ppl<2>(c, b, sv, zout, h, ctl, rsel, lean); break;
        case 3: prolong_onepass_ppl<3>(c, b, sv, zout, h, ctl, rsel, lean); break;
        default: prolong_onepass_ppl<4>(c, b, sv, zout, h, ctl, rsel, lean); break;
    }
    count(c);
}

// the x/r update fused with the first two sweeps (OpUpdSweep): s -> zt0
bool update_sweep_ok(const SolveArgs& a, unsigned long long T) {
    return T >= 2 && (a.dia.kind || spmv_tma_ok(a));
}

// a later sweep s_out = s_in + w D^-1 (r' - A s_in) after the fused update,
// r' = r[(it + 1) & 1]
static void launch_sweep_rpar(const LaunchCtx& c, const SolveArgs& a, const double* zin, double* zout) {
    const GPlain gp{zin};
    if (a.dia.kind && a.wdc != 0.0 && launch_march_op(c, a, MOpSweep<true>{zin, nullptr, a.wd, zout, a.wdc})) {
    } else if (a.dia.kind && a.wdc == 0.0 && launch_march_op(c, a, MOpSweep<false>{zin, nullptr, a.wd, zout, 0.0})) {
    } else if (a.dia.kind && a.wdc != 0.0)
        launch_dia_op<1>(c, a, OpSweep<GPlain, false, true>{gp, a.r, a.wd, zout, a.wdc, true});
    else if (a.dia.kind)
        launch_dia_op<1>(c, a, OpSweep<GPlain, false>{gp, a.r, a.wd, zout, 0.0, true});
    else
        launch_spmv_op<1>(c, a, OpSweep<GPlain, false>{gp, a.r, a.wd, zout, 0.0, true});
    count(c);
}
void launch_sweeps_rpar(const LaunchCtx& c, const SolveArgs& a, unsigned long long T, double** cur) {
    for (unsigned long long j = 3; j <= T; ++j) {
        double* nxt = (*cur == a.zt0) ? a.zt1 : a.zt0;
        launch_sweep_rpar(c, a, *cur, nxt);
        *cur = nxt;
    }
}
void launch_update_sweep(const LaunchCtx& c, const SolveArgs& a) {
    if (a.dia.kind && a.wdc != 0.0 && launch_march_op(c, a, MOpUpdSweep<true>{})) {
    } else if (a.dia.kind && a.wdc == 0.0 && launch_march_op(c, a, MOpUpdSweep<false>{})) {
    } else if (a.dia.kind && a.wdc != 0.0) launch_dia_op<1>(c, a, OpUpdSweep<true>{});
    else if (a.dia.kind) launch_dia_op<1>(c, a, OpUpdSweep<false>{});
    else launch_spmv_op<1>(c, a, OpUpdSweep<false>{});
    count(c);
}

// sweeps s = S_T(r) (T = nu1 + nu2 even, first sweep implicit), returns s (null for T = 0)
const double* launch_onepass_sweeps(const LaunchCtx& c, const SolveArgs& a, unsigned long long T) {
    double* cur = nullptr;
    for (unsigned long long j = 2; j <= T; ++j) {
        double* nxt = (cur == a.zt0) ? a.zt1 : a.zt0;
        launch_sweep(c, a, cur == nullptr, cur, nxt, false);
        cur = nxt;
    }
    return cur;
}

void launch_update_onepass(const LaunchCtx& c, const SolveArgs& a) {
    launch_elems(c, k_update_onepass, a.n, a);
    count(c);
}

// one iteration's tail after k_spmv_p / k_update_onepass
void launch_onepass_tail(const LaunchCtx& c, const SolveArgs& a, unsigned long long T,
                         cudaGraphConditionalHandle h, int ctl) {
    const double* sv = launch_onepass_sweeps(c, a, T);
    launch_prolong_onepass(c, a, sv, a.z, h, ctl, 0, 0);
}

// one iteration after k_spmv_p: fused update + sweeps (T = 2) when possible
void launch_onepass_iteration_tail(const LaunchCtx& c, const SolveArgs& a, unsigned long long T,
                                   cudaGraphConditionalHandle h, int ctl) {
    if (update_sweep_ok(a, T) && launch_lfused(c, a, T, false)) {  // s_T -> zt0
        launch_prolong_onepass(c, a, a.zt0, a.z, h, ctl, 1, 0);
        return;
    }
    if (update_sweep_ok(a, T)) {
        launch_update_sweep(c, a);  // s_2 -> zt0
        double* cur = a.zt0;
        launch_sweeps_rpar(c, a, T, &cur);
        launch_prolong_onepass(c, a, cur, a.z, h, ctl, 1, 0);
        return;
    }
    launch_update_onepass(c, a);
    launch_onepass_tail(c, a, T, h, ctl);
}

// PCG prologue z = M r_0 with the one-pass partials of r_0: c = W^T r_0 directly
void launch_onepass_apply(const LaunchCtx& c, const SolveArgs& a, unsigned long long T) {
    launch_update_restrict(c, a, false);
    launch_onepass_tail(c, a, T, 0, 0);
}

// ---------------------------------------------------------- lean cycle host --
// The lean cycle needs the warp-specialised pass (it stages p's old rows) and
// a smoother (T >= 2) on the diagonal-form or TMA-staged SpMV kernels.
bool lean_supported(const SolveArgs& a, unsigned long long T) {
    static const bool off = std::getenv("NLSP_LEAN") && std::atoi(std::getenv("NLSP_LEAN")) == 0;
    if (off || !NLSP_OP_TMA || a.k > kOnePassK || T < 2 || (T & 1)) return false;
    if (!(a.dia.kind || spmv_tma_ok(a))) return false;
    return op_fit(a, kOpRingBudget) >= 2;
}

// K1: q = A p in the gather, x += alpha p, r -= alpha q, ||r|| and p.q
void launch_spmv_upd(const LaunchCtx& c, const SolveArgs& a) {
    if (a.dia.kind) launch_dia_op<1>(c, a, OpSpmvUpd{});
    else launch_spmv_op<1>(c, a, OpSpmvUpd{});
    count(c);
}

// K2 (+ the later sweeps of T > 2): s = S_T(r), r.s, the coarse step; returns s
const double* launch_lean_sweeps(const LaunchCtx& c, const SolveArgs& a, unsigned long long T) {
    // all T sweeps in one line march: s_T -> zt0 (T = 2 stays the direct kernel:
    // one sweep pair has nothing to chain, measured 290 vs 297 us at C1 2048^2)
    if (T > 2 && launch_lfused(c, a, T, true)) return a.zt0;
    if (a.dia.kind && a.wdc != 0.0) launch_dia_op<1>(c, a, OpSweepLean<true>{});
    else if (a.dia.kind) launch_dia_op<1>(c, a, OpSweepLean<false>{});
    else launch_spmv_op<1>(c, a, OpSweepLean<false>{});
    count(c);
    double* cur = a.zt0;
    for (unsigned long long j = 3; j <= T; ++j) {
        double* nxt = (cur == a.zt0) ? a.zt1 : a.zt0;
        const GPlain gp{cur};
        const bool last = j == T;
        if (a.dia.kind && a.wdc != 0.0) {
            if (last) launch_dia_op<1>(c, a, OpSweep<GPlain, true, true>{gp, a.r, a.wd, nxt, a.wdc});
            else launch_dia_op<1>(c, a, OpSweep<GPlain, false, true>{gp, a.r, a.wd, nxt, a.wdc});
        } else if (a.dia.kind) {
            if (last) launch_dia_op<1>(c, a, OpSweep<GPlain, true>{gp, a.r, a.wd, nxt});
            else launch_dia_op<1>(c, a, OpSweep<GPlain, false>{gp, a.r, a.wd, nxt});
        } else {
            if (last) launch_spmv_op<1>(c, a, OpSweep<GPlain, true>{gp, a.r, a.wd, nxt});
            else launch_spmv_op<1>(c, a, OpSweep<GPlain, false>{gp, a.r, a.wd, nxt});
        }
        count(c);
        cur = nxt;
    }
    return cur;
}

// one lean iteration: c0 launches its first kernel, c1 the rest (PDL)
void launch_lean_iteration(const LaunchCtx& c0, const LaunchCtx& c1, const SolveArgs& a,
                           unsigned long long T, cudaGraphConditionalHandle h, int ctl) {
    launch_spmv_upd(c0, a);
    const double* sv = launch_lean_sweeps(c1, a, T);
    launch_prolong_onepass(c1, a, sv, a.p0, h, ctl, 0, 1);
}

// lean prologue: c = W^T r_0 directly, e_0, s = S_T(r_0) with r.s, the coarse
// scalars, then the pass: p_0 = s + W e_0, u_0, v_0 -> alpha_0
void launch_lean_apply(const LaunchCtx& c, const SolveArgs& a, unsigned long long T) {
    launch_update_restrict(c, a, false);
    double* cur = nullptr;
    for (unsigned long long j = 2; j <= T; ++j) {
        double* nxt = (cur == a.zt0) ? a.zt1 : a.zt0;
        launch_sweep(c, a, cur == nullptr, cur, nxt, j == T);
        cur = nxt;
    }
    k_lean_init<<<1, kThreads, 0, c.s>>>(a, cur != nullptr ? 1 : 0);
    count(c);
    launch_prolong_onepass(c, a, cur, a.p0, 0, 0, 0, 2);
}

}  // namespace nlsp
