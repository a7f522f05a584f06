// paper_2601_20174_b200/csrc/nlsp_gpu.cu — the C-ABI (include/nlsp_gpu.h):
// handles, device memory, setup orchestration and the device-resident PCG loop
// (one CUDA graph per solve: prologue, a WHILE conditional node whose body is
// one PCG iteration, epilogue). Reference interface cited per entry point.
#include <cuda_runtime.h>

#include <algorithm>
#include <climits>
#include <cmath>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "host_rng.hpp"
#include "internal.cuh"
#include "nlsp_gpu.h"

namespace nlsp {
// solve_kernels.cu
void launch_state_init(const LaunchCtx&, PcgState*, double, long long);
void launch_bnorm(const LaunchCtx&, const SolveArgs&);
void launch_init_simple(const LaunchCtx&, const SolveArgs&, int);
void launch_init_ctl(const LaunchCtx&, PcgState*);
void launch_state_continue(const LaunchCtx&, PcgState*, long long, long long);
void launch_spmv_p(const LaunchCtx&, const SolveArgs&);
void launch_update(const LaunchCtx&, const SolveArgs&, int);
void launch_loop_ctl(const LaunchCtx&, PcgState*, cudaGraphConditionalHandle, int);
void launch_true_res(const LaunchCtx&, const SolveArgs&);
void launch_spmv_args(const LaunchCtx&, const SolveArgs&, const double*, double*);
void launch_spmv(const LaunchCtx&, int, const int*, const int*, const double*, const double*,
                 double*);
void launch_sweep(const LaunchCtx&, const SolveArgs&, bool, const double*, double*, bool);
void launch_restrict(const LaunchCtx&, const SolveArgs&, int, const double*);
void launch_prolong(const LaunchCtx&, const SolveArgs&, int, bool, const double*, double*,
                    cudaGraphConditionalHandle, int);
void launch_twolevel_apply(const LaunchCtx&, const SolveArgs&, unsigned long long,
                           unsigned long long);
void launch_update_restrict(const LaunchCtx&, const SolveArgs&, bool);
void launch_folded_tail(const LaunchCtx&, const SolveArgs&, unsigned long long, unsigned long long,
                        cudaGraphConditionalHandle, int);
void launch_folded_apply(const LaunchCtx&, const SolveArgs&, unsigned long long, unsigned long long);
bool onepass_supported(int k);
void launch_prolong_onepass(const LaunchCtx&, const SolveArgs&, const double*, double*,
                            cudaGraphConditionalHandle, int, int, int);
bool lean_supported(const SolveArgs&, unsigned long long);
void launch_spmv_upd(const LaunchCtx&, const SolveArgs&);
const double* launch_lean_sweeps(const LaunchCtx&, const SolveArgs&, unsigned long long);
void launch_lean_iteration(const LaunchCtx&, const LaunchCtx&, const SolveArgs&, unsigned long long,
                           cudaGraphConditionalHandle, int);
void launch_lean_apply(const LaunchCtx&, const SolveArgs&, unsigned long long);
bool update_sweep_ok(const SolveArgs&, unsigned long long);
void launch_sweeps_rpar(const LaunchCtx&, const SolveArgs&, unsigned long long, double**);
void launch_update_sweep(const LaunchCtx&, const SolveArgs&);
void launch_onepass_iteration_tail(const LaunchCtx&, const SolveArgs&, unsigned long long,
                                   cudaGraphConditionalHandle, int);
const double* launch_onepass_sweeps(const LaunchCtx&, const SolveArgs&, unsigned long long);
void launch_update_onepass(const LaunchCtx&, const SolveArgs&);
void launch_onepass_tail(const LaunchCtx&, const SolveArgs&, unsigned long long, cudaGraphConditionalHandle, int);
void launch_onepass_apply(const LaunchCtx&, const SolveArgs&, unsigned long long);
int ppl_for(int k);
// cluster_solve.cu
int cluster_plan(int n, int k, int width, bool two_w, int* rows_out,
                 size_t* smem_out);
cudaError_t launch_cluster_pcg(cudaStream_t s, const ClusterArgs& a, int ncta, size_t smem);
int cluster_plan_batch(int count, const int* n, const int* k, const int* width, const bool* two_w, int* rows,
                       size_t* smem_out);
cudaError_t launch_cluster_pcg_batch(cudaStream_t s, const ClusterArgs* dargs, int count, int ncta, size_t smem);
// setup_kernels.cu
void launch_csr_import(const LaunchCtx&, int, long long, const unsigned long long*,
                       const unsigned long long*, const double*, int*, int*, double*, int*, int*);
void launch_wd(const LaunchCtx&, int, const double*, double, double*, int*);
bool launch_block_op_dia(const LaunchCtx&, int, int, const DiaArgs&, const double*, int, const double*,
                         double*);
void launch_block_op(const LaunchCtx&, int, int, const int*, const int*, const double*,
                     const double*, int, const double*, double*);
int gram_grid(const LaunchCtx&, long long);
void launch_gram(const LaunchCtx&, long long, int, int, const double*, const double*, double*,
                 double*);
void launch_eigh(const LaunchCtx&, int, const double*, double*, double*, double*, double*, int*,
                 int*);
void launch_dense_mm(const LaunchCtx&, long long, int, int, const double*, const double*,
                     const double*, double*);
void launch_colsign(const LaunchCtx&, long long, int, double*, double*, long long*, double*,
                    double*);
void launch_chol(const LaunchCtx&, int, const double*, double*, double, int*);
void launch_coarse_inverse(const LaunchCtx&, int, const double*, double*);
void launch_tri_inv_t(const LaunchCtx&, int, const double*, double*);
void launch_symmetrize(const LaunchCtx&, int, double*);
void launch_shift_diag(const LaunchCtx&, int, double*, double);
void launch_coldot(const LaunchCtx&, long long, int, const double*, int, const double*, double*, double*);
void launch_col_axpy(const LaunchCtx&, long long, int, const double*, int, double*, const double*);
void launch_col_move(const LaunchCtx&, long long, int, double*, int, double*, const double*, int, long long);
void launch_transpose(const LaunchCtx&, long long, int, const double*, double*);
bool march_planned(const LaunchCtx&, const SolveArgs&);
bool launch_lfused(const LaunchCtx&, const SolveArgs&, unsigned long long, bool);
int lfused_pattern(const SolveArgs&, unsigned long long);
void launch_s0_scatter(const LaunchCtx&, const double*, long long, long long, int, const int*, double*);
void launch_mt_stream(const LaunchCtx&, unsigned long long*, long long, int, const unsigned long long*, int,
                      unsigned long long, unsigned long long, unsigned long long*, unsigned long long*);
void launch_box_muller(const LaunchCtx&, double*, unsigned long long, const unsigned long long*, int*);
void launch_sigma(const LaunchCtx&, int, int, const double*, const double*, double*, double*,
                  int*);
// setup_kernels.cu (SA)
void launch_sa_assemble(const LaunchCtx&, int, int, const int*, const int*, const double*, const int*,
                        const double*, const double*, double, double*);
// mlp.cu
int mlp_splitk_parts(const LaunchCtx&, int, int);
void launch_mlp_layer(const LaunchCtx&, const double*, const double*, const double*, const double*,
                      int, int, bool, const double*, double*, double*);
void launch_mlp_input(const LaunchCtx&, int, int, const double*, double*, int, double*, int*);
void launch_unflatten(const LaunchCtx&, int, int, const double*, double*);
}  // namespace nlsp

using namespace nlsp;

namespace {
std::atomic<unsigned long long> g_next_id{1};
}

struct nlsp_csr {
    unsigned long long id;
    int device;
    int n;
    long long nnz;
    int* rp;
    int* ci;
    double* v;
    double* diag;
    int diag_ok;  // all A_ii > 0
    int max_row;
    int tile_nnz64, tile_nnz128, tile_nnz256;  // max nonzeros of any 64/128/256-row tile
    std::vector<int> rp_host;  // row_ptr kept on the host for small systems (cluster plan)
    DiaArgs dia{};             // diagonal form (dia.kind == 0: none)
    void* dia_mask = nullptr;
    double* dia_rv = nullptr;
    PackArgs pk{};             // implicit-column form of the CSR arrays (pk.mask == nullptr: none)
    unsigned* pk_mask = nullptr;
    unsigned long long pass_bytes = 0;  // matrix bytes one solve-kernel pass streams
};

struct nlsp_dense {
    unsigned long long id;
    int device;
    unsigned long long rows, cols;
    double* d;
};

struct nlsp_twolevel {
    unsigned long long id;
    int device;
    int n, k, ld;
    unsigned long long nu1, nu2;
    double omega;
    double* basis;   // n x ld
    double* L;       // k x k
    double* Ainv;    // A_c^-1 = L^-T L^-1, k x k (coarse solve as one mat-vec)
    double* coarse;  // k x k
    double* wd;      // n
    double* W1;      // (I - w D^-1 A)^nu1 P, n x ld (folded cycle)
    double* W2;      // (I - w D^-1 A)^nu2 P, n x ld (aliases W1 when nu1 == nu2)
    bool folded;     // folded cycle (default) or the literal schedule (NLSP_CYCLE=literal)
    bool onepass;    // PCG streams W once per iteration (nu1 == nu2, k <= 64; NLSP_CYCLE=folded: twice)
    bool lean;       // one-pass with beta before and alpha after the pass (NLSP_CYCLE=onepass: off)
    double* M;       // W^T A W, k x k (one-pass restriction recurrence)
};

struct GraphKey {
    unsigned long long a = 0, m = 0;
    int kind = -1;
    long long ws_gen = -1;
    bool operator==(const GraphKey& o) const {
        return a == o.a && m == o.m && kind == o.kind && ws_gen == o.ws_gen;
    }
};

struct nlsp_ctx {
    int device = 0;
    int num_sms = 148;
    cudaStream_t s = nullptr;
    cudaStream_t s_body = nullptr;
    std::string err;
    unsigned long long launches = 0;
    LaunchCtx lc{};
    PcgState* st = nullptr;      // device
    PcgState* st_host = nullptr; // pinned
    int* flags = nullptr;        // device int[16]
    int* flags_host = nullptr;   // pinned
    // workspace (sized for ws_n rows, ws_ld coarse columns, ws_hist history)
    long long ws_n = 0, ws_hist = 0;
    long long ws_gen = 0;
    double *x = nullptr, *r = nullptr, *r1 = nullptr, *q = nullptr, *z = nullptr, *p0 = nullptr, *p1 = nullptr,
           *zt0 = nullptr, *zt1 = nullptr, *b = nullptr, *e = nullptr, *partials = nullptr,
           *hist = nullptr;
    double *ow = nullptr, *opart = nullptr;  // one-pass cycle: [u | v | w], per-CTA partials
    cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr;
    cudaGraphExec_t gexec = nullptr;
    GraphKey gkey;
    cudaGraphExec_t gexec_cont = nullptr;  // the loop without its prologue: later history segments
    GraphKey gkey_cont;
    // residual history of the last solve (SolveReport::residual_history): the
    // device keeps one segment of ws_hist entries; completed segments are moved
    // here, the last one stays on the device until nlsp_pcg_history asks
    std::vector<double> hist_done;
    unsigned long long hist_tail = 0;
    bool last_qr_robust = false;  // the last qr_thin took the shifted CholeskyQR3 path
    // pinned staging of the host-drawn S^(0) (nlsp_generate_smoothed_vectors):
    // two chunks of the normal stream in flight to the device
    double* s0_pin[2] = {nullptr, nullptr};
    cudaEvent_t s0_ev[2] = {nullptr, nullptr};
    // S^(0) drawn on the device (nlsp_ctx_set_s0_draw; s0_device.cu): the jump
    // polynomials of mt19937_64 (mt_jump_table.inc), uploaded on first use
    int s0_draw = NLSP_S0_DRAW_HOST;
    unsigned long long* mt_polys = nullptr;
    int last_s0_draw = NLSP_S0_DRAW_HOST;  // where the last generate_smoothed_vectors drew S^(0)
    double last_svd_defect = 0.0;  // orthonormality defect of the last svd_basis' U_k before any polish
    int last_svd_solid = 0;        // its columns above the singular-value cutoff
    bool use_graph = true;
    bool use_cluster = true;  // single-cluster solver for small systems
    cudaMemPool_t pool = nullptr;  // scratch of setup calls (salloc / sfree)
    bool coarse_inverse = true;  // coarse solve through A_c^-1 (NLSP_COARSE=chol: substitutions)
    unsigned long long gk_pro = 0, gk_body = 0, gk_epi = 0;  // kernels per graph part
};

// ------------------------------------------------------------------ helpers --
namespace {

nlsp_status set_err(nlsp_ctx* c, nlsp_status st, const std::string& msg) {
    if (c) c->err = msg;
    return st;
}

nlsp_status cuda_fail(nlsp_ctx* c, cudaError_t e, const char* what) {
    const nlsp_status st = (e == cudaErrorMemoryAllocation) ? NLSP_E_OOM : NLSP_E_CUDA;
    cudaGetLastError();
    return set_err(c, st, std::string(what) + ": " + cudaGetErrorString(e));
}

#define CU(expr)                                                  \
    do {                                                          \
        cudaError_t e_ = (expr);                                  \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, #expr);  \
    } while (0)

#define CHECK_LAUNCH()                                                   \
    do {                                                                 \
        cudaError_t e_ = cudaGetLastError();                             \
        if (e_ != cudaSuccess) return cuda_fail(ctx, e_, "kernel launch"); \
    } while (0)

nlsp_status map_dev_error(nlsp_ctx* c, int code, const char* where) {
    switch (code) {
        case kErrNone: return NLSP_OK;
        case kErrValidation: return set_err(c, NLSP_E_VALIDATION, std::string(where) + ": validation error");
        case kErrNumeric: return set_err(c, NLSP_E_NUMERIC, std::string(where) + ": numeric error");
        case kErrNotSpd: return set_err(c, NLSP_E_NOT_SPD, std::string(where) + ": operator not SPD");
        case kErrRank: return set_err(c, NLSP_E_RANK_DEFICIENT, std::string(where) + ": rank-deficient basis");
        case kErrConvergence: return set_err(c, NLSP_E_CONVERGENCE, std::string(where) + ": no convergence");
        default: return set_err(c, NLSP_E_NUMERIC, std::string(where) + ": device error");
    }
}

// Handle-owned device memory (matrices, bases, workspaces) comes from one
// stream-ordered pool per device that never releases memory to the OS, so
// rebuilding a preconditioner or re-uploading a matrix reuses pages instead of
// mapping multi-GB allocations anew (tens to hundreds of ms at C4). Allocation
// is ordered on the legacy stream and completed before use; cudaFree of a pool
// allocation synchronises the device and returns the block to the pool.
static cudaMemPool_t device_pool() {
    static std::mutex mu;
    static cudaMemPool_t pools[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    std::lock_guard<std::mutex> lk(mu);
    if (!pools[dev]) {
        cudaMemPoolProps pp{};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = dev;
        unsigned long long keep = ~0ull;
        if (cudaMemPoolCreate(&pools[dev], &pp) != cudaSuccess ||
            cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep) != cudaSuccess) {
            cudaGetLastError();
            pools[dev] = nullptr;
        }
    }
    return pools[dev];
}

template <class T>
cudaError_t dalloc(T** p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    cudaMemPool_t pool = device_pool();
    if (!pool) return cudaMalloc(reinterpret_cast<void**>(p), count * sizeof(T));
    cudaError_t e = cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), count * sizeof(T), pool, 0);
    if (!e) e = cudaStreamSynchronize(0);
    return e;
}

void dfree(void* p) {
    if (p) cudaFree(p);
}

// Scratch of the setup calls comes from the context's stream-ordered pool
// (release threshold: never), so repeated builds reuse memory instead of paying
// cudaMalloc/cudaFree of multi-GB buffers (and their implicit device syncs).
template <class T>
cudaError_t salloc(nlsp_ctx* c, T** p, size_t count) {
    *p = nullptr;
    if (count == 0) count = 1;
    return cudaMallocFromPoolAsync(reinterpret_cast<void**>(p), count * sizeof(T), c->pool, c->s);
}

void sfree(nlsp_ctx* c, void* p) {
    if (p) cudaFreeAsync(p, c->s);
}

// per-CTA partial size of launch_gram: it tiles C in blocks of <= 128 x 128
size_t gram_tile(int ca, int cb) { return (size_t)std::min(ca, 128) * (size_t)std::min(cb, 128); }

nlsp_status bind(nlsp_ctx* ctx) {
    if (!ctx) return NLSP_E_VALIDATION;
    CU(cudaSetDevice(ctx->device));
    return NLSP_OK;
}

void free_ws(nlsp_ctx* c) {
    for (double** p : {&c->x, &c->r, &c->r1, &c->q, &c->z, &c->p0, &c->p1, &c->zt0, &c->zt1, &c->b,
                       &c->e, &c->partials, &c->hist, &c->ow, &c->opart}) {
        dfree(*p);
        *p = nullptr;
    }
    c->ws_n = 0;
    c->ws_hist = 0;
}

// Device residual-history segment: a solve longer than this runs in segments
// (run_pcg), so the device never holds max_iters entries (10 n in the
// reference's harness: 328 MB at C4). NLSP_HIST_CHUNK overrides (tests).
long long hist_chunk() {
    static const long long v = [] {
        const char* e = std::getenv("NLSP_HIST_CHUNK");
        const long long c = e ? std::atoll(e) : (1ll << 20);
        return c < 1 ? 1ll : c;
    }();
    return v;
}
long long hist_segment(unsigned long long max_iters) {
    const unsigned long long c = (unsigned long long)hist_chunk();
    return (long long)(max_iters < c ? (max_iters ? max_iters : 1) : c);
}

// vectors for n rows, coarse vector and partials, history of hist entries
nlsp_status ensure_ws(nlsp_ctx* ctx, long long n, long long hist) {
    if (n > ctx->ws_n) {
        const long long hist_keep = ctx->ws_hist;
        free_ws(ctx);
        for (double** p : {&ctx->x, &ctx->r, &ctx->r1, &ctx->q, &ctx->z, &ctx->p0, &ctx->p1, &ctx->zt0,
                           &ctx->zt1, &ctx->b})
            CU(dalloc(p, (size_t)n + 16));  // padded for 16-B bulk copies of tile slices
        CU(dalloc(&ctx->e, (size_t)kMaxCoarse + 2));
        CU(dalloc(&ctx->partials, (size_t)kMaxGrid * 256));
        CU(dalloc(&ctx->ow, (size_t)6 * (kOnePassK + 2)));
        CU(dalloc(&ctx->opart, (size_t)kMaxGrid * 3 * (kOnePassK + 2)));
        // q feeds the one-pass partials of the PCG prologue (weighted by 0)
        CU(cudaMemsetAsync(ctx->q, 0, ((size_t)n + 16) * 8, ctx->s));
        ctx->ws_n = n;
        ctx->ws_gen++;
        hist = hist > hist_keep ? hist : hist_keep;
    }
    if (hist > ctx->ws_hist || !ctx->hist) {
        dfree(ctx->hist);
        ctx->hist = nullptr;
        const long long cap = hist > 1 ? hist : 1;
        CU(dalloc(&ctx->hist, (size_t)cap));
        ctx->ws_hist = cap;
        ctx->ws_gen++;
    }
    return NLSP_OK;
}

SolveArgs make_args(nlsp_ctx* c, const nlsp_csr* a, const nlsp_twolevel* m) {
    SolveArgs s{};
    s.n = a->n;
    s.rp = a->rp;
    s.ci = a->ci;
    s.v = a->v;
    s.diag = a->diag;
    s.tile_nnz64 = a->tile_nnz64;
    s.tile_nnz128 = a->tile_nnz128;
    s.tile_nnz256 = a->tile_nnz256;
    s.max_row = a->max_row;
    s.dia = a->dia;
    s.pk = a->pk;
    s.wd = m ? m->wd : nullptr;
    s.wdc = 0.0;
    if (m && a->dia.kind == 1) {
        // every stored entry on an offset is bitwise equal, so every row's
        // omega * (1 / A_ii) (k_wd) is this one value
        for (int t = 0; t < a->dia.d; ++t)
            if (a->dia.off[t] == 0 && a->dia.val[t] > 0.0) s.wdc = m->omega * (1.0 / a->dia.val[t]);
    }
    s.P = m ? m->basis : nullptr;
    s.L = m ? m->L : nullptr;
    s.Ainv = (m && (c->coarse_inverse || m->k > kWideK)) ? m->Ainv : nullptr;
    s.W1 = m ? m->W1 : nullptr;
    s.W2 = m ? m->W2 : nullptr;
    s.k = m ? m->k : 0;
    s.x = c->x;
    s.r = c->r;
    s.r1 = c->r1;
    s.q = c->q;
    s.z = c->z;
    s.p0 = c->p0;
    s.p1 = c->p1;
    s.zt0 = c->zt0;
    s.zt1 = c->zt1;
    s.b = c->b;
    s.hist = c->hist;
    s.st = c->st;
    s.partials = c->partials;
    s.e = c->e;
    s.M = m ? m->M : nullptr;
    s.ow = c->ow;
    s.opart = c->opart;
    return s;
}

// NLSP_QR=robust forces the shifted CholeskyQR3 path of qr_thin_dev (tests)
const bool g_force_sqr = std::getenv("NLSP_QR") && std::strcmp(std::getenv("NLSP_QR"), "robust") == 0;
const bool g_pdl = !(std::getenv("NLSP_PDL") && std::strcmp(std::getenv("NLSP_PDL"), "0") == 0);
// NLSP_PDL_FIRST=1: the first kernel of an unrolled iteration launched with PDL
// too (off: measured slower, C4 443 -> 455 us, C3 413 -> 440 us per iteration)
const bool g_pdl_first = std::getenv("NLSP_PDL_FIRST") && std::strcmp(std::getenv("NLSP_PDL_FIRST"), "1") == 0;
const int g_unroll = [] {
    const char* u = std::getenv("NLSP_UNROLL");
    const int v = u ? std::atoi(u) : 4;  // measured: +1.4 % at C2, +1.8 % at C5 over 1
    return v < 1 ? 1 : (v > 8 ? 8 : v);
}();

// One PCG iteration (the WHILE body). mode: 0 two-level, 1 identity, 2 Jacobi.
void enqueue_iteration(const LaunchCtx& lc, const SolveArgs& a, int mode, const nlsp_twolevel* m,
                       cudaGraphConditionalHandle h, int use_cond, bool pdl_first = false) {
    if (mode == 0 && m->lean) {
        // every kernel after the first of an iteration is launched with PDL, and
        // the first too when it follows another iteration of the same WHILE body
        LaunchCtx lp = lc, l0 = lc;
        lp.pdl = g_pdl;
        l0.pdl = g_pdl && pdl_first;
        launch_lean_iteration(l0, lp, a, m->nu1 + m->nu2, h, use_cond ? 2 : 1);
        return;
    }
    launch_spmv_p(lc, a);
    if (mode == 0 && m->onepass) {
        // x, r, ||r||, c by its recurrence, e (+ the sweeps when fused); prolongation.
        // Each of these kernels starts with pdl_entry(): launched with PDL, it is
        // scheduled while its predecessor drains (NLSP_PDL=0: plain launches)
        LaunchCtx lp = lc;
        lp.pdl = g_pdl;
        launch_onepass_iteration_tail(lp, a, m->nu1 + m->nu2, h, use_cond ? 2 : 1);
        return;
    }
    if (mode == 0 && m->folded) {
        launch_update_restrict(lc, a, true);  // x, r, ||r||, c = W1^T r, e
        // the prolongation ends the iteration and runs the loop control too
        launch_folded_tail(lc, a, m->nu1, m->nu2, h, use_cond ? 2 : 1);
        return;
    }
    launch_update(lc, a, mode);
    if (mode == 0) launch_twolevel_apply(lc, a, m->nu1, m->nu2);
    launch_loop_ctl(lc, a.st, h, use_cond);
}

// prologue: state, r = b, x = 0, ||b||, z = M r, rz
void enqueue_prologue(const LaunchCtx& lc, const SolveArgs& a, int mode, const nlsp_twolevel* m,
                      const double* params_dev) {
    (void)params_dev;
    launch_bnorm(lc, a);
    if (mode == 0 && m->lean) launch_lean_apply(lc, a, m->nu1 + m->nu2);
    else if (mode == 0 && m->onepass) launch_onepass_apply(lc, a, m->nu1 + m->nu2);
    else if (mode == 0 && m->folded) launch_folded_apply(lc, a, m->nu1, m->nu2);
    else if (mode == 0) launch_twolevel_apply(lc, a, m->nu1, m->nu2);
    else launch_init_simple(lc, a, mode == 2 ? 1 : 0);
    launch_init_ctl(lc, a.st);
}

int kind_mode(int kind) { return kind == NLSP_PRECOND_TWOLEVEL ? 0 : (kind == NLSP_PRECOND_JACOBI ? 2 : 1); }

// The solve graph: prologue, WHILE(body), true residual. prologue = false: the
// continuation graph of a later history segment (the loop resumes from the
// device state).
nlsp_status build_graph(nlsp_ctx* ctx, const SolveArgs& a, int mode, const nlsp_twolevel* m,
                        bool prologue = true) {
    cudaGraphExec_t& gx = prologue ? ctx->gexec : ctx->gexec_cont;
    if (gx) {
        cudaGraphExecDestroy(gx);
        gx = nullptr;
    }
    cudaGraph_t g = nullptr;
    LaunchCtx lc = ctx->lc;
    unsigned long long scratch = 0;
    if (prologue) ctx->gk_pro = ctx->gk_body = ctx->gk_epi = 0;
    lc.launches = prologue ? &ctx->gk_pro : &scratch;
    CU(cudaStreamBeginCapture(ctx->s, cudaStreamCaptureModeThreadLocal));
    if (prologue) enqueue_prologue(lc, a, mode, m, nullptr);
    cudaStreamCaptureStatus cs;
    cudaGraph_t cg = nullptr;
    const cudaGraphNode_t* deps = nullptr;
    size_t ndeps = 0;
    cudaError_t e = cudaStreamGetCaptureInfo(ctx->s, &cs, nullptr, &cg, &deps, &ndeps);
    cudaGraphConditionalHandle h{};
    cudaGraphNode_t cnode{};
    cudaGraph_t body = nullptr;
    if (e == cudaSuccess) e = cudaGraphConditionalHandleCreate(&h, cg, 1, cudaGraphCondAssignDefault);
    if (e == cudaSuccess) {
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        e = cudaGraphAddNode(&cnode, cg, deps, ndeps, &cp);
        if (e == cudaSuccess) body = cp.conditional.phGraph_out[0];
    }
    if (e == cudaSuccess)
        e = cudaStreamUpdateCaptureDependencies(ctx->s, &cnode, 1, cudaStreamSetCaptureDependencies);
    if (e == cudaSuccess)
        e = cudaStreamBeginCaptureToGraph(ctx->s_body, body, nullptr, nullptr, 0,
                                          cudaStreamCaptureModeThreadLocal);
    if (e == cudaSuccess) {
        LaunchCtx lb = lc;
        lb.s = ctx->s_body;
        lb.launches = prologue ? &ctx->gk_body : &scratch;
        // NLSP_UNROLL iterations per WHILE body execution (kernels of an
        // iteration after convergence exit at once; each iteration's last
        // kernel still sets the condition)
        for (int u = 0; u < g_unroll; ++u) enqueue_iteration(lb, a, mode, m, h, 1, u > 0 && g_pdl_first);
        e = cudaStreamEndCapture(ctx->s_body, &body);
    }
    lc.launches = prologue ? &ctx->gk_epi : &scratch;
    if (e == cudaSuccess) launch_true_res(lc, a);
    cudaError_t e2 = cudaStreamEndCapture(ctx->s, &g);
    if (e != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        return cuda_fail(ctx, e, "graph build");
    }
    if (e2 != cudaSuccess) return cuda_fail(ctx, e2, "graph capture");
    e = cudaGraphInstantiate(&gx, g, 0);
    cudaGraphDestroy(g);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "graph instantiate");
    return NLSP_OK;
}

// Runs the solve on ctx->b -> ctx->x. Caller has ensured the workspace.
// The loop runs in history segments of ws_hist iterations (hist_chunk): the
// device loop stops at the segment end, the host moves the segment's history
// out and resumes the loop from the device state (a solve that converges
// within the first segment — every BASELINE configuration — is one graph
// launch).
nlsp_status run_pcg(nlsp_ctx* ctx, const nlsp_csr* a, int kind, const nlsp_twolevel* m,
                    double delta, unsigned long long max_iters, nlsp_solve_report* rep) {
    const int mode = kind_mode(kind);
    const SolveArgs args = make_args(ctx, a, m);
    const unsigned long long H = (unsigned long long)ctx->ws_hist;
    unsigned long long seg_end = std::min<unsigned long long>(max_iters, H);
    ctx->hist_done.clear();
    ctx->hist_tail = 0;
    launch_state_init(ctx->lc, ctx->st, delta, (long long)seg_end);
    CHECK_LAUNCH();
    unsigned long long klaunch = 1;
    bool graph_ok = false;
    // small systems: the whole solve in one launch of one thread-block cluster.
    // It cannot pause at a segment end: a solve still running after H
    // iterations (never at the BASELINE sizes) restarts on the multi-kernel path.
    bool cluster_ok = false;
    int c_rows = 0, c_ncta = 0;
    size_t c_smem = 0;
    if (mode == 0 && m->folded && ctx->use_cluster && !a->rp_host.empty())
        c_ncta = cluster_plan(a->n, m->k, a->max_row, m->W2 != m->W1, &c_rows, &c_smem);
    if (c_ncta) {
        ClusterArgs ca{a->n, m->k, m->ld, c_rows, (int)m->nu1, (int)m->nu2, a->max_row, a->rp, a->ci, a->v,
                       m->wd, m->W1, m->W2, m->L, args.Ainv, ctx->b, ctx->x, ctx->hist, (long long)H,
                       ctx->st};
        CU(cudaEventRecord(ctx->ev0, ctx->s));
        const cudaError_t ce = launch_cluster_pcg(ctx->s, ca, c_ncta, c_smem);
        if (ce == cudaSuccess) {
            cluster_ok = true;
            klaunch += 1;
            ctx->launches += 1;
            if (max_iters > H) {
                CU(cudaMemcpyAsync(ctx->st_host, ctx->st, sizeof(PcgState), cudaMemcpyDeviceToHost, ctx->s));
                CU(cudaStreamSynchronize(ctx->s));
                const PcgState& cs = *ctx->st_host;
                if (!cs.error && !cs.converged && (unsigned long long)cs.iterations == seg_end) {
                    cluster_ok = false;
                    launch_state_init(ctx->lc, ctx->st, delta, (long long)seg_end);
                    CHECK_LAUNCH();
                    klaunch += 1;
                }
            }
            if (cluster_ok) ctx->launches += 1;  // the state init
        } else {
            cudaGetLastError();
            ctx->use_cluster = false;  // not schedulable here: multi-kernel path
        }
    }
    if (!cluster_ok && ctx->use_graph) {
        GraphKey key{a->id, m ? m->id : 0, kind, ctx->ws_gen};
        if (!ctx->gexec || !(ctx->gkey == key)) {
            if (build_graph(ctx, args, mode, m) == NLSP_OK) {
                ctx->gkey = key;
            } else {
                ctx->use_graph = false;  // fall back to stream-ordered launches
                ctx->gexec = nullptr;
                ctx->gkey = GraphKey{};
            }
        }
    }
    // one history segment on the multi-kernel path: the graph, or the
    // stream-ordered loop in chunks of iterations (converged kernels exit early)
    unsigned long long segments = 0;
    auto run_segment = [&](bool first, unsigned long long seg_iters) -> nlsp_status {
        ++segments;
        if (graph_ok) {
            if (!first) {
                GraphKey key{a->id, m ? m->id : 0, kind, ctx->ws_gen};
                if (!ctx->gexec_cont || !(ctx->gkey_cont == key)) {
                    const nlsp_status bs = build_graph(ctx, args, mode, m, false);
                    if (bs) return bs;
                    ctx->gkey_cont = key;
                }
            }
            CU(cudaGraphLaunch(first ? ctx->gexec : ctx->gexec_cont, ctx->s));
            return NLSP_OK;
        }
        if (first) {
            enqueue_prologue(ctx->lc, args, mode, m, nullptr);
            CHECK_LAUNCH();
        }
        unsigned long long done_iters = 0;
        const unsigned long long chunk = 16;
        for (;;) {
            for (unsigned long long i = 0; i < chunk && done_iters < seg_iters; ++i, ++done_iters)
                enqueue_iteration(ctx->lc, args, mode, m, cudaGraphConditionalHandle{}, 0);
            CHECK_LAUNCH();
            CU(cudaMemcpyAsync(ctx->st_host, ctx->st, sizeof(PcgState), cudaMemcpyDeviceToHost, ctx->s));
            CU(cudaStreamSynchronize(ctx->s));
            if (ctx->st_host->done || done_iters >= seg_iters) break;
        }
        launch_true_res(ctx->lc, args);
        CHECK_LAUNCH();
        return NLSP_OK;
    };
    // solve_ms starts after the (cached) graph build
    if (!cluster_ok) {
        CU(cudaEventRecord(ctx->ev0, ctx->s));
        graph_ok = ctx->use_graph && ctx->gexec;
        const nlsp_status ss = run_segment(true, seg_end);
        if (ss) return ss;
    }
    CU(cudaMemcpyAsync(ctx->st_host, ctx->st, sizeof(PcgState), cudaMemcpyDeviceToHost, ctx->s));
    CU(cudaStreamSynchronize(ctx->s));
    while (!cluster_ok && !ctx->st_host->error && !ctx->st_host->converged &&
           (unsigned long long)ctx->st_host->iterations == seg_end && seg_end < max_iters) {
        // segment full: keep its history, resume the loop
        const size_t old = ctx->hist_done.size();
        const unsigned long long base = seg_end;
        ctx->hist_done.resize(old + (size_t)(seg_end - (unsigned long long)ctx->st_host->hist_base));
        CU(cudaMemcpyAsync(ctx->hist_done.data() + old, ctx->hist, sizeof(double) * (ctx->hist_done.size() - old),
                           cudaMemcpyDeviceToHost, ctx->s));
        seg_end = std::min<unsigned long long>(max_iters, base + H);
        launch_state_continue(ctx->lc, ctx->st, (long long)seg_end, (long long)base);
        CHECK_LAUNCH();
        klaunch += 1;
        const nlsp_status ss = run_segment(false, seg_end - base);
        if (ss) return ss;
        CU(cudaMemcpyAsync(ctx->st_host, ctx->st, sizeof(PcgState), cudaMemcpyDeviceToHost, ctx->s));
        CU(cudaStreamSynchronize(ctx->s));
    }
    CU(cudaEventRecord(ctx->ev1, ctx->s));
    CU(cudaStreamSynchronize(ctx->s));
    const PcgState& st = *ctx->st_host;
    if (graph_ok) {
        // kernels counted while capturing each graph part; the WHILE body ran
        // st.body_runs times (k_loop_ctl counts itself)
        // (body_runs counts iterations, g_unroll of them per body execution)
        klaunch += ctx->gk_pro + ctx->gk_body * (unsigned long long)st.body_runs / g_unroll +
                   ctx->gk_epi * segments;
        ctx->launches += klaunch;
    }
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
    if (rep) {
        rep->iterations = (unsigned long long)st.iterations;
        rep->converged = st.converged;
        rep->precond_kind = kind;
        rep->true_relative_residual = st.true_res;
        rep->final_relative_residual = st.last_rel;
        rep->solve_ms = ms;
        rep->coarse_dim = m ? (unsigned long long)m->k : 0;
        rep->kernel_launches = klaunch;
    }
    if ((unsigned long long)st.iterations > ctx->hist_done.size())
        ctx->hist_tail = (unsigned long long)st.iterations - ctx->hist_done.size();
    if (st.error) return map_dev_error(ctx, st.error, "pcg");
    return NLSP_OK;
}

// The one-pass cycle carries the restriction by a recurrence; its
// drift against the direct W^T r is measured every iteration on the device.
// Past NLSP_DRIFT_TOL (default 1e-10) the solve is re-run from x0 = 0 on the
// folded cycle (W streamed twice, the restriction direct), which applies the
// same operator without the recurrence.
const double g_drift_tol = [] {
    const char* e = std::getenv("NLSP_DRIFT_TOL");
    return e ? std::atof(e) : 1e-10;
}();

nlsp_status run_pcg_guarded(nlsp_ctx* ctx, const nlsp_csr* a, int kind, const nlsp_twolevel* m,
                            double delta, unsigned long long max_iters, nlsp_solve_report* rep) {
    nlsp_status st = run_pcg(ctx, a, kind, m, delta, max_iters, rep);
    // the lean cycle's second guard: the predicted p.Ap against the direct one
    const double drift = (m && m->lean && kind == NLSP_PRECOND_TWOLEVEL)
                             ? std::max(ctx->st_host->drift_max, ctx->st_host->pap_drift)
                             : ctx->st_host->drift_max;
    if (rep) {
        rep->onepass_drift = drift;
        rep->cycle_fallback = 0;
    }
    if (st != NLSP_OK || kind != NLSP_PRECOND_TWOLEVEL || !m->onepass || !(drift > g_drift_tol)) return st;
    nlsp_twolevel folded = *m;  // same device arrays, W streamed twice per iteration
    folded.onepass = false;
    folded.lean = false;
    folded.id = m->id | (1ull << 63);
    const double ms0 = rep ? rep->solve_ms : 0.0;
    const unsigned long long l0 = rep ? rep->kernel_launches : 0;
    st = run_pcg(ctx, a, kind, &folded, delta, max_iters, rep);
    if (rep) {
        rep->onepass_drift = drift;
        rep->cycle_fallback = 1;
        rep->solve_ms += ms0;
        rep->kernel_launches += l0;
    }
    return st;
}

// Copies the last solve's history: completed segments from the host, the last
// one from the device.
nlsp_status copy_history(nlsp_ctx* ctx, double* out, unsigned long long cap) {
    const unsigned long long nd = std::min<unsigned long long>(cap, ctx->hist_done.size());
    if (nd) std::memcpy(out, ctx->hist_done.data(), sizeof(double) * nd);
    const unsigned long long nt = std::min<unsigned long long>(cap - nd, ctx->hist_tail);
    if (nt) CU(cudaMemcpy(out + nd, ctx->hist, sizeof(double) * nt, cudaMemcpyDeviceToHost));
    return NLSP_OK;
}

nlsp_status check_pcg_args(nlsp_ctx* ctx, const nlsp_csr* a, int kind, const nlsp_twolevel* m) {
    if (!a) return set_err(ctx, NLSP_E_VALIDATION, "pcg: null matrix");
    if (kind < 0 || kind > 2) return set_err(ctx, NLSP_E_VALIDATION, "pcg: unknown preconditioner");
    if (kind == NLSP_PRECOND_TWOLEVEL) {
        if (!m) return set_err(ctx, NLSP_E_VALIDATION, "pcg: two-level preconditioner is NULL");
        if (m->n != a->n) return set_err(ctx, NLSP_E_VALIDATION, "pcg: dimension mismatch");
    }
    // a non-positive diagonal under the Jacobi preconditioner fails on the device
    // (k_init_simple), after the zero-rhs check, in the reference's order
    return NLSP_OK;
}

}  // namespace

// ==================================================================== C-ABI ==
extern "C" {

const char* nlsp_version(void) { return "nlsp-b200 0.1 (sm_100a)"; }

nlsp_status nlsp_ctx_create(int device, nlsp_ctx** out) {
    if (!out) return NLSP_E_VALIDATION;
    *out = nullptr;
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        cudaGetLastError();
        return NLSP_E_CUDA;
    }
    if (device < 0 || device >= count) return NLSP_E_VALIDATION;
    cudaDeviceProp prop{};
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10) return NLSP_E_CUDA;
    auto* ctx = new nlsp_ctx();
    ctx->device = device;
    ctx->num_sms = prop.multiProcessorCount;
    if (cudaSetDevice(device) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->s_body, cudaStreamNonBlocking) != cudaSuccess ||
        cudaMalloc(&ctx->st, sizeof(PcgState)) != cudaSuccess ||
        cudaMallocHost(&ctx->st_host, sizeof(PcgState)) != cudaSuccess ||
        cudaMalloc(&ctx->flags, 16 * sizeof(int)) != cudaSuccess ||
        cudaMallocHost(&ctx->flags_host, 16 * sizeof(int)) != cudaSuccess ||
        cudaEventCreate(&ctx->ev0) != cudaSuccess || cudaEventCreate(&ctx->ev1) != cudaSuccess ||
        cudaEventCreate(&ctx->ev2) != cudaSuccess || cudaEventCreate(&ctx->ev3) != cudaSuccess) {
        cudaGetLastError();
        nlsp_ctx_destroy(ctx);
        return NLSP_E_CUDA;
    }
    {
        cudaMemPoolProps pp{};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = device;
        unsigned long long keep = ~0ull;
        if (cudaMemPoolCreate(&ctx->pool, &pp) != cudaSuccess ||
            cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &keep) != cudaSuccess) {
            cudaGetLastError();
            nlsp_ctx_destroy(ctx);
            return NLSP_E_CUDA;
        }
    }
    cudaMemset(ctx->st, 0, sizeof(PcgState));
    ctx->lc.s = ctx->s;
    ctx->lc.num_sms = ctx->num_sms;
    ctx->lc.launches = &ctx->launches;
    const char* loop = std::getenv("NLSP_LOOP");
    ctx->use_graph = !(loop && std::strcmp(loop, "host") == 0);
    const char* clu = std::getenv("NLSP_CLUSTER");
    ctx->use_cluster = !(clu && std::strcmp(clu, "0") == 0);
    const char* co = std::getenv("NLSP_COARSE");
    ctx->coarse_inverse = !(co && std::strcmp(co, "chol") == 0);
    const char* sd = std::getenv("NLSP_S0_DRAW");
    ctx->s0_draw = (sd && std::strcmp(sd, "device") == 0) ? NLSP_S0_DRAW_DEVICE : NLSP_S0_DRAW_HOST;
    *out = ctx;
    return NLSP_OK;
}

void nlsp_ctx_destroy(nlsp_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    if (ctx->s) cudaStreamSynchronize(ctx->s);
    if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
    if (ctx->gexec_cont) cudaGraphExecDestroy(ctx->gexec_cont);
    for (int b = 0; b < 2; ++b) {
        if (ctx->s0_pin[b]) cudaFreeHost(ctx->s0_pin[b]);
        if (ctx->s0_ev[b]) cudaEventDestroy(ctx->s0_ev[b]);
    }
    free_ws(ctx);
    dfree(ctx->mt_polys);
    dfree(ctx->st);
    dfree(ctx->flags);
    if (ctx->st_host) cudaFreeHost(ctx->st_host);
    if (ctx->flags_host) cudaFreeHost(ctx->flags_host);
    for (cudaEvent_t ev : {ctx->ev0, ctx->ev1, ctx->ev2, ctx->ev3})
        if (ev) cudaEventDestroy(ev);
    if (ctx->s_body) cudaStreamDestroy(ctx->s_body);
    if (ctx->s) cudaStreamDestroy(ctx->s);
    if (ctx->pool) cudaMemPoolDestroy(ctx->pool);
    delete ctx;
}

const char* nlsp_last_error(const nlsp_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

void* nlsp_ctx_stream(nlsp_ctx* ctx) { return ctx ? static_cast<void*>(ctx->s) : nullptr; }

uint64_t nlsp_ctx_kernel_launches(const nlsp_ctx* ctx) { return ctx ? ctx->launches : 0; }

nlsp_status nlsp_ctx_synchronize(nlsp_ctx* ctx) {
    nlsp_status b = bind(ctx);
    if (b) return b;
    CU(cudaStreamSynchronize(ctx->s));
    return NLSP_OK;
}

// ---------------------------------------------------------------------- CSR --
// Diagonal form of a CSR matrix (DiaArgs, internal.cuh): the sorted set of
// column offsets (at most kMaxDia), per-row presence bits and either the one
// value every entry of an offset shares (kind 1) or a d x n value slab (kind 2).
// Returns false when the offsets do not fit or the form would not stream fewer
// bytes than the CSR arrays.
// When the offsets fit but the value slab does not pay, pk / pmask receive the
// implicit-column form (PackArgs, internal.cuh) and the function returns false.
static bool detect_dia(uint64_t n, uint64_t nnz, const uint64_t* rp, const uint64_t* ci,
                       const double* v, DiaArgs& d, std::vector<unsigned char>& mask,
                       std::vector<double>& rv, PackArgs& pk, std::vector<unsigned>& pmask) {
    if (n == 0 || nnz == 0) return false;
    long long offs[kMaxDia];
    int D = 0;
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const long long o = (long long)ci[k] - (long long)i;
            const long long* at = std::lower_bound(offs, offs + D, o);
            if (at < offs + D && *at == o) continue;
            if (D == kMaxDia) return false;
            const int pos = (int)(at - offs);
            for (int t = D; t > pos; --t) offs[t] = offs[t - 1];
            offs[pos] = o;
            ++D;
        }
    const int mb = D <= 8 ? 1 : (D <= 16 ? 2 : 4);
    double cv[kMaxDia];
    bool seen[kMaxDia] = {false}, constant = true;
    mask.assign((size_t)n * mb, 0);
    for (uint64_t i = 0; i < n; ++i) {
        unsigned m = 0;
        for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const int t = (int)(std::lower_bound(offs, offs + D, (long long)ci[k] - (long long)i) - offs);
            m |= 1u << t;
            if (!seen[t]) {
                cv[t] = v[k];
                seen[t] = true;
            } else if (std::memcmp(&cv[t], &v[k], sizeof(double)) != 0) {
                constant = false;
            }
        }
        std::memcpy(mask.data() + (size_t)i * mb, &m, mb);  // little endian
    }
    const double csr_bytes = 12.0 * (double)nnz + 4.0 * (double)(n + 1);
    const double dia_bytes = (double)n * (mb + (constant ? 0 : 8 * D));
    if (!constant && dia_bytes > 0.8 * csr_bytes) {
        pk = PackArgs{};
        pk.d = D;
        for (int t = 0; t < D; ++t) pk.off[t] = (int)offs[t];
        pmask.assign((size_t)n, 0u);
        for (uint64_t i = 0; i < n; ++i) {
            unsigned m = 0;
            std::memcpy(&m, mask.data() + (size_t)i * mb, mb);
            pmask[i] = m;
        }
        return false;
    }
    if (!constant) {
        rv.assign((size_t)D * n, 0.0);
        for (uint64_t i = 0; i < n; ++i)
            for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
                const int t = (int)(std::lower_bound(offs, offs + D, (long long)ci[k] - (long long)i) - offs);
                rv[(size_t)t * n + i] = v[k];
            }
    }
    d = DiaArgs{};
    d.kind = constant ? 1 : 2;
    d.d = D;
    d.mbytes = mb;
    for (int t = 0; t < D; ++t) {
        d.off[t] = (int)offs[t];
        d.val[t] = constant ? cv[t] : 0.0;
    }
    // structured-grid geometry for the plane-march kernels (march.cuh): the
    // plane stride P (a positive offset) for which every offset is dz P + dd
    // with dz in {-1, 0, 1} and the smallest halo max |dd| (<= P / 4), P | n
    for (int c = 0; c < D; ++c) {
        const long long P = offs[c];
        if (P < 2 || (long long)n % P != 0 || (long long)n / P < 3) continue;
        long long h = 0;
        for (int t = 0; t < D; ++t) {
            const long long o = offs[t];
            const long long dz = o > P / 2 ? 1 : (o < -P / 2 ? -1 : 0);
            const long long r = o - dz * P;
            h = std::max(h, r < 0 ? -r : r);
            if (o > P + P / 2 || o < -P - P / 2) h = P;  // beyond the neighbouring planes
        }
        if (h >= 1 && 4 * h <= P && (d.plane == 0 || h < d.halo)) {
            d.plane = P;
            d.halo = (int)h;
        }
    }
    return true;
}

nlsp_status nlsp_csr_upload(nlsp_ctx* ctx, uint64_t n, uint64_t nnz, const uint64_t* row_ptr,
                            const uint64_t* col_idx, const double* values, nlsp_csr** out) {
    if (!out) return set_err(ctx, NLSP_E_VALIDATION, "csr_upload: null out");
    *out = nullptr;
    nlsp_status b = bind(ctx);
    if (b) return b;
    if (n >= (1ull << 31) || nnz >= (1ull << 31))
        return set_err(ctx, NLSP_E_VALIDATION, "csr_upload: n and nnz must be < 2^31");
    if (!row_ptr || (nnz && (!col_idx || !values)))
        return set_err(ctx, NLSP_E_VALIDATION, "csr_upload: null array");
    if (row_ptr[0] != 0 || row_ptr[n] != nnz)
        return set_err(ctx, NLSP_E_VALIDATION, "csr_upload: row_ptr must start at 0 and end at nnz");
    auto* a = new nlsp_csr();
    a->id = g_next_id++;
    a->device = ctx->device;
    a->n = (int)n;
    a->nnz = (long long)nnz;
    unsigned long long *rp64 = nullptr, *ci64 = nullptr;
    auto fail = [&](cudaError_t e, const char* w) {
        sfree(ctx, rp64);
        sfree(ctx, ci64);
        nlsp_csr_destroy(a);
        return cuda_fail(ctx, e, w);
    };
    cudaError_t e;
    // TMA-staged tiles: max nonzeros per 64 / 128-row tile; arrays padded so the
    // 16-B-rounded bulk copies of the last tile stay inside the allocations
    a->tile_nnz64 = a->tile_nnz128 = a->tile_nnz256 = 0;
    for (uint64_t r0 = 0; r0 < n; r0 += 64) {
        auto span = [&](uint64_t len) {
            const uint64_t r1 = r0 + len < n ? r0 + len : n;
            return (int)(row_ptr[r1] - row_ptr[r0]);
        };
        a->tile_nnz64 = std::max(a->tile_nnz64, span(64));
        if ((r0 & 127) == 0) a->tile_nnz128 = std::max(a->tile_nnz128, span(128));
        if ((r0 & 255) == 0) a->tile_nnz256 = std::max(a->tile_nnz256, span(256));
    }
    if ((e = dalloc(&a->rp, n + 1 + 16)) || (e = dalloc(&a->ci, nnz + 16)) || (e = dalloc(&a->v, nnz + 16)) ||
        (e = dalloc(&a->diag, n)) || (e = salloc(ctx, &rp64, n + 1)) || (e = salloc(ctx, &ci64, nnz)))
        return fail(e, "csr_upload alloc");
    if ((e = cudaMemcpyAsync(rp64, row_ptr, (n + 1) * 8, cudaMemcpyHostToDevice, ctx->s)) ||
        (nnz && (e = cudaMemcpyAsync(ci64, col_idx, nnz * 8, cudaMemcpyHostToDevice, ctx->s))) ||
        (nnz && (e = cudaMemcpyAsync(a->v, values, nnz * 8, cudaMemcpyHostToDevice, ctx->s))) ||
        (e = cudaMemsetAsync(ctx->flags, 0, 16 * sizeof(int), ctx->s)))
        return fail(e, "csr_upload copy");
    if (n == 0) {
        cudaMemsetAsync(a->rp, 0, sizeof(int), ctx->s);
    } else {
        launch_csr_import(ctx->lc, (int)n, (long long)nnz, rp64, ci64, a->v, a->rp, a->ci, a->diag,
                          ctx->flags, ctx->flags + 1);
    }
    if ((e = cudaGetLastError())) return fail(e, "csr_import launch");
    if ((e = cudaMemcpyAsync(ctx->flags_host, ctx->flags, 16 * sizeof(int), cudaMemcpyDeviceToHost,
                             ctx->s)) ||
        (e = cudaStreamSynchronize(ctx->s)))
        return fail(e, "csr_upload sync");
    sfree(ctx, rp64);
    sfree(ctx, ci64);
    rp64 = ci64 = nullptr;
    const int fl = ctx->flags_host[0];
    if (fl) {
        nlsp_csr_destroy(a);
        return set_err(ctx, NLSP_E_VALIDATION,
                       (fl & 1) ? "csr_upload: row_ptr not monotone"
                       : (fl & 2) ? "csr_upload: column index out of range"
                                  : "csr_upload: columns must be sorted without duplicates");
    }
    a->max_row = ctx->flags_host[1];
    if (n <= 65536) a->rp_host.assign(row_ptr, row_ptr + n + 1);
    a->pass_bytes = 12ull * nnz + 4ull * (n + 1);
    {
        const char* de = std::getenv("NLSP_DIA");
        std::vector<unsigned char> mask;
        std::vector<double> rv;
        std::vector<unsigned> pmask;
        PackArgs pk{};
        DiaArgs d{};
        const char* pe = std::getenv("NLSP_PACK");
        if (!(de && de[0] == '0') && detect_dia(n, nnz, row_ptr, col_idx, values, d, mask, rv, pk, pmask)) {
            if ((e = dalloc(reinterpret_cast<unsigned char**>(&a->dia_mask), mask.size() + 16)) ||
                (e = cudaMemcpyAsync(a->dia_mask, mask.data(), mask.size(), cudaMemcpyHostToDevice, ctx->s)))
                return fail(e, "csr_upload diagonal form");
            if (d.kind == 2) {
                if ((e = dalloc(&a->dia_rv, rv.size() + 16)) ||
                    (e = cudaMemcpyAsync(a->dia_rv, rv.data(), rv.size() * 8, cudaMemcpyHostToDevice, ctx->s)))
                    return fail(e, "csr_upload diagonal values");
            }
            if ((e = cudaStreamSynchronize(ctx->s))) return fail(e, "csr_upload diagonal sync");
            d.mask = a->dia_mask;
            d.rv = a->dia_rv;
            a->dia = d;
            a->pass_bytes = (unsigned long long)n * (d.mbytes + (d.kind == 2 ? 8ull * d.d : 0ull));
        } else if (!pmask.empty() && pe && pe[0] == '1' && a->tile_nnz64 >= 64 && a->tile_nnz256 >= 256) {
            // implicit columns (opt-in, NLSP_PACK=1): the staged tiles carry one mask
            // per row where the column indices were (the 64- and 256-row tiles'
            // column regions hold them). Off by default: 30 % fewer matrix bytes at
            // C5, but the per-nonzero decode (next set bit -> offset -> address)
            // sits in front of every gather of kernels that are latency-bound, not
            // bandwidth-bound: measured 117 -> 144 us per iteration at C5.
            if ((e = dalloc(&a->pk_mask, pmask.size() + 16)) ||
                (e = cudaMemcpyAsync(a->pk_mask, pmask.data(), pmask.size() * 4, cudaMemcpyHostToDevice, ctx->s)) ||
                (e = cudaStreamSynchronize(ctx->s)))
                return fail(e, "csr_upload implicit columns");
            pk.mask = a->pk_mask;
            a->pk = pk;
            a->pass_bytes = 8ull * nnz + 4ull * (n + 1) + 4ull * n;
        }
    }
    // diag_ok: any A_ii <= 0 ?
    {
        int* f = ctx->flags + 2;
        double* tmp = nullptr;
        if ((e = salloc(ctx, &tmp, n)) || (e = cudaMemsetAsync(f, 0, sizeof(int), ctx->s))) {
            sfree(ctx, tmp);
            return fail(e, "csr_upload diag");
        }
        launch_wd(ctx->lc, (int)n, a->diag, 1.0, tmp, f);
        e = cudaMemcpyAsync(ctx->flags_host + 2, f, sizeof(int), cudaMemcpyDeviceToHost, ctx->s);
        sfree(ctx, tmp);
        if (!e) e = cudaStreamSynchronize(ctx->s);
        if (e) return fail(e, "csr_upload diag sync");
        a->diag_ok = ctx->flags_host[2] == 0;
    }
    *out = a;
    return NLSP_OK;
}

void nlsp_csr_destroy(nlsp_csr* a) {
    if (!a) return;
    cudaSetDevice(a->device);
    dfree(a->rp);
    dfree(a->ci);
    dfree(a->v);
    dfree(a->diag);
    dfree(a->dia_mask);
    dfree(a->dia_rv);
    dfree(a->pk_mask);
    delete a;
}

nlsp_status nlsp_csr_format(const nlsp_csr* a, int* kind, int* offsets, uint64_t* pass_bytes) {
    if (!a) return NLSP_E_VALIDATION;
    if (kind) *kind = a->dia.kind ? a->dia.kind : (a->pk.mask ? 3 : 0);
    if (offsets) *offsets = a->dia.kind ? a->dia.d : (a->pk.mask ? a->pk.d : 0);
    if (pass_bytes) *pass_bytes = a->pass_bytes;
    return NLSP_OK;
}

nlsp_status nlsp_csr_geometry(nlsp_ctx* ctx, const nlsp_csr* a, uint64_t* plane, int* halo, int* march) {
    if (!a) return NLSP_E_VALIDATION;
    if (plane) *plane = a->dia.kind ? (uint64_t)a->dia.plane : 0;
    if (halo) *halo = a->dia.kind ? a->dia.halo : 0;
    if (march) {
        SolveArgs s{};
        s.n = a->n;
        s.dia = a->dia;
        *march = (ctx && march_planned(ctx->lc, s)) ? 1 : 0;
    }
    return NLSP_OK;
}

void nlsp_csr_dims(const nlsp_csr* a, uint64_t* n, uint64_t* nnz) {
    if (n) *n = a ? (uint64_t)a->n : 0;
    if (nnz) *nnz = a ? (uint64_t)a->nnz : 0;
}

nlsp_status nlsp_spmv_device(nlsp_ctx* ctx, const nlsp_csr* a, const double* x, double* y) {
    nlsp_status b = bind(ctx);
    if (b) return b;
    if (!a) return set_err(ctx, NLSP_E_VALIDATION, "spmv: null matrix");
    if (a->n) launch_spmv_args(ctx->lc, make_args(ctx, a, nullptr), x, y);
    CHECK_LAUNCH();
    CU(cudaStreamSynchronize(ctx->s));
    return NLSP_OK;
}

nlsp_status nlsp_spmv(nlsp_ctx* ctx, const nlsp_csr* a, const double* x, double* y) {
    nlsp_status b = bind(ctx);
    if (b) return b;
    if (!a || !x || !y) return set_err(ctx, NLSP_E_VALIDATION, "spmv: null argument");
    b = ensure_ws(ctx, a->n, 1);
    if (b) return b;
    const size_t bytes = (size_t)a->n * 8;
    CU(cudaMemcpyAsync(ctx->zt0, x, bytes, cudaMemcpyHostToDevice, ctx->s));
    if (a->n) launch_spmv_args(ctx->lc, make_args(ctx, a, nullptr), ctx->zt0, ctx->zt1);
    CHECK_LAUNCH();
    CU(cudaMemcpyAsync(y, ctx->zt1, bytes, cudaMemcpyDeviceToHost, ctx->s));
    CU(cudaStreamSynchronize(ctx->s));
    return NLSP_OK;
}

nlsp_status nlsp_csr_diagonal(nlsp_ctx* ctx, const nlsp_csr* a, double* d) {
    nlsp_status b = bind(ctx);
    if (b) return b;
    if (!a || !d) return set_err(ctx, NLSP_E_VALIDATION, "diagonal: null argument");
    CU(cudaMemcpy(d, a->diag, (size_t)a->n * 8, cudaMemcpyDeviceToHost));
    return NLSP_OK;
}

// -------------------------------------------------------------------- dense --
static nlsp_status dense_alloc(nlsp_ctx* ctx, uint64_t rows, uint64_t cols, nlsp_dense** out) {
    auto* d = new nlsp_dense();
    d->id = g_next_id++;
    d->device = ctx->device;
    d->rows = rows;
    d->cols = cols;
    cudaError_t e = dalloc(&d->d, rows * cols);
    if (e) {
        delete d;
        return cuda_fail(ctx, e, "dense alloc");
    }
    *out = d;
    return NLSP_OK;
}

nlsp_status nlsp_dense_upload(nlsp_ctx* ctx, uint64_t rows, uint64_t cols, const double* host,
                              nlsp_dense** out) {
    if (!out) return set_err(ctx, NLSP_E_VALIDATION, "dense_upload: null out");
    *out = nullptr;
    nlsp_status b = bind(ctx);
    if (b) return b;
    if (rows * cols && !host) return set_err(ctx, NLSP_E_VALIDATION, "dense_upload: null data");
    nlsp_dense* d = nullptr;
    b = dense_alloc(ctx, rows, cols, &d);
    if (b) return b;
    if (rows * cols) {
        cudaError_t e = cudaMemcpy(d->d, host, rows * cols * 8, cudaMemcpyHostToDevice);
        if (e) {
            nlsp_dense_destroy(d);
            return cuda_fail(ctx, e, "dense_upload copy");
        }
    }
    *out = d;
    return NLSP_OK;
}

nlsp_status nlsp_dense_export(nlsp_ctx* ctx, const nlsp_dense* d, double* host) {
    nlsp_status b = bind(ctx);
    if (b) return b;
    if (!d || (!host && d->rows * d->cols)) return set_err(ctx, NLSP_E_VALIDATION, "dense_export: null");
    CU(cudaStreamSynchronize(ctx->s));
    if (d->rows * d->cols) CU(cudaMemcpy(host, d->d, d->rows * d->cols * 8, cudaMemcpyDeviceToHost));
    return NLSP_OK;
}

void nlsp_dense_dims(const nlsp_dense* d, uint64_t* rows, uint64_t* cols) {
    if (rows) *rows = d ? d->rows : 0;
    if (cols) *cols = d ? d->cols : 0;
}

void* nlsp_dense_data(const nlsp_dense* d) { return d ? d->d : nullptr; }

void nlsp_dense_destroy(nlsp_dense* d) {
    if (!d) return;
    cudaSetDevice(d->device);
    dfree(d->d);
    delete d;
}

// ---------------------------------------------------------------- smoothing --
nlsp_status nlsp_jacobi_sweeps(nlsp_ctx* ctx, const nlsp_csr* a, double omega, uint64_t sweeps,
                               double* x, const double* b) {
    nlsp_status st = bind(ctx);
    if (st) return st;
    if (!a || !x || !b) return set_err(ctx, NLSP_E_VALIDATION, "jacobi sweep: null argument");
    if (omega < 0.0 || omega > 1.0)
        return set_err(ctx, NLSP_E_VALIDATION, "jacobi: omega must lie in [0, 1]");
    if (!a->diag_ok) return set_err(ctx, NLSP_E_NUMERIC, "jacobi: non-positive diagonal");
    st = ensure_ws(ctx, a->n, 1);
    if (st) return st;
    double* wd = nullptr;
    CU(salloc(ctx, &wd, a->n));
    launch_wd(ctx->lc, a->n, a->diag, omega, wd, ctx->flags + 3);
    const size_t bytes = (size_t)a->n * 8;
    CU(cudaMemcpyAsync(ctx->zt0, x, bytes, cudaMemcpyHostToDevice, ctx->s));
    CU(cudaMemcpyAsync(ctx->r, b, bytes, cudaMemcpyHostToDevice, ctx->s));
    CU(cudaMemsetAsync(ctx->st, 0, sizeof(PcgState), ctx->s));
    nlsp_twolevel fake{};
    fake.wd = wd;
    SolveArgs args = make_args(ctx, a, &fake);
    double* cur = ctx->zt0;
    for (uint64_t s = 0; s < sweeps; ++s) {
        double* nxt = (cur == ctx->zt0) ? ctx->zt1 : ctx->zt0;
        launch_sweep(ctx->lc, args, false, cur, nxt, false);
        cur = nxt;
    }
    CHECK_LAUNCH();
    sfree(ctx, wd);
    CU(cudaMemcpyAsync(x, cur, bytes, cudaMemcpyDeviceToHost, ctx->s));
    CU(cudaStreamSynchronize(ctx->s));
    return NLSP_OK;
}

static nlsp_status smooth_impl(nlsp_ctx* ctx, const nlsp_csr* a, nlsp_dense* s, uint64_t sweeps,
                               double omega) {
    if (omega < 0.0 || omega > 1.0)
        return set_err(ctx, NLSP_E_VALIDATION, "jacobi: omega must lie in [0, 1]");
    if (!a->diag_ok) return set_err(ctx, NLSP_E_NUMERIC, "jacobi: non-positive diagonal");
    if (s->rows != (uint64_t)a->n)
        return set_err(ctx, NLSP_E_VALIDATION, "jacobi sweep: dimension mismatch");
    if (sweeps == 0 || s->cols == 0 || a->n == 0) return NLSP_OK;
    double *wd = nullptr, *tmp = nullptr;
    CU(salloc(ctx, &wd, a->n));
    cudaError_t e = salloc(ctx, &tmp, s->rows * s->cols);
    if (e) {
        sfree(ctx, wd);
        return cuda_fail(ctx, e, "smooth alloc");
    }
    launch_wd(ctx->lc, a->n, a->diag, omega, wd, ctx->flags + 3);
    double* cur = s->d;
    double* other = tmp;
    for (uint64_t k = 0; k < sweeps; ++k) {
        if (!launch_block_op_dia(ctx->lc, 0, a->n, a->dia, wd, (int)s->cols, cur, other))
            launch_block_op(ctx->lc, 0, a->n, a->rp, a->ci, a->v, wd, (int)s->cols, cur, other);
        double* t = cur;
        cur = other;
        other = t;
    }
    e = cudaGetLastError();
    if (!e && cur != s->d)
        e = cudaMemcpyAsync(s->d, cur, s->rows * s->cols * 8, cudaMemcpyDeviceToDevice, ctx->s);
    sfree(ctx, wd);
    sfree(ctx, tmp);
    if (!e) e = cudaStreamSynchronize(ctx->s);
    if (e) return cuda_fail(ctx, e, "smooth");
    return NLSP_OK;
}

nlsp_status nlsp_smooth_vectors(nlsp_ctx* ctx, const nlsp_csr* a, nlsp_dense* s, uint64_t sweeps,
                                double omega) {
    nlsp_status st = bind(ctx);
    if (st) return st;
    if (!a || !s) return set_err(ctx, NLSP_E_VALIDATION, "smooth: null argument");
    return smooth_impl(ctx, a, s, sweeps, omega);
}

nlsp_status nlsp_ctx_set_s0_draw(nlsp_ctx* ctx, int32_t mode) {
    if (!ctx) return NLSP_E_VALIDATION;
    if (mode != NLSP_S0_DRAW_HOST && mode != NLSP_S0_DRAW_DEVICE)
        return set_err(ctx, NLSP_E_VALIDATION, "set_s0_draw: unknown mode");
    ctx->s0_draw = mode;
    return NLSP_OK;
}

int32_t nlsp_ctx_last_s0_draw(const nlsp_ctx* ctx) { return ctx ? ctx->last_s0_draw : -1; }

namespace {
constexpr int kS0Log2B = 18;  // words per device substream (s0_device.cu)

// The first `count` normals of Rng(stream_seed) into dst (device, count
// doubles), drawn on the device. *redo is set when the stream holds a zero u1
// (the reference would redraw it and shift every later value): the caller then
// draws on the host. words_only: dst receives the raw mt19937_64 words instead.
nlsp_status s0_draw_device(nlsp_ctx* ctx, std::uint64_t stream_seed, unsigned long long count, double* dst,
                           bool* redo, bool words_only = false) {
    *redo = false;
    if (count == 0) return NLSP_OK;
    const unsigned long long total = (count + 1) / 2 * 2;
    const long long nsub = (long long)((total + (1ull << kS0Log2B) - 1) >> kS0Log2B);
    int levels = 0;
    while ((1ll << levels) < nsub) ++levels;
    if (kS0Log2B + levels - 1 > nlsp_host::kMtJumpMaxLog2) {  // beyond the tabulated jumps
        *redo = true;
        return NLSP_OK;
    }
    if (!ctx->mt_polys) {
        CU(cudaMalloc(&ctx->mt_polys, sizeof(nlsp_host::kMtJump)));
        CU(cudaMemcpy(ctx->mt_polys, nlsp_host::kMtJump, sizeof(nlsp_host::kMtJump), cudaMemcpyHostToDevice));
    }
    unsigned long long* win = nullptr;
    unsigned long long* tail = nullptr;
    cudaError_t e = cudaSuccess;
    auto cleanup = [&]() {
        sfree(ctx, win);
        sfree(ctx, tail);
    };
    std::uint64_t w0[nlsp_host::kMtN];
    nlsp_host::mt64_seed(stream_seed, w0);
    if ((e = salloc(ctx, &win, (size_t)nsub * nlsp_host::kMtN)) || (e = salloc(ctx, &tail, 2)) ||
        (e = cudaMemcpyAsync(win, w0, sizeof(w0), cudaMemcpyHostToDevice, ctx->s)) ||
        (e = cudaMemsetAsync(ctx->flags, 0, sizeof(int), ctx->s))) {
        cleanup();
        return cuda_fail(ctx, e, "s0 device draw alloc");
    }
    launch_mt_stream(ctx->lc, win, nsub, kS0Log2B, ctx->mt_polys, nlsp_host::kMtJumpMinLog2, total, count,
                     reinterpret_cast<unsigned long long*>(dst), tail);
    if (!words_only) launch_box_muller(ctx->lc, dst, count, tail, ctx->flags);
    e = cudaGetLastError();
    if (!e) e = cudaMemcpyAsync(ctx->flags_host, ctx->flags, sizeof(int), cudaMemcpyDeviceToHost, ctx->s);
    if (!e) e = cudaStreamSynchronize(ctx->s);
    cleanup();
    if (e) return cuda_fail(ctx, e, "s0 device draw");
    *redo = ctx->flags_host[0] != 0;
    return NLSP_OK;
}
}  // namespace

// test hook: the first `count` raw words of std::mt19937_64(seed), generated
// on the device by the jump tree, copied to the host
nlsp_status nlsp_mt19937_64_words(nlsp_ctx* ctx, uint64_t seed, uint64_t count, uint64_t* out) {
    nlsp_status st = bind(ctx);
    if (st) return st;
    if (!out && count) return set_err(ctx, NLSP_E_VALIDATION, "mt19937_64_words: null out");
    if (count == 0) return NLSP_OK;
    double* d = nullptr;
    const unsigned long long even = (count + 1) / 2 * 2;
    cudaError_t e = salloc(ctx, &d, (size_t)even);
    if (e) return cuda_fail(ctx, e, "mt19937_64_words alloc");
    bool redo = false;
    st = s0_draw_device(ctx, seed, even, d, &redo, true);
    if (!st && redo) st = set_err(ctx, NLSP_E_VALIDATION, "mt19937_64_words: count beyond the tabulated jumps");
    if (!st) {
        e = cudaMemcpyAsync(out, d, sizeof(uint64_t) * count, cudaMemcpyDeviceToHost, ctx->s);
        if (!e) e = cudaStreamSynchronize(ctx->s);
        if (e) st = cuda_fail(ctx, e, "mt19937_64_words copy");
    }
    sfree(ctx, d);
    return st;
}

// S^(0) streams from the host generator to the device chunk by chunk (4 M
// normal pairs = 64 MB): each chunk is Box-Muller-transformed into one of two
// pinned staging buffers while the previous one is in flight (cudaMemcpyAsync
// on ctx->s), so the 4.2 GB upload at C4 hides behind the sequential
// mt19937_64 draw. Rows under the Dirichlet mask take no values from the
// stream (smoothing.hpp:84-92): the live rows' chunk is scattered on the
// device (k_s0_scatter).
nlsp_status nlsp_generate_smoothed_vectors(nlsp_ctx* ctx, const nlsp_csr* a, const uint8_t* mask,
                                           uint64_t k, uint64_t sweeps, double omega,
                                           uint64_t seed, nlsp_dense** out) {
    if (!out) return set_err(ctx, NLSP_E_VALIDATION, "generate_smoothed_vectors: null out");
    *out = nullptr;
    nlsp_status st = bind(ctx);
    if (st) return st;
    if (!a) return set_err(ctx, NLSP_E_VALIDATION, "generate_smoothed_vectors: null matrix");
    if (k < 1) return set_err(ctx, NLSP_E_VALIDATION, "generate_smoothed_vectors: K must be positive");
    const unsigned long long n = (unsigned long long)a->n;
    constexpr unsigned long long kChunkPairs = 1ull << 22;
    nlsp_dense* d = nullptr;
    st = dense_alloc(ctx, n, k, &d);
    if (st) return st;
    std::vector<int> live;
    unsigned long long nlive = n;
    if (mask) {
        for (unsigned long long i = 0; i < n; ++i)
            if (!mask[i]) live.push_back((int)i);
        nlive = live.size();
    }
    int* dlive = nullptr;
    double* dstage[2] = {nullptr, nullptr};
    ctx->last_s0_draw = NLSP_S0_DRAW_HOST;
    if (ctx->s0_draw == NLSP_S0_DRAW_DEVICE) {
        // the stream's nlive * k normals straight into S (or, under a mask, into
        // a buffer of the live rows that is then scattered)
        bool redo = false;
        double* dlivebuf = nullptr;
        cudaError_t de = cudaSuccess;
        if (mask) {
            if ((de = cudaMemsetAsync(d->d, 0, sizeof(double) * n * k, ctx->s)) ||
                (de = salloc(ctx, &dlive, (size_t)std::max<unsigned long long>(nlive, 1))) ||
                (nlive && (de = cudaMemcpyAsync(dlive, live.data(), sizeof(int) * nlive, cudaMemcpyHostToDevice, ctx->s))) ||
                (de = salloc(ctx, &dlivebuf, (size_t)(nlive * k + 2)))) {
                sfree(ctx, dlive);
                sfree(ctx, dlivebuf);
                nlsp_dense_destroy(d);
                return cuda_fail(ctx, de, "generate_smoothed_vectors alloc");
            }
        }
        st = s0_draw_device(ctx, nlsp_host::mix_seed(seed, 0x736d6f6f), nlive * k, mask ? dlivebuf : d->d, &redo);
        if (!st && !redo && mask && nlive)
            launch_s0_scatter(ctx->lc, dlivebuf, 0, (long long)(nlive * k), (int)k, dlive, d->d);
        if (mask) {
            if (!st) de = cudaStreamSynchronize(ctx->s);  // live (host vector) is read by the copy above
            sfree(ctx, dlive);
            sfree(ctx, dlivebuf);
            dlive = nullptr;
            if (!st && de) st = cuda_fail(ctx, de, "generate_smoothed_vectors scatter");
        }
        if (st) {
            nlsp_dense_destroy(d);
            return st;
        }
        if (!redo) {
            ctx->last_s0_draw = NLSP_S0_DRAW_DEVICE;
            st = smooth_impl(ctx, a, d, sweeps, omega);
            if (st) {
                nlsp_dense_destroy(d);
                return st;
            }
            *out = d;
            return NLSP_OK;
        }
        // a zero u1 in the stream (or a stream beyond the jump table): the host draw below
    }
    for (int b = 0; b < 2; ++b) {
        cudaError_t pe = cudaSuccess;
        if (!ctx->s0_pin[b]) pe = cudaMallocHost(&ctx->s0_pin[b], sizeof(double) * 2 * kChunkPairs);
        if (!pe && !ctx->s0_ev[b]) pe = cudaEventCreateWithFlags(&ctx->s0_ev[b], cudaEventDisableTiming);
        if (pe) {
            nlsp_dense_destroy(d);
            return cuda_fail(ctx, pe, "generate_smoothed_vectors staging");
        }
    }
    auto cleanup = [&]() {
        sfree(ctx, dlive);
        sfree(ctx, dstage[0]);
        sfree(ctx, dstage[1]);
    };
    cudaError_t e = cudaSuccess;
    if (mask) {
        if ((e = cudaMemsetAsync(d->d, 0, sizeof(double) * n * k, ctx->s)) ||
            (e = salloc(ctx, &dlive, (size_t)std::max<unsigned long long>(nlive, 1))) ||
            (nlive && (e = cudaMemcpyAsync(dlive, live.data(), sizeof(int) * nlive, cudaMemcpyHostToDevice, ctx->s))) ||
            (e = salloc(ctx, &dstage[0], 2 * kChunkPairs)) || (e = salloc(ctx, &dstage[1], 2 * kChunkPairs))) {
            cleanup();
            nlsp_dense_destroy(d);
            return cuda_fail(ctx, e, "generate_smoothed_vectors alloc");
        }
    }
    struct DeviceSink {
        nlsp_ctx* ctx;
        double* dst;
        int* live;
        double* const* stage;
        unsigned long long count, m;
        int cur = 0;
        bool used[2] = {false, false};
        cudaError_t err = cudaSuccess;
        double* buffer(unsigned long long, unsigned long long) {
            if (used[cur] && !err) err = cudaEventSynchronize(ctx->s0_ev[cur]);
            return ctx->s0_pin[cur];
        }
        void done(unsigned long long base, unsigned long long np) {
            const unsigned long long e0 = 2 * base, cnt = std::min(2 * np, count - e0);
            if (!err) {
                if (!live) {
                    err = cudaMemcpyAsync(dst + e0, ctx->s0_pin[cur], sizeof(double) * cnt, cudaMemcpyHostToDevice,
                                          ctx->s);
                } else {
                    err = cudaMemcpyAsync(stage[cur], ctx->s0_pin[cur], sizeof(double) * cnt, cudaMemcpyHostToDevice,
                                          ctx->s);
                    if (!err) launch_s0_scatter(ctx->lc, stage[cur], (long long)e0, (long long)cnt, (int)m, live, dst);
                }
            }
            if (!err) err = cudaEventRecord(ctx->s0_ev[cur], ctx->s);
            used[cur] = true;
            cur ^= 1;
        }
    } sink{ctx, d->d, mask ? dlive : nullptr, dstage, nlive * k, k};
    nlsp_host::normal_stream_chunks(nlsp_host::mix_seed(seed, 0x736d6f6f), nlive * k, sink, kChunkPairs);
    e = sink.err;
    if (!e) e = cudaStreamSynchronize(ctx->s);  // the staging buffers are reused by the next call
    cleanup();
    if (e) {
        nlsp_dense_destroy(d);
        return cuda_fail(ctx, e, "generate_smoothed_vectors upload");
    }
    st = smooth_impl(ctx, a, d, sweeps, omega);
    if (st) {
        nlsp_dense_destroy(d);
        return st;
    }
    *out = d;
    return NLSP_OK;
}

// ---------------------------------------------------------------- SVD basis --
nlsp_status nlsp_svd_basis(nlsp_ctx* ctx, const nlsp_dense* s, uint64_t k, nlsp_dense** p_out,
                           double* sigma, int32_t* eigh_sweeps) {
    if (!p_out) return set_err(ctx, NLSP_E_VALIDATION, "svd_basis: null out");
    *p_out = nullptr;
    nlsp_status st = bind(ctx);
    if (st) return st;
    if (!s) return set_err(ctx, NLSP_E_VALIDATION, "svd_basis: null matrix");
    const long long n = (long long)s->rows;
    const int m = (int)std::min<unsigned long long>(s->cols, 1u << 30);
    if (m == 0 || n == 0) return set_err(ctx, NLSP_E_VALIDATION, "svd_oracle: empty matrix");
    // svd.hpp:161-165: the eigensolve runs on the Gram of the smaller dimension
    // (S^T S for a tall S, S S^T for a wide one), gdim = r = min(n, m)
    const bool wide = (long long)m > n;
    const int gdim = wide ? (int)n : m;
    if (gdim > 1024) return set_err(ctx, NLSP_E_VALIDATION, "svd_basis: min(rows, cols) at most 1024");
    if (k > (uint64_t)gdim) return set_err(ctx, NLSP_E_VALIDATION, "first_cols: k exceeds column count");
    if (k > 256) return set_err(ctx, NLSP_E_VALIDATION, "svd_basis: at most 256 basis columns");
    if (k == 0) {
        nlsp_dense* d = nullptr;
        st = dense_alloc(ctx, n, 0, &d);
        if (!st) *p_out = d;
        return st;
    }
    const long long grow = wide ? (long long)m : n;  // rows the Gram streams
    const int g = gram_grid(ctx->lc, grow);
    double *part = nullptr, *G = nullptr, *ev = nullptr, *V = nullptr, *sa = nullptr, *sv = nullptr,
           *sig = nullptr, *W = nullptr, *pmag = nullptr, *pval = nullptr, *sign = nullptr, *T = nullptr,
           *vcol = nullptr, *cpart = nullptr, *cval = nullptr, *Gk = nullptr;
    long long* pidx = nullptr;
    nlsp_dense* P = nullptr;
    auto cleanup = [&]() {
        for (double* p : {part, G, ev, V, sa, sv, sig, W, pmag, pval, sign, T, vcol, cpart, cval, Gk}) sfree(ctx, p);
        sfree(ctx, pidx);
    };
    auto fail = [&](nlsp_status code, const std::string& msg) {
        cleanup();
        if (P) nlsp_dense_destroy(P);
        return set_err(ctx, code, msg);
    };
    cudaError_t e;
    const size_t gg = (size_t)gdim * gdim;
    if ((e = salloc(ctx, &part, (size_t)g * gram_tile(gdim, gdim))) || (e = salloc(ctx, &G, gg)) ||
        (e = salloc(ctx, &ev, gdim)) || (e = salloc(ctx, &V, gg)) || (e = salloc(ctx, &sa, gg)) ||
        (e = salloc(ctx, &sv, gg)) || (e = salloc(ctx, &sig, gdim)) || (e = salloc(ctx, &W, (size_t)gdim * k)) ||
        (e = salloc(ctx, &pmag, (size_t)ctx->num_sms * kColsignPerSm * k)) ||
        (e = salloc(ctx, &pval, (size_t)ctx->num_sms * kColsignPerSm * k)) ||
        (e = salloc(ctx, &pidx, (size_t)ctx->num_sms * kColsignPerSm * k)) || (e = salloc(ctx, &sign, k)) ||
        (wide && (e = salloc(ctx, &T, (size_t)n * m)))) {
        cleanup();
        return cuda_fail(ctx, e, "svd_basis alloc");
    }
    CU(cudaMemsetAsync(ctx->flags, 0, 16 * sizeof(int), ctx->s));
    // Gram (svd.hpp:161-166), eigensolve (:167), sigma with the rounding floor
    // and the first k eigenvectors W (:174-183)
    if (wide) {
        launch_transpose(ctx->lc, n, m, s->d, T);
        launch_gram(ctx->lc, m, gdim, gdim, T, T, part, G);
    } else {
        launch_gram(ctx->lc, n, m, m, s->d, s->d, part, G);
    }
    launch_eigh(ctx->lc, gdim, G, ev, V, sa, sv, ctx->flags + 4, ctx->flags + 5);
    launch_sigma(ctx->lc, gdim, (int)k, ev, V, sig, W, ctx->flags + 6);
    e = cudaGetLastError();
    if (!e) e = cudaMemcpyAsync(ctx->flags_host, ctx->flags, 16 * sizeof(int), cudaMemcpyDeviceToHost, ctx->s);
    if (!e) e = cudaStreamSynchronize(ctx->s);
    if (e) {
        cleanup();
        return cuda_fail(ctx, e, "svd_basis");
    }
    if (eigh_sweeps) *eigh_sweeps = ctx->flags_host[5];
    if (ctx->flags_host[4] == kErrValidation) return fail(NLSP_E_VALIDATION, "svd_oracle: non-finite entries");
    if (ctx->flags_host[4]) return fail(NLSP_E_CONVERGENCE, "jacobi_eigh: no convergence after 30 sweeps");
    if (sigma) CU(cudaMemcpy(sigma, sig, sizeof(double) * gdim, cudaMemcpyDeviceToHost));
    const int solid = ctx->flags_host[6];
    st = dense_alloc(ctx, n, k, &P);
    if (st) {
        cleanup();
        return st;
    }
    if (wide) {
        // U = the eigenvectors of S S^T themselves (svd.hpp:186, 205)
        CU(cudaMemcpyAsync(P->d, W, sizeof(double) * (size_t)n * k, cudaMemcpyDeviceToDevice, ctx->s));
    } else {
        // U_j = S V_j / sigma_j for the solid columns (svd.hpp:189-202; the
        // columns past `solid` are overwritten by the completion below)
        launch_dense_mm(ctx->lc, n, m, (int)k, s->d, W, sig, P->d);
        const int gd = std::max(1, std::min(ctx->num_sms * 2, (int)((n + 255) / 256)));
        if ((e = salloc(ctx, &vcol, (size_t)n)) || (e = salloc(ctx, &cpart, (size_t)gd + 64)) ||
            (e = salloc(ctx, &cval, 2)) || (e = salloc(ctx, &Gk, (size_t)k * k))) {
            cleanup();
            nlsp_dense_destroy(P);
            return cuda_fail(ctx, e, "svd_basis alloc");
        }
        const int kk = (int)k;
        // complete_orthonormal (svd.hpp:101-126): column j from the coordinate
        // vector e_cand with the largest residual > 0.5, candidates in order
        for (int j = solid; j < kk; ++j) {
            bool placed = false;
            for (long long cand = 0; cand < n && !placed; ++cand) {
                launch_col_move(ctx->lc, n, kk, P->d, -1, vcol, nullptr, 0, cand);
                for (int pass = 0; pass < 2; ++pass)
                    for (int p = 0; p < j; ++p) {
                        launch_coldot(ctx->lc, n, kk, P->d, p, vcol, cpart, cval);
                        launch_col_axpy(ctx->lc, n, kk, P->d, p, vcol, cval);
                    }
                launch_coldot(ctx->lc, n, kk, P->d, -1, vcol, cpart, cval + 1);
                double nrm = 0.0;
                CU(cudaMemcpyAsync(&nrm, cval + 1, sizeof(double), cudaMemcpyDeviceToHost, ctx->s));
                CU(cudaStreamSynchronize(ctx->s));
                if (nrm > 0.5) {
                    launch_col_move(ctx->lc, n, kk, P->d, j, vcol, cval + 1, 1, 0);
                    placed = true;
                }
            }
            if (!placed) return fail(NLSP_E_NUMERIC, "complete_orthonormal: no candidate found");
        }
        // orthonormality_defect (dense.hpp:175-182) of the k columns; past 1e-11
        // the Gram-Schmidt polish (svd.hpp:128-145). (The reference measures
        // the defect over all min(n, m) columns; a polish triggered only by
        // the later columns moves the first k by less than their own defect,
        // < 1e-11.)
        launch_gram(ctx->lc, n, kk, kk, P->d, P->d, part, Gk);
        std::vector<double> gk((size_t)k * k);
        CU(cudaMemcpyAsync(gk.data(), Gk, sizeof(double) * gk.size(), cudaMemcpyDeviceToHost, ctx->s));
        CU(cudaStreamSynchronize(ctx->s));
        double defect = 0.0;
        for (int i = 0; i < kk; ++i)
            for (int j = 0; j < kk; ++j) defect = std::max(defect, std::fabs(gk[(size_t)i * k + j] - (i == j ? 1.0 : 0.0)));
        ctx->last_svd_defect = defect;
        ctx->last_svd_solid = solid;
        if (defect > 1e-11) {
            for (int j = 0; j < kk; ++j) {
                launch_col_move(ctx->lc, n, kk, P->d, j, vcol, nullptr, 0, 0);
                for (int p = 0; p < j; ++p) {
                    launch_coldot(ctx->lc, n, kk, P->d, p, vcol, cpart, cval);
                    launch_col_axpy(ctx->lc, n, kk, P->d, p, vcol, cval);
                }
                launch_coldot(ctx->lc, n, kk, P->d, -1, vcol, cpart, cval + 1);
                double nrm = 0.0;
                CU(cudaMemcpyAsync(&nrm, cval + 1, sizeof(double), cudaMemcpyDeviceToHost, ctx->s));
                CU(cudaStreamSynchronize(ctx->s));
                if (nrm == 0.0) return fail(NLSP_E_NUMERIC, "reorthonormalize: zero column");
                launch_col_move(ctx->lc, n, kk, P->d, j, vcol, cval + 1, 1, 0);
            }
        }
    }
    // sign convention (svd.hpp:209-225)
    launch_colsign(ctx->lc, n, (int)k, P->d, pmag, pidx, pval, sign);
    e = cudaGetLastError();
    if (!e) e = cudaStreamSynchronize(ctx->s);
    cleanup();
    if (e) {
        nlsp_dense_destroy(P);
        return cuda_fail(ctx, e, "svd_basis products");
    }
    *p_out = P;
    return NLSP_OK;
}

// qr_thin (qr.hpp:18-45) on the device: Q (n x k, orthonormal, R with a
// positive diagonal, so the same Q as the reference's two-pass MGS up to
// rounding) from the basis B.
//
// CholeskyQR2 (R1 = chol(B^T B), Q1 = B R1^-1; R2 = chol(Q1^T Q1), Q = Q1 R2^-1)
// when B is well conditioned: every first-pass pivot L_jj (= MGS's
// post-elimination norm of column j, up to the Gram's rounding of
// eps ||B||_F^2) is at least 1e-6 ||B||_F, so the reference's rank test
// (nrm < 1e-12 ||B||_F) cannot trigger and Q is orthonormal to rounding.
// Otherwise the Gram has lost the small pivots to rounding (they square the
// condition number), and shifted CholeskyQR3 takes over: R1 = chol(B^T B + s I)
// with s = 11 (n k + k (k + 1)) u ||B||_F^2, then CholeskyQR2 on B R1^-1 —
// orthonormal for cond(B) up to ~1/u. Its rank test is the reference's own on
// the diagonal of R = Q^T B (the post-elimination norms, resolved to
// ~u ||B||_F): R_jj < 1e-12 ||B||_F -> RankDeficiencyError; a second-stage
// Cholesky breakdown means B is numerically rank-deficient too.
// Scratch: Q1, Y (n x k), part, G, U (k x k); L (k x k + 8) ends as garbage.
static nlsp_status qr_thin_dev(nlsp_ctx* ctx, long long n, int k, const double* B, double* Q, double* Q1, double* Y,
                        double* part, double* G, double* U, double* L) {
    const LaunchCtx& lc = ctx->lc;
    CU(cudaMemsetAsync(ctx->flags + 8, 0, 3 * sizeof(int), ctx->s));
    launch_gram(lc, n, k, k, B, B, part, G);
    launch_chol(lc, k, G, L, 0.0, ctx->flags + 8);
    std::vector<double> gd(k), ld(k);
    CU(cudaMemcpy2DAsync(gd.data(), 8, G, (size_t)(k + 1) * 8, 8, k, cudaMemcpyDeviceToHost, ctx->s));
    CU(cudaMemcpy2DAsync(ld.data(), 8, L, (size_t)(k + 1) * 8, 8, k, cudaMemcpyDeviceToHost, ctx->s));
    CU(cudaMemcpyAsync(ctx->flags_host + 8, ctx->flags + 8, sizeof(int), cudaMemcpyDeviceToHost, ctx->s));
    CU(cudaStreamSynchronize(ctx->s));
    double fro2 = 0.0, lmin = HUGE_VAL;
    for (int j = 0; j < k; ++j) {
        fro2 += gd[j];
        lmin = std::min(lmin, ld[j]);
    }
    const double fro = std::sqrt(std::max(fro2, 0.0));
    if (!(fro > 0.0)) return set_err(ctx, NLSP_E_RANK_DEFICIENT, "qr_thin: rank-deficient at column 0");
    const bool fast = ctx->flags_host[8] == 0 && lmin >= 1e-6 * fro && !g_force_sqr;
    if (fast) {
        launch_tri_inv_t(lc, k, L, U);
        launch_dense_mm(lc, n, k, k, B, U, nullptr, Q1);
        launch_gram(lc, n, k, k, Q1, Q1, part, G);
        launch_chol(lc, k, G, L, 0.0, ctx->flags + 9);
        launch_tri_inv_t(lc, k, L, U);
        launch_dense_mm(lc, n, k, k, Q1, U, nullptr, Q);
        ctx->last_qr_robust = false;
        return NLSP_OK;
    }
    // shifted CholeskyQR3
    const double u = std::ldexp(1.0, -53);
    const double shift = 11.0 * ((double)n * k + (double)k * (k + 1)) * u * fro2;
    launch_gram(lc, n, k, k, B, B, part, G);
    launch_shift_diag(lc, k, G, shift);
    launch_chol(lc, k, G, L, 0.0, ctx->flags + 9);
    launch_tri_inv_t(lc, k, L, U);
    launch_dense_mm(lc, n, k, k, B, U, nullptr, Q1);
    launch_gram(lc, n, k, k, Q1, Q1, part, G);
    launch_chol(lc, k, G, L, 0.0, ctx->flags + 10);
    launch_tri_inv_t(lc, k, L, U);
    launch_dense_mm(lc, n, k, k, Q1, U, nullptr, Y);
    launch_gram(lc, n, k, k, Y, Y, part, G);
    launch_chol(lc, k, G, L, 0.0, ctx->flags + 10);
    launch_tri_inv_t(lc, k, L, U);
    launch_dense_mm(lc, n, k, k, Y, U, nullptr, Q);
    // R = Q^T B: its diagonal holds the post-elimination norms
    launch_gram(lc, n, k, k, Q, B, part, G);
    CU(cudaGetLastError());
    CU(cudaMemcpy2DAsync(gd.data(), 8, G, (size_t)(k + 1) * 8, 8, k, cudaMemcpyDeviceToHost, ctx->s));
    CU(cudaMemcpyAsync(ctx->flags_host + 9, ctx->flags + 9, 2 * sizeof(int), cudaMemcpyDeviceToHost, ctx->s));
    CU(cudaStreamSynchronize(ctx->s));
    ctx->last_qr_robust = true;
    for (int j = 0; j < k; ++j)
        if (!(gd[j] >= 1e-12 * fro))
            return set_err(ctx, NLSP_E_RANK_DEFICIENT, "qr_thin: rank-deficient at column " + std::to_string(j));
    if (ctx->flags_host[9] || ctx->flags_host[10])
        return set_err(ctx, NLSP_E_RANK_DEFICIENT, "qr_thin: rank-deficient basis");
    return NLSP_OK;
}

// -------------------------------------------------------- two-level operator --
nlsp_status nlsp_twolevel_build(nlsp_ctx* ctx, const nlsp_csr* a, const nlsp_dense* basis,
                                double omega, uint64_t nu1, uint64_t nu2, nlsp_twolevel** out) {
    if (!out) return set_err(ctx, NLSP_E_VALIDATION, "two-level: null out");
    *out = nullptr;
    nlsp_status st = bind(ctx);
    if (st) return st;
    if (!a || !basis) return set_err(ctx, NLSP_E_VALIDATION, "two-level: null argument");
    // smoother_ is constructed first (two_level.hpp:25), then the basis checks
    if (omega < 0.0 || omega > 1.0)
        return set_err(ctx, NLSP_E_VALIDATION, "jacobi: omega must lie in [0, 1]");
    if (!a->diag_ok) return set_err(ctx, NLSP_E_NUMERIC, "jacobi: non-positive diagonal");
    if (basis->cols == 0) return set_err(ctx, NLSP_E_VALIDATION, "two-level: empty coarse space");
    if (basis->rows != (uint64_t)a->n)
        return set_err(ctx, NLSP_E_VALIDATION, "two-level: basis row count must match matrix dimension");
    const int k = (int)basis->cols;
    const long long n = a->n;
    if (k > kMaxCoarse)
        return set_err(ctx, NLSP_E_VALIDATION, "two-level: coarse dimension above 2048 unsupported");
    if ((long long)k > n) return set_err(ctx, NLSP_E_VALIDATION, "qr_thin: requires rows >= cols");
    auto* m = new nlsp_twolevel();
    m->id = g_next_id++;
    m->device = ctx->device;
    m->n = (int)n;
    m->k = k;
    m->ld = k + (k & 1);
    m->nu1 = nu1;
    m->nu2 = nu2;
    m->omega = omega;
    {
        const char* cyc = std::getenv("NLSP_CYCLE");
        // wide coarse spaces (k > 256) run the folded cycle only
        m->folded = !(cyc && std::strcmp(cyc, "literal") == 0) || k > kWideK;
        m->onepass = m->folded && nu1 == nu2 && onepass_supported(k) &&
                     !(cyc && std::strcmp(cyc, "folded") == 0);
    }
    const size_t kk = (size_t)k * k;
    const int g = gram_grid(ctx->lc, n);
    double *part = nullptr, *G = nullptr, *U = nullptr, *Q1 = nullptr, *Q = nullptr, *Y = nullptr;
    auto cleanup = [&]() {
        for (double* p : {part, G, U, Q1, Q, Y}) sfree(ctx, p);
    };
    auto fail_cuda = [&](cudaError_t e, const char* w) {
        cleanup();
        nlsp_twolevel_destroy(m);
        return cuda_fail(ctx, e, w);
    };
    cudaError_t e;
    if ((e = dalloc(&m->basis, (size_t)n * m->ld)) || (e = dalloc(&m->L, kk + 8)) ||
        (e = dalloc(&m->Ainv, kk)) || (e = dalloc(&m->coarse, kk)) || (e = dalloc(&m->wd, n)) ||
        (e = salloc(ctx, &part, (size_t)g * gram_tile(k, k))) || (e = salloc(ctx, &G, kk)) || (e = salloc(ctx, &U, kk)) ||
        (e = salloc(ctx, &Q1, (size_t)n * k)) || (e = salloc(ctx, &Q, (size_t)n * k)) ||
        (e = salloc(ctx, &Y, (size_t)n * k)))
        return fail_cuda(e, "two-level alloc");
    if ((e = cudaMemsetAsync(ctx->flags, 0, 16 * sizeof(int), ctx->s))) return fail_cuda(e, "memset");
    launch_wd(ctx->lc, (int)n, a->diag, omega, m->wd, ctx->flags + 7);
    {
        // qr_thin (qr.hpp:18-45): CholeskyQR2, or shifted CholeskyQR3 for an
        // ill-conditioned basis (qr_thin_dev)
        const nlsp_status qs = qr_thin_dev(ctx, n, k, basis->d, Q, Q1, Y, part, G, U, m->L);
        if (qs) {
            cleanup();
            nlsp_twolevel_destroy(m);
            return qs;
        }
    }
    // Galerkin A_c = Q^T (A Q), exact symmetrisation, Cholesky (two_level.hpp:33-52)
    if (!launch_block_op_dia(ctx->lc, 1, (int)n, a->dia, nullptr, k, Q, Y))
        launch_block_op(ctx->lc, 1, (int)n, a->rp, a->ci, a->v, nullptr, k, Q, Y);
    launch_gram(ctx->lc, n, k, k, Q, Y, part, m->coarse);
    launch_symmetrize(ctx->lc, k, m->coarse);
    launch_chol(ctx->lc, k, m->coarse, m->L, 0.0, ctx->flags + 10);
    launch_tri_inv_t(ctx->lc, k, m->L, U);
    launch_coarse_inverse(ctx->lc, k, U, m->Ainv);
    // basis with an even leading dimension (zero pad column for odd k)
    if (!(e = cudaGetLastError()))
        e = cudaMemcpy2DAsync(m->basis, (size_t)m->ld * 8, Q, (size_t)k * 8, (size_t)k * 8, n,
                              cudaMemcpyDeviceToDevice, ctx->s);
    if (!e && m->ld != k)
        e = cudaMemset2DAsync(m->basis + k, (size_t)m->ld * 8, 0, 8, n, ctx->s);
    // folded cycle bases W = (I - w D^-1 A)^nu P: nu homogeneous block sweeps
    // of the orthonormal basis (smoothing.hpp:50-60 applied to its k columns)
    auto fold = [&](unsigned long long nu, double** out) -> cudaError_t {
        cudaError_t err = dalloc(out, (size_t)n * m->ld);
        if (err) return err;
        double* cur = Q;
        double* other = Y;  // Y and Q1 are free scratch (n x k) at this point
        for (unsigned long long s = 0; s < nu; ++s) {
            double* dst = (cur == Y) ? Q1 : Y;
            if (!launch_block_op_dia(ctx->lc, 0, (int)n, a->dia, m->wd, k, cur, dst))
                launch_block_op(ctx->lc, 0, (int)n, a->rp, a->ci, a->v, m->wd, k, cur, dst);
            cur = dst;
        }
        (void)other;
        err = cudaMemcpy2DAsync(*out, (size_t)m->ld * 8, cur, (size_t)k * 8, (size_t)k * 8, n,
                                cudaMemcpyDeviceToDevice, ctx->s);
        if (!err && m->ld != k) err = cudaMemset2DAsync(*out + k, (size_t)m->ld * 8, 0, 8, n, ctx->s);
        if (!err && m->onepass) {
            // M = W^T (A W) for the one-pass restriction recurrence
            double* aw = (cur == Y) ? Q1 : Y;
            err = dalloc(&m->M, kk);
            if (err) return err;
            if (!launch_block_op_dia(ctx->lc, 1, (int)n, a->dia, nullptr, k, cur, aw))
                launch_block_op(ctx->lc, 1, (int)n, a->rp, a->ci, a->v, nullptr, k, cur, aw);
            launch_gram(ctx->lc, n, k, k, cur, aw, part, m->M);
            launch_symmetrize(ctx->lc, k, m->M);
        }
        return err;
    };
    if (!e && m->folded) {
        e = fold(nu1, &m->W1);
        if (!e) {
            if (nu2 == nu1) m->W2 = m->W1;
            else e = fold(nu2, &m->W2);
        }
    }
    if (!e) e = cudaMemcpyAsync(ctx->flags_host, ctx->flags, 16 * sizeof(int), cudaMemcpyDeviceToHost, ctx->s);
    if (!e) e = cudaStreamSynchronize(ctx->s);
    if (e) return fail_cuda(e, "two-level build");
    cleanup();
    const int* f = ctx->flags_host;
    if (f[7]) {
        nlsp_twolevel_destroy(m);
        return set_err(ctx, NLSP_E_NUMERIC, "jacobi: non-positive diagonal");
    }
    if (f[9]) {  // CholeskyQR2's second pass
        nlsp_twolevel_destroy(m);
        return set_err(ctx, NLSP_E_RANK_DEFICIENT, "qr_thin: rank-deficient basis");
    }
    if (f[10]) {
        nlsp_twolevel_destroy(m);
        return map_dev_error(ctx, f[10], "cholesky");
    }
    {
        const char* cyc = std::getenv("NLSP_CYCLE");
        m->lean = m->onepass && !(cyc && std::strcmp(cyc, "onepass") == 0) &&
                  lean_supported(make_args(ctx, a, m), nu1 + nu2);
    }
    *out = m;
    return NLSP_OK;
}

void nlsp_twolevel_destroy(nlsp_twolevel* m) {
    if (!m) return;
    cudaSetDevice(m->device);
    if (m->W2 && m->W2 != m->W1) dfree(m->W2);
    for (double* p : {m->basis, m->L, m->Ainv, m->coarse, m->wd, m->W1, m->M}) dfree(p);
    delete m;
}

int nlsp_twolevel_cycle(const nlsp_twolevel* m) {
    if (!m) return -1;
    return m->lean ? 3 : (m->onepass ? 2 : (m->folded ? 1 : 0));
}

void nlsp_twolevel_dims(const nlsp_twolevel* m, uint64_t* n, uint64_t* k) {
    if (n) *n = m ? (uint64_t)m->n : 0;
    if (k) *k = m ? (uint64_t)m->k : 0;
}

nlsp_status nlsp_twolevel_export(nlsp_ctx* ctx, const nlsp_twolevel* m, double* basis, double* chol,
                                 double* coarse) {
    nlsp_status st = bind(ctx);
    if (st) return st;
    if (!m) return set_err(ctx, NLSP_E_VALIDATION, "two-level export: null handle");
    CU(cudaStreamSynchronize(ctx->s));
    const size_t kk = (size_t)m->k * m->k * 8;
    if (basis)
        CU(cudaMemcpy2D(basis, (size_t)m->k * 8, m->basis, (size_t)m->ld * 8, (size_t)m->k * 8,
                        (size_t)m->n, cudaMemcpyDeviceToHost));
    if (chol) CU(cudaMemcpy(chol, m->L, kk, cudaMemcpyDeviceToHost));
    if (coarse) CU(cudaMemcpy(coarse, m->coarse, kk, cudaMemcpyDeviceToHost));
    return NLSP_OK;
}

nlsp_status nlsp_twolevel_apply(nlsp_ctx* ctx, const nlsp_twolevel* m, const nlsp_csr* a,
                                const double* r, double* z) {
    nlsp_status st = bind(ctx);
    if (st) return st;
    if (!m || !a || !r || !z) return set_err(ctx, NLSP_E_VALIDATION, "two-level apply: null argument");
    if (a->n != m->n) return set_err(ctx, NLSP_E_VALIDATION, "two-level apply: dimension mismatch");
    st = ensure_ws(ctx, a->n, 1);
    if (st) return st;
    const size_t bytes = (size_t)a->n * 8;
    CU(cudaMemcpyAsync(ctx->r, r, bytes, cudaMemcpyHostToDevice, ctx->s));
    CU(cudaMemsetAsync(ctx->st, 0, sizeof(PcgState), ctx->s));
    const SolveArgs args = make_args(ctx, a, m);
    if (m->folded) launch_folded_apply(ctx->lc, args, m->nu1, m->nu2);
    else launch_twolevel_apply(ctx->lc, args, m->nu1, m->nu2);
    CHECK_LAUNCH();
    CU(cudaMemcpyAsync(z, ctx->z, bytes, cudaMemcpyDeviceToHost, ctx->s));
    CU(cudaStreamSynchronize(ctx->s));
    return NLSP_OK;
}

// ---------------------------------------------------------------------- PCG --
nlsp_status nlsp_pcg(nlsp_ctx* ctx, const nlsp_csr* a, int kind, const nlsp_twolevel* m,
                     const double* b, double delta, uint64_t max_iters, double* x,
                     nlsp_solve_report* rep, double* residual_history) {
    nlsp_status st = bind(ctx);
    if (st) return st;
    st = check_pcg_args(ctx, a, kind, m);
    if (st) return st;
    if (!b || !x) return set_err(ctx, NLSP_E_VALIDATION, "pcg: null vector");
    st = ensure_ws(ctx, a->n, hist_segment(max_iters));
    if (st) return st;
    const size_t bytes = (size_t)a->n * 8;
    CU(cudaEventRecord(ctx->ev2, ctx->s));
    CU(cudaMemcpyAsync(ctx->b, b, bytes, cudaMemcpyHostToDevice, ctx->s));
    nlsp_solve_report local{};
    nlsp_solve_report* r = rep ? rep : &local;
    std::memset(r, 0, sizeof(*r));
    st = run_pcg_guarded(ctx, a, kind, m, delta, max_iters, r);
    if (st) return st;
    if (residual_history) {
        st = copy_history(ctx, residual_history, r->iterations);
        if (st) return st;
    }
    CU(cudaMemcpyAsync(x, ctx->x, bytes, cudaMemcpyDeviceToHost, ctx->s));
    CU(cudaEventRecord(ctx->ev3, ctx->s));
    CU(cudaStreamSynchronize(ctx->s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev2, ctx->ev3);
    r->total_ms = ms;
    r->h2d_bytes = bytes;
    r->d2h_bytes = bytes + sizeof(PcgState) + (residual_history ? r->iterations * 8 : 0);
    return NLSP_OK;
}

nlsp_status nlsp_pcg_device(nlsp_ctx* ctx, const nlsp_csr* a, int kind, const nlsp_twolevel* m,
                            const double* b_dev, double delta, uint64_t max_iters, double* x_dev,
                            nlsp_solve_report* rep, double* residual_history) {
    nlsp_status st = bind(ctx);
    if (st) return st;
    st = check_pcg_args(ctx, a, kind, m);
    if (st) return st;
    if (!b_dev || !x_dev) return set_err(ctx, NLSP_E_VALIDATION, "pcg: null vector");
    st = ensure_ws(ctx, a->n, hist_segment(max_iters));
    if (st) return st;
    const size_t bytes = (size_t)a->n * 8;
    CU(cudaEventRecord(ctx->ev2, ctx->s));
    CU(cudaMemcpyAsync(ctx->b, b_dev, bytes, cudaMemcpyDeviceToDevice, ctx->s));
    nlsp_solve_report local{};
    nlsp_solve_report* r = rep ? rep : &local;
    std::memset(r, 0, sizeof(*r));
    st = run_pcg_guarded(ctx, a, kind, m, delta, max_iters, r);
    if (st) return st;
    if (residual_history) {
        st = copy_history(ctx, residual_history, r->iterations);
        if (st) return st;
    }
    CU(cudaMemcpyAsync(x_dev, ctx->x, bytes, cudaMemcpyDeviceToDevice, ctx->s));
    CU(cudaEventRecord(ctx->ev3, ctx->s));
    CU(cudaStreamSynchronize(ctx->s));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev2, ctx->ev3);
    r->total_ms = ms;
    r->h2d_bytes = 0;
    r->d2h_bytes = sizeof(PcgState) + (residual_history ? r->iterations * 8 : 0);
    return NLSP_OK;
}

nlsp_status nlsp_pcg_history(nlsp_ctx* ctx, double* out, uint64_t cap, uint64_t* count) {
    nlsp_status st = bind(ctx);
    if (st) return st;
    const unsigned long long total = ctx->hist_done.size() + ctx->hist_tail;
    if (count) *count = total;
    if (!out || !cap) return NLSP_OK;
    return copy_history(ctx, out, std::min<unsigned long long>(cap, total));
}

// ---------------------------------------------------------------- profiling --
int nlsp_pcg_profile(nlsp_ctx* ctx, const nlsp_csr* a, int kind, const nlsp_twolevel* m,
                     const double* b_dev, uint64_t iters, nlsp_kernel_stat* stats, int cap) {
    if (bind(ctx) || check_pcg_args(ctx, a, kind, m) || !b_dev || !stats || cap <= 0) return -1;
    if (ensure_ws(ctx, a->n, (long long)iters + 1)) return -1;
    const int mode = kind_mode(kind);
    const SolveArgs args = make_args(ctx, a, m);
    cudaMemcpyAsync(ctx->b, b_dev, (size_t)a->n * 8, cudaMemcpyDeviceToDevice, ctx->s);
    launch_state_init(ctx->lc, ctx->st, 0.0, (long long)iters);
    enqueue_prologue(ctx->lc, args, mode, m, nullptr);
    struct Acc {
        const char* name;
        double bytes;
        unsigned long long launches = 0;
        double ms = 0.0;
    };
    const double n = a->n, nnz = (double)a->nnz, k = m ? m->k : 0;
    const double csr = 12.0 * nnz + 4.0 * (n + 1);
    const double pass = (double)a->pass_bytes;  // CSR, or the diagonal form when detected
    // algorithmic bytes per launch; slots by name below
    enum { kSpmvP = 0, kUpd, kRes, kPro, kPost, kUR, kSmooth, kCtl, kUO, kPO, kUS, kUSF, kSU, kSL, kPL, kSLF, kSL1, kSlots };
    const bool onepass = mode == 0 && m->onepass;
    const unsigned long long T = m ? m->nu1 + m->nu2 : 0;
    std::vector<Acc> acc = {
        {"spmv_p", pass + 32.0 * n},                 // reads z, p; writes p, q
        {"update", (mode == 0 ? 48.0 : (mode == 1 ? 56.0 : 64.0)) * n},
        {"restrict", csr + 8.0 * n * k + 16.0 * n},  // literal: P, r, w (implicit z1)
        {"prolong", 8.0 * n * k + 24.0 * n},         // literal: P, r, w; writes z2
        {"post_sweep", pass + 32.0 * n},             // z2, r, w; writes z
        {"update_restrict", 8.0 * n * k + 48.0 * n}, // folded: W1, x, p, q, r; writes x, r
        // sweeps (the first from zero: r, w, s; later: s, r, w, s'), w not read when constant
        {"smooth", pass + ((m && m->nu1 + m->nu2 == 2) ? 24.0 : 32.0) * n - (args.wdc != 0.0 ? 8.0 * n : 0.0)},
        {"loop_ctl", 0.0},
        {"update_onepass", 48.0 * n},  // x, p, q, r; writes x, r (+ the 2k column sums)
        // one-pass prolongation: W, s (+ A s: one more matrix pass), r; writes z
        {"prolong_onepass", 8.0 * n * k + (T ? pass + 24.0 * n : 16.0 * n)},
        // x/r update fused with the T = 2 sweeps: A, x, p, q, r, w; writes x, r', s
        {"update_sweep", pass + (args.wdc != 0.0 ? 56.0 : 64.0) * n},
        // ... fused with ALL T sweeps (lmarch.cuh): A, x, p, q, r; writes x, r', s_T
        {"update_sweeps_fused", pass + 56.0 * n},
        // lean cycle: A, p (gathered), x, r; writes x, r
        {"spmv_update", pass + 40.0 * n},
        // ... A, r (gathered), w; writes s
        {"sweep_lean", pass + (args.wdc != 0.0 ? 16.0 : 24.0) * n},
        // ... W, A (A s), s, r, p; writes p
        {"prolong_lean", 8.0 * n * k + pass + 32.0 * n},
        // ... all T sweeps in one line march: A, r; writes s_T
        {"sweeps_fused_lean", pass + 16.0 * n},
        // ... separate kernels at T > 2: the T - 1 launches together
        {"sweeps_lean", (double)(T > 1 ? T - 1 : 1) * pass + (args.wdc != 0.0 ? 16.0 : 24.0) * n +
                            (double)(T > 2 ? T - 2 : 0) * (args.wdc != 0.0 ? 24.0 : 32.0) * n},
    };
    if ((int)acc.size() != kSlots) return -1;
    std::vector<cudaEvent_t> evs(2);
    for (auto& e : evs) cudaEventCreate(&e);
    auto timed = [&](int slot, auto&& fn) {
        cudaEventRecord(evs[0], ctx->s);
        fn();
        cudaEventRecord(evs[1], ctx->s);
        cudaEventSynchronize(evs[1]);
        float t = 0.f;
        cudaEventElapsedTime(&t, evs[0], evs[1]);
        acc[slot].ms += t;
        acc[slot].launches++;
    };
    const bool folded = mode == 0 && m->folded;
    const bool simple_apply = mode == 0 && !folded && m->nu1 == 1 && m->nu2 == 1;
    const bool lean = mode == 0 && m->lean;
    for (uint64_t it = 0; it < iters; ++it) {
        if (lean) {
            timed(kSU, [&] { launch_spmv_upd(ctx->lc, args); });
            const double* sv = nullptr;
            const int slot = (T > 2 && lfused_pattern(args, T)) ? kSLF : (T == 2 ? kSL : kSL1);
            timed(slot, [&] { sv = launch_lean_sweeps(ctx->lc, args, T); });
            timed(kPL, [&] { launch_prolong_onepass(ctx->lc, args, sv, ctx->p0, 0, 1, 0, 1); });
            continue;
        }
        timed(kSpmvP, [&] { launch_spmv_p(ctx->lc, args); });
        bool fused = false;
        if (onepass && update_sweep_ok(args, T)) {
            cudaEventRecord(evs[0], ctx->s);
            fused = launch_lfused(ctx->lc, args, T, false);
            if (fused) {
                cudaEventRecord(evs[1], ctx->s);
                cudaEventSynchronize(evs[1]);
                float tf = 0.f;
                cudaEventElapsedTime(&tf, evs[0], evs[1]);
                acc[kUSF].ms += tf;
                acc[kUSF].launches++;
            }
        }
        if (fused) {
            timed(kPO, [&] { launch_prolong_onepass(ctx->lc, args, ctx->zt0, ctx->z, 0, 1, 1, 0); });
        } else if (onepass && update_sweep_ok(args, T)) {
            timed(kUS, [&] { launch_update_sweep(ctx->lc, args); });
            double* cur = ctx->zt0;
            for (unsigned long long j = 3; j <= T; ++j) {
                double* c1 = cur;
                timed(kSmooth, [&] { launch_sweeps_rpar(ctx->lc, args, 3, &c1); });  // one sweep
                cur = c1;
            }
            timed(kPO, [&] { launch_prolong_onepass(ctx->lc, args, cur, ctx->z, 0, 1, 1, 0); });
        } else if (onepass) {
            timed(kUO, [&] { launch_update_onepass(ctx->lc, args); });
            double* cur = nullptr;
            for (unsigned long long j = 2; j <= T; ++j) {
                double* nxt = (cur == ctx->zt0) ? ctx->zt1 : ctx->zt0;
                timed(kSmooth, [&] { launch_sweep(ctx->lc, args, cur == nullptr, cur, nxt, false); });
                cur = nxt;
            }
            timed(kPO, [&] { launch_prolong_onepass(ctx->lc, args, cur, ctx->z, 0, 1, 0, 0); });
        } else if (folded) {
            timed(kUR, [&] { launch_update_restrict(ctx->lc, args, true); });
            // launch_folded_tail, each launch timed on its own
            SolveArgs b = args;
            b.P = m->W2;
            if (T <= 1) {
                timed(kPro, [&] { launch_prolong(ctx->lc, b, T == 0 ? 0 : 1, true, nullptr, ctx->z, 0, 1); });
            } else {
                double* cur = nullptr;
                for (unsigned long long j = 2; j <= T; ++j) {
                    double* nxt = (cur == ctx->zt0) ? ctx->zt1 : ctx->zt0;
                    timed(kSmooth, [&] { launch_sweep(ctx->lc, args, cur == nullptr, cur, nxt, false); });
                    cur = nxt;
                }
                timed(kPro, [&] { launch_prolong(ctx->lc, b, 2, true, cur, ctx->z, 0, 1); });
            }
        } else {
            timed(kUpd, [&] { launch_update(ctx->lc, args, mode); });
            if (mode == 0) {
                if (simple_apply) {
                    timed(kRes, [&] { launch_restrict(ctx->lc, args, 1, nullptr); });
                    timed(kPro, [&] { launch_prolong(ctx->lc, args, 1, false, nullptr, ctx->zt0, 0, 0); });
                    timed(kPost, [&] { launch_sweep(ctx->lc, args, false, ctx->zt0, ctx->z, true); });
                } else {
                    timed(kRes, [&] { launch_twolevel_apply(ctx->lc, args, m->nu1, m->nu2); });
                }
            }
        }
        if (!folded) timed(kCtl, [&] { launch_loop_ctl(ctx->lc, ctx->st, cudaGraphConditionalHandle{}, 0); });
    }
    for (auto& e : evs) cudaEventDestroy(e);
    cudaStreamSynchronize(ctx->s);
    int w = 0;
    for (auto& x : acc) {
        if (!x.launches || w >= cap) continue;
        std::snprintf(stats[w].name, sizeof(stats[w].name), "%s", x.name);
        stats[w].launches = x.launches;
        stats[w].total_ms = x.ms;
        stats[w].bytes_per_launch = x.bytes;
        ++w;
    }
    return w;
}

}  // extern "C"

// ------------------------------------------------------- MLP inference (8f.4) --
struct nlsp_mlp {
    unsigned long long id;
    int device;
    std::vector<uint64_t> w;  // layer widths
    struct Off {
        size_t w, b, gain, offset;
    };
    std::vector<Off> off;
    double* params = nullptr;
    uint64_t np = 0;
};

nlsp_status nlsp_mlp_upload(nlsp_ctx* ctx, const uint64_t* widths, uint64_t nwidths, const double* params,
                            uint64_t nparams, nlsp_mlp** out) {
    if (!out) return set_err(ctx, NLSP_E_VALIDATION, "mlp: null out");
    *out = nullptr;
    nlsp_status st = bind(ctx);
    if (st) return st;
    if (!widths || !params || nwidths < 2)
        return set_err(ctx, NLSP_E_VALIDATION, "mlp: need at least input and output widths");
    auto* m = new nlsp_mlp();
    m->id = g_next_id++;
    m->device = ctx->device;
    m->w.assign(widths, widths + nwidths);
    size_t total = 0;
    for (size_t l = 0; l + 1 < m->w.size(); ++l) {
        if (m->w[l] == 0 || m->w[l + 1] == 0 || m->w[l] >= (1ull << 31) || m->w[l + 1] >= (1ull << 31)) {
            delete m;
            return set_err(ctx, NLSP_E_VALIDATION, "mlp: layer widths must be in [1, 2^31)");
        }
        nlsp_mlp::Off o{};
        o.w = total;
        total += m->w[l] * m->w[l + 1];
        o.b = total;
        total += m->w[l + 1];
        if (l + 2 < m->w.size()) {
            o.gain = total;
            total += m->w[l + 1];
            o.offset = total;
            total += m->w[l + 1];
        }
        m->off.push_back(o);
    }
    if (total != nparams) {
        delete m;
        return set_err(ctx, NLSP_E_VALIDATION, "mlp: parameter count does not match the widths");
    }
    m->np = nparams;
    cudaError_t e = dalloc(&m->params, nparams);
    if (!e) e = cudaMemcpyAsync(m->params, params, nparams * 8, cudaMemcpyHostToDevice, ctx->s);
    if (!e) e = cudaStreamSynchronize(ctx->s);
    if (e) {
        nlsp_mlp_destroy(m);
        return cuda_fail(ctx, e, "mlp upload");
    }
    *out = m;
    return NLSP_OK;
}

void nlsp_mlp_destroy(nlsp_mlp* m) {
    if (!m) return;
    cudaSetDevice(m->device);
    dfree(m->params);
    delete m;
}

// forward pass on device vectors; scratch from the context pool
static nlsp_status mlp_forward_dev(nlsp_ctx* ctx, const nlsp_mlp* m, const double* x, double* y) {
    uint64_t maxw = 0, maxs = 0;
    const size_t L = m->w.size() - 1;
    for (size_t l = 0; l < L; ++l) {
        const int fi = (int)m->w[l], fo = (int)m->w[l + 1];
        if (l + 1 < L) maxw = std::max<uint64_t>(maxw, fo);
        uint64_t sc = fo;
        if (fi > 4096) sc = (uint64_t)mlp_splitk_parts(ctx->lc, fi, fo) * fo;
        maxs = std::max(maxs, sc);
    }
    double *a = nullptr, *b = nullptr, *scr = nullptr;
    cudaError_t e;
    if ((e = salloc(ctx, &a, std::max<uint64_t>(maxw, 1))) || (e = salloc(ctx, &b, std::max<uint64_t>(maxw, 1))) ||
        (e = salloc(ctx, &scr, maxs))) {
        sfree(ctx, a);
        sfree(ctx, b);
        return cuda_fail(ctx, e, "mlp scratch");
    }
    const double* cur = x;
    for (size_t l = 0; l < L; ++l) {
        const bool hidden = l + 1 < L;
        double* dst = hidden ? ((cur == a) ? b : a) : y;
        const auto& o = m->off[l];
        launch_mlp_layer(ctx->lc, m->params + o.w, m->params + o.b, hidden ? m->params + o.gain : nullptr,
                         hidden ? m->params + o.offset : nullptr, (int)m->w[l], (int)m->w[l + 1], hidden, cur,
                         dst, scr);
        cur = dst;
    }
    sfree(ctx, a);
    sfree(ctx, b);
    sfree(ctx, scr);
    CU(cudaGetLastError());
    return NLSP_OK;
}

nlsp_status nlsp_mlp_forward(nlsp_ctx* ctx, const nlsp_mlp* m, const double* in, double* out) {
    nlsp_status st = bind(ctx);
    if (st) return st;
    if (!m || !in || !out) return set_err(ctx, NLSP_E_VALIDATION, "mlp forward: null argument");
    const uint64_t wi = m->w.front(), wo = m->w.back();
    double *x = nullptr, *y = nullptr;
    cudaError_t e;
    if ((e = salloc(ctx, &x, wi)) || (e = salloc(ctx, &y, wo))) {
        sfree(ctx, x);
        return cuda_fail(ctx, e, "mlp forward alloc");
    }
    CU(cudaMemcpyAsync(x, in, wi * 8, cudaMemcpyHostToDevice, ctx->s));
    st = mlp_forward_dev(ctx, m, x, y);
    if (!st) CU(cudaMemcpyAsync(out, y, wo * 8, cudaMemcpyDeviceToHost, ctx->s));
    sfree(ctx, x);
    sfree(ctx, y);
    CU(cudaStreamSynchronize(ctx->s));
    return st;
}

nlsp_status nlsp_mlp_infer_basis(nlsp_ctx* ctx, const nlsp_mlp* m, const nlsp_dense* s, nlsp_dense** q_out) {
    if (!q_out) return set_err(ctx, NLSP_E_VALIDATION, "infer_basis: null out");
    *q_out = nullptr;
    nlsp_status st = bind(ctx);
    if (st) return st;
    if (!m || !s) return set_err(ctx, NLSP_E_VALIDATION, "infer_basis: null argument");
    const uint64_t n = s->rows, K = s->cols;
    if (n * K != m->w.front()) return set_err(ctx, NLSP_E_VALIDATION, "mlp forward: width mismatch");
    const uint64_t r = m->w.back() / n;
    if (r * n != m->w.back()) return set_err(ctx, NLSP_E_VALIDATION, "reshape: length mismatch");
    if (n < r) return set_err(ctx, NLSP_E_VALIDATION, "orthonormalize: requires rows >= cols");
    if (r > 256) return set_err(ctx, NLSP_E_VALIDATION, "infer_basis: at most 256 basis columns");
    const int g = gram_grid(ctx->lc, (long long)n);
    const int nparts = ctx->num_sms * 2;
    const size_t rr = (size_t)r * r;
    double *part = nullptr, *x = nullptr, *raw = nullptr, *P = nullptr, *G = nullptr, *gp = nullptr,
           *Lf = nullptr, *U = nullptr, *Q1 = nullptr;
    auto cleanup = [&]() {
        for (double* p : {part, x, raw, P, G, gp, Lf, U, Q1}) sfree(ctx, p);
    };
    cudaError_t e;
    if ((e = salloc(ctx, &part, nparts)) || (e = salloc(ctx, &x, n * K)) || (e = salloc(ctx, &raw, n * r)) ||
        (e = salloc(ctx, &P, n * r)) || (e = salloc(ctx, &G, rr)) || (e = salloc(ctx, &gp, (size_t)g * gram_tile((int)r, (int)r))) ||
        (e = salloc(ctx, &Lf, rr)) || (e = salloc(ctx, &U, rr)) || (e = salloc(ctx, &Q1, n * r))) {
        cleanup();
        return cuda_fail(ctx, e, "infer_basis alloc");
    }
    CU(cudaMemsetAsync(ctx->flags, 0, 16 * sizeof(int), ctx->s));
    // x = vec(S / ||S||_F), forward, reshape (train.hpp:52-61)
    launch_mlp_input(ctx->lc, (int)n, (int)K, s->d, part, nparts, x, ctx->flags + 11);
    st = mlp_forward_dev(ctx, m, x, raw);
    if (st) {
        cleanup();
        return st;
    }
    launch_unflatten(ctx->lc, (int)n, (int)r, raw, P);
    // orthonormalize_differentiable (orthonormalize.hpp:25-59) as CholeskyQR2:
    // the first pass's pivots are MGS's post-elimination norms (absolute 1e-10 test)
    nlsp_dense* Q = nullptr;
    st = dense_alloc(ctx, n, r, &Q);
    if (st) {
        cleanup();
        return st;
    }
    launch_gram(ctx->lc, (long long)n, (int)r, (int)r, P, P, gp, G);
    launch_chol(ctx->lc, (int)r, G, Lf, -1e-10, ctx->flags + 12);
    launch_tri_inv_t(ctx->lc, (int)r, Lf, U);
    launch_dense_mm(ctx->lc, (long long)n, (int)r, (int)r, P, U, nullptr, Q1);
    launch_gram(ctx->lc, (long long)n, (int)r, (int)r, Q1, Q1, gp, G);
    launch_chol(ctx->lc, (int)r, G, Lf, 0.0, ctx->flags + 13);
    launch_tri_inv_t(ctx->lc, (int)r, Lf, U);
    launch_dense_mm(ctx->lc, (long long)n, (int)r, (int)r, Q1, U, nullptr, Q->d);
    e = cudaGetLastError();
    if (!e) e = cudaMemcpyAsync(ctx->flags_host, ctx->flags, 16 * sizeof(int), cudaMemcpyDeviceToHost, ctx->s);
    if (!e) e = cudaStreamSynchronize(ctx->s);
    cleanup();
    if (e) {
        nlsp_dense_destroy(Q);
        return cuda_fail(ctx, e, "infer_basis");
    }
    const int* f = ctx->flags_host;
    if (f[11]) {
        nlsp_dense_destroy(Q);
        return set_err(ctx, NLSP_E_VALIDATION, "infer_basis: zero vector set");
    }
    if (f[12] || f[13]) {
        nlsp_dense_destroy(Q);
        return set_err(ctx, NLSP_E_RANK_DEFICIENT, "orthonormalize: a column vanished after elimination");
    }
    *q_out = Q;
    return NLSP_OK;
}

// ------------------------------------------------- smoothed aggregation (8f.3) --
// aggregate_nodes (sa.hpp:18-76), restated on the host: the greedy passes are
// sequential by construction (each pass reads the ids it has just assigned).
static void sa_aggregate_host(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                              double theta, std::vector<uint64_t>& agg, uint64_t& nc) {
    const uint64_t kUnset = ~0ull;
    std::vector<double> diag(n, 0.0);
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t k = rp[i]; k < rp[i + 1]; ++k)
            if (ci[k] == i) {
                diag[i] = v[k];
                break;
            }
    std::vector<uint64_t> sstart(n + 1, 0), strong;
    strong.reserve(rp[n]);
    for (uint64_t i = 0; i < n; ++i) {
        sstart[i] = strong.size();
        for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const uint64_t j = ci[k];
            if (j == i) continue;
            if (std::abs(v[k]) >= theta * std::sqrt(std::abs(diag[i] * diag[j]))) strong.push_back(j);
        }
    }
    sstart[n] = strong.size();
    agg.assign(n, kUnset);
    uint64_t next = 0;
    for (uint64_t i = 0; i < n; ++i) {  // pass 1: seeds with untouched strong neighbourhoods
        if (agg[i] != kUnset || sstart[i] == sstart[i + 1]) continue;
        bool touched = false;
        for (uint64_t s2 = sstart[i]; s2 < sstart[i + 1]; ++s2)
            if (agg[strong[s2]] != kUnset) {
                touched = true;
                break;
            }
        if (touched) continue;
        agg[i] = next;
        for (uint64_t s2 = sstart[i]; s2 < sstart[i + 1]; ++s2) agg[strong[s2]] = next;
        ++next;
    }
    for (uint64_t i = 0; i < n; ++i) {  // pass 2: strongest neighbouring aggregate
        if (agg[i] != kUnset) continue;
        double best = -1.0;
        uint64_t best_agg = kUnset;
        for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const uint64_t j = ci[k];
            if (j == i || agg[j] == kUnset) continue;
            bool is_strong = false;
            for (uint64_t s2 = sstart[i]; s2 < sstart[i + 1]; ++s2)
                if (strong[s2] == j) {
                    is_strong = true;
                    break;
                }
            if (!is_strong) continue;
            if (std::abs(v[k]) > best) {
                best = std::abs(v[k]);
                best_agg = agg[j];
            }
        }
        if (best_agg != kUnset) agg[i] = best_agg;
    }
    for (uint64_t i = 0; i < n; ++i) {  // pass 3: the rest
        if (agg[i] != kUnset) continue;
        agg[i] = next;
        for (uint64_t s2 = sstart[i]; s2 < sstart[i + 1]; ++s2)
            if (agg[strong[s2]] == kUnset) agg[strong[s2]] = next;
        ++next;
    }
    nc = next;
}

nlsp_status nlsp_sa_aggregate(uint64_t n, uint64_t nnz, const uint64_t* row_ptr, const uint64_t* col_idx,
                              const double* values, double theta, uint64_t* agg, uint64_t* nc) {
    if (!row_ptr || !agg || !nc || (nnz && (!col_idx || !values))) return NLSP_E_VALIDATION;
    if (row_ptr[0] != 0 || row_ptr[n] != nnz) return NLSP_E_VALIDATION;
    std::vector<uint64_t> a;
    uint64_t c = 0;
    sa_aggregate_host(n, row_ptr, col_idx, values, theta, a, c);
    std::copy(a.begin(), a.end(), agg);
    *nc = c;
    return NLSP_OK;
}

nlsp_status nlsp_sa_prolongator(nlsp_ctx* ctx, uint64_t n, uint64_t nnz, const uint64_t* row_ptr,
                                const uint64_t* col_idx, const double* values, double theta, double omega,
                                nlsp_dense** p_out) {
    if (!p_out) return set_err(ctx, NLSP_E_VALIDATION, "sa_prolongator: null out");
    *p_out = nullptr;
    nlsp_status st = bind(ctx);
    if (st) return st;
    if (!row_ptr || (nnz && (!col_idx || !values)) || row_ptr[0] != 0 || row_ptr[n] != nnz)
        return set_err(ctx, NLSP_E_VALIDATION, "sa_prolongator: bad CSR arrays");
    if (n >= (1ull << 31) || nnz >= (1ull << 31))
        return set_err(ctx, NLSP_E_VALIDATION, "sa_prolongator: n and nnz must be < 2^31");
    for (uint64_t k = 0; k < nnz; ++k)
        if (col_idx[k] >= n) return set_err(ctx, NLSP_E_VALIDATION, "sa_prolongator: column index out of range");
    std::vector<uint64_t> agg;
    uint64_t nc = 0;
    sa_aggregate_host(n, row_ptr, col_idx, values, theta, agg, nc);
    if (nc == 0) return set_err(ctx, NLSP_E_NUMERIC, "sa_prolongator: no aggregates formed");
    // t_c = 1 / sqrt(|aggregate c|); A_ii > 0 (sa.hpp:84-99)
    std::vector<uint64_t> size(nc, 0);
    for (uint64_t i = 0; i < n; ++i) ++size[agg[i]];
    std::vector<double> tval(nc), diag(n, 0.0);
    for (uint64_t c = 0; c < nc; ++c) tval[c] = 1.0 / std::sqrt(static_cast<double>(size[c]));
    std::vector<int> rp32(n + 1), ci32(std::max<uint64_t>(nnz, 1)), agg32(n);
    for (uint64_t i = 0; i <= n; ++i) rp32[i] = (int)row_ptr[i];
    for (uint64_t k = 0; k < nnz; ++k) ci32[k] = (int)col_idx[k];
    for (uint64_t i = 0; i < n; ++i) {
        agg32[i] = (int)agg[i];
        for (uint64_t k = row_ptr[i]; k < row_ptr[i + 1]; ++k)
            if (col_idx[k] == i) {
                diag[i] = values[k];
                break;
            }
        if (diag[i] <= 0.0) return set_err(ctx, NLSP_E_NUMERIC, "sa_prolongator: non-positive diagonal");
    }
    nlsp_dense* P = nullptr;
    st = dense_alloc(ctx, n, nc, &P);
    if (st) return st;
    int *drp = nullptr, *dci = nullptr, *dagg = nullptr;
    double *dv = nullptr, *dt = nullptr, *dd = nullptr;
    auto cleanup = [&]() {
        sfree(ctx, drp);
        sfree(ctx, dci);
        sfree(ctx, dagg);
        sfree(ctx, dv);
        sfree(ctx, dt);
        sfree(ctx, dd);
    };
    cudaError_t e;
    if ((e = salloc(ctx, &drp, n + 1)) || (e = salloc(ctx, &dci, std::max<uint64_t>(nnz, 1))) ||
        (e = salloc(ctx, &dagg, n)) || (e = salloc(ctx, &dv, std::max<uint64_t>(nnz, 1))) ||
        (e = salloc(ctx, &dt, nc)) || (e = salloc(ctx, &dd, n)) ||
        (e = cudaMemcpyAsync(drp, rp32.data(), (n + 1) * 4, cudaMemcpyHostToDevice, ctx->s)) ||
        (nnz && (e = cudaMemcpyAsync(dci, ci32.data(), nnz * 4, cudaMemcpyHostToDevice, ctx->s))) ||
        (nnz && (e = cudaMemcpyAsync(dv, values, nnz * 8, cudaMemcpyHostToDevice, ctx->s))) ||
        (e = cudaMemcpyAsync(dagg, agg32.data(), n * 4, cudaMemcpyHostToDevice, ctx->s)) ||
        (e = cudaMemcpyAsync(dt, tval.data(), nc * 8, cudaMemcpyHostToDevice, ctx->s)) ||
        (e = cudaMemcpyAsync(dd, diag.data(), n * 8, cudaMemcpyHostToDevice, ctx->s)) ||
        (e = cudaMemsetAsync(P->d, 0, n * nc * 8, ctx->s))) {
        cleanup();
        nlsp_dense_destroy(P);
        return cuda_fail(ctx, e, "sa_prolongator upload");
    }
    launch_sa_assemble(ctx->lc, (int)n, (int)nc, drp, dci, dv, dagg, dt, dd, omega, P->d);
    e = cudaGetLastError();
    cleanup();
    if (!e) e = cudaStreamSynchronize(ctx->s);
    if (e) {
        nlsp_dense_destroy(P);
        return cuda_fail(ctx, e, "sa_prolongator");
    }
    *p_out = P;
    return NLSP_OK;
}

// ------------------------------------------------------------- batched solves --
// Many independent small systems in one launch: one single-cluster solver per
// system (the reference's harness runs its test instances through parallel_for,
// pipeline.hpp:356). Systems that do not fit a cluster are solved one by one.
nlsp_status nlsp_pcg_batch(nlsp_ctx* ctx, uint64_t count, const nlsp_csr* const* a,
                           const nlsp_twolevel* const* m, const double* const* b, double delta,
                           uint64_t max_iters, double* const* x, nlsp_solve_report* reps,
                           nlsp_status* statuses) {
    nlsp_status st = bind(ctx);
    if (st) return st;
    if (count == 0) return NLSP_OK;
    if (!a || !m || !b || !x) return set_err(ctx, NLSP_E_VALIDATION, "pcg_batch: null array");
    std::vector<int> in_batch, ns, ks, ws, rows;
    std::vector<char> tw;
    for (uint64_t i = 0; i < count; ++i) {
        if (!a[i] || !m[i] || !b[i] || !x[i]) return set_err(ctx, NLSP_E_VALIDATION, "pcg_batch: null system");
        st = check_pcg_args(ctx, a[i], NLSP_PRECOND_TWOLEVEL, m[i]);
        if (st) return st;
        int r = 0;
        size_t sm = 0;
        const bool fits = m[i]->folded && ctx->use_cluster && !a[i]->rp_host.empty() &&
                          cluster_plan(a[i]->n, m[i]->k, a[i]->max_row, m[i]->W2 != m[i]->W1, &r, &sm) > 0;
        if (fits) {
            in_batch.push_back((int)i);
            ns.push_back(a[i]->n);
            ks.push_back(m[i]->k);
            ws.push_back(a[i]->max_row);
            tw.push_back(m[i]->W2 != m[i]->W1);
        }
    }
    nlsp_status first = NLSP_OK;
    auto record = [&](uint64_t i, nlsp_status s_i) {
        if (statuses) statuses[i] = s_i;
        if (s_i && !first) first = s_i;
    };
    const int cnt = (int)in_batch.size();
    if (cnt) {
        rows.resize(cnt);
        size_t smem = 0;
        std::vector<bool> twb(tw.begin(), tw.end());
        std::unique_ptr<bool[]> twa(new bool[cnt]);
        for (int j = 0; j < cnt; ++j) twa[j] = twb[j];
        const int ncta = cluster_plan_batch(cnt, ns.data(), ks.data(), ws.data(), twa.get(), rows.data(), &smem);
        if (!ncta) return set_err(ctx, NLSP_E_VALIDATION, "pcg_batch: systems do not fit one cluster size");
        // per-system state, b, x in one pool allocation each (no residual
        // history: the batch reports iterations and the last residual only)
        std::vector<size_t> voff(cnt + 1, 0);
        for (int j = 0; j < cnt; ++j) voff[j + 1] = voff[j] + (size_t)ns[j] + 16;
        struct Scratch {
            nlsp_ctx* c;
            PcgState* dst = nullptr;
            double *db = nullptr, *dx = nullptr;
            ClusterArgs* dargs = nullptr;
            ~Scratch() {  // every return path gives the pool blocks back
                sfree(c, dst);
                sfree(c, db);
                sfree(c, dx);
                sfree(c, dargs);
            }
        } sc{ctx};
        PcgState*& dst = sc.dst;
        double*& db = sc.db;
        double*& dx = sc.dx;
        ClusterArgs*& dargs = sc.dargs;
        cudaError_t e;
        if ((e = salloc(ctx, &dst, cnt)) || (e = salloc(ctx, &db, voff[cnt])) || (e = salloc(ctx, &dx, voff[cnt])) ||
            (e = salloc(ctx, &dargs, cnt)))
            return cuda_fail(ctx, e, "pcg_batch alloc");
        // a system that fails before its loop (zero rhs) leaves x = 0, not pool garbage
        CU(cudaMemsetAsync(dx, 0, sizeof(double) * voff[cnt], ctx->s));
        std::vector<ClusterArgs> args(cnt);
        CU(cudaEventRecord(ctx->ev2, ctx->s));
        for (int j = 0; j < cnt; ++j) {
            const uint64_t i = in_batch[j];
            const nlsp_csr* A = a[i];
            const nlsp_twolevel* M = m[i];
            CU(cudaMemcpyAsync(db + voff[j], b[i], (size_t)A->n * 8, cudaMemcpyHostToDevice, ctx->s));
            launch_state_init(ctx->lc, dst + j, delta,
                              (long long)std::min<uint64_t>(max_iters, (uint64_t)LLONG_MAX));
            const SolveArgs sa = make_args(ctx, A, M);
            args[j] = ClusterArgs{A->n, M->k, M->ld, rows[j], (int)M->nu1, (int)M->nu2, A->max_row, A->rp, A->ci, A->v,
                                  M->wd, M->W1, M->W2, M->L, sa.Ainv, db + voff[j], dx + voff[j],
                                  nullptr, 0, dst + j};
        }
        CU(cudaMemcpyAsync(dargs, args.data(), sizeof(ClusterArgs) * cnt, cudaMemcpyHostToDevice, ctx->s));
        CU(cudaEventRecord(ctx->ev0, ctx->s));
        e = launch_cluster_pcg_batch(ctx->s, dargs, cnt, ncta, smem);
        if (e) return cuda_fail(ctx, e, "pcg_batch launch");
        ctx->launches += 1 + cnt;
        CU(cudaEventRecord(ctx->ev1, ctx->s));
        std::vector<PcgState> hs(cnt);
        CU(cudaMemcpyAsync(hs.data(), dst, sizeof(PcgState) * cnt, cudaMemcpyDeviceToHost, ctx->s));
        for (int j = 0; j < cnt; ++j)
            CU(cudaMemcpyAsync(x[in_batch[j]], dx + voff[j], (size_t)ns[j] * 8, cudaMemcpyDeviceToHost, ctx->s));
        CU(cudaEventRecord(ctx->ev3, ctx->s));
        CU(cudaStreamSynchronize(ctx->s));
        float ms = 0.f, tot = 0.f;
        cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1);
        cudaEventElapsedTime(&tot, ctx->ev2, ctx->ev3);
        for (int j = 0; j < cnt; ++j) {
            const uint64_t i = in_batch[j];
            const PcgState& p = hs[j];
            if (reps) {
                nlsp_solve_report& r = reps[i];
                std::memset(&r, 0, sizeof(r));
                r.iterations = (uint64_t)p.iterations;
                r.converged = p.converged;
                r.precond_kind = NLSP_PRECOND_TWOLEVEL;
                r.true_relative_residual = p.true_res;
                r.final_relative_residual = p.last_rel;
                r.solve_ms = ms;  // the batch's device time
                r.total_ms = tot;
                r.coarse_dim = (uint64_t)m[i]->k;
                r.kernel_launches = 1;
                r.h2d_bytes = (uint64_t)ns[j] * 8;
                r.d2h_bytes = (uint64_t)ns[j] * 8 + sizeof(PcgState);
            }
            record(i, p.error == kErrNotSpd ? NLSP_E_NOT_SPD : (p.error ? NLSP_E_VALIDATION : NLSP_OK));
        }
    }
    // the rest one by one on the general path
    for (uint64_t i = 0; i < count; ++i) {
        if (std::find(in_batch.begin(), in_batch.end(), (int)i) != in_batch.end()) continue;
        nlsp_solve_report local{};
        const nlsp_status s_i = nlsp_pcg(ctx, a[i], NLSP_PRECOND_TWOLEVEL, m[i], b[i], delta, max_iters, x[i],
                                         reps ? &reps[i] : &local, nullptr);
        record(i, s_i);
    }
    if (first) return set_err(ctx, first, "pcg_batch: at least one system failed (see statuses)");
    return NLSP_OK;
}
