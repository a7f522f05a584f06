/* include/nlsp_gpu.h — C-ABI of the B200 (sm_100a) two-level PCG library
 * (paper_2601_20174_b200/libnlsp_gpu.so).
 *
 * This is the drop-in boundary for the reference's solver/preconditioner
 * interface (/root/reference/proj/include/nlsp/, header-only C++). Every entry
 * point names the reference symbol it replaces. Plain pointers and sizes only;
 * host pointers are borrowed for the duration of the call, device buffers are
 * owned by the opaque handles. One context per host thread; handles other than
 * the context are immutable after creation and may be shared read-only between
 * contexts on the same device (the reference: objects immutable after
 * construction).
 *
 * Errors: the reference throws (errors.hpp:10-49); here every call returns an
 * nlsp_status and leaves a message in nlsp_last_error(ctx). include/nlsp_gpu.hpp
 * maps the codes back onto the nlsp:: exception types.
 *
 * There is no CPU fallback: without a usable sm_100 device every compute entry
 * point returns NLSP_E_CUDA.
 */
#ifndef NLSP_GPU_H
#define NLSP_GPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    NLSP_OK = 0,
    NLSP_E_VALIDATION = 1,     /* nlsp::ValidationError (CLI exit 1)           */
    NLSP_E_NUMERIC = 2,        /* nlsp::NumericError                           */
    NLSP_E_NOT_SPD = 3,        /* nlsp::NotSpdError                            */
    NLSP_E_RANK_DEFICIENT = 4, /* nlsp::RankDeficiencyError                    */
    NLSP_E_CONVERGENCE = 5,    /* nlsp::ConvergenceError                       */
    NLSP_E_CUDA = 6,           /* device missing / CUDA failure                */
    NLSP_E_OOM = 7             /* device allocation failed                     */
} nlsp_status;

typedef enum {
    NLSP_PRECOND_IDENTITY = 0, /* IdentityPreconditioner, two_level.hpp:103-106 */
    NLSP_PRECOND_JACOBI = 1,   /* JacobiPreconditioner, two_level.hpp:107-118   */
    NLSP_PRECOND_TWOLEVEL = 2  /* TwoLevelPreconditioner, two_level.hpp:22-89   */
} nlsp_precond_kind;

typedef struct nlsp_ctx nlsp_ctx;
typedef struct nlsp_csr nlsp_csr;
typedef struct nlsp_dense nlsp_dense;
typedef struct nlsp_twolevel nlsp_twolevel;

/* Mirrors SolveReport (two_level.hpp:121-132); the residual history is
 * returned through the separate residual_history argument of nlsp_pcg. */
typedef struct {
    uint64_t iterations;           /* completed x/r updates                          */
    int32_t converged;             /* recurrence ||r||/||b|| < delta reached         */
    int32_t precond_kind;          /* nlsp_precond_kind                              */
    double true_relative_residual; /* ||b - A x|| / ||b|| recomputed at exit         */
    double final_relative_residual;/* last recurrence entry (history back())         */
    double solve_ms;               /* device time of the solve (CUDA events)         */
    double total_ms;               /* solve incl. host<->device copies of b, x      */
    uint64_t coarse_dim;           /* k for the two-level preconditioner, else 0     */
    uint64_t kernel_launches;      /* this library's kernels launched by the solve   */
    uint64_t h2d_bytes;            /* host->device bytes copied by the call          */
    uint64_t d2h_bytes;            /* device->host bytes copied by the call          */
    double onepass_drift;          /* one-pass cycle guard: max over the solve of
                                      |c_rec - W^T r|_inf / |W^T r|_inf, the restriction's
                                      recurrence against its direct value; on
                                      the lean cycle the larger of that and
                                      |p.Ap predicted - direct| / direct               */
    int32_t cycle_fallback;        /* 1: the drift passed NLSP_DRIFT_TOL (default 1e-10)
                                      and the solve was re-run on the folded cycle        */
    int32_t reserved;
} nlsp_solve_report;

/* ------------------------------------------------------------ context ---- */
nlsp_status nlsp_ctx_create(int device, nlsp_ctx** out);
void nlsp_ctx_destroy(nlsp_ctx* ctx);
const char* nlsp_last_error(const nlsp_ctx* ctx);
/* the cudaStream_t every call of this context is ordered on */
void* nlsp_ctx_stream(nlsp_ctx* ctx);
nlsp_status nlsp_ctx_synchronize(nlsp_ctx* ctx);
const char* nlsp_version(void);
/* number of kernels this library has launched on ctx since creation */
uint64_t nlsp_ctx_kernel_launches(const nlsp_ctx* ctx);

/* ---------------------------------------------------------------- CSR ---- */
/* SparseCsrMatrix (sparse.hpp:19-113): size_t row_ptr/col_idx, fp64 values;
 * columns sorted, no duplicates. Stored on the device with int32 indices;
 * NLSP_E_VALIDATION for nnz >= 2^31, n >= 2^31, or a violated invariant. */
nlsp_status nlsp_csr_upload(nlsp_ctx* ctx, uint64_t n, uint64_t nnz, const uint64_t* row_ptr,
                            const uint64_t* col_idx, const double* values, nlsp_csr** out);
void nlsp_csr_destroy(nlsp_csr* a);
void nlsp_csr_dims(const nlsp_csr* a, uint64_t* n, uint64_t* nnz);

/* The device form the solve kernels stream (no reference
 * counterpart): kind 0 = CSR; 1 = diagonal form with one value per offset
 * (constant-coefficient stencil: per-row presence bits only); 2 = diagonal
 * form with per-row values; 3 = CSR rows with implicit columns (a banded
 * matrix with too many absent offsets for kind 2: row_ptr and values as they
 * are, one 32-bit presence mask per row in place of the column indices).
 * `offsets` = number of distinct column offsets (kinds 1, 2, 3), `pass_bytes`
 * = matrix bytes one SpMV pass of the PCG loop reads (the byte model of the
 * roofline). Detected at nlsp_csr_upload; NLSP_DIA=0 keeps CSR; kind 3 is
 * opt-in (NLSP_PACK=1: measured slower than explicit columns).
 * Results are bitwise those of the CSR kernels (same per-row fma order). */
nlsp_status nlsp_csr_format(const nlsp_csr* a, int* kind, int* offsets, uint64_t* pass_bytes);
/* The structured-grid geometry of the diagonal form (no reference
 * counterpart): every offset is dz * plane + d with dz in {-1, 0, 1},
 * |d| <= halo (plane = 0: none). march = 1 when the PCG loop's gather kernels
 * run as plane marches on ctx's device (march.cuh; NLSP_MARCH=0
 * disables, =1 forces for any n). */
nlsp_status nlsp_csr_geometry(nlsp_ctx* ctx, const nlsp_csr* a, uint64_t* plane, int* halo, int* march);
/* spmv (sparse.hpp:116-128), y = A x; host buffers of length n */
nlsp_status nlsp_spmv(nlsp_ctx* ctx, const nlsp_csr* a, const double* x, double* y);
/* device-buffer variant (x, y device pointers of length n) */
nlsp_status nlsp_spmv_device(nlsp_ctx* ctx, const nlsp_csr* a, const double* x, double* y);
/* diagonal() (sparse.hpp:74-78), host buffer of length n */
nlsp_status nlsp_csr_diagonal(nlsp_ctx* ctx, const nlsp_csr* a, double* d);

/* -------------------------------------------------------------- dense ---- */
/* DenseMatrix (dense.hpp:17-50): row-major fp64 */
nlsp_status nlsp_dense_upload(nlsp_ctx* ctx, uint64_t rows, uint64_t cols, const double* host,
                              nlsp_dense** out);
nlsp_status nlsp_dense_export(nlsp_ctx* ctx, const nlsp_dense* d, double* host);
void nlsp_dense_dims(const nlsp_dense* d, uint64_t* rows, uint64_t* cols);
void nlsp_dense_destroy(nlsp_dense* d);
/* device address of the row-major data (for the *_device entry points) */
void* nlsp_dense_data(const nlsp_dense* d);

/* ----------------------------------------------------------- smoothing ---- */
/* `sweeps` weighted-Jacobi sweeps x <- x + w D^-1 (b - A x)
 * (JacobiSmoother::sweep, smoothing.hpp:34-41); x in/out, b host, length n. */
nlsp_status nlsp_jacobi_sweeps(nlsp_ctx* ctx, const nlsp_csr* a, double omega, uint64_t sweeps,
                               double* x, const double* b);
/* homogeneous block sweeps on s in place (smoothing.hpp:50-60) */
nlsp_status nlsp_smooth_vectors(nlsp_ctx* ctx, const nlsp_csr* a, nlsp_dense* s, uint64_t sweeps,
                                double omega);
/* generate_smoothed_vectors (smoothing.hpp:81-100): S^(0) drawn from the
 * reference's Rng stream (rng.hpp:22-49), then swept on the device. mask may be
 * NULL (no Dirichlet rows). Where S^(0) is drawn is a context setting:
 *   NLSP_S0_DRAW_HOST (default): on the host cores, every thread jumping its own
 *     mt19937_64 generator to its slice of the one stream, glibc's log / sin /
 *     cos — bit-identical to the reference's serial loop; streamed to the device
 *     through pinned chunks.
 *   NLSP_S0_DRAW_DEVICE: on the device. The mt19937_64 words are the same bit
 *     for bit (jump-ahead, csrc/s0_device.cu); the Box-Muller transform uses
 *     CUDA's log / sincos, so a normal can differ from the reference's in its
 *     last bits (<= 4 ulp) — no host draw, no 8 n k byte upload.
 * The environment variable NLSP_S0_DRAW=device selects the device draw for
 * contexts created afterwards. */
enum { NLSP_S0_DRAW_HOST = 0, NLSP_S0_DRAW_DEVICE = 1 };
nlsp_status nlsp_ctx_set_s0_draw(nlsp_ctx* ctx, int32_t mode);
/* where the last nlsp_generate_smoothed_vectors of this context drew S^(0)
 * (the device draw hands over to the host when the stream holds a zero
 * uniform, which the reference redraws: probability 2^-53 per pair) */
int32_t nlsp_ctx_last_s0_draw(const nlsp_ctx* ctx);
nlsp_status nlsp_generate_smoothed_vectors(nlsp_ctx* ctx, const nlsp_csr* a, const uint8_t* mask,
                                           uint64_t k, uint64_t sweeps, double omega,
                                           uint64_t seed, nlsp_dense** out);
/* the first `count` outputs of std::mt19937_64(seed), generated on the device
 * by the jump tree of the device draw (a check of its integer part: they are
 * bit for bit the host generator's) */
nlsp_status nlsp_mt19937_64_words(nlsp_ctx* ctx, uint64_t seed, uint64_t count, uint64_t* out);

/* ----------------------------------------------------------- SVD basis ---- */
/* first_cols(svd_oracle(S).left_vectors, k) (svd.hpp:155-227, dense.hpp:158-164)
 * for a tall S (rows >= cols): Gram S^T S, Jacobi eigensolve, U_k = S V_k / sigma_k,
 * largest-|entry|-nonnegative sign convention. sigma (length cols) and
 * eigh_sweeps may be NULL. */
nlsp_status nlsp_svd_basis(nlsp_ctx* ctx, const nlsp_dense* s, uint64_t k, nlsp_dense** p_out,
                           double* sigma, int32_t* eigh_sweeps);

/* --------------------------------------------------- two-level operator ---- */
/* TwoLevelPreconditioner(a, basis_any, omega, nu1, nu2) (two_level.hpp:24-53):
 * orthonormalise the basis (CholeskyQR2 in place of qr_thin's MGS), form the
 * Galerkin operator P^T A P, symmetrise exactly, Cholesky-factor it. */
nlsp_status nlsp_twolevel_build(nlsp_ctx* ctx, const nlsp_csr* a, const nlsp_dense* basis,
                                double omega, uint64_t nu1, uint64_t nu2, nlsp_twolevel** out);
void nlsp_twolevel_destroy(nlsp_twolevel* m);
void nlsp_twolevel_dims(const nlsp_twolevel* m, uint64_t* n, uint64_t* k);
/* The schedule nlsp_pcg runs this operator with (same operator,
 * different pass structure): 0 literal (two_level.hpp:60-81 op by op), 1 folded
 * (W1 = G^nu1 P, W2 = G^nu2 P streamed twice per iteration), 2 one-pass (nu1 ==
 * nu2, k <= 64: W streamed once per iteration, the restriction by its
 * recurrence), 3 lean one-pass (nu1 == nu2 >= 1: beta known before and alpha
 * right after the pass, q = A p never stored; the default where it applies).
 * NLSP_CYCLE=literal|folded|onepass selects the first three. */
int nlsp_twolevel_cycle(const nlsp_twolevel* m);
/* basis_ (n x k), Cholesky factor L (k x k, lower), A_c (k x k); any may be NULL */
nlsp_status nlsp_twolevel_export(nlsp_ctx* ctx, const nlsp_twolevel* m, double* basis,
                                 double* chol, double* coarse);
/* apply (two_level.hpp:60-81): z = M^-1 r, host buffers of length n */
nlsp_status nlsp_twolevel_apply(nlsp_ctx* ctx, const nlsp_twolevel* m, const nlsp_csr* a,
                                const double* r, double* z);

/* ------------------------------------------------------------------ PCG ---- */
/* pcg<Preconditioner> (two_level.hpp:141-191) with x0 = 0. m must be non-NULL
 * for NLSP_PRECOND_TWOLEVEL and is ignored otherwise. b, x host buffers of
 * length n. The whole iteration loop runs on the device; max_iters may be any
 * value (SIZE_MAX: no limit). The device keeps the residual history in
 * segments of at most 2^20 entries (a longer solve pauses at each segment end
 * to move it to the host), so no buffer is sized by max_iters. Read the history
 * after the call with nlsp_pcg_history; residual_history (may be NULL) is the
 * one-shot form: it receives rep->iterations entries, so it must hold as many
 * as the solve may run. */
nlsp_status nlsp_pcg(nlsp_ctx* ctx, const nlsp_csr* a, int kind, const nlsp_twolevel* m,
                     const double* b, double delta, uint64_t max_iters, double* x,
                     nlsp_solve_report* rep, double* residual_history);
/* device-resident variant: b, x device pointers (length n); residual_history is
 * a HOST pointer (may be NULL). */
nlsp_status nlsp_pcg_device(nlsp_ctx* ctx, const nlsp_csr* a, int kind, const nlsp_twolevel* m,
                            const double* b_dev, double delta, uint64_t max_iters, double* x_dev,
                            nlsp_solve_report* rep, double* residual_history);
/* SolveReport::residual_history (two_level.hpp:123, one ||r_k||/||b|| per
 * iteration) of the last nlsp_pcg / nlsp_pcg_device call on ctx: *count = its
 * length (= that call's rep->iterations), and min(cap, *count) entries are
 * copied to the host buffer out (out may be NULL to query the length). Valid
 * until the next solve on ctx. */
nlsp_status nlsp_pcg_history(nlsp_ctx* ctx, double* out, uint64_t cap, uint64_t* count);

/* ------------------------------------------------------------ profiling ---- */
/* Runs `iters` PCG iterations kernel by kernel (no graph) on device-resident b
 * and records CUDA events around every launch. Fills, for up to `cap` kernel
 * kinds, the name, the number of launches and the summed device ms. Returns the
 * number of kinds written. */
typedef struct {
    char name[32];
    uint64_t launches;
    double total_ms;
    double bytes_per_launch; /* algorithmic bytes (DESIGN.md byte model) */
} nlsp_kernel_stat;
int nlsp_pcg_profile(nlsp_ctx* ctx, const nlsp_csr* a, int kind, const nlsp_twolevel* m,
                     const double* b_dev, uint64_t iters, nlsp_kernel_stat* stats, int cap);

/* ---- many small systems at once ------------------------------------------ */
/* count independent two-level PCG solves (the reference's harness runs its
 * test instances through parallel_for, pipeline.hpp:356) in ONE launch: one
 * single-cluster solver per system that fits one (n <= 65536, k <= 256,
 * folded cycle), the others one by one through nlsp_pcg. Host b[i], x[i];
 * reps[i] / statuses[i] per system (either may be NULL). Returns the first
 * failing status (NOT_SPD, VALIDATION for a zero right-hand side), else OK. */
nlsp_status nlsp_pcg_batch(nlsp_ctx* ctx, uint64_t count, const nlsp_csr* const* a,
                           const nlsp_twolevel* const* m, const double* const* b, double delta,
                           uint64_t max_iters, double* const* x, nlsp_solve_report* reps,
                           nlsp_status* statuses);

/* ---- smoothed aggregation: the SA coarse space ------------ */
/* aggregate_nodes(a, theta) (sa.hpp:18-76) on the host CSR (reference
 * layout): one aggregate id per node and their count. Needs no device. */
nlsp_status nlsp_sa_aggregate(uint64_t n, uint64_t nnz, const uint64_t* row_ptr, const uint64_t* col_idx,
                              const double* values, double theta, uint64_t* agg, uint64_t* nc);

/* sa_prolongator(a, theta, omega) (sa.hpp:78-109): P = (I - omega D^-1 A) T,
 * dense n x n_c on the device (T the normalised aggregate indicator). The
 * aggregation runs on the host, the assembly on the device. NUMERIC for a
 * non-positive diagonal or no aggregates. Feed P to nlsp_twolevel_build
 * (coarse dimensions up to 2048). */
nlsp_status nlsp_sa_prolongator(nlsp_ctx* ctx, uint64_t n, uint64_t nnz, const uint64_t* row_ptr,
                                const uint64_t* col_idx, const double* values, double theta, double omega,
                                nlsp_dense** p_out);

/* ---- NLSS basis: MLP inference --------------------------- */
typedef struct nlsp_mlp nlsp_mlp;

/* MlpModel (mlp.hpp:47-320) on the device from its widths and flat parameter
 * buffer in the reference's layout (nlsp_io_mlp_load / nlsp_io_mlp_init,
 * include/nlsp_io.h). VALIDATION on fewer than 2 widths or a count mismatch. */
nlsp_status nlsp_mlp_upload(nlsp_ctx* ctx, const uint64_t* widths, uint64_t nwidths,
                            const double* params, uint64_t nparams, nlsp_mlp** out);
void nlsp_mlp_destroy(nlsp_mlp* m);

/* MlpModel::forward (mlp.hpp:113-161): host vectors of the input / output
 * width; hidden layers Linear -> LayerNorm(gain, offset) -> GELU. */
nlsp_status nlsp_mlp_forward(nlsp_ctx* ctx, const nlsp_mlp* m, const double* in, double* out);

/* infer_basis(model, S) (train.hpp:52-62): Q (n x r, r = output width / n) =
 * orthonormalize(reshape_column_major(forward(vec_colmajor(S / ||S||_F)))).
 * The orthonormalisation is CholeskyQR2 (same Q as the reference's two-pass
 * MGS up to rounding); RANK_DEFICIENT when a column's post-elimination norm
 * falls below 1e-10 (orthonormalize.hpp:52-54), VALIDATION on width mismatch
 * or ||S||_F = 0. */
nlsp_status nlsp_mlp_infer_basis(nlsp_ctx* ctx, const nlsp_mlp* m, const nlsp_dense* s,
                                 nlsp_dense** q_out);

#ifdef __cplusplus
}
#endif
#endif
