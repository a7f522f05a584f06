// paper_2601_20174_b200/csrc/internal.cuh — shared internals of libnlsp_gpu.so.
//
// Layout in HBM:
//   CSR A      int32 row_ptr[n+1], int32 col_idx[nnz], fp64 values[nnz]  (12 B/nnz)
//   basis P    fp64 n x k row-major, leading dimension k (even k keeps 16-B rows)
//   vectors    fp64 n each: x, r, q, z, p[2] (ping-pong), zt[2] (sweep temps), b
//   state      one PcgState (scalars + flags) + per-CTA reduction partials
#pragma once

#include <cstdio>

#include <cuda_runtime.h>

#include <cstdint>

namespace nlsp {

constexpr int kThreads = 256;      // CTA size of the row kernels
constexpr int kGroup = 8;          // lanes per CSR row / basis row
constexpr int kRowsPerWarp = 32 / kGroup;
constexpr int kMaxGrid = 148 * 8;  // upper bound on row-kernel grids (partials sizing)
constexpr int kMaxCoarse = 2048;   // largest supported coarse dimension k
constexpr int kWideK = 256;        // k above this: the wide restriction / prolongation kernels
constexpr int kWideGrid = 144;     // CTAs of the wide restriction (partials: grid * (k + 1))
// c = W1^T r of the wide path lives at the tail of the partials buffer
constexpr long long kWideCOffset = (long long)kMaxGrid * 256 - (kMaxCoarse + 8);
// one-pass cycle: coarse dimensions it runs at (8-lane register tiles, PPL <= 4)
constexpr int kOnePassK = 64;

enum DevError : int {
    kErrNone = 0,
    kErrValidation = 1,
    kErrNumeric = 2,
    kErrNotSpd = 3,
    kErrRank = 4,
    kErrConvergence = 5,
};

// Device-resident PCG scalars (two_level.hpp:141-191 locals).
struct PcgState {
    double rz, rz_new, pap, alpha, beta, rr, bnorm, delta, true_res, last_rel;
    long long it, max_it, iterations, body_runs;
    long long hist_base;       // iteration of hist[0]: the history is kept in segments (nlsp_gpu.cu run_pcg)
    int done, converged, error, first;
    unsigned int counter[16];  // last-CTA tickets, one slot per kernel kind
    int op_grid;               // CTAs of the last one-pass prolongation (its partials' stride)
    double alpha_prev;         // alpha of the previous iteration (one-pass restriction)
    double drift_max;          // max over the solve of |c_rec - W^T r| / |W^T r| (one-pass guard)
    // lean one-pass cycle (solve_kernels.cu): c.e and e.Me of the
    // current coarse correction, the p.Ap predicted after the pass over W, and
    // the max over the solve of |predicted - direct| / direct (its guard)
    double lean_ce, lean_eme, pap_pred, pap_drift;
};

// Ticket slots (each kernel kind reuses its own counter; counters return to 0).
enum Ticket : int {
    kTkBnorm = 0, kTkSpmvP, kTkUpdate, kTkSweep, kTkRestrict, kTkProlong, kTkTrue,
    kTkInit, kTkGeneric
};

// Diagonal (offset) form of A, detected at upload (nlsp_gpu.cu):
// when the CSR columns of every row sit at one of d <= 32 fixed offsets from
// the row, A is stored as per-row presence bits over the sorted offsets plus
// either one value per offset (kind 1, every entry on an offset bitwise equal:
// constant-coefficient stencils) or a column-major value slab vals[t n + i]
// (kind 2). Row sums run over the present offsets in ascending order = the
// CSR column order, so results are bitwise those of the CSR kernels.
constexpr int kMaxDia = 32;
struct DiaArgs {
    int kind;   // 0: CSR only, 1: constant values, 2: per-row values
    int d;      // number of offsets
    int mbytes; // presence-mask bytes per row: 1, 2 or 4
    int off[kMaxDia];
    double val[kMaxDia];
    const void* mask;  // n presence masks (bit t: offset t present)
    const double* rv;  // kind 2: d x n values (0 where absent)
    // structured grid (march.cuh): every offset is dz * plane + d, dz in
    // {-1, 0, 1}, |d| <= halo, n % plane == 0; plane == 0: none detected
    long long plane;
    int halo;
};

// Implicit-column form of a CSR matrix (nlsp_gpu.cu detect_dia): a banded
// matrix whose stored entries sit at d <= 32 fixed offsets from the row, but
// with varying values and too many absent offsets for the value slab of the
// diagonal form to pay (C5: 13 of 21 offsets stored per row). The CSR row_ptr
// and values stay as they are; the column indices (4 B per nonzero) are
// replaced by one 32-bit presence mask per row: the j-th stored entry of row i
// is at column i + off[t_j], t_j the j-th set bit. Same entries in the same
// order, so every row sum is bitwise the CSR one. mask == nullptr: not in use.
struct PackArgs {
    int d;
    int off[kMaxDia];
    const unsigned* mask;
};

// Everything a solve kernel needs, passed by value.
struct SolveArgs {
    int n;
    const int* rp;
    const int* ci;
    const double* v;
    const double* wd;    // omega * (1 / A_ii)    (two-level smoother)
    double wdc;          // wd when it is one constant (constant-coefficient diagonal form), else 0
    const double* diag;  // A_ii                   (Jacobi preconditioner)
    const double* P;     // basis, n x k row-major, ld = k
    const double* L;     // Cholesky factor of A_c, k x k row-major
    const double* Ainv;  // A_c^-1 = L^-T L^-1 (k x k), or null: triangular solves
    const double* W1;    // (I - w D^-1 A)^nu1 P, n x ld (restriction basis)
    const double* W2;    // (I - w D^-1 A)^nu2 P, n x ld (prolongation basis; may alias W1)
    int k;
    int tile_nnz64;   // max nonzeros in any run of 64 / 128 consecutive rows
    int tile_nnz128;  // (stage sizes of the TMA-staged kernels)
    int tile_nnz256;
    int max_row;      // longest CSR row
    double* x;
    double* r;
    double* r1;          // second residual buffer (fused update + sweep, by iteration parity)
    double* q;
    double* z;
    double* p0;
    double* p1;
    double* zt0;
    double* zt1;
    const double* b;
    double* hist;        // device residual history segment: entry it - st->hist_base
    PcgState* st;
    double* partials;    // kMaxGrid * max(k, 4)
    double* e;           // coarse correction, k
    // one-pass cycle (solve_kernels.cu): M = W^T A W (k x k),
    // ow = [u_even | u_odd | v | c | M e] column sums (5 ld; c = the last
    // recurrence value, for the drift guard; M e: lean cycle), opart = per-CTA
    // partials of [u | v], column-major
    const double* M;
    double* ow;
    double* opart;
    DiaArgs dia;         // diagonal form of A (dia.kind == 0: CSR kernels)
    PackArgs pk;         // implicit-column form of the CSR arrays (pk.mask == nullptr: explicit columns)
};

constexpr int kColsignPerSm = 8;  // CTAs per SM of the column-sign scan

// The single-cluster solver (cluster_solve.cu): one CTA per row block.
struct ClusterArgs {
    int n, k, ld, rows;  // rows per CTA
    int nu1, nu2;
    int width;           // ELL width = longest row
    const int* rp;
    const int* ci;
    const double* v;
    const double* wd;
    const double* W1;
    const double* W2;    // may equal W1
    const double* L;
    const double* Ainv;  // A_c^-1 or null
    const double* b;
    double* x;           // out
    double* hist;        // residual history (may be null: batched solves keep none)
    long long hist_cap;  // entries hist holds; later iterations are not recorded
    PcgState* st;
};

// Checked builds (make -C paper_2601_20174_b200 checked -> variants/
// libnlsp_gpu_checked.so, scripts/gpu_checked.sh): device-side bounds checks on
// every staged copy and shared-memory window, in place of compute-sanitizer
// (closed on this pool). A failed check prints its site and traps, so the call
// returns a CUDA error and the test fails. Compiled out otherwise.
#ifdef NLSP_CHECKED
#define NLSP_CHECK(cond)                                                                             \
    do {                                                                                             \
        if (!(cond)) {                                                                               \
            printf("NLSP_CHECK failed: %s (%s:%d) block %d thread %d\n", #cond, __FILE__, __LINE__, \
                   (int)blockIdx.x, (int)threadIdx.x);                                               \
            __trap();                                                                                \
        }                                                                                            \
    } while (0)
#else
#define NLSP_CHECK(cond) \
    do {                 \
    } while (0)
#endif

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ double group_sum(double v) {
    v += __shfl_xor_sync(0xffffffffu, v, 4);
    v += __shfl_xor_sync(0xffffffffu, v, 2);
    v += __shfl_xor_sync(0xffffffffu, v, 1);
    return v;
}

// Programmatic dependent launch: wait until the preceding grid has completed
// and its memory is visible (a no-op without PDL), then let the next grid be
// scheduled. Called first thing by every kernel that may be launched with
// LaunchCtx::pdl.
__device__ __forceinline__ void pdl_entry() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// Streaming 16-B load that does not allocate in L1 (basis rows, CSR arrays).
__device__ __forceinline__ double2 ld_stream2(const double* p) {
    double2 r;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
                 : "=d"(r.x), "=d"(r.y)
                 : "l"(p));
    return r;
}

}  // namespace nlsp

// Host-side launch helpers (defined in the .cu files).
namespace nlsp {
struct LaunchCtx {
    cudaStream_t s;
    int num_sms;
    unsigned long long* launches;  // incremented per kernel launch
    // launch with programmatic stream serialization (PDL): the kernel may be
    // scheduled while its predecessor drains; it must start with pdl_entry()
    bool pdl = false;
};
}  // namespace nlsp
