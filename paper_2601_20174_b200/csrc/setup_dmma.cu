// paper_2601_20174_b200/csrc/setup_dmma.cu — the setup contractions on the FP64
// tensor pipe (DMMA, `mma.sync.m8n8k4.f64`; sm_100a has no tcgen05 f64 kind):
//
//   k_gram_dmma      C = X^T Y per CTA (tall X, Y; the m x m Gram S^T S of
//                    svd_oracle, svd.hpp:162-166, the CholeskyQR2 Grams and the
//                    Galerkin Q^T (A Q), two_level.hpp:33-51)
//   k_dense_mm_dmma  Y = X W (/ sigma) (U_k = S V_k / sigma_k, svd.hpp:189-202, and
//                    the CholeskyQR2 products Q = B R^-1)
//
// Both stream row tiles of the tall operand through shared memory with
// cp.async (2 stages) and keep the small operand / the accumulators on chip.
// Fragment layouts (PTX ISA, mma m8n8k4 .f64): A 8x4 row-major, lane holds
// A[lane/4][lane%4]; B 4x8 col-major, lane holds B[lane%4][lane/4]; C/D 8x8,
// lane holds D[lane/4][2(lane%4) + {0,1}].
//
// Rounding differs from the reference's sequential sums only in summation
// order (fp64 products, fp64 accumulation); the parity tests bound P, sigma
// and A_c against the reference at 1e-10 / 1e-12.
#include <cstdlib>

#include "internal.cuh"

namespace nlsp {

namespace {

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// 8-byte async copy global -> shared, zero-filled when !valid
__device__ __forceinline__ void cp8(double* dst, const double* src, bool valid) {
    const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
    const int n = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

}  // namespace

// ------------------------------------------------------------------- Gram --
// C tile (TM x TN) = X[:, i0:i0+bi]^T Y[:, j0:j0+bj] over this CTA's 16-row
// tiles (grid-stride); 8 warps as 4 (rows of C) x 2 (cols of C), warp tile
// (8 WM) x (8 WN). SAME: X == Y over the same columns (one staged tile).
template <int WM, int WN, bool SAME>
__global__ void __launch_bounds__(256) k_gram_dmma(long long rows, int bi, int bj, int lda, int ldb,
                                                   const double* __restrict__ X,
                                                   const double* __restrict__ Y,
                                                   double* __restrict__ part) {
    constexpr int TM = 4 * WM * 8, TN = 2 * WN * 8, RB = 16;
    constexpr int LX = TM + 4, LY = TN + 4;  // +4 doubles: conflict-free fragment loads
    extern __shared__ __align__(16) double sm[];
    double* xs = sm;                                 // [2][RB][LX]
    double* ys = SAME ? xs : sm + 2 * RB * LX;       // [2][RB][LY]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp >> 1, wn = warp & 1;
    const long long tiles = (rows + RB - 1) / RB;
    auto load = [&](long long tile, int stg) {
        const long long r0 = tile * RB;
        for (int idx = tid; idx < RB * TM; idx += 256) {
            const int r = idx / TM, c = idx - r * TM;
            const long long row = r0 + r;
            const bool ok = row < rows && c < bi;
            cp8(xs + stg * RB * LX + r * LX + c, ok ? X + row * lda + c : X, ok);
        }
        if (!SAME)
            for (int idx = tid; idx < RB * TN; idx += 256) {
                const int r = idx / TN, c = idx - r * TN;
                const long long row = r0 + r;
                const bool ok = row < rows && c < bj;
                cp8(ys + stg * RB * LY + r * LY + c, ok ? Y + row * ldb + c : Y, ok);
            }
        cp_commit();
    };
    double acc[WM][WN][2];
#pragma unroll
    for (int a = 0; a < WM; ++a)
#pragma unroll
        for (int b = 0; b < WN; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    long long tile = blockIdx.x;
    if (tile < tiles) load(tile, 0);
    for (int i = 0; tile < tiles; tile += gridDim.x, ++i) {
        const int stg = i & 1;
        const bool more = tile + gridDim.x < tiles;
        if (more) load(tile + gridDim.x, stg ^ 1);
        if (more) cp_wait<1>();
        else cp_wait<0>();
        __syncthreads();
        const double* xb = xs + stg * RB * LX + (lane & 3) * LX + wm * WM * 8 + (lane >> 2);
        const double* yb = ys + stg * RB * LY + (lane & 3) * LY + wn * WN * 8 + (lane >> 2);
#pragma unroll
        for (int kk = 0; kk < RB; kk += 4) {
            double fa[WM], fb[WN];
#pragma unroll
            for (int a = 0; a < WM; ++a) fa[a] = xb[kk * LX + a * 8];
#pragma unroll
            for (int b = 0; b < WN; ++b) fb[b] = yb[kk * LY + b * 8];
#pragma unroll
            for (int a = 0; a < WM; ++a)
#pragma unroll
                for (int b = 0; b < WN; ++b) dmma(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
        }
        __syncthreads();  // this stage is refilled next-but-one iteration
    }
    double* out = part + (long long)blockIdx.x * bi * bj;
#pragma unroll
    for (int a = 0; a < WM; ++a)
#pragma unroll
        for (int b = 0; b < WN; ++b) {
            const int row = wm * WM * 8 + a * 8 + (lane >> 2);
            const int col = wn * WN * 8 + b * 8 + 2 * (lane & 3);
            if (row < bi) {
                if (col < bj) out[row * bj + col] = acc[a][b][0];
                if (col + 1 < bj) out[row * bj + col + 1] = acc[a][b][1];
            }
        }
}

// The symmetric Gram X^T X (svd_oracle's S^T S, the CholeskyQR Grams): only the
// 8x8 blocks on and above the diagonal are computed — NB (NB + 1) / 2 of the
// NB^2 — and mirrored on the way out. Warp w < NB/2 owns block rows w and
// NB - 1 - w, NB + 1 blocks each (balanced). NB = bi / 8 rounded up (12 or 16).
template <int NB>
__global__ void __launch_bounds__(256) k_gram_dmma_sym(long long rows, int bi, int lda, const double* __restrict__ X,
                                                       double* __restrict__ part) {
    constexpr int TM = NB * 8, RB = 16, LX = TM + 4;
    extern __shared__ __align__(16) double sm[];
    double* xs = sm;  // [2][RB][LX]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long tiles = (rows + RB - 1) / RB;
    auto load = [&](long long tile, int stg) {
        const long long r0 = tile * RB;
        for (int idx = tid; idx < RB * TM; idx += 256) {
            const int r = idx / TM, c = idx - r * TM;
            const long long row = r0 + r;
            const bool ok = row < rows && c < bi;
            cp8(xs + stg * RB * LX + r * LX + c, ok ? X + row * lda + c : X, ok);
        }
        cp_commit();
    };
    const bool active = warp < NB / 2;
    const int ra = warp, rb = NB - 1 - warp;  // this warp's two block rows
    double acc0[NB][2], acc1[NB][2];
#pragma unroll
    for (int c = 0; c < NB; ++c) acc0[c][0] = acc0[c][1] = acc1[c][0] = acc1[c][1] = 0.0;
    long long tile = blockIdx.x;
    if (tile < tiles) load(tile, 0);
    for (int i = 0; tile < tiles; tile += gridDim.x, ++i) {
        const int stg = i & 1;
        const bool more = tile + gridDim.x < tiles;
        if (more) load(tile + gridDim.x, stg ^ 1);
        if (more) cp_wait<1>();
        else cp_wait<0>();
        __syncthreads();
        if (active) {
            const double* xb = xs + stg * RB * LX + (lane & 3) * LX + (lane >> 2);
#pragma unroll
            for (int kk = 0; kk < RB; kk += 4) {
                double f[NB];
#pragma unroll
                for (int c = 0; c < NB; ++c) f[c] = c >= ra ? xb[kk * LX + c * 8] : 0.0;
                const double fa = xb[kk * LX + ra * 8], fb = xb[kk * LX + rb * 8];
#pragma unroll
                for (int c = 0; c < NB; ++c) {
                    if (c >= ra) dmma(acc0[c][0], acc0[c][1], fa, f[c]);
                    if (c >= rb) dmma(acc1[c][0], acc1[c][1], fb, f[c]);
                }
            }
        }
        __syncthreads();  // this stage is refilled next-but-one iteration
    }
    if (!active) return;
    double* out = part + (long long)blockIdx.x * bi * bi;
    auto put = [&](int br, int c, const double (&acc)[NB][2]) {
        const int row = br * 8 + (lane >> 2);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int col = c * 8 + 2 * (lane & 3) + h;
            if (row < bi && col < bi) {
                out[row * bi + col] = acc[c][h];
                if (c != br) out[col * bi + row] = acc[c][h];  // the mirrored block
            }
        }
    };
#pragma unroll
    for (int c = 0; c < NB; ++c) {
        if (c >= ra) put(ra, c, acc0);
        if (c >= rb) put(rb, c, acc1);
    }
}

// Tile configuration covering a bi x bj block (<= 128 x 128); returns false
// when the block is larger.
bool launch_gram_dmma(cudaStream_t s, int g, long long rows, int bi, int bj, int lda, int ldb,
                      const double* X, const double* Y, double* part) {
    const bool same = X == Y && bi == bj && lda == ldb;
    const int w = bi > bj ? bi : bj;
    static const bool sym_on = !(std::getenv("NLSP_GRAM_SYM") && std::atoi(std::getenv("NLSP_GRAM_SYM")) == 0);
    if (same && sym_on && bi > 64) {
        // symmetric: half the DMMA blocks (k_gram_dmma_sym)
        const int nb = (bi + 7) / 8;
        if (nb <= 12) {
            const size_t smem = 2 * 16 * (12 * 8 + 4) * 8;
            cudaFuncSetAttribute(k_gram_dmma_sym<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_gram_dmma_sym<12><<<g, 256, smem, s>>>(rows, bi, lda, X, part);
        } else {
            const size_t smem = 2 * 16 * (16 * 8 + 4) * 8;
            cudaFuncSetAttribute(k_gram_dmma_sym<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            k_gram_dmma_sym<16><<<g, 256, smem, s>>>(rows, bi, lda, X, part);
        }
        return true;
    }
#define NLSP_GD(WM, WN)                                                                           \
    do {                                                                                          \
        constexpr int TM = 4 * (WM) * 8, TN = 2 * (WN) * 8;                                       \
        const size_t smem = same ? 2 * 16 * (TM + 4) * 8 : 2 * 16 * (TM + 4 + TN + 4) * 8;      \
        if (same) {                                                                               \
            cudaFuncSetAttribute(k_gram_dmma<WM, WN, true>,                                       \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
            k_gram_dmma<WM, WN, true><<<g, 256, smem, s>>>(rows, bi, bj, lda, ldb, X, Y, part);  \
        } else {                                                                                  \
            cudaFuncSetAttribute(k_gram_dmma<WM, WN, false>,                                      \
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);         \
            k_gram_dmma<WM, WN, false><<<g, 256, smem, s>>>(rows, bi, bj, lda, ldb, X, Y, part); \
        }                                                                                         \
    } while (0)
    if (w <= 32) NLSP_GD(1, 2);
    else if (w <= 64) NLSP_GD(2, 4);
    else if (w <= 128) NLSP_GD(4, 8);
    else return false;
#undef NLSP_GD
    return true;
}

// ------------------------------------------------------------- X W / sigma --
// Y (rows x kout) = X (rows x m) W (m x kout) (/ sigma_j), m <= 128,
// kout <= 64. W (padded) stays in shared memory; 32-row X tiles stream
// through 2 cp.async stages. 8 warps as 2 (16 rows each) x 4 (16 cols each).
__global__ void __launch_bounds__(256) k_dense_mm_dmma(long long rows, int m, int kout,
                                                       const double* __restrict__ X,
                                                       const double* __restrict__ W,
                                                       const double* __restrict__ sigma,
                                                       double* __restrict__ Y) {
    constexpr int RT = 32, TN = 64, LW = TN + 4;
    const int mp = (m + 3) & ~3;  // k-steps of 4 (zero padded)
    const int LXm = mp + 4;
    extern __shared__ __align__(16) double sm[];
    double* ws = sm;              // [mp][LW]
    double* xs = sm + mp * LW;    // [2][RT][LXm]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wr = warp >> 2, wc = warp & 3;
    for (int idx = tid; idx < mp * TN; idx += 256) {
        const int i = idx / TN, j = idx - i * TN;
        ws[i * LW + j] = (i < m && j < kout) ? W[(long long)i * kout + j] : 0.0;
    }
    const long long tiles = (rows + RT - 1) / RT;
    auto load = [&](long long tile, int stg) {
        const long long r0 = tile * RT;
        double* dst = xs + stg * RT * LXm;
        for (int idx = tid; idx < RT * mp; idx += 256) {
            const int r = idx / mp, c = idx - r * mp;
            const long long row = r0 + r;
            const bool ok = row < rows && c < m;
            cp8(dst + r * LXm + c, ok ? X + row * m + c : X, ok);
        }
        cp_commit();
    };
    double sig[2][2];
#pragma unroll
    for (int b = 0; b < 2; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int col = wc * 16 + b * 8 + 2 * (lane & 3) + h;
            sig[b][h] = (sigma && col < kout) ? sigma[col] : 1.0;
        }
    long long tile = blockIdx.x;
    if (tile < tiles) load(tile, 0);
    for (int i = 0; tile < tiles; tile += gridDim.x, ++i) {
        const int stg = i & 1;
        const bool more = tile + gridDim.x < tiles;
        if (more) load(tile + gridDim.x, stg ^ 1);
        if (more) cp_wait<1>();
        else cp_wait<0>();
        __syncthreads();
        double acc[2][2][2];
#pragma unroll
        for (int a = 0; a < 2; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
        const double* xb = xs + stg * RT * LXm + (wr * 16 + (lane >> 2)) * LXm + (lane & 3);
        const double* wb = ws + (lane & 3) * LW + wc * 16 + (lane >> 2);
        for (int kk = 0; kk < mp; kk += 4) {
            double fa[2], fb[2];
#pragma unroll
            for (int a = 0; a < 2; ++a) fa[a] = xb[a * 8 * LXm + kk];
#pragma unroll
            for (int b = 0; b < 2; ++b) fb[b] = wb[kk * LW + b * 8];
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 2; ++b) dmma(acc[a][b][0], acc[a][b][1], fa[a], fb[b]);
        }
        const long long r0 = tile * RT;
#pragma unroll
        for (int a = 0; a < 2; ++a) {
            const long long row = r0 + wr * 16 + a * 8 + (lane >> 2);
            if (row >= rows) continue;
#pragma unroll
            for (int b = 0; b < 2; ++b) {
                const int col = wc * 16 + b * 8 + 2 * (lane & 3);
                if (col < kout) Y[row * kout + col] = sigma ? acc[a][b][0] / sig[b][0] : acc[a][b][0];
                if (col + 1 < kout)
                    Y[row * kout + col + 1] = sigma ? acc[a][b][1] / sig[b][1] : acc[a][b][1];
            }
        }
        __syncthreads();  // this stage is refilled next-but-one iteration
    }
}

bool launch_dense_mm_dmma(cudaStream_t s, int num_sms, long long rows, int m, int kout, const double* X,
                          const double* W, const double* sigma, double* Y) {
    if (m > 128 || kout > 64 || m < 1 || kout < 1) return false;
    const int mp = (m + 3) & ~3;
    const size_t smem = ((size_t)mp * 68 + 2 * 32 * (size_t)(mp + 4)) * 8;
    cudaFuncSetAttribute(k_dense_mm_dmma, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    long long g = (rows + 31) / 32;
    if (g > num_sms) g = num_sms;
    if (g < 1) g = 1;
    k_dense_mm_dmma<<<(int)g, 256, smem, s>>>(rows, m, kout, X, W, sigma, Y);
    return true;
}

}  // namespace nlsp
