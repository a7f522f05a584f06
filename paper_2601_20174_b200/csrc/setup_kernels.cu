// paper_2601_20174_b200/csrc/setup_kernels.cu — setup path on sm_100a:
//
//   k_csr_import     size_t CSR -> int32 CSR, invariant checks, diagonal
//   k_block_sweep    S <- S + w D^-1 (0 - A S)   (smoothing.hpp:50-60), also plain Y = A X
//   k_gram_partial   C = X^T Y per CTA (+ k_gram_reduce), register-tiled fp64
//   k_eigh           cyclic-by-rounds parallel Jacobi on the m x m Gram (svd.hpp:23-88)
//   k_dense_mm       Y = X W (/ sigma) for the tall-skinny basis products
//   k_colsign_*      largest-|entry|-nonnegative column signs (svd.hpp:209-225)
//   k_chol / k_tri_inv_lower / k_symmetrize   single-CTA k x k kernels
#include <cfloat>
#include <cstdlib>

#include "internal.cuh"

namespace nlsp {

// ------------------------------------------------------------ CSR import --
// flags bit 0: bad row_ptr, bit 1: column out of range, bit 2: unsorted or
// duplicate column
__global__ void k_csr_import(int n, long long nnz, const unsigned long long* rp64,
                             const unsigned long long* ci64, const double* v, int* rp, int* ci,
                             double* diag, int* flags, int* max_row) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const unsigned long long b = rp64[i], e = rp64[i + 1];
        rp[i] = static_cast<int>(b);
        if (i == n - 1) rp[n] = static_cast<int>(e);
        if (e < b || e > (unsigned long long)nnz) {
            atomicOr(flags, 1);
            diag[i] = 0.0;
            continue;
        }
        atomicMax(max_row, static_cast<int>(e - b));
        double d = 0.0;
        long long prev = -1;
        for (unsigned long long k = b; k < e; ++k) {
            const unsigned long long c = ci64[k];
            if (c >= (unsigned long long)n) {
                atomicOr(flags, 2);
                ci[k] = 0;
                continue;
            }
            if ((long long)c <= prev) atomicOr(flags, 4);
            prev = (long long)c;
            ci[k] = static_cast<int>(c);
            if ((long long)c == i) d = v[k];
        }
        diag[i] = d;
    }
}

// w_i = omega * (1 / A_ii) (JacobiSmoother ctor, smoothing.hpp:19-29, then the
// sweep's omega_ * inv_diag_[i]); flag NumericError on A_ii <= 0
__global__ void k_wd(int n, const double* diag, double omega, double* wd, int* flag) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        const double d = diag[i];
        if (d <= 0.0) {
            atomicOr(flag, 1);
            wd[i] = 0.0;
        } else {
            wd[i] = omega * (1.0 / d);
        }
    }
}

// ----------------------------------------------------------- block sweep --
// L lanes per row, columns j = lane + L t. Each output entry accumulates the
// row's nonzeros in column order with one fma per term (the -O3 -march build of
// spmm, sparse.hpp:131-146), then x + w (0 - ax) (smoothing.hpp:50-60).
// MODE 0: sweep (out = fma(w, -acc, in)); MODE 1: plain out = acc.
template <int L, int T, int MODE>
__global__ void __launch_bounds__(256) k_block_sweep(int n, const int* __restrict__ rp,
                                                     const int* __restrict__ ci,
                                                     const double* __restrict__ v,
                                                     const double* __restrict__ wd, int m,
                                                     const double* __restrict__ in,
                                                     double* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    const int lr = lane % L;
    const int sub = lane / L;
    constexpr int RPW = 32 / L;
    const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
    for (int c0 = 0; c0 < m; c0 += L * T) {
        for (long long base = wid * RPW; base < n; base += nw * RPW) {
            const long long row = base + sub;
            if (row >= n) continue;
            double acc[T];
#pragma unroll
            for (int t = 0; t < T; ++t) acc[t] = 0.0;
            const int b = rp[row], e = rp[row + 1];
            for (int k = b; k < e; ++k) {
                const double aik = v[k];
                const double* xr = in + (long long)ci[k] * m;
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    const int j = c0 + lr + L * t;
                    if (j < m) acc[t] = fma(aik, xr[j], acc[t]);
                }
            }
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const int j = c0 + lr + L * t;
                if (j < m) {
                    const long long o = row * m + j;
                    if (MODE == 0) out[o] = fma(wd[row], 0.0 - acc[t], in[o]);
                    else out[o] = acc[t];
                }
            }
        }
    }
}

// The same block sweep over the diagonal form of A (exact 5/7/9-offset
// patterns): the offsets are kernel parameters, so every neighbour row of x is
// loaded at once (clamped rows, no column-index load in front of them), then
// each output entry accumulates the present offsets in ascending order (= the
// CSR column order): bitwise the CSR kernel's result.
// HINT: S (the block being swept) is read with an L2 evict_last policy and the
// output written with evict-first (st.global.cs): a row of S is read again
// +-P rows (26 MB of S at C4) after its first use, and the streaming output
// would otherwise push it out of L2 in between (2.2x S read from DRAM).
__device__ __forceinline__ unsigned long long l2_keep_policy() {
    unsigned long long p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ double ld_keep(const double* a, unsigned long long pol) {
    double v;
    asm volatile("ld.global.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(a), "l"(pol));
    return v;
}

template <int D, int T, int MODE, bool HINT>
__global__ void __launch_bounds__(256) k_block_sweep_dia(int n, DiaArgs dia, const double* __restrict__ wd,
                                                         int m, const double* __restrict__ in,
                                                         double* __restrict__ out) {
    const unsigned long long pol = HINT ? l2_keep_policy() : 0ull;
    const int lane = threadIdx.x & 31;
    const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
    const int mb = dia.mbytes;
    for (int c0 = 0; c0 < m; c0 += 32 * T) {
        for (long long row = wid; row < n; row += nw) {
            unsigned msk;
            if (mb == 1) msk = static_cast<const unsigned char*>(dia.mask)[row];
            else if (mb == 2) msk = static_cast<const unsigned short*>(dia.mask)[row];
            else msk = static_cast<const unsigned*>(dia.mask)[row];
            double xv[D][T], av[D];
#pragma unroll
            for (int t = 0; t < D; ++t) {
                const long long nb = min(max(row + dia.off[t], 0LL), (long long)n - 1);
                av[t] = dia.kind == 2 ? dia.rv[(size_t)t * n + row] : dia.val[t];
                const double* xr = in + nb * m;
#pragma unroll
                for (int u = 0; u < T; ++u) {
                    const int j = c0 + lane + 32 * u;
                    xv[t][u] = j < m ? (HINT ? ld_keep(xr + j, pol) : xr[j]) : 0.0;
                }
            }
            double acc[T];
#pragma unroll
            for (int u = 0; u < T; ++u) acc[u] = 0.0;
#pragma unroll
            for (int t = 0; t < D; ++t)
                if ((msk >> t) & 1u) {
#pragma unroll
                    for (int u = 0; u < T; ++u) acc[u] = fma(av[t], xv[t][u], acc[u]);
                }
#pragma unroll
            for (int u = 0; u < T; ++u) {
                const int j = c0 + lane + 32 * u;
                if (j < m) {
                    const long long o = row * m + j;
                    const double r = MODE == 0 ? fma(wd[row], 0.0 - acc[u], in[o]) : acc[u];
                    if (HINT) __stcs(out + o, r);
                    else out[o] = r;
                }
            }
        }
    }
}

// ------------------------------------------------------------------ Gram --
// C = X^T Y for tall X (rows x ca), Y (rows x cb), row-major. 256 threads as a
// 16 x 16 grid; thread (ti, tj) owns a TI x TJ block of C. Row tiles of X and Y
// are staged in shared memory; each CTA writes its partial C.
template <int TI>
__global__ void __launch_bounds__(256) k_gram_partial(long long rows, int ca, int cb, int lda,
                                                      int ldb, const double* __restrict__ X,
                                                      const double* __restrict__ Y,
                                                      double* __restrict__ part) {
    constexpr int RB = 16;
    extern __shared__ double sm[];
    double* xs = sm;                 // RB x (16*TI)
    double* ys = sm + RB * 16 * TI;  // RB x (16*TI)
    const int W = 16 * TI;
    const int ti = threadIdx.x / 16, tj = threadIdx.x % 16;
    double acc[TI][TI];
#pragma unroll
    for (int a = 0; a < TI; ++a)
#pragma unroll
        for (int b = 0; b < TI; ++b) acc[a][b] = 0.0;
    const long long tiles = (rows + RB - 1) / RB;
    for (long long tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const long long r0 = tile * RB;
        for (int idx = threadIdx.x; idx < RB * W; idx += blockDim.x) {
            const int rr = idx / W, cc = idx % W;
            const long long row = r0 + rr;
            xs[idx] = (row < rows && cc < ca) ? X[row * lda + cc] : 0.0;
            ys[idx] = (row < rows && cc < cb) ? Y[row * ldb + cc] : 0.0;
        }
        __syncthreads();
#pragma unroll 4
        for (int rr = 0; rr < RB; ++rr) {
            double xa[TI], yb[TI];
#pragma unroll
            for (int a = 0; a < TI; ++a) xa[a] = xs[rr * W + ti * TI + a];
#pragma unroll
            for (int b = 0; b < TI; ++b) yb[b] = ys[rr * W + tj * TI + b];
#pragma unroll
            for (int a = 0; a < TI; ++a)
#pragma unroll
                for (int b = 0; b < TI; ++b) acc[a][b] = fma(xa[a], yb[b], acc[a][b]);
        }
        __syncthreads();
    }
    double* out = part + (long long)blockIdx.x * ca * cb;
#pragma unroll
    for (int a = 0; a < TI; ++a)
#pragma unroll
        for (int b = 0; b < TI; ++b) {
            const int i = ti * TI + a, j = tj * TI + b;
            if (i < ca && j < cb) out[i * cb + j] = acc[a][b];
        }
}

// fixed-order sum of the CTA partials of a ca x cb block into C (row stride ldc)
__global__ void k_gram_reduce(int nparts, int ca, int cb, const double* part, double* c, int ldc) {
    const int count = ca * cb;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < count;
         idx += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int p = 0; p < nparts; ++p) s += part[(long long)p * count + idx];
        c[(idx / cb) * ldc + idx % cb] = s;
    }
}

// ------------------------------------------------------------- eigensolve --
// Jacobi eigensolver for a symmetric m x m matrix in one CTA. A sweep visits
// every (p, q) pair once, as m-1 rounds of m/2 disjoint rotations (round-robin
// tournament), each rotation formed with the reference's formulas
// (svd.hpp:44-65) and applied as A <- J^T A J, V <- V J. Same convergence test
// (off-norm <= 1e-12 ||A||_F, at most 30 sweeps) and stable descending sort as
// svd.hpp:29-40,70-87. A is held as its packed upper triangle.
struct EighArgs {
    int m;
    double* a_packed;  // m(m+1)/2, shared or global scratch
    double* v;         // m x m, shared or global scratch
    const double* g;   // input m x m (global)
    double* evals;     // out m (descending)
    double* evecs;     // out m x m, columns
    int* status;       // out: 0 ok, kErrConvergence
    int* sweeps_out;
};

__device__ __forceinline__ int pidx(int i, int j, int m) {  // i <= j
    return i * m - (i * (i - 1)) / 2 + (j - i);
}
__device__ __forceinline__ double& pel(double* a, int i, int j, int m) {
    return i <= j ? a[pidx(i, j, m)] : a[pidx(j, i, m)];
}

__global__ void __launch_bounds__(1024) k_eigh(EighArgs args, int use_shared) {
    extern __shared__ double sm[];
    const int m = args.m;
    const int mp = m + (m & 1);  // even number of tournament players
    double* a = use_shared ? sm : args.a_packed;
    double* v = use_shared ? sm + (m * (m + 1)) / 2 : args.v;
    __shared__ double cs_c[512], cs_s[512];
    __shared__ int pp[512], pq[512];
    __shared__ double red[32];
    __shared__ double total_s, off_s;
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int idx = tid; idx < m * m; idx += nt) {
        const int i = idx / m, j = idx % m;
        v[idx] = (i == j) ? 1.0 : 0.0;
        if (i <= j) a[pidx(i, j, m)] = args.g[idx];
    }
    __syncthreads();
    // ||A||_F over the full matrix (frobenius_norm, dense.hpp:129)
    auto block_sum = [&](double t) {
        t = warp_sum(t);
        if ((tid & 31) == 0) red[tid >> 5] = t;
        __syncthreads();
        double r = 0.0;
        if (tid < 32) {
            r = tid < (nt >> 5) ? red[tid] : 0.0;
            r = warp_sum(r);
        }
        __syncthreads();
        return r;  // valid in thread 0 (and warp 0)
    };
    double t = 0.0;
    for (int idx = tid; idx < m * m; idx += nt) {
        const int i = idx / m, j = idx % m;
        const double x = pel(a, i, j, m);
        t = fma(x, x, t);
    }
    t = block_sum(t);
    if (tid == 0) total_s = sqrt(t);
    __syncthreads();
    const double total = total_s;
    // the (u, w) 2x2 blocks of every round are the same for a thread: decode
    // them once (up to kEighBlk per thread; larger m decodes per round)
    constexpr int kEighBlk = 4;
    const int np_ = mp / 2;
    const int nblocks_ = np_ * (np_ + 1) / 2;
    const bool pre_blk = nblocks_ <= kEighBlk * nt;
    auto decode = [&](int bi, int& u, int& w) {
        // row u of the upper triangle starts at u np - u (u - 1) / 2 (closed
        // form, then a +-1 fix-up)
        const double b2 = 2.0 * np_ + 1.0;
        u = (int)((b2 - sqrt(b2 * b2 - 8.0 * bi)) * 0.5);
        auto row_start = [&](int uu) { return uu * np_ - (uu * (uu - 1)) / 2; };
        if (u < 0) u = 0;
        if (u > np_ - 1) u = np_ - 1;
        while (u > 0 && row_start(u) > bi) --u;
        while (u < np_ - 1 && row_start(u + 1) <= bi) ++u;
        w = u + (bi - row_start(u));
    };
    int blk_u[kEighBlk], blk_w[kEighBlk];
#pragma unroll
    for (int j = 0; j < kEighBlk; ++j) {
        blk_u[j] = blk_w[j] = -1;
        const int bi = tid + j * nt;
        if (pre_blk && bi < nblocks_) decode(bi, blk_u[j], blk_w[j]);
    }
    // V update mapping: a fixed rotation w per thread when nt is a multiple of np
    const bool v_fixed = (nt % np_) == 0;
    const int v_w = tid % np_, v_i0 = tid / np_, v_step = nt / np_;
    int sweeps = 0;
    int status = isfinite(total) ? 0 : kErrValidation;  // svd.hpp:156 all_finite gate
    for (; status == 0;) {
        double o = 0.0;
        for (int idx = tid; idx < m * m; idx += nt) {
            const int i = idx / m, j = idx % m;
            if (i < j) {
                const double x = a[pidx(i, j, m)];
                o = fma(2.0 * x, x, o);
            }
        }
        o = block_sum(o);
        if (tid == 0) off_s = sqrt(o);
        __syncthreads();
        if (!(off_s > 1e-12 * total && total > 0.0)) break;
        if (sweeps >= 30) {
            status = kErrConvergence;
            break;
        }
        ++sweeps;
        for (int round = 0; round < mp - 1; ++round) {
            // pairing (circle method) and rotation parameters
            for (int w = tid; w < mp / 2; w += nt) {
                auto player = [&](int pos) {
                    return pos == 0 ? 0 : 1 + ((pos - 1 + round) % (mp - 1));
                };
                int p = player(w), q = player(mp - 1 - w);
                if (p > q) { const int tmp = p; p = q; q = tmp; }
                pp[w] = p;
                pq[w] = q;
                double c = 1.0, s = 0.0;
                if (q < m) {
                    const double apq = a[pidx(p, q, m)];
                    if (apq != 0.0) {
                        const double theta = (a[pidx(q, q, m)] - a[pidx(p, p, m)]) / (2.0 * apq);
                        const double tt = (theta >= 0.0 ? 1.0 : -1.0) /
                                          (fabs(theta) + sqrt(theta * theta + 1.0));
                        c = 1.0 / sqrt(tt * tt + 1.0);
                        s = tt * c;
                    }
                }
                cs_c[w] = c;
                cs_s[w] = s;
            }
            __syncthreads();
            // A <- J^T A J on 2x2 blocks (pair u rows, pair w cols), u <= w
            const int np = mp / 2;
            const int nblocks = np * (np + 1) / 2;
            auto block = [&](int u, int w) {
                const int p1 = pp[u], q1 = pq[u], p2 = pp[w], q2 = pq[w];
                const double c1 = cs_c[u], s1 = cs_s[u], c2 = cs_c[w], s2 = cs_s[w];
                const bool q1v = q1 < m, q2v = q2 < m;
                if (u == w) {
                    if (!q1v) return;
                    const double xpp = a[pidx(p1, p1, m)], xpq = a[pidx(p1, q1, m)],
                                 xqq = a[pidx(q1, q1, m)];
                    // columns: y(., p) = c x(., p) - s x(., q); y(., q) = s x(., p) + c x(., q)
                    const double ypp = c1 * xpp - s1 * xpq, ypq = s1 * xpp + c1 * xpq;
                    const double yqp = c1 * xpq - s1 * xqq, yqq = s1 * xpq + c1 * xqq;
                    // rows: z(p, .) = c y(p, .) - s y(q, .); z(q, .) = s y(p, .) + c y(q, .)
                    a[pidx(p1, p1, m)] = c1 * ypp - s1 * yqp;
                    a[pidx(p1, q1, m)] = c1 * ypq - s1 * yqq;
                    a[pidx(q1, q1, m)] = s1 * ypq + c1 * yqq;
                } else {
                    // rows {p1, q1} (rotation 1), cols {p2, q2} (rotation 2)
                    const double xpp = pel(a, p1, p2, m);
                    const double xpq = q2v ? pel(a, p1, q2, m) : 0.0;
                    const double xqp = q1v ? pel(a, q1, p2, m) : 0.0;
                    const double xqq = (q1v && q2v) ? pel(a, q1, q2, m) : 0.0;
                    const double ypp = c2 * xpp - s2 * xpq, ypq = s2 * xpp + c2 * xpq;
                    const double yqp = c2 * xqp - s2 * xqq, yqq = s2 * xqp + c2 * xqq;
                    pel(a, p1, p2, m) = c1 * ypp - s1 * yqp;
                    if (q2v) pel(a, p1, q2, m) = c1 * ypq - s1 * yqq;
                    if (q1v) pel(a, q1, p2, m) = s1 * ypp + c1 * yqp;
                    if (q1v && q2v) pel(a, q1, q2, m) = s1 * ypq + c1 * yqq;
                }
            };
            if (pre_blk) {
#pragma unroll
                for (int j = 0; j < kEighBlk; ++j)
                    if (blk_u[j] >= 0) block(blk_u[j], blk_w[j]);
            } else {
                for (int bi = tid; bi < nblocks; bi += nt) {
                    int u, w;
                    decode(bi, u, w);
                    block(u, w);
                }
            }
            // V <- V J (svd.hpp:61-65)
            if (v_fixed) {
                const int p = pp[v_w], q = pq[v_w];
                if (q < m) {
                    const double c = cs_c[v_w], s = cs_s[v_w];
                    for (int i = v_i0; i < m; i += v_step) {
                        const double vip = v[i * m + p], viq = v[i * m + q];
                        v[i * m + p] = c * vip - s * viq;
                        v[i * m + q] = s * vip + c * viq;
                    }
                }
            } else {
                for (int idx = tid; idx < m * np; idx += nt) {
                    const int i = idx / np, w = idx % np;
                    const int p = pp[w], q = pq[w];
                    if (q >= m) continue;
                    const double c = cs_c[w], s = cs_s[w];
                    const double vip = v[i * m + p], viq = v[i * m + q];
                    v[i * m + p] = c * vip - s * viq;
                    v[i * m + q] = s * vip + c * viq;
                }
            }
            __syncthreads();
        }
    }
    // stable descending order: rank_i = #{j : ev_j > ev_i} + #{j < i : ev_j == ev_i}
    for (int i = tid; i < m; i += nt) {
        const double ei = a[pidx(i, i, m)];
        int rank = 0;
        for (int j = 0; j < m; ++j) {
            const double ej = a[pidx(j, j, m)];
            rank += (ej > ei) || (ej == ei && j < i);
        }
        args.evals[rank] = ei;
        for (int r = 0; r < m; ++r) args.evecs[r * m + rank] = v[r * m + i];
    }
    if (tid == 0) {
        *args.status = status;
        *args.sweeps_out = sweeps;
    }
}

// ------------------------------------------------------------- dense mm --
// Y[i, j] = (sum_l X[i, l] W[l, j]) (/ sigma[j]) for j < kout, accumulated in
// l order (svd.hpp:193-199). One warp per row; W staged in shared memory.
template <int T>
__global__ void __launch_bounds__(256) k_dense_mm(long long rows, int m, int kout,
                                                  const double* __restrict__ X,
                                                  const double* __restrict__ Wg,
                                                  const double* __restrict__ sigma,
                                                  double* __restrict__ Y, int use_shared) {
    extern __shared__ double sw[];
    const double* W = Wg;
    if (use_shared) {
        for (int idx = threadIdx.x; idx < m * kout; idx += blockDim.x) sw[idx] = Wg[idx];
        __syncthreads();
        W = sw;
    }
    const int lane = threadIdx.x & 31;
    const long long wid = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
    const long long nw = (gridDim.x * (long long)blockDim.x) >> 5;
    for (long long row = wid; row < rows; row += nw) {
        const double* xr = X + row * m;
        for (int c0 = 0; c0 < kout; c0 += 32 * T) {  // column blocks (kout > 32 T)
            double acc[T];
#pragma unroll
            for (int t = 0; t < T; ++t) acc[t] = 0.0;
            for (int l0 = 0; l0 < m; l0 += 32) {
                const double xl = (l0 + lane < m) ? xr[l0 + lane] : 0.0;
                const int lim = min(32, m - l0);
                for (int u = 0; u < lim; ++u) {
                    const double s = __shfl_sync(0xffffffffu, xl, u);
                    const double* wr = W + (long long)(l0 + u) * kout;
#pragma unroll
                    for (int t = 0; t < T; ++t) {
                        const int j = c0 + lane + 32 * t;
                        if (j < kout) acc[t] = fma(s, wr[j], acc[t]);
                    }
                }
            }
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const int j = c0 + lane + 32 * t;
                if (j < kout) Y[row * kout + j] = sigma ? acc[t] / sigma[j] : acc[t];
            }
        }
    }
}

// -------------------------------------------------------------- col signs --
// per CTA: for each column, (max |x|, first row attaining it, x at that row)
__global__ void k_colmax_partial(long long rows, int k, const double* __restrict__ P,
                                 double* pmag, long long* pidx_out, double* pval) {
    // thread (sub, j): column j over rows blockIdx * tpc + sub, stepping by
    // gridDim * tpc, in increasing order (first maximum kept); a CTA step reads
    // tpc whole rows (coalesced), 4 steps' loads in flight per thread
    extern __shared__ unsigned char smraw[];
    double* bm = reinterpret_cast<double*>(smraw);
    long long* bi = reinterpret_cast<long long*>(bm + blockDim.x);
    double* bv = reinterpret_cast<double*>(bi + blockDim.x);
    const int tpc = blockDim.x / k;
    const int t = threadIdx.x, j = t % k, sub = t / k;
    double best = -1.0, val = 0.0;
    long long arg = -1;
    if (sub < tpc) {
        const long long step = (long long)gridDim.x * tpc;
        for (long long i0 = (long long)blockIdx.x * tpc + sub; i0 < rows; i0 += 4 * step) {
            double x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const long long i = i0 + u * step;
                x[u] = i < rows ? P[i * k + j] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const long long i = i0 + u * step;
                const double mag = fabs(x[u]);
                if (i < rows && mag > best) {
                    best = mag;
                    arg = i;
                    val = x[u];
                }
            }
        }
    }
    bm[t] = best;
    bi[t] = arg;
    bv[t] = val;
    __syncthreads();
    if (t < k) {
        for (int q = 1; q < tpc; ++q) {
            const double m2 = bm[q * k + t];
            const long long i2 = bi[q * k + t];
            if (i2 >= 0 && (m2 > best || (m2 == best && (arg < 0 || i2 < arg)))) {
                best = m2;
                arg = i2;
                val = bv[q * k + t];
            }
        }
        pmag[(long long)blockIdx.x * k + t] = best;
        pidx_out[(long long)blockIdx.x * k + t] = arg;
        pval[(long long)blockIdx.x * k + t] = val;
    }
}

__global__ void k_colsign_final(int nparts, int k, const double* pmag, const long long* pidx_in,
                                const double* pval, double* sign) {
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        double best = -1.0, val = 0.0;
        long long arg = -1;
        for (int p = 0; p < nparts; ++p) {
            const double m2 = pmag[(long long)p * k + j];
            const long long i2 = pidx_in[(long long)p * k + j];
            if (i2 < 0) continue;
            if (m2 > best || (m2 == best && (arg < 0 || i2 < arg))) {
                best = m2;
                arg = i2;
                val = pval[(long long)p * k + j];
            }
        }
        sign[j] = (arg >= 0 && val < 0.0) ? -1.0 : 1.0;
    }
}

__global__ void k_colscale(long long rows, int k, double* P, const double* sign) {
    // thread (sub, j) flips column j over its rows only when sign_j < 0
    const int tpc = blockDim.x / k;
    const int t = threadIdx.x, j = t % k, sub = t / k;
    if (sub >= tpc || !(sign[j] < 0.0)) return;
    const long long step = (long long)gridDim.x * tpc;
    for (long long i = (long long)blockIdx.x * tpc + sub; i < rows; i += step) P[i * k + j] = -P[i * k + j];
}

// ----------------------------------------------------- smoothed aggregation --
// P = (I - omega D^-1 A) T (sa.hpp:78-109): row i starts at T(i, agg_i) and
// subtracts (omega / A_ii) a_ij T(j, agg_j) in the row's CSR order, contracted
// like the reference's default build (p(i, col) -= scaled * t(j, col)).
__global__ void k_sa_assemble(int n, int nc, const int* __restrict__ rp, const int* __restrict__ ci,
                              const double* __restrict__ v, const int* __restrict__ agg,
                              const double* __restrict__ tval, const double* __restrict__ diag,
                              double omega, double* __restrict__ P) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
         i += (long long)gridDim.x * blockDim.x) {
        double* row = P + i * nc;
        row[agg[i]] = tval[agg[i]];
        const double w = omega / diag[i];
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int col = agg[ci[k]];
            const double scaled = w * v[k];
            row[col] = fma(-scaled, tval[col], row[col]);
        }
    }
}

// ------------------------------------------------------- small k x k ops --
// Cholesky with the reference's symmetry gate (1e-10 max|a|) and pivot test
// (cholesky.hpp:15-37). rank_tol > 0 additionally flags pivots below it as
// rank deficiency (qr_thin's 1e-12 ||M||_F test on R_jj, qr.hpp:38-40), with
// rank_tol computed here from the trace when rank_rel > 0.
__global__ void __launch_bounds__(256) k_chol(int k, const double* __restrict__ A,
                                              double* __restrict__ L, double rank_rel,
                                              int* status) {
    __shared__ double red[256];
    __shared__ double djj;
    __shared__ int fail;
    const int tid = threadIdx.x, nt = blockDim.x;
    double mx = 0.0, tr = 0.0;
    for (int idx = tid; idx < k * k; idx += nt) {
        mx = fmax(mx, fabs(A[idx]));
        L[idx] = 0.0;
    }
    for (int i = tid; i < k; i += nt) tr += A[i * k + i];
    red[tid] = mx;
    __syncthreads();
    for (int s = nt / 2; s > 0; s >>= 1) {
        if (tid < s) red[tid] = fmax(red[tid], red[tid + s]);
        __syncthreads();
    }
    const double scale = red[0] > 0.0 ? red[0] : 1.0;
    __syncthreads();
    red[tid] = tr;
    __syncthreads();
    for (int s = nt / 2; s > 0; s >>= 1) {
        if (tid < s) red[tid] += red[tid + s];
        __syncthreads();
    }
    // rank_rel > 0: tolerance relative to sqrt(trace) (qr_thin); < 0: absolute
    // |rank_rel| on the pivots (orthonormalize_differentiable's 1e-10 norm test)
    const double rank_tol = rank_rel > 0.0 ? rank_rel * sqrt(fmax(red[0], 0.0)) : -rank_rel;
    if (tid == 0) fail = 0;
    __syncthreads();
    for (int idx = tid; idx < k * k; idx += nt) {
        const int i = idx / k, j = idx % k;
        if (j > i && fabs(A[i * k + j] - A[j * k + i]) > 1e-10 * scale) atomicOr(&fail, 1);
    }
    __syncthreads();
    if (fail) {
        if (tid == 0) *status = kErrNotSpd;
        return;
    }
    for (int j = 0; j < k; ++j) {
        if (tid == 0) {
            double d = A[j * k + j];
            for (int q = 0; q < j; ++q) d = fma(-L[j * k + q], L[j * k + q], d);
            if (d <= 0.0) {
                fail = rank_rel != 0.0 ? 2 : 1;
            } else {
                const double sd = sqrt(d);
                if (rank_rel != 0.0 && sd < rank_tol) fail = 2;
                djj = sd;
                L[j * k + j] = sd;
            }
        }
        __syncthreads();
        if (fail) break;
        const double lj = djj;
        for (int i = j + 1 + tid; i < k; i += nt) {
            double s = A[i * k + j];
            for (int q = 0; q < j; ++q) s = fma(-L[i * k + q], L[j * k + q], s);
            L[i * k + j] = s / lj;
        }
        __syncthreads();
    }
    if (tid == 0) *status = fail == 0 ? 0 : (fail == 2 ? kErrRank : kErrNotSpd);
}

// U = L^-T (upper triangular), column j of L^-1 by forward substitution
__global__ void k_tri_inv_lower_t(int k, const double* __restrict__ L, double* __restrict__ U) {
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < k; j += gridDim.x * blockDim.x) {
        // x = L^-1 e_j ; x_i = 0 for i < j
        for (int i = 0; i < k; ++i) {
            double xi;
            if (i < j) {
                xi = 0.0;
            } else {
                double s = (i == j) ? 1.0 : 0.0;
                for (int q = j; q < i; ++q) s = fma(-L[i * k + q], U[j * k + q], s);
                xi = s / L[i * k + i];
            }
            U[j * k + i] = xi;  // row j of U^T... U stored as (L^-1)^T: U[j][i] = (L^-1)[i][j]
        }
    }
}

// ---- wide k x k factorizations (k > 256, e.g. the SA coarse space) --------
// Same entrywise formulas as k_chol / k_tri_inv_lower_t, with the inner sums
// split across a warp: the Cholesky runs one launch per column (the column's
// rows in parallel across the grid), the triangular inverse a warp per column.
__global__ void __launch_bounds__(1024) k_chol_prep(int k, const double* __restrict__ A, double* __restrict__ L,
                                                    double rank_rel, double* tol, int* status) {
    __shared__ double red[32];
    __shared__ int fail;
    const int tid = threadIdx.x;
    double mx = 0.0, tr = 0.0;
    for (long long idx = tid; idx < (long long)k * k; idx += blockDim.x) {
        mx = fmax(mx, fabs(A[idx]));
        L[idx] = 0.0;
    }
    for (int i = tid; i < k; i += blockDim.x) tr += A[(long long)i * k + i];
    // block max / sum
    for (int o = 16; o; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        tr += __shfl_xor_sync(0xffffffffu, tr, o);
    }
    if (tid == 0) fail = 0;
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    double scale = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) scale = fmax(scale, red[w]);
    __syncthreads();
    if ((tid & 31) == 0) red[tid >> 5] = tr;
    __syncthreads();
    double trace = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) trace += red[w];
    scale = scale > 0.0 ? scale : 1.0;
    for (long long idx = tid; idx < (long long)k * k; idx += blockDim.x) {
        const long long i = idx / k, j = idx % k;
        if (j > i && fabs(A[i * k + j] - A[j * k + i]) > 1e-10 * scale) atomicOr(&fail, 1);
    }
    __syncthreads();
    if (tid == 0) {
        *tol = rank_rel > 0.0 ? rank_rel * sqrt(fmax(trace, 0.0)) : -rank_rel;
        *status = fail ? kErrNotSpd : 0;
    }
}

// column j: d = A_jj - sum_q L_jq^2 (every CTA, warp 0), then rows i > j
__global__ void __launch_bounds__(256) k_chol_col(int k, int j, const double* __restrict__ A,
                                                  double* __restrict__ L, double rank_rel,
                                                  const double* tol, int* status) {
    __shared__ double djj;
    __shared__ int bad;
    if (*status) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* lj = L + (long long)j * k;
    if (warp == 0) {
        double s = 0.0;
        for (int q = lane; q < j; q += 32) s = fma(lj[q], lj[q], s);
        s = warp_sum(s);
        if (lane == 0) {
            const double d = A[(long long)j * k + j] - s;
            bad = 0;
            if (d <= 0.0) {
                bad = rank_rel != 0.0 ? kErrRank : kErrNotSpd;
            } else {
                const double sd = sqrt(d);
                if (rank_rel != 0.0 && sd < *tol) bad = kErrRank;
                djj = sd;
            }
        }
    }
    __syncthreads();
    if (bad) {
        if (blockIdx.x == 0 && threadIdx.x == 0) *status = bad;
        return;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) L[(long long)j * k + j] = djj;
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (int i = j + 1 + blockIdx.x * (blockDim.x >> 5) + warp; i < k; i += warps) {
        const double* li = L + (long long)i * k;
        double s = 0.0;
        for (int q = lane; q < j; q += 32) s = fma(li[q], lj[q], s);
        s = warp_sum(s);
        if (lane == 0) L[(long long)i * k + j] = (A[(long long)i * k + j] - s) / djj;
    }
}

// U = (L^-1)^T, a warp per column j of L^-1 (row j of U): forward substitution
__global__ void __launch_bounds__(256) k_tri_inv_warp(int k, const double* __restrict__ L, double* __restrict__ U) {
    const int lane = threadIdx.x & 31;
    const int warps = gridDim.x * (blockDim.x >> 5);
    for (int j = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); j < k; j += warps) {
        double* u = U + (long long)j * k;
        for (int q = lane; q < j; q += 32) u[q] = 0.0;
        for (int i = j; i < k; ++i) {
            const double* li = L + (long long)i * k;
            double s = 0.0;
            for (int q = j + lane; q < i; q += 32) s = fma(li[q], u[q], s);
            s = warp_sum(s);
            if (lane == 0) u[i] = ((i == j ? 1.0 : 0.0) - s) / li[i];
            __syncwarp();
        }
    }
}

// A_c^-1 = L^-T L^-1 from U = (L^-1)^T: (A_c^-1)_ab = sum_{m >= max(a,b)} U_am U_bm
// (the coarse solve of the two-level cycle becomes one k x k mat-vec)
__global__ void k_coarse_inverse(int k, const double* __restrict__ U, double* __restrict__ Ainv) {
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < k * k; idx += gridDim.x * blockDim.x) {
        const int a = idx / k, b = idx % k;
        double s = 0.0;
        for (int m = max(a, b); m < k; ++m) s = fma(U[a * k + m], U[b * k + m], s);
        Ainv[idx] = s;
    }
}

// c_ij = c_ji = (c_ij + c_ji) / 2 (two_level.hpp:46-51)
__global__ void k_symmetrize(int k, double* C) {
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < k * k;
         idx += gridDim.x * blockDim.x) {
        const int i = idx / k, j = idx % k;
        if (i < j) {
            const double v = 0.5 * (C[i * k + j] + C[j * k + i]);
            C[i * k + j] = v;
            C[j * k + i] = v;
        }
    }
}

// S^(0) of a masked system: the stream's elements [e0, e0 + cnt) over the live
// rows (row live[e / m], column e % m) into S (generate_smoothed_vectors)
__global__ void k_s0_scatter(const double* __restrict__ src, long long e0, long long cnt, int m,
                             const int* __restrict__ live, double* __restrict__ S) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < cnt; t += (long long)gridDim.x * blockDim.x) {
        const long long e = e0 + t;
        S[(long long)live[e / m] * m + e % m] = src[t];
    }
}

// G += shift I (shifted CholeskyQR, nlsp_gpu.cu qr_thin_dev)
__global__ void k_shift_diag(int k, double* G, double shift) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < k; i += gridDim.x * blockDim.x)
        G[(long long)i * k + i] += shift;
}

// ---- column Gram-Schmidt on a row-major n x ld basis (svd.hpp:101-145) ----
// svd_oracle's rare branches: completing a numerically rank-deficient U
// (complete_orthonormal) and the polish when U^T U drifts past 1e-11
// (reorthonormalize_columns). One column at a time, as the reference does;
// every dot product is a fixed-order two-stage sum (deterministic).
// v is a separate n-vector; col < 0 selects v as the left operand.
__global__ void __launch_bounds__(256) k_coldot_partial(long long n, int ld, const double* __restrict__ U, int col,
                                                        const double* __restrict__ v, double* part) {
    __shared__ double red[256];
    double s = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double a = col >= 0 ? U[i * ld + col] : v[i];
        s = fma(a, v[i], s);
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int o = 128; o; o >>= 1) {
        if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}
// out[0] = sum of the partials; sqrt_out: out[0] = sqrt(sum)
__global__ void k_coldot_final(int nparts, const double* part, double* out, int sqrt_out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double s = 0.0;
        for (int p = 0; p < nparts; ++p) s += part[p];
        out[0] = sqrt_out ? sqrt(s) : s;
    }
}
// v -= c u_col  (c read on the device: no host round trip per projection)
__global__ void k_col_axpy(long long n, int ld, const double* __restrict__ U, int col, double* v,
                           const double* __restrict__ c) {
    const double cc = c[0];
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        v[i] -= cc * U[i * ld + col];
}
// v = u_col (get) or u_col = v / nrm (put); v = e_cand when col < 0
__global__ void k_col_move(long long n, int ld, double* U, int col, double* v, const double* nrm, int put,
                           long long cand) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        if (col < 0) v[i] = (i == cand) ? 1.0 : 0.0;
        else if (put) U[i * ld + col] = v[i] / nrm[0];
        else v[i] = U[i * ld + col];
    }
}
// Y (cols x rows) = X^T for a row-major rows x cols X (the wide-S Gram S S^T)
__global__ void k_transpose(long long rows, int cols, const double* __restrict__ X, double* __restrict__ Y) {
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < rows * cols;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long i = idx / cols, j = idx % cols;
        Y[j * rows + i] = X[idx];
    }
}

// sigma_i = sqrt(max(0, lambda_i <= floor ? 0 : lambda_i)), floor = 64 eps lambda_0
// (svd.hpp:174-179); W[:, :k] = V[:, :k]; flag if any sigma_j (j < k) <= 1e-13 sigma_0
__global__ void k_sigma(int m, int k, const double* evals, const double* evecs, double* sigma,
                        double* W, int* status) {
    __shared__ double smax;
    if (threadIdx.x == 0) {
        const double fl = evals[0] * 64.0 * DBL_EPSILON;
        for (int i = 0; i < m; ++i) {
            const double lam = evals[i] <= fl ? 0.0 : evals[i];
            sigma[i] = sqrt(fmax(0.0, lam));
        }
        smax = sigma[0];
        // solid: the leading sigma_j above the cutoff 1e-13 sigma_max (svd.hpp:185-200);
        // U's later columns come from complete_orthonormal instead
        int solid = 0;
        while (solid < k && sigma[solid] > smax * 1e-13) ++solid;
        *status = solid;
    }
    __syncthreads();
    for (int idx = threadIdx.x; idx < m * k; idx += blockDim.x) {
        const int l = idx / k, j = idx % k;
        W[idx] = evecs[l * m + j];
    }
}

// =========================================================== launchers ==

namespace {
inline void count(const LaunchCtx& c) { ++*c.launches; }
int grid_for(const LaunchCtx& c, long long work, int threads, int per_sm = 4) {
    long long g = (work + threads - 1) / threads;
    const long long cap = (long long)c.num_sms * per_sm;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return static_cast<int>(g);
}
}  // namespace

void launch_csr_import(const LaunchCtx& c, int n, long long nnz, const unsigned long long* rp64,
                       const unsigned long long* ci64, const double* v, int* rp, int* ci,
                       double* diag, int* flags, int* max_row) {
    k_csr_import<<<grid_for(c, n, 256, 8), 256, 0, c.s>>>(n, nnz, rp64, ci64, v, rp, ci, diag,
                                                          flags, max_row);
    count(c);
}

void launch_wd(const LaunchCtx& c, int n, const double* diag, double omega, double* wd, int* flag) {
    k_wd<<<grid_for(c, n, 256), 256, 0, c.s>>>(n, diag, omega, wd, flag);
    count(c);
}

// mode 0: sweep, 1: plain product
void launch_block_op(const LaunchCtx& c, int mode, int n, const int* rp, const int* ci,
                     const double* v, const double* wd, int m, const double* in, double* out) {
    const int g = grid_for(c, (long long)n * 32, 256, 8);
#define NLSP_BS(L, T)                                                                         \
    do {                                                                                      \
        if (mode == 0) k_block_sweep<L, T, 0><<<g, 256, 0, c.s>>>(n, rp, ci, v, wd, m, in, out); \
        else k_block_sweep<L, T, 1><<<g, 256, 0, c.s>>>(n, rp, ci, v, wd, m, in, out);        \
    } while (0)
    if (m <= 8) NLSP_BS(8, 1);
    else if (m <= 16) NLSP_BS(16, 1);
    else if (m <= 32) NLSP_BS(32, 1);
    else if (m <= 64) NLSP_BS(32, 2);
    else if (m <= 96) NLSP_BS(32, 3);
    else NLSP_BS(32, 4);
#undef NLSP_BS
    count(c);
}

// the diagonal-form block sweep for the exact 5/7/9-offset forms and m > 16;
// false: not applicable (the caller uses the CSR kernel)
bool launch_block_op_dia(const LaunchCtx& c, int mode, int n, const DiaArgs& dia, const double* wd, int m,
                         const double* in, double* out) {
    static const bool on = !(std::getenv("NLSP_BSWEEP_DIA") && std::atoi(std::getenv("NLSP_BSWEEP_DIA")) == 0);
    // measured at C4: 26.8 -> 38.4 ms for the 10 sweeps with the hints, so
    // they stay off unless NLSP_BSWEEP_HINT=1
    static const bool hint = std::getenv("NLSP_BSWEEP_HINT") && std::atoi(std::getenv("NLSP_BSWEEP_HINT")) == 1;
    // measured: faster than the CSR kernel for constant coefficients and wide
    // blocks (C4 smoothing, m = 128: 3.66 -> 2.68 ms per sweep; C3, m = 96:
    // -10 %), slower for per-row values (C2 +57 %) and m <= 64 (the builds, +9 %)
    if (!on || dia.kind != 1 || m <= 64 || m > 128 || !(dia.d == 5 || dia.d == 7 || dia.d == 9)) return false;
    const int g = grid_for(c, (long long)n * 32, 256, 8);
#define NLSP_BD(D, T)                                                                                   \
    do {                                                                                                \
        if (mode == 0 && hint) k_block_sweep_dia<D, T, 0, true><<<g, 256, 0, c.s>>>(n, dia, wd, m, in, out); \
        else if (mode == 0) k_block_sweep_dia<D, T, 0, false><<<g, 256, 0, c.s>>>(n, dia, wd, m, in, out); \
        else k_block_sweep_dia<D, T, 1, false><<<g, 256, 0, c.s>>>(n, dia, wd, m, in, out);             \
    } while (0)
#define NLSP_BDT(D)                  \
    do {                             \
        if (m <= 32) NLSP_BD(D, 1);  \
        else if (m <= 64) NLSP_BD(D, 2); \
        else if (m <= 96) NLSP_BD(D, 3); \
        else NLSP_BD(D, 4);          \
    } while (0)
    if (dia.d == 5) NLSP_BDT(5);
    else if (dia.d == 7) NLSP_BDT(7);
    else NLSP_BDT(9);
#undef NLSP_BDT
#undef NLSP_BD
    count(c);
    return true;
}

// C (ca x cb) = X^T Y; part must hold grid * ca * cb doubles (grid <= kMaxGrid)
bool launch_gram_dmma(cudaStream_t s, int g, long long rows, int bi, int bj, int lda, int ldb,
                      const double* X, const double* Y, double* part);
bool launch_dense_mm_dmma(cudaStream_t s, int num_sms, long long rows, int m, int kout, const double* X,
                          const double* W, const double* sigma, double* Y);

// FP64 tensor-pipe (DMMA) contractions unless NLSP_DMMA=0 (then the
// register-tiled FFMA kernels below)
static bool use_dmma() {
    static const bool on = [] {
        const char* e = std::getenv("NLSP_DMMA");
        return !(e && e[0] == '0');
    }();
    return on;
}

int gram_grid(const LaunchCtx& c, long long rows) {
    // at least 256 rows per CTA: fewer partials to reduce for short, wide Grams
    long long g = (rows + 255) / 256;
    const long long cap = (long long)c.num_sms * 2;
    if (g > cap) g = cap;
    if (g < 1) g = 1;
    return static_cast<int>(g);
}

// C (ca x cb) = X^T Y in register tiles of at most 128 x 128 columns; part must
// hold gram_grid(rows) * min(ca,128) * min(cb,128) doubles
void launch_gram(const LaunchCtx& c, long long rows, int ca, int cb, const double* X,
                 const double* Y, double* part, double* C) {
    const int g = gram_grid(c, rows);
    for (int i0 = 0; i0 < ca; i0 += 128)
        for (int j0 = 0; j0 < cb; j0 += 128) {
            const int bi = ca - i0 < 128 ? ca - i0 : 128, bj = cb - j0 < 128 ? cb - j0 : 128;
            if (use_dmma() &&
                launch_gram_dmma(c.s, g, rows, bi, bj, ca, cb, X + i0, Y + j0, part)) {
                count(c);
                k_gram_reduce<<<grid_for(c, (long long)bi * bj, 256), 256, 0, c.s>>>(
                    g, bi, bj, part, C + (long long)i0 * cb + j0, cb);
                count(c);
                continue;
            }
            const int w = bi > bj ? bi : bj;
            const int ti = (w + 15) / 16;
#define NLSP_G(T)                                                                              \
    do {                                                                                       \
        const size_t smem = 2 * 16 * 16 * (T) * sizeof(double);                                \
        k_gram_partial<T><<<g, 256, smem, c.s>>>(rows, bi, bj, ca, cb, X + i0, Y + j0, part);  \
    } while (0)
            switch (ti) {
                case 1: NLSP_G(1); break;
                case 2: NLSP_G(2); break;
                case 3: NLSP_G(3); break;
                case 4: NLSP_G(4); break;
                case 5: NLSP_G(5); break;
                case 6: NLSP_G(6); break;
                case 7: NLSP_G(7); break;
                default: NLSP_G(8); break;
            }
#undef NLSP_G
            count(c);
            k_gram_reduce<<<grid_for(c, (long long)bi * bj, 256), 256, 0, c.s>>>(g, bi, bj, part,
                                                                                  C + (long long)i0 * cb + j0, cb);
            count(c);
        }
}

void launch_eigh(const LaunchCtx& c, int m, const double* g, double* evals, double* evecs,
                 double* scratch_a, double* scratch_v, int* status, int* sweeps) {
    EighArgs a{m, scratch_a, scratch_v, g, evals, evecs, status, sweeps};
    const size_t need = (size_t)(m * (m + 1) / 2 + m * m) * sizeof(double);
    const int use_shared = need <= 200 * 1024;
    if (use_shared) {
        cudaFuncSetAttribute(k_eigh, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)need);
        k_eigh<<<1, 1024, need, c.s>>>(a, 1);
    } else {
        k_eigh<<<1, 1024, 0, c.s>>>(a, 0);
    }
    count(c);
}

void launch_dense_mm(const LaunchCtx& c, long long rows, int m, int kout, const double* X,
                     const double* W, const double* sigma, double* Y) {
    if (use_dmma() && launch_dense_mm_dmma(c.s, c.num_sms, rows, m, kout, X, W, sigma, Y)) {
        count(c);
        return;
    }
    const size_t wbytes = (size_t)m * kout * sizeof(double);
    const int use_shared = wbytes <= 96 * 1024;
    const int g = grid_for(c, rows * 32, 256, 8);
#define NLSP_MM(T)                                                                          \
    do {                                                                                    \
        if (use_shared) {                                                                   \
            cudaFuncSetAttribute(k_dense_mm<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                 (int)wbytes);                                              \
            k_dense_mm<T><<<g, 256, wbytes, c.s>>>(rows, m, kout, X, W, sigma, Y, 1);       \
        } else {                                                                            \
            k_dense_mm<T><<<g, 256, 0, c.s>>>(rows, m, kout, X, W, sigma, Y, 0);            \
        }                                                                                   \
    } while (0)
    const int t = (kout + 31) / 32;
    if (t <= 1) NLSP_MM(1);
    else if (t == 2) NLSP_MM(2);
    else if (t <= 4) NLSP_MM(4);
    else NLSP_MM(8);
#undef NLSP_MM
    count(c);
}

void launch_colsign(const LaunchCtx& c, long long rows, int k, double* P, double* pmag,
                    long long* pidx_buf, double* pval, double* sign) {
    const int g = grid_for(c, rows, 256, kColsignPerSm);  // pmag / pidx / pval: num_sms * 8 * k
    const size_t smem = 256 * (sizeof(double) * 2 + sizeof(long long));
    k_colmax_partial<<<g, 256, smem, c.s>>>(rows, k, P, pmag, pidx_buf, pval);
    count(c);
    k_colsign_final<<<1, 256, 0, c.s>>>(g, k, pmag, pidx_buf, pval, sign);
    count(c);
    k_colscale<<<grid_for(c, rows, 256 / k, 8), 256, 0, c.s>>>(rows, k, P, sign);
    count(c);
}

void launch_sa_assemble(const LaunchCtx& c, int n, int nc, const int* rp, const int* ci, const double* v,
                        const int* agg, const double* tval, const double* diag, double omega, double* P) {
    k_sa_assemble<<<grid_for(c, n, 128), 128, 0, c.s>>>(n, nc, rp, ci, v, agg, tval, diag, omega, P);
    count(c);
}

void launch_chol(const LaunchCtx& c, int k, const double* A, double* L, double rank_rel,
                 int* status) {
    if (k <= 256) {
        k_chol<<<1, 256, 0, c.s>>>(k, A, L, rank_rel, status);
        count(c);
        return;
    }
    // wide: one launch per column; the rank tolerance sits just past the
    // factor (callers allocate L with k*k + 8 doubles for k > 256)
    double* tol = L + (long long)k * k;
    k_chol_prep<<<1, 1024, 0, c.s>>>(k, A, L, rank_rel, tol, status);
    count(c);
    const int grid = (k + 63) / 64;  // 8 warps per CTA, ~8 rows per warp
    for (int j = 0; j < k; ++j) {
        k_chol_col<<<grid, 256, 0, c.s>>>(k, j, A, L, rank_rel, tol, status);
        count(c);
    }
}

void launch_tri_inv_t(const LaunchCtx& c, int k, const double* L, double* U) {
    if (k <= 256) k_tri_inv_lower_t<<<(k + 127) / 128, 128, 0, c.s>>>(k, L, U);
    else k_tri_inv_warp<<<(k + 7) / 8, 256, 0, c.s>>>(k, L, U);
    count(c);
}

void launch_coarse_inverse(const LaunchCtx& c, int k, const double* U, double* Ainv) {
    k_coarse_inverse<<<(k * k + 255) / 256, 256, 0, c.s>>>(k, U, Ainv);
    count(c);
}

// dot / norm of columns (k_coldot_*): out[0] = u_col . v (col >= 0) or
// sqrt(v . v) (col < 0); part holds num_sms * 2 partials
void launch_coldot(const LaunchCtx& c, long long n, int ld, const double* U, int col, const double* v, double* part,
                   double* out) {
    const int g = grid_for(c, n, 256, 2);
    k_coldot_partial<<<g, 256, 0, c.s>>>(n, ld, U, col, v, part);
    k_coldot_final<<<1, 32, 0, c.s>>>(g, part, out, col < 0 ? 1 : 0);
    count(c);
    count(c);
}
void launch_col_axpy(const LaunchCtx& c, long long n, int ld, const double* U, int col, double* v, const double* cc) {
    k_col_axpy<<<grid_for(c, n, 256), 256, 0, c.s>>>(n, ld, U, col, v, cc);
    count(c);
}
void launch_col_move(const LaunchCtx& c, long long n, int ld, double* U, int col, double* v, const double* nrm,
                     int put, long long cand) {
    k_col_move<<<grid_for(c, n, 256), 256, 0, c.s>>>(n, ld, U, col, v, nrm, put, cand);
    count(c);
}
void launch_transpose(const LaunchCtx& c, long long rows, int cols, const double* X, double* Y) {
    k_transpose<<<grid_for(c, rows * cols, 256), 256, 0, c.s>>>(rows, cols, X, Y);
    count(c);
}

void launch_s0_scatter(const LaunchCtx& c, const double* src, long long e0, long long cnt, int m, const int* live,
                       double* S) {
    k_s0_scatter<<<grid_for(c, cnt, 256), 256, 0, c.s>>>(src, e0, cnt, m, live, S);
    count(c);
}

void launch_shift_diag(const LaunchCtx& c, int k, double* G, double shift) {
    k_shift_diag<<<(k + 255) / 256, 256, 0, c.s>>>(k, G, shift);
    count(c);
}

void launch_symmetrize(const LaunchCtx& c, int k, double* C) {
    k_symmetrize<<<(k * k + 255) / 256, 256, 0, c.s>>>(k, C);
    count(c);
}

void launch_sigma(const LaunchCtx& c, int m, int k, const double* evals, const double* evecs,
                  double* sigma, double* W, int* status) {
    k_sigma<<<1, 256, 0, c.s>>>(m, k, evals, evecs, sigma, W, status);
    count(c);
}

}  // namespace nlsp
