// paper_2601_20174_b200/csrc/cluster_solve.cu — the whole PCG solve of a small
// system in ONE launch of one thread-block cluster.
//
// Systems of a few thousand unknowns (config C1, the paper's N = 64 FEM
// setting) are launch- and latency-bound on the multi-kernel path: each PCG
// iteration is 4 dependent grid-wide kernels of a few microseconds. Here a
// cluster of up to 16 CTAs keeps the system on chip for the entire solve:
// CTA q owns rows [q R, q R + R) and holds, in shared memory, their matrix rows
// as a column-major ELL slice, their rows of the folded bases W1 / W2
// (two_level cycle) column-major, omega D^-1, b and every PCG
// vector. Each ELL entry stores the shared::cluster ADDRESS of its column's
// slot (owner CTA, local row) instead of the column index, so a gather x[col]
// of any vector is one `ld.shared::cluster` at (entry + the vector's offset) —
// local or remote (DSMEM) alike, no division, no branch. Every dot product /
// the restriction is a cluster all-reduce (each CTA pushes its partial into
// every CTA's slot, one cluster barrier, each CTA sums the slots in rank order
// — deterministic and identical in every CTA). Three cluster barriers per PCG
// iteration for nu1 + nu2 = 2: (p.Ap), (||r||^2 with W1^T r fused), (r.z).
//
// Arithmetic is that of the folded multi-kernel path (same per-row summation
// order of A x, same sweeps, the same coarse solve: A_c^-1 c as one k x k
// mat-vec, or the triangular substitutions with NLSP_COARSE=chol); only the
// reduction order differs.
#include <cooperative_groups.h>

#include <algorithm>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace nlsp {

constexpr int kClusterThreads = 512;
constexpr int kClusterWarps = kClusterThreads / 32;
constexpr int kMaxClusterCtas = 16;
constexpr int kInvMax = 64;  // coarse inverse held in shared memory up to this k

// shared-memory layout (identical in every CTA of the cluster)
struct ClusterLayout {
    unsigned ea, ev_, wd, b, x, r, p0, p1, q, z, s0, s1, w1, w2, red, e, tot, wsum, Lm, Ai, bytes;
    __host__ __device__ ClusterLayout(int R, int W, int ld, int k, bool two_w, int ncta) {
        unsigned o = 0;
        auto take = [&](unsigned bytes) {
            const unsigned at = o;
            o += (bytes + 15u) & ~15u;
            return at;
        };
        ev_ = take(W * R * 8);  // ELL values [W][R]
        ea = take(W * R * 4);   // ELL shared::cluster addresses [W][R]
        wd = take(R * 8);
        b = take(R * 8);
        x = take(R * 8);
        r = take(R * 8);
        p0 = take(R * 8);
        p1 = take(R * 8);
        q = take(R * 8);
        z = take(R * 8);
        s0 = take(R * 8);
        s1 = take(R * 8);
        w1 = take(R * ld * 8);  // [ld][R]
        w2 = two_w ? take(R * ld * 8) : w1;
        red = take(2 * ncta * (ld + 4) * 8);  // double-buffered all-reduce slots
        e = take((ld + 4) * 8);
        tot = take((ld + 4) * 8);
        wsum = take(kClusterWarps * (ld + 4) * 8);
        Lm = take(k * k * 8);  // L, or A_c^-1 for k <= kInvMax
        Ai = Lm;
        bytes = o;
    }
};

namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ unsigned mapa_u32(unsigned a, unsigned rank) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
// volatile keeps these in program order relative to the cluster barriers;
// independent loads still overlap in flight
__device__ __forceinline__ double ld_dsm(unsigned a) {
    double v;
    asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void st_dsm(unsigned a, double v) {
    asm volatile("st.shared::cluster.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// sum_s v[s][i] * f(gather(s, i)) over the ELL row, in CSR order (padding
// entries carry value 0 and point at a valid local slot)
template <int NG, class F>
__device__ __forceinline__ double ell_row(const unsigned* ea, const double* ev, int W, int R, int i,
                                          unsigned off0, unsigned off1, const F& f) {
    double s = 0.0;
#pragma unroll 4
    for (int t = 0; t < W; ++t) {
        const unsigned a = ea[t * R + i];
        const double g0 = ld_dsm(a + off0);
        const double g1 = NG == 2 ? ld_dsm(a + off1) : 0.0;
        s = fma(ev[t * R + i], f(g0, g1), s);
    }
    return s;
}

}  // namespace

__device__ __forceinline__ void cluster_pcg_body(const ClusterArgs& a) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ double wsc[kClusterWarps];
    const int ncta = (int)cl.num_blocks();
    const int q = (int)cl.block_rank();
    const int R = a.rows, ld = a.ld, k = a.k, W = a.width;
    const int row0 = q * R;
    const int nr = max(0, min(R, a.n - row0));
    const ClusterLayout Lo(R, W, ld, k, a.W2 != a.W1, ncta);
    const unsigned base = smem_u32(sm);
    auto D = [&](unsigned off) { return reinterpret_cast<double*>(sm + off); };
    unsigned* ea = reinterpret_cast<unsigned*>(sm + Lo.ea);
    double* ev = D(Lo.ev_);
    double *wd = D(Lo.wd), *bv = D(Lo.b), *xv = D(Lo.x), *rv = D(Lo.r), *qv = D(Lo.q), *zv = D(Lo.z);
    double* pv[2] = {D(Lo.p0), D(Lo.p1)};
    double* sv[2] = {D(Lo.s0), D(Lo.s1)};
    double *w1 = D(Lo.w1), *w2 = D(Lo.w2), *red = D(Lo.red), *ec = D(Lo.e), *tot = D(Lo.tot);
    double *wsum = D(Lo.wsum), *Lm = D(Lo.Lm), *Ai = D(Lo.Ai);
    const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
    const int nw = nt >> 5;
    PcgState* st = a.st;

    // ---- load the CTA's slice of the system into shared memory
    const unsigned pad = mapa_u32(base, (unsigned)q);  // a valid local slot
    for (int idx = tid; idx < W * R; idx += nt) {
        const int t = idx / R, i = idx - t * R;
        unsigned ad = pad;
        double v = 0.0;
        if (i < nr) {
            const int k0 = a.rp[row0 + i], k1 = a.rp[row0 + i + 1];
            if (k0 + t < k1) {
                const int col = a.ci[k0 + t];
                const int o = col / R;
                ad = mapa_u32(base, (unsigned)o) + (unsigned)(col - o * R) * 8u;
                v = a.v[k0 + t];
            }
        }
        ea[idx] = ad;
        ev[idx] = v;
    }
    for (int i = tid; i < R; i += nt) {
        const bool own = i < nr;
        wd[i] = own ? a.wd[row0 + i] : 0.0;
        bv[i] = own ? a.b[row0 + i] : 0.0;
        xv[i] = 0.0;
        rv[i] = bv[i];
        pv[0][i] = pv[1][i] = qv[i] = zv[i] = sv[0][i] = sv[1][i] = 0.0;
    }
    for (int idx = tid; idx < R * ld; idx += nt) {
        const int i = idx / ld, j = idx - i * ld;
        const bool own = i < nr;
        w1[j * R + i] = own ? a.W1[(long long)(row0 + i) * ld + j] : 0.0;
        if (a.W2 != a.W1) w2[j * R + i] = own ? a.W2[(long long)(row0 + i) * ld + j] : 0.0;
    }
    const bool inv = a.Ainv != nullptr && k <= kInvMax;
    for (int i = tid; i < k * k; i += nt) {
        if (inv) Ai[i] = a.Ainv[i];
        else Lm[i] = a.L[i];
    }
    const int stride = ld + 4;
    int rbuf = 0;
    cl.sync();  // every CTA's slice is resident before any DSMEM access

    // scalar all-reduce of a per-thread value; every thread gets the sum
    auto reduce_scalar = [&](double v) -> double {
        v = warp_sum(v);
        if (lane == 0) wsc[warp] = v;
        __syncthreads();
        double* slot0 = red + (size_t)rbuf * ncta * stride;
        if (tid < ncta) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += wsc[w];
            st_dsm(mapa_u32(smem_u32(slot0 + q * stride), (unsigned)tid), t);
        }
        cl.sync();
        double t = 0.0;
        for (int c = 0; c < ncta; ++c) t += slot0[c * stride];
        rbuf ^= 1;
        return t;
    };

    // ||r||^2 and c = W1^T r (own rows) in one all-reduce, then the coarse
    // solve e = (L L^T)^-1 c into ec (two_level.hpp:98-115); returns ||r||^2
    auto restrict_solve = [&](double rr) -> double {
        const int cnt = ld + 1;
        for (int j0 = 0; j0 < ld; j0 += 8) {
            double acc[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) acc[u] = 0.0;
            for (int i = tid; i < nr; i += nt) {
                const double ri = rv[i];
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    if (j0 + u < ld) acc[u] = fma(w1[(j0 + u) * R + i], ri, acc[u]);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const double t = warp_sum(acc[u]);
                if (lane == 0 && j0 + u < ld) wsum[warp * stride + j0 + u] = t;
            }
        }
        rr = warp_sum(rr);
        if (lane == 0) wsum[warp * stride + ld] = rr;
        __syncthreads();
        double* slot0 = red + (size_t)rbuf * ncta * stride;
        if (tid < cnt) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += wsum[w * stride + tid];
            const unsigned my = smem_u32(slot0 + q * stride + tid);
            for (int dst = 0; dst < ncta; ++dst) st_dsm(mapa_u32(my, (unsigned)dst), t);
        }
        cl.sync();
        if (tid < cnt) {
            double t = 0.0;
            for (int c = 0; c < ncta; ++c) t += slot0[c * stride + tid];
            tot[tid] = t;
        }
        rbuf ^= 1;
        __syncthreads();
        if (inv) {
            if (tid < k) {
                double s = 0.0;
                for (int j = 0; j < k; ++j) s = fma(Ai[tid * k + j], tot[j], s);
                ec[tid] = s;
            }
        } else if (tid < 32) {
            // L y = c, L^T e = y (cholesky.hpp:41-57) by warp 0
            for (int i = tid; i < k; i += 32) ec[i] = tot[i];
            for (int j = 0; j < k; ++j) {
                __syncwarp();
                const double yj = ec[j] / Lm[j * k + j];
                __syncwarp();
                if (tid == 0) ec[j] = yj;
                for (int i = j + 1 + tid; i < k; i += 32) ec[i] = fma(-Lm[i * k + j], yj, ec[i]);
            }
            for (int j = k - 1; j >= 0; --j) {
                __syncwarp();
                const double xj = ec[j] / Lm[j * k + j];
                __syncwarp();
                if (tid == 0) ec[j] = xj;
                for (int i = tid; i < j; i += 32) ec[i] = fma(-Lm[j * k + i], xj, ec[i]);
            }
        }
        if (tid == 0 && (k & 1)) ec[k] = 0.0;
        const double rr_tot = tot[ld];
        __syncthreads();
        return rr_tot;
    };

    // z = S_T(r) + W2 e (folded cycle tail); returns r.z (all-reduced). The
    // sweep outputs are published by a barrier only when another sweep gathers
    // them; z itself by the r.z all-reduce.
    auto tail = [&]() -> double {
        const int T = a.nu1 + a.nu2;
        double* cur = nullptr;  // s_1 = w D^-1 r implicit
        int cb = 0;
        for (int j = 2; j <= T; ++j) {
            double* nxt = sv[cb];
            for (int i = tid; i < nr; i += nt) {
                double y;
                if (cur == nullptr)
                    y = ell_row<2>(ea, ev, W, R, i, Lo.wd, Lo.r,
                                   [](double g0, double g1) { return g0 * g1; });
                else
                    y = ell_row<1>(ea, ev, W, R, i, (unsigned)((unsigned char*)cur - sm), 0u,
                                   [](double g0, double) { return g0; });
                const double si = cur == nullptr ? wd[i] * rv[i] : cur[i];
                nxt[i] = fma(wd[i], rv[i] - y, si);
            }
            if (j < T) cl.sync();  // the next sweep gathers this one's output
            cur = nxt;
            cb ^= 1;
        }
        double rz = 0.0;
        for (int i = tid; i < nr; i += nt) {
            double s = 0.0;
            for (int j = 0; j < ld; ++j) s = fma(w2[j * R + i], ec[j], s);
            const double zp = T == 0 ? 0.0 : (cur == nullptr ? wd[i] * rv[i] : cur[i]);
            const double zi = zp + s;
            zv[i] = zi;
            rz = fma(rv[i], zi, rz);
        }
        return reduce_scalar(rz);
    };

    // ---- prologue: ||b|| (fused with W1^T b), z = M b, rz (two_level.hpp:143-156)
    double bb = 0.0;
    for (int i = tid; i < nr; i += nt) bb = fma(bv[i], bv[i], bb);
    const double bnorm = sqrt(restrict_solve(bb));
    if (bnorm == 0.0) {
        if (q == 0 && tid == 0) {
            st->error = kErrValidation;
            st->done = 1;
        }
        cl.sync();
        return;
    }
    double rz = tail();
    const long long max_it = st->max_it;
    const double delta = st->delta;
    double beta = 0.0;
    long long it = 0;
    int converged = 0, err = 0;
    double last_rel = 0.0;
    for (; it < max_it; ++it) {
        double* pc = pv[it & 1];
        double* pp = pv[(it + 1) & 1];
        // p = z + beta p (gathered on the fly), q = A p, p.q (:159-163)
        double pap_part = 0.0;
        for (int i = tid; i < nr; i += nt) {
            double y, pi;
            if (it == 0) {
                y = ell_row<1>(ea, ev, W, R, i, Lo.z, 0u, [](double g0, double) { return g0; });
                pi = zv[i];
            } else {
                const unsigned opp = (unsigned)((unsigned char*)pp - sm);
                y = ell_row<2>(ea, ev, W, R, i, Lo.z, opp,
                               [beta](double g0, double g1) { return fma(beta, g1, g0); });
                pi = fma(beta, pp[i], zv[i]);
            }
            pc[i] = pi;
            qv[i] = y;
            pap_part = fma(pi, y, pap_part);
        }
        const double pap = reduce_scalar(pap_part);
        if (pap <= 0.0) {
            err = kErrNotSpd;
            break;
        }
        const double alpha = rz / pap;
        // x += alpha p, r -= alpha q, ||r|| (:164-176) fused with W1^T r and
        // the coarse solve of the next preconditioner application
        double rr = 0.0;
        for (int i = tid; i < nr; i += nt) {
            xv[i] = fma(alpha, pc[i], xv[i]);
            const double ri = fma(-alpha, qv[i], rv[i]);
            rv[i] = ri;
            rr = fma(ri, ri, rr);
        }
        const double rel = sqrt(restrict_solve(rr)) / bnorm;
        last_rel = rel;
        if (q == 0 && tid == 0 && a.hist && it < a.hist_cap) a.hist[it] = rel;
        if (rel < delta) {
            converged = 1;
            ++it;
            break;
        }
        // z = M r (folded cycle), beta = rz' / rz (:177-182)
        const double rz_new = tail();
        beta = rz_new / rz;
        rz = rz_new;
    }
    // true residual ||b - A x|| / ||b|| (:185-189)
    cl.sync();
    double tr = 0.0;
    for (int i = tid; i < nr; i += nt) {
        const double y = ell_row<1>(ea, ev, W, R, i, Lo.x, 0u, [](double g0, double) { return g0; });
        const double d = bv[i] - y;
        tr = fma(d, d, tr);
    }
    const double true_res = sqrt(reduce_scalar(tr)) / bnorm;
    for (int i = tid; i < nr; i += nt) a.x[row0 + i] = xv[i];
    if (q == 0 && tid == 0) {
        st->iterations = it;
        st->converged = converged;
        st->error = err;
        st->done = 1;
        st->bnorm = bnorm;
        st->true_res = err ? 0.0 : true_res;
        st->last_rel = last_rel;
        st->body_runs = it;
    }
    cl.sync();  // no CTA exits while others may still read its shared memory
}

__global__ void __launch_bounds__(kClusterThreads, 1) k_cluster_pcg(ClusterArgs a) { cluster_pcg_body(a); }

// Independent systems in ONE launch, one cluster each (nlsp_pcg_batch): the
// cluster index selects the system's arguments.
__global__ void __launch_bounds__(kClusterThreads, 1) k_cluster_pcg_batch(const ClusterArgs* __restrict__ args) {
    cg::cluster_group cl = cg::this_cluster();
    const ClusterArgs a = args[blockIdx.x / cl.num_blocks()];
    cluster_pcg_body(a);
}

// Cluster size and rows per CTA for an n x n system with rows of at most
// `width` nonzeros, or 0 when the slices do not fit in shared memory. Prefers
// the smallest cluster whose CTAs hold at most one row per thread.
int cluster_plan(int n, int k, int width, bool two_w, int* rows_out, size_t* smem_out) {
    const int ld = k + (k & 1);
    if (k > 256 || n < 1) return 0;
    int best = 0;
    for (int ncta = 1; ncta <= kMaxClusterCtas; ncta *= 2) {
        const int R = (n + ncta - 1) / ncta;
        const ClusterLayout Lo(R, std::max(width, 1), ld, k, two_w, ncta);
        if (Lo.bytes > 200 * 1024) continue;
        if (!best) {
            best = ncta;
            *rows_out = R;
            *smem_out = Lo.bytes;
        }
        if (R <= kClusterThreads) {
            *rows_out = R;
            *smem_out = Lo.bytes;
            return ncta;
        }
    }
    return best;
}

cudaError_t launch_cluster_pcg(cudaStream_t s, const ClusterArgs& a, int ncta, size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(k_cluster_pcg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e) return e;
    e = cudaFuncSetAttribute(k_cluster_pcg, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(ncta);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ncta;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    e = cudaOccupancyMaxActiveClusters(&nclusters, k_cluster_pcg, &cfg);
    if (e || nclusters < 1) return e ? e : cudaErrorInvalidConfiguration;
    return cudaLaunchKernelEx(&cfg, k_cluster_pcg, a);
}

// Common cluster size for a batch: the largest any system needs, each
// system's rows re-split over it; returns 0 if any system does not fit.
int cluster_plan_batch(int count, const int* n, const int* k, const int* width, const bool* two_w, int* rows,
                       size_t* smem_out) {
    // the smallest cluster each system fits in: many systems share the SMs,
    // so fewer SMs per system beat fewer rows per thread
    int ncta = 1;
    for (int i = 0; i < count; ++i) {
        int c = 0;
        for (int t = 1; t <= kMaxClusterCtas && !c; t *= 2) {
            const int R = (n[i] + t - 1) / t;
            if (ClusterLayout(R, std::max(width[i], 1), k[i] + (k[i] & 1), k[i], two_w[i], t).bytes <= 200 * 1024)
                c = t;
        }
        if (!c || k[i] > 256) return 0;
        ncta = std::max(ncta, c);
    }
    size_t smem = 0;
    for (int i = 0; i < count; ++i) {
        rows[i] = (n[i] + ncta - 1) / ncta;
        const ClusterLayout Lo(rows[i], std::max(width[i], 1), k[i] + (k[i] & 1), k[i], two_w[i], ncta);
        if (Lo.bytes > 200 * 1024) return 0;
        smem = std::max<size_t>(smem, Lo.bytes);
    }
    *smem_out = smem;
    return ncta;
}

cudaError_t launch_cluster_pcg_batch(cudaStream_t s, const ClusterArgs* dargs, int count, int ncta, size_t smem) {
    cudaError_t e = cudaFuncSetAttribute(k_cluster_pcg_batch, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    if (e) return e;
    e = cudaFuncSetAttribute(k_cluster_pcg_batch, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e) return e;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(count * ncta);
    cfg.blockDim = dim3(kClusterThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = ncta;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    e = cudaOccupancyMaxActiveClusters(&nclusters, k_cluster_pcg_batch, &cfg);
    if (e || nclusters < 1) return e ? e : cudaErrorInvalidConfiguration;
    return cudaLaunchKernelEx(&cfg, k_cluster_pcg_batch, dargs);
}

}  // namespace nlsp
