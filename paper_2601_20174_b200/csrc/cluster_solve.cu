// paper_2601_20174_b200/csrc/cluster_solve.cu — the whole PCG solve of a small
// system in ONE launch of one thread-block cluster.
//
// Systems of a few thousand unknowns (config C1, the paper's N = 64 FEM
// setting) are launch- and latency-bound on the multi-kernel path: each PCG
// iteration is 4 dependent grid-wide kernels of a few microseconds. Here a
// cluster of up to 16 CTAs keeps the system on chip for the entire solve:
// CTA q owns rows [q R, q R + R) and holds their CSR slice, their rows of the
// folded bases W1 / W2 (two_level cycle), omega D^-1, b and every
// PCG vector in shared memory. Gathers x[col] of other CTAs' rows are
// distributed-shared-memory (DSMEM) loads; every dot product / the restriction
// is a cluster all-reduce (each CTA pushes its partial into every CTA's slot,
// one cluster barrier, each CTA sums the slots in rank order — deterministic and
// identical in every CTA); the k x k Cholesky solve runs redundantly in every
// CTA. Arithmetic is that of the multi-kernel folded path; only reduction order
// differs.
#include <cooperative_groups.h>

#include <algorithm>

#include "internal.cuh"

namespace cg = cooperative_groups;

namespace nlsp {

constexpr int kClusterThreads = 256;
constexpr int kMaxClusterCtas = 16;

// shared-memory layout (identical in every CTA of the cluster)
struct ClusterLayout {
    unsigned rp, ci, v, wd, b, x, r, p0, p1, q, z, s0, s1, w1, w2, red, e, Lm, wpart, bytes;
    __host__ __device__ ClusterLayout(int R, int max_nnz, int ld, int k, bool two_w, int ncta) {
        unsigned o = 0;
        auto take = [&](unsigned bytes) {
            const unsigned at = o;
            o += (bytes + 15u) & ~15u;
            return at;
        };
        rp = take((R + 1) * 4);
        ci = take(max_nnz * 4);
        v = take(max_nnz * 8);
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
        w1 = take(R * ld * 8);
        w2 = two_w ? take(R * ld * 8) : w1;
        red = take(2 * ncta * (ld + 4) * 8);  // double-buffered all-reduce slots
        e = take((ld + 4) * 8);
        Lm = take(k * k * 8);
        wpart = take((kClusterThreads / 32) * (ld + 4) * 8);  // per-warp restriction partials
        bytes = o;
    }
};

namespace {

__device__ __forceinline__ double block_sum_t(double v, double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) scratch[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += scratch[w];
    return t;
}

}  // namespace

// y = A x for own rows, x gathered from whichever CTA owns the column; x is the
// value array at local offset `xo` in every CTA; `fx` transforms (used for the
// implicit first sweep s = w D^-1 r and the p = z + beta p gather).
template <class Fx>
__device__ __forceinline__ double cluster_row_dot(cg::cluster_group& cl, const int* rps,
                                                  const int* cis, const double* vs, int lr, int R,
                                                  const Fx& fx) {
    double s = 0.0;
    for (int kk = rps[lr]; kk < rps[lr + 1]; ++kk) {
        const int col = cis[kk];
        s = fma(vs[kk], fx(col / R, col % R), s);
    }
    return s;
}

__global__ void __launch_bounds__(kClusterThreads) k_cluster_pcg(ClusterArgs a) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ __align__(16) unsigned char sm[];
    __shared__ double scratch[32];
    const int ncta = (int)cl.num_blocks();
    const int q = (int)cl.block_rank();
    const int R = a.rows, ld = a.ld, k = a.k;
    const int row0 = q * R;
    const int nr = max(0, min(R, a.n - row0));
    const ClusterLayout Lo(R, a.max_nnz, ld, k, a.W2 != a.W1, ncta);
    int* rps = reinterpret_cast<int*>(sm + Lo.rp);
    int* cis = reinterpret_cast<int*>(sm + Lo.ci);
    double* vs = reinterpret_cast<double*>(sm + Lo.v);
    double* wd = reinterpret_cast<double*>(sm + Lo.wd);
    double* bv = reinterpret_cast<double*>(sm + Lo.b);
    double* xv = reinterpret_cast<double*>(sm + Lo.x);
    double* rv = reinterpret_cast<double*>(sm + Lo.r);
    double* pv[2] = {reinterpret_cast<double*>(sm + Lo.p0), reinterpret_cast<double*>(sm + Lo.p1)};
    double* qv = reinterpret_cast<double*>(sm + Lo.q);
    double* zv = reinterpret_cast<double*>(sm + Lo.z);
    double* sv[2] = {reinterpret_cast<double*>(sm + Lo.s0), reinterpret_cast<double*>(sm + Lo.s1)};
    double* w1 = reinterpret_cast<double*>(sm + Lo.w1);
    double* w2 = reinterpret_cast<double*>(sm + Lo.w2);
    double* red = reinterpret_cast<double*>(sm + Lo.red);
    double* ev = reinterpret_cast<double*>(sm + Lo.e);
    double* Lm = reinterpret_cast<double*>(sm + Lo.Lm);
    double* wpart = reinterpret_cast<double*>(sm + Lo.wpart);
    const int tid = threadIdx.x, nt = blockDim.x;
    PcgState* st = a.st;

    // ---- load the CTA's slice of the system into shared memory
    const int base = nr ? a.rp[row0] : 0;
    for (int i = tid; i <= nr; i += nt) rps[i] = (nr ? a.rp[row0 + i] : 0) - base;
    const int nnz_loc = nr ? a.rp[row0 + nr] - base : 0;
    for (int i = tid; i < nnz_loc; i += nt) {
        cis[i] = a.ci[base + i];
        vs[i] = a.v[base + i];
    }
    for (int i = tid; i < R; i += nt) {
        const bool own = i < nr;
        wd[i] = own ? a.wd[row0 + i] : 0.0;
        bv[i] = own ? a.b[row0 + i] : 0.0;
        xv[i] = 0.0;
        rv[i] = bv[i];
        pv[0][i] = pv[1][i] = qv[i] = zv[i] = sv[0][i] = sv[1][i] = 0.0;
    }
    for (int i = tid; i < nr * ld; i += nt) {
        w1[i] = a.W1[(long long)row0 * ld + i];
        if (a.W2 != a.W1) w2[i] = a.W2[(long long)row0 * ld + i];
    }
    for (int i = tid; i < k * k; i += nt) Lm[i] = a.L[i];
    int rbuf = 0;
    // all-reduce of `cnt` doubles from `part` (shared, this CTA's partial) into
    // `out` (shared, every CTA): push to every CTA's slot q, one barrier, sum
    // the slots in rank order
    auto allreduce = [&](const double* part, int cnt, double* out) {
        const int stride = ld + 4;
        double* slot0 = red + (size_t)rbuf * ncta * stride;
        for (int idx = tid; idx < ncta * cnt; idx += nt) {
            const int dst = idx / cnt, j = idx % cnt;
            double* remote = cl.map_shared_rank(slot0, dst);
            remote[q * stride + j] = part[j];
        }
        cl.sync();
        for (int j = tid; j < cnt; j += nt) {
            double t = 0.0;
            for (int c = 0; c < ncta; ++c) t += slot0[c * stride + j];
            out[j] = t;
        }
        __syncthreads();
        rbuf ^= 1;
    };
    __shared__ double part[264];
    __shared__ double tot[264];
    cl.sync();  // every CTA's slice is resident before any DSMEM gather

    // remote readers
    auto remote_val = [&](double* local_arr, int owner, int li) -> double {
        return owner == q ? local_arr[li] : cl.map_shared_rank(local_arr, owner)[li];
    };
    // scalar all-reduce of a per-thread value
    auto sum_scalar = [&](double v) -> double {
        const double t = block_sum_t(v, scratch);
        if (tid == 0) part[0] = t;
        __syncthreads();
        allreduce(part, 1, tot);
        return tot[0];
    };

    // restriction c = W1^T r (own rows), all-reduce, coarse solve L L^T e = c
    auto restrict_solve = [&]() {
        // lane j of warp w accumulates column j over rows w, w+8, ...; warps
        // combine in a fixed order
        const int warp = tid >> 5, lane = tid & 31, nw = nt >> 5;
        for (int j = lane; j < ld; j += 32) {
            double accj = 0.0;
            for (int i = warp; i < nr; i += nw) accj = fma(w1[i * ld + j], rv[i], accj);
            wpart[warp * (ld + 4) + j] = accj;
        }
        __syncthreads();
        for (int j = tid; j < ld; j += nt) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += wpart[w * (ld + 4) + j];
            part[j] = t;
        }
        __syncthreads();
        allreduce(part, ld, tot);
        // L y = c, L^T e = y (cholesky.hpp:41-57) by warp 0, column-oriented
        if (tid < 32) {
            for (int i = tid; i < k; i += 32) ev[i] = tot[i];
            for (int j = 0; j < k; ++j) {
                __syncwarp();
                const double yj = ev[j] / Lm[j * k + j];
                __syncwarp();
                if (tid == 0) ev[j] = yj;
                for (int i = j + 1 + tid; i < k; i += 32) ev[i] = fma(-Lm[i * k + j], yj, ev[i]);
            }
            for (int j = k - 1; j >= 0; --j) {
                __syncwarp();
                const double xj = ev[j] / Lm[j * k + j];
                __syncwarp();
                if (tid == 0) ev[j] = xj;
                for (int i = tid; i < j; i += 32) ev[i] = fma(-Lm[j * k + i], xj, ev[i]);
            }
            if (tid == 0 && (k & 1)) ev[k] = 0.0;
        }
        __syncthreads();
    };

    // z = S_T(r) + W2 e (folded cycle tail); returns r.z (all-reduced)
    auto tail = [&]() -> double {
        const int T = a.nu1 + a.nu2;
        double* cur = nullptr;  // s_1 = w D^-1 r implicit
        int cb = 0;
        for (int j = 2; j <= T; ++j) {
            double* nxt = sv[cb];
            for (int i = tid; i < nr; i += nt) {
                double y;
                if (cur == nullptr)
                    y = cluster_row_dot(cl, rps, cis, vs, i, R, [&](int o, int li) {
                        return remote_val(wd, o, li) * remote_val(rv, o, li);
                    });
                else
                    y = cluster_row_dot(cl, rps, cis, vs, i, R,
                                        [&](int o, int li) { return remote_val(cur, o, li); });
                const double si = cur == nullptr ? wd[i] * rv[i] : cur[i];
                nxt[i] = fma(wd[i], rv[i] - y, si);
            }
            cl.sync();  // the next sweep gathers this one's output
            cur = nxt;
            cb ^= 1;
        }
        double rz = 0.0;
        for (int i = tid; i < nr; i += nt) {
            double s = 0.0;
            for (int j = 0; j < ld; ++j) s = fma(w2[i * ld + j], ev[j], s);
            const double zp = T == 0 ? 0.0 : (cur == nullptr ? wd[i] * rv[i] : cur[i]);
            const double zi = zp + s;
            zv[i] = zi;
            rz = fma(rv[i], zi, rz);
        }
        return sum_scalar(rz);
    };

    // ---- prologue: ||b||, z = M b, rz (two_level.hpp:143-156)
    double bb = 0.0;
    for (int i = tid; i < nr; i += nt) bb = fma(bv[i], bv[i], bb);
    const double bnorm = sqrt(sum_scalar(bb));
    if (bnorm == 0.0) {
        if (q == 0 && tid == 0) {
            st->error = kErrValidation;
            st->done = 1;
        }
        return;
    }
    restrict_solve();
    double rz = tail();
    cl.sync();  // z complete everywhere before p = z is gathered
    const long long max_it = st->max_it;
    const double delta = st->delta;
    double beta = 0.0;
    long long it = 0;
    int converged = 0, err = 0;
    for (; it < max_it; ++it) {
        double* pc = pv[it & 1];
        double* pp = pv[(it + 1) & 1];
        const bool first = it == 0;
        // p = z + beta p (gathered on the fly), q = A p, p.q (:159-163)
        double pap_part = 0.0;
        for (int i = tid; i < nr; i += nt) {
            const double y = cluster_row_dot(cl, rps, cis, vs, i, R, [&](int o, int li) {
                const double zz = remote_val(zv, o, li);
                return first ? zz : fma(beta, remote_val(pp, o, li), zz);
            });
            const double pi = first ? zv[i] : fma(beta, pp[i], zv[i]);
            pc[i] = pi;
            qv[i] = y;
            pap_part = fma(pi, y, pap_part);
        }
        const double pap = sum_scalar(pap_part);
        if (pap <= 0.0) {
            err = kErrNotSpd;
            break;
        }
        const double alpha = rz / pap;
        // x += alpha p, r -= alpha q, ||r|| (:164-176)
        double rr = 0.0;
        for (int i = tid; i < nr; i += nt) {
            xv[i] = fma(alpha, pc[i], xv[i]);
            const double ri = fma(-alpha, qv[i], rv[i]);
            rv[i] = ri;
            rr = fma(ri, ri, rr);
        }
        const double rel = sqrt(sum_scalar(rr)) / bnorm;
        if (q == 0 && tid == 0) a.hist[it] = rel;
        if (rel < delta) {
            converged = 1;
            ++it;
            break;
        }
        // z = M r (folded cycle), beta = rz' / rz (:177-182)
        restrict_solve();
        const double rz_new = tail();
        beta = rz_new / rz;
        rz = rz_new;
        cl.sync();  // z and p complete everywhere before the next gathers
    }
    // true residual ||b - A x|| / ||b|| (:185-189)
    cl.sync();
    double tr = 0.0;
    for (int i = tid; i < nr; i += nt) {
        const double y = cluster_row_dot(cl, rps, cis, vs, i, R,
                                         [&](int o, int li) { return remote_val(xv, o, li); });
        const double d = bv[i] - y;
        tr = fma(d, d, tr);
    }
    const double true_res = sqrt(sum_scalar(tr)) / bnorm;
    for (int i = tid; i < nr; i += nt) a.x[row0 + i] = xv[i];
    if (q == 0 && tid == 0) {
        st->iterations = err ? it : it;
        st->converged = converged;
        st->error = err;
        st->done = 1;
        st->bnorm = bnorm;
        st->true_res = err ? 0.0 : true_res;
        st->last_rel = it > 0 ? a.hist[it - 1] : 0.0;
        st->body_runs = it;
    }
    cl.sync();  // no CTA exits while others may still read its shared memory
}

// Cluster size and rows per CTA for an n x n system (row_ptr on the host), or 0
// when its slices do not fit in shared memory.
int cluster_plan(int n, int k, const int* rp_host, bool two_w, int* rows_out, int* max_nnz_out,
                 size_t* smem_out) {
    const int ld = k + (k & 1);
    if (k > 256) return 0;
    for (int ncta = 2; ncta <= kMaxClusterCtas; ncta *= 2) {
        const int R = (n + ncta - 1) / ncta;
        int mx = 0;
        for (int q = 0; q < ncta; ++q) {
            const int r0 = q * R, r1 = std::min(n, r0 + R);
            if (r0 < r1) mx = std::max(mx, rp_host[r1] - rp_host[r0]);
        }
        const ClusterLayout Lo(R, mx, ld, k, two_w, ncta);
        if (Lo.bytes <= 200 * 1024) {
            *rows_out = R;
            *max_nnz_out = mx;
            *smem_out = Lo.bytes;
            return ncta;
        }
    }
    return 0;
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

}  // namespace nlsp
