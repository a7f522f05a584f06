// paper_2601_20174_b200/csrc/mlp.cu — MLP inference for the NLSS basis
// (SURVEY §8f.4): infer_basis (train.hpp:52-62) = orthonormalize(reshape(
// MlpModel::forward(vec(S / ||S||_F)))) with the forward pass of mlp.hpp:113-161
// (hidden layers Linear -> LayerNorm(gain, offset) -> GELU, plain Linear out).
//
// The network is a batch-1 GEMV chain over the flattened vector set: at the
// paper's N = 64 (n = 4 225, K = 32) the input and output widths are n K =
// 135 200, so the first and last weight matrices are 138 MB each and the pass
// is HBM-bound on streaming them once:
//   k_gemv_splitk  wide fan-in (first layer): 8 output rows per CTA share each
//                  x element loaded (x stays in L2), the fan-in split into
//                  chunks across CTAs; fixed-order partial sums
//   k_gemv_rows    narrow fan-in (hidden, last layer): a warp per output row,
//                  x in shared memory, coalesced row reads, bias fused
//   k_finish       bias + partial sums (split-K), LayerNorm over the features,
//                  gain/offset, GELU — one CTA (features <= a few thousand)
// Rounding differs from the reference's 4-accumulator dot (mlp.hpp:28-40) in
// summation order only.
#include "internal.cuh"

namespace nlsp {

namespace {

__device__ __forceinline__ double block_sum(double v, double* sh) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) sh[warp] = v;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < nw; ++w) t += sh[w];
    return t;
}

__device__ __forceinline__ double gelu(double x) {
    return 0.5 * x * (1.0 + erf(x * 0.70710678118654752440));  // mlp.hpp:16
}

}  // namespace

// per-CTA partial sums of squares (frobenius_norm, dense.hpp:129)
__global__ void k_sumsq_partial(long long count, const double* __restrict__ s, double* part) {
    __shared__ double sh[32];
    double acc = 0.0;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count;
         i += (long long)gridDim.x * blockDim.x)
        acc = fma(s[i], s[i], acc);
    const double t = block_sum(acc, sh);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
}

// x[j n + i] = s[i k + j] / ||S||_F (flatten_column_major of the normalised
// set, train.hpp:33-38, 57-59); flag = 1 when ||S||_F == 0
__global__ void k_flatten_scaled(int n, int k, const double* __restrict__ s, const double* part,
                                 int nparts, double* __restrict__ x, int* flag) {
    __shared__ double fro;
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int p = 0; p < nparts; ++p) t += part[p];
        fro = sqrt(t);
        if (blockIdx.x == 0 && !(fro > 0.0)) *flag = 1;
    }
    __syncthreads();
    const double f = fro;
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * k;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long i = idx / k, j = idx - i * k;
        x[j * n + i] = s[idx] / f;
    }
}

// partial[c fo + o] = sum over chunk c of W[o, :] x, rows o0 .. o0 + R - 1
template <int R>
__global__ void __launch_bounds__(256) k_gemv_splitk(const double* __restrict__ W,
                                                     const double* __restrict__ x, int fi, int fo,
                                                     int chunk, double* __restrict__ partial) {
    __shared__ double sh[32];
    const int o0 = blockIdx.x * R;
    const long long c0 = (long long)blockIdx.y * chunk;
    const long long c1 = min((long long)fi, c0 + chunk);
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    for (long long i = c0 + threadIdx.x; i < c1; i += blockDim.x) {
        const double xv = __ldg(x + i);
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (o0 + r < fo) acc[r] = fma(__ldcs(W + (long long)(o0 + r) * fi + i), xv, acc[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const double t = block_sum(acc[r], sh);
        if (threadIdx.x == 0 && o0 + r < fo) partial[(long long)blockIdx.y * fo + o0 + r] = t;
    }
}

// z[o] = b[o] + W[o, :] x, one warp per row, x staged in shared memory
__global__ void __launch_bounds__(256) k_gemv_rows(const double* __restrict__ W,
                                                   const double* __restrict__ x,
                                                   const double* __restrict__ b, int fi, int fo,
                                                   double* __restrict__ z) {
    extern __shared__ double xs[];
    for (int i = threadIdx.x; i < fi; i += blockDim.x) xs[i] = x[i];
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * (blockDim.x >> 5);
    for (long long o = blockIdx.x * (long long)(blockDim.x >> 5) + (threadIdx.x >> 5); o < fo; o += warps) {
        const double* w = W + o * fi;
        double acc = 0.0;
        for (int i = lane; i < fi; i += 32) acc = fma(__ldcs(w + i), xs[i], acc);
        acc = warp_sum(acc);
        if (lane == 0) z[o] = b[o] + acc;
    }
}

// out = b + sum_c partial[c] (nparts > 0) or z as given (nparts == 0); hidden
// layers then LayerNorm over the fo features (mlp.hpp:132-150) and GELU
__global__ void __launch_bounds__(1024) k_finish(const double* __restrict__ partial, int nparts,
                                                 const double* __restrict__ z_in,
                                                 const double* __restrict__ b, int fo,
                                                 const double* __restrict__ gain,
                                                 const double* __restrict__ offset, int hidden,
                                                 double* __restrict__ out) {
    __shared__ double sh[32];
    for (int o = threadIdx.x; o < fo; o += blockDim.x) {
        double z;
        if (nparts > 0) {
            double t = 0.0;
            for (int c = 0; c < nparts; ++c) t += partial[(long long)c * fo + o];
            z = b[o] + t;
        } else {
            z = z_in[o];
        }
        out[o] = z;
    }
    if (!hidden) return;
    __syncthreads();
    double sum = 0.0;
    for (int o = threadIdx.x; o < fo; o += blockDim.x) sum += out[o];
    const double mean = block_sum(sum, sh) / (double)fo;
    double var = 0.0;
    for (int o = threadIdx.x; o < fo; o += blockDim.x) {
        const double d = out[o] - mean;
        var = fma(d, d, var);
    }
    var = block_sum(var, sh) / (double)fo;
    const double inv_std = 1.0 / sqrt(var + 1e-5);  // kLayerNormEps, mlp.hpp:25
    for (int o = threadIdx.x; o < fo; o += blockDim.x) {
        const double xh = (out[o] - mean) * inv_std;
        out[o] = gelu(gain[o] * xh + offset[o]);
    }
}

// P[i r + j] = raw[j n + i] (reshape_column_major, train.hpp:40-47)
__global__ void k_unflatten(int n, int r, const double* __restrict__ raw, double* __restrict__ P) {
    for (long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x; idx < (long long)n * r;
         idx += (long long)gridDim.x * blockDim.x) {
        const long long i = idx / r, j = idx - i * r;
        P[idx] = raw[j * n + i];
    }
}

// ---------------------------------------------------------------- launchers --
namespace {
inline void count(const LaunchCtx& c) { ++*c.launches; }
}  // namespace

int mlp_splitk_parts(const LaunchCtx& c, int fi, int fo) {
    // ~4 CTAs per SM, chunks of at least 2048 inputs
    const int rows = (fo + 7) / 8;
    int parts = (4 * c.num_sms + rows - 1) / rows;
    parts = max(1, min(parts, fi / 2048));
    return parts;
}

void launch_mlp_layer(const LaunchCtx& c, const double* W, const double* b, const double* gain,
                      const double* offset, int fi, int fo, bool hidden, const double* x,
                      double* out, double* scratch) {
    if (fi > 4096) {
        const int parts = mlp_splitk_parts(c, fi, fo);
        const int chunk = (fi + parts - 1) / parts;
        dim3 grid((fo + 7) / 8, parts);
        k_gemv_splitk<8><<<grid, 256, 0, c.s>>>(W, x, fi, fo, chunk, scratch);
        count(c);
        k_finish<<<1, 1024, 0, c.s>>>(scratch, parts, nullptr, b, fo, gain, offset, hidden ? 1 : 0, out);
        count(c);
        return;
    }
    const int warps = 8;
    long long g = ((long long)fo + warps - 1) / warps;
    if (g > (long long)c.num_sms * 8) g = (long long)c.num_sms * 8;
    const size_t smem = (size_t)fi * sizeof(double);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_gemv_rows, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    double* z = hidden ? scratch : out;
    k_gemv_rows<<<(int)g, 256, smem, c.s>>>(W, x, b, fi, fo, z);
    count(c);
    if (hidden) {
        k_finish<<<1, 1024, 0, c.s>>>(nullptr, 0, z, b, fo, gain, offset, 1, out);
        count(c);
    }
}

void launch_mlp_input(const LaunchCtx& c, int n, int k, const double* s, double* part, int nparts,
                      double* x, int* flag) {
    k_sumsq_partial<<<nparts, 256, 0, c.s>>>((long long)n * k, s, part);
    count(c);
    k_flatten_scaled<<<c.num_sms * 4, 256, 0, c.s>>>(n, k, s, part, nparts, x, flag);
    count(c);
}

void launch_unflatten(const LaunchCtx& c, int n, int r, const double* raw, double* P) {
    k_unflatten<<<c.num_sms * 4, 256, 0, c.s>>>(n, r, raw, P);
    count(c);
}

}  // namespace nlsp
