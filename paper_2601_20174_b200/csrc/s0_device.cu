// paper_2601_20174_b200/csrc/s0_device.cu — S^(0) of generate_smoothed_vectors
// drawn on the device (smoothing.hpp:84-92, rng.hpp:22-49).
//
// The reference fills S^(0) row by row from ONE sequential std::mt19937_64
// stream. The stream is GF(2)-linear, so it splits exactly: substream t covers
// words [t B, (t + 1) B), B = 2^18, and starts from the generator's window
// t B words ahead of the seeded one (mt_jump.hpp). The windows of all
// substreams come from a binary tree of jumps (k_mt_jump: one CTA per jump,
// window(t + s) = XOR of the windows of t's continued stream at the set
// coefficients of x^(s B) mod phi), then every warp generates its substream's
// words (k_mt_words) and a pair-parallel kernel applies Box-Muller in place
// (k_box_muller). The mt19937_64 words are bit for bit the host stream's
// (tests/test_gpu_kernels.py); the normals go through CUDA's log / sincos
// instead of glibc's, so they can differ from the reference's in the last
// bits — the device draw is therefore opt-in (nlsp_ctx_set_s0_draw), and
// the host stream (host_rng.hpp) stays the default and the parity reference.
#include "internal.cuh"

namespace nlsp {

inline void count(const LaunchCtx& c) { ++*c.launches; }

namespace {
using u64 = unsigned long long;
constexpr int kN = 312, kM = 156;
constexpr u64 kA = 0xB5026F5AA96619E9ull, kUM = 0xFFFFFFFF80000000ull, kLM = 0x7FFFFFFFull;

__device__ __forceinline__ u64 mt_next(u64 x0, u64 x1, u64 xm) {
    const u64 y = (x0 & kUM) | (x1 & kLM);
    return xm ^ (y >> 1) ^ ((y & 1ull) ? kA : 0ull);
}
__device__ __forceinline__ u64 mt_temper(u64 x) {
    x ^= (x >> 29) & 0x5555555555555555ull;
    x ^= (x << 17) & 0x71D67FFFEDA60000ull;
    x ^= (x << 37) & 0xFFF7EEE000000000ull;
    x ^= x >> 43;
    return x;
}

// next block of 312 words from `src` into `dst` (a different buffer), whole CTA
__device__ __forceinline__ void cta_next_block(const u64* src, u64* dst) {
    const int i = threadIdx.x;
    if (i < kM) dst[i] = mt_next(src[i], src[i + 1], src[i + kM]);
    __syncthreads();
    if (i >= kM && i < kN) dst[i] = mt_next(src[i], i + 1 < kN ? src[i + 1] : dst[0], dst[i - kM]);
    __syncthreads();
}
}  // namespace

// window(t + s) from window(t) for t = 2 s blockIdx.x: the XOR of the windows
// at positions i of t's continued stream over the set coefficients g_i of
// x^(s B) mod phi (312 words of bits, degree < 19937). Thread w accumulates
// word w of the result; the stream is regenerated block by block in a ring of
// two blocks (position i + w lies in block i / 312 or the next).
__global__ void __launch_bounds__(320) k_mt_jump(u64* __restrict__ win, long long s, long long nsub,
                                                 const u64* __restrict__ poly) {
    __shared__ u64 ring[2 * kN];
    __shared__ u64 g[kN];
    const long long t = 2 * s * (long long)blockIdx.x;
    if (t + s >= nsub) return;
    const int w = threadIdx.x;
    if (w < kN) {
        ring[w] = win[t * kN + w];
        g[w] = poly[w];
    }
    __syncthreads();
    cta_next_block(ring, ring + kN);
    u64 acc = 0;
    for (int b = 0; b < 64; ++b) {  // 64 blocks of 312 coefficients = 312 words of 64
        if (w < kN) {
            int pos = (b & 1) * kN + w;  // (i + w) mod 624 for i = 312 b
            const int i0 = kN * b;
#pragma unroll 8
            for (int ii = 0; ii < kN; ++ii) {
                const int i = i0 + ii;
                const u64 bit = (g[i >> 6] >> (i & 63)) & 1ull;
                acc ^= ring[pos] & (0ull - bit);
                pos = pos + 1 == 2 * kN ? 0 : pos + 1;
            }
        }
        __syncthreads();
        // block b + 2 replaces block b
        cta_next_block(ring + ((b + 1) & 1) * kN, ring + (b & 1) * kN);
    }
    if (w < kN) win[(t + s) * kN + w] = acc;
}

// The words of substream t = [t B, min((t + 1) B, total)) by one warp (total =
// the even number of words the count elements take): the
// window in shared memory, each block of 312 new words in two half steps of
// 156 independent words (lanes take words lane + 32 j), tempered on the way out.
constexpr int kWordsWarps = 4;
__global__ void __launch_bounds__(32 * kWordsWarps) k_mt_words(const u64* __restrict__ win, long long nsub,
                                                             int log2b, u64 total, u64 count,
                                                             u64* __restrict__ out, u64* __restrict__ tail) {
    __shared__ u64 st[kWordsWarps][kN];
    const int lane = threadIdx.x & 31, wq = threadIdx.x >> 5;
    const long long t = (long long)blockIdx.x * kWordsWarps + wq;
    if (t >= nsub) return;
    u64* mt = st[wq];
    for (int i = lane; i < kN; i += 32) mt[i] = win[t * kN + i];
    __syncwarp();
    const u64 w0 = (u64)t << log2b;
    const u64 cnt = min((u64)1 << log2b, total - w0);
    for (u64 done = 0; done < cnt; done += kN) {
        u64 v[5];
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int i = lane + 32 * j;
            v[j] = i < kM ? mt_next(mt[i], mt[i + 1], mt[i + kM]) : 0ull;
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int i = lane + 32 * j;
            if (i < kM) mt[i] = v[j];
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int i = kM + lane + 32 * j;
            v[j] = i < kN ? mt_next(mt[i], i + 1 < kN ? mt[i + 1] : mt[0], mt[i - kM]) : 0ull;
        }
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const int i = kM + lane + 32 * j;
            if (i < kN) mt[i] = v[j];
        }
        __syncwarp();
        for (int i = lane; i < kN; i += 32) {
            const u64 idx = done + i;
            if (idx < cnt) {
                const u64 word = mt_temper(mt[i]);
                // an odd element count leaves the last pair's second word past the
                // end of the destination (count = total - 1): it goes to `tail`
                if (w0 + idx < count) out[w0 + idx] = word;
                else tail[0] = word;
            }
        }
    }
}

// Box-Muller in place (rng.hpp:37-49): pair p holds the stream's words 2p and
// 2p + 1 and becomes r cos a, r sin a with u = (word >> 11) 2^-53. A zero u1
// would make the reference redraw it and shift the rest of the stream
// (probability 2^-53 per pair): it raises `flag` and the host stream takes over.
__global__ void __launch_bounds__(256) k_box_muller(double* __restrict__ out, u64 count, const u64* __restrict__ tail,
                                                    int* __restrict__ flag) {
    const u64 pairs = (count + 1) / 2;
    for (u64 p = blockIdx.x * (u64)blockDim.x + threadIdx.x; p < pairs; p += (u64)gridDim.x * blockDim.x) {
        const bool both = 2 * p + 1 < count;
        u64 a0, a1;
        if (both) {
            const ulonglong2 wv = *reinterpret_cast<const ulonglong2*>(out + 2 * p);
            a0 = wv.x;
            a1 = wv.y;
        } else {
            a0 = reinterpret_cast<const u64*>(out)[2 * p];
            a1 = tail[0];
        }
        const double u1 = (double)(a0 >> 11) * 0x1.0p-53;
        const double u2 = (double)(a1 >> 11) * 0x1.0p-53;
        if (u1 <= 0.0) {
            atomicOr(flag, 1);
            continue;
        }
        const double r = sqrt(-2.0 * log(u1));
        const double a = 2.0 * 3.141592653589793 * u2;
        double sn, cs;
        sincos(a, &sn, &cs);
        if (both) *reinterpret_cast<double2*>(out + 2 * p) = make_double2(r * cs, r * sn);
        else out[2 * p] = r * cs;
    }
}

// the raw stream words only (tests: bit for bit the host generator's)
void launch_mt_stream(const LaunchCtx& c, unsigned long long* win, long long nsub, int log2b,
                      const unsigned long long* polys, int poly_min_log2, unsigned long long total_words,
                      unsigned long long count_elems, unsigned long long* out, unsigned long long* tail) {
    long long top = 1;
    while (top < nsub) top <<= 1;
    for (long long s = top >> 1; s >= 1; s >>= 1) {
        int lg = 0;
        while ((1ll << lg) < s) ++lg;
        const long long jumps = (nsub + 2 * s - 1) / (2 * s);
        k_mt_jump<<<(unsigned)jumps, 320, 0, c.s>>>(win, s, nsub, polys + (size_t)(log2b + lg - poly_min_log2) * kN);
        count(c);
    }
    k_mt_words<<<(unsigned)((nsub + kWordsWarps - 1) / kWordsWarps), 32 * kWordsWarps, 0, c.s>>>(win, nsub, log2b,
                                                                                              total_words, count_elems, out, tail);
    count(c);
}

void launch_box_muller(const LaunchCtx& c, double* out, unsigned long long elems, const unsigned long long* tail,
                       int* flag) {
    const u64 pairs = (elems + 1) / 2;
    long long blocks = (long long)((pairs + 255) / 256);
    const long long cap = (long long)c.num_sms * 16;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    k_box_muller<<<(unsigned)blocks, 256, 0, c.s>>>(out, elems, tail, flag);
    count(c);
}

}  // namespace nlsp
