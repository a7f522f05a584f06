// paper_2601_20174_b200/csrc/tma_rows.cuh — TMA-staged row-tile engine.
//
// The CSR row kernels are latency-bound on the dependent chain
// row_ptr -> (values, columns) -> gather. Here a producer warp streams each
// tile of TR consecutive rows into shared memory with bulk async copies
// (cp.async.bulk, the 1-D TMA path; UBLKCP in SASS): the tile's row_ptr slice,
// its contiguous run of values and column indices, and optionally the tile's TR
// rows of the basis P (contiguous too, n x ld row-major). An S-stage ring of
// full/empty mbarriers keeps S tiles in flight per CTA, so HBM sees S tiles of
// requests per CTA while 8 consumer warps work on the current one; the only
// global latency left on the consumer side is the gather x[col], which is
// mostly an L1/L2 hit for the banded operators of the configs.
#pragma once

#include "internal.cuh"

namespace nlsp {

constexpr int kConsumerWarps = 8;
constexpr int kTmaThreads = (kConsumerWarps + 1) * 32;  // + 1 producer warp
constexpr int kGroups = kConsumerWarps * 32 / kGroup;    // 32 row groups per CTA

__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* b, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// try_wait with a suspend-time hint (ns): the waiting thread is parked until
// the phase completes or the hint runs out, instead of the short
// system-dependent limit. ncu source counters of the lean pass at C4 without
// it: 18.7 M SYNCS + 17.5 M YIELD for 1.2 M completed waits, a third of the
// kernel's instructions spent polling. NLSP_MBAR_HINT=0 compiles the plain form.
#ifndef NLSP_MBAR_HINT
#define NLSP_MBAR_HINT 20000
#endif
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned phase) {
    const unsigned addr = smem_u32(b);
    unsigned ok = 0;
    do {
#if NLSP_MBAR_HINT > 0
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(addr), "r"(phase), "r"((unsigned)NLSP_MBAR_HINT)
            : "memory");
#else
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(addr), "r"(phase)
            : "memory");
#endif
    } while (!ok);
}
// Wait of a warp that runs AHEAD of the critical path (the pass's stencil warps:
// their tile's data arrives several tile-times before the W-product warps need
// A s): sleep between polls instead of spinning (ncu: 9.9 M polls for 64 k waits).
__device__ __forceinline__ void mbar_wait_relaxed(unsigned long long* b, unsigned phase, unsigned ns) {
    const unsigned addr = smem_u32(b);
    for (;;) {
        unsigned ok = 0;
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(ok)
            : "r"(addr), "r"(phase)
            : "memory");
        if (ok) break;
        __nanosleep(ns);
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         unsigned long long* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__host__ __device__ constexpr unsigned round16(unsigned b) { return (b + 15u) & ~15u; }

// Byte layout of one stage for a tile of TR rows, at most `tile_nnz` nonzeros
// and (with basis rows) ld doubles per row.
struct StageLayout {
    unsigned rp_off, v_off, c_off, p_off, bytes;
    __host__ __device__ StageLayout(int TR, int tile_nnz, int ld, bool with_p) {
        rp_off = 0;
        v_off = round16((TR + 4) * 4);
        c_off = v_off + round16((tile_nnz + 2) * 8);
        p_off = c_off + round16((tile_nnz + 8) * 4);
        bytes = p_off + (with_p ? round16(TR * ld * 8) : 0u);
    }
};

// Producer side: stage tile `tile` (rows [r0, r0 + rows), nonzeros [a0, a1))
// into `stage_base`.
__device__ __forceinline__ void stage_tile(const int* __restrict__ rp, const int* __restrict__ ci,
                                           const double* __restrict__ v,
                                           const double* __restrict__ P, int ld, int n, int TR,
                                           int tile, int a0, int a1, unsigned char* stage_base,
                                           const StageLayout& L, unsigned long long* full,
                                           const unsigned* __restrict__ pmask = nullptr) {
    const int r0 = tile * TR;
    const int rows = min(TR, n - r0);
    const int s0 = a0 & ~1, c0 = a0 & ~3;
    const unsigned rbytes = ((rows + 1 + 3) & ~3) * 4;
    const unsigned vbytes = ((a1 - s0 + 1) & ~1) * 8;
    // implicit columns (PackArgs): the rows' presence masks go where the column indices would
    const unsigned cbytes = pmask ? ((rows + 3) & ~3) * 4 : ((a1 - c0 + 3) & ~3) * 4;
    const unsigned pbytes = P ? (unsigned)rows * ld * 8 : 0u;
    NLSP_CHECK(rows > 0 && rows <= TR && a0 >= 0 && a1 >= a0);
    NLSP_CHECK(L.rp_off + rbytes <= L.v_off && L.v_off + vbytes <= L.c_off);
    NLSP_CHECK(L.c_off + cbytes <= (P ? L.p_off : L.bytes) && (!P || L.p_off + pbytes <= L.bytes));
    mbar_arrive_tx(full, rbytes + vbytes + cbytes + pbytes);
    bulk_g2s(stage_base + L.rp_off, rp + r0, rbytes, full);
    if (vbytes) bulk_g2s(stage_base + L.v_off, v + s0, vbytes, full);
    if (cbytes) {
        if (pmask) bulk_g2s(stage_base + L.c_off, pmask + r0, cbytes, full);
        else bulk_g2s(stage_base + L.c_off, ci + c0, cbytes, full);
    }
    if (pbytes) bulk_g2s(stage_base + L.p_off, P + (long long)r0 * ld, pbytes, full);
}

// The producer warp: for this CTA's tiles (blockIdx.x + i * gridDim.x), the 32
// lanes first load the row_ptr boundaries of 32 upcoming tiles in parallel,
// then lane 0 waits for each stage to be released and issues its bulk copies.
// The row_ptr latency is paid once per 32 tiles instead of once per tile.
template <int S>
__device__ __forceinline__ void produce_tiles(const int* __restrict__ rp, const int* __restrict__ ci,
                                              const double* __restrict__ v,
                                              const double* __restrict__ P, int ld, int n, int TR,
                                              unsigned char* stages, const StageLayout& L,
                                              unsigned long long* full, unsigned long long* empty,
                                              const unsigned* __restrict__ pmask = nullptr) {
    const int lane = threadIdx.x & 31;
    const int ntiles = (n + TR - 1) / TR;
    for (int base = 0;; base += 32) {
        if ((long long)blockIdx.x + (long long)base * gridDim.x >= ntiles) break;
        const long long my = (long long)blockIdx.x + (long long)(base + lane) * gridDim.x;
        int b0 = 0, b1 = 0;
        if (my < ntiles) {
            const int r0 = (int)my * TR;
            b0 = __ldg(rp + r0);
            b1 = __ldg(rp + min(r0 + TR, n));
        }
        for (int j = 0; j < 32; ++j) {
            const long long tile = (long long)blockIdx.x + (long long)(base + j) * gridDim.x;
            if (tile >= ntiles) break;
            const int a0 = __shfl_sync(0xffffffffu, b0, j);
            const int a1 = __shfl_sync(0xffffffffu, b1, j);
            if (lane == 0) {
                const int i = base + j;
                const int stg = i % S;
                if (i >= S) mbar_wait(&empty[stg], ((i / S) - 1) & 1);
                stage_tile(rp, ci, v, P, ld, n, TR, (int)tile, a0, a1, stages + stg * L.bytes, L,
                           &full[stg], pmask);
            }
            __syncwarp();
        }
    }
}

// Consumer side, transposed mapping: G lanes per row, lane = s * R + r with
// R = 32 / G consecutive rows per warp step, so lanes r, r+1, ... of one slot s
// gather x[col] of consecutive rows — for banded operators (sorted columns,
// col = row + offset) the gather of a slot is one contiguous run. Warp w takes
// local rows (w * U + u) * R + r, u < U. Each lane accumulates its slots in
// ascending column order; the G partial sums are combined by xor-shuffles.
template <int G, int U, int CH, class Gat>
__device__ __forceinline__ void staged_rows_dot(const unsigned char* stage_base,
                                                const StageLayout& L, int rows, int warp,
                                                int lane, const Gat& g, int (&lr)[U],
                                                bool (&valid)[U], double (&y)[U]) {
    constexpr int R = 32 / G;
    const int r = lane % R, s = lane / R;
    const int* rps = reinterpret_cast<const int*>(stage_base + L.rp_off);
    const double* vs = reinterpret_cast<const double*>(stage_base + L.v_off);
    const int* cs = reinterpret_cast<const int*>(stage_base + L.c_off);
    const int a0 = rps[0];
    const int s0 = a0 & ~1, c0 = a0 & ~3;
    int b[U], e[U];
    int len = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        lr[u] = (warp * U + u) * R + r;
        valid[u] = lr[u] < rows;
        b[u] = valid[u] ? rps[lr[u]] : 0;
        e[u] = valid[u] ? rps[lr[u] + 1] : 0;
        len = max(len, e[u] - b[u]);
        y[u] = 0.0;
    }
    for (int off = s; off < len; off += G * CH) {
        double vv[U][CH], xv[U][CH];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int k = b[u] + off + c * G;
                vv[u][c] = 0.0;
                xv[u][c] = 0.0;
                if (k < e[u]) {
                    vv[u][c] = vs[k - s0];
                    xv[u][c] = g(cs[k - c0]);
                }
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int c = 0; c < CH; ++c) y[u] = fma(vv[u][c], xv[u][c], y[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int m = R; m < 32; m <<= 1) y[u] += __shfl_xor_sync(0xffffffffu, y[u], m);
}

// The same for the implicit-column form (PackArgs, internal.cuh; one lane per
// row): the staged column region holds the rows' presence masks, the j-th
// nonzero of row i is at column i + offs[t_j], t_j the j-th set bit of its mask.
// offs: the offsets in shared memory. Same values in the same order: y is
// bitwise the explicit-column result.
template <int U, int CH, class Gat>
__device__ __forceinline__ void staged_rows_dot_masked(const unsigned char* stage_base,
                                                       const StageLayout& L, int rows, int r0, int warp,
                                                       int lane, const Gat& g, const int* offs,
                                                       int (&lr)[U], bool (&valid)[U], double (&y)[U]) {
    const int* rps = reinterpret_cast<const int*>(stage_base + L.rp_off);
    const double* vs = reinterpret_cast<const double*>(stage_base + L.v_off);
    const unsigned* ms = reinterpret_cast<const unsigned*>(stage_base + L.c_off);
    const int s0 = rps[0] & ~1;
    int b[U], e[U];
    unsigned m[U];
    int len = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        lr[u] = (warp * U + u) * 32 + lane;
        valid[u] = lr[u] < rows;
        b[u] = valid[u] ? rps[lr[u]] : 0;
        e[u] = valid[u] ? rps[lr[u] + 1] : 0;
        m[u] = valid[u] ? ms[lr[u]] : 0u;
        len = max(len, e[u] - b[u]);
        y[u] = 0.0;
    }
    for (int off = 0; off < len; off += CH) {
        double vv[U][CH], xv[U][CH];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int c = 0; c < CH; ++c) {
                const int k = b[u] + off + c;
                vv[u][c] = 0.0;
                xv[u][c] = 0.0;
                if (k < e[u]) {
                    const int t = __ffs(m[u]) - 1;
                    m[u] &= m[u] - 1u;
                    NLSP_CHECK(t >= 0);
                    vv[u][c] = vs[k - s0];
                    xv[u][c] = g(r0 + lr[u] + offs[t]);
                }
            }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int c = 0; c < CH; ++c) y[u] = fma(vv[u][c], xv[u][c], y[u]);  // absent: + 0 * 0, as above
    }
}

// Consumer side: y[u] = sum_k v_k g(col_k) for the U local rows lr[u] of this
// 8-lane group, reading row_ptr / values / columns from the staged tile.
template <int U, class Gat>
__device__ __forceinline__ void staged_group_dot(const unsigned char* stage_base,
                                                 const StageLayout& L, const int (&lr)[U],
                                                 const bool (&valid)[U], const Gat& g, int l,
                                                 double (&y)[U]) {
    const int* rps = reinterpret_cast<const int*>(stage_base + L.rp_off);
    const double* vs = reinterpret_cast<const double*>(stage_base + L.v_off);
    const int* cs = reinterpret_cast<const int*>(stage_base + L.c_off);
    const int a0 = rps[0];
    const int s0 = a0 & ~1, c0 = a0 & ~3;
    int b[U], e[U];
    int len = 0;
#pragma unroll
    for (int u = 0; u < U; ++u) {
        b[u] = valid[u] ? rps[lr[u]] : 0;
        e[u] = valid[u] ? rps[lr[u] + 1] : 0;
        len = max(len, e[u] - b[u]);
        y[u] = 0.0;
    }
    for (int off = l; off < len; off += kGroup) {
        double vv[U], xv[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int k = b[u] + off;
            vv[u] = 0.0;
            xv[u] = 0.0;
            if (k < e[u]) {
                vv[u] = vs[k - s0];
                xv[u] = g(cs[k - c0]);
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) y[u] = fma(vv[u], xv[u], y[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) y[u] = group_sum(y[u]);
}

}  // namespace nlsp
