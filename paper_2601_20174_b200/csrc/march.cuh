// paper_2601_20174_b200/csrc/march.cuh — the plane-march stencil engine for
// the gather-bound kernels of the PCG loop (included by solve_kernels.cu).
//
// When the diagonal form of A is a structured-grid stencil — every offset is
// dz * P + d with dz in {-1, 0, 1} and |d| <= h, the rows split into Z = n / P
// planes of P rows (3D: P = nx ny, h = nx; 2D: P = nx, h = 1) — each CTA
// marches through a contiguous run of planes of one slab [c0, c0 + C) of the
// plane. A producer warp streams, per plane, the slab's window
// [z P + c0 - h, z P + c0 + C + h) of every gathered array plus the slab's
// own-row arrays (matrix values, masks, pointwise operands) into an R-deep
// shared-memory ring with bulk copies (cp.async.bulk, mbarrier complete_tx),
// several planes ahead of the consumers. The 8 consumer warps first transform
// the newly landed plane in place (the gathered quantity, e.g. p = z + beta p)
// and then evaluate the stencil of the previous plane entirely from shared
// memory: every element is read from HBM once per kernel (the halos of
// neighbouring slabs hit L2), where the direct kernel (k_spmv_dia) issues
// |offsets| x (gathered arrays) L1/L2 requests per row.
//
// Each row's sum runs over the present offsets in ascending order, the same
// fma chain as k_spmv_dia and the CSR kernels, so every row value is bitwise
// theirs; only the grid-wide dot products are summed in another order.
// (Included inside namespace nlsp, after the row ops it builds on.)
#pragma once

constexpr int kMarchConsumers = 10;                      // consumer warps
constexpr int kMarchThreads = (kMarchConsumers + 1) * 32;  // + 1 producer warp
constexpr int kMarchMaxArrays = 16;                     // staged arrays per plane (halo + own)

// The launch-time geometry (march_plan in the launcher below).
struct MarchGeom {
    long long P;   // plane stride (rows)
    int h;         // in-plane halo (rows)
    int C;         // rows per slab (P % C == 0)
    int S;         // slabs per plane
    int Z;         // planes
    int R;         // ring depth (planes in flight)
    unsigned slot; // bytes per ring slot
    unsigned hcap, ocap, mcap;  // bytes per staged halo array / own array / mask
};

__device__ __forceinline__ long long floor16(long long b) { return b >= 0 ? (b & ~15ll) : -(((-b) + 15) & ~15ll); }

// Byte position of element e of an array whose window starts at element ws
// (es bytes per element) inside its 16-B aligned staging area.
__device__ __forceinline__ unsigned stage_pos(long long e, long long ws, int es) {
    return (unsigned)(e * es - floor16(ws * es));
}

// Bulk copy of elements [ws, we) of src (clamped to [0, n)) into dst laid out
// by stage_pos. Returns the bytes issued (0 when the range is empty).
__device__ __forceinline__ unsigned stage_range(unsigned char* dst, const void* src, long long ws, long long we,
                                                long long n, int es, unsigned long long* bar) {
    const long long a = ws < 0 ? 0 : ws, b = we > n ? n : we;
    if (a >= b) return 0;
    const long long sb = (a * es) & ~15ll, se = (b * es + 15) & ~15ll;
    const long long base = floor16(ws * es);
    NLSP_CHECK(sb - base >= 0 && se - base <= (we - ws) * es + 32);
    bulk_g2s(dst + (sb - base), static_cast<const unsigned char*>(src) + sb, (unsigned)(se - sb), bar);
    return (unsigned)(se - sb);
}

__device__ __forceinline__ unsigned stage_bytes(long long ws, long long we, long long n, int es) {
    const long long a = ws < 0 ? 0 : ws, b = we > n ? n : we;
    if (a >= b) return 0;
    return (unsigned)(((b * es + 15) & ~15ll) - ((a * es) & ~15ll));
}

// shared loads by 32-bit address (plain loads: ordered by the barriers' memory
// clobbers, free to interleave between rows)
__device__ __forceinline__ double lds_f64(unsigned addr) {
    return *static_cast<const double*>(__cvta_shared_to_generic(addr));
}
template <typename MT>
__device__ __forceinline__ unsigned lds_mask(unsigned addr) {
    return *static_cast<const MT*>(__cvta_shared_to_generic(addr));
}

__device__ __forceinline__ void consumer_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(kMarchConsumers * 32) : "memory");
}

// Op interface (see MOpSpmvP): NH gathered arrays staged with halo, NO own-row
// arrays; init(a), hsrc(j) / osrc(j) pointers, convert(hv) in place on one
// window element, row(i, y, hc, oc, s) with the centre values of the halo
// arrays and the own values; NV / TICKET / finish or CTA hooks as the row ops.
template <class Op, int MAXD, typename MT, bool RV, bool EXACT>
__global__ void __launch_bounds__(kMarchThreads, 2) k_march(SolveArgs a, Op op, MarchGeom g) {
    pdl_entry();
    PcgState* st = a.st;
    if (st->done) return;
    op.init(a);
    constexpr int NH = Op::NH, NO = Op::NO + (RV ? MAXD : 0);
    static_assert(NH + NO <= kMarchMaxArrays, "too many staged arrays");
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long* full = reinterpret_cast<unsigned long long*>(smem);
    unsigned long long* empty = full + 16;
    unsigned char* ring = smem + 256;
    const int R = g.R;
    if (threadIdx.x == 0) {
        for (int s = 0; s < R; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kMarchConsumers);
        }
        fence_barrier_init();
    }
    __syncthreads();
    const long long n = a.n;
    const int d = EXACT ? MAXD : a.dia.d;
    const int mb = (int)sizeof(MT);
    const long long T = (long long)g.S * g.Z;
    const long long t0 = (long long)blockIdx.x * T / gridDim.x, t1 = (long long)(blockIdx.x + 1) * T / gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // staging areas inside a slot
    auto harea = [&](unsigned char* slot, int j) { return slot + (unsigned)j * g.hcap; };
    auto oarea = [&](unsigned char* slot, int j) { return slot + NH * g.hcap + (unsigned)j * g.ocap; };
    auto marea = [&](unsigned char* slot) { return slot + NH * g.hcap + NO * g.ocap; };

    constexpr int NVS = Op::NV > 0 ? Op::NV : 1;
    double s[NVS];
#pragma unroll
    for (int j = 0; j < NVS; ++j) s[j] = 0.0;

    if (warp == kMarchConsumers) {
        // ---------------------------------------------------------- producer
        if (lane == 0) {
            long long cnt = 0;
            for (long long t = t0; t < t1;) {
                const int sl = (int)(t / g.Z);
                const int za = (int)(t % g.Z);
                const int zb = (int)min((long long)g.Z, za + (t1 - t));
                for (int zl = za - 1; zl <= zb; ++zl, ++cnt) {
                    const int slot = (int)(cnt % R);
                    if (cnt >= R) mbar_wait(&empty[slot], (unsigned)(((cnt / R) & 1) ^ 1));
                    unsigned char* sp = ring + (size_t)slot * g.slot;
                    if (zl < 0 || zl >= g.Z) {
                        mbar_arrive(&full[slot]);
                        continue;
                    }
                    const long long e0 = (long long)zl * g.P + (long long)sl * g.C;
                    const long long ws = e0 - g.h, we = e0 + g.C + g.h;
                    unsigned bytes = 0;
#pragma unroll
                    for (int j = 0; j < NH; ++j) bytes += stage_bytes(ws, we, n, 8);
#pragma unroll
                    for (int j = 0; j < Op::NO; ++j) bytes += stage_bytes(e0, e0 + g.C, n, 8);
                    if constexpr (RV) bytes += (unsigned)d * stage_bytes(e0, e0 + g.C, n, 8);
                    bytes += stage_bytes(e0, e0 + g.C, n, mb);
                    mbar_arrive_tx(&full[slot], bytes);
#pragma unroll
                    for (int j = 0; j < NH; ++j) stage_range(harea(sp, j), op.hsrc(j), ws, we, n, 8, &full[slot]);
#pragma unroll
                    for (int j = 0; j < Op::NO; ++j)
                        stage_range(oarea(sp, j), op.osrc(j), e0, e0 + g.C, n, 8, &full[slot]);
                    if constexpr (RV) {
#pragma unroll
                        for (int j = 0; j < MAXD; ++j)
                            if (j < d)
                                stage_range(oarea(sp, Op::NO + j), a.dia.rv + (size_t)j * n, e0, e0 + g.C, n, 8,
                                            &full[slot]);
                    }
                    stage_range(marea(sp), a.dia.mask, e0, e0 + g.C, n, mb, &full[slot]);
                }
                t += zb - za;
            }
        }
    } else {
        // ---------------------------------------------------------- consumers
        // per offset: plane step dz and in-plane shift dd
        int dz[MAXD], dd[MAXD];
#pragma unroll
        for (int t = 0; t < MAXD; ++t) {
            const int o = t < d ? a.dia.off[t] : 0;
            dz[t] = o > g.h ? 1 : (o < -g.h ? -1 : 0);
            dd[t] = (int)(o - (long long)dz[t] * g.P);
        }
        constexpr unsigned kFull = MAXD >= 32 ? ~0u : ((1u << MAXD) - 1u);
        const int tid = threadIdx.x;
        long long cnt = 0;
        auto slot_of = [&](long long c) { return ring + (size_t)(c % R) * g.slot; };
        // in-place transform of a landed plane's halo windows
        auto convert = [&](long long c, int zl, int sl) {
            mbar_wait(&full[c % R], (unsigned)((c / R) & 1));
            if (!Op::CONVERT || zl < 0 || zl >= g.Z) return;
            unsigned char* sp = slot_of(c);
            const long long ws = (long long)zl * g.P + (long long)sl * g.C - g.h;
            const unsigned lead = stage_pos(ws, ws, 8);
            double* hv[NH];
#pragma unroll
            for (int j = 0; j < NH; ++j) hv[j] = reinterpret_cast<double*>(harea(sp, j) + lead);
            const int W = g.C + 2 * g.h;
#pragma unroll 4
            for (int x = tid; x < W; x += kMarchConsumers * 32) op.convert(hv, x);
        };
        for (long long t = t0; t < t1;) {
            const int sl = (int)(t / g.Z);
            const int za = (int)(t % g.Z);
            const int zb = (int)min((long long)g.Z, za + (t1 - t));
            const long long base = cnt;  // load index of plane za - 1
            convert(base, za - 1, sl);
            convert(base + 1, za, sl);
            for (int z = za; z < zb; ++z) {
                const long long cz = base + (z - za + 1);
                convert(cz + 1, z + 1, sl);
                consumer_sync();
                // 32-bit shared addresses (few live registers: two CTAs per SM)
                const unsigned sp[3] = {smem_u32(slot_of(cz - 1)), smem_u32(slot_of(cz)), smem_u32(slot_of(cz + 1))};
                const long long e0 = (long long)z * g.P + (long long)sl * g.C;
                // window starts of planes z - 1, z, z + 1 differ by P: one lead
                // per plane (P may be odd in rows)
                unsigned hq[3];
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const long long ws = e0 + (long long)(q - 1) * g.P - g.h;
                    hq[q] = sp[q] + stage_pos(ws, ws, 8);
                }
                const unsigned olead = stage_pos(e0, e0, 8);
                const unsigned ob = sp[1] + NH * g.hcap + olead;
                const unsigned mk = sp[1] + NH * g.hcap + NO * g.ocap + stage_pos(e0, e0, mb);
                // the gathered quantity's window position of row 0 + offset t
                unsigned ga[MAXD];
#pragma unroll
                for (int t = 0; t < MAXD; ++t) {
                    ga[t] = (dz[t] < 0 ? hq[0] : (dz[t] > 0 ? hq[2] : hq[1])) + 8u * (unsigned)(g.h + dd[t]);
                    NLSP_CHECK(t >= d || (g.h + dd[t] >= 0 && g.h + dd[t] + g.C <= g.C + 2 * g.h));
                }
                const int rows = (int)min((long long)g.C, n - e0);
                // two rows in flight per thread: their fma chains interleave
#pragma unroll 2
                for (int c = tid; c < rows; c += kMarchConsumers * 32) {
                    const unsigned m = lds_mask<MT>(mk + (unsigned)c * mb);
                    const unsigned c8 = 8u * (unsigned)c;
                    double gv[MAXD];
#pragma unroll
                    for (int t = 0; t < MAXD; ++t) gv[t] = t < d ? lds_f64(ga[t] + c8) : 0.0;
                    double y = 0.0;
                    if (EXACT && m == kFull) {
#pragma unroll
                        for (int t = 0; t < MAXD; ++t)
                            y = fma(RV ? lds_f64(ob + (Op::NO + t) * g.ocap + c8) : a.dia.val[t], gv[t], y);
                    } else {
#pragma unroll
                        for (int t = 0; t < MAXD; ++t)
                            if (t < d && ((m >> t) & 1u))
                                y = fma(RV ? lds_f64(ob + (Op::NO + t) * g.ocap + c8) : a.dia.val[t], gv[t], y);
                    }
                    double hc[NH], oc[Op::NO > 0 ? Op::NO : 1];
#pragma unroll
                    for (int j = 0; j < NH; ++j) hc[j] = lds_f64(hq[1] + j * g.hcap + 8u * (unsigned)g.h + c8);
#pragma unroll
                    for (int j = 0; j < Op::NO; ++j) oc[j] = lds_f64(ob + j * g.ocap + c8);
                    op.row(e0 + c, y, hc, oc, s);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&empty[(cz - 1) % R]);
            }
            // the march's last two planes are no longer needed either
            const long long cend = base + (zb - za + 2);
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&empty[(cend - 2) % R]);
                mbar_arrive(&empty[(cend - 1) % R]);
            }
            cnt = cend;
            t += zb - za;
        }
    }
    if constexpr (Op::NV > 0) {
        double v[Op::NV], tot[Op::NV];
#pragma unroll
        for (int j = 0; j < Op::NV; ++j) v[j] = s[j];
        if constexpr (HasCtaHooks<Op>::value) {
            op.cta_pre(a);
            if (grid_reduce<Op::NV>(v, a.partials, &st->counter[Op::TICKET], tot)) op.cta_last(a, tot);
        } else if (grid_reduce<Op::NV>(v, a.partials, &st->counter[Op::TICKET], tot) && threadIdx.x == 0) {
            op.finish(st, tot);
        }
    }
}

// ---------------------------------------------------------------- ops --
// p = z + beta p_prev in the staged windows, q = A p, p.q -> alpha (OpSpmvP)
struct MOpSpmvP {
    static constexpr int NV = 1, NH = 2, NO = 0;
    static constexpr int TICKET = kTkSpmvP;
    static constexpr bool CONVERT = true;
    const double* z;
    const double* pp;
    double* pc;
    double* q;
    double beta;
    bool first;
    __device__ __forceinline__ void init(const SolveArgs& a) {
        const bool odd = a.st->it & 1;
        z = a.z;
        pp = odd ? a.p0 : a.p1;
        pc = odd ? a.p1 : a.p0;
        q = a.q;
        beta = a.st->beta;
        first = a.st->first != 0;
    }
    __device__ __forceinline__ const double* hsrc(int j) const { return j == 0 ? z : pp; }
    __device__ __forceinline__ const double* osrc(int) const { return nullptr; }
    __device__ __forceinline__ void convert(double* const* hv, int x) const {
        hv[0][x] = first ? hv[0][x] : fma(beta, hv[1][x], hv[0][x]);  // GPupd
    }
    __device__ __forceinline__ void row(long long i, double y, const double* hc, const double*, double* s) const {
        pc[i] = hc[0];
        q[i] = y;
        s[0] = fma(hc[0], y, s[0]);
    }
    __device__ __forceinline__ void finish(PcgState* st, const double* tot) const {
        OpSpmvP{}.finish(st, tot);
    }
};

// The x/r update fused with the first two sweeps (OpUpdSweep): windows of r and
// q (and w D^-1 unless constant) become s1 = w (r - alpha q) and r_new; own x, p.
template <bool CW>
struct MOpUpdSweep {
    static constexpr int NV = 1, NH = CW ? 2 : 3, NO = 2;
    static constexpr int TICKET = kTkUpdate;
    static constexpr bool CTA_HOOKS = true;
    static constexpr bool CONVERT = true;
    OpUpdSweep<CW> u;
    __device__ __forceinline__ void init(const SolveArgs& a) { u.init(a); }
    __device__ __forceinline__ const double* hsrc(int j) const { return j == 0 ? u.rc : (j == 1 ? u.q : u.wd); }
    __device__ __forceinline__ const double* osrc(int j) const { return j == 0 ? u.x : u.p; }
    __device__ __forceinline__ void convert(double* const* hv, int x) const {
        const double t = fma(-u.alpha, hv[1][x], hv[0][x]);  // r_new = r - alpha q
        const double w = CW ? u.wc : hv[NH - 1][x];
        hv[0][x] = w * t;  // s1 = w D^-1 r_new (GWdr)
        hv[1][x] = t;
    }
    __device__ __forceinline__ void row(long long i, double y, const double* hc, const double* oc,
                                        double* s) const {
        const double ri = hc[1], wi = CW ? u.wc : hc[NH - 1];
        const double gi = hc[0];  // = wi * ri, the same product
        u.sout[i] = fma(wi, ri - y, gi);
        u.rn[i] = ri;
        u.x[i] = fma(u.alpha, oc[1], oc[0]);
        s[0] = fma(ri, ri, s[0]);
    }
    __device__ __forceinline__ void cta_pre(const SolveArgs& a) const { u.cta_pre(a); }
    __device__ __forceinline__ void cta_last(const SolveArgs& a, const double* tot) const { u.cta_last(a, tot); }
    __device__ __forceinline__ void finish(PcgState*, const double*) const {}
};

// A later sweep s_out = s_in + w D^-1 (r' - A s_in) (OpSweep with rpar)
template <bool CW>
struct MOpSweep {
    static constexpr int NV = 0, NH = 1, NO = CW ? 1 : 2;
    static constexpr int TICKET = kTkSweep;
    static constexpr bool CONVERT = false;
    const double* zin;
    const double* r;
    const double* wd;
    double* zout;
    double wc;
    __device__ __forceinline__ void init(const SolveArgs& a) { r = (a.st->it & 1) ? a.r : a.r1; }
    __device__ __forceinline__ const double* hsrc(int) const { return zin; }
    __device__ __forceinline__ const double* osrc(int j) const { return j == 0 ? r : wd; }
    __device__ __forceinline__ void convert(double* const*, int) const {}
    __device__ __forceinline__ void row(long long i, double y, const double* hc, const double* oc,
                                        double*) const {
        const double wi = CW ? wc : oc[1];
        zout[i] = fma(wi, oc[0] - y, hc[0]);
    }
    __device__ __forceinline__ void finish(PcgState*, const double*) const {}
};

