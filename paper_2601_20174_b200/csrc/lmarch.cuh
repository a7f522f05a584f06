// paper_2601_20174_b200/csrc/lmarch.cuh — the fused line march: the x/r update
// and all the smoothing sweeps of a PCG iteration in ONE kernel, for 2D
// constant-coefficient stencils (included by solve_kernels.cu after the row ops).
//
// The rows are walked as grid LINES of Lw rows (a grid row of the mesh): a CTA
// owns a slab of C consecutive columns and marches from line to line, one
// thread per column. Each thread loads its own column of the next line once
// (the loads of the next D lines are in flight in registers), and everything a
// stencil needs from the neighbouring rows comes from shared-memory rings of
// recent lines, one __syncthreads per line. Slabs overlap by a few columns, so
// there is no halo exchange. (A plain per-kernel line march — one SpMV-family
// kernel per launch in this execution shape, with 1, 2 or 4 columns per thread
// — was measured at parity with or slower than the direct kernels on C2, C3 and
// C4, as the plane march of march.cuh was: DESIGN.md §3. What pays is chaining
// the sweeps, which removes whole passes over the vectors.)
#pragma once

// The stencil patterns the march is specialised for (offsets ascending, as the
// diagonal form stores them): per offset t the line step dl and column shift dx.
// The launcher checks the matrix's offsets against the pattern.
template <int PAT>
struct LinePat;
template <>
struct LinePat<9> {  // 2D 3 x 3
    __host__ __device__ static constexpr int dl(int t) { return t / 3 - 1; }
    __host__ __device__ static constexpr int dx(int t) { return t % 3 - 1; }
};
template <>
struct LinePat<5> {  // 2D plus
    __host__ __device__ static constexpr int dl(int t) { return t == 0 ? -1 : (t == 4 ? 1 : 0); }
    __host__ __device__ static constexpr int dx(int t) { return t == 1 ? -1 : (t == 3 ? 1 : 0); }
};

struct LineGeom {
    int Lw;   // rows per line (n % Lw == 0)
    int C;    // CTA threads = columns a slab loads
    int Ci;   // columns a slab evaluates: C - 2 pad
    int pad;  // columns loaded but not evaluated on either side of a slab
    int S;    // slabs per line
    int NL;   // lines
};

// ---- the x/r update and ALL the sweeps of a two-level cycle in one march ----
// For nu1 + nu2 = T sweeps the one-pass iteration runs, between q = A p and the
// prolongation, the fused update + first two sweeps and T - 2 further sweep
// kernels (C3, T = 4: three stencil passes over the vectors). A line march can
// chain them: stage 0 forms r' = r - alpha q, s_1 = w r' and x' for a line;
// stencil stage k = 1 .. NS (NS = T - 1) forms s_{k+1} = s_k + w (r' - A s_k)
// for the line two behind stage k - 1, reading s_k from a shared-memory ring of
// lines that stage k - 1 filled in earlier steps — so one __syncthreads per
// step orders everything — and only the last stage's s_T goes back to HBM.
// Per row: r, q, x, p and the mask are read once, x', r' and s_T written once
// (72 n bytes + the run ends' extra lines instead of 56 n + (T - 2) 32 n).
// A run of lines [la, lb) starts stage 0 NS lines early and every stage k covers
// [la - (NS - k), lb + (NS - k)); slabs overlap by pad >= NS columns, since a
// slab's outermost valid column moves in by one per stencil stage.
// Constant-coefficient forms only (w D^-1 one constant, values per offset).
// Rows are bitwise those of the separate kernels: same operands, same fma
// chains; only ||r'||^2 is summed in another order.
// Ring depths. A step is [stage writes and reads, __syncthreads]. Stage k - 1
// writes line L of s_k at step j and stage k reads it last at step j + 3 (as the
// line behind L + 1), so the slot may be rewritten from step j + 4 on: 4 slots.
// r' and the mask of line L are written by stage 0 at step j and read last by
// stage NS at step j + 2 NS <= j + 6: 8 slots.
constexpr int kFusedC = 128;     // CTA threads = columns a slab loads
constexpr int kFusedSlots = 8;   // r', masks
constexpr int kFusedSSlots = 4;  // s_1 .. s_NS

#ifndef NLSP_LFUSED_MINB
#define NLSP_LFUSED_MINB 8
#endif
// LEAN (the lean cycle, solve_kernels.cu): the residual was already updated by
// OpSpmvUpd, so stage 0 only reads r and the mask and nothing but s_T is
// written (16 n bytes per iteration where the separate lean sweeps move
// 16 n + (T - 2) 24 n); the reduction is r.s_T, and the CTA hooks are
// OpSweepLean's.
template <int PAT, typename MT, int NS, int D, bool LEAN = false>
__global__ void __launch_bounds__(128, NLSP_LFUSED_MINB) k_lfused(SolveArgs a, OpUpdSweep<true> op, LineGeom g) {
    static_assert(NS >= 1 && 2 * NS + 2 <= kFusedSlots, "ring depth");
    pdl_entry();
    PcgState* st = a.st;
    if (st->done) return;
    op.init(a);
    using Pat = LinePat<PAT>;
    extern __shared__ __align__(16) unsigned char smem[];
    constexpr int W = kFusedC + 2;  // one spare column on either side of a line
    // rings: s_1 .. s_NS (NS of them), then r'; then the masks
    double* ringS = reinterpret_cast<double*>(smem);
    double* ringR = ringS + NS * kFusedSSlots * W;
    MT* ringM = reinterpret_cast<MT*>(ringR + kFusedSlots * W);
    const int c = threadIdx.x;
    const MT* __restrict__ mask = static_cast<const MT*>(a.dia.mask);
    constexpr unsigned kFull = (1u << PAT) - 1u;
    const double alpha = op.alpha, wc = op.wc;
    double s[1] = {0.0};

    struct Raw {
        double r, q, x, p;
        unsigned m;
    };
    const double* rsrc = LEAN ? a.r : op.rc;
    auto load_line = [&](Raw& v, int row) {
        v.r = rsrc[row];
        if (!LEAN) {
            v.q = op.q[row];
            v.x = op.x[row];
            v.p = op.p[row];
        }
        v.m = mask[row];
    };

    const int T = g.S * g.NL;
    const int t0 = (int)((long long)blockIdx.x * T / gridDim.x), t1 = (int)((long long)(blockIdx.x + 1) * T / gridDim.x);
    for (int t = t0; t < t1;) {
        const int sl = t / g.NL;
        const int la = t - sl * g.NL;
        const int lb = min(g.NL, la + (t1 - t));
        const int x = sl * g.Ci - g.pad + c;  // this thread's column of the line
        const bool evaluates = c >= g.pad && c < g.pad + g.Ci && x < g.Lw;
        const int xl = x < 0 ? 0 : (x > g.Lw - 1 ? g.Lw - 1 : x);
        // stage 0 covers lines la - NS .. lb - 1 + NS; the last stage trails it by 2 NS lines
        const int n0 = lb - la + 2 * NS;  // stage-0 steps
        const int NP = n0 + 2 * NS;       // steps of the run
        auto line_row = [&](int L) { return (L < 0 ? 0 : (L >= g.NL ? g.NL - 1 : L)) * g.Lw + xl; };
        // stage k evaluates lines [lo_k, lo_k + cnt_k): its share of the run, inside the grid
        int lo[NS + 1];
        unsigned cnt[NS + 1];
#pragma unroll
        for (int k = 1; k <= NS; ++k) {
            lo[k] = max(la - (NS - k), 0);
            cnt[k] = (unsigned)max(min(lb + (NS - k), g.NL) - lo[k], 0);
        }
        // this thread's own column of the three lines stage k reads (s_k of lines
        // Ak - 1, Ak, Ak + 1): it wrote them itself, so they stay in registers
        // and only the left and right neighbours come from the rings
        double own[NS + 1][3];
#pragma unroll
        for (int k = 0; k <= NS; ++k) own[k][0] = own[k][1] = own[k][2] = 0.0;
        Raw rq[D];
#pragma unroll
        for (int u = 0; u < D; ++u) load_line(rq[u], line_row(la - NS + u));
        int orow = (la - 3 * NS) * g.Lw + x;  // the last stage's row at step j: line la - NS + j - 2 NS
        __syncthreads();  // the previous run's last step still reads the rings
        for (int jb = 0; jb < NP; jb += D) {
#pragma unroll
            for (int u = 0; u < D; ++u) {
                const int j = jb + u;
                if (j < NP) {
                    const int A0 = la - NS + j;
                    // ring line offsets of the lines A0 + q, q = 0 .. 3 (s rings) and
                    // A0 - 2 k (r', masks): every stage's lines are among them
                    int b4[4], b8[NS + 1];
#pragma unroll
                    for (int q = 0; q < 4; ++q) b4[q] = ((A0 + 64 + q) & (kFusedSSlots - 1)) * W + 1 + c;
#pragma unroll
                    for (int k = 0; k <= NS; ++k) b8[k] = ((A0 + 64 - 2 * k) & (kFusedSlots - 1)) * W + 1 + c;
                    // this step's line of stage 0: take it from the prefetch ring, refill the ring
                    Raw v = rq[u];
                    if (j + D < n0) load_line(rq[u], line_row(A0 + D));
                    // ---- stencil stages, last first: s_{k+1} of the line 2 k behind stage 0.
                    // own[k - 1] then still holds s_k of lines Ak - 1, Ak, Ak + 1 (stage
                    // k - 1 pushes this step's line after stage k has run)
#pragma unroll
                    for (int k = NS; k >= 1; --k) {
                        const int Ak = A0 - 2 * k;
                        double zo = 0.0;
                        if ((unsigned)(Ak - lo[k]) < cnt[k]) {
                            const double* in = ringS + (k - 1) * kFusedSSlots * W;
                            // lines Ak - 1, Ak, Ak + 1 = A0 + (-2 k - 1, -2 k, -2 k + 1)
                            const int b[3] = {b4[(4 * NS - 2 * k - 1) & 3], b4[(4 * NS - 2 * k) & 3],
                                              b4[(4 * NS - 2 * k + 1) & 3]};
                            const unsigned m = ringM[b8[k]];
                            double gv[PAT];
#pragma unroll
                            for (int tt = 0; tt < PAT; ++tt)
                                gv[tt] = Pat::dx(tt) == 0 ? own[k - 1][Pat::dl(tt) + 1] : in[b[Pat::dl(tt) + 1] + Pat::dx(tt)];
                            double y = 0.0;
                            if (m == kFull) {
#pragma unroll
                                for (int tt = 0; tt < PAT; ++tt) y = fma(a.dia.val[tt], gv[tt], y);
                            } else {
#pragma unroll
                                for (int tt = 0; tt < PAT; ++tt)
                                    if ((m >> tt) & 1u) y = fma(a.dia.val[tt], gv[tt], y);
                            }
                            const double rk = ringR[b8[k]];
                            zo = fma(wc, rk - y, own[k - 1][1]);
                            if (k < NS) ringS[k * kFusedSSlots * W + b4[(4 * NS - 2 * k) & 3]] = zo;
                            else if (evaluates) {
                                op.sout[orow] = zo;
                                if (LEAN) s[0] = fma(rk, zo, s[0]);  // r.s_T
                            }
                        }
                        if (k < NS) {  // every step pushes (a line outside the stage's range: a placeholder)
                            own[k][0] = own[k][1];
                            own[k][1] = own[k][2];
                            own[k][2] = zo;
                        }
                    }
                    // ---- stage 0: r' = r - alpha q, s_1 = w r', x' = x + alpha p
                    {
                        const double rn = LEAN ? v.r : fma(-alpha, v.q, v.r);
                        const double s1 = wc * rn;
                        own[0][0] = own[0][1];
                        own[0][1] = own[0][2];
                        own[0][2] = s1;
                        if (j < n0) {
                            ringS[b4[0]] = s1;
                            ringR[b8[0]] = rn;
                            ringM[b8[0]] = (MT)v.m;
                            if (!LEAN && evaluates && (unsigned)(A0 - la) < (unsigned)(lb - la)) {
                                const int row = orow + 2 * NS * g.Lw;
                                op.rn[row] = rn;
                                op.x[row] = fma(alpha, v.p, v.x);
                                s[0] = fma(rn, rn, s[0]);
                            }
                        }
                    }
                    orow += g.Lw;
                    __syncthreads();
                }
            }
        }
        t += lb - la;
    }
    double v[1] = {s[0]}, tot[1];
    op.cta_pre(a);  // the column sums of the last pass over W (both cycles)
    if (grid_reduce<1>(v, a.partials, &st->counter[kTkUpdate], tot)) {
        if (!LEAN) op.cta_last(a, tot);
        else if (threadIdx.x == 0) st->rz_new = tot[0];
    }
}
