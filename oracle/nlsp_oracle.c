/* oracle/nlsp_oracle.c — TEST INFRASTRUCTURE ONLY: the CPU oracle.
 *
 * A plain-C restatement of the reference's two-level-preconditioned CG path
 * (/root/reference/proj/include/nlsp/, cited as file:line). Sequential loops in
 * the reference's order, compiled with -ffp-contract=off (oracle/Makefile).
 *
 * Pinned by tests/test_oracle_pin.py: bitwise against the reference's own code
 * built with -ffp-contract=off (oracle/_ref/libnlsp_ref_strict.so) and within
 * rounding of the default build; also against every hand-checked case in the
 * reference's tests (tests/unit/test_linalg.cpp, test_smoothing.cpp,
 * test_two_level.cpp) and the committed golden fixtures in tests/golden/.
 *
 * Never loaded by the product library; see nlsp_oracle.h.
 */
#include "nlsp_oracle.h"

#include <float.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static _Thread_local char g_err[256];

static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}

const char* orc_last_error(void) { return g_err; }

/* ---------------------------------------------------------------- rng.hpp -- */

/* splitmix64 finaliser, rng.hpp:12-17 */
uint64_t orc_mix_seed(uint64_t seed, uint64_t tag) {
    uint64_t z = seed + 0x9e3779b97f4a7c15ULL * (tag + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* std::mt19937_64 (the engine behind Rng, rng.hpp:22,71), standard parameters */
typedef struct {
    uint64_t mt[312];
    int idx;
    double cached;
    int has_cached;
} orc_rng;

static void rng_init(orc_rng* g, uint64_t seed) {
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
    g->cached = 0.0;
    g->has_cached = 0;
}

static uint64_t rng_u64(orc_rng* g) {
    if (g->idx >= 312) {
        const uint64_t upper = 0xFFFFFFFF80000000ULL, lower = 0x7FFFFFFFULL;
        for (int i = 0; i < 312; ++i) {
            uint64_t y = (g->mt[i] & upper) | (g->mt[(i + 1) % 312] & lower);
            uint64_t next = g->mt[(i + 156) % 312] ^ (y >> 1);
            if (y & 1ULL) next ^= 0xB5026F5AA96619E9ULL;
            g->mt[i] = next;
        }
        g->idx = 0;
    }
    uint64_t x = g->mt[g->idx++];
    x ^= (x >> 29) & 0x5555555555555555ULL;
    x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
    x ^= (x << 37) & 0xFFF7EEE000000000ULL;
    x ^= x >> 43;
    return x;
}

/* top 53 bits, rng.hpp:29-31 */
static double rng_uniform(orc_rng* g) { return (double)(rng_u64(g) >> 11) * 0x1.0p-53; }

/* Box-Muller with the sine value cached, rng.hpp:36-49 */
static double rng_normal(orc_rng* g) {
    if (g->has_cached) {
        g->has_cached = 0;
        return g->cached;
    }
    double u1 = rng_uniform(g);
    double u2 = rng_uniform(g);
    while (u1 <= 0.0) u1 = rng_uniform(g);
    const double r = sqrt(-2.0 * log(u1));
    const double a = 2.0 * 3.141592653589793 * u2;
    g->cached = r * sin(a);
    g->has_cached = 1;
    return r * cos(a);
}

void orc_rng_u64_fill(uint64_t seed, uint64_t count, uint64_t* out) {
    orc_rng g;
    rng_init(&g, seed);
    for (uint64_t i = 0; i < count; ++i) out[i] = rng_u64(&g);
}

void orc_rng_normal_fill(uint64_t seed, uint64_t count, double* out) {
    orc_rng g;
    rng_init(&g, seed);
    for (uint64_t i = 0; i < count; ++i) out[i] = rng_normal(&g);
}

/* rng.hpp:33 */
void orc_rng_uniform_fill(uint64_t seed, uint64_t count, double lo, double hi, double* out) {
    orc_rng g;
    rng_init(&g, seed);
    for (uint64_t i = 0; i < count; ++i) out[i] = lo + (hi - lo) * rng_uniform(&g);
}

/* ------------------------------------------------------------- sparse.hpp -- */

/* y_i = sum_k v_k x[col_k] in row-traversal order, sparse.hpp:116-128 */
static void spmv_raw(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                     const double* x, double* y) {
    for (uint64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) s += v[k] * x[ci[k]];
        y[i] = s;
    }
}

int orc_spmv(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
             const double* x, double* y) {
    spmv_raw(n, rp, ci, v, x, y);
    return ORC_OK;
}

/* at(i,i) by linear search, sparse.hpp:68-78 */
static double diag_at(const uint64_t* rp, const uint64_t* ci, const double* v, uint64_t i) {
    for (uint64_t k = rp[i]; k < rp[i + 1]; ++k)
        if (ci[k] == i) return v[k];
    return 0.0;
}

/* Y = A X, X row-major n x m, sparse.hpp:131-146 */
static void spmm_raw(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                     uint64_t m, const double* x, double* y) {
    memset(y, 0, sizeof(double) * n * m);
    for (uint64_t i = 0; i < n; ++i) {
        double* yi = y + i * m;
        for (uint64_t k = rp[i]; k < rp[i + 1]; ++k) {
            const double aik = v[k];
            const double* xr = x + ci[k] * m;
            for (uint64_t j = 0; j < m; ++j) yi[j] += aik * xr[j];
        }
    }
}

/* ---------------------------------------------------------- smoothing.hpp -- */

/* JacobiSmoother ctor, smoothing.hpp:19-29 */
int orc_inv_diag(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                 double omega, double* dinv) {
    if (omega < 0.0 || omega > 1.0) return fail(ORC_VALIDATION, "jacobi: omega must lie in [0, 1]");
    for (uint64_t i = 0; i < n; ++i) {
        const double d = diag_at(rp, ci, v, i);
        if (d <= 0.0) return fail(ORC_NUMERIC, "jacobi: non-positive diagonal");
        dinv[i] = 1.0 / d;
    }
    return ORC_OK;
}

/* x <- x + w D^-1 (b - A x), smoothing.hpp:34-41 */
static void sweep_vec(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                      const double* dinv, double omega, double* x, const double* b, double* ax) {
    spmv_raw(n, rp, ci, v, x, ax);
    for (uint64_t i = 0; i < n; ++i) x[i] += omega * dinv[i] * (b[i] - ax[i]);
}

int orc_jacobi_sweep(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                     double omega, uint64_t sweeps, double* x, const double* b) {
    double* dinv = malloc(sizeof(double) * (n ? n : 1));
    double* ax = malloc(sizeof(double) * (n ? n : 1));
    int st = orc_inv_diag(n, rp, ci, v, omega, dinv);
    for (uint64_t s = 0; st == ORC_OK && s < sweeps; ++s) sweep_vec(n, rp, ci, v, dinv, omega, x, b, ax);
    free(dinv);
    free(ax);
    return st;
}

/* block sweep with b = 0, smoothing.hpp:50-60 */
static void sweep_block(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                        const double* dinv, double omega, uint64_t m, double* x, double* ax) {
    spmm_raw(n, rp, ci, v, m, x, ax);
    for (uint64_t i = 0; i < n; ++i) {
        const double w = omega * dinv[i];
        for (uint64_t j = 0; j < m; ++j) {
            const double rhs = 0.0;
            x[i * m + j] += w * (rhs - ax[i * m + j]);
        }
    }
}

int orc_block_sweeps(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                     uint64_t m, double* s, uint64_t sweeps, double omega) {
    double* dinv = malloc(sizeof(double) * (n ? n : 1));
    int st = orc_inv_diag(n, rp, ci, v, omega, dinv);
    if (st == ORC_OK && sweeps) {
        double* ax = malloc(sizeof(double) * (n * m > 0 ? n * m : 1));
        for (uint64_t k = 0; k < sweeps; ++k) sweep_block(n, rp, ci, v, dinv, omega, m, s, ax);
        free(ax);
    }
    free(dinv);
    return st;
}

/* smoothing.hpp:81-100: i-major N(0,1) fill from Rng(mix_seed(seed, "smoo")),
 * Dirichlet rows zero (and draw nothing), then `sweeps` homogeneous sweeps */
int orc_generate_smoothed_vectors(uint64_t n, const uint64_t* rp, const uint64_t* ci,
                                  const double* v, const uint8_t* mask, uint64_t k,
                                  uint64_t sweeps, double omega, uint64_t seed, double* s_out) {
    if (k < 1) return fail(ORC_VALIDATION, "generate_smoothed_vectors: K must be positive");
    orc_rng g;
    rng_init(&g, orc_mix_seed(seed, 0x736d6f6fULL));
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < k; ++j) s_out[i * k + j] = (mask && mask[i]) ? 0.0 : rng_normal(&g);
    return orc_block_sweeps(n, rp, ci, v, k, s_out, sweeps, omega);
}

/* -------------------------------------------------------------- dense.hpp -- */

/* C = A^T B, row-k outer loop with the zero skip, dense.hpp:83-97 */
void orc_matmul_tn(uint64_t rows, uint64_t ca, uint64_t cb, const double* a, const double* b,
                   double* c) {
    memset(c, 0, sizeof(double) * ca * cb);
    for (uint64_t k = 0; k < rows; ++k) {
        const double* ak = a + k * ca;
        const double* bk = b + k * cb;
        for (uint64_t i = 0; i < ca; ++i) {
            const double aki = ak[i];
            if (aki == 0.0) continue;
            double* ci = c + i * cb;
            for (uint64_t j = 0; j < cb; ++j) ci[j] += aki * bk[j];
        }
    }
}

/* dense.hpp:122-129 */
static double frobenius(uint64_t rows, uint64_t cols, const double* m) {
    double s = 0.0;
    for (uint64_t i = 0; i < rows * cols; ++i) s += m[i] * m[i];
    return sqrt(s);
}

/* max |A^T A - I|, dense.hpp:175-182 */
double orc_orthonormality_defect(uint64_t rows, uint64_t cols, const double* a) {
    double* g = malloc(sizeof(double) * (cols * cols > 0 ? cols * cols : 1));
    orc_matmul_tn(rows, cols, cols, a, a, g);
    double d = 0.0;
    for (uint64_t i = 0; i < cols; ++i)
        for (uint64_t j = 0; j < cols; ++j) {
            const double e = fabs(g[i * cols + j] - (i == j ? 1.0 : 0.0));
            if (e > d) d = e;
        }
    free(g);
    return d;
}

/* ---------------------------------------------------------------- svd.hpp -- */

/* cyclic two-sided Jacobi, off-norm < 1e-12 ||A||_F, <= 30 sweeps, then a
 * stable descending sort; svd.hpp:23-88 */
int orc_jacobi_eigh(uint64_t n, const double* g, double* evals, double* evecs, int* sweeps_out) {
    double* a = malloc(sizeof(double) * (n * n > 0 ? n * n : 1));
    double* v = calloc(n * n > 0 ? n * n : 1, sizeof(double));
    memcpy(a, g, sizeof(double) * n * n);
    for (uint64_t i = 0; i < n; ++i) v[i * n + i] = 1.0;
    const double total = frobenius(n, n, a);
    int sweeps = 0;
    for (;;) {
        double off = 0.0;
        for (uint64_t i = 0; i < n; ++i)
            for (uint64_t j = i + 1; j < n; ++j) off += 2.0 * a[i * n + j] * a[i * n + j];
        off = sqrt(off);
        if (!(off > 1e-12 * total && total > 0.0)) break;
        if (sweeps >= 30) {
            free(a);
            free(v);
            return fail(ORC_CONVERGENCE, "jacobi_eigh: no convergence after 30 sweeps");
        }
        ++sweeps;
        for (uint64_t p = 0; p + 1 < n; ++p) {
            for (uint64_t q = p + 1; q < n; ++q) {
                const double apq = a[p * n + q];
                if (apq == 0.0) continue;
                const double theta = (a[q * n + q] - a[p * n + p]) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) /
                                 (fabs(theta) + sqrt(theta * theta + 1.0));
                const double c = 1.0 / sqrt(t * t + 1.0);
                const double s = t * c;
                for (uint64_t i = 0; i < n; ++i) {
                    const double aip = a[i * n + p], aiq = a[i * n + q];
                    a[i * n + p] = c * aip - s * aiq;
                    a[i * n + q] = s * aip + c * aiq;
                }
                for (uint64_t j = 0; j < n; ++j) {
                    const double apj = a[p * n + j], aqj = a[q * n + j];
                    a[p * n + j] = c * apj - s * aqj;
                    a[q * n + j] = s * apj + c * aqj;
                }
                for (uint64_t i = 0; i < n; ++i) {
                    const double vip = v[i * n + p], viq = v[i * n + q];
                    v[i * n + p] = c * vip - s * viq;
                    v[i * n + q] = s * vip + c * viq;
                }
            }
        }
    }
    /* stable sort of indices by eigenvalue, descending (insertion sort is stable) */
    uint64_t* order = malloc(sizeof(uint64_t) * (n ? n : 1));
    for (uint64_t i = 0; i < n; ++i) order[i] = i;
    for (uint64_t i = 1; i < n; ++i) {
        const uint64_t key = order[i];
        uint64_t j = i;
        while (j > 0 && a[key * n + key] > a[order[j - 1] * n + order[j - 1]]) {
            order[j] = order[j - 1];
            --j;
        }
        order[j] = key;
    }
    for (uint64_t j = 0; j < n; ++j) {
        evals[j] = a[order[j] * n + order[j]];
        for (uint64_t i = 0; i < n; ++i) evecs[i * n + j] = v[i * n + order[j]];
    }
    *sweeps_out = sweeps;
    free(order);
    free(a);
    free(v);
    return ORC_OK;
}

/* svd.hpp:101-126 */
static int complete_orthonormal(uint64_t n, uint64_t r, double* u, uint64_t have) {
    double* v = malloc(sizeof(double) * (n ? n : 1));
    for (uint64_t j = have; j < r; ++j) {
        int placed = 0;
        for (uint64_t cand = 0; cand < n && !placed; ++cand) {
            for (uint64_t i = 0; i < n; ++i) v[i] = (i == cand) ? 1.0 : 0.0;
            for (int pass = 0; pass < 2; ++pass) {
                for (uint64_t p = 0; p < j; ++p) {
                    double c = 0.0;
                    for (uint64_t i = 0; i < n; ++i) c += u[i * r + p] * v[i];
                    for (uint64_t i = 0; i < n; ++i) v[i] -= c * u[i * r + p];
                }
            }
            double nrm = 0.0;
            for (uint64_t i = 0; i < n; ++i) nrm += v[i] * v[i];
            nrm = sqrt(nrm);
            if (nrm > 0.5) {
                for (uint64_t i = 0; i < n; ++i) u[i * r + j] = v[i] / nrm;
                placed = 1;
            }
        }
        if (!placed) {
            free(v);
            return fail(ORC_NUMERIC, "complete_orthonormal: no candidate found");
        }
    }
    free(v);
    return ORC_OK;
}

/* svd.hpp:130-147 */
static int reorthonormalize_columns(uint64_t n, uint64_t r, double* u) {
    double* v = malloc(sizeof(double) * (n ? n : 1));
    for (uint64_t j = 0; j < r; ++j) {
        for (uint64_t i = 0; i < n; ++i) v[i] = u[i * r + j];
        for (uint64_t p = 0; p < j; ++p) {
            double c = 0.0;
            for (uint64_t i = 0; i < n; ++i) c += u[i * r + p] * v[i];
            for (uint64_t i = 0; i < n; ++i) v[i] -= c * u[i * r + p];
        }
        double nrm = 0.0;
        for (uint64_t i = 0; i < n; ++i) nrm += v[i] * v[i];
        nrm = sqrt(nrm);
        if (nrm == 0.0) {
            free(v);
            return fail(ORC_NUMERIC, "reorthonormalize: zero column");
        }
        for (uint64_t i = 0; i < n; ++i) u[i * r + j] = v[i] / nrm;
    }
    free(v);
    return ORC_OK;
}

/* Thin SVD through the Gram of the smaller dimension, svd.hpp:155-227.
 * u: rows x r, sigma: r, v: cols x r, r = min(rows, cols). */
int orc_svd(uint64_t rows, uint64_t cols, const double* s, double* u, double* sigma, double* vout,
            int* sweeps) {
    for (uint64_t i = 0; i < rows * cols; ++i)
        if (!isfinite(s[i])) return fail(ORC_VALIDATION, "svd_oracle: non-finite entries");
    const uint64_t n = rows, m = cols, r = n < m ? n : m;
    if (r == 0) return fail(ORC_VALIDATION, "svd_oracle: empty matrix");
    const int gram_right = (m <= n);
    double* gram = malloc(sizeof(double) * r * r);
    if (gram_right) {
        orc_matmul_tn(n, m, m, s, s, gram);
    } else {
        double* st = malloc(sizeof(double) * n * m);
        for (uint64_t i = 0; i < n; ++i)
            for (uint64_t j = 0; j < m; ++j) st[j * n + i] = s[i * m + j];
        orc_matmul_tn(m, n, n, st, st, gram);
        free(st);
    }
    double* ev = malloc(sizeof(double) * r);
    double* small = malloc(sizeof(double) * r * r); /* eigenvectors, r x r */
    int st = orc_jacobi_eigh(r, gram, ev, small, sweeps);
    free(gram);
    if (st != ORC_OK) {
        free(ev);
        free(small);
        return st;
    }
    const double lam_floor = ev[0] * 64.0 * DBL_EPSILON;
    for (uint64_t i = 0; i < r; ++i) {
        const double lam = ev[i] <= lam_floor ? 0.0 : ev[i];
        sigma[i] = sqrt(lam > 0.0 ? lam : 0.0);
    }
    const double cutoff = sigma[0] * 1e-13;
    const uint64_t big_rows = gram_right ? n : m;
    double* big = calloc(big_rows * r, sizeof(double));
    uint64_t solid = 0;
    for (uint64_t j = 0; j < r; ++j) {
        if (sigma[j] <= cutoff) break;
        for (uint64_t i = 0; i < big_rows; ++i) {
            double acc = 0.0;
            if (gram_right)
                for (uint64_t k = 0; k < m; ++k) acc += s[i * m + k] * small[k * r + j];
            else
                for (uint64_t k = 0; k < n; ++k) acc += s[k * m + i] * small[k * r + j];
            big[i * r + j] = acc / sigma[j];
        }
        solid = j + 1;
    }
    st = complete_orthonormal(big_rows, r, big, solid);
    if (st == ORC_OK && orc_orthonormality_defect(big_rows, r, big) > 1e-11)
        st = reorthonormalize_columns(big_rows, r, big);
    if (st != ORC_OK) {
        free(ev);
        free(small);
        free(big);
        return st;
    }
    double* left = gram_right ? big : small;
    double* right = gram_right ? small : big;
    const uint64_t lrows = gram_right ? n : n, rrows = gram_right ? m : m;
    for (uint64_t j = 0; j < r; ++j) {
        uint64_t arg = 0;
        double best = -1.0;
        for (uint64_t i = 0; i < lrows; ++i) {
            const double mag = fabs(left[i * r + j]);
            if (mag > best) {
                best = mag;
                arg = i;
            }
        }
        if (left[arg * r + j] < 0.0) {
            for (uint64_t i = 0; i < lrows; ++i) left[i * r + j] = -left[i * r + j];
            for (uint64_t i = 0; i < rrows; ++i) right[i * r + j] = -right[i * r + j];
        }
    }
    memcpy(u, left, sizeof(double) * n * r);
    memcpy(vout, right, sizeof(double) * m * r);
    free(ev);
    free(small);
    free(big);
    return ORC_OK;
}

/* ----------------------------------------------------------------- qr.hpp -- */

/* MGS with a second elimination pass, diag(R) >= 0, qr.hpp:18-45 */
int orc_qr_thin(uint64_t n, uint64_t k, const double* m, double* q, double* r) {
    if (n < k) return fail(ORC_VALIDATION, "qr_thin: requires rows >= cols");
    const double scale = frobenius(n, k, m);
    memset(q, 0, sizeof(double) * n * k);
    memset(r, 0, sizeof(double) * k * k);
    double* v = malloc(sizeof(double) * (n ? n : 1));
    for (uint64_t j = 0; j < k; ++j) {
        for (uint64_t i = 0; i < n; ++i) v[i] = m[i * k + j];
        for (int pass = 0; pass < 2; ++pass) {
            for (uint64_t p = 0; p < j; ++p) {
                double c = 0.0;
                for (uint64_t i = 0; i < n; ++i) c += q[i * k + p] * v[i];
                for (uint64_t i = 0; i < n; ++i) v[i] -= c * q[i * k + p];
                r[p * k + j] += c;
            }
        }
        double nrm = 0.0;
        for (uint64_t i = 0; i < n; ++i) nrm += v[i] * v[i];
        nrm = sqrt(nrm);
        if (nrm < 1e-12 * scale) {
            free(v);
            return fail(ORC_RANK_DEFICIENT, "qr_thin: rank-deficient");
        }
        r[j * k + j] = nrm;
        for (uint64_t i = 0; i < n; ++i) q[i * k + j] = v[i] / nrm;
    }
    free(v);
    return ORC_OK;
}

/* ----------------------------------------------------------- cholesky.hpp -- */

/* LL^T with the 1e-10 symmetry gate and pivot > 0, cholesky.hpp:15-37 */
int orc_cholesky(uint64_t n, const double* a, double* l) {
    double mx = 0.0;
    for (uint64_t i = 0; i < n * n; ++i) mx = fabs(a[i]) > mx ? fabs(a[i]) : mx;
    const double scale = mx > 0.0 ? mx : 1.0;
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = i + 1; j < n; ++j)
            if (fabs(a[i * n + j] - a[j * n + i]) > 1e-10 * scale)
                return fail(ORC_NOT_SPD, "cholesky: matrix not symmetric");
    memset(l, 0, sizeof(double) * n * n);
    for (uint64_t j = 0; j < n; ++j) {
        double d = a[j * n + j];
        for (uint64_t k = 0; k < j; ++k) d -= l[j * n + k] * l[j * n + k];
        if (d <= 0.0) return fail(ORC_NOT_SPD, "cholesky: non-positive pivot");
        l[j * n + j] = sqrt(d);
        for (uint64_t i = j + 1; i < n; ++i) {
            double s = a[i * n + j];
            for (uint64_t k = 0; k < j; ++k) s -= l[i * n + k] * l[j * n + k];
            l[i * n + j] = s / l[j * n + j];
        }
    }
    return ORC_OK;
}

/* forward then backward substitution, cholesky.hpp:41-57 */
void orc_cholesky_solve_factored(uint64_t n, const double* l, const double* rhs, double* x) {
    double* y = malloc(sizeof(double) * (n ? n : 1));
    for (uint64_t i = 0; i < n; ++i) {
        double s = rhs[i];
        for (uint64_t k = 0; k < i; ++k) s -= l[i * n + k] * y[k];
        y[i] = s / l[i * n + i];
    }
    for (uint64_t ii = n; ii-- > 0;) {
        double s = y[ii];
        for (uint64_t k = ii + 1; k < n; ++k) s -= l[k * n + ii] * x[k];
        x[ii] = s / l[ii * n + ii];
    }
    free(y);
}

/* ---------------------------------------------------------- two_level.hpp -- */

struct orc_twolevel {
    uint64_t n, k, nu1, nu2;
    double omega;
    double* basis;  /* n x k, orthonormal (qr_thin(basis_any).q) */
    double* coarse; /* k x k symmetrised Galerkin operator */
    double* l;      /* k x k Cholesky factor */
    double* dinv;   /* smoother inv_diag */
};

void orc_twolevel_destroy(orc_twolevel* t) {
    if (!t) return;
    free(t->basis);
    free(t->coarse);
    free(t->l);
    free(t->dinv);
    free(t);
}

/* TwoLevelPreconditioner ctor, two_level.hpp:24-53 */
int orc_twolevel_create(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                        uint64_t k, const double* basis_any, double omega, uint64_t nu1,
                        uint64_t nu2, orc_twolevel** out) {
    *out = NULL;
    orc_twolevel* t = calloc(1, sizeof *t);
    t->n = n;
    t->k = k;
    t->nu1 = nu1;
    t->nu2 = nu2;
    t->omega = omega;
    t->dinv = malloc(sizeof(double) * (n ? n : 1));
    int st = orc_inv_diag(n, rp, ci, v, omega, t->dinv); /* smoother_ member init first */
    if (st == ORC_OK && k == 0) st = fail(ORC_VALIDATION, "two-level: empty coarse space");
    if (st != ORC_OK) {
        orc_twolevel_destroy(t);
        return st;
    }
    t->basis = malloc(sizeof(double) * n * k);
    double* r = malloc(sizeof(double) * k * k);
    st = orc_qr_thin(n, k, basis_any, t->basis, r);
    free(r);
    if (st != ORC_OK) {
        orc_twolevel_destroy(t);
        return st;
    }
    t->coarse = malloc(sizeof(double) * k * k);
    double* col = malloc(sizeof(double) * (n ? n : 1));
    double* acol = malloc(sizeof(double) * (n ? n : 1));
    for (uint64_t j = 0; j < k; ++j) {
        for (uint64_t i = 0; i < n; ++i) col[i] = t->basis[i * k + j];
        spmv_raw(n, rp, ci, v, col, acol);
        for (uint64_t i = 0; i < k; ++i) {
            double s = 0.0;
            for (uint64_t row = 0; row < n; ++row) s += t->basis[row * k + i] * acol[row];
            t->coarse[i * k + j] = s;
        }
    }
    free(col);
    free(acol);
    for (uint64_t i = 0; i < k; ++i)
        for (uint64_t j = i + 1; j < k; ++j) {
            const double val = 0.5 * (t->coarse[i * k + j] + t->coarse[j * k + i]);
            t->coarse[i * k + j] = val;
            t->coarse[j * k + i] = val;
        }
    t->l = malloc(sizeof(double) * k * k);
    st = orc_cholesky(k, t->coarse, t->l);
    if (st != ORC_OK) {
        orc_twolevel_destroy(t);
        return st;
    }
    *out = t;
    return ORC_OK;
}

/* The operator of an already-built preconditioner from its parts (orthonormal
 * basis, symmetric A_c): smoother and Cholesky as in the constructor
 * (two_level.hpp:25,52), the QR/Galerkin body skipped. Used to time the solve
 * loop at sizes where the constructor's column-strided loops take minutes. */
int orc_twolevel_from_parts(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                            uint64_t k, const double* basis, const double* coarse, double omega,
                            uint64_t nu1, uint64_t nu2, orc_twolevel** out) {
    *out = NULL;
    orc_twolevel* t = calloc(1, sizeof *t);
    t->n = n;
    t->k = k;
    t->nu1 = nu1;
    t->nu2 = nu2;
    t->omega = omega;
    t->dinv = malloc(sizeof(double) * (n ? n : 1));
    int st = orc_inv_diag(n, rp, ci, v, omega, t->dinv);
    if (st == ORC_OK && k == 0) st = fail(ORC_VALIDATION, "two-level: empty coarse space");
    if (st != ORC_OK) {
        orc_twolevel_destroy(t);
        return st;
    }
    t->basis = malloc(sizeof(double) * n * k);
    memcpy(t->basis, basis, sizeof(double) * n * k);
    t->coarse = malloc(sizeof(double) * k * k);
    memcpy(t->coarse, coarse, sizeof(double) * k * k);
    t->l = malloc(sizeof(double) * k * k);
    st = orc_cholesky(k, t->coarse, t->l);
    if (st != ORC_OK) {
        orc_twolevel_destroy(t);
        return st;
    }
    *out = t;
    return ORC_OK;
}

void orc_twolevel_export(const orc_twolevel* t, double* basis, double* chol, double* coarse) {
    if (basis) memcpy(basis, t->basis, sizeof(double) * t->n * t->k);
    if (chol) memcpy(chol, t->l, sizeof(double) * t->k * t->k);
    if (coarse) memcpy(coarse, t->coarse, sizeof(double) * t->k * t->k);
}

/* one two-grid cycle from zero, two_level.hpp:60-81 */
static void twolevel_apply_raw(const orc_twolevel* t, const uint64_t* rp, const uint64_t* ci,
                               const double* v, const double* rhs, double* z, double* work) {
    const uint64_t n = t->n, k = t->k;
    double* ax = work;          /* n */
    double* res = work + n;     /* n */
    double* crhs = work + 2 * n; /* k */
    double* cerr = crhs + k;    /* k */
    memset(z, 0, sizeof(double) * n);
    for (uint64_t s = 0; s < t->nu1; ++s) sweep_vec(n, rp, ci, v, t->dinv, t->omega, z, rhs, ax);
    spmv_raw(n, rp, ci, v, z, ax);
    for (uint64_t i = 0; i < n; ++i) res[i] = rhs[i] - ax[i];
    memset(crhs, 0, sizeof(double) * k);
    for (uint64_t i = 0; i < n; ++i)
        for (uint64_t j = 0; j < k; ++j) crhs[j] += t->basis[i * k + j] * res[i];
    orc_cholesky_solve_factored(k, t->l, crhs, cerr);
    for (uint64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (uint64_t j = 0; j < k; ++j) s += t->basis[i * k + j] * cerr[j];
        z[i] += s;
    }
    for (uint64_t s = 0; s < t->nu2; ++s) sweep_vec(n, rp, ci, v, t->dinv, t->omega, z, rhs, ax);
}

int orc_twolevel_apply(const orc_twolevel* t, uint64_t n, const uint64_t* rp,
                       const uint64_t* ci, const double* v, const double* r, double* z) {
    if (n != t->n) return fail(ORC_VALIDATION, "two-level apply: dimension mismatch");
    double* work = malloc(sizeof(double) * (2 * n + 2 * t->k + 1));
    twolevel_apply_raw(t, rp, ci, v, r, z, work);
    free(work);
    return ORC_OK;
}

/* preconditioned CG from x0 = 0, recurrence-residual stop, two_level.hpp:141-191 */
int orc_pcg(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v, int kind,
            const orc_twolevel* t, const double* b, double delta, uint64_t max_iters, double* x,
            double* hist, uint64_t hist_cap, uint64_t* iterations, int* converged,
            double* true_res) {
    if (kind == 2 && (!t || t->n != n)) return fail(ORC_VALIDATION, "pcg: dimension mismatch");
    double b_norm = 0.0;
    for (uint64_t i = 0; i < n; ++i) b_norm += b[i] * b[i];
    b_norm = sqrt(b_norm);
    if (b_norm == 0.0) return fail(ORC_VALIDATION, "pcg: zero right-hand side");
    const uint64_t nn = n ? n : 1;
    double* r = malloc(sizeof(double) * nn);
    double* z = malloc(sizeof(double) * nn);
    double* p = malloc(sizeof(double) * nn);
    double* ap = malloc(sizeof(double) * nn);
    double* d = NULL;
    double* work = malloc(sizeof(double) * (2 * nn + 2 * (t ? t->k : 0) + 1));
    int st = ORC_OK;
    memset(x, 0, sizeof(double) * n);
    memcpy(r, b, sizeof(double) * n);
    *iterations = 0;
    *converged = 0;
    if (kind == 1) { /* JacobiPreconditioner, two_level.hpp:107-118 */
        d = malloc(sizeof(double) * nn);
        for (uint64_t i = 0; i < n; ++i) d[i] = diag_at(rp, ci, v, i);
    }
#define APPLY_M(rin, zout)                                                                   \
    do {                                                                                     \
        if (kind == 0) {                                                                     \
            memcpy(zout, rin, sizeof(double) * n);                                           \
        } else if (kind == 1) {                                                              \
            for (uint64_t i_ = 0; i_ < n; ++i_) {                                            \
                if (d[i_] <= 0.0) {                                                          \
                    st = fail(ORC_NUMERIC, "jacobi preconditioner: non-positive diagonal");  \
                    goto done;                                                               \
                }                                                                            \
                zout[i_] = rin[i_] / d[i_];                                                  \
            }                                                                                \
        } else {                                                                             \
            twolevel_apply_raw(t, rp, ci, v, rin, zout, work);                               \
        }                                                                                    \
    } while (0)
    APPLY_M(r, z);
    memcpy(p, z, sizeof(double) * n);
    double rz = 0.0;
    for (uint64_t i = 0; i < n; ++i) rz += r[i] * z[i];
    for (uint64_t iter = 0; iter < max_iters; ++iter) {
        spmv_raw(n, rp, ci, v, p, ap);
        double pap = 0.0;
        for (uint64_t i = 0; i < n; ++i) pap += p[i] * ap[i];
        if (pap <= 0.0) {
            st = fail(ORC_NOT_SPD, "pcg: p^T A p <= 0, operator not SPD");
            goto done;
        }
        const double alpha = rz / pap;
        for (uint64_t i = 0; i < n; ++i) {
            x[i] += alpha * p[i];
            r[i] -= alpha * ap[i];
        }
        double r_norm = 0.0;
        for (uint64_t i = 0; i < n; ++i) r_norm += r[i] * r[i];
        r_norm = sqrt(r_norm);
        if (hist && iter < hist_cap) hist[iter] = r_norm / b_norm;
        *iterations = iter + 1;
        if (r_norm / b_norm < delta) {
            *converged = 1;
            break;
        }
        APPLY_M(r, z);
        double rz_next = 0.0;
        for (uint64_t i = 0; i < n; ++i) rz_next += r[i] * z[i];
        const double beta = rz_next / rz;
        rz = rz_next;
        for (uint64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
#undef APPLY_M
    spmv_raw(n, rp, ci, v, x, ap);
    double tr = 0.0;
    for (uint64_t i = 0; i < n; ++i) tr += (b[i] - ap[i]) * (b[i] - ap[i]);
    *true_res = sqrt(tr) / b_norm;
done:
    free(r);
    free(z);
    free(p);
    free(ap);
    free(d);
    free(work);
    return st;
}
