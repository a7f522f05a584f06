// paper_2601_20174_b200/csrc/inputs.cpp — seeded synthetic inputs for the
// BASELINE.json configs C1–C5. Host C++, no CUDA. See
// include/nlsp_inputs.h for the contract.
//
// The reference has none of these operators (only P1 FEM, fem.hpp:121-236);
// the generators follow BASELINE.json's config text. Conventions shared by all
// of them (and recorded in DESIGN.md §Inputs):
//   * Dirichlet unknowns eliminated for C1–C4, kept as identity
//     rows for C5 like apply_dirichlet (fem.hpp:184-200);
//   * no h^2 scaling (C1 has diagonal 4 / off-diagonal -1 as specified);
//   * rows assembled with sorted columns, exact zeros dropped
//     (SparseCsrMatrix::from_triplets invariants, sparse.hpp:24-53);
//   * RHS stream Rng(mix_seed(seed, "rhs")), GRF stream mix_seed(seed, "grf"),
//     Young's-modulus stream mix_seed(seed, "youn").

#include "nlsp_inputs.h"

#include "host_rng.hpp"

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

constexpr std::uint64_t kTagRhs = 0x726873;      // "rhs"
constexpr std::uint64_t kTagGrf = 0x677266;      // "grf"
constexpr std::uint64_t kTagYoung = 0x796f756e;  // "youn"

using nlsp_host::mix_seed;
using nlsp_host::normal_stream;
using nlsp_host::Rng;

struct Csr {
    std::uint64_t n = 0;
    std::vector<std::uint64_t> rp, ci;
    std::vector<double> v;
};

// Row builder: columns pushed in ascending order; exact zeros dropped.
struct RowSink {
    Csr& a;
    explicit RowSink(Csr& m, std::uint64_t n) : a(m) {
        a.n = n;
        a.rp.assign(1, 0);
        a.rp.reserve(n + 1);
    }
    void put(std::uint64_t col, double val) {
        if (val != 0.0) {
            a.ci.push_back(col);
            a.v.push_back(val);
        }
    }
    void end_row() { a.rp.push_back(a.ci.size()); }
};

// C1: 5-point FD Laplacian on an nx*ny interior grid, Dirichlet eliminated.
void gen_poisson2d(std::uint64_t nx, std::uint64_t ny, Csr& a) {
    RowSink s(a, nx * ny);
    a.ci.reserve(5 * nx * ny);
    a.v.reserve(5 * nx * ny);
    for (std::uint64_t y = 0; y < ny; ++y)
        for (std::uint64_t x = 0; x < nx; ++x) {
            const std::uint64_t i = y * nx + x;
            if (y > 0) s.put(i - nx, -1.0);
            if (x > 0) s.put(i - 1, -1.0);
            s.put(i, 4.0);
            if (x + 1 < nx) s.put(i + 1, -1.0);
            if (y + 1 < ny) s.put(i + nx, -1.0);
            s.end_row();
        }
}

// C4: 7-point FD Laplacian on an nx*ny*nz interior grid.
void gen_poisson3d(std::uint64_t nx, std::uint64_t ny, std::uint64_t nz, Csr& a) {
    const std::uint64_t pl = nx * ny;
    RowSink s(a, pl * nz);
    a.ci.reserve(7 * pl * nz);
    a.v.reserve(7 * pl * nz);
    for (std::uint64_t z = 0; z < nz; ++z)
        for (std::uint64_t y = 0; y < ny; ++y)
            for (std::uint64_t x = 0; x < nx; ++x) {
                const std::uint64_t i = (z * ny + y) * nx + x;
                if (z > 0) s.put(i - pl, -1.0);
                if (y > 0) s.put(i - nx, -1.0);
                if (x > 0) s.put(i - 1, -1.0);
                s.put(i, 6.0);
                if (x + 1 < nx) s.put(i + 1, -1.0);
                if (y + 1 < ny) s.put(i + nx, -1.0);
                if (z + 1 < nz) s.put(i + pl, -1.0);
                s.end_row();
            }
}

// C3: -div(K grad u), K = R(theta) diag(1, eps) R(theta)^T, standard 9-point
// stencil (central u_xx, u_yy; 4-point cross derivative), h^2 dropped.
// Symbol 2k11(1-cos x) + 2k22(1-cos y) + 2k12 sin x sin y >= 0 since det K > 0,
// so the eliminated-Dirichlet operator is SPD (not an M-matrix).
void gen_aniso9(std::uint64_t nx, std::uint64_t ny, double eps, double theta, Csr& a) {
    const double c = std::cos(theta), sn = std::sin(theta);
    const double k11 = c * c + eps * sn * sn;
    const double k22 = sn * sn + eps * c * c;
    const double k12 = (1.0 - eps) * c * sn;
    const double w_c = 2.0 * k11 + 2.0 * k22, w_ew = -k11, w_ns = -k22;
    const double w_ne = -0.5 * k12, w_nw = 0.5 * k12; // NE/SW and NW/SE pairs
    RowSink s(a, nx * ny);
    a.ci.reserve(9 * nx * ny);
    a.v.reserve(9 * nx * ny);
    for (std::uint64_t y = 0; y < ny; ++y)
        for (std::uint64_t x = 0; x < nx; ++x) {
            const std::uint64_t i = y * nx + x;
            const bool w = x > 0, e = x + 1 < nx, sth = y > 0, nth = y + 1 < ny;
            if (sth) {
                if (w) s.put(i - nx - 1, w_ne); // SW pairs with NE
                s.put(i - nx, w_ns);
                if (e) s.put(i - nx + 1, w_nw); // SE pairs with NW
            }
            if (w) s.put(i - 1, w_ew);
            s.put(i, w_c);
            if (e) s.put(i + 1, w_ew);
            if (nth) {
                if (w) s.put(i + nx - 1, w_nw);
                s.put(i + nx, w_ns);
                if (e) s.put(i + nx + 1, w_ne);
            }
            s.end_row();
        }
}

// Gaussian random field on the nx*ny cell centres of the unit square with
// covariance variance * exp(-r^2 / (2 l^2)), by process convolution: white
// noise on a padded grid convolved with the separable kernel exp(-r^2 / l^2)
// (whose self-convolution is exp(-r^2 / (2 l^2))), truncated at 4 l, scaled to
// the target variance. Exact in the fine-grid limit; no FFT needed.
std::vector<double> grf(std::uint64_t nx, std::uint64_t ny, double corr_len, double variance,
                        std::uint64_t seed) {
    const double h = 1.0 / static_cast<double>(std::max(nx, ny));
    const std::int64_t R = static_cast<std::int64_t>(std::ceil(4.0 * corr_len / h));
    std::vector<double> w(2 * R + 1);
    double wsq = 0.0;
    for (std::int64_t d = -R; d <= R; ++d) {
        const double t = static_cast<double>(d) * h / corr_len;
        w[d + R] = std::exp(-t * t);
        wsq += w[d + R] * w[d + R];
    }
    const std::uint64_t px = nx + 2 * R, py = ny + 2 * R;
    std::vector<double> noise(px * py);
    normal_stream(seed, noise.size(), noise.data());
    std::vector<double> tmp(py * nx, 0.0);
    unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
    auto par = [&](std::uint64_t count, auto&& body) {
        std::vector<std::thread> th;
        const std::uint64_t per = (count + hw - 1) / hw;
        for (unsigned t = 0; t < hw; ++t) {
            const std::uint64_t lo = t * per, hi = std::min(count, lo + per);
            if (lo < hi) th.emplace_back([&, lo, hi] { for (auto r = lo; r < hi; ++r) body(r); });
        }
        for (auto& x : th) x.join();
    };
    par(py, [&](std::uint64_t yy) {
        const double* row = noise.data() + yy * px;
        for (std::uint64_t x = 0; x < nx; ++x) {
            double acc = 0.0;
            for (std::int64_t d = 0; d <= 2 * R; ++d) acc += w[d] * row[x + d];
            tmp[yy * nx + x] = acc;
        }
    });
    std::vector<double> g(nx * ny, 0.0);
    const double scale = std::sqrt(variance) / wsq;
    par(ny, [&](std::uint64_t y) {
        double* out = g.data() + y * nx;
        for (std::int64_t d = 0; d <= 2 * R; ++d) {
            const double wd = w[d];
            const double* src = tmp.data() + (y + d) * nx;
            for (std::uint64_t x = 0; x < nx; ++x) out[x] += wd * src[x];
        }
        for (std::uint64_t x = 0; x < nx; ++x) out[x] *= scale;
    });
    return g;
}

// C2: cell-centred FV for -div(a grad u) on nx*ny cells, a = exp(g); interior
// faces use the harmonic mean 2 a_i a_j / (a_i + a_j), Dirichlet faces the
// half-cell transmissibility 2 a_i. Rows sorted S, W, C, E, N.
void gen_diffusion_fv(std::uint64_t nx, std::uint64_t ny, const std::vector<double>& a_cell,
                      Csr& a) {
    RowSink s(a, nx * ny);
    a.ci.reserve(5 * nx * ny);
    a.v.reserve(5 * nx * ny);
    auto hm = [](double p, double q) { return 2.0 * p * q / (p + q); };
    for (std::uint64_t y = 0; y < ny; ++y)
        for (std::uint64_t x = 0; x < nx; ++x) {
            const std::uint64_t i = y * nx + x;
            const double ai = a_cell[i];
            const double ts = y > 0 ? hm(ai, a_cell[i - nx]) : 2.0 * ai;
            const double tw = x > 0 ? hm(ai, a_cell[i - 1]) : 2.0 * ai;
            const double te = x + 1 < nx ? hm(ai, a_cell[i + 1]) : 2.0 * ai;
            const double tn = y + 1 < ny ? hm(ai, a_cell[i + nx]) : 2.0 * ai;
            if (y > 0) s.put(i - nx, -ts);
            if (x > 0) s.put(i - 1, -tw);
            s.put(i, ((ts + tw) + te) + tn);
            if (x + 1 < nx) s.put(i + 1, -te);
            if (y + 1 < ny) s.put(i + nx, -tn);
            s.end_row();
        }
}

// Q1 plane-strain element stiffness for E = 1 on a square element (independent
// of the element size in 2D), 2x2 Gauss. Local nodes (0,0),(1,0),(1,1),(0,1);
// dofs [u0x,u0y,u1x,u1y,...].
void q1_stiffness(double nu, double ke[8][8]) {
    const double f = 1.0 / ((1.0 + nu) * (1.0 - 2.0 * nu));
    const double D[3][3] = {{f * (1.0 - nu), f * nu, 0.0},
                            {f * nu, f * (1.0 - nu), 0.0},
                            {0.0, 0.0, f * (1.0 - 2.0 * nu) / 2.0}};
    const double xi_n[4] = {-1, 1, 1, -1}, eta_n[4] = {-1, -1, 1, 1};
    const double gp = 1.0 / std::sqrt(3.0);
    for (int i = 0; i < 8; ++i)
        for (int j = 0; j < 8; ++j) ke[i][j] = 0.0;
    for (int gi = 0; gi < 2; ++gi)
        for (int gj = 0; gj < 2; ++gj) {
            const double xi = gi ? gp : -gp, eta = gj ? gp : -gp;
            // element [0,1]^2: x = (xi+1)/2 → dN/dx = 2 dN/dxi, detJ = 1/4
            double dNdx[4], dNdy[4];
            for (int a = 0; a < 4; ++a) {
                dNdx[a] = 2.0 * 0.25 * xi_n[a] * (1.0 + eta * eta_n[a]);
                dNdy[a] = 2.0 * 0.25 * eta_n[a] * (1.0 + xi * xi_n[a]);
            }
            double B[3][8] = {};
            for (int a = 0; a < 4; ++a) {
                B[0][2 * a] = dNdx[a];
                B[1][2 * a + 1] = dNdy[a];
                B[2][2 * a] = dNdy[a];
                B[2][2 * a + 1] = dNdx[a];
            }
            for (int i = 0; i < 8; ++i)
                for (int j = 0; j < 8; ++j) {
                    double acc = 0.0;
                    for (int p = 0; p < 3; ++p)
                        for (int q = 0; q < 3; ++q) acc += B[p][i] * D[p][q] * B[q][j];
                    ke[i][j] += acc * 0.25; // detJ, unit weights
                }
        }
}

// C5: Q1 plane strain on ex*ey elements of the unit square, (ex+1)(ey+1) nodes,
// dofs interleaved (2 per node). E piecewise constant on blocks x blocks
// checkerboard cells, log-uniform in [lo, hi]. Nodes on x = 0 are clamped and
// kept as identity rows (apply_dirichlet, fem.hpp:184-200).
void gen_elasticity(std::uint64_t ex, std::uint64_t ey, std::uint64_t blocks, double lo,
                    double hi, double nu, std::uint64_t seed, Csr& a, std::vector<std::uint8_t>& mask,
                    std::vector<double>& young) {
    const std::uint64_t nxn = ex + 1, nyn = ey + 1, nodes = nxn * nyn, n = 2 * nodes;
    Rng er(mix_seed(seed, kTagYoung));
    std::vector<double> eb(blocks * blocks);
    for (auto& e : eb) e = lo * std::pow(hi / lo, er.uniform());
    young.assign(ex * ey, 0.0);
    for (std::uint64_t y = 0; y < ey; ++y)
        for (std::uint64_t x = 0; x < ex; ++x)
            young[y * ex + x] = eb[(y * blocks / ey) * blocks + (x * blocks / ex)];
    double ke[8][8];
    q1_stiffness(nu, ke);
    mask.assign(n, 0);
    for (std::uint64_t y = 0; y < nyn; ++y) {
        mask[2 * (y * nxn)] = 1;
        mask[2 * (y * nxn) + 1] = 1;
    }
    RowSink s(a, n);
    a.ci.reserve(18 * n);
    a.v.reserve(18 * n);
    // element (x, y) local node L -> global node
    auto gnode = [&](std::uint64_t x, std::uint64_t y, int L) {
        const std::uint64_t dx = (L == 1 || L == 2), dy = (L >= 2);
        return (y + dy) * nxn + (x + dx);
    };
    double row[18];
    for (std::uint64_t ny_ = 0; ny_ < nyn; ++ny_)
        for (std::uint64_t nx_ = 0; nx_ < nxn; ++nx_) {
            const std::uint64_t node = ny_ * nxn + nx_;
            for (int c = 0; c < 2; ++c) {
                const std::uint64_t dof = 2 * node + c;
                if (mask[dof]) {
                    s.put(dof, 1.0);
                    s.end_row();
                    continue;
                }
                // slots: neighbour (dy, dx) in {-1,0,1}^2 sorted by node id, x2 dofs
                for (double& r : row) r = 0.0;
                for (int oy = -1; oy <= 0; ++oy)
                    for (int ox = -1; ox <= 0; ++ox) {
                        const std::int64_t exx = static_cast<std::int64_t>(nx_) + ox;
                        const std::int64_t eyy = static_cast<std::int64_t>(ny_) + oy;
                        if (exx < 0 || eyy < 0 || exx >= static_cast<std::int64_t>(ex) ||
                            eyy >= static_cast<std::int64_t>(ey))
                            continue;
                        const double E = young[eyy * ex + exx];
                        int me = -1;
                        for (int L = 0; L < 4; ++L)
                            if (gnode(exx, eyy, L) == node) me = L;
                        for (int L = 0; L < 4; ++L) {
                            const std::uint64_t gn = gnode(exx, eyy, L);
                            const std::int64_t gx = gn % nxn, gy = gn / nxn;
                            const int slot = static_cast<int>(((gy - ny_ + 1) * 3 + (gx - nx_ + 1)));
                            for (int d = 0; d < 2; ++d) row[2 * slot + d] += E * ke[2 * me + c][2 * L + d];
                        }
                    }
                for (int slot = 0; slot < 9; ++slot) {
                    const std::int64_t gx = static_cast<std::int64_t>(nx_) + slot % 3 - 1;
                    const std::int64_t gy = static_cast<std::int64_t>(ny_) + slot / 3 - 1;
                    if (gx < 0 || gy < 0 || gx >= static_cast<std::int64_t>(nxn) ||
                        gy >= static_cast<std::int64_t>(nyn))
                        continue;
                    const std::uint64_t gnode_id = gy * nxn + gx;
                    for (int d = 0; d < 2; ++d) {
                        const std::uint64_t col = 2 * gnode_id + d;
                        if (mask[col]) continue; // eliminated coupling to a clamped dof
                        s.put(col, row[2 * slot + d]);
                    }
                }
                s.end_row();
            }
        }
}

} // namespace

struct nlsp_problem {
    Csr a;
    std::vector<double> rhs;
    std::vector<std::uint8_t> mask;
    std::vector<double> coef;
};

extern "C" {

const char* nlsp_inputs_last_error(void) { return g_err.c_str(); }

std::uint64_t nlsp_mix_seed(std::uint64_t seed, std::uint64_t tag) { return mix_seed(seed, tag); }

void nlsp_rng_normal_fill(std::uint64_t seed, std::uint64_t count, double* out) {
    normal_stream(seed, count, out);
}

// The serial loop over Rng(seed).normal() itself (std::mt19937_64, no jumps):
// what nlsp_rng_normal_fill's threaded stream must reproduce bit for bit.
// zero_below widens the rejection `while (u1 <= 0)` for tests of that path.
void nlsp_rng_normal_serial(std::uint64_t seed, std::uint64_t count, double zero_below, double* out) {
    std::mt19937_64 gen(seed);
    auto uni = [&]() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; };
    for (std::uint64_t i = 0; i < count; i += 2) {
        double u1 = uni();
        const double u2 = uni();
        while (u1 <= zero_below) u1 = uni();
        const double r = std::sqrt(-2.0 * std::log(u1));
        const double a = 2.0 * 3.141592653589793 * u2;
        out[i] = r * std::cos(a);
        if (i + 1 < count) out[i + 1] = r * std::sin(a);
    }
}

// nlsp_rng_normal_fill with its knobs exposed: chunk size in pairs, the widened
// rejection, and a cap on the worker threads (0: all)
void nlsp_rng_normal_chunks(std::uint64_t seed, std::uint64_t count, std::uint64_t chunk_pairs,
                            double zero_below, std::uint32_t max_workers, double* out) {
    struct ToArray {
        double* out;
        std::uint64_t count;
        std::vector<double> scratch;
        double* buffer(std::uint64_t base, std::uint64_t np) {
            if (2 * (base + np) <= count) return out + 2 * base;
            scratch.assign(2 * np, 0.0);
            return scratch.data();
        }
        void done(std::uint64_t base, std::uint64_t np) {
            if (2 * (base + np) > count)
                std::copy(scratch.begin(), scratch.begin() + (count - 2 * base), out + 2 * base);
        }
    } sink{out, count, {}};
    nlsp_host::normal_stream_chunks(seed, count, sink, chunk_pairs, zero_below, max_workers);
}

// raw std::mt19937_64 outputs (the check of the jump-ahead generators)
void nlsp_mt19937_64_fill(std::uint64_t seed, std::uint64_t skip, std::uint64_t count, std::uint64_t* out) {
    std::mt19937_64 gen(seed);
    gen.discard(skip);
    for (std::uint64_t i = 0; i < count; ++i) out[i] = gen();
}

// the same words from a generator jumped `skip` words ahead (mt_jump.hpp);
// skip must be a multiple of 2^17. Returns 0 on success.
int nlsp_mt19937_64_jump_fill(std::uint64_t seed, std::uint64_t skip, std::uint64_t count, std::uint64_t* out) {
    std::uint64_t w[nlsp_host::kMtN], j[nlsp_host::kMtN];
    nlsp_host::mt64_seed(seed, w);
    if (!nlsp_host::mt64_jump(w, skip, j)) return 1;
    nlsp_host::Mt64 gen(j);
    for (std::uint64_t i = 0; i < count; ++i) out[i] = gen();
    return 0;
}

void nlsp_rng_uniform_fill(std::uint64_t seed, std::uint64_t count, double lo, double hi,
                           double* out) {
    Rng r(seed);
    for (std::uint64_t i = 0; i < count; ++i) out[i] = r.uniform(lo, hi);
}

void nlsp_smoothed_s0(std::uint64_t seed, std::uint64_t n, std::uint64_t m, const std::uint8_t* mask,
                      double* out) {
    nlsp_host::smoothed_s0(seed, n, m, mask, out);
}

int nlsp_problem_create(const nlsp_problem_spec* spec, nlsp_problem** out) {
    *out = nullptr;
    if (!spec) {
        g_err = "null spec";
        return 1;
    }
    auto p = new nlsp_problem();
    const std::uint64_t nx = spec->nx, ny = spec->ny ? spec->ny : spec->nx,
                        nz = spec->nz ? spec->nz : spec->nx;
    if (nx == 0) {
        g_err = "grid size must be positive";
        delete p;
        return 1;
    }
    switch (spec->kind) {
        case NLSP_PROBLEM_POISSON2D_FD: gen_poisson2d(nx, ny, p->a); break;
        case NLSP_PROBLEM_POISSON3D_FD: gen_poisson3d(nx, ny, nz, p->a); break;
        case NLSP_PROBLEM_ANISO2D_9PT: gen_aniso9(nx, ny, spec->epsilon, spec->theta, p->a); break;
        case NLSP_PROBLEM_DIFFUSION2D_FV: {
            if (!(spec->corr_len > 0.0) || !(spec->variance >= 0.0)) {
                g_err = "GRF needs corr_len > 0 and variance >= 0";
                delete p;
                return 1;
            }
            auto g = grf(nx, ny, spec->corr_len, spec->variance, mix_seed(spec->seed, kTagGrf));
            p->coef.resize(g.size());
            for (std::size_t i = 0; i < g.size(); ++i) p->coef[i] = std::exp(g[i]);
            gen_diffusion_fv(nx, ny, p->coef, p->a);
            break;
        }
        case NLSP_PROBLEM_ELASTICITY2D_Q1: {
            const std::uint64_t blocks = spec->blocks ? spec->blocks : 1;
            if (!(spec->young_lo > 0.0) || !(spec->young_hi >= spec->young_lo) ||
                !(spec->poisson > -1.0 && spec->poisson < 0.5)) {
                g_err = "elasticity needs 0 < young_lo <= young_hi and -1 < nu < 0.5";
                delete p;
                return 1;
            }
            gen_elasticity(nx, ny, blocks, spec->young_lo, spec->young_hi, spec->poisson,
                           spec->seed, p->a, p->mask, p->coef);
            break;
        }
        default:
            g_err = "unknown problem kind";
            delete p;
            return 1;
    }
    const std::uint64_t n = p->a.n;
    if (p->mask.empty()) p->mask.assign(n, 0);
    p->rhs.resize(n);
    if (spec->rhs_uniform) {
        Rng r(mix_seed(spec->seed, kTagRhs));
        for (auto& v : p->rhs) v = r.uniform(-1.0, 1.0);
    } else {
        normal_stream(mix_seed(spec->seed, kTagRhs), n, p->rhs.data());
    }
    for (std::uint64_t i = 0; i < n; ++i)
        if (p->mask[i]) p->rhs[i] = 0.0;
    *out = p;
    return 0;
}

void nlsp_problem_destroy(nlsp_problem* p) { delete p; }
std::uint64_t nlsp_problem_n(const nlsp_problem* p) { return p->a.n; }
std::uint64_t nlsp_problem_nnz(const nlsp_problem* p) { return p->a.v.size(); }
std::uint64_t nlsp_problem_coef_len(const nlsp_problem* p) { return p->coef.size(); }

void nlsp_problem_export(const nlsp_problem* p, std::uint64_t* row_ptr, std::uint64_t* col_idx,
                         double* values, double* rhs, std::uint8_t* mask) {
    if (row_ptr) std::memcpy(row_ptr, p->a.rp.data(), sizeof(std::uint64_t) * p->a.rp.size());
    if (col_idx) std::memcpy(col_idx, p->a.ci.data(), sizeof(std::uint64_t) * p->a.ci.size());
    if (values) std::memcpy(values, p->a.v.data(), sizeof(double) * p->a.v.size());
    if (rhs) std::memcpy(rhs, p->rhs.data(), sizeof(double) * p->rhs.size());
    if (mask) std::memcpy(mask, p->mask.data(), p->mask.size());
}

void nlsp_problem_export_coef(const nlsp_problem* p, double* coef) {
    if (coef && !p->coef.empty()) std::memcpy(coef, p->coef.data(), sizeof(double) * p->coef.size());
}

} // extern "C"
