// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never measured
// as the product).
//
// A thin extern "C" shim over the UNMODIFIED reference headers
// (/root/reference/proj/include/nlsp/*.hpp, included by path, never copied),
// compiled by oracle/Makefile into oracle/_ref/libnlsp_ref*.so. It is the
// "real reference" arm used to
//   * pin the C restatement in oracle/nlsp_oracle.c (tests/test_oracle_pin.py),
//   * generate the golden fixtures under tests/golden/ (tests/golden/make_golden.py),
//   * time the reference CPU solve for bench.py --impl reference / cpu_baseline.
//
// Two builds are produced from this one file:
//   libnlsp_ref.so         -O3 -march=x86-64-v3      (the reference's default
//                           "-O3 -march=native" build, pinned to a portable ISA so
//                           the .so runs on the GPU box's host CPU)
//   libnlsp_ref_strict.so  same + -ffp-contract=off  (sequential-rounding build,
//                           bitwise comparable to the restatement)
//
// Private members of the reference classes are read (not modified) so the
// Galerkin operator and its Cholesky factor can be exported for parity.

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <fstream>
#include <functional>
#include <limits>
#include <memory>
#include <numbers>
#include <numeric>
#include <random>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#define private public
#include "nlsp/cholesky.hpp"
#include "nlsp/dense.hpp"
#include "nlsp/errors.hpp"
#include "nlsp/fem.hpp"
#include "nlsp/instance_io.hpp"
#include "nlsp/mlp.hpp"
#include "nlsp/train.hpp"
#include "nlsp/qr.hpp"
#include "nlsp/rng.hpp"
#include "nlsp/sa.hpp"
#include "nlsp/smoothing.hpp"
#include "nlsp/sparse.hpp"
#include "nlsp/svd.hpp"
#include "nlsp/two_level.hpp"
#undef private

using namespace nlsp;

namespace {

thread_local std::string g_err;

// status codes shared with include/nlsp_gpu.h (nlsp_status)
enum { ST_OK = 0, ST_VALIDATION = 1, ST_NUMERIC = 2, ST_NOT_SPD = 3, ST_RANK = 4,
       ST_CONVERGENCE = 5, ST_IO = 8, ST_OTHER = 9 };

template <class F>
int guarded(F&& f) {
    try {
        f();
        return ST_OK;
    } catch (const ValidationError& e) {
        g_err = e.what();
        return ST_VALIDATION;
    } catch (const NotSpdError& e) {
        g_err = e.what();
        return ST_NOT_SPD;
    } catch (const RankDeficiencyError& e) {
        g_err = e.what();
        return ST_RANK;
    } catch (const ConvergenceError& e) {
        g_err = e.what();
        return ST_CONVERGENCE;
    } catch (const NumericError& e) {
        g_err = e.what();
        return ST_NUMERIC;
    } catch (const IoError& e) {
        g_err = e.what();
        return ST_IO;
    } catch (const std::exception& e) {
        g_err = e.what();
        return ST_OTHER;
    }
}

DenseMatrix dense_from(std::uint64_t rows, std::uint64_t cols, const double* a) {
    DenseMatrix m(rows, cols);
    if (rows * cols) std::memcpy(m.data(), a, sizeof(double) * rows * cols);
    return m;
}

void dense_to(const DenseMatrix& m, double* out) {
    if (m.rows() * m.cols()) std::memcpy(out, m.data(), sizeof(double) * m.rows() * m.cols());
}

struct RefTwoLevel {
    std::unique_ptr<TwoLevelPreconditioner> m;
};

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// --- CSR ------------------------------------------------------------------
// Builds through SparseCsrMatrix::from_triplets (sparse.hpp:24-53) so the
// reference's own invariants (sorted, duplicates summed, zeros dropped) apply.
void* ref_csr_create(std::uint64_t n, std::uint64_t nnz, const std::uint64_t* rp,
                     const std::uint64_t* ci, const double* v) {
    void* out = nullptr;
    int st = guarded([&] {
        std::vector<std::tuple<std::size_t, std::size_t, double>> t;
        t.reserve(nnz);
        for (std::uint64_t i = 0; i < n; ++i)
            for (std::uint64_t k = rp[i]; k < rp[i + 1]; ++k) t.emplace_back(i, ci[k], v[k]);
        out = new SparseCsrMatrix(SparseCsrMatrix::from_triplets(n, std::move(t)));
    });
    return st == ST_OK ? out : nullptr;
}

void ref_csr_destroy(void* h) { delete static_cast<SparseCsrMatrix*>(h); }

std::uint64_t ref_csr_nnz(void* h) { return static_cast<SparseCsrMatrix*>(h)->nnz(); }

std::uint64_t ref_csr_dim(void* h) { return static_cast<SparseCsrMatrix*>(h)->dim(); }

// export the (possibly re-normalised) CSR arrays
void ref_csr_export(void* h, std::uint64_t* rp, std::uint64_t* ci, double* v) {
    auto* a = static_cast<SparseCsrMatrix*>(h);
    for (std::size_t i = 0; i <= a->dim(); ++i) rp[i] = a->row_ptr()[i];
    for (std::size_t k = 0; k < a->nnz(); ++k) {
        ci[k] = a->col_idx()[k];
        v[k] = a->values()[k];
    }
}

// triplet construction straight through the reference (for the dedup test)
void* ref_csr_from_triplets(std::uint64_t n, std::uint64_t count, const std::uint64_t* ti,
                            const std::uint64_t* tj, const double* tv, int* status) {
    void* out = nullptr;
    *status = guarded([&] {
        std::vector<std::tuple<std::size_t, std::size_t, double>> t;
        for (std::uint64_t k = 0; k < count; ++k) t.emplace_back(ti[k], tj[k], tv[k]);
        out = new SparseCsrMatrix(SparseCsrMatrix::from_triplets(n, std::move(t)));
    });
    return out;
}

int ref_spmv(void* h, std::uint64_t xlen, const double* x, double* y) {
    return guarded([&] {
        auto* a = static_cast<SparseCsrMatrix*>(h);
        std::vector<double> xv(x, x + xlen);
        auto yv = spmv(*a, xv);
        std::copy(yv.begin(), yv.end(), y);
    });
}

// --- P1 FEM instances (fem.hpp:223-236): unstructured CSR test inputs --------
// family 0 diffusion, 1 anisotropic, 2 screened Poisson. Two-phase: query the
// size (out arrays NULL), then fill.
int ref_fem_instance(int family, std::uint64_t grid_n, double jitter, std::uint64_t seed,
                     std::uint64_t* n_out, std::uint64_t* nnz_out, std::uint64_t* rp,
                     std::uint64_t* ci, double* v, double* rhs, std::uint8_t* mask) {
    return guarded([&] {
        auto inst = make_instance(static_cast<PdeFamily>(family), grid_n, jitter, seed);
        const auto& a = inst.matrix;
        *n_out = a.dim();
        *nnz_out = a.nnz();
        if (!rp) return;
        for (std::size_t i = 0; i <= a.dim(); ++i) rp[i] = a.row_ptr()[i];
        for (std::size_t k = 0; k < a.nnz(); ++k) {
            ci[k] = a.col_idx()[k];
            v[k] = a.values()[k];
        }
        for (std::size_t i = 0; i < a.dim(); ++i) {
            rhs[i] = inst.rhs[i];
            mask[i] = inst.mesh.boundary_mask[i] ? 1 : 0;
        }
    });
}

// --- on-disk inputs (sparse.hpp:148-194, instance_io.hpp:99-185) ------------
int ref_save_instance(int family, std::uint64_t grid_n, double jitter, std::uint64_t seed,
                      const char* dir) {
    return guarded([&] {
        auto inst = make_instance(static_cast<PdeFamily>(family), grid_n, jitter, seed);
        save_instance(inst, dir);
    });
}

// load_matrix_market -> CSR handle (ref_csr_export / ref_csr_destroy), or NULL
// with *status set
void* ref_load_matrix_market(const char* path, int* status) {
    SparseCsrMatrix* out = nullptr;
    *status = guarded([&] { out = new SparseCsrMatrix(load_matrix_market(path)); });
    return out;
}

int ref_save_matrix_market(void* h, const char* path) {
    return guarded([&] { save_matrix_market(*static_cast<SparseCsrMatrix*>(h), path); });
}

void* ref_load_instance(const char* dir, int* status) {
    PdeInstance* out = nullptr;
    *status = guarded([&] { out = new PdeInstance(load_instance(dir)); });
    return out;
}

void ref_instance_destroy(void* h) { delete static_cast<PdeInstance*>(h); }

// family, grid_n, seed, jitter, alpha, n (matrix), vertices, triangles
void ref_instance_meta(void* h, int* family, std::uint64_t* grid_n, std::uint64_t* seed, double* jitter,
                       double* alpha, std::uint64_t* n, std::uint64_t* nv, std::uint64_t* nt) {
    const auto& in = *static_cast<PdeInstance*>(h);
    *family = static_cast<int>(in.family);
    *grid_n = in.grid_n;
    *seed = in.seed;
    *jitter = in.jitter;
    *alpha = in.coefficients.alpha;
    *n = in.matrix.dim();
    *nv = in.mesh.vertices.size();
    *nt = in.mesh.triangles.size();
}

// a copy of the matrix as a CSR handle; rhs (n), mask (nv), vertices (nv x 2),
// triangles (nt x 3), coefficients (nt x 1|3)
void* ref_instance_matrix(void* h) { return new SparseCsrMatrix(static_cast<PdeInstance*>(h)->matrix); }

void ref_instance_arrays(void* h, double* rhs, std::uint8_t* mask, double* vert, std::uint64_t* tri,
                         double* coeff) {
    const auto& in = *static_cast<PdeInstance*>(h);
    for (std::size_t i = 0; i < in.rhs.size(); ++i) rhs[i] = in.rhs[i];
    for (std::size_t v = 0; v < in.mesh.vertices.size(); ++v) {
        mask[v] = in.mesh.boundary_mask[v] ? 1 : 0;
        vert[2 * v] = in.mesh.vertices[v].x;
        vert[2 * v + 1] = in.mesh.vertices[v].y;
    }
    for (std::size_t t = 0; t < in.mesh.triangles.size(); ++t)
        for (int q = 0; q < 3; ++q) tri[3 * t + q] = in.mesh.triangles[t].v[q];
    const auto& c = in.coefficients;
    switch (in.family) {
        case PdeFamily::Diffusion:
            for (std::size_t t = 0; t < c.g.size(); ++t) coeff[t] = c.g[t];
            break;
        case PdeFamily::Anisotropic:
            for (std::size_t t = 0; t < c.tensor.size(); ++t) {
                coeff[3 * t] = c.tensor[t].k11;
                coeff[3 * t + 1] = c.tensor[t].k12;
                coeff[3 * t + 2] = c.tensor[t].k22;
            }
            break;
        case PdeFamily::ScreenedPoisson:
            for (std::size_t t = 0; t < c.kappa.size(); ++t) coeff[t] = c.kappa[t];
            break;
    }
}

// --- smoothed aggregation (sa.hpp:18-109) -----------------------------------
// aggregate ids (n) and their count
int ref_aggregate_nodes(void* h, double theta, std::uint64_t* agg, std::uint64_t* nc) {
    return guarded([&] {
        std::size_t c = 0;
        const auto a = aggregate_nodes(*static_cast<SparseCsrMatrix*>(h), theta, &c);
        for (std::size_t i = 0; i < a.size(); ++i) agg[i] = a[i];
        *nc = c;
    });
}

// dense P (n x nc, row-major); two-phase: p == NULL queries nc
int ref_sa_prolongator(void* h, double theta, double omega, std::uint64_t* nc, double* p) {
    return guarded([&] {
        const auto m = sa_prolongator(*static_cast<SparseCsrMatrix*>(h), theta, omega);
        *nc = m.cols();
        if (p) dense_to(m, p);
    });
}

// --- MLP inference (mlp.hpp:57-161, train.hpp:52-62) -------------------------
int ref_mlp_create_save(const std::uint64_t* widths, std::uint64_t nw, std::uint64_t seed,
                        const char* path) {
    return guarded([&] {
        MlpModel m(std::vector<std::size_t>(widths, widths + nw), seed);
        m.save(path, "created by oracle/ref_driver.cpp");
    });
}

// parameters of a checkpoint (two-phase: params == NULL queries the count)
int ref_mlp_params(const char* path, std::uint64_t* np, double* params) {
    return guarded([&] {
        const auto m = MlpModel::load(path);
        *np = m.num_params();
        if (params) std::copy(m.params().begin(), m.params().end(), params);
    });
}

int ref_mlp_forward(const char* path, const double* in, double* out) {
    return guarded([&] {
        const auto m = MlpModel::load(path);
        const std::vector<double> x(in, in + m.input_width());
        const auto y = m.forward(x);
        std::copy(y.begin(), y.end(), out);
    });
}

// infer_basis(model, S) (train.hpp:52-62): S n x k row-major -> q n x r row-major
int ref_infer_basis(const char* path, std::uint64_t n, std::uint64_t k, const double* s, double* q,
                    std::uint64_t* r_out, double* ms) {
    return guarded([&] {
        const auto m = MlpModel::load(path);
        const auto sm = dense_from(n, k, s);
        const auto t0 = std::chrono::steady_clock::now();
        const auto b = infer_basis(m, sm);
        const auto t1 = std::chrono::steady_clock::now();
        if (ms) *ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        *r_out = b.cols();
        if (q) dense_to(b, q);
    });
}

// --- RNG (rng.hpp) ----------------------------------------------------------
std::uint64_t ref_mix_seed(std::uint64_t seed, std::uint64_t tag) { return mix_seed(seed, tag); }

void ref_rng_normal(std::uint64_t seed, std::uint64_t count, double* out) {
    Rng r(seed);
    for (std::uint64_t i = 0; i < count; ++i) out[i] = r.normal();
}

void ref_rng_uniform(std::uint64_t seed, std::uint64_t count, double lo, double hi, double* out) {
    Rng r(seed);
    for (std::uint64_t i = 0; i < count; ++i) out[i] = r.uniform(lo, hi);
}

void ref_rng_u64(std::uint64_t seed, std::uint64_t count, std::uint64_t* out) {
    Rng r(seed);
    for (std::uint64_t i = 0; i < count; ++i) out[i] = r.next_u64();
}

// --- smoothing (smoothing.hpp) -------------------------------------------------
int ref_jacobi_inv_diag(void* h, double omega, double* dinv) {
    return guarded([&] {
        JacobiSmoother sm(*static_cast<SparseCsrMatrix*>(h), omega);
        std::copy(sm.inv_diag().begin(), sm.inv_diag().end(), dinv);
    });
}

// `sweeps` weighted-Jacobi sweeps x <- x + w D^-1 (b - A x) on one vector
int ref_jacobi_sweep(void* h, double omega, std::uint64_t sweeps, double* x, const double* b) {
    return guarded([&] {
        auto* a = static_cast<SparseCsrMatrix*>(h);
        JacobiSmoother sm(*a, omega);
        std::vector<double> xv(x, x + a->dim()), bv(b, b + a->dim());
        for (std::uint64_t s = 0; s < sweeps; ++s) sm.sweep(*a, xv, bv);
        std::copy(xv.begin(), xv.end(), x);
    });
}

// generate_smoothed_vectors (smoothing.hpp:81-100); s_out is n x k row-major
int ref_generate_smoothed_vectors(void* h, const std::uint8_t* mask, std::uint64_t k,
                                  std::uint64_t sweeps, double omega, std::uint64_t seed,
                                  double* s_out) {
    return guarded([&] {
        auto* a = static_cast<SparseCsrMatrix*>(h);
        std::vector<bool> m(a->dim(), false);
        if (mask)
            for (std::size_t i = 0; i < a->dim(); ++i) m[i] = mask[i] != 0;
        auto sv = generate_smoothed_vectors(*a, m, k, sweeps, omega, seed);
        dense_to(sv.s, s_out);
    });
}

// homogeneous block sweeps on a supplied S (smoothing.hpp:50-60), in place
int ref_block_sweeps(void* h, std::uint64_t m, double* s, std::uint64_t sweeps, double omega) {
    return guarded([&] {
        auto* a = static_cast<SparseCsrMatrix*>(h);
        JacobiSmoother sm(*a, omega);
        DenseMatrix x = dense_from(a->dim(), m, s);
        for (std::uint64_t k = 0; k < sweeps; ++k) sm.sweep(*a, x);
        dense_to(x, s);
    });
}

// --- dense kernels ------------------------------------------------------------
int ref_matmul_tn(std::uint64_t rows, std::uint64_t ca, std::uint64_t cb, const double* a,
                  const double* b, double* c) {
    return guarded([&] { dense_to(matmul_tn(dense_from(rows, ca, a), dense_from(rows, cb, b)), c); });
}

int ref_jacobi_eigh(std::uint64_t n, const double* g, double* evals, double* evecs, int* sweeps) {
    return guarded([&] {
        auto r = jacobi_eigh(dense_from(n, n, g));
        std::copy(r.eigenvalues.begin(), r.eigenvalues.end(), evals);
        dense_to(r.eigenvectors, evecs);
        *sweeps = r.sweeps_used;
    });
}

// svd_oracle (svd.hpp:155-227): U rows x r, sigma r, V cols x r, r = min(rows, cols)
int ref_svd(std::uint64_t rows, std::uint64_t cols, const double* s, double* u, double* sigma,
            double* v, int* sweeps) {
    return guarded([&] {
        auto f = svd_oracle(dense_from(rows, cols, s));
        dense_to(f.left_vectors, u);
        std::copy(f.singular_values.begin(), f.singular_values.end(), sigma);
        dense_to(f.right_vectors, v);
        *sweeps = f.sweeps_used;
    });
}

double ref_orthonormality_defect(std::uint64_t rows, std::uint64_t cols, const double* a) {
    return orthonormality_defect(dense_from(rows, cols, a));
}

int ref_principal_angles(std::uint64_t rows, std::uint64_t cols, const double* a, const double* b,
                         double* angles) {
    return guarded([&] {
        auto r = principal_angles(dense_from(rows, cols, a), dense_from(rows, cols, b));
        std::copy(r.begin(), r.end(), angles);
    });
}

double ref_captured_energy(std::uint64_t rows, std::uint64_t k, std::uint64_t m, const double* p,
                           const double* s) {
    double out = -1.0;
    guarded([&] { out = captured_energy(dense_from(rows, k, p), dense_from(rows, m, s)); });
    return out;
}

int ref_qr_thin(std::uint64_t n, std::uint64_t k, const double* m, double* q, double* r) {
    return guarded([&] {
        auto f = qr_thin(dense_from(n, k, m));
        dense_to(f.q, q);
        dense_to(f.r, r);
    });
}

int ref_cholesky(std::uint64_t n, const double* a, double* l) {
    return guarded([&] {
        CholeskyFactor f(dense_from(n, n, a));
        dense_to(f.l_, l);
    });
}

int ref_cholesky_solve(std::uint64_t n, const double* a, const double* rhs, double* x) {
    return guarded([&] {
        CholeskyFactor f(dense_from(n, n, a));
        auto y = f.solve(std::vector<double>(rhs, rhs + n));
        std::copy(y.begin(), y.end(), x);
    });
}

// --- two-level preconditioner (two_level.hpp:22-89) ---------------------------
void* ref_twolevel_create(void* h, std::uint64_t k, const double* basis, double omega,
                          std::uint64_t nu1, std::uint64_t nu2, int* status) {
    RefTwoLevel* out = nullptr;
    *status = guarded([&] {
        auto* a = static_cast<SparseCsrMatrix*>(h);
        auto t = std::make_unique<RefTwoLevel>();
        t->m = std::make_unique<TwoLevelPreconditioner>(*a, dense_from(a->dim(), k, basis), omega,
                                                        nu1, nu2);
        out = t.release();
    });
    return out;
}

void ref_twolevel_destroy(void* t) { delete static_cast<RefTwoLevel*>(t); }

// A TwoLevelPreconditioner whose members are set from given parts instead of
// running the constructor body: basis_ = an orthonormal basis, coarse_ =
// CholeskyFactor(A_c) (the reference's own factorisation, cholesky.hpp:15-37),
// smoother_ = JacobiSmoother(a, omega). Used only to time the reference's own
// apply/pcg (two_level.hpp:60-81,141-191) at full size, where the constructor's
// column-strided QR + Galerkin loops alone take ~20 min.
void* ref_twolevel_from_parts(void* h, std::uint64_t k, const double* basis, const double* coarse,
                              double omega, std::uint64_t nu1, std::uint64_t nu2, int* status) {
    RefTwoLevel* out = nullptr;
    *status = guarded([&] {
        auto* a = static_cast<SparseCsrMatrix*>(h);
        // constructed on a 1x1 identity problem (trivially cheap), then re-seated
        const auto tiny = SparseCsrMatrix::identity(1);
        DenseMatrix one(1, 1, 1.0);
        auto t = std::make_unique<RefTwoLevel>();
        t->m = std::make_unique<TwoLevelPreconditioner>(tiny, one, omega, nu1, nu2);
        t->m->basis_ = dense_from(a->dim(), k, basis);
        t->m->coarse_ = std::make_unique<CholeskyFactor>(dense_from(k, k, coarse));
        t->m->smoother_ = JacobiSmoother(*a, omega);
        out = t.release();
    });
    return out;
}

// `threads` concurrent reference pcg solves of the same system (the reference
// parallelises across instances only, pipeline.hpp:356 / parallel.hpp:26-55;
// objects are safe for concurrent pcg). Returns wall ms and the
// per-thread iteration count of thread 0.
int ref_pcg_parallel(void* h, int kind, void* t, const double* b, double delta,
                     std::uint64_t max_iters, int threads, double* wall_ms,
                     std::uint64_t* iterations) {
    return guarded([&] {
        auto* a = static_cast<SparseCsrMatrix*>(h);
        std::vector<double> bv(b, b + a->dim());
        std::vector<std::uint64_t> its(threads, 0);
        std::vector<std::string> errs(threads);
        auto work = [&](int i) {
            try {
                PcgResult r;
                if (kind == 0) r = pcg(*a, bv, IdentityPreconditioner{}, delta, max_iters);
                else if (kind == 1) r = pcg(*a, bv, JacobiPreconditioner{}, delta, max_iters);
                else r = pcg(*a, bv, *static_cast<RefTwoLevel*>(t)->m, delta, max_iters);
                its[i] = r.report.iterations;
            } catch (const std::exception& e) {
                errs[i] = e.what();
            }
        };
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> th;
        for (int i = 0; i < threads; ++i) th.emplace_back(work, i);
        for (auto& x : th) x.join();
        const auto t1 = std::chrono::steady_clock::now();
        *wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        *iterations = its[0];
        for (auto& e : errs)
            if (!e.empty()) throw NumericError(e);
    });
}

// basis_ (n x k), the Cholesky factor L (k x k) and A_c = L L^T (recomposed
// from the reference's own factor, k x k)
void ref_twolevel_export(void* t, double* basis, double* chol, double* coarse) {
    auto* m = static_cast<RefTwoLevel*>(t)->m.get();
    if (basis) dense_to(m->basis_, basis);
    const auto& l = m->coarse_->l_;
    if (chol) dense_to(l, chol);
    if (coarse) {
        const std::size_t k = l.rows();
        for (std::size_t i = 0; i < k; ++i)
            for (std::size_t j = 0; j < k; ++j) {
                double s = 0.0;
                for (std::size_t p = 0; p <= std::min(i, j); ++p) s += l(i, p) * l(j, p);
                coarse[i * k + j] = s;
            }
    }
}

// The Galerkin operator exactly as the constructor forms it before
// factorising (two_level.hpp:33-51), recomputed from basis_ with the same
// loops so it can be compared entrywise.
void ref_twolevel_galerkin(void* t, void* h, double* coarse) {
    auto* m = static_cast<RefTwoLevel*>(t)->m.get();
    auto* a = static_cast<SparseCsrMatrix*>(h);
    const auto& b = m->basis_;
    const std::size_t nc = b.cols();
    DenseMatrix c(nc, nc);
    std::vector<double> col(a->dim());
    for (std::size_t j = 0; j < nc; ++j) {
        for (std::size_t i = 0; i < a->dim(); ++i) col[i] = b(i, j);
        const auto acol = spmv(*a, col);
        for (std::size_t i = 0; i < nc; ++i) {
            double s = 0.0;
            for (std::size_t row = 0; row < a->dim(); ++row) s += b(row, i) * acol[row];
            c(i, j) = s;
        }
    }
    for (std::size_t i = 0; i < nc; ++i)
        for (std::size_t j = i + 1; j < nc; ++j) {
            const double v = 0.5 * (c(i, j) + c(j, i));
            c(i, j) = v;
            c(j, i) = v;
        }
    dense_to(c, coarse);
}

int ref_twolevel_apply(void* t, void* h, const double* r, double* z) {
    return guarded([&] {
        auto* m = static_cast<RefTwoLevel*>(t)->m.get();
        auto* a = static_cast<SparseCsrMatrix*>(h);
        auto zv = m->apply(*a, std::vector<double>(r, r + a->dim()));
        std::copy(zv.begin(), zv.end(), z);
    });
}

// --- PCG (two_level.hpp:141-191) ------------------------------------------------
// kind: 0 identity, 1 Jacobi (diagonal), 2 two-level (t must be non-NULL).
// hist receives min(iterations, hist_cap) entries.
int ref_pcg(void* h, int kind, void* t, const double* b, double delta, std::uint64_t max_iters,
            double* x, double* hist, std::uint64_t hist_cap, std::uint64_t* iterations,
            int* converged, double* true_res, double* solve_ms) {
    return guarded([&] {
        auto* a = static_cast<SparseCsrMatrix*>(h);
        std::vector<double> bv(b, b + a->dim());
        const auto t0 = std::chrono::steady_clock::now();
        PcgResult res;
        if (kind == 0)
            res = pcg(*a, bv, IdentityPreconditioner{}, delta, max_iters);
        else if (kind == 1)
            res = pcg(*a, bv, JacobiPreconditioner{}, delta, max_iters);
        else
            res = pcg(*a, bv, *static_cast<RefTwoLevel*>(t)->m, delta, max_iters);
        const auto t1 = std::chrono::steady_clock::now();
        *solve_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        std::copy(res.solution.begin(), res.solution.end(), x);
        *iterations = res.report.iterations;
        *converged = res.report.converged ? 1 : 0;
        *true_res = res.report.true_relative_residual;
        if (hist) {
            const std::size_t c = std::min<std::size_t>(hist_cap, res.report.residual_history.size());
            std::copy(res.report.residual_history.begin(), res.report.residual_history.begin() + c,
                      hist);
        }
    });
}

} // extern "C"
