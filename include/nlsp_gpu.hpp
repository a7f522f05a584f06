// include/nlsp_gpu.hpp — header-only C++ shim over the C-ABI (nlsp_gpu.h) that
// gives reference-style call sites (two_level.hpp:22-191, smoothing.hpp:81-100,
// svd.hpp:155-227) a B200 backend:
//
//     nlsp_gpu::Device dev;                                   // one per host thread
//     nlsp_gpu::Matrix A(dev, a);                             // any SparseCsrMatrix-like
//     auto sv = nlsp_gpu::generate_smoothed_vectors(dev, A, mask, K, s1, omega, seed);
//     auto u  = nlsp_gpu::svd_basis(dev, sv, rank);           // first_cols(svd_oracle(S).U, rank)
//     nlsp_gpu::TwoLevelPreconditioner M(dev, A, u, omega, nu1, nu2);
//     nlsp_gpu::PcgResult r = nlsp_gpu::pcg(dev, A, b, M, delta, max_iters);
//
// Reference-signature overloads (pcg(a, b, M, delta, max_iters),
// build_preconditioner, apply_two_level, M.apply(a, r)) take the reference's
// own SparseCsrMatrix and run on a thread-local default device; see below.
//
// `a` may be the reference's nlsp::SparseCsrMatrix itself (dim(), row_ptr(),
// col_idx(), values() with size_t indices, sparse.hpp:62-66) and a basis may be
// its nlsp::DenseMatrix (rows(), cols(), data(), dense.hpp:23-30). Errors throw:
// with NLSP_GPU_REFERENCE_ERRORS defined (after including the reference's
// nlsp/errors.hpp) the reference's own exception types, otherwise the
// same-named types below. The whole PCG loop stays on the device (one call).
#pragma once

#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "nlsp_gpu.h"

namespace nlsp_gpu {

#ifdef NLSP_GPU_REFERENCE_ERRORS
using ValidationError = ::nlsp::ValidationError;
using NumericError = ::nlsp::NumericError;
using NotSpdError = ::nlsp::NotSpdError;
using RankDeficiencyError = ::nlsp::RankDeficiencyError;
using ConvergenceError = ::nlsp::ConvergenceError;
#else
struct ValidationError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NumericError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct NotSpdError : NumericError {
    using NumericError::NumericError;
};
struct RankDeficiencyError : NumericError {
    using NumericError::NumericError;
};
struct ConvergenceError : NumericError {
    using NumericError::NumericError;
};
#endif
struct DeviceError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

inline void check(nlsp_status s, const nlsp_ctx* ctx) {
    if (s == NLSP_OK) return;
    const std::string msg = ctx ? nlsp_last_error(ctx) : "nlsp_gpu";
    switch (s) {
        case NLSP_E_VALIDATION: throw ValidationError(msg);
        case NLSP_E_NUMERIC: throw NumericError(msg);
        case NLSP_E_NOT_SPD: throw NotSpdError(msg);
        case NLSP_E_RANK_DEFICIENT: throw RankDeficiencyError(msg);
        case NLSP_E_CONVERGENCE: throw ConvergenceError(msg);
        default: throw DeviceError(msg.empty() ? "no usable sm_100 device" : msg);
    }
}

class Device {
public:
    explicit Device(int device = 0) {
        nlsp_ctx* c = nullptr;
        check(nlsp_ctx_create(device, &c), nullptr);
        ctx_.reset(c);
    }
    nlsp_ctx* get() const { return ctx_.get(); }
    void* stream() const { return nlsp_ctx_stream(ctx_.get()); }
    // where generate_smoothed_vectors draws S^(0): NLSP_S0_DRAW_HOST (default,
    // bit-identical to the reference's Rng stream) or NLSP_S0_DRAW_DEVICE
    void set_s0_draw(int mode) { check(nlsp_ctx_set_s0_draw(ctx_.get(), mode), ctx_.get()); }
    int last_s0_draw() const { return nlsp_ctx_last_s0_draw(ctx_.get()); }

private:
    struct Del {
        void operator()(nlsp_ctx* c) const { nlsp_ctx_destroy(c); }
    };
    std::unique_ptr<nlsp_ctx, Del> ctx_;
};

// Device copy of a CSR matrix (sparse.hpp:19-113 invariants are checked).
class Matrix {
public:
    Matrix(Device& dev, std::uint64_t n, const std::vector<std::uint64_t>& row_ptr,
           const std::vector<std::uint64_t>& col_idx, const std::vector<double>& values)
        : dev_(&dev), n_(n) {
        if (row_ptr.size() != n + 1 || col_idx.size() != values.size())
            throw ValidationError("Matrix: inconsistent CSR arrays");
        nlsp_csr* a = nullptr;
        check(nlsp_csr_upload(dev.get(), n, values.size(), row_ptr.data(), col_idx.data(),
                              values.data(), &a),
              dev.get());
        csr_.reset(a);
    }
    // any SparseCsrMatrix-like (the reference's nlsp::SparseCsrMatrix included)
    template <class Csr, class = decltype(std::declval<const Csr&>().row_ptr())>
    Matrix(Device& dev, const Csr& a) : dev_(&dev), n_(a.dim()) {
        std::vector<std::uint64_t> rp(a.row_ptr().begin(), a.row_ptr().end());
        std::vector<std::uint64_t> ci(a.col_idx().begin(), a.col_idx().end());
        nlsp_csr* h = nullptr;
        check(nlsp_csr_upload(dev.get(), n_, a.values().size(), rp.data(), ci.data(),
                              a.values().data(), &h),
              dev.get());
        csr_.reset(h);
    }
    std::uint64_t dim() const { return n_; }
    const nlsp_csr* get() const { return csr_.get(); }
    Device& device() const { return *dev_; }

    std::vector<double> spmv(const std::vector<double>& x) const {  // sparse.hpp:116-128
        if (x.size() != n_) throw ValidationError("spmv: dimension mismatch");
        std::vector<double> y(n_);
        check(nlsp_spmv(dev_->get(), csr_.get(), x.data(), y.data()), dev_->get());
        return y;
    }

private:
    struct Del {
        void operator()(nlsp_csr* a) const { nlsp_csr_destroy(a); }
    };
    Device* dev_;
    std::uint64_t n_;
    std::unique_ptr<nlsp_csr, Del> csr_;
};

// Device-resident row-major dense matrix (DenseMatrix, dense.hpp:17-50).
class Dense {
public:
    Dense() = default;
    Dense(Device& dev, std::uint64_t rows, std::uint64_t cols, const double* host) : dev_(&dev) {
        nlsp_dense* d = nullptr;
        check(nlsp_dense_upload(dev.get(), rows, cols, host, &d), dev.get());
        d_.reset(d);
    }
    template <class DM, class = decltype(std::declval<const DM&>().data())>
    Dense(Device& dev, const DM& m) : Dense(dev, m.rows(), m.cols(), m.data()) {}
    Dense(Device& dev, nlsp_dense* owned) : dev_(&dev) { d_.reset(owned); }
    std::uint64_t rows() const {
        std::uint64_t r = 0;
        nlsp_dense_dims(d_.get(), &r, nullptr);
        return r;
    }
    std::uint64_t cols() const {
        std::uint64_t c = 0;
        nlsp_dense_dims(d_.get(), nullptr, &c);
        return c;
    }
    std::vector<double> host() const {
        std::vector<double> out(rows() * cols());
        check(nlsp_dense_export(dev_->get(), d_.get(), out.data()), dev_->get());
        return out;
    }
    const nlsp_dense* get() const { return d_.get(); }
    nlsp_dense* get() { return d_.get(); }
    Device& device() const { return *dev_; }

private:
    struct Del {
        void operator()(nlsp_dense* d) const { nlsp_dense_destroy(d); }
    };
    Device* dev_ = nullptr;
    std::unique_ptr<nlsp_dense, Del> d_;
};

// generate_smoothed_vectors (smoothing.hpp:81-100): S stays on the device
inline Dense generate_smoothed_vectors(Device& dev, const Matrix& a,
                                       const std::vector<bool>& boundary_mask, std::uint64_t k,
                                       std::uint64_t sweeps, double omega, std::uint64_t seed) {
    if (!boundary_mask.empty() && boundary_mask.size() != a.dim())
        throw ValidationError("generate_smoothed_vectors: mask size mismatch");
    std::vector<std::uint8_t> m(boundary_mask.begin(), boundary_mask.end());
    nlsp_dense* s = nullptr;
    check(nlsp_generate_smoothed_vectors(dev.get(), a.get(), m.empty() ? nullptr : m.data(), k,
                                         sweeps, omega, seed, &s),
          dev.get());
    return Dense(dev, s);
}

// first_cols(svd_oracle(S).left_vectors, k) on the device (svd.hpp:155-227)
inline Dense svd_basis(Device& dev, const Dense& s, std::uint64_t k,
                       std::vector<double>* singular_values = nullptr) {
    nlsp_dense* p = nullptr;
    std::vector<double> sig(s.cols());
    check(nlsp_svd_basis(dev.get(), s.get(), k, &p, sig.data(), nullptr), dev.get());
    if (singular_values) *singular_values = std::move(sig);
    return Dense(dev, p);
}

// TwoLevelPreconditioner(a, basis_any, omega, nu1, nu2) (two_level.hpp:22-89)
class TwoLevelPreconditioner {
public:
    TwoLevelPreconditioner(Device& dev, const Matrix& a, const Dense& basis, double omega,
                           std::uint64_t nu1, std::uint64_t nu2)
        : dev_(&dev), nu1_(nu1), nu2_(nu2) {
        nlsp_twolevel* m = nullptr;
        check(nlsp_twolevel_build(dev.get(), a.get(), basis.get(), omega, nu1, nu2, &m), dev.get());
        m_.reset(m);
        nlsp_twolevel_dims(m, &n_, &k_);
    }
    template <class DM, class = decltype(std::declval<const DM&>().data())>
    TwoLevelPreconditioner(Device& dev, const Matrix& a, const DM& basis_any, double omega,
                           std::uint64_t nu1, std::uint64_t nu2)
        : TwoLevelPreconditioner(dev, a, Dense(dev, basis_any), omega, nu1, nu2) {}

    std::uint64_t coarse_dim() const { return k_; }
    std::uint64_t nu1() const { return nu1_; }
    std::uint64_t nu2() const { return nu2_; }
    const nlsp_twolevel* get() const { return m_.get(); }

    std::vector<double> basis() const {
        std::vector<double> b(n_ * k_);
        check(nlsp_twolevel_export(dev_->get(), m_.get(), b.data(), nullptr, nullptr), dev_->get());
        return b;
    }
    std::vector<double> apply(const Matrix& a, const std::vector<double>& rhs) const {
        if (rhs.size() != a.dim()) throw ValidationError("two-level apply: dimension mismatch");
        std::vector<double> z(a.dim());
        check(nlsp_twolevel_apply(a.device().get(), m_.get(), a.get(), rhs.data(), z.data()), a.device().get());
        return z;
    }
    // m.apply(a, r) with the reference's matrix (two_level.hpp:60): uploaded once
    // per thread (device_matrix, below)
    template <class Csr, class = decltype(std::declval<const Csr&>().row_ptr())>
    std::vector<double> apply(const Csr& a, const std::vector<double>& rhs) const;

private:
    struct Del {
        void operator()(nlsp_twolevel* m) const { nlsp_twolevel_destroy(m); }
    };
    Device* dev_;
    std::uint64_t nu1_, nu2_, n_ = 0, k_ = 0;
    std::unique_ptr<nlsp_twolevel, Del> m_;
};

struct IdentityPreconditioner {};  // two_level.hpp:103-106
struct JacobiPreconditioner {};    // two_level.hpp:107-118

// SolveReport / PcgResult (two_level.hpp:121-137). With NLSP_GPU_REFERENCE_TYPES
// (defined after including the reference's nlsp/two_level.hpp) they ARE the
// reference's structs, so `nlsp::PcgResult r = pcg(...)` compiles unchanged.
#ifdef NLSP_GPU_REFERENCE_TYPES
using SolveReport = ::nlsp::SolveReport;
using PcgResult = ::nlsp::PcgResult;
#else
struct SolveReport {
    std::size_t iterations = 0;
    std::vector<double> residual_history;  // ||r_k|| / ||b|| per iteration
    bool converged = false;
    double true_relative_residual = 0.0;
    double inference_ms = 0.0;
    double setup_ms = 0.0;
    double solve_ms = 0.0;
    double total_ms = 0.0;
    std::string method;
    std::size_t coarse_dim = 0;
};
struct PcgResult {
    std::vector<double> solution;
    SolveReport report;
};
#endif

namespace detail {
inline PcgResult run(Device& dev, const Matrix& a, const std::vector<double>& b, int kind,
                     const nlsp_twolevel* m, double delta, std::size_t max_iters) {
    if (b.size() != a.dim()) throw ValidationError("pcg: dimension mismatch");
    PcgResult out;
    out.solution.resize(a.dim());
    nlsp_solve_report rep{};
    check(nlsp_pcg(dev.get(), a.get(), kind, m, b.data(), delta, max_iters, out.solution.data(), &rep,
                   nullptr),
          dev.get());
    // the history, sized by the iterations run (not by max_iters)
    std::vector<double> hist(rep.iterations);
    std::uint64_t cnt = 0;
    check(nlsp_pcg_history(dev.get(), hist.empty() ? nullptr : hist.data(), hist.size(), &cnt), dev.get());
    out.report.iterations = rep.iterations;
    out.report.residual_history = std::move(hist);
    out.report.converged = rep.converged != 0;
    out.report.true_relative_residual = rep.true_relative_residual;
    out.report.solve_ms = rep.solve_ms;
    out.report.total_ms = rep.total_ms;
    out.report.coarse_dim = rep.coarse_dim;
    out.report.method = kind == NLSP_PRECOND_TWOLEVEL ? "two_level" : (kind == NLSP_PRECOND_JACOBI ? "jacobi" : "plain");
    return out;
}
}  // namespace detail

// pcg (two_level.hpp:141-191), the whole loop on the device
inline PcgResult pcg(Device& dev, const Matrix& a, const std::vector<double>& b,
                     const TwoLevelPreconditioner& m, double delta, std::size_t max_iters) {
    return detail::run(dev, a, b, NLSP_PRECOND_TWOLEVEL, m.get(), delta, max_iters);
}
inline PcgResult pcg(Device& dev, const Matrix& a, const std::vector<double>& b,
                     const IdentityPreconditioner&, double delta, std::size_t max_iters) {
    return detail::run(dev, a, b, NLSP_PRECOND_IDENTITY, nullptr, delta, max_iters);
}
inline PcgResult pcg(Device& dev, const Matrix& a, const std::vector<double>& b,
                     const JacobiPreconditioner&, double delta, std::size_t max_iters) {
    return detail::run(dev, a, b, NLSP_PRECOND_JACOBI, nullptr, delta, max_iters);
}

// ---- the reference's own signatures (two_level.hpp:91-101, 141-191) --------
// Reference call sites keep their SparseCsrMatrix and std::vector arguments:
//
//     auto M = nlsp_gpu::build_preconditioner(a, basis, omega, nu1, nu2);  // the one changed line
//     nlsp::PcgResult r = pcg(a, b, M, delta, max_iters);                  // unchanged: ADL picks
//     auto z = apply_two_level(M, a, r);                                   // the device overloads
//
// A thread-local default Device (NLSP_GPU_DEVICE, default 0; one context per
// host thread, as the C-ABI requires) and a small per-thread upload cache stand
// in for the explicit Device/Matrix. The reference's matrices are immutable
// after construction (sparse.hpp:19-113), so a cached upload is keyed by the
// object's address, its arrays' addresses and sizes, and a sampled fingerprint
// of its entries.
namespace detail {
struct CsrKey {
    const void* obj = nullptr;
    const void* rp = nullptr;
    const void* ci = nullptr;
    const void* v = nullptr;
    std::uint64_t n = 0, nnz = 0, fp = 0;
    bool operator==(const CsrKey& o) const {
        return obj == o.obj && rp == o.rp && ci == o.ci && v == o.v && n == o.n && nnz == o.nnz && fp == o.fp;
    }
};
template <class Csr>
CsrKey csr_key(const Csr& a) {
    CsrKey k;
    k.obj = &a;
    k.rp = a.row_ptr().data();
    k.ci = a.col_idx().data();
    k.v = a.values().data();
    k.n = a.dim();
    k.nnz = a.values().size();
    std::uint64_t h = 1469598103934665603ull;  // FNV-1a over <= 64 sampled entries
    const std::uint64_t step = k.nnz > 64 ? k.nnz / 64 : 1;
    for (std::uint64_t i = 0; i < k.nnz; i += step) {
        std::uint64_t bits;
        const double d = a.values()[i];
        std::memcpy(&bits, &d, sizeof bits);
        h = (h ^ bits ^ ((std::uint64_t)a.col_idx()[i] << 17)) * 1099511628211ull;
    }
    k.fp = h;
    return k;
}
struct ThreadState {
    Device dev;  // declared first: destroyed after the cached matrices
    std::vector<std::pair<CsrKey, std::unique_ptr<Matrix>>> cache;
    ThreadState() : dev(std::getenv("NLSP_GPU_DEVICE") ? std::atoi(std::getenv("NLSP_GPU_DEVICE")) : 0) {}
};
inline ThreadState& tls() {
    thread_local ThreadState t;
    return t;
}
}  // namespace detail

// the calling thread's default device
inline Device& default_device() { return detail::tls().dev; }

// the device copy of a reference matrix on this thread's device (cached; the
// four most recent matrices are kept)
template <class Csr, class = decltype(std::declval<const Csr&>().row_ptr())>
const Matrix& device_matrix(const Csr& a) {
    auto& t = detail::tls();
    const detail::CsrKey key = detail::csr_key(a);
    for (auto& e : t.cache)
        if (e.first == key) return *e.second;
    if (t.cache.size() >= 4) t.cache.erase(t.cache.begin());
    t.cache.emplace_back(key, std::make_unique<Matrix>(t.dev, a));
    return *t.cache.back().second;
}

// build_preconditioner (two_level.hpp:91-95): any SparseCsrMatrix-like a and any
// DenseMatrix-like basis (row-major rows() x cols())
template <class Csr, class DM, class = decltype(std::declval<const Csr&>().row_ptr()),
          class = decltype(std::declval<const DM&>().data())>
TwoLevelPreconditioner build_preconditioner(const Csr& a, const DM& basis, double omega, std::size_t nu1,
                                            std::size_t nu2) {
    return TwoLevelPreconditioner(default_device(), device_matrix(a), basis, omega, nu1, nu2);
}
// (the basis already on the device, e.g. svd_basis's output)
template <class Csr, class = decltype(std::declval<const Csr&>().row_ptr())>
TwoLevelPreconditioner build_preconditioner(const Csr& a, const Dense& basis, double omega, std::size_t nu1,
                                            std::size_t nu2) {
    return TwoLevelPreconditioner(default_device(), device_matrix(a), basis, omega, nu1, nu2);
}

// generate_smoothed_vectors(A, boundary_mask, K, sweeps, omega, seed)
// (smoothing.hpp:81-100) with the reference's arguments; S stays on the device
template <class Csr, class = decltype(std::declval<const Csr&>().row_ptr())>
Dense generate_smoothed_vectors(const Csr& a, const std::vector<bool>& boundary_mask, std::size_t k,
                                std::size_t sweeps, double omega, std::uint64_t seed) {
    return generate_smoothed_vectors(default_device(), device_matrix(a), boundary_mask, k, sweeps, omega, seed);
}
// first_cols(svd_oracle(S).left_vectors, k) (svd.hpp:155-227, dense.hpp:158-164)
// on the device of S
inline Dense svd_first_cols(const Dense& s, std::size_t k, std::vector<double>* singular_values = nullptr) {
    return svd_basis(s.device(), s, k, singular_values);
}

#ifdef NLSP_GPU_REFERENCE_TYPES
// exact (non-template) overloads for the reference's own matrix type, so that an
// unqualified pcg(a, b, M, ...) prefers them over the template nlsp::pcg<P>
inline PcgResult pcg(const ::nlsp::SparseCsrMatrix& a, const std::vector<double>& b,
                     const TwoLevelPreconditioner& m, double delta, std::size_t max_iters) {
    return detail::run(default_device(), device_matrix(a), b, NLSP_PRECOND_TWOLEVEL, m.get(), delta, max_iters);
}
inline std::vector<double> apply_two_level(const TwoLevelPreconditioner& m, const ::nlsp::SparseCsrMatrix& a,
                                           const std::vector<double>& rhs) {
    return m.apply(device_matrix(a), rhs);
}
#else
template <class Csr, class = decltype(std::declval<const Csr&>().row_ptr())>
PcgResult pcg(const Csr& a, const std::vector<double>& b, const TwoLevelPreconditioner& m, double delta,
              std::size_t max_iters) {
    return detail::run(default_device(), device_matrix(a), b, NLSP_PRECOND_TWOLEVEL, m.get(), delta, max_iters);
}
template <class Csr, class = decltype(std::declval<const Csr&>().row_ptr())>
std::vector<double> apply_two_level(const TwoLevelPreconditioner& m, const Csr& a, const std::vector<double>& rhs) {
    return m.apply(device_matrix(a), rhs);
}
#endif
template <class Csr, class = decltype(std::declval<const Csr&>().row_ptr())>
PcgResult pcg(const Csr& a, const std::vector<double>& b, const IdentityPreconditioner&, double delta,
              std::size_t max_iters) {
    return detail::run(default_device(), device_matrix(a), b, NLSP_PRECOND_IDENTITY, nullptr, delta, max_iters);
}
template <class Csr, class = decltype(std::declval<const Csr&>().row_ptr())>
PcgResult pcg(const Csr& a, const std::vector<double>& b, const JacobiPreconditioner&, double delta,
              std::size_t max_iters) {
    return detail::run(default_device(), device_matrix(a), b, NLSP_PRECOND_JACOBI, nullptr, delta, max_iters);
}

template <class Csr, class>
std::vector<double> TwoLevelPreconditioner::apply(const Csr& a, const std::vector<double>& rhs) const {
    return apply(device_matrix(a), rhs);
}

}  // namespace nlsp_gpu
