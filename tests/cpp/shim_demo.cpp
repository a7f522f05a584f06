// tests/cpp/shim_demo.cpp — the reference's bench_single SVD row
// (pipeline.hpp:303-346) written against include/nlsp_gpu.hpp.
//
// Built twice by __graft_entry__.build():
//   shim_demo      with local SparseCsrMatrix/DenseMatrix-like types
//   shim_demo_ref  with the reference's own nlsp::SparseCsrMatrix and
//                  nlsp::ValidationError (only where /root/reference exists),
//                  showing the shim accepts the reference's types unchanged.
//
// usage: shim_demo <dir>   where <dir> holds, in dense.hpp's binary layout
// (u64 rows, u64 cols, f64 row-major): csr_rp.bin, csr_ci.bin, csr_v.bin (as
// n x 1 columns of doubles), rhs.bin, params.bin = [k, m, s1, nu1, nu2, omega,
// delta, s0_seed]. Writes x.bin and prints one JSON line.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <fstream>
#include <string>
#include <tuple>
#include <vector>

#ifdef WITH_REFERENCE
#include "nlsp/dense.hpp"
#include "nlsp/errors.hpp"
#include "nlsp/sparse.hpp"
#include "nlsp/two_level.hpp"
#define NLSP_GPU_REFERENCE_ERRORS
#define NLSP_GPU_REFERENCE_TYPES
#endif
#include "nlsp_gpu.hpp"

namespace {

std::vector<double> load(const std::string& path, std::uint64_t* rows = nullptr) {
    std::ifstream in(path, std::ios::binary);
    std::uint64_t dims[2] = {0, 0};
    in.read(reinterpret_cast<char*>(dims), sizeof dims);
    std::vector<double> v(dims[0] * dims[1]);
    in.read(reinterpret_cast<char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
    if (rows) *rows = dims[0];
    return v;
}

void save(const std::string& path, const std::vector<double>& v) {
    std::ofstream out(path, std::ios::binary);
    const std::uint64_t dims[2] = {v.size(), 1};
    out.write(reinterpret_cast<const char*>(dims), sizeof dims);
    out.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * 8));
}

#ifndef WITH_REFERENCE
// the accessor surface of nlsp::DenseMatrix (dense.hpp:17-30)
struct LocalDense {
    std::size_t r, c;
    std::vector<double> a;
    LocalDense(std::size_t rows, std::size_t cols) : r(rows), c(cols), a(rows * cols) {}
    std::size_t rows() const { return r; }
    std::size_t cols() const { return c; }
    double* data() { return a.data(); }
    const double* data() const { return a.data(); }
};
// the accessor surface of nlsp::SparseCsrMatrix (sparse.hpp:62-66)
struct LocalCsr {
    std::size_t n;
    std::vector<std::size_t> rp, ci;
    std::vector<double> v;
    std::size_t dim() const { return n; }
    const std::vector<std::size_t>& row_ptr() const { return rp; }
    const std::vector<std::size_t>& col_idx() const { return ci; }
    const std::vector<double>& values() const { return v; }
};
#endif

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) {
        std::fprintf(stderr, "usage: %s <dir>\n", argv[0]);
        return 2;
    }
    const std::string dir = argv[1];
    const auto rp_d = load(dir + "/csr_rp.bin"), ci_d = load(dir + "/csr_ci.bin");
    const auto v = load(dir + "/csr_v.bin"), rhs = load(dir + "/rhs.bin"), prm = load(dir + "/params.bin");
    const std::size_t n = rp_d.size() - 1;
#ifdef WITH_REFERENCE
    std::vector<std::tuple<std::size_t, std::size_t, double>> trip;
    for (std::size_t i = 0; i < n; ++i)
        for (std::size_t k = (std::size_t)rp_d[i]; k < (std::size_t)rp_d[i + 1]; ++k)
            trip.emplace_back(i, (std::size_t)ci_d[k], v[k]);
    const auto a = nlsp::SparseCsrMatrix::from_triplets(n, std::move(trip));
#else
    LocalCsr a{n, {}, {}, v};
    for (double x : rp_d) a.rp.push_back((std::size_t)x);
    for (double x : ci_d) a.ci.push_back((std::size_t)x);
#endif
    const std::uint64_t k = (std::uint64_t)prm[0], m = (std::uint64_t)prm[1], s1 = (std::uint64_t)prm[2];
    const std::uint64_t nu1 = (std::uint64_t)prm[3], nu2 = (std::uint64_t)prm[4];
    const double omega = prm[5], delta = prm[6];
    const std::uint64_t seed = (std::uint64_t)prm[7];

    nlsp_gpu::Device dev;
    nlsp_gpu::Matrix A(dev, a);
    auto s = nlsp_gpu::generate_smoothed_vectors(dev, A, {}, m, s1, omega, seed);
    std::vector<double> sigma;
    auto u = nlsp_gpu::svd_basis(dev, s, k, &sigma);
    nlsp_gpu::TwoLevelPreconditioner precond(dev, A, u, omega, nu1, nu2);
    const auto res = nlsp_gpu::pcg(dev, A, rhs, precond, delta, 10 * n);
    const auto plain = nlsp_gpu::pcg(dev, A, rhs, nlsp_gpu::IdentityPreconditioner{}, delta, 10 * n);
    save(dir + "/x.bin", res.solution);

    // The reference's own call site, unchanged but for the namespace of
    // build_preconditioner (two_level.hpp:91-101, 141-191): the matrix stays the
    // reference's SparseCsrMatrix, the basis a host DenseMatrix, and the
    // unqualified pcg / apply_two_level resolve to the device overloads.
#ifdef WITH_REFERENCE
    using HostDense = nlsp::DenseMatrix;
    using nlsp::PcgResult;
#else
    using HostDense = LocalDense;
    using nlsp_gpu::PcgResult;
#endif
    // the setup through the reference-signature helpers as well
    auto s_ref = nlsp_gpu::generate_smoothed_vectors(a, std::vector<bool>{}, m, s1, omega, seed);
    const auto u_ref = nlsp_gpu::svd_first_cols(s_ref, k).host();
    const auto uh = u.host();
    double u_diff = 0.0;
    for (std::size_t i = 0; i < uh.size(); ++i) u_diff = std::fmax(u_diff, std::fabs(u_ref[i] - uh[i]));
    HostDense basis(n, k);
    std::copy(uh.begin(), uh.end(), basis.data());
    auto M = nlsp_gpu::build_preconditioner(a, basis, omega, nu1, nu2);
#ifdef WITH_REFERENCE
    PcgResult ref_style = pcg(a, rhs, M, delta, 10 * n);
    const auto z_free = apply_two_level(M, a, rhs);
#else
    PcgResult ref_style = nlsp_gpu::pcg(a, rhs, M, delta, 10 * n);
    const auto z_free = nlsp_gpu::apply_two_level(M, a, rhs);
#endif
    const auto z_member = M.apply(a, rhs);
    const auto z_dev = precond.apply(A, rhs);
    double z_diff = 0.0, z_norm = 0.0, x_diff = 0.0;
    for (std::size_t i = 0; i < n; ++i) {
        z_diff = std::fmax(z_diff, std::fabs(z_free[i] - z_dev[i]) + std::fabs(z_member[i] - z_dev[i]));
        z_norm = std::fmax(z_norm, std::fabs(z_dev[i]));
        x_diff = std::fmax(x_diff, std::fabs(ref_style.solution[i] - res.solution[i]));
    }

    // error mapping: the reference's ValidationError for a zero right-hand side
    bool zero_rhs_rejected = false;
    try {
        nlsp_gpu::pcg(dev, A, std::vector<double>(n, 0.0), precond, delta, 10);
    } catch (const nlsp_gpu::ValidationError&) {
        zero_rhs_rejected = true;
    }
    std::printf(
        "{\"n\": %zu, \"iterations\": %zu, \"converged\": %d, \"true_relative_residual\": %.6e, "
        "\"plain_iterations\": %zu, \"history_len\": %zu, \"zero_rhs_rejected\": %d, "
        "\"solve_ms\": %.3f, \"ref_style_iterations\": %zu, \"ref_style_history_len\": %zu, "
        "\"ref_style_method\": \"%s\", \"ref_style_x_maxdiff\": %.3e, \"apply_rel_diff\": %.3e, "
        "\"ref_style_basis_maxdiff\": %.3e, "
        "\"reference_types\": %d}\n",
        n, res.report.iterations, res.report.converged ? 1 : 0, res.report.true_relative_residual,
        plain.report.iterations, res.report.residual_history.size(), zero_rhs_rejected ? 1 : 0,
        res.report.solve_ms, ref_style.report.iterations, ref_style.report.residual_history.size(),
        ref_style.report.method.c_str(), x_diff, z_diff / (z_norm > 0 ? z_norm : 1.0), u_diff,
#ifdef WITH_REFERENCE
        1
#else
        0
#endif
    );
    return 0;
}
