/* oracle/nlsp_oracle.h — TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C restatement of the reference hot path (NeuraLSP `nlsp`, header-only
 * C++ under /root/reference/proj/include/nlsp/). Every function cites the
 * reference lines it restates. Built with -ffp-contract=off, so every operation
 * rounds exactly where the reference's source expression does: bitwise equal to
 * the reference compiled with -ffp-contract=off (oracle/_ref/libnlsp_ref_strict.so)
 * and within rounding of the reference's default -O3 -march=... build.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may load
 * this library, and only as the checker. The product (libnlsp_gpu.so) never
 * links it.
 *
 * Status codes equal nlsp_status in include/nlsp_gpu.h.
 */
#ifndef NLSP_ORACLE_H
#define NLSP_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ORC_OK = 0,
    ORC_VALIDATION = 1,
    ORC_NUMERIC = 2,
    ORC_NOT_SPD = 3,
    ORC_RANK_DEFICIENT = 4,
    ORC_CONVERGENCE = 5
};

const char* orc_last_error(void);

/* rng.hpp:12-73 */
uint64_t orc_mix_seed(uint64_t seed, uint64_t tag);
void orc_rng_u64_fill(uint64_t seed, uint64_t count, uint64_t* out);
void orc_rng_normal_fill(uint64_t seed, uint64_t count, double* out);
void orc_rng_uniform_fill(uint64_t seed, uint64_t count, double lo, double hi, double* out);

/* CSR with the reference's size_t index layout (sparse.hpp:108-112) */
int orc_spmv(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
             const double* x, double* y);
int orc_inv_diag(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                 double omega, double* dinv);
int orc_jacobi_sweep(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                     double omega, uint64_t sweeps, double* x, const double* b);
int orc_block_sweeps(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                     uint64_t m, double* s, uint64_t sweeps, double omega);
int orc_generate_smoothed_vectors(uint64_t n, const uint64_t* rp, const uint64_t* ci,
                                  const double* v, const uint8_t* mask, uint64_t k,
                                  uint64_t sweeps, double omega, uint64_t seed, double* s_out);

/* dense.hpp / svd.hpp / qr.hpp / cholesky.hpp */
void orc_matmul_tn(uint64_t rows, uint64_t ca, uint64_t cb, const double* a, const double* b,
                   double* c);
double orc_orthonormality_defect(uint64_t rows, uint64_t cols, const double* a);
int orc_jacobi_eigh(uint64_t n, const double* g, double* evals, double* evecs, int* sweeps);
int orc_svd(uint64_t rows, uint64_t cols, const double* s, double* u, double* sigma, double* v,
            int* sweeps);
int orc_qr_thin(uint64_t n, uint64_t k, const double* m, double* q, double* r);
int orc_cholesky(uint64_t n, const double* a, double* l);
void orc_cholesky_solve_factored(uint64_t n, const double* l, const double* rhs, double* x);

/* two_level.hpp:22-191 */
typedef struct orc_twolevel orc_twolevel;
int orc_twolevel_create(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                        uint64_t k, const double* basis_any, double omega, uint64_t nu1,
                        uint64_t nu2, orc_twolevel** out);
void orc_twolevel_destroy(orc_twolevel* t);
int orc_twolevel_from_parts(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v,
                            uint64_t k, const double* basis, const double* coarse, double omega,
                            uint64_t nu1, uint64_t nu2, orc_twolevel** out);
/* basis_ (n x k), L (k x k), symmetrised Galerkin operator A_c (k x k) */
void orc_twolevel_export(const orc_twolevel* t, double* basis, double* chol, double* coarse);
int orc_twolevel_apply(const orc_twolevel* t, uint64_t n, const uint64_t* rp,
                       const uint64_t* ci, const double* v, const double* r, double* z);

/* kind: 0 identity, 1 Jacobi (diagonal), 2 two-level */
int orc_pcg(uint64_t n, const uint64_t* rp, const uint64_t* ci, const double* v, int kind,
            const orc_twolevel* t, const double* b, double delta, uint64_t max_iters, double* x,
            double* hist, uint64_t hist_cap, uint64_t* iterations, int* converged,
            double* true_res);

#ifdef __cplusplus
}
#endif
#endif
