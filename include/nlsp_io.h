/* include/nlsp_io.h — the reference's on-disk inputs for the solver path
 * (SURVEY §8f.2), host C++ in paper_2601_20174_b200/csrc/io.cpp →
 * libnlsp_io.so.
 *
 * Two entry points feed nlsp_csr_upload / nlsp_pcg (include/nlsp_gpu.h) with
 * what the reference's pipeline reads from disk:
 *
 *   nlsp_io_load_matrix_market   load_matrix_market   (sparse.hpp:168-194)
 *   nlsp_io_save_matrix_market   save_matrix_market   (sparse.hpp:148-166)
 *   nlsp_io_load_instance        load_instance        (instance_io.hpp:137-185)
 *
 * Semantics follow the reference exactly: the same header checks and error
 * classes, entries read as whitespace-separated tokens the way
 * `std::istream >> size_t >> size_t >> double` reads them, a "symmetric"
 * header mirrors off-diagonal entries, and the triplets go through
 * SparseCsrMatrix::from_triplets (sparse.hpp:24-53): (row, col) order,
 * duplicates summed, exact zeros dropped, out-of-range indices rejected.
 * Doubles are parsed correctly rounded (as strtod), so a file written with
 * %.17g reloads bit for bit. Duplicate (row, col) entries are summed in file
 * order; the reference's unstable std::sort leaves that order unspecified
 * (files written by save_matrix_market never contain duplicates).
 *
 * The CSR arrays use the reference layout (uint64 row_ptr[n+1], col_idx[nnz],
 * fp64 values[nnz]) and are owned by the caller after a successful load: free
 * them with nlsp_io_csr_free / nlsp_io_instance_free.
 */
#ifndef NLSP_IO_H
#define NLSP_IO_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status values shared with nlsp_status (include/nlsp_gpu.h) */
#define NLSP_IO_OK 0
#define NLSP_IO_E_VALIDATION 1 /* nlsp::ValidationError (bad index, manifest, family) */
#define NLSP_IO_E_IO 8         /* nlsp::IoError (open / header / truncated)          */

typedef struct {
    uint64_t n, nnz;
    uint64_t* row_ptr; /* n + 1 */
    uint64_t* col_idx; /* nnz */
    double* values;    /* nnz */
} nlsp_host_csr;

/* load_matrix_market(path) (sparse.hpp:168-194). */
int nlsp_io_load_matrix_market(const char* path, nlsp_host_csr* out);

/* save_matrix_market(a, path) (sparse.hpp:148-166): "real symmetric", lower
 * triangle, 1-based, %.17g values. */
int nlsp_io_save_matrix_market(const nlsp_host_csr* a, const char* path);

void nlsp_io_csr_free(nlsp_host_csr* a);

/* PdeInstance (fem.hpp:202-211) as load_instance reads it
 * (instance_io.hpp:137-185): manifest.txt, vertices.csv, triangles.csv,
 * matrix.mtx, rhs.csv, coefficients.csv. */
typedef struct {
    int family;       /* 0 diffusion, 1 anisotropic, 2 screened_poisson */
    uint64_t grid_n;  /* manifest N    */
    uint64_t seed;    /* manifest seed */
    double jitter;    /* manifest jitter */
    double alpha;     /* screened Poisson reaction weight (manifest alpha), else 0 */
    nlsp_host_csr matrix;
    double* rhs;             /* matrix.n */
    uint64_t n_vertices;
    double* vertices;        /* n_vertices x 2 (x, y) */
    uint8_t* boundary_mask;  /* n_vertices (1 = Dirichlet row; the mask of generate_smoothed_vectors) */
    uint64_t n_triangles;
    uint64_t* triangles;     /* n_triangles x 3 */
    uint64_t coeff_cols;     /* 1 (g or kappa) or 3 (k11, k12, k22) */
    double* coefficients;    /* n_triangles x coeff_cols */
} nlsp_instance;

int nlsp_io_load_instance(const char* dir, nlsp_instance* out);
void nlsp_io_instance_free(nlsp_instance* inst);

/* MlpModel (mlp.hpp:47-320): layer widths and the flat parameter buffer in
 * the reference's order — per layer l: W_l (fan_out x fan_in, row-major), b_l,
 * and for hidden layers the LayerNorm gain_l, offset_l. */
typedef struct {
    uint64_t nwidths;
    uint64_t* widths;
    uint64_t nparams;
    double* params;
    char* manifest;  /* NUL-terminated checkpoint manifest text (may be empty) */
} nlsp_host_mlp;

/* MlpModel::load(path) (mlp.hpp:276-303): "NLSPCKP1" checkpoint; the Adam
 * state is read past, not kept. IoError on bad magic / count / truncation. */
int nlsp_io_mlp_load(const char* path, nlsp_host_mlp* out);

/* MlpModel::save(path, manifest) (mlp.hpp:255-274) with zero Adam state. */
int nlsp_io_mlp_save(const nlsp_host_mlp* m, const char* path);

/* MlpModel(widths, seed) (mlp.hpp:57-88): the reference's seeded He
 * initialisation (Rng(mix_seed(seed, 0x6d6c70)), bit-identical), gains 1. */
int nlsp_io_mlp_init(const uint64_t* widths, uint64_t nwidths, uint64_t seed, nlsp_host_mlp* out);

void nlsp_io_mlp_free(nlsp_host_mlp* m);

/* Message of the last failed call on this thread. */
const char* nlsp_io_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* NLSP_IO_H */
