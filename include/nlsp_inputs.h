/* include/nlsp_inputs.h — seeded synthetic inputs for the BASELINE.json configs.
 *
 * Host-side C++ (paper_2601_20174_b200/csrc/inputs.cpp → libnlsp_inputs.so).
 * None of these operators exist in the reference (it only has P1 FEM,
 * fem.hpp); they restate BASELINE.json configs C1–C5. Both the
 * GPU path and the CPU oracle consume the arrays these functions produce.
 *
 * The random streams restate the reference's Rng/mix_seed (rng.hpp:12-73):
 * std::mt19937_64, top-53-bit uniforms, Box–Muller with the cached sine value,
 * so the reference itself can regenerate every stream (tests pin this).
 *
 * CSR arrays use the reference layout (sparse.hpp:108-112): uint64 row_ptr
 * (n+1) and col_idx (nnz), fp64 values, columns sorted within a row, no
 * duplicates, no stored zeros.
 */
#ifndef NLSP_INPUTS_H
#define NLSP_INPUTS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    NLSP_PROBLEM_POISSON2D_FD = 1,   /* C1: 5-point FD, nx*ny interior, diag 4 / off -1 */
    NLSP_PROBLEM_DIFFUSION2D_FV = 2, /* C2: cell-centred FV, a = exp(GRF), harmonic faces */
    NLSP_PROBLEM_ANISO2D_9PT = 3,    /* C3: 9-point rotated-tensor stencil */
    NLSP_PROBLEM_POISSON3D_FD = 4,   /* C4: 7-point FD, nx*ny*nz interior */
    NLSP_PROBLEM_ELASTICITY2D_Q1 = 5 /* C5: Q1 plane strain, left edge clamped */
} nlsp_problem_kind;

typedef struct {
    int kind;            /* nlsp_problem_kind */
    uint64_t nx, ny, nz; /* grid (interior points / cells / elements per side) */
    uint64_t seed;       /* master seed: RHS, GRF and Young's-modulus streams */
    double epsilon;      /* C3 anisotropy ratio (1e-3) */
    double theta;        /* C3 rotation angle (pi/6) */
    double corr_len;     /* C2 GRF correlation length, fraction of the domain (0.1) */
    double variance;     /* C2 GRF variance (1.0) */
    uint64_t blocks;     /* C5 checkerboard blocks per side (16) */
    double young_lo;     /* C5 log-uniform Young's modulus range [lo, hi] (1, 1e3) */
    double young_hi;
    double poisson;      /* C5 Poisson ratio (0.3) */
    int rhs_uniform;     /* 0: RHS ~ N(0,1); 1: RHS ~ U[-1,1] (C3) */
} nlsp_problem_spec;

typedef struct nlsp_problem nlsp_problem;

/* Builds the operator and right-hand side. Returns 0 on success, 1 on bad
 * arguments (message via nlsp_inputs_last_error). */
int nlsp_problem_create(const nlsp_problem_spec* spec, nlsp_problem** out);
void nlsp_problem_destroy(nlsp_problem* p);
uint64_t nlsp_problem_n(const nlsp_problem* p);
uint64_t nlsp_problem_nnz(const nlsp_problem* p);
/* copy-out; any pointer may be NULL. mask: 1 for Dirichlet rows kept as
 * identity rows (C5), all-zero for eliminated-BC operators. coef: per-cell
 * coefficient field (C2 a = exp(g)) or per-element E (C5), may be NULL. */
void nlsp_problem_export(const nlsp_problem* p, uint64_t* row_ptr, uint64_t* col_idx,
                         double* values, double* rhs, uint8_t* mask);
uint64_t nlsp_problem_coef_len(const nlsp_problem* p);
void nlsp_problem_export_coef(const nlsp_problem* p, double* coef);
const char* nlsp_inputs_last_error(void);

/* Reference RNG restatement (rng.hpp:12-73). */
uint64_t nlsp_mix_seed(uint64_t seed, uint64_t tag);
void nlsp_rng_normal_fill(uint64_t seed, uint64_t count, double* out);
void nlsp_rng_uniform_fill(uint64_t seed, uint64_t count, double lo, double hi, double* out);
/* nlsp_rng_normal_fill produces the stream of Rng(seed).normal() on several
 * threads, each jumping its own mt19937_64 to its slice (csrc/mt_jump.hpp).
 * The checks of that: the plain serial loop; the threaded stream with its
 * chunk size (pairs), widened u1 rejection and worker cap exposed; raw
 * mt19937_64 outputs after `skip` words by discard and by jump-ahead (skip a
 * multiple of 2^17; returns 0 on success). */
void nlsp_rng_normal_serial(uint64_t seed, uint64_t count, double zero_below, double* out);
void nlsp_rng_normal_chunks(uint64_t seed, uint64_t count, uint64_t chunk_pairs, double zero_below,
                            uint32_t max_workers, double* out);
void nlsp_mt19937_64_fill(uint64_t seed, uint64_t skip, uint64_t count, uint64_t* out);
int nlsp_mt19937_64_jump_fill(uint64_t seed, uint64_t skip, uint64_t count, uint64_t* out);

/* S^(0) exactly as generate_smoothed_vectors fills it before sweeping
 * (smoothing.hpp:88-96): Rng(mix_seed(seed, 0x736d6f6f)), row-major i outer /
 * j inner, rows with mask[i] != 0 are zero and draw nothing. mask may be NULL. */
void nlsp_smoothed_s0(uint64_t seed, uint64_t n, uint64_t m, const uint8_t* mask, double* out);

#ifdef __cplusplus
}
#endif
#endif
