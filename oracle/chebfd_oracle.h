/* CPU restatement of the ChebFD hot path -- TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library, and only as the checker.  The product library
 * (paper_1510_04895_b200/csrc) never links it.
 *
 * Every function restates one reference function line by line (file:line
 * relative to /root/reference/proj) with a single row chunk (the reference
 * with CHEBFD_THREADS=1), so integer/generator/RNG outputs and every
 * row-local floating-point result are bit-identical to the reference, and
 * the chunked reductions equal the reference's 1-thread results.
 *
 * Pinning: tests/test_oracle.py checks this library against
 *   (a) golden fixtures written by tests/golden/make_golden.py from the real
 *       reference (oracle/_ref/libchebfd_ref.so, built by oracle/Makefile);
 *   (b) the reference's own known-answer tests (SURVEY.md §8c list);
 *   (c) oracle/_ref directly, when it is present.
 *
 * Complex numbers are interleaved (re, im) doubles, i.e. the memory layout of
 * std::complex<double>.  Block vectors are D x nb row-major
 * (block_vector.hpp:15-16).  kind: 0 = real64, 1 = complex128 (scalar.hpp:12).
 */
#ifndef CHEBFD_ORACLE_H
#define CHEBFD_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG: std::mt19937_64 + libstdc++ normal_distribution ---- */
typedef struct {
    uint64_t mt[312];
    int mti;
    int have_saved;
    double saved;
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed);
uint64_t orc_rng_next(orc_rng* r);
void orc_rng_discard(orc_rng* r, uint64_t n);
double orc_rng_canonical(orc_rng* r);
double orc_rng_normal(orc_rng* r);

/* BlockVector::randomize (block_vector.hpp:42-51) */
void orc_randomize(int kind, int64_t dim, int64_t width, uint64_t seed, void* out);

/* ---- models (models.cpp) ---- */
/* boundary: 0 periodic_xy_open_z, 1 periodic_all, 2 open_all (models.hpp:13) */
/* Two-call pattern: pass NULL arrays to get dim/nnz, then call again with
 * arrays of size dim+1 / nnz / nnz. */
int orc_graphene(int64_t lx, int64_t ly, double t, double disorder, int boundary, uint64_t seed,
                 int64_t* dim, int64_t* nnz, int64_t* offs, int64_t* cols, double* vals);
int orc_topological_insulator(int64_t lx, int64_t ly, int64_t lz, double t, double disorder,
                              int boundary, uint64_t seed, int64_t* dim, int64_t* nnz,
                              int64_t* offs, int64_t* cols, double* vals /* complex */);

/* ---- filter coefficients (filter.cpp) ---- */
/* kernel kind: 0 none, 1 fejer, 2 jackson, 3 lanczos(mu) (filter.hpp:12) */
int orc_window_coeffs(double tlo, double thi, double blo, double bhi, int degree, double* out);
int orc_kernel_coeffs(int kind, int mu, int degree, double* out);
int orc_make_filter(double tlo, double thi, double blo, double bhi, int degree, int kind, int mu,
                    double* combined, double* alpha, double* beta);
double orc_eval_scalar(const double* combined, int degree, double alpha, double beta, double x);

/* ---- kernels (kernels.hpp), CSR with int64 offsets/cols ---- */
typedef struct {
    int kind;
    int64_t dim;
    const int64_t* offs;
    const int64_t* cols;
    const double* vals; /* complex: interleaved */
} orc_csr;

int orc_spmmvm(const orc_csr* a, const double* x, int64_t nb, double alpha, double beta,
               double* y);
int orc_spmmvm_fused(const orc_csr* a, const double* u, double* w, double* x, int64_t nb,
                     double alpha, double beta, double coeff, double* dots);
int orc_recurrence_step(const orc_csr* a, const double* u, double* w, int64_t nb, double alpha,
                        double beta);
void orc_block_axpy_scal(int kind, int64_t dim, int64_t nb, double* x, const double* u,
                         const double* w, double c0, double c1, double c2);
void orc_column_dots(int kind, int64_t dim, int64_t nb, const double* x, const double* y,
                     double* d);
void orc_gram(int kind, int64_t dim, const double* x, int64_t nx, const double* y, int64_t ny,
              double* g);
void orc_block_mult_small(int kind, int64_t dim, int64_t nb, const double* x, const double* b,
                          int64_t bcols, double* y);
void orc_column_norms(int kind, int64_t dim, int64_t nb, const double* x, double* out);

/* apply_filter (filter.hpp:73-116); moments: (degree+1) x nb or NULL */
int orc_apply_filter(const orc_csr* a, double* x, int64_t nb, const double* combined, int degree,
                     double alpha, double beta, double* moments);

/* bench conventions (bench.cpp:28-34) */
double orc_per_row_flops(double n_nzr, int f_a, int f_m);
double orc_per_row_bytes(double n_nzr, int s_d, int s_i, int n_b);

#ifdef __cplusplus
}
#endif
#endif
