/* oracle.h — CPU restatement of the reference eigenid hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2002_04989_b200/,
 * include/, the C-ABI library) links, loads or calls this code.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * use it, and only as the checker or the timed CPU baseline.
 *
 * Parity status: PINNED.  The restatement is checked bit-for-bit against the
 * unmodified reference compiled from /root/reference/proj/src into
 * oracle/_ref/libeigenid_ref.so (tests/test_oracle.py, tests/golden/).
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj.
 */
#ifndef EIGENID_ORACLE_H
#define EIGENID_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Error codes, mirroring include/eigenid/errors.hpp:11-107. */
enum {
  ORC_OK = 0,
  ORC_E_MATRIX_TOO_SMALL = 1,  /* MatrixTooSmall       errors.hpp:31-34 */
  ORC_E_DEGENERATE = 2,        /* DegenerateEigenvalue errors.hpp:58-66 */
  ORC_E_CONVERGENCE = 3,       /* ConvergenceFailure   errors.hpp:51-54 */
  ORC_E_NONFINITE = 4,         /* NonFiniteIntermediate errors.hpp:69-72 */
  ORC_E_INTERNAL = 5,          /* InternalInconsistency errors.hpp:74-77 */
  ORC_E_CONFIG = 6,            /* ConfigError          errors.hpp:89-92 */
  ORC_E_INDEX = 7,             /* IndexOutOfRange      errors.hpp:26-29 */
  ORC_E_SIGN_RECOVERY = 8,     /* SignRecoveryFailure  errors.hpp:79-82 */
  ORC_E_DIMENSION = 9,         /* DimensionMismatch    errors.hpp:46-49 */
  ORC_E_ALLOC = 30
};

typedef struct {
  int code;
  int64_t index; /* eigenvalue index for degeneracy, -1 otherwise */
  double gap;    /* DegenerateEigenvalue::gap() */
  char msg[256];
} orc_err;

/* ---- seeded inputs: src/matrix_io.cpp:39-71, :171-181; src/matrix.cpp ---- */
void orc_random_symmetric(uint64_t seed, size_t n, int uniform, double* out);
void orc_gaussian_stream(uint64_t seed, size_t count, double* out);
/* C3 input, SURVEY §8 d3 (bit-identical to eigenid_c3_matrix) */
void orc_c3_matrix(uint64_t seed, size_t n, double* out);
uint64_t orc_splitmix64(uint64_t x); /* src/bench.cpp:78-83 */
void orc_minor(const double* a, size_t n, size_t j, double* out); /* matrix.cpp:51-68 */

/* C5 synthetic interlacing spectra: lambda sorted strictly
 * increasing from uniform_open draws; mu_{j,k} = l_k + u_jk (l_{k+1} - l_k). */
void orc_c5_lambda(uint64_t seed, size_t n, double* lambda);
void orc_c5_mu_row(uint64_t seed, const double* lambda, size_t n, size_t j,
                   double* mu);

/* ---- eigensolver: src/eigensolve.cpp ---- */
/* tred1 without Q (eigensolve.cpp:19-69).  max_steps limits the number of
 * Householder steps (SIZE_MAX = full); used only to bound CPU-baseline
 * samples.  offdiag has n-1 entries. */
void orc_tridiagonalize(const double* a, size_t n, size_t max_steps,
                        double* diag, double* offdiag);
/* implicit-shift QL + ascending sort (eigensolve.cpp:72-128). d in/out. */
int orc_ql(double* d, const double* offdiag, size_t n, orc_err* err);
int orc_eigenvalues(const double* a, size_t n, double* out, orc_err* err);

/* ---- identity engine: src/identity.cpp ---- */
int orc_check_fully_nondegenerate(const double* s, size_t n, double tol,
                                  orc_err* err); /* identity.cpp:141-149 */
/* One |v_ij|^2: evaluate() (identity.cpp:185-238).  log_domain selects
 * IdentityConfig::Evaluation::kLogDomain.  Returns status; *raw and *value
 * receive raw_value / value; *method: 1 batched, 3 log-domain. */
int orc_evaluate(const double* lambda, const double* mu, size_t n, size_t i,
                 size_t batch, double tol, int log_domain, double* raw,
                 double* value, int* method, orc_err* err);
/* log_domain_product over an explicit pairing (identity.cpp:98-122). */
int orc_log_domain_product(const double* num, const double* den, size_t len,
                           double* out, orc_err* err);
/* Identity stage only, rows j0..j1 of out[j*n+i] from given spectra
 * (mu is row-major, row j has n-1 ascending values).  Threads >= 1. */
int orc_identity_rows(const double* lambda, const double* mu, size_t n,
                      size_t j0, size_t j1, size_t batch, double tol,
                      int log_domain, int threads, double* out, orc_err* err);
/* Full pipeline all_magnitudes (identity.cpp:294-316).  lambda_out (n) and
 * mu_out (n*(n-1)) are optional. */
int orc_all_magnitudes(const double* a, size_t n, size_t batch, double tol,
                       int log_domain, int threads, double* out,
                       double* lambda_out, double* mu_out, orc_err* err);
/* Minor spectra for a list of minor indices, one minor per thread
 * (identity.cpp:303-306). mu is count x (n-1). */
/* ---- sign recovery: src/signs.cpp:48-120 ---- */
/* Signed eigenvector from squared magnitudes (n entries in out). */
int orc_recover_signs(const double* a, size_t n, size_t i, const double* mags,
                      size_t nmags, double lambda_i, double sign_tol,
                      double* out, orc_err* err);

int orc_minor_spectra(const double* a, size_t n, const size_t* js,
                      size_t count, int threads, double* mu, orc_err* err);

#ifdef __cplusplus
}
#endif
#endif
