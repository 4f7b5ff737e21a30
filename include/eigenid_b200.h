/* eigenid_b200.h — C-ABI of the B200-native eigenvector–eigenvalue identity.
 *
 * This is the drop-in boundary for the reference hot path
 * IdentityEngine::all_magnitudes (proj/src/identity.cpp:294-316) and the
 * eigenvalue solver under it (proj/src/eigensolve.cpp:19-132).  The C++ host
 * layer (include/eigenid/*.hpp, paper_2002_04989_b200/host/) and the Python
 * mirror (paper_2002_04989_b200/engine.py) call only these entry points.
 *
 * Conventions
 *  - All matrices are dense row-major FP64, symmetric; only the lower triangle
 *    is read (the reference's build() guarantees exact symmetry,
 *    proj/src/matrix.cpp:10-38).
 *  - Output layout matches the reference: out[j*n + i] = |v_ij|^2, i the
 *    ascending eigenvalue index, j the component (identity.cpp:311-313).
 *  - Minor spectra mu are row-major, row j = ascending eigenvalues of M_j.
 *  - Host-pointer entry points are synchronous and return an int status
 *    (EIGENID_OK or an error code); `err` (nullable) receives the detail.
 *    No exception ever crosses this boundary; the host layers re-throw the
 *    matching eigenid::Error subclass (proj/include/eigenid/errors.hpp).
 *  - *_device entry points take device pointers and a cudaStream_t (passed as
 *    void*), enqueue work, and report errors at the next eigenid_gpu_sync()
 *    (or the next host-pointer call, which also reads the status).  The
 *    status is sticky: the FIRST error of the enqueued calls is reported,
 *    and every stage of a later enqueued call stops early once it is set.
 *  - Input matrices are checked for non-finite entries on the device
 *    (EIGENID_E_NONFINITE_ENTRY, err->index = entry, before any solve), as
 *    SymmetricMatrix::build does (matrix.cpp:17-18).
 *  - A degenerate lambda(A) (EIGENID_E_DEGENERATE) stops the minor solves
 *    early: lambda(A) is solved first, beside the minors, and the minors'
 *    work queues stop pulling once the degeneracy check fails
 *    (identity.cpp:299-300 throws before any minor solve).
 *  - A bisection that exhausts its iteration budget, or a non-finite
 *    tridiagonal, is EIGENID_E_CONVERGENCE (eigensolve.cpp:90-93).
 *  - There is no CPU fallback: a missing device is EIGENID_E_DEVICE.
 */
#ifndef EIGENID_B200_H
#define EIGENID_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EIGENID_B200_ABI_VERSION 1

/* Status codes; 1..7 mirror the reference's typed errors. */
enum eigenid_status {
  EIGENID_OK = 0,
  EIGENID_E_MATRIX_TOO_SMALL = 1, /* MatrixTooSmall        errors.hpp:31-34 */
  EIGENID_E_DEGENERATE = 2,       /* DegenerateEigenvalue  errors.hpp:58-66 */
  EIGENID_E_CONVERGENCE = 3,      /* ConvergenceFailure    errors.hpp:51-54 */
  EIGENID_E_NONFINITE = 4,        /* NonFiniteIntermediate errors.hpp:69-72 */
  EIGENID_E_INTERNAL = 5,         /* InternalInconsistency errors.hpp:74-77 */
  EIGENID_E_CONFIG = 6,           /* ConfigError           errors.hpp:89-92 */
  EIGENID_E_INDEX = 7,            /* IndexOutOfRange       errors.hpp:26-29 */
  EIGENID_E_SIGN_RECOVERY = 8,    /* SignRecoveryFailure   errors.hpp:79-82 */
  EIGENID_E_DIMENSION = 9,        /* DimensionMismatch     errors.hpp:46-49 */
  EIGENID_E_NONFINITE_ENTRY = 10, /* NonFiniteEntry        errors.hpp:21-24,
                                     raised by build(), matrix.cpp:17-18 */
  EIGENID_E_ASYMMETRIC = 11,      /* AsymmetricInput       errors.hpp:16-19
                                     (host mirrors only: the ABI reads the
                                     lower triangle) */
  EIGENID_E_DEVICE = 20,          /* new: CUDA failure / no device          */
  EIGENID_E_ALLOC = 21            /* new: device allocation failed          */
};

typedef struct eigenid_gpu_err {
  int code;        /* eigenid_status */
  int64_t index;   /* eigenvalue index (degeneracy) or matrix index; -1 */
  double gap;      /* DegenerateEigenvalue::gap() */
  int cuda_error;  /* cudaError_t when code == EIGENID_E_DEVICE */
  char msg[256];
} eigenid_gpu_err;

/* Mirrors IdentityConfig (proj/include/eigenid/identity.hpp:81-93); the
 * reference's `workers` has no device meaning and is absent. */
typedef struct eigenid_gpu_config {
  size_t batch_size;     /* >= 1, default 64 */
  double degeneracy_tol; /* >= 0, default 1e-12, relative to spectral range */
  int log_domain;        /* 1 = Evaluation::kLogDomain */
} eigenid_gpu_config;

typedef struct eigenid_gpu_ctx eigenid_gpu_ctx;

/* Version of this ABI (EIGENID_B200_ABI_VERSION). */
int eigenid_gpu_abi_version(void);
/* Number of visible CUDA devices (0 when none). */
int eigenid_gpu_device_count(void);

/* Context: device buffers and one stream, created once per engine like the
 * reference's worker pool (identity.hpp:95-98, SPEC D5).  Calls on one
 * context are serialised by an internal mutex (thread_pool.hpp:26-28). */
int eigenid_gpu_create(eigenid_gpu_ctx** ctx, int device, eigenid_gpu_err* err);
int eigenid_gpu_destroy(eigenid_gpu_ctx* ctx);
void* eigenid_gpu_stream(eigenid_gpu_ctx* ctx); /* cudaStream_t */
int eigenid_gpu_sync(eigenid_gpu_ctx* ctx, eigenid_gpu_err* err);

/* Multi-GPU context over devices first_device .. first_device+num_gpus-1 of
 * this process (one stream per GPU, one NCCL communicator per GPU from
 * ncclCommInitAll; NCCL is loaded on demand, reusing an already loaded
 * libnccl.so.2).  eigenid_gpu_all_magnitudes on it shards the minor index j
 * over the devices (device d owns rows [d n/P, (d+1) n/P)), recomputes
 * lambda(A) on each, and all-gathers the rows with NCCL before the D2H —
 * the fan-out the reference runs on its thread pool (identity.cpp:303-314).
 * The result is bit-identical for every num_gpus.  Other entry points use
 * the first device. */
int eigenid_gpu_create_multi(eigenid_gpu_ctx** ctx, int first_device, int num_gpus,
                             eigenid_gpu_err* err);
int eigenid_gpu_num_devices(eigenid_gpu_ctx* ctx);
void* eigenid_gpu_device_stream(eigenid_gpu_ctx* ctx, int d); /* cudaStream_t of device d */

/* Device-resident multi-GPU all_magnitudes: d_a[d] is A (n x n) on device
 * d, d_out[d] a full n x n buffer on device d; on return (after
 * eigenid_gpu_sync) every d_out[d] holds the whole matrix (NCCL
 * all-gather of the per-device rows).  Enqueues only. */
int eigenid_gpu_all_magnitudes_multi_device(eigenid_gpu_ctx* ctx, const double* const* d_a,
                                            size_t n, const eigenid_gpu_config* cfg,
                                            double* const* d_out, eigenid_gpu_err* err);

/* ---- host-pointer entry points (reference-facing) ------------------- */

/* Spectrum eigenvalues(const SymmetricMatrix&)   eigensolve.hpp:46,
 * eigensolve.cpp:130-132.  out: n ascending eigenvalues. */
int eigenid_gpu_eigenvalues(eigenid_gpu_ctx* ctx, const double* a, size_t n,
                            double* out, eigenid_gpu_err* err);

/* IdentityEngine::all_magnitudes   identity.hpp:133-135, identity.cpp:294-316.
 * out: n*n, out[j*n+i].  lambda_out (n) / mu_out (n*(n-1)) nullable. */
int eigenid_gpu_all_magnitudes(eigenid_gpu_ctx* ctx, const double* a, size_t n,
                               const eigenid_gpu_config* cfg, double* out,
                               double* lambda_out, double* mu_out,
                               eigenid_gpu_err* err);

/* Batched all_magnitudes over `count` independent n x n matrices stored
 * back to back (a + t*n*n); out + t*n*n.  (SURVEY §8(b) addition, config C2.)
 * On error, err->index is the first failing matrix. */
int eigenid_gpu_all_magnitudes_batched(eigenid_gpu_ctx* ctx, const double* a,
                                       size_t count, size_t n,
                                       const eigenid_gpu_config* cfg,
                                       double* out, eigenid_gpu_err* err);

/* Minor spectra rows j0..j1-1 (and lambda(A)) — the n minor solves of
 * identity.cpp:303-306.  mu: (j1-j0) x (n-1). lambda nullable. */
int eigenid_gpu_minor_spectra(eigenid_gpu_ctx* ctx, const double* a, size_t n,
                              size_t j0, size_t j1, double* lambda, double* mu,
                              eigenid_gpu_err* err);

/* Identity stage only (evaluate(), identity.cpp:185-238) from given spectra,
 * rows j0..j1-1.  mu: (j1-j0) x (n-1); out: (j1-j0) x n.  (config C5.) */
int eigenid_gpu_identity(eigenid_gpu_ctx* ctx, const double* lambda,
                         const double* mu, size_t n, size_t j0, size_t j1,
                         const eigenid_gpu_config* cfg, double* out,
                         eigenid_gpu_err* err);

/* One eigenvector's component magnitudes |v_ij|^2, j = 0..n-1
 * (IdentityEngine::vector_magnitudes, identity.cpp:276-292): n+1 solves.
 * out: n values; out_raw (nullable): pre-clamp values. */
int eigenid_gpu_vector_magnitudes(eigenid_gpu_ctx* ctx, const double* a,
                                  size_t n, size_t i,
                                  const eigenid_gpu_config* cfg, double* out,
                                  double* out_raw, eigenid_gpu_err* err);

/* One component (IdentityEngine::component_magnitude, identity.cpp:240-251;
 * log_domain_magnitude :253-274 when cfg->log_domain).  Cached spectra are
 * used when both lambda (n) and mu_j (n-1) are given (no solves); otherwise
 * lambda(A) and the spectrum of M_j are solved on the device (2 solves).
 * method: 1 batched, 3 log-domain (EvaluationMethod). */
int eigenid_gpu_component_magnitude(eigenid_gpu_ctx* ctx, const double* a,
                                    size_t n, size_t i, size_t j,
                                    const double* lambda, const double* mu_j,
                                    const eigenid_gpu_config* cfg,
                                    double* value, double* raw, int* method,
                                    eigenid_gpu_err* err);

/* MagnitudeResult (identity.hpp:66-74). */
typedef struct eigenid_gpu_magnitude {
  double value;          /* clamped to [0, 1] */
  double raw_value;      /* pre-clamp */
  uint64_t i, j;
  int method;            /* EvaluationMethod: 0 baseline, 1 batched,
                            2 batched-parallel, 3 log-domain */
  double condition_flag; /* min |lambda_i - lambda_k| / range */
} eigenid_gpu_magnitude;

/* The reference's per-component entry points with the full MagnitudeResult:
 *   variant 0  IdentityEngine::component_magnitude   identity.cpp:240-251
 *   variant 1  IdentityEngine::log_domain_magnitude  identity.cpp:253-274
 *   variant 2  component_magnitude_baseline          identity.cpp:151-183
 *              (natural pairing, running products; EIGENID_E_NONFINITE when
 *              a product leaves the finite range; always solves)
 * lambda / mu_j: cached spectra (both or neither; ignored by variant 2). */
int eigenid_gpu_component(eigenid_gpu_ctx* ctx, const double* a, size_t n, size_t i,
                          size_t j, const double* lambda, const double* mu_j,
                          const eigenid_gpu_config* cfg, int variant,
                          eigenid_gpu_magnitude* out, eigenid_gpu_err* err);

/* IdentityEngine::vector_magnitudes (identity.cpp:276-292) with one
 * MagnitudeResult per component j (out: n entries). */
int eigenid_gpu_vector(eigenid_gpu_ctx* ctx, const double* a, size_t n, size_t i,
                       const eigenid_gpu_config* cfg, eigenid_gpu_magnitude* out,
                       eigenid_gpu_err* err);

/* log_domain_product (identity.cpp:98-122) of explicit factor lists
 * (FactorPairing numerator / denominator, len each), on the device. */
int eigenid_gpu_log_domain_product(eigenid_gpu_ctx* ctx, const double* num,
                                   const double* den, size_t len, double* out,
                                   eigenid_gpu_err* err);

/* tridiagonalize (eigensolve.hpp:41): a tridiagonal form orthogonally
 * similar to A from the device reduction (two-stage, not tred1's sequence:
 * same eigenvalues, different (diag, offdiag)).  offdiag: n-1 values. */
int eigenid_gpu_tridiagonalize(eigenid_gpu_ctx* ctx, const double* a, size_t n,
                               double* diag, double* offdiag, eigenid_gpu_err* err);

/* eigenvalues(TridiagonalForm) (eigensolve.cpp:72-128): ascending
 * eigenvalues of the given tridiagonal by Sturm bisection on the device. */
int eigenid_gpu_tridiagonal_eigenvalues(eigenid_gpu_ctx* ctx, const double* diag,
                                        const double* offdiag, size_t n, double* out,
                                        eigenid_gpu_err* err);

/* Sign recovery (recover_signs, signs.cpp:48-120; identity.hpp:159-166):
 * the signed eigenvector i from its squared magnitudes (n_magnitudes must
 * equal n, else EIGENID_E_DIMENSION) and lambda_i.  The largest magnitude is
 * anchored, the other n-1 row equations of (A - lambda_i I) v = 0 are solved
 * on the device (blocked LU with partial pivoting), only their signs are
 * kept, the first component above sign_tol is made positive.  A zero pivot
 * or a residual above 1e-6 ||A||_F is EIGENID_E_SIGN_RECOVERY.  `i` is
 * accepted for interface parity and unused, as in the reference. */
int eigenid_gpu_recover_signs(eigenid_gpu_ctx* ctx, const double* a, size_t n,
                              size_t i, const double* magnitudes,
                              size_t n_magnitudes, double lambda_i,
                              double sign_tol, double* out_v,
                              eigenid_gpu_err* err);

/* Reference-style per-call instrumentation: eigenvalue solves performed by
 * this context (identity.hpp:137-144).  all_magnitudes adds n+1. */
size_t eigenid_gpu_solve_count(eigenid_gpu_ctx* ctx);
void eigenid_gpu_reset_solve_count(eigenid_gpu_ctx* ctx);

/* ---- device-pointer entry points (inputs resident in HBM) ------------ */

/* recover_signs on device-resident A (n x n), magnitudes (n) and d_out (n). */
int eigenid_gpu_recover_signs_device(eigenid_gpu_ctx* ctx, const double* d_a,
                                     size_t n, const double* d_magnitudes,
                                     double lambda_i, double sign_tol,
                                     double* d_out, eigenid_gpu_err* err);

/* Full pipeline for minor rows j0..j1-1 of a device-resident A: computes
 * lambda(A) (redundantly per shard) and the minor spectra, then the identity
 * rows.  d_out: (j1-j0) x n.  d_lambda (n) / d_mu ((j1-j0) x (n-1))
 * nullable.  This is the per-rank shard of the multi-GPU path. */
int eigenid_gpu_all_magnitudes_device(eigenid_gpu_ctx* ctx, const double* d_a,
                                      size_t n, size_t j0, size_t j1,
                                      const eigenid_gpu_config* cfg,
                                      double* d_out, double* d_lambda,
                                      double* d_mu, eigenid_gpu_err* err);

/* Batched small matrices, device pointers. */
int eigenid_gpu_all_magnitudes_batched_device(eigenid_gpu_ctx* ctx,
                                              const double* d_a, size_t count,
                                              size_t n,
                                              const eigenid_gpu_config* cfg,
                                              double* d_out,
                                              eigenid_gpu_err* err);

/* Identity stage, device pointers (rows j0..j1-1; d_mu row r = minor j0+r). */
int eigenid_gpu_identity_device(eigenid_gpu_ctx* ctx, const double* d_lambda,
                                const double* d_mu, size_t n, size_t j0,
                                size_t j1, const eigenid_gpu_config* cfg,
                                double* d_out, eigenid_gpu_err* err);

/* C5 synthetic interlacing spectra generated on the device;
 * bit-identical to oracle's orc_c5_mu_row. d_mu: (j1-j0) x (n-1). */
int eigenid_gpu_c5_mu_device(eigenid_gpu_ctx* ctx, uint64_t seed,
                             const double* d_lambda, size_t n, size_t j0,
                             size_t j1, double* d_mu, eigenid_gpu_err* err);

/* random_symmetric (proj/src/matrix_io.cpp:171-181, host): n*n draws of a
 * seeded mt19937_64 — Box-Muller Gaussian (uniform = 0) or uniform(-1,1)
 * (uniform = 1) — symmetrised as build(kSymmetrize) does; bit-identical to the
 * reference.  The seeded input generator of the benchmark configs. */
void eigenid_random_symmetric(uint64_t seed, size_t n, int uniform,
                              double* out);
/* The raw SeededDraws stream (matrix_io.cpp:44-65): `count` Gaussian
 * (kind 0) or uniform(-1,1) (kind 1) draws. */
void eigenid_seeded_draws(uint64_t seed, size_t count, int kind, double* out);

/* C3 input: Q diag(linspace(-1,1)) Q^T with Q the sign-fixed
 * Householder QR factor of an n x n seeded Gaussian matrix, symmetrised as
 * build(kSymmetrize) does.  Deterministic plain loops (no BLAS): the same
 * bytes on every host. */
void eigenid_c3_matrix(uint64_t seed, size_t n, double* out);

/* Number of kernels this context has launched (instrumentation for the
 * bench's gpu_launches field). */
uint64_t eigenid_gpu_launch_count(eigenid_gpu_ctx* ctx);

/* Per-stage device timing of the large-n pipeline (CUDA events on the
 * context stream): stage1 (dense->band), stage2 (bulge chase), bisection of
 * lambda(A), bisection of the minors, identity.  Off by default. */
void eigenid_gpu_set_profiling(eigenid_gpu_ctx* ctx, int on);
/* Copies up to `cap` stage times (ms) of the last large-n call; returns the
 * count written. */
int eigenid_gpu_stage_times(eigenid_gpu_ctx* ctx, double* ms, int cap);

#ifdef __cplusplus
}
#endif
#endif /* EIGENID_B200_H */
