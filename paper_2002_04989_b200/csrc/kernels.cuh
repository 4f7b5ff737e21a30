// kernels.cuh — launch interfaces of the device stages, shared by the
// kernel files and the pipeline in api.cu (one definition per argument
// struct, so the two sides cannot drift apart).
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>

#include "common.cuh"

namespace eigenid_b200 {

// ---- small.cu: whole pipeline for n <= 64
cudaError_t launch_small_all(const double* dA, size_t count, int n, int batch,
                             double tol, int log_domain, double* dout,
                             double* dlam, double* dmu, DevStatus* dstatus,
                             cudaStream_t stream);

// ---- band.cu: stage 1, dense -> band
struct Stage1Args {
  const double* A;    // n x n row-major
  int n;
  const int* js;      // solve list: js[s] = minor index, -1 = A itself
  int nsolves;
  double* ws;         // per-slot workspace
  long long ws_stride;
  int ldw;            // leading dimension of the slot matrix
  double* band;       // per-solve band, column-major [col][0..2kB]
  long long band_stride;
  int* counter;       // work queue (zeroed before launch unless reset == 0)
  DevStatus* status;  // sticky call status: nonzero code = abort; wait time-outs are recorded here
  int slot0;          // workspace slot of blockIdx.x == 0
  const double* scale;  // [0]: exact power-of-two input scale (nullable = 1)
  // "the main grid is running" flag (nullable): the main launch sets it, a
  // helper launch joins the queue only if it is set — when kernels are
  // serialised (ncu, CUDA_LAUNCH_BLOCKING) the one-CTA helper would
  // otherwise drain the whole queue alone before the main grid starts
  int* running;
  int helper;         // 1: this launch is the helper
};
// Two compiled layouts of the same kernel (band.cu header): wide (16 warps,
// one CTA per SM) and narrow (8 warps, two CTAs per SM).
namespace wide {
cudaError_t launch_stage1(const Stage1Args& a, int grid, cudaStream_t st,
                          bool reset = true);
int stage1_ctas_per_sm();
}  // namespace wide
namespace narrow {
cudaError_t launch_stage1(const Stage1Args& a, int grid, cudaStream_t st,
                          bool reset = true);
int stage1_ctas_per_sm();
}  // namespace narrow
namespace wide8 {
cudaError_t launch_stage1(const Stage1Args& a, int grid, cudaStream_t st,
                          bool reset = true);
int stage1_ctas_per_sm();
}  // namespace wide8
namespace widesp {
cudaError_t launch_stage1(const Stage1Args& a, int grid, cudaStream_t st,
                          bool reset = true);
int stage1_ctas_per_sm();
}  // namespace widesp
int stage1_band_ld();
int stage1_bandwidth();
long long stage1_ws_doubles(int n, int ldw);  // per-slot workspace

// ---- bulge.cu: stage 2, band -> tridiagonal
struct Stage2Args {
  double* band;            // per solve: m columns x kCLD
  long long band_stride;
  const int* js;           // -1 = A itself (m = n), else m = n - 1
  int nsolves;
  int n;
  double* d;               // per solve: m diagonal
  double* e2;              // per solve: m-1 squared off-diagonal
  double* ae;              // per solve: m-1 |off-diagonal|
  long long de_stride;
  int* counter;            // work queue (zeroed before launch)
  DevStatus* status; // sticky call status: nonzero code = abort; wait time-outs are recorded here
  int device;              // for the SM count
  int compact = 0;         // 1: register-capped variant (co-resides with stage 1)
};
cudaError_t launch_stage2(const Stage2Args& a, cudaStream_t st);

// ---- bisect.cu: Sturm bisection of the tridiagonals
struct BisectArgs {
  const double* d;
  const double* e2;
  const double* ae;
  long long de_stride;
  const int* js;
  int nsolves;
  int first_solve;       // solve index of the first CTA (blockIdx.x offset)
  int n;
  const double* lam;     // interlacing brackets (nullptr: Gershgorin only)
  double* out;           // row r = solve first_solve + r ... see out_ld
  long long out_ld;
  int split;             // CTAs per solve (eigenvalue ranges), >= 1
  DevStatus* status;     // ConvergenceFailure; nonzero code on entry = abort
  const double* scale;   // [0] input scale (brackets), [1] its inverse (output); nullable
  int max_it;            // secant/bisection budget per eigenvalue
};
// Exact power-of-two scale of A when max|a_ij| is far outside [2^-400, 2^400]
// (the reference's tred1 scales every row, eigensolve.cpp:28; the blocked
// reduction would overflow its column norms instead).  scale[0] = 2^-e,
// scale[1] = 2^e; both 1 for ordinary inputs, so their results are untouched.
cudaError_t launch_input_scale(const double* dA, long long count, double* dscale,
                               cudaStream_t st, int* launches);
cudaError_t launch_bisect(const BisectArgs& a, int nsolves_here, int mmax,
                          cudaStream_t st, int* launches);

// ---- identity.cu
int identity_nb(int n, int batch);
cudaError_t launch_identity(const double* dlam, const double* dmu, int n,
                            int rows, int batch, double* dden, double* drcp,
                            double* dout, unsigned long long* dflag_count,
                            long long* dflags, long long flag_cap,
                            DevStatus* dstatus, int log_domain, cudaStream_t st,
                            int* launches);
cudaError_t launch_degeneracy(const double* dlam, int n, double tol,
                              DevStatus* dstatus, cudaStream_t st,
                              int* launches);
cudaError_t launch_c5_mu(uint64_t seed, const double* dlam, int n, int j0,
                         int rows, double* dmu, cudaStream_t st, int* launches);
cudaError_t launch_component(const double* dlam, const double* dmu, int n,
                             int i, int batch, double tol, int log_domain,
                             int variant, double* dout4, DevStatus* dstatus,
                             cudaStream_t st, int* launches);
cudaError_t launch_vector(const double* dlam, const double* dmu, int n, int i,
                          int batch, int log_domain, double* draw, double* dmethod,
                          DevStatus* dstatus, cudaStream_t st, int* launches);
cudaError_t launch_log_product(const double* dnum, const double* dden, long long len,
                               double* dout, DevStatus* dstatus, cudaStream_t st,
                               int* launches);
// Tridiagonal helpers (bisect.cu): signed (d, e) of a reduced band, and the
// (d*s, (e*s)^2, |e*s|) the bisection reads from an explicit tridiagonal.
cudaError_t launch_band_tridiag(const double* band, int ldab, int n, double* d,
                                double* e, cudaStream_t st, int* launches);
cudaError_t launch_tridiag_prepare(const double* de, int n, const double* scale,
                                   double* d, double* e2, double* ae, cudaStream_t st,
                                   int* launches);

// ---- recover.cu: sign recovery (signs.cpp:48-120)
struct RecoverState;
long long recover_ws_doubles(int n);
size_t recover_state_bytes();
cudaError_t launch_recover_signs(const double* dA, int n, const double* dmags,
                                 double lambda, double sign_tol, double* dv,
                                 double* dws, RecoverState* st_dev, cudaStream_t s,
                                 int* launches);
// host view of the state the epilogue needs
struct RecoverResult {
  int singular;
  double res2, fro2;
};
cudaError_t recover_result(const RecoverState* st_dev, RecoverResult* out, cudaStream_t s);

}  // namespace eigenid_b200
