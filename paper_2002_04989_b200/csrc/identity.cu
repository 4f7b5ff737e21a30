// identity.cu — K3: the fused identity kernel (product stage of
// all_magnitudes, identity.cpp:308-314 -> evaluate(), :185-238).
//
// For every (i, j) it forms exactly the reference's value: sorted pairing
// (== reversed natural order), batches of B pairs, per batch
// ratio = num/den, raw = product of ratios in batch order, log-domain retry
// when raw is not finite, clamp to [0, 1].  Identical spectra therefore give
// bit-identical output.
//
// B200 mapping:
//  * The denominator product of a batch depends on (i, batch) only, so it is
//    hoisted into a table den[i][b] (plus its correctly rounded reciprocal)
//    built once by den_table_kernel: the inner loop is one DSUB + one DMUL
//    per (i, j, k) triple instead of the reference's 2 DSUB + 2 DMUL.
//  * The per-batch division num/den is a reciprocal multiply with one FMA
//    correction (Markstein), which is correctly rounded whenever the quotient
//    is in the normal range; outside it falls back to __ddiv_rn.
//  * CTA tile: 256 i (lanes, 8 per thread, coalesced stores along i) x 32 j
//    (8 warps x 4 rows); mu for the 32 rows is staged through shared memory
//    in 64-wide k chunks with cp.async double buffering; inside a warp every
//    mu load is a broadcast.
#include "kernels.cuh"

namespace eigenid_b200 {

constexpr int kIdTI = 256;   // i per CTA
constexpr int kIdTJ = 32;    // j per CTA
constexpr int kIdQI = 8;     // i per thread
constexpr int kIdPJ = 4;     // j per thread (per warp)
constexpr int kIdCH = 64;    // k chunk staged in shared memory

// den[i*nb + b] = prod over batch b (sorted order) of (lambda_i - lambda_k'),
// rcp = RN(1/den).  Same multiplication order as identity.cpp:206-213.
__global__ void den_table_kernel(const double* __restrict__ lam, int n,
                                 int batch, int nb, double* __restrict__ den,
                                 double* __restrict__ rcp) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= (long long)n * nb) return;
  const int i = (int)(t / nb), b = (int)(t % nb);
  const double li = lam[i];
  const int s0 = b * batch, s1 = min(s0 + batch, n - 1);
  double dn = 1.0;
  for (int s = s0; s < s1; ++s) {
    const int k = n - 2 - s;
    dn = __dmul_rn(dn, __dsub_rn(li, lam[k + (k >= i)]));
  }
  den[t] = dn;
  rcp[t] = __drcp_rn(dn);
}

// exponent field within [2^-959, 2^960]: an integer test that keeps the
// FP64 pipe free for the products
__device__ __forceinline__ bool mid_range(double v) {
  const unsigned e = ((unsigned)__double2hiint(v) >> 20) & 0x7ffu;
  return e - 64u < 1920u;  // 64 <= e < 1984
}

__device__ __forceinline__ double div_rn_fast(double a, double b, double r) {
  const double q = __dmul_rn(a, r);
  const double res = __fma_rn(-q, b, a);
  const double q2 = __fma_rn(res, r, q);
  if (!(mid_range(q2) && mid_range(a) && mid_range(b))) return __ddiv_rn(a, b);
  return q2;
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(saddr),
               "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() {
  asm volatile("cp.async.commit_group;\n" ::);
}
__device__ __forceinline__ void cp_async_wait_1() {
  asm volatile("cp.async.wait_group 1;\n" ::);
}
__device__ __forceinline__ void cp_async_wait_0() {
  asm volatile("cp.async.wait_group 0;\n" ::);
}

// Stages mu rows [jt, jt+32) for sorted indices s in [s0, s0+64) as
// smu[row][s - s0] = mu_row[n-2-s] (rows past `rows` clamp to the last row;
// s past n-2 is padding and never consumed).
__device__ __forceinline__ void stage_mu(double* smu, const double* mu,
                                         long long ldmu, int rows, int jt,
                                         int n, int s0) {
  for (int t = threadIdx.x; t < kIdTJ * kIdCH; t += blockDim.x) {
    const int r = t / kIdCH, c = t % kIdCH;
    const int row = min(jt + r, rows - 1);
    const int s = min(s0 + c, n - 2);
    cp_async8(smu + r * (kIdCH + 1) + c, mu + row * ldmu + (n - 2 - s));
  }
}

// out row r (= minor j0 + r), column i.  mu row r likewise.  flags collects
// (r, i) pairs whose raw product is not finite, for the log-domain retry.
__global__ void __launch_bounds__(256, 1)
identity_kernel(const double* __restrict__ lam, const double* __restrict__ mu,
                int n, int rows, int batch, int nb,
                const double* __restrict__ den, const double* __restrict__ rcp,
                double* __restrict__ out, unsigned long long* flag_count,
                long long* flags, long long flag_cap, const DevStatus* status) {
  if (*(volatile const int*)&status->code) return;  // the call already failed
  __shared__ double smu[2][kIdTJ * (kIdCH + 1)];
  __shared__ double sden[2][2 * kIdTI];  // den, rcp of the batch ending in a chunk
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int i0 = blockIdx.x * kIdTI, jt = blockIdx.y * kIdTJ;
  const long long ldmu = n - 1;

  double li[kIdQI];
  int ii[kIdQI];
#pragma unroll
  for (int q = 0; q < kIdQI; ++q) {
    ii[q] = i0 + lane + 32 * q;
    li[q] = lam[min(ii[q], n - 1)];
  }
  double acc[kIdQI][kIdPJ], num[kIdQI][kIdPJ];
#pragma unroll
  for (int q = 0; q < kIdQI; ++q)
#pragma unroll
    for (int p = 0; p < kIdPJ; ++p) {
      acc[q][p] = 1.0;
      num[q][p] = 1.0;
    }

  const int total = n - 1;  // number of factor pairs
  const int nchunks = (total + kIdCH - 1) / kIdCH;
  // With batch >= kIdCH at most one full batch ends inside a chunk, plus the
  // short final batch in the last chunk.  The den/rcp rows (this CTA's 256 i)
  // of the LAST batch ending in a chunk are staged with the chunk (cp.async);
  // any other batch ending there (only the one before a short final batch)
  // reads den/rcp from global memory at its end.
  const bool staged_den = batch >= kIdCH;
  // the last batch whose final pair lies in chunk c, or -1
  auto chunk_bend = [&](int c) -> int {
    const int s0 = c * kIdCH, s1 = min(s0 + kIdCH, total);
    if (s1 == total) return (total - 1) / batch;
    const int bend = s1 / batch - 1;
    return (bend < 0 || (bend + 1) * batch - 1 < s0) ? -1 : bend;
  };
  auto stage_den = [&](int c, int buf) {
    if (!staged_den) return;
    const int bend = chunk_bend(c);
    if (bend < 0) return;
    for (int t = threadIdx.x; t < kIdTI; t += blockDim.x) {
      const long long g = (long long)min(i0 + t, n - 1) * nb + bend;
      cp_async8(&sden[buf][t], den + g);
      cp_async8(&sden[buf][kIdTI + t], rcp + g);
    }
  };
  stage_mu(smu[0], mu, ldmu, rows, jt, n, 0);
  stage_den(0, 0);
  cp_async_commit();
  int batch_end = min(batch, total);
  int b = 0;
  for (int c = 0; c < nchunks; ++c) {
    if (c + 1 < nchunks) {
      stage_mu(smu[(c + 1) & 1], mu, ldmu, rows, jt, n, (c + 1) * kIdCH);
      stage_den(c + 1, (c + 1) & 1);
      cp_async_commit();
      cp_async_wait_1();
    } else {
      cp_async_wait_0();
    }
    __syncthreads();
    const double* sm = smu[c & 1] + (warp * kIdPJ) * (kIdCH + 1);
    const int s0 = c * kIdCH, s1 = min(s0 + kIdCH, total);
    const int cb = staged_den ? chunk_bend(c) : -1;
    int s = s0;
    while (s < s1) {
      const int stop = min(s1, batch_end);
      for (; s < stop; ++s) {
        double m[kIdPJ];
#pragma unroll
        for (int p = 0; p < kIdPJ; ++p) m[p] = sm[p * (kIdCH + 1) + (s - s0)];
#pragma unroll
        for (int q = 0; q < kIdQI; ++q)
#pragma unroll
          for (int p = 0; p < kIdPJ; ++p)
            num[q][p] = __dmul_rn(num[q][p], __dsub_rn(li[q], m[p]));
      }
      if (s == batch_end) {
#pragma unroll
        for (int q = 0; q < kIdQI; ++q) {
          double dq, rq;
          if (staged_den && b == cb) {
            dq = sden[c & 1][lane + 32 * q];
            rq = sden[c & 1][kIdTI + lane + 32 * q];
          } else {
            const long long t = (long long)min(ii[q], n - 1) * nb + b;
            dq = den[t];
            rq = rcp[t];
          }
#pragma unroll
          for (int p = 0; p < kIdPJ; ++p) {
            acc[q][p] = __dmul_rn(acc[q][p], div_rn_fast(num[q][p], dq, rq));
            num[q][p] = 1.0;
          }
        }
        ++b;
        batch_end = min(batch_end + batch, total);
      }
    }
    __syncthreads();
  }

#pragma unroll
  for (int p = 0; p < kIdPJ; ++p) {
    const int r = jt + warp * kIdPJ + p;
    if (r >= rows) continue;
    double* orow = out + (long long)r * n;
#pragma unroll
    for (int q = 0; q < kIdQI; ++q) {
      if (ii[q] >= n) continue;
      const double raw = acc[q][p];
      if (isfinite(raw)) {
        orow[ii[q]] = clamp01(raw);
      } else {
        // NaN marks the entry for the retry; past the flag buffer's capacity
        // the retry finds it by scanning the output instead
        orow[ii[q]] = __longlong_as_double(0x7ff8000000000000ll);
        const unsigned long long slot = atomicAdd(flag_count, 1ull);
        if ((long long)slot < flag_cap) flags[slot] = (long long)r * n + ii[q];
      }
    }
  }
}

// Log-domain retry for flagged components (identity.cpp:227-231), and the
// whole stage when IdentityConfig::Evaluation::kLogDomain is selected.
__device__ __forceinline__ void log_domain_fix_one(const double* __restrict__ lam,
                                                   const double* __restrict__ mu,
                                                   int n, long long idx,
                                                   double* __restrict__ out,
                                                   DevStatus* status) {
  const int r = (int)(idx / n), i = (int)(idx % n);
  double v;
  const int rc = identity_log_domain(lam, mu + (long long)r * (n - 1), n, i, &v);
  if (rc)
    set_status(status, rc, i, 0.0, r);
  else
    out[idx] = clamp01(v);
}

// When more components were flagged than the buffer holds (e.g. a matrix
// scaled by 1e6, where every batch product overflows), the whole output is
// scanned for the NaN markers identity_kernel left instead.
__global__ void log_domain_fix_kernel(const double* __restrict__ lam,
                                      const double* __restrict__ mu, int n,
                                      int rows,
                                      const unsigned long long* flag_count,
                                      const long long* flags, long long flag_cap,
                                      double* __restrict__ out,
                                      DevStatus* status) {
  if (*(volatile const int*)&status->code) return;
  const unsigned long long cnt = *flag_count;
  const unsigned long long stride = (unsigned long long)gridDim.x * blockDim.x;
  const unsigned long long t0 =
      blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
  if (cnt > (unsigned long long)flag_cap) {
    const unsigned long long total = (unsigned long long)rows * n;
    for (unsigned long long t = t0; t < total; t += stride)
      if (isnan(out[t])) log_domain_fix_one(lam, mu, n, (long long)t, out, status);
    return;
  }
  for (unsigned long long t = t0; t < cnt; t += stride)
    log_domain_fix_one(lam, mu, n, flags[t], out, status);
}

__global__ void log_domain_all_kernel(const double* __restrict__ lam,
                                      const double* __restrict__ mu, int n,
                                      int rows, double* __restrict__ out,
                                      DevStatus* status) {
  if (*(volatile const int*)&status->code) return;
  const long long total = (long long)rows * n;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
       t < total; t += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(t / n), i = (int)(t % n);
    double v;
    const int rc = identity_log_domain(lam, mu + (long long)r * (n - 1), n, i, &v);
    if (rc)
      set_status(status, rc, i, 0.0, r);
    else
      out[t] = clamp01(v);
  }
}

// check_fully_nondegenerate (identity.cpp:141-149) on the device.
__global__ void degeneracy_kernel(const double* __restrict__ lam, int n,
                                  double tol, DevStatus* status) {
  const double range = lam[n - 1] - lam[0];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k + 1 < n;
       k += gridDim.x * blockDim.x) {
    const double g = lam[k + 1] - lam[k];
    if (g <= tol * range) {
      // lowest k wins, as in the reference's sequential scan
      atomicMin((unsigned long long*)&status[1].index, (unsigned long long)k);
      status[1].code = 2;
    }
  }
}

__global__ void degeneracy_finish_kernel(const double* __restrict__ lam,
                                         DevStatus* status) {
  if (status[1].code == 2 && status[0].code == 0) {
    const long long k = status[1].index;
    status[0].code = 2;
    status[0].phase = 1;
    status[0].index = k;
    status[0].gap = lam[k + 1] - lam[k];
  }
}

// C5 synthetic minor spectra, bit-identical to orc_c5_mu_row.
__device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ULL;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ULL;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebULL;
  return x ^ (x >> 31);
}

__global__ void c5_mu_kernel(uint64_t seed, const double* __restrict__ lam,
                             int n, int j0, int rows, double* __restrict__ mu) {
  const long long total = (long long)rows * (n - 1);
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
       t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long r = t / (n - 1);
    const int k = (int)(t % (n - 1));
    const uint64_t j = (uint64_t)(j0 + r);
    const uint64_t h = splitmix64(seed ^ ((j << 32) ^ (uint64_t)k));
    const double u = __dmul_rn(__dadd_rn((double)(h >> 11), 0.5), 0x1.0p-53);
    const double lo = lam[k], hi = lam[k + 1];
    const double w = __dsub_rn(hi, lo);
    double v = __dadd_rn(lo, __dmul_rn(u, w));
    if (!(v > lo && v < hi)) v = __dmul_rn(0.5, __dadd_rn(lo, hi));
    mu[t] = v;
  }
}

// One component (i, j), the reference's per-component entry points:
//   variant 0: evaluate() (identity.cpp:185-238) — checked_min_gap for i
//              (:189), batched sorted-pairing product with the log-domain
//              retry, or the log domain outright when cfg is kLogDomain;
//   variant 2: component_magnitude_baseline (:151-183) — natural pairing,
//              sequential running products, NonFiniteIntermediate when one
//              leaves the finite range.
// out4 = {value, raw, method (EvaluationMethod), condition_flag}.
__global__ void component_kernel(const double* __restrict__ lam,
                                 const double* __restrict__ mu, int n, int i,
                                 int batch, double tol, int log_domain,
                                 int variant, double* out4, DevStatus* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double min_gap = 1.0 / 0.0;
  for (int k = 0; k < n; ++k)
    if (k != i) min_gap = fmin(min_gap, fabs(lam[i] - lam[k]));
  const double range = lam[n - 1] - lam[0];
  if (min_gap <= tol * range) {
    set_status(status, 2, i, min_gap, -1, 1);
    return;
  }
  double raw;
  int method = 1;
  if (variant == 2) {
    const double li = lam[i];
    double num = 1.0, den = 1.0;
    for (int k = 0; k + 1 < n; ++k) {
      num = __dmul_rn(num, __dsub_rn(li, mu[k]));
      if (!isfinite(num)) { set_status(status, 4, i, 0.0, 1); return; }
    }
    for (int k = 0; k < n; ++k) {
      if (k == i) continue;
      den = __dmul_rn(den, __dsub_rn(li, lam[k]));
      if (!isfinite(den)) { set_status(status, 4, i, 0.0, 2); return; }
    }
    raw = __ddiv_rn(num, den);
    if (!isfinite(raw)) { set_status(status, 4, i, 0.0, 3); return; }
    method = 0;
  } else if (log_domain) {
    const int rc = identity_log_domain(lam, mu, n, i, &raw);
    if (rc) { set_status(status, rc, i, 0.0); return; }
    method = 3;
  } else {
    raw = identity_batched(lam, mu, n, i, batch);
    if (!isfinite(raw)) {
      const int rc = identity_log_domain(lam, mu, n, i, &raw);
      if (rc) { set_status(status, rc, i, 0.0); return; }
      method = 3;
    }
  }
  out4[0] = clamp01(raw);
  out4[1] = raw;
  out4[2] = method;
  out4[3] = min_gap / range;
}

// raw |v_ij|^2 of one eigenvector i for every row j (vector_magnitudes,
// identity.cpp:276-292) and the method each took (1 batched, 3 log-domain).
__global__ void vector_kernel(const double* __restrict__ lam,
                              const double* __restrict__ mu, int n, int i,
                              int batch, int log_domain, double* __restrict__ raw_out,
                              double* __restrict__ method_out, DevStatus* status) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += gridDim.x * blockDim.x) {
    const double* mj = mu + (long long)j * (n - 1);
    double raw = 0.0;
    int method = 1;
    if (!log_domain) raw = identity_batched(lam, mj, n, i, batch);
    if (log_domain || !isfinite(raw)) {
      const int rc = identity_log_domain(lam, mj, n, i, &raw);
      if (rc) set_status(status, rc, i, 0.0, j);
      method = 3;
    }
    raw_out[j] = raw;
    if (method_out) method_out[j] = method;
  }
}

// log_domain_product (identity.cpp:98-122) of explicit factor lists, in list
// order: out = exp(sum ln|num| - sum ln|den|); a zero numerator gives 0, a
// zero denominator DegenerateEigenvalue(gap 0), a negative sign
// InternalInconsistency.
__global__ void log_product_kernel(const double* __restrict__ num,
                                   const double* __restrict__ den, long long len,
                                   double* out, DevStatus* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double log_sum = 0.0;
  bool negative = false, zero = false;
  for (long long k = 0; k < len; ++k) {
    const double x = num[k];
    if (x == 0.0) {
      zero = true;
    } else {
      log_sum += log(fabs(x));
      if (x < 0.0) negative = !negative;
    }
  }
  for (long long k = 0; k < len; ++k) {
    const double x = den[k];
    if (x == 0.0) { set_status(status, 2, -1, 0.0); return; }
    log_sum -= log(fabs(x));
    if (x < 0.0) negative = !negative;
  }
  if (zero) { *out = 0.0; return; }
  if (negative) { set_status(status, 5, -1, 0.0); return; }
  *out = exp(log_sum);
}

cudaError_t launch_component(const double* dlam, const double* dmu, int n,
                             int i, int batch, double tol, int log_domain,
                             int variant, double* dout4, DevStatus* dstatus,
                             cudaStream_t st, int* launches) {
  component_kernel<<<1, 32, 0, st>>>(dlam, dmu, n, i, batch, tol, log_domain,
                                     variant, dout4, dstatus);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_vector(const double* dlam, const double* dmu, int n, int i,
                          int batch, int log_domain, double* draw, double* dmethod,
                          DevStatus* dstatus, cudaStream_t st, int* launches) {
  vector_kernel<<<(n + 127) / 128, 128, 0, st>>>(dlam, dmu, n, i, batch, log_domain,
                                                 draw, dmethod, dstatus);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_log_product(const double* dnum, const double* dden, long long len,
                               double* dout, DevStatus* dstatus, cudaStream_t st,
                               int* launches) {
  log_product_kernel<<<1, 32, 0, st>>>(dnum, dden, len, dout, dstatus);
  ++*launches;
  return cudaGetLastError();
}

// ---- launchers ----------------------------------------------------------

int identity_nb(int n, int batch) { return (n - 1 + batch - 1) / batch; }

cudaError_t launch_identity(const double* dlam, const double* dmu, int n,
                            int rows, int batch, double* dden, double* drcp,
                            double* dout, unsigned long long* dflag_count,
                            long long* dflags, long long flag_cap,
                            DevStatus* dstatus, int log_domain,
                            cudaStream_t st, int* launches) {
  if (rows <= 0) return cudaSuccess;
  if (log_domain) {
    log_domain_all_kernel<<<148 * 8, 256, 0, st>>>(dlam, dmu, n, rows, dout,
                                                   dstatus);
    ++*launches;
    return cudaGetLastError();
  }
  const int nb = identity_nb(n, batch);
  const long long nt = (long long)n * nb;
  den_table_kernel<<<(unsigned)((nt + 255) / 256), 256, 0, st>>>(dlam, n, batch,
                                                                 nb, dden, drcp);
  cudaMemsetAsync(dflag_count, 0, sizeof(unsigned long long), st);
  dim3 grid((n + kIdTI - 1) / kIdTI, (rows + kIdTJ - 1) / kIdTJ);
  identity_kernel<<<grid, 256, 0, st>>>(dlam, dmu, n, rows, batch, nb, dden,
                                        drcp, dout, dflag_count, dflags,
                                        flag_cap, dstatus);
  log_domain_fix_kernel<<<148 * 4, 256, 0, st>>>(dlam, dmu, n, rows, dflag_count,
                                                 dflags, flag_cap, dout, dstatus);
  *launches += 3;
  return cudaGetLastError();
}

cudaError_t launch_degeneracy(const double* dlam, int n, double tol,
                              DevStatus* dstatus, cudaStream_t st,
                              int* launches) {
  degeneracy_kernel<<<(n + 255) / 256, 256, 0, st>>>(dlam, n, tol, dstatus);
  degeneracy_finish_kernel<<<1, 1, 0, st>>>(dlam, dstatus);
  *launches += 2;
  return cudaGetLastError();
}

cudaError_t launch_c5_mu(uint64_t seed, const double* dlam, int n, int j0,
                         int rows, double* dmu, cudaStream_t st,
                         int* launches) {
  c5_mu_kernel<<<148 * 16, 256, 0, st>>>(seed, dlam, n, j0, rows, dmu);
  ++*launches;
  return cudaGetLastError();
}

}  // namespace eigenid_b200
