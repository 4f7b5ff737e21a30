// small.cu — K1s: fused all_magnitudes for n <= 64, one CTA per matrix.
//
// Replaces, for small n, the whole reference pipeline
// IdentityEngine::all_magnitudes (identity.cpp:294-316):
//   * minor_matrix (matrix.cpp:51-68) becomes an index remap on the SMEM copy
//     of A — no (n-1)^2 copy through memory;
//   * each of the n+1 eigenvalue solves (eigensolve.cpp:19-132) is one warp:
//     Householder tridiagonalisation in shared memory (tred1 scheme,
//     eigensolve.cpp:24-61) followed by lane-per-eigenvalue Sturm bisection
//     (replacing QL + sort, :72-128 — the output is ascending by
//     construction);
//   * the identity stage evaluate() (identity.cpp:185-238) runs over the n^2
//     (i, j) pairs of the CTA with the reference's exact pairing / batch /
//     combine order, so identical spectra give bit-identical |v_ij|^2.
// A, lambda and all n minor spectra never leave shared memory; HBM traffic is
// A in (8 n^2 B) and |v|^2 out (8 n^2 B) per matrix.  Config C2 (4096 x n=32)
// runs 4096 CTAs; C1 (n=64) one.
#include "kernels.cuh"

namespace eigenid_b200 {

// Warp-level Householder tridiagonalisation of the m x m symmetric matrix S
// (leading dimension ld, both triangles stored).  Same reflector scheme as
// tred1 (eigensolve.cpp:24-61): rows reduced from the last upward, scale by
// sum |x|, g = -sign(f) sqrt(h).  Outputs diag d[0..m), e2[k] = offdiag_k^2
// and ae[k] = |offdiag_k| for k = 0..m-2.
__device__ void warp_tridiagonalize(double* S, int ld, int m, double* d,
                                    double* e2, double* ae, double* uu,
                                    double* qq) {
  const int lane = threadIdx.x & 31;
  for (int i = m - 1; i >= 1; --i) {
    const int l = i - 1;
    double* row = S + i * ld;
    double ei;
    if (l == 0) {
      ei = row[0];
    } else {
      double sc = 0.0;
      for (int k = lane; k <= l; k += 32) sc += fabs(row[k]);
      sc = warp_sum(sc);
      if (sc == 0.0) {
        ei = row[l];
      } else {
        double h = 0.0;
        for (int k = lane; k <= l; k += 32) {
          const double u = row[k] / sc;
          uu[k] = u;
          h += u * u;
        }
        h = warp_sum(h);
        __syncwarp();
        const double f = uu[l];
        const double g = f >= 0.0 ? -sqrt(h) : sqrt(h);
        ei = sc * g;
        h -= f * g;
        __syncwarp();
        if (lane == 0) uu[l] = f - g;
        __syncwarp();
        // p = S u / h ; K = u.p / 2h ; q = p - K u
        double fp = 0.0;
        for (int j = lane; j <= l; j += 32) {
          const double* sj = S + j * ld;
          double acc = 0.0;
          for (int k = 0; k <= l; ++k) acc += sj[k] * uu[k];
          const double p = acc / h;
          qq[j] = p;
          fp += p * uu[j];
        }
        fp = warp_sum(fp);
        const double hh = fp / (h + h);
        for (int j = lane; j <= l; j += 32) qq[j] -= hh * uu[j];
        __syncwarp();
        // S -= u q^T + q u^T on the leading (l+1) x (l+1) block
        for (int j = lane; j <= l; j += 32) {
          double* sj = S + j * ld;
          const double uj = uu[j], qj = qq[j];
          for (int k = 0; k <= l; ++k) sj[k] -= uj * qq[k] + qj * uu[k];
        }
        __syncwarp();
      }
    }
    if (lane == 0) {
      e2[i - 1] = ei * ei;
      ae[i - 1] = fabs(ei);
    }
    __syncwarp();
  }
  for (int k = lane; k < m; k += 32) d[k] = S[k * ld + k];
  __syncwarp();
}

// All eigenvalues of (d, e2) by lane-per-eigenvalue bisection from the
// Gershgorin interval; writes ascending values to out[0..m).
__device__ void warp_bisect_all(double* d, double* e2, const double* ae, int m,
                                double* out) {
  const int lane = threadIdx.x & 31;
  double lo = 1e308, hi = -1e308, tn = 0.0;
  for (int k = lane; k < m; k += 32) {
    const double r = (k > 0 ? ae[k - 1] : 0.0) + (k + 1 < m ? ae[k] : 0.0);
    lo = fmin(lo, d[k] - r);
    hi = fmax(hi, d[k] + r);
    tn = fmax(tn, fabs(d[k]) + r);
  }
  lo = warp_min(lo);
  hi = warp_max(hi);
  tn = warp_max(tn);
  // exact power-of-two scaling to ||T|| <= 1 for the division-free count
  const double sc = pow2_scale(tn);
  __syncwarp();
  for (int k = lane; k < m; k += 32) {
    d[k] *= sc;
    // (|e| sc)^2, not e^2 sc^2: the same bits for ordinary inputs, and no
    // overflow of e^2 for entries near 1e300 (tred1 scales its rows)
    if (k + 1 < m) e2[k] = (ae[k] * sc) * (ae[k] * sc);
  }
  __syncwarp();
  const double fudge = 2.0 * kEps * tn * m + 1e-300;
  lo = (lo - fudge) * sc;
  hi = (hi + fudge) * sc;
  const double atol = kEps * tn * sc;
  for (int k = lane; k < m; k += 32)
    out[k] = bisect_one(d, e2, m, k, lo, hi, atol) / sc;
  __syncwarp();
  // Bisection results are monotone up to the stopping tolerance; enforce the
  // ascending contract of Spectrum (eigensolve.hpp:10-11) exactly.
  if (lane == 0) {
    for (int k = 1; k < m; ++k) {
      const double v = out[k];
      int t = k - 1;
      while (t >= 0 && out[t] > v) {
        out[t + 1] = out[t];
        --t;
      }
      out[t + 1] = v;
    }
  }
  __syncwarp();
}

// Degeneracy check (identity.cpp:141-149) and the identity stage for one
// matrix whose lambda / mu sit in shared memory (all threads of the CTA).
__device__ void small_identity_phase(const double* lam, const double* mu, int n,
                                     int batch, double tol, int log_domain,
                                     long long mat, double* __restrict__ out,
                                     double* __restrict__ lambda_out,
                                     double* __restrict__ mu_out,
                                     DevStatus* status) {
  __shared__ int degenerate;
  if (threadIdx.x == 0) {
    degenerate = 0;
    const double range = lam[n - 1] - lam[0];
    for (int k = 0; k + 1 < n; ++k)
      if (lam[k + 1] - lam[k] <= tol * range) {
        set_status(status, 2, k, lam[k + 1] - lam[k], mat, 1);
        degenerate = 1;
        break;
      }
  }
  __syncthreads();
  if (degenerate) return;

  if (lambda_out)
    for (int t = threadIdx.x; t < n; t += blockDim.x)
      lambda_out[mat * n + t] = lam[t];
  if (mu_out)
    for (int t = threadIdx.x; t < n * (n - 1); t += blockDim.x)
      mu_out[mat * (long long)n * (n - 1) + t] = mu[t];

  double* og = out + mat * (long long)n * n;
  for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
    const int j = t / n, i = t % n;
    const double* mj = mu + j * (n - 1);
    double raw;
    if (log_domain) {
      const int rc = identity_log_domain(lam, mj, n, i, &raw);
      if (rc) {
        set_status(status, rc, i, 0.0, mat);
        continue;
      }
    } else {
      raw = identity_batched(lam, mj, n, i, batch);
      if (!isfinite(raw)) {
        const int rc = identity_log_domain(lam, mj, n, i, &raw);
        if (rc) {
          set_status(status, rc, i, 0.0, mat);
          continue;
        }
      }
    }
    og[t] = clamp01(raw);
  }
}


__global__ void small_all_magnitudes_kernel(const double* __restrict__ A,
                                            int n, int batch, double tol,
                                            int log_domain,
                                            double* __restrict__ out,
                                            double* __restrict__ lambda_out,
                                            double* __restrict__ mu_out,
                                            DevStatus* status) {
  extern __shared__ double sm[];
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long mat = blockIdx.x;
  const int ldA = n | 1;  // odd leading dimension: conflict-free columns
  double* sA = sm;                       // n x ldA
  double* lam = sA + n * ldA;            // n
  double* mu = lam + n;                  // n x (n-1)
  double* wbase = mu + n * (n - 1);      // per-warp scratch
  const int wsz = n * ldA + 5 * n;
  double* S = wbase + warp * wsz;
  double* d = S + n * ldA;
  double* e2 = d + n;
  double* ae = e2 + n;
  double* uu = ae + n;
  double* qq = uu + n;

  const double* Ag = A + mat * (long long)n * n;
  for (int t = threadIdx.x; t < n * n; t += blockDim.x)
    sA[(t / n) * ldA + (t % n)] = Ag[t];
  __syncthreads();

  // n + 1 solves: s < n is minor M_s, s == n is A itself.
  for (int s = warp; s <= n; s += nw) {
    const int m = (s == n) ? n : n - 1;
    for (int t = lane; t < m * m; t += 32) {
      const int r = t / m, c = t % m;
      const int rr = (s < n && r >= s) ? r + 1 : r;
      const int cc = (s < n && c >= s) ? c + 1 : c;
      S[r * ldA + c] = sA[rr * ldA + cc];
    }
    __syncwarp();
    warp_tridiagonalize(S, ldA, m, d, e2, ae, uu, qq);
    warp_bisect_all(d, e2, ae, m, s == n ? lam : mu + s * (n - 1));
  }
  __syncthreads();

  small_identity_phase(lam, mu, n, batch, tol, log_domain, mat, out, lambda_out,
                       mu_out, status);
}

// Split form for few matrices (C1): the n+1 solves of matrix blockIdx.y are
// spread over gridDim.x CTAs (one warp per solve), spectra go to global
// memory, then small_identity_kernel finishes each matrix.
__global__ void small_solves_kernel(const double* __restrict__ A, int n,
                                    double* __restrict__ lam_g,
                                    double* __restrict__ mu_g) {
  extern __shared__ double sm[];
  const int nw = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long mat = blockIdx.y;
  const int s = blockIdx.x * nw + warp;
  if (s > n) return;
  const int ld = n | 1;
  double* S = sm + warp * (n * ld + 5 * n);
  double* d = S + n * ld;
  double* e2 = d + n;
  double* ae = e2 + n;
  double* uu = ae + n;
  double* qq = uu + n;
  const double* Ag = A + mat * (long long)n * n;
  const int m = (s == n) ? n : n - 1;
  for (int t = lane; t < m * m; t += 32) {
    const int r = t / m, c = t % m;
    const int rr = (s < n && r >= s) ? r + 1 : r;
    const int cc = (s < n && c >= s) ? c + 1 : c;
    S[r * ld + c] = Ag[rr * n + cc];
  }
  __syncwarp();
  warp_tridiagonalize(S, ld, m, d, e2, ae, uu, qq);
  warp_bisect_all(d, e2, ae, m, s == n ? lam_g + mat * n
                                       : mu_g + (mat * n + s) * (long long)(n - 1));
}

__global__ void small_identity_kernel(const double* __restrict__ lam_g,
                                      const double* __restrict__ mu_g, int n,
                                      int batch, double tol, int log_domain,
                                      double* __restrict__ out,
                                      DevStatus* status) {
  extern __shared__ double sm[];
  const long long mat = blockIdx.x;
  double* lam = sm;
  double* mu = sm + n;
  for (int t = threadIdx.x; t < n; t += blockDim.x) lam[t] = lam_g[mat * n + t];
  for (int t = threadIdx.x; t < n * (n - 1); t += blockDim.x)
    mu[t] = mu_g[mat * (long long)n * (n - 1) + t];
  __syncthreads();
  small_identity_phase(lam, mu, n, batch, tol, log_domain, mat, out, nullptr,
                       nullptr, status);
}

size_t small_smem_bytes(int n, int warps) {
  const int ldA = n | 1;
  return sizeof(double) *
         (size_t)(n * ldA + n + n * (n - 1) + warps * (n * ldA + 5 * n));
}

int small_warps_for(int n) { return n <= 16 ? 2 : 4; }

cudaError_t launch_small_split(const double* dA, size_t count, int n,
                               int batch, double tol, int log_domain,
                               double* dout, double* dlam, double* dmu,
                               DevStatus* dstatus, cudaStream_t stream) {
  const int warps = 2;
  const size_t smem1 = sizeof(double) * (size_t)warps * (n * (n | 1) + 5 * n);
  cudaError_t e = cudaFuncSetAttribute(small_solves_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem1);
  if (e != cudaSuccess) return e;
  dim3 g1((n + 1 + warps - 1) / warps, (unsigned)count);
  small_solves_kernel<<<g1, warps * 32, smem1, stream>>>(dA, n, dlam, dmu);
  const size_t smem2 = sizeof(double) * (size_t)(n + n * (n - 1));
  e = cudaFuncSetAttribute(small_identity_kernel,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem2);
  if (e != cudaSuccess) return e;
  small_identity_kernel<<<(unsigned)count, 256, smem2, stream>>>(
      dlam, dmu, n, batch, tol, log_domain, dout, dstatus);
  return cudaGetLastError();
}

cudaError_t launch_small_all(const double* dA, size_t count, int n, int batch,
                             double tol, int log_domain, double* dout,
                             double* dlam, double* dmu, DevStatus* dstatus,
                             cudaStream_t stream) {
  if (count * 4 < 148 && dlam && dmu)  // few matrices: spread the solves
    return launch_small_split(dA, count, n, batch, tol, log_domain, dout, dlam,
                              dmu, dstatus, stream);
  const int warps = small_warps_for(n);
  const size_t smem = small_smem_bytes(n, warps);
  cudaError_t e = cudaFuncSetAttribute(small_all_magnitudes_kernel,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)smem);
  if (e != cudaSuccess) return e;
  small_all_magnitudes_kernel<<<(unsigned)count, warps * 32, smem, stream>>>(
      dA, n, batch, tol, log_domain, dout, dlam, dmu, dstatus);
  return cudaGetLastError();
}

}  // namespace eigenid_b200
