// bisect.cu — K2: Sturm-count bisection for the tridiagonals of stage 2.
//
// Replaces the implicit-shift QL + std::sort of eigensolve.cpp:72-128.
// Output is ascending by construction (a final check enforces the Spectrum
// contract exactly).  For the minors the bracket of eigenvalue k is the
// interlacing interval [lambda_k(A), lambda_{k+1}(A)] widened by the solver
// error and verified by Sturm counts at both ends; if
// either check fails the Gershgorin interval is used instead.
// One CTA per minor stages (d, e^2) in shared memory (64 KB at m = 4095);
// one thread per eigenvalue, so every Sturm step of a warp is a broadcast
// shared-memory read.
#include "kernels.cuh"

namespace eigenid_b200 {

constexpr int kBisNT = 256;
// Three CTAs per SM (64 KB of (d, e^2) each at m = 4095; <= 85 registers).
// Two eigenvalues in flight per thread (two interleaved Sturm chains) measured
// 29 % slower: the recurrence is issue-bound, not latency-bound.
constexpr int kBisMinBlocks = 3;  // eigenvalues in flight per thread

__device__ double block_reduce_max(double v, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = warp_max(v);
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  double t = red[0];
  for (int w = 1; w < kBisNT / 32; ++w) t = fmax(t, red[w]);
  __syncthreads();
  return t;
}
__device__ double block_reduce_min(double v, double* red) {
  return -block_reduce_max(-v, red);
}

// One eigenvalue's bracketing / secant state machine (see bisect_kernel).
struct BisectLane {
  int k = 0;
  bool active = false, gersh = false, failed = false;
  int failed_k = -1;
  int stage = 0, it = 0, side = 0, clo = 0, chi = 0, elo = 0, ehi = 0;
  double lo = 0.0, hi = 0.0, plo = 0.0, phi = 0.0, w1 = 0.0, w2 = 0.0;

  __device__ __forceinline__ void start(const double* lam, double delta, double glo,
                                        double ghi, double sc, double glo_s,
                                        double ghi_s, double as) {
    stage = 0;
    if (lam) {
      gersh = false;
      lo = fmax(lam[k] * as - delta, glo) * sc;
      hi = fmin(lam[k + 1] * as + delta, ghi) * sc;
    } else {
      gersh = true;
      lo = glo_s;
      hi = ghi_s;
    }
  }
  // Next evaluation point; an eigenvalue that has converged is written out
  // and the slot moves on to k + stride (active is cleared past k1).
  __device__ __forceinline__ double next_x(double atol, double* out, double sc, int stride,
                                           int k1, const double* lam, double delta,
                                           double glo, double ghi, double glo_s,
                                           double ghi_s, double as, double us,
                                           int max_it) {
    double x = 0.0;
    if (stage == 2) {
      bool fin = false;
      const double w = hi - lo;
      const double tol = fmax(atol, 2.0 * kEps * fmax(fabs(lo), fabs(hi)));
      if (w <= tol || it >= max_it) {
        fin = true;
      } else {
        x = lo + 0.5 * w;
        const bool slow = it >= 2 && w > 0.5 * w2;
        if (clo == k && chi == k + 1 && !slow) {
          const int de = ehi - elo;
          double r = phi / plo;
          r = de > 1000 ? -1e300 : (de < -1000 ? -1e-300 : scalbn(r, de));
          const double xs = lo + w / (1.0 - r);
          const double g = 0.5 * tol;
          x = fmin(fmax(xs, lo + g), hi - g);
          if (!(x > lo && x < hi)) x = lo + 0.5 * w;
        } else {
          side = 0;
        }
        w2 = w1;
        w1 = w;
        if (!(x > lo && x < hi)) fin = true;  // a few ulps wide
      }
      if (fin) {
#ifdef EIGENID_BISECT_STATS
        atomicAdd(&g_bis_hist[it < 63 ? it : 63], 1ull);
#endif
        const double v = (lo + 0.5 * (hi - lo)) / sc * us;
        // iteration budget exhausted or a non-finite tridiagonal: the
        // reference's QL raises ConvergenceFailure (eigensolve.cpp:90-93)
        if (((it >= max_it && w > tol) || !isfinite(v)) && !failed) {
          failed = true;
          failed_k = k;
        }
        out[k] = v;
        k += stride;
        active = k < k1;
        if (active) {
          start(lam, delta, glo, ghi, sc, glo_s, ghi_s, as);
          x = lo;
        }
      }
    } else {
      x = stage == 0 ? lo : hi;
    }
    return x;
  }
  __device__ __forceinline__ void update(int cx, double px, int ex, double x, double glo_s,
                                         double ghi_s) {
    if (stage == 0) {
      clo = cx;
      plo = px;
      elo = ex;
      if (!gersh && !(cx <= k && lo < hi)) {
        gersh = true;  // interlacing check failed: Gershgorin bracket
        lo = glo_s;
        hi = ghi_s;
      } else {
        stage = 1;
      }
    } else if (stage == 1) {
      chi = cx;
      phi = px;
      ehi = ex;
      if (!gersh && !(cx > k)) {
        gersh = true;
        lo = glo_s;
        hi = ghi_s;
        stage = 0;
      } else {
        stage = 2;
        it = 0;
        side = 0;
        w1 = w2 = 0.0;
      }
    } else {
      if (cx > k) {
        hi = x;
        phi = px;
        ehi = ex;
        chi = cx;
        if (side == 1) plo *= 0.5;  // Illinois: retained end twice
        side = 1;
      } else {
        lo = x;
        plo = px;
        elo = ex;
        clo = cx;
        if (side == -1) phi *= 0.5;
        side = -1;
      }
      ++it;
    }
  }
};

__global__ void __launch_bounds__(kBisNT, kBisMinBlocks) bisect_kernel(BisectArgs a) {
  extern __shared__ double sm[];
  __shared__ double red[kBisNT / 32];
  __shared__ int unsorted;
  const int solve = a.first_solve + blockIdx.x / a.split;
  const int part = blockIdx.x % a.split;
  if (*(volatile const int*)&a.status->code) return;  // the call already failed
  const int m = a.js[solve] < 0 ? a.n : a.n - 1;
  double* sd = sm;
  double* se2 = sm + m;
  const double* gd = a.d + solve * a.de_stride;
  const double* ge2 = a.e2 + solve * a.de_stride;
  const double* gae = a.ae + solve * a.de_stride;
  double glo = 1e308, ghi = -1e308, tn = 0.0;
  for (int k = threadIdx.x; k < m; k += kBisNT) {
    const double dk = gd[k];
    sd[k] = dk;
    if (k + 1 < m) se2[k] = ge2[k];
    const double r = (k > 0 ? gae[k - 1] : 0.0) + (k + 1 < m ? gae[k] : 0.0);
    glo = fmin(glo, dk - r);
    ghi = fmax(ghi, dk + r);
    tn = fmax(tn, fabs(dk) + r);
  }
  glo = block_reduce_min(glo, red);
  ghi = block_reduce_max(ghi, red);
  tn = block_reduce_max(tn, red);
  // exact power-of-two scaling to ||T|| <= 1 for the division-free count
  const double sc = pow2_scale(tn);
  for (int k = threadIdx.x; k < m; k += kBisNT) {
    sd[k] *= sc;
    if (k + 1 < m) se2[k] *= sc * sc;
  }
  __syncthreads();
  const double fudge = 2.0 * kEps * tn * m + 1e-300;
  glo -= fudge;
  ghi += fudge;
  const double atol = kEps * tn * sc;
  const double delta = 8.0 * (m + 1) * kEps * tn;
  double* out = a.out + (long long)(solve - a.first_solve) * a.out_ld;
  const int per = (m + a.split - 1) / a.split;
  const int k0 = part * per, k1 = min(m, k0 + per);
  // Each thread owns eigenvalues k = k0 + tid, + kBisNT, ... and runs them as
  // a state machine (BisectLane), one Sturm evaluation per round: bracket low
  // end, high end, then safeguarded secant/bisection (the arithmetic of
  // bisect_from).  A lane whose eigenvalue converges starts its next one in the
  // same round, so the warp's rounds follow the mean, not the maximum,
  // evaluation count.  The interlacing bracket (minors) is verified by the
  // counts at both ends; if either check fails the lane restarts on the
  // Gershgorin interval.
  const double glo_s = glo * sc, ghi_s = ghi * sc;
  const double as = a.scale ? a.scale[0] : 1.0, us = a.scale ? a.scale[1] : 1.0;
  BisectLane ln;
  ln.k = k0 + threadIdx.x;
  ln.active = ln.k < k1;
  if (ln.active) ln.start(a.lam, delta, glo, ghi, sc, glo_s, ghi_s, as);
  while (__any_sync(0xffffffffu, ln.active)) {
    double x = 0.0;
    if (ln.active)
      x = ln.next_x(atol, out, sc, kBisNT, k1, a.lam, delta, glo, ghi, glo_s, ghi_s, as,
                    us, a.max_it);
    if (ln.active) {
      double px;
      int ex;
      const int cx = sturm_det(sd, se2, m, x, &px, &ex);
      ln.update(cx, px, ex, x, glo_s, ghi_s);
    }
  }
  if (ln.failed) set_status(a.status, 3, ln.failed_k, 0.0, solve);
  if (a.split > 1) return;  // cross-CTA order is checked by sort_fix_kernel
  __syncthreads();
  if (threadIdx.x == 0) unsorted = 0;
  __syncthreads();
  for (int k = threadIdx.x; k + 1 < m; k += kBisNT)
    if (out[k + 1] < out[k]) unsorted = 1;
  __syncthreads();
  if (unsorted && threadIdx.x == 0) {
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
}

// Enforces ascending order of one spectrum written by a split bisection.
__global__ void sort_fix_kernel(double* out, int m) {
  __shared__ int unsorted;
  if (threadIdx.x == 0) unsorted = 0;
  __syncthreads();
  for (int k = threadIdx.x; k + 1 < m; k += blockDim.x)
    if (out[k + 1] < out[k]) unsorted = 1;
  __syncthreads();
  if (unsorted && threadIdx.x == 0) {
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
}

// max|a| -> exact power-of-two scale (see kernels.cuh)
__global__ void input_maxabs_kernel(const double* __restrict__ a, long long count,
                                    unsigned long long* maxbits) {
  double m = 0.0;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < count;
       t += (long long)gridDim.x * blockDim.x)
    m = fmax(m, fabs(a[t]));
  m = warp_max(m);
  // non-negative doubles order like their bit patterns
  if ((threadIdx.x & 31) == 0) atomicMax(maxbits, (unsigned long long)__double_as_longlong(m));
}
__global__ void input_scale_kernel(const unsigned long long* maxbits, double* scale) {
  const double m = __longlong_as_double((long long)*maxbits);
  double s = 1.0, u = 1.0;
  if (m > 0x1p400 || (m > 0.0 && m < 0x1p-400)) {
    const int e = ilogb(m);
    s = scalbn(1.0, -e);
    u = scalbn(1.0, e);
  }
  scale[0] = s;
  scale[1] = u;
}

cudaError_t launch_input_scale(const double* dA, long long count, double* dscale,
                               cudaStream_t st, int* launches) {
  auto* bits = reinterpret_cast<unsigned long long*>(dscale + 2);
  cudaError_t e = cudaMemsetAsync(bits, 0, sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  long long blocks = (count + 255) / 256;
  if (blocks > 2048) blocks = 2048;
  input_maxabs_kernel<<<(unsigned)blocks, 256, 0, st>>>(dA, count, bits);
  input_scale_kernel<<<1, 1, 0, st>>>(bits, dscale);
  *launches += 2;
  return cudaGetLastError();
}

// Signed tridiagonal of a band after the chase: d_k = AB[k][0], e_k = AB[k][1].
__global__ void band_tridiag_kernel(const double* __restrict__ band, int ldab, int n,
                                    double* d, double* e) {
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    d[k] = band[(long long)k * ldab];
    if (k + 1 < n) e[k] = band[(long long)k * ldab + 1];
  }
}
cudaError_t launch_band_tridiag(const double* band, int ldab, int n, double* d,
                                double* e, cudaStream_t st, int* launches) {
  band_tridiag_kernel<<<(n + 255) / 256, 256, 0, st>>>(band, ldab, n, d, e);
  ++*launches;
  return cudaGetLastError();
}

// de = [d (n) | e (n-1)] -> d*s, (|e| s)^2, |e| s with the exact input scale.
__global__ void tridiag_prepare_kernel(const double* __restrict__ de, int n,
                                       const double* scale, double* d, double* e2,
                                       double* ae) {
  const double s = scale[0];
  for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
    d[k] = de[k] * s;
    if (k + 1 < n) {
      const double a = fabs(de[n + k]) * s;
      ae[k] = a;
      e2[k] = a * a;
    }
  }
}
cudaError_t launch_tridiag_prepare(const double* de, int n, const double* scale,
                                   double* d, double* e2, double* ae, cudaStream_t st,
                                   int* launches) {
  tridiag_prepare_kernel<<<(n + 255) / 256, 256, 0, st>>>(de, n, scale, d, e2, ae);
  ++*launches;
  return cudaGetLastError();
}

cudaError_t launch_bisect(const BisectArgs& a, int nsolves_here, int mmax,
                          cudaStream_t st, int* launches) {
  const size_t smem = sizeof(double) * 2 * (size_t)mmax;
  cudaError_t e = cudaFuncSetAttribute(
      bisect_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  bisect_kernel<<<nsolves_here * a.split, kBisNT, smem, st>>>(a);
  ++*launches;
  if (a.split > 1) {
    for (int s = 0; s < nsolves_here; ++s) {
      sort_fix_kernel<<<1, 256, 0, st>>>(a.out + s * a.out_ld, mmax);
      ++*launches;
    }
  }
  return cudaGetLastError();
}

#ifdef EIGENID_BISECT_STATS
extern "C" void eigenid_debug_bisect_hist(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_bis_hist, sizeof(g_bis_hist));
}
#endif

}  // namespace eigenid_b200
