// common.cuh — shared device helpers for the eigenid B200 kernels.
//
// Arithmetic that must round exactly like the reference (the identity
// products, identity.cpp:206-225) uses the explicit __d*_rn intrinsics so
// nvcc can never contract it into FMAs.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace eigenid_b200 {

constexpr double kEps = 2.220446049250313080847e-16;   // DBL_EPSILON
constexpr double kSafeMin = 2.2250738585072014e-308;   // DBL_MIN

// Per-solve / per-call device status record (reduced with atomics).
struct DevStatus {
  int code;        // eigenid_status
  int phase;       // 1: lambda(A) degeneracy check (identity.cpp:141-149)
  long long index; // eigenvalue index (degeneracy) / component index
  double gap;
  long long aux;   // matrix index (batched) or output row
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__device__ __forceinline__ double warp_min(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Records the first error of a call (lowest code wins ties deterministically
// enough for reporting; any error aborts the call on the host side).
__device__ __forceinline__ void set_status(DevStatus* st, int code,
                                           long long index, double gap,
                                           long long aux = -1, int phase = 0) {
  if (atomicCAS(&st->code, 0, code) == 0) {
    st->index = index;
    st->gap = gap;
    st->aux = aux;
    st->phase = phase;
  }
}

// Power-of-two scale 2^-e with 2^e >= tn (exact rescaling of T).
__device__ __forceinline__ double pow2_scale(double tn) {
  if (!(tn > 0.0)) return 1.0;
  return scalbn(1.0, -(ilogb(tn) + 1));
}

// Sturm count plus the determinant det(T - x) = p * 2^e of the same
// division-free recurrence (sign(det) = (-1)^count); used for the secant
// (Illinois) acceleration of bisection.
__device__ __forceinline__ bool is_zero_bits(double v) {
  // +-0.0 test on the integer pipe (keeps the FP64 pipe for the recurrence)
  return ((__double2hiint(v) & 0x7fffffff) | __double2loint(v)) == 0;
}

__device__ __forceinline__ int biased_exp(double v) {
  return (__double2hiint(v) >> 20) & 0x7ff;
}

__device__ __forceinline__ int sturm_det(const double* __restrict__ d,
                                         const double* __restrict__ e2, int m,
                                         double x, double* pdet, int* edet) {
  double p0 = 1.0, p1 = d[0] - x;
  if (is_zero_bits(p1)) p1 = -0x1p-900;
  int cnt = __double2hiint(p1) < 0;
  int ex = 0;
  int k = 1;
  for (; k + 4 <= m; k += 4) {
    // Fast path: four steps without the zero fix-up, tracking whether any
    // p came out exactly zero (integer min of the magnitude bits); in that
    // rare case the block is recomputed with the fix-up, so the result is
    // bit-identical to applying it at every step.
    double q0 = p0, q1 = p1;
    int c = cnt;
    unsigned nz = 0xffffffffu;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const double p2 = fma(d[k + u] - x, q1, -e2[k + u - 1] * q0);
      nz = min(nz, (unsigned)((__double2hiint(p2) & 0x7fffffff) | __double2loint(p2)));
      c += (__double2hiint(p2) ^ __double2hiint(q1)) < 0;
      q0 = q1;
      q1 = p2;
    }
    if (nz == 0u) {
      q0 = p0;
      q1 = p1;
      c = cnt;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        double p2 = fma(d[k + u] - x, q1, -e2[k + u - 1] * q0);
        if (is_zero_bits(p2)) p2 = -q1 * 0x1p-900;
        c += (__double2hiint(p2) ^ __double2hiint(q1)) < 0;
        q0 = q1;
        q1 = p2;
      }
    }
    p0 = q0;
    p1 = q1;
    cnt = c;
    // renormalise by a power of two when the larger exponent leaves
    // [2^-256, 2^256] (integer test on the exponent fields)
    const int eb = max(biased_exp(p0), biased_exp(p1));
    if (eb > 1023 + 256 || eb < 1023 - 256) {
      const int sh = eb - 1023;
      const double f = __hiloint2double((1023 - sh) << 20, 0);
      p0 *= f;
      p1 *= f;
      ex += sh;
    }
  }
  for (; k < m; ++k) {
    double p2 = fma(d[k] - x, p1, -e2[k - 1] * p0);
    if (is_zero_bits(p2)) p2 = -p1 * 0x1p-900;
    cnt += (__double2hiint(p2) ^ __double2hiint(p1)) < 0;
    p0 = p1;
    p1 = p2;
  }
  *pdet = p1;
  *edet = ex;
  return cnt;
}

// Sturm count: number of eigenvalues of the symmetric tridiagonal (d, e2)
// strictly below x, division-free form p_k = (d_k - x) p_{k-1} - e2_{k-1}
// p_{k-2}, counting sign changes (Sturm sequence of leading minors).  The
// caller pre-scales (d, e2, x) by an exact power of two so that ||T|| <= 1,
// which bounds growth per step by 3; both p's are renormalised by a power of
// two every 4 steps.  A zero p_k is replaced by -p_{k-1} 2^-900, the p-form
// image of LAPACK dlaebz's q = -pivmin convention.  3 DP ops per step versus
// ~20 for the division of the q-form.
__device__ __forceinline__ int sturm_count(const double* __restrict__ d,
                                           const double* __restrict__ e2,
                                           int m, double x) {
  double pd;
  int ed;
  return sturm_det(d, e2, m, x, &pd, &ed);
}

// Eigenvalue k (0-based, ascending) of the scaled (d, e2) inside [lo, hi)
// with count(lo) <= k < count(hi).  Bisection until the bracket isolates
// eigenvalue k (count(lo) == k, count(hi) == k+1), then Illinois-modified
// regula falsi on det(T - x), which has exactly one sign change there, with
// Brent-style safeguards (bisect when two steps did not halve the bracket;
// trial points at least half a tolerance inside); every trial point still
// updates the bracket by its Sturm count, so the result is the same
// eigenvalue bisection would find.  Stops at
// hi - lo <= max(atol, 2 eps max(|lo|,|hi|)) — the accuracy the
// Householder reduction's backward error (~eps ||T||) supports.
#ifdef EIGENID_BISECT_STATS
static __device__ unsigned long long g_bis_hist[64];  // evaluations per eigenvalue
#endif
__device__ __forceinline__ double bisect_from(const double* __restrict__ d,
                                              const double* __restrict__ e2,
                                              int m, int k, double lo,
                                              double hi, double atol, int clo,
                                              double plo, int elo, int chi,
                                              double phi, int ehi) {
  int side = 0;
  int it = 0;
  double w1 = 0.0, w2 = 0.0;  // bracket widths one and two steps ago
  for (; it < 300; ++it) {
    const double w = hi - lo;
    const double tol = fmax(atol, 2.0 * kEps * fmax(fabs(lo), fabs(hi)));
    if (w <= tol) break;
    double x = lo + 0.5 * w;
    // secant (Illinois) step once eigenvalue k is isolated, unless the last
    // two steps did not halve the bracket; the trial point keeps half a
    // tolerance from both ends, so a converged secant estimate is bracketed
    // within one tolerance by the next one or two evaluations
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
    if (!(x > lo && x < hi)) break;  // interval is a few ulps wide
    double px;
    int ex;
    const int cx = sturm_det(d, e2, m, x, &px, &ex);
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
  }
#ifdef EIGENID_BISECT_STATS
  atomicAdd(&g_bis_hist[it < 63 ? it : 63], 1ull);
#endif
  return lo + 0.5 * (hi - lo);
}

__device__ __forceinline__ double bisect_one(const double* __restrict__ d,
                                             const double* __restrict__ e2,
                                             int m, int k, double lo, double hi,
                                             double atol) {
  double plo, phi;
  int elo, ehi;
  const int clo = sturm_det(d, e2, m, lo, &plo, &elo);
  const int chi = sturm_det(d, e2, m, hi, &phi, &ehi);
  return bisect_from(d, e2, m, k, lo, hi, atol, clo, plo, elo, chi, phi, ehi);
}

// One |v_ij|^2 exactly as evaluate() computes it (identity.cpp:185-238):
// the sorted pairing equals the reversed natural order, so
// sorted index s pairs lambda_i - mu[n-2-s] with lambda_i - lambda[k'],
// k = n-2-s, k' = k + (k >= i); batches of `batch` pairs, ratio num/den per
// batch, product of ratios in batch order.  Returns raw (pre-clamp); the
// caller retries in the log domain when it is not finite.
__device__ __forceinline__ double identity_batched(const double* __restrict__ lam,
                                                   const double* __restrict__ mu,
                                                   int n, int i, int batch) {
  const double li = lam[i];
  double raw = 1.0, num = 1.0, den = 1.0;
  int cnt = 0;
  for (int s = 0; s < n - 1; ++s) {
    const int k = n - 2 - s;
    const int kd = k + (k >= i);
    num = __dmul_rn(num, __dsub_rn(li, mu[k]));
    den = __dmul_rn(den, __dsub_rn(li, lam[kd]));
    if (++cnt == batch || s == n - 2) {
      raw = __dmul_rn(raw, __ddiv_rn(num, den));
      num = 1.0;
      den = 1.0;
      cnt = 0;
    }
  }
  return raw;
}

// log_domain_product over the sorted pairing (identity.cpp:98-122).
// Returns 0 on success, 2 (zero denominator -> DegenerateEigenvalue) or
// 5 (negative square -> InternalInconsistency).
__device__ __forceinline__ int identity_log_domain(const double* __restrict__ lam,
                                                   const double* __restrict__ mu,
                                                   int n, int i, double* out) {
  const double li = lam[i];
  double log_sum = 0.0;
  bool negative = false, zero = false;
  for (int s = 0; s < n - 1; ++s) {
    const double x = __dsub_rn(li, mu[n - 2 - s]);
    if (x == 0.0) {
      zero = true;
    } else {
      log_sum += log(fabs(x));
      if (x < 0.0) negative = !negative;
    }
  }
  for (int s = 0; s < n - 1; ++s) {
    const int k = n - 2 - s;
    const double x = __dsub_rn(li, lam[k + (k >= i)]);
    if (x == 0.0) return 2;
    log_sum -= log(fabs(x));
    if (x < 0.0) negative = !negative;
  }
  if (zero) {
    *out = 0.0;
    return 0;
  }
  if (negative) return 5;
  *out = exp(log_sum);
  return 0;
}

__device__ __forceinline__ double clamp01(double r) {
  return r < 0.0 ? 0.0 : (1.0 < r ? 1.0 : r);  // std::clamp(raw, 0, 1)
}

}  // namespace eigenid_b200
