// bulge.cu — K1L stage 2: symmetric band (bandwidth kB) -> tridiagonal by
// Householder bulge chasing, one warp per solve.
//
// Second half of the replacement for tridiagonalize (eigensolve.cpp:19-69).
// Sweep st annihilates column st below the subdiagonal with a length-kB
// reflector, then chases the bulge down the band block by block:
//   right-apply the previous reflector to the off-diagonal block
//   A[R', R], annihilate that block's first column with a new reflector,
//   left-apply it to the rest of the block, two-sided apply it to the
//   diagonal block A[R', R'].
// Fill from one sweep is cleaned by the next sweep at the same block
// position, so every step touches only two kB x kB blocks (band storage keeps
// 2kB+1 diagonals per column).  Each step stages the blocks in the warp's
// shared-memory slice; lanes own rows.
#include "common.cuh"

namespace eigenid_b200 {

constexpr int kCB = 32;              // bandwidth (must match band.cu kB)
constexpr int kCLD = 2 * kCB + 1;    // band diagonals stored per column
constexpr int kWarpsPerCta = 4;
constexpr int kSLD = kCB + 1;
constexpr int kWarpSmem = 2 * kCB * kSLD + 4 * kCB;

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
};

// Householder from x (lane r holds x_r, r < L); returns tau, writes v (v_0=1)
// to sv, beta to *beta.
__device__ __forceinline__ double warp_householder(double x, int L, double* sv,
                                                   double* beta) {
  const int lane = threadIdx.x & 31;
  const double alpha = __shfl_sync(0xffffffffu, x, 0);
  const double sig = warp_sum((lane >= 1 && lane < L) ? x * x : 0.0);
  double tau, b, scal;
  if (sig == 0.0) {
    tau = 0.0;
    b = alpha;
    scal = 0.0;
  } else {
    b = -copysign(sqrt(alpha * alpha + sig), alpha);
    tau = (b - alpha) / b;
    scal = 1.0 / (alpha - b);
  }
  if (lane < kCB) sv[lane] = (lane == 0) ? 1.0 : ((lane < L) ? x * scal : 0.0);
  __syncwarp();
  *beta = b;
  return tau;
}

// D (L x L, full symmetric in sD) <- H D H, H = I - tau v v^T.
__device__ __forceinline__ void warp_two_sided(double* sD, int L,
                                               const double* sv, double tau,
                                               double* sw) {
  const int lane = threadIdx.x & 31;
  double p = 0.0;
  if (lane < L) {
    const double* row = sD + lane * kSLD;
    for (int c = 0; c < L; ++c) p += row[c] * sv[c];
    p *= tau;
  }
  const double K = 0.5 * tau * warp_sum(lane < L ? p * sv[lane] : 0.0);
  const double w = p - K * (lane < L ? sv[lane] : 0.0);
  sw[lane] = w;
  __syncwarp();
  if (lane < L) {
    double* row = sD + lane * kSLD;
    const double vr = sv[lane];
    for (int c = 0; c < L; ++c) row[c] -= vr * sw[c] + w * sv[c];
  }
  __syncwarp();
}

__global__ void __launch_bounds__(kWarpsPerCta * 32)
bulge_chase_kernel(Stage2Args a) {
  extern __shared__ double smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int sidx = blockIdx.x * kWarpsPerCta + warp;
  if (sidx >= a.nsolves) return;
  double* sC = smem + warp * kWarpSmem;
  double* sD = sC + kCB * kSLD;
  double* sv = sD + kCB * kSLD;
  double* sv2 = sv + kCB;
  double* sw = sv2 + kCB;
  const int m = a.js[sidx] < 0 ? a.n : a.n - 1;
  double* AB = a.band + sidx * a.band_stride;
  auto at = [&](int r, int c) -> double& {  // r >= c, r - c <= 2kB
    return AB[(long long)c * kCLD + (r - c)];
  };

  for (int st = 0; st + 2 < m; ++st) {
    // ---- block 0: annihilate column st below the subdiagonal
    int R = st + 1;
    int L = min(kCB, m - 1 - st);
    double beta;
    const double x = lane < L ? at(st + 1 + lane, st) : 0.0;
    double tau = warp_householder(x, L, sv, &beta);
    if (lane < L) at(st + 1 + lane, st) = (lane == 0) ? beta : 0.0;
    // diagonal block D = A[R.., R..]
    for (int c = 0; c < L; ++c)
      if (lane >= c && lane < L) {
        const double v = at(R + lane, R + c);
        sD[lane * kSLD + c] = v;
        sD[c * kSLD + lane] = v;
      }
    __syncwarp();
    warp_two_sided(sD, L, sv, tau, sw);
    for (int c = 0; c < L; ++c)
      if (lane >= c && lane < L) at(R + lane, R + c) = sD[lane * kSLD + c];
    __syncwarp();
    // ---- chase
    while (true) {
      const int R1 = R + kCB;
      if (R1 > m - 1) break;
      const int L1 = min(kCB, m - R1);
      // C = A[R1.., R..] (L1 x L); lane = row
      double crow[kCB];
#pragma unroll
      for (int c = 0; c < kCB; ++c)
        crow[c] = (lane < L1 && c < L) ? at(R1 + lane, R + c) : 0.0;
      // right apply previous H: C -= tau (C v) v^T
      double y = 0.0;
#pragma unroll
      for (int c = 0; c < kCB; ++c) y += crow[c] * sv[c];
      y *= tau;
#pragma unroll
      for (int c = 0; c < kCB; ++c) crow[c] -= y * sv[c];
      // new reflector from column 0
      double beta2;
      const double tau2 = warp_householder(crow[0], L1, sv2, &beta2);
      crow[0] = (lane == 0) ? beta2 : 0.0;
      // left apply to columns 1..: w_c = sum_r v2_r C[r][c]
      if (lane < kCB) {
#pragma unroll
        for (int c = 0; c < kCB; ++c) sC[lane * kSLD + c] = crow[c];
      }
      __syncwarp();
      {
        double w = 0.0;
        if (lane >= 1 && lane < L)
          for (int r = 0; r < L1; ++r) w += sv2[r] * sC[r * kSLD + lane];
        sw[lane] = tau2 * w;
      }
      __syncwarp();
      if (lane < L1) {
        const double vr = sv2[lane];
#pragma unroll
        for (int c = 1; c < kCB; ++c) crow[c] -= vr * sw[c];
      }
#pragma unroll
      for (int c = 0; c < kCB; ++c)
        if (lane < L1 && c < L) at(R1 + lane, R + c) = crow[c];
      __syncwarp();
      // two-sided on the next diagonal block
      for (int c = 0; c < L1; ++c)
        if (lane >= c && lane < L1) {
          const double v = at(R1 + lane, R1 + c);
          sD[lane * kSLD + c] = v;
          sD[c * kSLD + lane] = v;
        }
      __syncwarp();
      warp_two_sided(sD, L1, sv2, tau2, sw);
      for (int c = 0; c < L1; ++c)
        if (lane >= c && lane < L1) at(R1 + lane, R1 + c) = sD[lane * kSLD + c];
      __syncwarp();
      if (lane < kCB) sv[lane] = sv2[lane];
      __syncwarp();
      tau = tau2;
      R = R1;
      L = L1;
    }
  }
  double* d = a.d + sidx * a.de_stride;
  double* e2 = a.e2 + sidx * a.de_stride;
  double* ae = a.ae + sidx * a.de_stride;
  for (int k = lane; k < m; k += 32) {
    d[k] = at(k, k);
    if (k + 1 < m) {
      const double e = at(k + 1, k);
      e2[k] = e * e;
      ae[k] = fabs(e);
    }
  }
}

cudaError_t launch_stage2(const Stage2Args& a, cudaStream_t st) {
  const size_t smem = sizeof(double) * kWarpSmem * kWarpsPerCta;
  cudaError_t e = cudaFuncSetAttribute(
      bulge_chase_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int grid = (a.nsolves + kWarpsPerCta - 1) / kWarpsPerCta;
  bulge_chase_kernel<<<grid, kWarpsPerCta * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace eigenid_b200
