// bulge.cu — K1L stage 2: symmetric band (bandwidth kB) -> tridiagonal by
// Householder bulge chasing.
//
// Second half of the replacement for tridiagonalize (eigensolve.cpp:19-69).
// Sweep st annihilates column st below the subdiagonal with a length-kB
// reflector, then chases the bulge down the band block by block:
//   right-apply the previous reflector to the off-diagonal block C = A[R', R],
//   annihilate C's first column with a new reflector, left-apply it to the
//   rest of C, two-sided apply it to the diagonal block D = A[R', R'].
// Fill left by one sweep is cleaned by the next sweep at the same block
// position, so a step touches only C and D (band storage keeps 2kB+1
// diagonals per column).
//
// Parallel layout: a CTA owns one solve at a time; its 16 warps form 8 warp
// pairs and each pair chases one sweep (pair p takes sweeps p, p+8, ...), so
// 8 consecutive sweeps are in flight: sweep s may run step k once sweep s-1
// has finished step k+1 (k+2 before prefetching step k+1), tracked by
// progress counters in shared memory.  The leading sweep pulls each block
// from HBM and the 7 following sweeps re-read it from L2.  Inside a pair,
// lane = row and warp h owns columns [16h, 16h+16) of the 32 x 32 blocks, so
// every step's row dot products are split across the two warps (combined
// through shared memory under a 64-thread named barrier), halving the
// per-step dependent chain.  The blocks of step k+1 are prefetched while step
// k computes (C into registers, D into a shared-memory double buffer by
// cp.async).  CTAs pull solves from an atomic work counter.
#include "common.cuh"

namespace eigenid_b200 {

constexpr int kCB = 32;              // bandwidth (must match band.cu kB)
constexpr int kCLD = 2 * kCB + 1;    // band diagonals stored per column
constexpr int kPairs = 8;            // sweeps in flight per CTA
constexpr int kWarpsPerCta = 2 * kPairs;
constexpr int kHalf = kCB / 2;       // columns per warp
constexpr int kSLD = kCB + 2;        // even: rows read as double2
constexpr int kBlk = kCB * kSLD;
// per pair: sC, sD[2], v, v2, w, w2, x[2][32], scalars
constexpr int kPairSmem = 3 * kBlk + 4 * kCB + 2 * kCB + 8;

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
};

__device__ __forceinline__ void cpa8(double* smem, const double* gmem, bool ok) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr),
               "l"(gmem), "r"(ok ? 8 : 0));
}
// Branch-free predicated store (the compiler otherwise emits one divergent
// branch per element of the store loops).
__device__ __forceinline__ void st_pred(double* p, double v, bool pred) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f64 [%0], %1;\n}\n" ::"l"(p),
      "d"(v), "r"((int)pred)
      : "memory");
}
__device__ __forceinline__ void cpa_commit2() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void cpa_wait_one() { asm volatile("cp.async.wait_group 1;\n" ::); }

// 64-thread barrier of warp pair p (named barriers 1..8).
__device__ __forceinline__ void pair_sync(int pair) {
  asm volatile("bar.sync %0, 64;\n" ::"r"(pair + 1) : "memory");
}

// Householder from x (lane r holds x_r, r < L), one warp: v (v_0 = 1) -> sv,
// returns tau, *beta (dlarfg convention).
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
  sv[lane] = (lane == 0) ? 1.0 : ((lane < L) ? x * scal : 0.0);
  *beta = b;
  return tau;
}

struct PairSmem {
  double* sC;     // 32 x kSLD: C rows for the left-apply transposition
  double* sD[2];  // 32 x kSLD: D block double buffer
  double* sv;     // previous / current reflector
  double* sv2;    // new reflector
  double* sw;     // left-apply column weights
  double* sw2;    // two-sided w vector
  double* sx;     // [2][32] partial row sums of the two halves
  double* sc;     // scalars: tau, tau2
};

// D <- H D H on the L x L block in sD (both triangles, zero outside L); each
// warp of the pair updates and stores its 16 columns of the lower triangle.
__device__ __forceinline__ void two_sided_pair(const PairSmem& S, double* sD,
                                               const double* sv, double tau,
                                               int L, double* AB, int R,
                                               int pair, int h) {
  const int lane = threadIdx.x & 31;
  double drow[kHalf];
  double pp[2] = {0.0, 0.0};
  const double2* dr2 = reinterpret_cast<const double2*>(sD + lane * kSLD + kHalf * h);
  const double2* v2p = reinterpret_cast<const double2*>(sv + kHalf * h);
#pragma unroll
  for (int c = 0; c < kHalf / 2; ++c) {
    const double2 dd = dr2[c], vv = v2p[c];
    drow[2 * c] = dd.x;
    drow[2 * c + 1] = dd.y;
    pp[0] += dd.x * vv.x;
    pp[1] += dd.y * vv.y;
  }
  S.sx[h * kCB + lane] = pp[0] + pp[1];
  pair_sync(pair);
  const double p = tau * (S.sx[lane] + S.sx[kCB + lane]);
  const double vr = sv[lane];
  const double K = 0.5 * tau * warp_sum(p * vr);
  const double w = p - K * vr;
  if (h == 0) S.sw2[lane] = w;
  pair_sync(pair);
  const double2* w2p = reinterpret_cast<const double2*>(S.sw2 + kHalf * h);
#pragma unroll
  for (int c = 0; c < kHalf / 2; ++c) {
    const double2 ww = w2p[c], vv = v2p[c];
    drow[2 * c] -= vr * ww.x + w * vv.x;
    drow[2 * c + 1] -= vr * ww.y + w * vv.y;
  }
  // lower triangle back to the band: column cg, rows cg..L-1
  double* base = AB + (long long)R * kCLD + lane;
#pragma unroll
  for (int c = 0; c < kHalf; ++c) {
    const int cg = kHalf * h + c;
    st_pred(base + cg * (kCLD - 1), drow[c], lane >= cg && lane < L);
  }
}

// cp.async of this warp's 16 columns of the symmetric L x L block at R.
__device__ __forceinline__ void prefetch_d_half(double* sD, const double* AB,
                                                int R, int L, int h) {
  const int lane = threadIdx.x & 31;
  const double* base = AB + (long long)R * kCLD;
#pragma unroll
  for (int c = 0; c < kHalf; ++c) {
    const int cg = kHalf * h + c;
    const bool ok = lane < L && cg < L;
    const int off = (cg <= lane) ? cg * kCLD + (lane - cg) : lane * kCLD + (cg - lane);
    cpa8(sD + lane * kSLD + cg, ok ? base + off : AB, ok);
  }
  cpa_commit2();
}

// This warp's 16 columns of C = A[R1.., R..] (lane = row).
__device__ __forceinline__ void load_c_half(double (&cr)[kHalf], const double* AB,
                                            int R1, int L1, int R, int L, int h) {
  const int lane = threadIdx.x & 31;
  const double* base = AB + (long long)R * kCLD + (R1 - R) + lane;
#pragma unroll
  for (int c = 0; c < kHalf; ++c) {
    const int cg = kHalf * h + c;
    cr[c] = (lane < L1 && cg < L) ? base[cg * (kCLD - 1)] : 0.0;
  }
}

__device__ __forceinline__ long long spos(int sweep, int step) {
  return (long long)sweep * 65536 + step;
}

// Blocks until sweep s-1 (owned by pair (p-1) mod 8) has finished step k.
__device__ __forceinline__ void wait_prev(volatile long long* prog, int pair,
                                          int s, int k) {
  if (s == 0) return;
  const int pp = (pair + kPairs - 1) % kPairs;
  const long long need = spos(s - 1, k);
  if ((threadIdx.x & 31) == 0)
    while (prog[pp] < need) __nanosleep(64);
  __syncwarp();
  __threadfence_block();
}

// Called by both warps of the pair after their stores of step k.
__device__ __forceinline__ void publish(volatile long long* prog, int pair,
                                        int h, int s, int k) {
  __threadfence_block();
  pair_sync(pair);
  if (h == 0 && (threadIdx.x & 31) == 0) prog[pair] = spos(s, k);
}

__global__ void __launch_bounds__(kWarpsPerCta * 32, 1)
bulge_chase_kernel(Stage2Args a) {
  extern __shared__ double smem[];
  __shared__ long long prog[kPairs];
  __shared__ int s_sidx;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int pair = warp >> 1, h = warp & 1;
  PairSmem S;
  {
    double* b = smem + pair * kPairSmem;
    S.sC = b;
    S.sD[0] = b + kBlk;
    S.sD[1] = b + 2 * kBlk;
    S.sv = b + 3 * kBlk;
    S.sv2 = S.sv + kCB;
    S.sw = S.sv2 + kCB;
    S.sw2 = S.sw + kCB;
    S.sx = S.sw2 + kCB;
    S.sc = S.sx + 2 * kCB;
  }

  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0) s_sidx = atomicAdd(a.counter, 1);
    if (threadIdx.x < kPairs) prog[threadIdx.x] = -1;
    __syncthreads();
    const int sidx = s_sidx;
    if (sidx >= a.nsolves) break;
    const int m = a.js[sidx] < 0 ? a.n : a.n - 1;
    double* AB = a.band + sidx * a.band_stride;

    for (int st = pair; st + 2 < m; st += kPairs) {
      const int R0 = st + 1;
      const int L0 = min(kCB, m - 1 - st);
      int Rk = R0 + kCB;
      bool have = Rk <= m - 1;
      int Lk = have ? min(kCB, m - Rk) : 0;
      // block 0 and the prefetch of step 1 need sweep st-1 past step 2
      wait_prev(prog, pair, st, 2);
      const double x = lane < L0 ? AB[(long long)st * kCLD + 1 + lane] : 0.0;
      prefetch_d_half(S.sD[0], AB, R0, L0, h);
      double ncrow[kHalf];
      if (have) {
        load_c_half(ncrow, AB, Rk, Lk, R0, L0, h);
        prefetch_d_half(S.sD[1], AB, Rk, Lk, h);
      }
      if (h == 0) {
        double beta;
        const double t0 = warp_householder(x, L0, S.sv, &beta);
        if (lane < L0) AB[(long long)st * kCLD + 1 + lane] = (lane == 0) ? beta : 0.0;
        if (lane == 0) S.sc[0] = t0;
      }
      if (have) cpa_wait_one(); else cpa_wait_all();
      pair_sync(pair);  // sv, tau and both halves of D_0 visible
      double tau = S.sc[0];
      two_sided_pair(S, S.sD[0], S.sv, tau, L0, AB, R0, pair, h);
      publish(prog, pair, h, st, 0);
      int R = R0, L = L0, buf = 1, k = 1;
      while (have) {
        // ---- step k on C = A[Rk.., R..] (Lk x L), D = A[Rk.., Rk..]
        double crow[kHalf];
#pragma unroll
        for (int c = 0; c < kHalf; ++c) crow[c] = ncrow[c];
        const int Rn = Rk + kCB;
        const bool haven = Rn <= m - 1;
        const int Ln = haven ? min(kCB, m - Rn) : 0;
        if (haven) {
          wait_prev(prog, pair, st, k + 2);
          load_c_half(ncrow, AB, Rn, Ln, Rk, Lk, h);
          prefetch_d_half(S.sD[buf ^ 1], AB, Rn, Ln, h);
        }
        // right-apply the previous reflector: C -= tau (C v) v^T
        {
          const double2* v2p = reinterpret_cast<const double2*>(S.sv + kHalf * h);
          double yy[2] = {0.0, 0.0};
#pragma unroll
          for (int c = 0; c < kHalf / 2; ++c) {
            const double2 vv = v2p[c];
            yy[0] += crow[2 * c] * vv.x;
            yy[1] += crow[2 * c + 1] * vv.y;
          }
          S.sx[h * kCB + lane] = yy[0] + yy[1];
          pair_sync(pair);
          const double y = tau * (S.sx[lane] + S.sx[kCB + lane]);
#pragma unroll
          for (int c = 0; c < kHalf / 2; ++c) {
            const double2 vv = v2p[c];
            crow[2 * c] -= y * vv.x;
            crow[2 * c + 1] -= y * vv.y;
          }
        }
        // new reflector from C's first column (owned by warp h = 0)
        if (h == 0) {
          double beta2;
          const double t2 = warp_householder(crow[0], Lk, S.sv2, &beta2);
          crow[0] = (lane == 0) ? beta2 : 0.0;
          if (lane == 0) S.sc[1] = t2;
        }
        pair_sync(pair);  // v2 and tau2 visible; sx free again
        const double tau2 = S.sc[1];
        // left-apply to columns 1..L-1 of this warp's half
        {
          double2* cr2 = reinterpret_cast<double2*>(S.sC + lane * kSLD + kHalf * h);
#pragma unroll
          for (int c = 0; c < kHalf / 2; ++c) cr2[c] = make_double2(crow[2 * c], crow[2 * c + 1]);
          __syncwarp();
          const int cl = lane & (kHalf - 1), rh = lane >> 4;
          const int cg = kHalf * h + cl;
          double w = 0.0;
#pragma unroll
          for (int r = 0; r < kHalf; ++r) {
            const int rr = kHalf * rh + r;
            w += S.sv2[rr] * S.sC[rr * kSLD + cg];
          }
          w += __shfl_xor_sync(0xffffffffu, w, 16);
          if (rh == 0) S.sw[cg] = (cg >= 1 && cg < L) ? tau2 * w : 0.0;
          __syncwarp();
          const double vr = S.sv2[lane];
          const double2* w2p = reinterpret_cast<const double2*>(S.sw + kHalf * h);
#pragma unroll
          for (int c = 0; c < kHalf / 2; ++c) {
            const double2 t = w2p[c];
            crow[2 * c] -= vr * t.x;
            crow[2 * c + 1] -= vr * t.y;
          }
        }
        {
          double* base = AB + (long long)R * kCLD + (Rk - R) + lane;
#pragma unroll
          for (int c = 0; c < kHalf; ++c) {
            const int cg = kHalf * h + c;
            st_pred(base + cg * (kCLD - 1), crow[c], lane < Lk && cg < L);
          }
        }
        // two-sided on the diagonal block (prefetched into sD[buf])
        if (haven) cpa_wait_one(); else cpa_wait_all();
        pair_sync(pair);  // both halves of D_k landed
        two_sided_pair(S, S.sD[buf], S.sv2, tau2, Lk, AB, Rk, pair, h);
        if (h == 0) S.sv[lane] = S.sv2[lane];
        publish(prog, pair, h, st, k);
        tau = tau2;
        R = Rk;
        L = Lk;
        Rk = Rn;
        Lk = Ln;
        have = haven;
        buf ^= 1;
        ++k;
      }
      publish(prog, pair, h, st, 65535);  // sweep done
    }
    __syncthreads();
    double* d = a.d + sidx * a.de_stride;
    double* e2 = a.e2 + sidx * a.de_stride;
    double* ae = a.ae + sidx * a.de_stride;
    for (int k = threadIdx.x; k < m; k += blockDim.x) {
      d[k] = AB[(long long)k * kCLD];
      if (k + 1 < m) {
        const double e = AB[(long long)k * kCLD + 1];
        e2[k] = e * e;
        ae[k] = fabs(e);
      }
    }
  }
}

cudaError_t launch_stage2(const Stage2Args& a, cudaStream_t st) {
  const size_t smem = sizeof(double) * kPairSmem * kPairs;
  cudaError_t e = cudaFuncSetAttribute(
      bulge_chase_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  e = cudaMemsetAsync(a.counter, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = a.nsolves < sms ? a.nsolves : sms;
  bulge_chase_kernel<<<grid, kWarpsPerCta * 32, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace eigenid_b200
