// bulge.cu — K1L stage 2: symmetric band (bandwidth kB) -> tridiagonal by
// Householder bulge chasing, one warp per solve.
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
// A CTA owns one solve at a time and its warps (nine) chase as many
// consecutive sweeps concurrently (warp w takes sweeps w, w + 9, ...): sweep
// s may run step k once sweep s-1 has finished step k+1 (k+2 before
// prefetching step k+1), tracked by per-warp progress counters in shared
// memory.  The leading sweep pulls each block from HBM and the following
// sweeps re-read it from L2/L1, so band traffic to HBM drops ~9x versus
// independent solves per warp.  One
// CTA per SM: the followers' re-reads need a large L1, so shared memory is
// kept to 13.4 KB per warp (two CTAs per SM — 16 warps at <= 128 registers —
// measured 2.1x slower: the L1 shrinks to ~30 KB and the re-reads go to L2).
// Within a sweep a step never reads what the previous step wrote, so the
// blocks of step k+1 are prefetched by cp.async while step k computes: C into
// sC once step k has taken its column sums from it, the packed lower
// triangle of D into sD once step k's two-sided update has read D into
// registers.  The left-apply's column sums come from the staged (not yet
// right-applied) C: C1^T v2 = C^T v2 - (y . v2) v1 for C1 = C - y v1^T.
#include "kernels.cuh"

#include <cstdlib>

namespace eigenid_b200 {

constexpr int kCB = 32;              // bandwidth (must match band.cu kB)
constexpr int kCLD = 2 * kCB + 1;    // band diagonals stored per column
// Warps (= sweeps in flight per solve) per CTA, by matrix size: nine for
// long sweeps (one SM sub-partition then holds three warps, so the register
// cap is 168 with small spills, and it still measured 1.1 % faster than
// eight at n = 4096), eight below (nine is 6 % slower at n = 1024); ten or
// more are slower everywhere.
constexpr int kWarpsLong = 9, kWarpsShort = 8;
constexpr int kWarpsLongMinN = 3072;
constexpr int kSLD = kCB + 1;
constexpr int kBlk = kCB * kSLD;
constexpr int kDP = kCB * (kCB + 1) / 2;        // packed lower triangle of D
constexpr int kWarpSmem = kBlk + kDP + 3 * kCB;  // sC, sD, v, v2, w
#ifndef EIGENID_BULGE_CTAS
#define EIGENID_BULGE_CTAS 1
#endif
constexpr int kBulgeCtasPerSm = EIGENID_BULGE_CTAS;

// Row-packed lower triangle: (r, c), r >= c.
__device__ __forceinline__ int dp(int r, int c) { return (r * (r + 1) >> 1) + c; }

__device__ __forceinline__ void cpa8(double* smem, const double* gmem, bool ok) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(saddr),
               "l"(gmem), "r"(ok ? 8 : 0));
}
// Branch-free predicated store (the compiler otherwise emits one divergent
// branch per element of the 32-iteration store loops).
__device__ __forceinline__ void st_pred(double* p, double v, bool pred) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q st.global.f64 [%0], %1;\n}\n" ::"l"(p),
      "d"(v), "r"((int)pred)
      : "memory");
}

__device__ __forceinline__ void cpa_commit2() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cpa_wait_all() { asm volatile("cp.async.wait_group 0;\n" ::); }
__device__ __forceinline__ void cpa_wait_one() { asm volatile("cp.async.wait_group 1;\n" ::); }
// Full-block (L = kCB) variants with immediate address offsets: element c of
// a column run lives kCLD-1 doubles further on, so every load/store is one
// instruction off a single base register (no per-element address or
// predicate arithmetic beyond the triangle test).
template <int C>
__device__ __forceinline__ void st_tri_full(double* base, const double (&v)[kCB], int lane) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ge.s32 q, %2, %3;\n @q st.global.f64 [%0+%4], %1;\n}\n" ::"l"(base),
      "d"(v[C]), "r"(lane), "n"(C), "n"(C * (kCLD - 1) * 8)
      : "memory");
  if constexpr (C + 1 < kCB) st_tri_full<C + 1>(base, v, lane);
}
template <int C>
__device__ __forceinline__ void st_full(double* base, const double (&v)[kCB]) {
  asm volatile("st.global.f64 [%0+%2], %1;\n" ::"l"(base), "d"(v[C]), "n"(C * (kCLD - 1) * 8)
               : "memory");
  if constexpr (C + 1 < kCB) st_full<C + 1>(base, v);
}
template <int C>
__device__ __forceinline__ void cpa_tri_full(unsigned sbase, const double* gbase, int lane) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ge.s32 q, %2, %3;\n @q cp.async.ca.shared.global [%0+%4], [%1+%5], 8;\n}\n" ::"r"(
          sbase),
      "l"(gbase), "r"(lane), "n"(C), "n"(C * 8), "n"(C * (kCLD - 1) * 8));
  if constexpr (C + 1 < kCB) cpa_tri_full<C + 1>(sbase, gbase, lane);
}
template <int C>
__device__ __forceinline__ void cpa_full(unsigned sbase, const double* gbase) {
  asm volatile("cp.async.ca.shared.global [%0+%2], [%1+%3], 8;\n" ::"r"(sbase), "l"(gbase),
               "n"(C * 8), "n"(C * (kCLD - 1) * 8));
  if constexpr (C + 1 < kCB) cpa_full<C + 1>(sbase, gbase);
}


// Householder from x (lane r holds x_r, r < L): v (v_0 = 1) -> sv, returns
// tau, *beta.  dlarfg convention.
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
  __syncwarp();
  *beta = b;
  return tau;
}

__device__ __forceinline__ void prefetch_d(double* sD, const double* AB, int R,
                                           int L) {
  // lower triangle of the L x L block: element (r, c), r >= c, lives at
  // column c, diagonal r - c of the band (one coalesced run per column);
  // out-of-range entries are zero-filled
  const int lane = threadIdx.x & 31;
  const double* base = AB + (long long)R * kCLD + lane;
  if (L == kCB) {
    cpa_tri_full<0>((unsigned)__cvta_generic_to_shared(sD + dp(lane, 0)), base, lane);
    cpa_commit2();
    return;
  }
#pragma unroll
  for (int c = 0; c < kCB; ++c) {
    if (lane >= c) {
      const bool ok = lane < L;
      cpa8(sD + dp(lane, c), ok ? base + c * (kCLD - 1) : AB, ok);
    }
  }
  cpa_commit2();
}

// D <- H D H on the L x L diagonal block whose lower triangle is held in sD
// (filled by cp.async; rows/cols >= L are zero; the upper triangle is read
// through the mirror).  Writes the lower triangle back to the band.  Once D
// is in registers, the next step's diagonal block (rows/cols nR.., nL of
// them; nL = 0: none) is prefetched into the same buffer.
template <bool FULL>
__device__ __forceinline__ void two_sided_store(double* sD, const double* sv,
                                                double tau, double* sw, int L,
                                                double* AB, int R, int nR, int nL) {
  const int lane = threadIdx.x & 31;
  double drow[kCB];
  double pp[4] = {0.0, 0.0, 0.0, 0.0};
  const double2* v2 = reinterpret_cast<const double2*>(sv);
#pragma unroll
  for (int c = 0; c < kCB; ++c) drow[c] = sD[c <= lane ? dp(lane, c) : dp(c, lane)];
  if (nL > 0) {
    __syncwarp();  // every lane has read its D row
    prefetch_d(sD, AB, nR, nL);
  }
#pragma unroll
  for (int h = 0; h < kCB / 2; ++h) {  // broadcast reads, two per LDS.128
    const double2 v = v2[h];
    pp[(2 * h) & 3] += drow[2 * h] * v.x;
    pp[(2 * h + 1) & 3] += drow[2 * h + 1] * v.y;
  }
  double p = (pp[0] + pp[1]) + (pp[2] + pp[3]);
  p *= tau;
  const double vr = sv[lane];
  const double K = 0.5 * tau * warp_sum(p * vr);
  const double w = p - K * vr;
  sw[lane] = w;
  __syncwarp();
  const double2* w2 = reinterpret_cast<const double2*>(sw);
#pragma unroll
  for (int h = 0; h < kCB / 2; ++h) {
    const double2 a = w2[h], v = v2[h];
    drow[2 * h] -= vr * a.x + w * v.x;
    drow[2 * h + 1] -= vr * a.y + w * v.y;
  }
  // lower triangle back to the band: column c, rows c..L-1 (coalesced in r)
  double* base = AB + (long long)R * kCLD + lane;
  if constexpr (FULL) {
    st_tri_full<0>(base, drow, lane);
  } else {
#pragma unroll
    for (int c = 0; c < kCB; ++c)
      st_pred(base + c * (kCLD - 1), drow[c], lane >= c && lane < L);
  }
  __syncwarp();
}

// C = A[R1.., R..] (L1 x L) into sC (row r = lane, padded rows); one
// coalesced run per column, out-of-range entries zero-filled.
__device__ __forceinline__ void prefetch_c(double* sC, const double* AB, int R1,
                                           int L1, int R, int L) {
  const int lane = threadIdx.x & 31;
  const double* base = AB + (long long)R * kCLD + (R1 - R) + lane;
  if (L1 == kCB && L == kCB) {
    cpa_full<0>((unsigned)__cvta_generic_to_shared(sC + lane * kSLD), base);
    cpa_commit2();
    return;
  }
#pragma unroll
  for (int c = 0; c < kCB; ++c) {
    const bool ok = lane < L1 && c < L;
    cpa8(sC + lane * kSLD + c, ok ? base + c * (kCLD - 1) : AB, ok);
  }
  cpa_commit2();
}

#ifdef EIGENID_PHASE_TIMING
__device__ unsigned long long g_bulge_cycles[8];
#define BPH(id)                                                         \
  do {                                                                  \
    const long long now_ = clock64();                                   \
    if (lane == 0 && blockIdx.x == 0 && warp == 0)                      \
      g_bulge_cycles[id] += (unsigned long long)(now_ - t_b_);          \
    t_b_ = now_;                                                        \
  } while (0)
#else
#define BPH(id) \
  do {          \
  } while (0)
#endif

__device__ __forceinline__ long long spos(int sweep, int step) {
  return (long long)sweep * 65536 + step;
}

// Blocks until sweep s-1 (owned by warp w-1 mod W) has finished step k.
// The wait is bounded (see band.cu: kWaitTimeoutCode): a lost progress update
// ends the call with a device error instead of hanging the process.
constexpr int kChaseTimeoutCode = 30;
constexpr long long kChaseTimeoutCycles = 30000000000LL;
template <int W>
__device__ __forceinline__ void wait_prev(volatile long long* prog, int warp,
                                          int s, int k, DevStatus* st) {
  if (s == 0) return;
  const int pw = (warp + W - 1) % W;
  const long long need = spos(s - 1, k);
  if ((threadIdx.x & 31) == 0) {
    unsigned spins = 0;
    long long t0 = 0;
    while (prog[pw] < need) {
      __nanosleep(64);
      if (((++spins) & 0xfffu) == 0) {
        if (*(volatile const int*)&st->code == kChaseTimeoutCode) break;
        const long long now = clock64();
        if (t0 == 0) {
          t0 = now;
        } else if (now - t0 > kChaseTimeoutCycles) {
          set_status(st, kChaseTimeoutCode, 100 + k, 0.0, blockIdx.x * 1000 + warp);
          break;
        }
      }
    }
  }
  __syncwarp();
  __threadfence_block();
}

__device__ __forceinline__ void publish(volatile long long* prog, int warp,
                                        int s, int k) {
  __syncwarp();
  __threadfence_block();
  if ((threadIdx.x & 31) == 0) prog[warp] = spos(s, k);
}

template <int kWarpsPerCta, int kMinBlocks>
__global__ void __launch_bounds__(kWarpsPerCta * 32, kMinBlocks)
bulge_chase_kernel(Stage2Args a) {
#ifdef EIGENID_PHASE_TIMING
  long long t_b_ = clock64();
#endif
  extern __shared__ double smem[];
  __shared__ long long prog[kWarpsPerCta];
  __shared__ int s_sidx;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sC = smem + warp * kWarpSmem;
  double* const sD = sC + kBlk;
  double* sv = sD + kDP;
  double* sv2 = sv + kCB;
  double* sw = sv2 + kCB;

  for (;;) {
    __syncthreads();
    if (threadIdx.x == 0)
      s_sidx = *(volatile const int*)&a.status->code ? a.nsolves
                                                     : atomicAdd(a.counter, 1);
    if (threadIdx.x < kWarpsPerCta) prog[threadIdx.x] = -1;
    __syncthreads();
    const int sidx = s_sidx;
    if (sidx >= a.nsolves) break;
    const int m = a.js[sidx] < 0 ? a.n : a.n - 1;
    double* AB = a.band + sidx * a.band_stride;

    for (int st = warp; st + 2 < m; st += kWarpsPerCta) {
      const int R0 = st + 1;
      const int L0 = min(kCB, m - 1 - st);
      int Rk = R0 + kCB;
      bool have = Rk <= m - 1;
      int Lk = have ? min(kCB, m - Rk) : 0;
      // block 0 and the prefetch of step 1 need sweep st-1 past step 2
      wait_prev<kWarpsPerCta>(prog, warp, st, 2, a.status);
      const double x = lane < L0 ? AB[(long long)st * kCLD + 1 + lane] : 0.0;
      prefetch_d(sD, AB, R0, L0);
      if (have) prefetch_c(sC, AB, Rk, Lk, R0, L0);
      double beta;
      double tau = warp_householder(x, L0, sv, &beta);
      if (lane < L0) AB[(long long)st * kCLD + 1 + lane] = (lane == 0) ? beta : 0.0;
      cpa_wait_all();
      __syncwarp();
      if (L0 == kCB)
        two_sided_store<true>(sD, sv, tau, sw, L0, AB, R0, Rk, Lk);
      else
        two_sided_store<false>(sD, sv, tau, sw, L0, AB, R0, Rk, Lk);
      publish(prog, warp, st, 0);
      int R = R0, L = L0, k = 1;
      while (have) {
        // ---- step k on C = A[Rk.., R..] (Lk x L), D = A[Rk.., Rk..]; both
        // were prefetched during step k-1
        cpa_wait_all();
        __syncwarp();
        double crow[kCB];
#pragma unroll
        for (int c = 0; c < kCB; ++c) crow[c] = sC[lane * kSLD + c];
        const int Rn = Rk + kCB;
        const bool haven = Rn <= m - 1;
        const int Ln = haven ? min(kCB, m - Rn) : 0;
        BPH(0);
        if (haven) wait_prev<kWarpsPerCta>(prog, warp, st, k + 2, a.status);  // before step k+1's prefetches
        BPH(6);
        BPH(1);
        // right-apply the previous reflector: C -= tau (C v) v^T
        const double2* v2 = reinterpret_cast<const double2*>(sv);
        double yy[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int h = 0; h < kCB / 2; ++h) {
          const double2 v = v2[h];
          yy[(2 * h) & 3] += crow[2 * h] * v.x;
          yy[(2 * h + 1) & 3] += crow[2 * h + 1] * v.y;
        }
        const double y = tau * ((yy[0] + yy[1]) + (yy[2] + yy[3]));
#pragma unroll
        for (int h = 0; h < kCB / 2; ++h) {
          const double2 v = v2[h];
          crow[2 * h] -= y * v.x;
          crow[2 * h + 1] -= y * v.y;
        }
        // new reflector from C's first column
        double beta2;
        const double tau2 = warp_householder(crow[0], Lk, sv2, &beta2);
        crow[0] = (lane == 0) ? beta2 : 0.0;
        BPH(2);
        // left-apply to columns 1..L-1: w_c = tau2 sum_r v2_r C1[r][c] with
        // C1 = C - y v^T, i.e. tau2 ((C^T v2)_c - (y . v2) v_c); lane c takes
        // column c of the staged C (conflict-free row reads)
        {
          const double2* u2 = reinterpret_cast<const double2*>(sv2);
          double cc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
          for (int h = 0; h < kCB / 2; ++h) {
            const double2 u = u2[h];
            cc[(2 * h) & 3] += sC[(2 * h) * kSLD + lane] * u.x;
            cc[(2 * h + 1) & 3] += sC[(2 * h + 1) * kSLD + lane] * u.y;
          }
          const double yv = warp_sum(y * sv2[lane]);
          const double cs = (cc[0] + cc[1]) + (cc[2] + cc[3]);
          const double w = tau2 * (cs - yv * sv[lane]);
          __syncwarp();  // every lane is done with sC and sw
          if (haven) prefetch_c(sC, AB, Rn, Ln, Rk, Lk);
          sw[lane] = (lane >= 1 && lane < L) ? w : 0.0;
        }
        __syncwarp();
        {
          const double vr = sv2[lane];
          const double2* w2 = reinterpret_cast<const double2*>(sw);
#pragma unroll
          for (int h = 0; h < kCB / 2; ++h) {
            const double2 a = w2[h];
            if (h > 0) crow[2 * h] -= vr * a.x;  // w_0 = 0: column 0 is final
            crow[2 * h + 1] -= vr * a.y;
          }
        }
        const bool full = Lk == kCB && L == kCB;
        {
          double* base = AB + (long long)R * kCLD + (Rk - R) + lane;
          if (full) {
            st_full<0>(base, crow);
          } else {
#pragma unroll
            for (int c = 0; c < kCB; ++c)
              st_pred(base + c * (kCLD - 1), crow[c], lane < Lk && c < L);
          }
        }
        BPH(3);
        BPH(4);
        if (Lk == kCB)
          two_sided_store<true>(sD, sv2, tau2, sw, Lk, AB, Rk, Rn, Ln);
        else
          two_sided_store<false>(sD, sv2, tau2, sw, Lk, AB, Rk, Rn, Ln);
        BPH(5);
        sv[lane] = sv2[lane];
        publish(prog, warp, st, k);
        tau = tau2;
        R = Rk;
        L = Lk;
        Rk = Rn;
        Lk = Ln;
        have = haven;
        ++k;
      }
      publish(prog, warp, st, 65535);  // sweep done
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

#ifdef EIGENID_PHASE_TIMING
extern "C" void eigenid_debug_bulge_cycles(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_bulge_cycles, sizeof(g_bulge_cycles));
}
#endif

template <int W, int B = kBulgeCtasPerSm>
static cudaError_t launch_chase(const Stage2Args& a, int grid, cudaStream_t st) {
  const size_t smem = sizeof(double) * kWarpSmem * W;
  cudaError_t e = cudaFuncSetAttribute(
      bulge_chase_kernel<W, B>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  bulge_chase_kernel<W, B><<<grid, W * 32, smem, st>>>(a);
  return cudaGetLastError();
}

cudaError_t launch_stage2(const Stage2Args& a, cudaStream_t st) {
  cudaError_t e;
  e = cudaMemsetAsync(a.counter, 0, sizeof(int), st);
  if (e != cudaSuccess) return e;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, a.device);
  const int slots = sms * kBulgeCtasPerSm;
  const int grid = a.nsolves < slots ? a.nsolves : slots;
  bool long_sweeps = a.n >= kWarpsLongMinN;
  // EIGENID_STAGE2_WARPS=8|9 overrides the size-based choice (tests, A/B).
  if (const char* w = std::getenv("EIGENID_STAGE2_WARPS")) {
    if (w[0] == '8') long_sweeps = false;
    if (w[0] == '9') long_sweeps = true;
  }
  // lambda(A)'s lone chase beside the narrow stage-1 layout: <= 128
  // registers so it fits on an SM that still runs a stage-1 CTA
  bool compact = a.compact;
  if (const char* c = std::getenv("EIGENID_STAGE2_COMPACT")) compact = compact || c[0] == '1';
  if (compact) return launch_chase<kWarpsShort, 2>(a, grid, st);
  return long_sweeps ? launch_chase<kWarpsLong>(a, grid, st)
                     : launch_chase<kWarpsShort>(a, grid, st);
}

}  // namespace eigenid_b200
