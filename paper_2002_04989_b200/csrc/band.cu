// band.cu — K1L stage 1: batched dense -> band (bandwidth kB) reduction of
// the n principal minors M_j (and A itself), FP64 on the DMMA tensor path.
//
// Replaces, for large n, the Householder tridiagonalisation of every minor
// (tridiagonalize, eigensolve.cpp:19-69, called per minor through
// identity.cpp:303-306 after minor_matrix, matrix.cpp:51-68).  The reference
// runs a one-stage tred1 whose symmetric mat-vec (:42-49) reads the whole
// trailing matrix once per column; here the reduction is two-stage:
//   stage 1 (this file): dense -> band, blocked Householder on panels of kB
//            columns; every flop of the trailing update is a dense
//            contraction run as mma.sync.m8n8k4.f64 (DMMA.8x8x4):
//              X  = A22 (V T)              (GEMM 1, s x s x kB)
//              A22 -= W2 V^T + V W2^T      (GEMM 2, s x s x 2kB)
//   stage 2 (bulge.cu): band -> tridiagonal by bulge chasing.
// One CTA owns one solve at a time (persistent over the solve list); the
// minor is materialised once into the CTA's HBM workspace by an index remap
// of A (no host-side minor copies), the panel / T / W2 work is BLAS2-sized
// and stays in L1/L2, and the band is written as kB+1.. 2kB+1 column-major
// diagonals ready for the chase.
#include "kernels.cuh"

#include <type_traits>

#ifndef EIGENID_STAGE1_NS  // band_narrow.cu compiles this file again as "narrow"
#define EIGENID_STAGE1_NS wide
#define EIGENID_STAGE1_PRIMARY 1
#endif

namespace eigenid_b200 {
namespace EIGENID_STAGE1_NS {

constexpr int kB = 32;      // bandwidth / panel width
// Four layouts of this file are compiled (namespaces narrow / wide / wide8 /
// widesp; api.cu picks narrow below n = 2048 and widesp from there, the other
// two stay selectable through EIGENID_STAGE1_LAYOUT for A/B runs):
//   narrow  8 warps, two CTAs per SM, 64-row fused blocks: the second CTA
//           fills the DMMA pipe during the other's panel phases, which weigh
//           more at small n (17 % faster than the wide layouts at n = 1024);
//   wide    16 warps, one CTA per SM, 128-row blocks: half the Bop / VT / X
//           re-reads per trailing element, half the workspace slots;
//   wide8, widesp: see EIGENID_STAGE1_RW and EIGENID_STAGE1_SP below.
#ifndef EIGENID_STAGE1_WIDE
#define EIGENID_STAGE1_WIDE 1
#endif
// A third layout, "wide8" (EIGENID_STAGE1_RW = 2): 8 warps, one CTA per SM,
// 128-row fused blocks with SIXTEEN rows per warp and up to 255 registers per
// thread: every Bop / VT fragment read from shared memory feeds two DMMAs
// instead of one and the transposed product shares its C fragment between
// two X tiles, so the fused tile needs ~30 % fewer shared-memory wavefronts
// (the L1 data pipe is the co-limiter of the 16-warp layouts).
#ifndef EIGENID_STAGE1_RW
#define EIGENID_STAGE1_RW 1
#endif
constexpr int kRW = EIGENID_STAGE1_RW;  // 8-row groups per warp in the fused pass
// Interior-tile copy fast path: same-box -1.1 % (wide) / -12 % (wide8) at
// n = 4096 with the mbarrier pipeline.  The skip of above-diagonal row groups
// measured 2 % SLOWER in both layouts (the skipping warps only reach the
// mid-tile barrier earlier) and stays off.
#ifndef EIGENID_FAST_STAGE
#define EIGENID_FAST_STAGE 1
#endif
#ifndef EIGENID_DIAG_SKIP
#define EIGENID_DIAG_SKIP 0
#endif
// unpredicated write-back of the updated C rows in interior row blocks
#ifndef EIGENID_FAST_STORE
#define EIGENID_FAST_STORE 1
#endif
static_assert(kRW == 1 || (kRW == 2 && EIGENID_STAGE1_WIDE), "layout");
// A fourth layout, "widesp" (EIGENID_STAGE1_SP = 1, with RW = 2): 16 warps and
// one CTA per SM like "wide", but the fused pass is warp-specialised.  Warps
// 0-7 compute with the wide8 tiling (sixteen rows per warp) after growing
// their register allocation with setmaxnreg; warps 8-15 shrink theirs and
// only issue the cp.async copies, running ahead of the compute warps through
// the full / empty mbarriers.  Every other phase (panel, Gram, W2, GEMM 1/2)
// uses all 16 warps at 128 registers.
#ifndef EIGENID_STAGE1_SP
#define EIGENID_STAGE1_SP 0
#endif
constexpr int kSP = EIGENID_STAGE1_SP;
static_assert(!kSP || kRW == 2, "widesp uses the sixteen-rows-per-warp tiling");
constexpr int kNT = (EIGENID_STAGE1_WIDE && (kRW == 1 || kSP)) ? 512 : 256;  // threads per CTA
constexpr int kNW = kNT / 32;                         // warps per CTA
constexpr int kCW = kSP ? kNW / 2 : kNW;              // warps that compute in the fused pass
constexpr int kPT = kNT - 32 * kCW;                   // copy-only threads of the fused pass
constexpr int kCtasPerSm = EIGENID_STAGE1_WIDE ? 1 : 2;
constexpr int kLDAB = 2 * kB + 1;  // band storage: diagonals 0..2kB per column

// Shared-memory layout (doubles); the GEMM region is reused by the panel /
// Gram phases.  Every warp owns 8 rows of a GEMM-2 / fused row block.
constexpr int kG2M = 8 * kCW * kRW, kG2N = 32, kG2K = 2 * kB;  // fused row block / tile / k
constexpr int kG2R = 8 * kNW;                          // GEMM 2 row block
constexpr int kG1M = 64, kG1K = 32, kG1LDA = 36, kG1LDB = 36, kG1TLD = 68;
constexpr int kMT1 = 8 * kG1M / kNT;                // 8-row m-tiles per warp
constexpr int kG1_A = kG1M * kG1LDA;                // pass 1: A chunk 128 x 32
constexpr int kG1_T = kG1K * kG1TLD;                // pass 2: A chunk 32 x 128
constexpr int kG1_B = kG1K * kG1LDB;                // VT chunk 32 x 32
constexpr int kSmallLD = kB + 1;
constexpr int kSmallMat = kB * kSmallLD;            // T, G/Y, M
constexpr int kGramPart = 8 * kSmallMat;             // 8 partial Gram slots
constexpr int cmax(int a, int b) { return a > b ? a : b; }
constexpr int kG1S = 3;                             // GEMM 1 cp.async stages
constexpr int kG2S = 3;                             // GEMM 2 cp.async stages
// Fused-pass cp.async stages: two in every layout (a third stage measured
// 0.7 % faster in wide, 4 % slower in widesp at n = 4096: 58 KB less L1).
#ifndef EIGENID_FUSED_STAGES
#define EIGENID_FUSED_STAGES 2
#endif
constexpr int kFS = EIGENID_FUSED_STAGES;            // fused-pass stages
constexpr int kXT = 16 / kCW;  // 8x8 tiles of the fused transposed product per warp
constexpr int kG2St = kG2N * kG2K + kG2R * kG2N;    // Bop rows + C tile
#ifndef EIGENID_STAGE1_FUSED
#define EIGENID_STAGE1_FUSED 1
#endif
// split arrive / sync around the fused tile's row product (see gemm_fused)
#ifndef EIGENID_SPLIT_BAR
#define EIGENID_SPLIT_BAR 1
#endif
// Fused pass (rest of panel p's update + SYMM of panel p+1): kFS stages of
// {Bop rows, C tile, VT(cb) rows} plus the row block's VT(rb) rows.
constexpr int kFVLD = 34, kFVRLD = 36;

constexpr int kFSt = kG2N * kG2K + kG2M * kG2N + kB * kFVLD;
constexpr int kFSmem = kFS * kFSt + kG2M * kFVRLD;
constexpr int kGemmSmem =
    cmax(cmax(kGramPart, kG2S * kG2St - 3 * kSmallMat),
         EIGENID_STAGE1_FUSED ? kFSmem - 2 * kSmallMat : 0);
// GEMM 1 also owns the G and A scratch matrices that follow the GEMM region
// (both dead while it runs; T, after them, is not).
constexpr int kGemm1Smem = kGemmSmem + 2 * kSmallMat;
// GEMM 2 owns G, A and T as well (all dead while it runs).
static_assert(kG2S * kG2St <= kGemmSmem + 3 * kSmallMat, "gemm2 smem");
// the fused pass owns G and A but not T (T of panel p+1 outlives it)
static_assert(!EIGENID_STAGE1_FUSED || kFSmem <= kGemmSmem + 2 * kSmallMat, "fused smem");
static_assert(kG1S * (kG1_A + kG1_B) <= kGemm1Smem &&
                  kG1S * (kG1_T + kG1_B) <= kGemm1Smem, "gemm1 smem");
constexpr int kRed = kNW + kNW * kB;
// T, G/Y, A persist across Gram calls; B and R live in the GEMM region
// (never alive across a gram() or GEMM call).  ~101 KB: two CTAs per SM.
constexpr int kStage1SmemDoubles = kGemmSmem + 3 * kSmallMat + kRed + 4 * kB;
static_assert(kGemmSmem >= kGramPart && kGemmSmem >= 2 * kSmallMat, "smem");

// unroll factors of the streaming panel passes (loads in flight per warp)
#ifndef EIGENID_GRAM_UNROLL
#define EIGENID_GRAM_UNROLL 2
#endif
#ifndef EIGENID_RT_UNROLL
#define EIGENID_RT_UNROLL 2
#endif
constexpr int kGramUnroll = EIGENID_GRAM_UNROLL, kRtUnroll = EIGENID_RT_UNROLL;

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, "
      "{%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem,
                                           int src_bytes) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(saddr),
               "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async16_full(double* smem, const double* gmem) {
  const unsigned saddr = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(saddr), "l"(gmem));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cpa_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cpa_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ double block_sum(double x, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  x = warp_sum(x);
  __syncthreads();
  if (lane == 0) red[warp] = x;
  __syncthreads();
  double t = 0.0;
#pragma unroll
  for (int w = 0; w < kNT / 32; ++w) t += red[w];
  return t;
}

// ---- panel QR ----------------------------------------------------------
// Householder QR of the s x kB panel P(r,q) = P0[r*ldw + q] (LAPACK
// dgeqr2/dlarfg convention, H = I - tau v v^T, v_0 = 1).  Lane q owns column
// q, warps stride over rows, so every row access is one coalesced 256-byte
// warp load; two streaming passes per column (w = v^T P, then the update
// fused with the next column's norm).  On exit the upper triangle holds R and
// the strictly lower part holds the reflectors v (LAPACK layout).
__device__ void panel_qr(double* P0, int ldw, int s, double* stau, double* red,
                         double* wsm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kr = min(kB, s - 1);
  double loc = 0.0;
  for (int r = 1 + tid; r < s; r += kNT) {
    const double x = P0[(long long)r * ldw];
    loc += x * x;
  }
  double sigma = block_sum(loc, red);
  for (int t = 0; t < kr; ++t) {
    const double alpha = P0[(long long)t * ldw + t];
    double tau, beta, scal;
    if (sigma == 0.0) {
      tau = 0.0;
      beta = alpha;
      scal = 0.0;
    } else {
      beta = -copysign(sqrt(alpha * alpha + sigma), alpha);
      tau = (beta - alpha) / beta;
      scal = 1.0 / (alpha - beta);
    }
    // pass A: acc_q = sum_{r>t} P(r,t) P(r,q)
    double acc = 0.0;
    for (int r0 = t + 1 + warp; r0 < s; r0 += 4 * kNW) {
      double row[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + kNW * u;
        row[u] = r < s ? P0[(long long)r * ldw + lane] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        acc += __shfl_sync(0xffffffffu, row[u], t) * row[u];
    }
    __syncthreads();
    red[kNW + warp * kB + lane] = acc;
    __syncthreads();
    if (warp == 0) {
      double w = 0.0;
#pragma unroll
      for (int ww = 0; ww < kNW; ++ww) w += red[kNW + ww * kB + lane];
      w = w * scal + P0[(long long)t * ldw + lane];
      wsm[lane] = (lane > t) ? tau * w : 0.0;
    }
    __syncthreads();
    // pass B: P(r,q) -= tau w_q v_r, v stored below the diagonal
    const double wq = wsm[lane];
    loc = 0.0;
    for (int r0 = t + warp; r0 < s; r0 += 4 * kNW) {
      double row[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + kNW * u;
        row[u] = r < s ? P0[(long long)r * ldw + lane] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int r = r0 + kNW * u;
        if (r < s) {
          const double x = __shfl_sync(0xffffffffu, row[u], t);
          const double v = (r == t) ? 1.0 : x * scal;
          double y = row[u];
          if (lane > t)
            y -= wq * v;
          else if (lane == t)
            y = (r == t) ? beta : v;
          if (lane >= t) P0[(long long)r * ldw + lane] = y;
          if (lane == t + 1 && r > t + 1) loc += y * y;
        }
      }
    }
    if (tid == 0) stau[t] = tau;
    sigma = block_sum(loc, red);
  }
  if (tid < kB && tid >= kr) stau[tid] = 0.0;
  __syncthreads();
}

// V (s x kB row-major, unit lower trapezoidal) from the LAPACK-layout panel.
__device__ void extract_v(const double* P0, int ldw, int s, double* Vg) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int r = warp; r < s; r += kNT / 32) {
    const double x = P0[(long long)r * ldw + lane];
    Vg[(long long)r * kB + lane] = r > lane ? x : (r == lane ? 1.0 : 0.0);
  }
  __syncthreads();
}

// out[q][p] = sum_{r<s} L(r,q) R(r,p) on the DMMA path: warp w takes the
// 4-row k-slices i = w (mod kNW); partials are summed through shared memory.
__device__ void gram(const double* L, int ldl, const double* R, int ldr, int s,
                     double* out, double* part) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kk = lane & 3, mm = lane >> 2;
  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll kGramUnroll
  for (int i = warp; 4 * i < s; i += kNT / 32) {
    const int r = 4 * i + kk;
    double a[4], b[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      a[t] = r < s ? L[(long long)r * ldl + 8 * t + mm] : 0.0;
      b[t] = r < s ? R[(long long)r * ldr + 8 * t + mm] : 0.0;
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt)
        dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
  }
  __syncthreads();
  // 8 partial slots; with 16 warps, warps 8..15 deposit first and warps
  // 0..7 add their own partial on top
  double* pw = part + (warp & 7) * kSmallMat;
  if (warp >= 8) {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        pw[(8 * mt + mm) * kSmallLD + 8 * nt + 2 * kk] = acc[mt][nt][0];
        pw[(8 * mt + mm) * kSmallLD + 8 * nt + 2 * kk + 1] = acc[mt][nt][1];
      }
  }
  if (kNW > 8) __syncthreads();
  if (warp < 8) {
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        double* q0 = pw + (8 * mt + mm) * kSmallLD + 8 * nt + 2 * kk;
        q0[0] = (kNW > 8 ? q0[0] : 0.0) + acc[mt][nt][0];
        q0[1] = (kNW > 8 ? q0[1] : 0.0) + acc[mt][nt][1];
      }
  }
  __syncthreads();
  for (int e = tid; e < kB * kB; e += kNT) {
    const int q = e / kB, p = e % kB;
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < 8; ++w) v += part[w * kSmallMat + q * kSmallLD + p];
    out[q * kSmallLD + p] = v;
  }
  __syncthreads();
}

// Y(r,:) = (Add ? Add(r,:) : 0) + alpha * L(r,:) Mt (Mt kB x kB in shared
// memory, ld kSmallLD) on the DMMA path: warp w owns the 32-row blocks
// w, w+8, ... and keeps the 32 x 32 output block in registers, so Y may alias
// L or Add.
__device__ void row_transform(const double* L, int ldl, const double* Mt,
                              double alpha, const double* Add, double* Y,
                              int s) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kk = lane & 3, mm = lane >> 2;
  for (int rb = 32 * warp; rb < s; rb += 32 * (kNT / 32)) {
    double acc[4][4][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll kRtUnroll
    for (int k4 = 0; k4 < kB / 4; ++k4) {
      const int k = 4 * k4 + kk;
      double af[4], bf[4];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int r = rb + 8 * mt + mm;
        af[mt] = r < s ? L[(long long)r * ldl + k] : 0.0;
      }
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) bf[nt] = Mt[k * kSmallLD + 8 * nt + mm];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
    }
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) {
      const int r = rb + 8 * mt + mm;
      if (r >= s) continue;
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = 8 * nt + 2 * kk;
        double2 y = make_double2(alpha * acc[mt][nt][0], alpha * acc[mt][nt][1]);
        if (Add) {
          const double2 ad = *reinterpret_cast<const double2*>(Add + (long long)r * kB + c);
          y.x += ad.x;
          y.y += ad.y;
        }
        *reinterpret_cast<double2*>(Y + (long long)r * kB + c) = y;
      }
    }
  }
  __syncthreads();
}

// ---- CholeskyQR2 panel with Householder reconstruction -----------------
// The panel's Householder representation (V, T) is rebuilt from an
// orthonormal basis Q1 of the panel (Ballard et al., "Reconstructing
// Householder vectors from tall-skinny QR"): Q1 - S = L U with S = -sign of
// each pivot, V = L, T = -U S L1^-T, and H = I - V T V^T satisfies
// H^T P = [S R; 0].  Q1, R come from two Cholesky-QR passes (Gram matrices on
// the DMMA path).  Five streaming passes over the panel replace the 2 kB
// latency-bound passes of column Householder; panels whose second Gram
// matrix is not within 1e-3 of I (cond(P) >~ 1e6), or whose Cholesky breaks
// down, fall back to panel_qr.

// Upper Cholesky factor R (G = R^T R) of the kB x kB matrix G; warp-level.
__device__ bool warp_chol(const double* G, double* R) {
  const int lane = threadIdx.x & 31;
  bool ok = true;
  for (int j = 0; j < kB; ++j) {
    double d = G[j * kSmallLD + j];
    for (int k = 0; k < j; ++k) d -= R[k * kSmallLD + j] * R[k * kSmallLD + j];
    if (!(d > 0.0)) ok = false;
    const double rjj = sqrt(fmax(d, 1e-300));
    if (lane > j) {
      double v = G[j * kSmallLD + lane];
      for (int k = 0; k < j; ++k) v -= R[k * kSmallLD + j] * R[k * kSmallLD + lane];
      R[j * kSmallLD + lane] = v / rjj;
    } else if (lane == j) {
      R[j * kSmallLD + j] = rjj;
    } else {
      R[j * kSmallLD + lane] = 0.0;
    }
    __syncwarp();
  }
  return ok;
}

// Inverse of an upper triangular kB x kB matrix; lane c solves column c.
__device__ void warp_upper_inv(const double* R, double* Ri) {
  const int c = threadIdx.x & 31;
  double x[kB];
#pragma unroll
  for (int i = kB - 1; i >= 0; --i) {
    double v = (i == c) ? 1.0 : 0.0;
#pragma unroll
    for (int k = i + 1; k < kB; ++k) v -= R[i * kSmallLD + k] * x[k];
    x[i] = (i <= c) ? v / R[i * kSmallLD + i] : 0.0;
  }
#pragma unroll
  for (int i = 0; i < kB; ++i) Ri[i * kSmallLD + c] = x[i];
  __syncwarp();
}

// Inverse of a unit lower triangular matrix (strict lower part of L).
__device__ void warp_unit_lower_inv(const double* L, double* Li) {
  const int c = threadIdx.x & 31;
  double x[kB];
#pragma unroll
  for (int i = 0; i < kB; ++i) {
    double v = (i == c) ? 1.0 : 0.0;
#pragma unroll
    for (int k = 0; k < i; ++k) v -= L[i * kSmallLD + k] * x[k];
    x[i] = (i >= c) ? v : 0.0;
  }
#pragma unroll
  for (int i = 0; i < kB; ++i) Li[i * kSmallLD + c] = x[i];
  __syncwarp();
}

// C = A B for upper triangular A, B (kB x kB); lane c computes column c.
__device__ void warp_upper_mul(const double* A, const double* B, double* C) {
  const int c = threadIdx.x & 31;
  for (int i = 0; i < kB; ++i) {
    double v = 0.0;
    for (int k = i; k <= c; ++k) v += A[i * kSmallLD + k] * B[k * kSmallLD + c];
    C[i * kSmallLD + c] = (i <= c) ? v : 0.0;
  }
  __syncwarp();
}

#ifdef EIGENID_PHASE_TIMING
__device__ unsigned long long g_phase_cycles[16];
// sub-phases of chol_panel (CTA 0) -> g_phase_cycles[8 + id]
#define SUBPH(id)                                                          \
  do {                                                                     \
    __syncthreads();                                                       \
    const long long now_ = clock64();                                      \
    if (threadIdx.x == 0)                                                  \
      atomicAdd(&g_phase_cycles[8 + (id)], (unsigned long long)(now_ - t_sp_)); \
    t_sp_ = now_;                                                          \
  } while (0)
#else
#define SUBPH(id) \
  do {            \
  } while (0)
#endif

__device__ bool chol_panel(double* P0, int ldw, int s, double* Vg, double* Xg,
                           double* sT, double* sG, double* sA, double* sB,
                           double* sR, double* sS, double* part, int* flag) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
#ifdef EIGENID_PHASE_TIMING
  long long t_sp_ = clock64();
#endif
  gram(P0, ldw, P0, ldw, s, sG, part);                    // G1 = P^T P
  SUBPH(0);
  if (warp == 0) {
    const bool ok = warp_chol(sG, sA);                     // R1
    if (lane == 0) *flag = ok;
    if (ok) warp_upper_inv(sA, sB);                        // R1^-1
  }
  __syncthreads();
  if (!*flag) return false;
  SUBPH(1);
  row_transform(P0, ldw, sB, 1.0, nullptr, Vg, s);         // Q = P R1^-1
  SUBPH(2);
  gram(Vg, kB, Vg, kB, s, sG, part);                      // G2 = Q^T Q
  SUBPH(3);
  if (warp == 0) {
    double dev = 0.0;
    for (int e = lane; e < kB * kB; e += 32) {
      const int q = e / kB, p = e % kB;
      dev = fmax(dev, fabs(sG[q * kSmallLD + p] - (q == p ? 1.0 : 0.0)));
    }
    dev = warp_max(dev);
    bool ok = dev <= 1e-3;
    if (ok) ok = warp_chol(sG, sB);                        // R2
    if (lane == 0) *flag = ok;
    if (ok) {
      warp_upper_mul(sB, sA, sR);                          // R = R2 R1
      warp_upper_inv(sB, sA);                              // R2^-1
    }
  }
  __syncthreads();
  if (!*flag) return false;
  SUBPH(4);
  row_transform(Vg, kB, sA, 1.0, nullptr, Xg, s);          // Q1 = Q R2^-1
  SUBPH(5);
  if (warp == 0) {
    // modified LU of the top block: Q1_top - S = L U (U' in sG upper)
    for (int r = 0; r < kB; ++r) sG[r * kSmallLD + lane] = Xg[r * kB + lane];
    __syncwarp();
    for (int i = 0; i < kB; ++i) {
      const double p = sG[i * kSmallLD + i];
      const double si = p >= 0.0 ? -1.0 : 1.0;
      __syncwarp();
      if (lane == 0) {
        sS[i] = si;
        sG[i * kSmallLD + i] = p - si;
      }
      __syncwarp();
      const double piv = sG[i * kSmallLD + i];
      if (lane > i) {
        const double l = sG[lane * kSmallLD + i] / piv;
        sG[lane * kSmallLD + i] = l;
        for (int c = i + 1; c < kB; ++c) sG[lane * kSmallLD + c] -= l * sG[i * kSmallLD + c];
      }
      __syncwarp();
    }
    // U'^-1 (upper part of sG) -> sB ; L1^-1 -> sA
    {
      const int c = lane;
      double x[kB];
#pragma unroll
      for (int i = kB - 1; i >= 0; --i) {
        double v = (i == c) ? 1.0 : 0.0;
#pragma unroll
        for (int k = i + 1; k < kB; ++k) v -= sG[i * kSmallLD + k] * x[k];
        x[i] = (i <= c) ? v / sG[i * kSmallLD + i] : 0.0;
      }
#pragma unroll
      for (int i = 0; i < kB; ++i) sB[i * kSmallLD + c] = x[i];
    }
    __syncwarp();
    warp_unit_lower_inv(sG, sA);
  }
  __syncthreads();
  // T = -U' S L1^-T  (upper)
  for (int e = tid; e < kB * kB; e += kNT) {
    const int i = e / kB, jj = e % kB;
    double v = 0.0;
    for (int k = i; k <= jj; ++k)
      v += sG[i * kSmallLD + k] * sS[k] * sA[jj * kSmallLD + k];
    sT[i * kSmallLD + jj] = (i <= jj) ? -v : 0.0;
  }
  // V: top rows L1 (unit lower), below Q1_bottom U'^-1 ; panel top <- S R
  for (int r = warp; r < kB; r += kNT / 32)
    Vg[r * kB + lane] = lane < r ? sG[r * kSmallLD + lane] : (lane == r ? 1.0 : 0.0);
  for (int r = warp; r < kB; r += kNT / 32)
    P0[(long long)r * ldw + lane] = lane >= r ? sS[r] * sR[r * kSmallLD + lane] : 0.0;
  __syncthreads();
  SUBPH(6);
  row_transform(Xg + kB * kB, kB, sB, 1.0, nullptr, Vg + kB * kB, s - kB);
  SUBPH(2);
  return true;
}

// ---- GEMM 1: X = A22 VT with A22 symmetric, lower triangle only ----------
// pass 1: X[r] = sum_{c <= r} A(r,c) VT(c)       (row blocks of 128)
// pass 2: X[c] += sum_{r > c} A(r,c) VT(r)       (column blocks of 128)
// Elements outside the lower triangle are masked to zero in the fragments,
// so only the lower triangle of A22 is ever read or kept up to date.
__device__ void gemm1(const double* A22, int ldw, int s, const double* VT,
                      double* X, double* sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kk = lane & 3, mm = lane >> 2;
  const int wm = warp >> 1, wn = warp & 1;
  // ---------------- pass 1
  {
    constexpr int kSt = kG1_A + kG1_B;  // one stage: A chunk, then VT chunk
    for (int rb = 0; rb < s; rb += kG1M) {
      const int kend = min(rb + kG1M, s);
      const int nk = (kend + kG1K - 1) / kG1K;
      double acc[kMT1][2][2];
#pragma unroll
      for (int a = 0; a < kMT1; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
      // one commit group per chunk (empty past the end) keeps the
      // wait_group arithmetic uniform
      auto stage = [&](int ki) {
        if (ki < nk) {
          const int kb = ki * kG1K, buf = ki % kG1S;
          for (int t = tid; t < kG1M * (kG1K / 2); t += kNT) {
            const int r = t >> 4, c2 = (t & 15) * 2;
            const int gr = rb + r, gc = kb + c2;
            int bytes = 0;
            if (gr < s && gc < kend) bytes = (gc + 1 < kend) ? 16 : 8;
            cp_async16(sm + buf * kSt + r * kG1LDA + c2,
                       bytes ? A22 + (long long)gr * ldw + gc : A22, bytes);
          }
          for (int t = tid; t < kG1K * (kB / 2); t += kNT) {
            const int r = t >> 4, c2 = (t & 15) * 2;
            const int gr = kb + r;
            const int bytes = gr < kend ? 16 : 0;
            cp_async16(sm + buf * kSt + kG1_A + r * kG1LDB + c2,
                       bytes ? VT + (long long)gr * kB + c2 : VT, bytes);
          }
        }
        cpa_commit();
      };
      __syncthreads();
#pragma unroll
      for (int p = 0; p < kG1S - 1; ++p) stage(p);
      for (int ki = 0; ki < nk; ++ki) {
        cpa_wait<kG1S - 2>();
        __syncthreads();
        stage(ki + kG1S - 1);
        const double* a = sm + (ki % kG1S) * kSt;
        const double* b = a + kG1_A;
        const int kb = ki * kG1K;
        const bool diag = kb + kG1K > rb;  // chunk may cross the diagonal
#pragma unroll
        for (int k4 = 0; k4 < kG1K / 4; ++k4) {
          const int kl = 4 * k4 + kk;
          double af[kMT1], bf[2];
#pragma unroll
          for (int mt = 0; mt < kMT1; ++mt) {
            const int ml = 8 * kMT1 * wm + 8 * mt + mm;
            const double v = a[ml * kG1LDA + kl];
            af[mt] = (diag && kb + kl > rb + ml) ? 0.0 : v;
          }
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) bf[nt] = b[kl * kG1LDB + 16 * wn + 8 * nt + mm];
#pragma unroll
          for (int mt = 0; mt < kMT1; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
              dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
        }
      }
      cpa_wait0();
#pragma unroll
      for (int mt = 0; mt < kMT1; ++mt) {
        const int r = rb + 8 * kMT1 * wm + 8 * mt + mm;
        if (r >= s) continue;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int c = 16 * wn + 8 * nt + 2 * kk;
          *reinterpret_cast<double2*>(X + (long long)r * kB + c) =
              make_double2(acc[mt][nt][0], acc[mt][nt][1]);
        }
      }
    }
  }
  __syncthreads();
  // ---------------- pass 2
  {
    constexpr int kSt = kG1_T + kG1_B;  // one stage: A chunk, then VT chunk
    for (int cb = 0; cb < s; cb += kG1M) {
      const int k0 = cb + 1;  // rows r > c >= cb
      if (k0 >= s) break;
      const int nk = (s - k0 + kG1K - 1) / kG1K;
      double acc[kMT1][2][2];
#pragma unroll
      for (int mt = 0; mt < kMT1; ++mt) {
        const int r = cb + 8 * kMT1 * wm + 8 * mt + mm;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int c = 16 * wn + 8 * nt + 2 * kk;
          if (r < s) {
            const double2 x = *reinterpret_cast<const double2*>(X + (long long)r * kB + c);
            acc[mt][nt][0] = x.x;
            acc[mt][nt][1] = x.y;
          } else {
            acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
          }
        }
      }
      const int cend = min(cb + kG1M, s);
      auto stage = [&](int ki) {
        if (ki < nk) {
          const int kb = k0 + ki * kG1K, buf = ki % kG1S;
          for (int t = tid; t < kG1K * (kG1M / 2); t += kNT) {
            const int r = t / (kG1M / 2), c2 = (t % (kG1M / 2)) * 2;
            const int gr = kb + r, gc = cb + c2;
            int bytes = 0;
            if (gr < s && gc < cend) bytes = (gc + 1 < cend) ? 16 : 8;
            cp_async16(sm + buf * kSt + r * kG1TLD + c2,
                       bytes ? A22 + (long long)gr * ldw + gc : A22, bytes);
          }
          for (int t = tid; t < kG1K * (kB / 2); t += kNT) {
            const int r = t >> 4, c2 = (t & 15) * 2;
            const int gr = kb + r;
            const int bytes = gr < s ? 16 : 0;
            cp_async16(sm + buf * kSt + kG1_T + r * kG1LDB + c2,
                       bytes ? VT + (long long)gr * kB + c2 : VT, bytes);
          }
        }
        cpa_commit();
      };
      __syncthreads();
#pragma unroll
      for (int p = 0; p < kG1S - 1; ++p) stage(p);
      for (int ki = 0; ki < nk; ++ki) {
        cpa_wait<kG1S - 2>();
        __syncthreads();
        stage(ki + kG1S - 1);
        const double* a = sm + (ki % kG1S) * kSt;
        const double* b = a + kG1_T;
        const int kb = k0 + ki * kG1K;
        const bool diag = kb < cb + kG1M;
#pragma unroll
        for (int k4 = 0; k4 < kG1K / 4; ++k4) {
          const int kl = 4 * k4 + kk;
          double af[kMT1], bf[2];
#pragma unroll
          for (int mt = 0; mt < kMT1; ++mt) {
            const int ml = 8 * kMT1 * wm + 8 * mt + mm;
            const double v = a[kl * kG1TLD + ml];
            af[mt] = (diag && kb + kl <= cb + ml) ? 0.0 : v;
          }
#pragma unroll
          for (int nt = 0; nt < 2; ++nt) bf[nt] = b[kl * kG1LDB + 16 * wn + 8 * nt + mm];
#pragma unroll
          for (int mt = 0; mt < kMT1; ++mt)
#pragma unroll
            for (int nt = 0; nt < 2; ++nt)
              dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
        }
      }
      cpa_wait0();
#pragma unroll
      for (int mt = 0; mt < kMT1; ++mt) {
        const int r = cb + 8 * kMT1 * wm + 8 * mt + mm;
        if (r >= s) continue;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int c = 16 * wn + 8 * nt + 2 * kk;
          *reinterpret_cast<double2*>(X + (long long)r * kB + c) =
              make_double2(acc[mt][nt][0], acc[mt][nt][1]);
        }
      }
    }
  }
  __syncthreads();
}

// ---- GEMM 2: A22 -= W2 V^T + V W2^T on the lower triangle ----------------
// As A22 += Aop Bop^T, Aop = -[W2 | V], Bop = [V | W2] (s x 2kB).  Row blocks
// of 64: warp w owns rows 8w..8w+7 and keeps its Aop fragments (16 k-steps)
// in registers for the whole row block; column tiles of 32 up to the
// diagonal stream their C tile (HBM) and Bop rows (L2) through a kG2S-stage
// cp.async pipeline in XOR-swizzled, unpadded shared memory, so two tiles
// are in flight while one is computed.  Bop fragments are 16-byte loads that
// feed two DMMAs (adjacent k values per lane).  Tiles crossing the diagonal also
// write their (never read) upper part.
__device__ void gemm2(double* A22, int ldw, int s, const double* W2,
                      const double* V, double* sm, int max_tiles = 1 << 30) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kk = lane & 3, mm = lane >> 2;
  const int crow = 8 * warp + mm;  // this lane's row within the row block
  for (int rb = 0; rb < s; rb += kG2R) {
    const int r = rb + crow;
    // k-pair q covers k = 8q .. 8q+7: lane kk takes k = 8q + 2kk in the
    // first DMMA of the pair and 8q + 2kk + 1 in the second, so both operands
    // of a pair are one 16-byte load
    double2 af[kG2K / 8];
#pragma unroll
    for (int q = 0; q < kG2K / 8; ++q) {
      const int k = 8 * q + 2 * kk;
      double2 v = make_double2(0.0, 0.0);
      if (r < s)
        v = *reinterpret_cast<const double2*>(k < kB ? W2 + (long long)r * kB + k
                                                     : V + (long long)r * kB + (k - kB));
      af[q] = make_double2(-v.x, -v.y);
    }
    const int cend = min(rb + kG2R, s);
    const int ncb = min((cend + kG2N - 1) / kG2N, max_tiles);
    auto stage = [&](int ci) {
      if (ci < ncb) {
        const int cb = ci * kG2N;
        double* st = sm + (ci % kG2S) * kG2St;
        for (int t = tid; t < kG2N * (kG2K / 2); t += kNT) {
          const int row = t >> 5, k2 = (t & 31) * 2;
          const int gr = cb + row;
          const int bytes = gr < s ? 16 : 0;
          const long long g = (long long)(bytes ? gr : 0) * kB;
          const double* src = k2 < kB ? V + g + k2 : W2 + g + (k2 - kB);
          cp_async16(st + row * kG2K + (k2 ^ (8 * (row & 1))), src, bytes);
        }
        double* cs = st + kG2N * kG2K;
        for (int t = tid; t < kG2R * (kG2N / 2); t += kNT) {
          const int row = t >> 4, c2 = (t & 15) * 2;
          const int gr = rb + row, gc = cb + c2;
          int bytes = 0;
          if (gr < s && gc < s) bytes = gc + 1 < s ? 16 : 8;
          cp_async16(cs + row * kG2N + (c2 ^ (8 * (row & 1))),
                     bytes ? A22 + (long long)gr * ldw + gc : A22, bytes);
        }
      }
      cpa_commit();
    };
    __syncthreads();  // the previous row block's last tile is consumed
#pragma unroll
    for (int p = 0; p < kG2S - 1; ++p) stage(p);
    for (int ci = 0; ci < ncb; ++ci) {
      cpa_wait<kG2S - 2>();
      __syncthreads();
      stage(ci + kG2S - 1);
      const double* b = sm + (ci % kG2S) * kG2St;
      const double* cs = b + kG2N * kG2K;
      double acc[kG2N / 8][2];
#pragma unroll
      for (int nt = 0; nt < kG2N / 8; ++nt) {
        const double2 x = *reinterpret_cast<const double2*>(
            cs + crow * kG2N + ((8 * nt + 2 * kk) ^ (8 * (crow & 1))));
        acc[nt][0] = x.x;
        acc[nt][1] = x.y;
      }
#pragma unroll
      for (int q = 0; q < kG2K / 8; ++q) {
        const int kl = (8 * q + 2 * kk) ^ (8 * (mm & 1));
        double2 bf[kG2N / 8];
#pragma unroll
        for (int nt = 0; nt < kG2N / 8; ++nt)
          bf[nt] = *reinterpret_cast<const double2*>(b + (8 * nt + mm) * kG2K + kl);
        // independent accumulators back to back (the DMMAs are volatile, so
        // this order is the issue order)
#pragma unroll
        for (int nt = 0; nt < kG2N / 8; ++nt) dmma(acc[nt][0], acc[nt][1], af[q].x, bf[nt].x);
#pragma unroll
        for (int nt = 0; nt < kG2N / 8; ++nt) dmma(acc[nt][0], acc[nt][1], af[q].y, bf[nt].y);
      }
      if (r < s) {
        const int cb = ci * kG2N;
#pragma unroll
        for (int nt = 0; nt < kG2N / 8; ++nt) {
          const int col = cb + 8 * nt + 2 * kk;
          double* p = A22 + (long long)r * ldw + col;
          if (col + 1 < s)
            *reinterpret_cast<double2*>(p) = make_double2(acc[nt][0], acc[nt][1]);
          else if (col < s)
            p[0] = acc[nt][0];
        }
      }
    }
    cpa_wait0();
  }
  __syncthreads();
}

// ---- next panel's columns: A22[:, 0:kB] -= (W2 V^T + V W2^T)[:, 0:kB] -------
// The one-tile-per-row-block case of GEMM 2 (same arithmetic, element by
// element), restructured for latency: the 32 Bop rows are staged once, then
// every warp streams its own 8-row groups — A-operand rows and C rows straight
// from global memory into registers, the next group's loads in flight while
// the current one runs its 64 DMMAs — with no CTA barrier per row block (GEMM 2
// spent ~2 us per 128 rows waiting for a cp.async round trip: 9.6 ms per solve
// at n = 4096).
__device__ void update_cols(double* A22, int ldw, int s, const double* W2, const double* V,
                            double* sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kk = lane & 3, mm = lane >> 2;
  __syncthreads();
  for (int t = tid; t < kG2N * (kG2K / 2); t += kNT) {
    const int row = t >> 5, k2 = (t & 31) * 2;
    const int bytes = row < s ? 16 : 0;
    const long long g = (long long)(bytes ? row : 0) * kB;
    const double* src = k2 < kB ? V + g + k2 : W2 + g + (k2 - kB);
    cp_async16(sm + row * kG2K + (k2 ^ (8 * (row & 1))), src, bytes);
  }
  cpa_commit();
  struct Group {
    double2 af[kG2K / 8];
    double2 c[kG2N / 8];
  };
  auto load = [&](int r, Group& g) {
#pragma unroll
    for (int q = 0; q < kG2K / 8; ++q) {
      const int k = 8 * q + 2 * kk;
      double2 v = make_double2(0.0, 0.0);
      if (r < s)
        v = *reinterpret_cast<const double2*>(k < kB ? W2 + (long long)r * kB + k
                                                     : V + (long long)r * kB + (k - kB));
      g.af[q] = make_double2(-v.x, -v.y);
    }
#pragma unroll
    for (int nt = 0; nt < kG2N / 8; ++nt)
      g.c[nt] = r < s ? *reinterpret_cast<const double2*>(A22 + (long long)r * ldw + 8 * nt + 2 * kk)
                      : make_double2(0.0, 0.0);
  };
  Group cur, nxt;
  int r = 8 * warp + mm;
  load(r, cur);
  cpa_wait0();
  __syncthreads();
  for (; r - mm < s; r += 8 * kNW) {
    load(r + 8 * kNW, nxt);  // rows past the end load nothing
    double acc[kG2N / 8][2];
#pragma unroll
    for (int nt = 0; nt < kG2N / 8; ++nt) {
      acc[nt][0] = cur.c[nt].x;
      acc[nt][1] = cur.c[nt].y;
    }
#pragma unroll
    for (int q = 0; q < kG2K / 8; ++q) {
      const int kl = (8 * q + 2 * kk) ^ (8 * (mm & 1));
      double2 bf[kG2N / 8];
#pragma unroll
      for (int nt = 0; nt < kG2N / 8; ++nt)
        bf[nt] = *reinterpret_cast<const double2*>(sm + (8 * nt + mm) * kG2K + kl);
#pragma unroll
      for (int nt = 0; nt < kG2N / 8; ++nt) dmma(acc[nt][0], acc[nt][1], cur.af[q].x, bf[nt].x);
#pragma unroll
      for (int nt = 0; nt < kG2N / 8; ++nt) dmma(acc[nt][0], acc[nt][1], cur.af[q].y, bf[nt].y);
    }
    if (r < s) {
#pragma unroll
      for (int nt = 0; nt < kG2N / 8; ++nt)
        *reinterpret_cast<double2*>(A22 + (long long)r * ldw + 8 * nt + 2 * kk) =
            make_double2(acc[nt][0], acc[nt][1]);
    }
    cur = nxt;
  }
  __syncthreads();
}

// ---- fused: rest of panel p's update + SYMM of panel p+1 -----------------
// A22n is the trailing matrix of panel p+1 (A22 of panel p without its first
// kB rows and columns, whose update was applied beforehand).  One pass over
// its lower tiles (64 x 32, row blocks in order, tiles up to the diagonal):
//   C  = C - W2p Vp^T - Vp W2p^T            (panel p; written back)
//   X[rb] += tril(C) VTn[cb]                 (registers, added per row block)
//   X[cb] += strict(C)^T VTn[rb]             (read-modify-write per tile)
// so the trailing matrix is read and written once per panel instead of being
// read three times and written once.  Xn must be zero on entry; every X
// element is accumulated in an order fixed by (n, panel), never by timing.
// Shared memory: two stages of {Bop rows (swizzled), C tile (swizzled),
// VTn[cb] rows} and the row block's VTn[rb] rows.
__device__ __forceinline__ int cswz(int row, int col) {
  return row * kG2N + (col ^ ((8 * (row & 1)) ^ (4 * ((row >> 1) & 1))));
}

// mbarrier helpers (CTA scope): arrive has release, try_wait acquire
// semantics, so shared-memory writes before an arrival are visible to a
// thread whose wait on that phase has returned.
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar)),
               "r"(count)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
// Device status code of a wait that ran out of time (reported by the host as
// EIGENID_E_DEVICE): every inter-warp wait of the library is bounded, so a
// lost arrival ends the call with an error instead of hanging the process.
constexpr int kWaitTimeoutCode = 30;
#ifndef EIGENID_WAIT_TIMEOUT_CYCLES
#define EIGENID_WAIT_TIMEOUT_CYCLES 30000000000LL  // ~15 s at 1.9 GHz
#endif
constexpr long long kWaitTimeoutCycles = EIGENID_WAIT_TIMEOUT_CYCLES;
__device__ __noinline__ void wait_timed_out(DevStatus* st, int site) {
  set_status(st, kWaitTimeoutCode, site, 0.0, blockIdx.x * 1000 + (threadIdx.x >> 5));
}
// Blocks until the barrier phase of the given parity has completed.  `site`
// names the wait in the timeout report; once any wait of the call has timed
// out, the others return at once so that the kernel unwinds.
// kSleepNs > 0: back off between polls (a try_wait that fails returns after
// ~100 cycles, so a waiting copy warp polls ~15 M times per second).
template <int kSleepNs = 0>
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity,
                                          DevStatus* st, int site) {
  const unsigned a = (unsigned)__cvta_generic_to_shared(bar);
  unsigned done = 0, spins = 0;
  long long t0 = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
    if (kSleepNs > 0 && !done) __nanosleep(kSleepNs);
    if (!done && ((++spins) & 0xffu) == 0) {
      if (*(volatile const int*)&st->code == kWaitTimeoutCode) return;
      const long long now = clock64();
      if (t0 == 0) {
        t0 = now;
      } else if (now - t0 > kWaitTimeoutCycles) {
        wait_timed_out(st, site);
        return;
      }
    }
  }
}

// Arrival on an mbarrier triggered by the completion of every cp.async this
// thread has issued so far (.noinc: it counts against the expected arrivals).
__device__ __forceinline__ void cpa_mbar_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_inval(unsigned long long* bar) {
  asm volatile("mbarrier.inval.shared::cta.b64 [%0];\n" ::"r"(
                   (unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}

// EIGENID_PIPE_MBAR: the fused pass's stage pipeline runs on mbarriers
// instead of cp.async groups + a CTA barrier per tile.  "full[b]" (one
// arrival per thread, triggered by the completion of its copies) tells a
// warp that stage b holds its tile; "empty[b]" (one arrival per warp after
// its transposed product) tells the copy issue that every warp is done with
// stage b.  A warp that finishes a tile early starts the next tile's update
// at once (it needs only data, not the other warps), and the next stage's
// copies are issued after the update, when the stage they overwrite has long
// been released: the only CTA-wide rendezvous left in a tile is the mid-tile
// "C rows complete" mbarrier.
#ifndef EIGENID_PIPE_MBAR
#define EIGENID_PIPE_MBAR 1
#endif
#ifndef EIGENID_ISSUE_POINT
#define EIGENID_ISSUE_POINT 0
#endif
static_assert(!EIGENID_PIPE_MBAR || EIGENID_SPLIT_BAR, "pipe");

// Row blocks of the fused pass are aligned to the END of the trailing matrix
// (rounded up to a whole 32-column tile, so block starts stay multiples of 32
// and a row block still crosses the diagonal in four tiles): the short block
// is the FIRST one (rows fused_rb0 .. < 0 do not exist and are zero-filled /
// skipped through row_ok), where it costs the few tiles up to the diagonal,
// instead of the last one, where it would cost a full row of tiles (on average
// 49 of 128 rows idle: 3.5 % of the DMMAs at n = 4096).
__device__ __forceinline__ int fused_rb0(int sn) {
  const int end = (sn + kG2N - 1) / kG2N * kG2N;
  return -((kG2M - end % kG2M) % kG2M);
}
__device__ __forceinline__ bool row_ok(int r, int sn) { return (unsigned)r < (unsigned)sn; }

#if !EIGENID_STAGE1_SP
__device__ void gemm_fused(double* A22n, int ldw, int sn, const double* W2p,
                           const double* Vp, const double* VTn, double* Xn,
                           double* sm, DevStatus* status) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kk = lane & 3, mm = lane >> 2;
  // this lane's rows within the row block: crow0 + 8 mt, mt < kRW
  const int crow0 = 8 * kRW * warp + mm;
  double* sVr = sm + kFS * kFSt;
#if EIGENID_SPLIT_BAR
  // "every warp's updated C rows are in shared memory": one arrival per warp
  // per tile, phases alternate tile by tile
  __shared__ alignas(8) unsigned long long cbar_storage;
  unsigned long long* cbar = &cbar_storage;
  unsigned cphase = 0;
#if EIGENID_PIPE_MBAR
  __shared__ alignas(8) unsigned long long pbar_storage[2 * kFS];  // full[], empty[]
  unsigned long long* const fullb = pbar_storage;
  unsigned long long* const emptyb = pbar_storage + kFS;
  unsigned fbits = 0;  // bit b: parity of the next phase to wait for on full[b]
  unsigned ebits = 0;  // bit b: phases begun on empty[b] (mod 2)
  if (tid == 0) {
    for (int b = 0; b < kFS; ++b) {
      mbar_init(fullb + b, kNT);
      mbar_init(emptyb + b, kNW);
    }
  }
#endif
  if (tid == 0) mbar_init(cbar, kNW);
  __syncthreads();
#endif
  for (int rb = fused_rb0(sn); rb < sn; rb += kG2M) {
    double2 af[kRW][kG2K / 8];
#pragma unroll
    for (int mt = 0; mt < kRW; ++mt) {
      const int r = rb + crow0 + 8 * mt;
#pragma unroll
      for (int q = 0; q < kG2K / 8; ++q) {
        const int k = 8 * q + 2 * kk;
        double2 v = make_double2(0.0, 0.0);
        if (row_ok(r, sn))
          v = *reinterpret_cast<const double2*>(k < kB ? W2p + (long long)r * kB + k
                                                       : Vp + (long long)r * kB + (k - kB));
        af[mt][q] = make_double2(-v.x, -v.y);
      }
    }
    double xr[kRW][kG2N / 8][2];
#pragma unroll
    for (int mt = 0; mt < kRW; ++mt)
#pragma unroll
      for (int nt = 0; nt < kG2N / 8; ++nt) xr[mt][nt][0] = xr[mt][nt][1] = 0.0;
    const int cend = min(rb + kG2M, sn);
    const int ncb = (cend + kG2N - 1) / kG2N;
    auto stage = [&](int ci) {
      if (ci < ncb) {
        const int cb = ci * kG2N;
        double* st = sm + (ci % kFS) * kFSt;
        for (int t = tid; t < kG2N * (kG2K / 2); t += kNT) {
          const int row = t >> 5, k2 = (t & 31) * 2;
          const int gr = cb + row;
          const int bytes = row_ok(gr, sn) ? 16 : 0;
          const long long g = (long long)(bytes ? gr : 0) * kB;
          const double* src = k2 < kB ? Vp + g + k2 : W2p + g + (k2 - kB);
          cp_async16(st + row * kG2K + (k2 ^ (8 * (row & 1))), src, bytes);
        }
        double* cs = st + kG2N * kG2K;
        for (int t = tid; t < kG2M * (kG2N / 2); t += kNT) {
          const int row = t >> 4, c2 = (t & 15) * 2;
          const int gr = rb + row, gc = cb + c2;
          int bytes = 0;
          if (row_ok(gr, sn) && gc < sn) bytes = gc + 1 < sn ? 16 : 8;
          cp_async16(cs + cswz(row, c2), bytes ? A22n + (long long)gr * ldw + gc : A22n,
                     bytes);
        }
        double* vc = cs + kG2M * kG2N;
        for (int t = tid; t < kB * (kB / 2); t += kNT) {
          const int row = t >> 4, c2 = (t & 15) * 2;
          const int gr = cb + row;
          const int bytes = row_ok(gr, sn) ? 16 : 0;
          cp_async16(vc + row * kFVLD + c2, VTn + (long long)(bytes ? gr : 0) * kB + c2,
                     bytes);
        }
#if EIGENID_PIPE_MBAR
        cpa_mbar_arrive(fullb + (ci % kFS));
#endif
      }
#if !EIGENID_PIPE_MBAR
      cpa_commit();
#endif
    };
    // Interior row blocks (every row and column of every tile in range: all
    // but the last partial block): each thread's copies of a tile sit at
    // fixed offsets from three pointers that advance by one tile, so a stage
    // is a handful of unpredicated cp.async off immediate offsets instead of
    // ~230 instructions of index and predicate arithmetic.
    const bool interior = rb >= 0 && rb + kG2M <= sn;
    auto stage_fast = [&](int ci) {
      if (ci < ncb) {
        constexpr int kBopIt = kG2N * (kG2K / 2) / kNT, kBopRows = kNT / 32;
        constexpr int kCIt = kG2M * (kG2N / 2) / kNT, kCRows = kNT / 16;
        constexpr int kVIt = kB * (kB / 2) / kNT;
        static_assert(kBopRows % 2 == 0 && kCRows % 4 == 0, "swizzle terms must not change");
        double* st = sm + (ci % kFS) * kFSt;
        const long long off = (long long)ci * (kG2N * kB);  // cb * kB
        const int brow = tid >> 5, bk2 = (tid & 31) * 2;
        const double* bsrc =
            (bk2 < kB ? Vp + bk2 : W2p + (bk2 - kB)) + off + (long long)brow * kB;
        double* bdst = st + brow * kG2K + (bk2 ^ (8 * (brow & 1)));
#pragma unroll
        for (int i = 0; i < kBopIt; ++i)
          cp_async16_full(bdst + i * kBopRows * kG2K, bsrc + i * kBopRows * kB);
        const int crw = tid >> 4, cc2 = (tid & 15) * 2;
        const double* csrc = A22n + (long long)(rb + crw) * ldw + ci * kG2N + cc2;
        double* cdst = st + kG2N * kG2K + cswz(crw, cc2);
#pragma unroll
        for (int i = 0; i < kCIt; ++i)
          cp_async16_full(cdst + i * kCRows * kG2N, csrc + (long long)i * kCRows * ldw);
        const double* vsrc = VTn + off + (long long)crw * kB + cc2;
        double* vdst = st + kG2N * kG2K + kG2M * kG2N + crw * kFVLD + cc2;
#pragma unroll
        for (int i = 0; i < kVIt; ++i)
          cp_async16_full(vdst + i * kCRows * kFVLD, vsrc + i * kCRows * kB);
#if EIGENID_PIPE_MBAR
        cpa_mbar_arrive(fullb + (ci % kFS));
#endif
      }
#if !EIGENID_PIPE_MBAR
      cpa_commit();
#endif
    };
    __syncthreads();  // the previous row block is done with every buffer
    for (int t = tid; t < kG2M * (kB / 2); t += kNT) {
      const int row = t >> 4, c2 = (t & 15) * 2;
      const int gr = rb + row;
      const int bytes = row_ok(gr, sn) ? 16 : 0;
      cp_async16(sVr + row * kFVRLD + c2, VTn + (long long)(bytes ? gr : 0) * kB + c2,
                 bytes);
    }
#pragma unroll
    for (int p = 0; p < kFS - 1; ++p) {
      if (EIGENID_FAST_STAGE && interior)
        stage_fast(p);
      else
        stage(p);
    }
    // Tile body, specialised on whether the tile may cross the diagonal
    // (only then are the triangular masks needed).
    auto tile = [&](int ci, auto diag_tag) {
      constexpr bool diag = decltype(diag_tag)::value;
      const int cb = ci * kG2N;
      const double* b = sm + (ci % kFS) * kFSt;
      double* cs = const_cast<double*>(b) + kG2N * kG2K;
      const double* vc = cs + kG2M * kG2N;
      // X[cb] block of this warp for the transposed product below, loaded
      // early so the read overlaps the rank-2kB update
      const int mt2 = warp / (4 / kXT), nb = (warp % (4 / kXT)) * kXT;
      const int xrow = cb + 8 * mt2 + mm;
      double x2[kXT][2];
#pragma unroll
      for (int u = 0; u < kXT; ++u) {
        const int xc = 8 * (nb + u) + 2 * kk;
        if (xrow < sn) {
          double2 t;
          asm volatile("ld.global.v2.f64 {%0, %1}, [%2];\n"
                       : "=d"(t.x), "=d"(t.y)
                       : "l"(Xn + (long long)xrow * kB + xc));
          x2[u][0] = t.x;
          x2[u][1] = t.y;
        } else {
          x2[u][0] = x2[u][1] = 0.0;
        }
      }
      // A diagonal-crossing tile's rows above the diagonal (tile rows < d =
      // cb - rb) hold only upper-triangle elements, which nothing reads: an
      // 8-row group that lies wholly there skips its update and row product
      // (their contributions are exact zeros), and the transposed product
      // below starts at contraction row d.
      const int dskip = (EIGENID_DIAG_SKIP && diag) ? cb - rb : 0;
      bool live[kRW];
#pragma unroll
      for (int mt = 0; mt < kRW; ++mt)
        live[mt] = !diag || 8 * kRW * warp + 8 * mt + 7 >= dskip;
      // ---- rank-2kB update of this lane's C rows
      double acc[kRW][kG2N / 8][2];
#pragma unroll
      for (int mt = 0; mt < kRW; ++mt) {
        if (!live[mt]) continue;
#pragma unroll
        for (int nt = 0; nt < kG2N / 8; ++nt) {
          const double2 x = *reinterpret_cast<const double2*>(
              cs + cswz(crow0 + 8 * mt, 8 * nt + 2 * kk));
          acc[mt][nt][0] = x.x;
          acc[mt][nt][1] = x.y;
        }
      }
#pragma unroll
      for (int q = 0; q < kG2K / 8; ++q) {
        const int kl = (8 * q + 2 * kk) ^ (8 * (mm & 1));
        double2 bf[kG2N / 8];
#pragma unroll
        for (int nt = 0; nt < kG2N / 8; ++nt)
          bf[nt] = *reinterpret_cast<const double2*>(b + (8 * nt + mm) * kG2K + kl);
        // independent accumulators back to back
#pragma unroll
        for (int mt = 0; mt < kRW; ++mt) {
          if (!live[mt]) continue;
#pragma unroll
          for (int nt = 0; nt < kG2N / 8; ++nt)
            dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt][q].x, bf[nt].x);
        }
#pragma unroll
        for (int mt = 0; mt < kRW; ++mt) {
          if (!live[mt]) continue;
#pragma unroll
          for (int nt = 0; nt < kG2N / 8; ++nt)
            dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt][q].y, bf[nt].y);
        }
      }
      // updated C rows to shared memory for the transposed product
      auto store_smem = [&]() {
#pragma unroll
        for (int mt = 0; mt < kRW; ++mt) {
          if (!live[mt]) continue;
#pragma unroll
          for (int nt = 0; nt < kG2N / 8; ++nt)
            *reinterpret_cast<double2*>(cs + cswz(crow0 + 8 * mt, 8 * nt + 2 * kk)) =
                make_double2(acc[mt][nt][0], acc[mt][nt][1]);
        }
      };
#if EIGENID_SPLIT_BAR
      // store first, then arrive (non-blocking) on the "C tile complete"
      // mbarrier (one arrival per warp), and run this warp's independent row
      // product before waiting for the others: the DMMA pipe is fed across
      // the barrier instead of draining at it
      store_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(cbar);
#if EIGENID_PIPE_MBAR
      // copies of tile ci + kFS - 1: the stage they overwrite held tile ci-1,
      // released by every warp after its transposed product (long ago by now)
      auto issue_next = [&]() {
        if (ci + kFS - 1 < ncb) {
          const int nb2 = (ci + kFS - 1) % kFS;
          if (ci >= 1) mbar_wait(emptyb + nb2, ((ebits >> nb2) & 1u) ^ 1u, status, 1);
          if (EIGENID_FAST_STAGE && interior)
            stage_fast(ci + kFS - 1);
          else
            stage(ci + kFS - 1);
        }
      };
      // EIGENID_ISSUE_POINT: 0 = here (before the row product), 1 = after the
      // row product, 2 = half of the warps of each SM sub-partition at each
      const bool issue_early = EIGENID_ISSUE_POINT == 0 ||
                               (EIGENID_ISSUE_POINT == 2 && ((warp >> 2) & 1) == 0);
      if (issue_early) issue_next();
#endif
#endif
      // ---- X[rb] += tril(C) VTn[cb] straight from the accumulators: the
      // m8n8k4 accumulator of column tile q holds C[row][8q+2kk .. +1], which
      // is exactly this lane's A-fragment pair for k-pair q (no shared-memory
      // round trip, no barrier)
#pragma unroll
      for (int q = 0; q < kB / 8; ++q) {
        const int k = 8 * q + 2 * kk;
        double b0[kG2N / 8], b1[kG2N / 8];
#pragma unroll
        for (int nt = 0; nt < kG2N / 8; ++nt) {
          b0[nt] = vc[k * kFVLD + 8 * nt + mm];
          b1[nt] = vc[(k + 1) * kFVLD + 8 * nt + mm];
        }
#pragma unroll
        for (int mt = 0; mt < kRW; ++mt) {
          if (!live[mt]) continue;
          const int r = rb + crow0 + 8 * mt;
          const double ax = (diag && cb + k > r) ? 0.0 : acc[mt][q][0];
          const double ay = (diag && cb + k + 1 > r) ? 0.0 : acc[mt][q][1];
#pragma unroll
          for (int nt = 0; nt < kG2N / 8; ++nt) dmma(xr[mt][nt][0], xr[mt][nt][1], ax, b0[nt]);
#pragma unroll
          for (int nt = 0; nt < kG2N / 8; ++nt) dmma(xr[mt][nt][0], xr[mt][nt][1], ay, b1[nt]);
        }
      }
      if (EIGENID_FAST_STORE && interior) {  // every row and column in range
#pragma unroll
        for (int mt = 0; mt < kRW; ++mt) {
          if (!live[mt]) continue;
          double* p = A22n + (long long)(rb + crow0 + 8 * mt) * ldw + cb + 2 * kk;
#pragma unroll
          for (int nt = 0; nt < kG2N / 8; ++nt)
            *reinterpret_cast<double2*>(p + 8 * nt) =
                make_double2(acc[mt][nt][0], acc[mt][nt][1]);
        }
      } else {
#pragma unroll
        for (int mt = 0; mt < kRW; ++mt) {
          if (!live[mt]) continue;
          const int r = rb + crow0 + 8 * mt;
#pragma unroll
          for (int nt = 0; nt < kG2N / 8; ++nt) {
            const int col = cb + 8 * nt + 2 * kk;
            if (row_ok(r, sn)) {
              double* p = A22n + (long long)r * ldw + col;
              if (col + 1 < sn)
                *reinterpret_cast<double2*>(p) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
              else if (col < sn)
                p[0] = acc[mt][nt][0];
            }
          }
        }
      }
#if EIGENID_PIPE_MBAR
      if (!issue_early) issue_next();
#endif
#if EIGENID_SPLIT_BAR
#ifndef EIGENID_EXP_NO_CBAR
      mbar_wait(cbar, cphase, status, 2);
#endif
      cphase ^= 1u;
#else
      store_smem();
      __syncthreads();
#endif
      // ---- X[cb] += strict(C)^T VTn[rb]   (warp: X rows 8*mt2.., 8*kXT cols)
#ifndef EIGENID_EXP_NO_XT
      {
        const int ccol = 8 * mt2 + mm;  // tile column of C = X row
#pragma unroll 4
        for (int k4 = dskip / 4; k4 < kG2M / 4; ++k4) {
          const int krow = 4 * k4 + kk;  // tile row of C = contraction index
          const double v = cs[cswz(krow, ccol)];
          const double a = (diag && rb + krow <= cb + ccol) ? 0.0 : v;
#pragma unroll
          for (int u = 0; u < kXT; ++u)
            dmma(x2[u][0], x2[u][1], a, sVr[krow * kFVRLD + 8 * (nb + u) + mm]);
        }
        if (xrow < sn) {
#pragma unroll
          for (int u = 0; u < kXT; ++u)
            *reinterpret_cast<double2*>(Xn + (long long)xrow * kB + 8 * (nb + u) + 2 * kk) =
                make_double2(x2[u][0], x2[u][1]);
        }
      }
#endif
#if EIGENID_PIPE_MBAR
      __syncwarp();
      if (lane == 0) mbar_arrive(emptyb + (ci % kFS));
      ebits ^= 1u << (ci % kFS);
#endif
    };
    for (int ci = 0; ci < ncb; ++ci) {
#if EIGENID_PIPE_MBAR
      mbar_wait(fullb + (ci % kFS), (fbits >> (ci % kFS)) & 1u, status, 3);
      fbits ^= 1u << (ci % kFS);
#else
      cpa_wait<kFS - 2>();
#ifndef EIGENID_EXP_NO_TILE_SYNC
      __syncthreads();
#endif
      if (EIGENID_FAST_STAGE && interior)
        stage_fast(ci + kFS - 1);
      else
        stage(ci + kFS - 1);
#endif
      if (ci * kG2N + kB > rb)
        tile(ci, std::true_type{});
      else
        tile(ci, std::false_type{});
    }
    // X[rb] += the row-part accumulators (after this row block's transposed
    // contributions to the same rows)
    __syncthreads();
#pragma unroll
    for (int mt = 0; mt < kRW; ++mt) {
      const int r = rb + crow0 + 8 * mt;
      if (row_ok(r, sn)) {
#pragma unroll
        for (int nt = 0; nt < kG2N / 8; ++nt) {
          double2* p = reinterpret_cast<double2*>(Xn + (long long)r * kB + 8 * nt + 2 * kk);
          double2 x = *p;
          x.x += xr[mt][nt][0];
          x.y += xr[mt][nt][1];
          *p = x;
        }
      }
    }
  }
  __syncthreads();
#if EIGENID_SPLIT_BAR
  if (tid == 0) {
    mbar_inval(cbar);
#if EIGENID_PIPE_MBAR
    for (int b = 0; b < 2 * kFS; ++b) mbar_inval(pbar_storage + b);
#endif
  }
#endif
}

#else  // EIGENID_STAGE1_SP
template <int N>
__device__ __forceinline__ void reg_inc() {
  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(N));
}
template <int N>
__device__ __forceinline__ void reg_dec() {
  asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(N));
}
// barrier over the compute warps only
__device__ __forceinline__ void bar_compute() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kCW) : "memory");
}
#ifdef EIGENID_EXP_DROP_ARRIVE
__device__ int g_drop_once = 1;
#endif
#ifndef EIGENID_SP_SKIP0
#define EIGENID_SP_SKIP0 1
#endif
// back-off of the copy warps' polls: measured 1 % SLOWER at 100 / 300 / 1000 ns
// (the copies of tile g+2 go out later), so they poll without sleeping
// order of a tile's copies: the C tile (DRAM) before the Bop rows (mostly L2)
#ifndef EIGENID_SP_C_FIRST
#define EIGENID_SP_C_FIRST 0
#endif
#ifndef EIGENID_SP_COPY_SLEEP_NS
#define EIGENID_SP_COPY_SLEEP_NS 0
#endif
#ifndef EIGENID_SP_SKIP
#define EIGENID_SP_SKIP 0
#endif
#ifndef EIGENID_SP_REGS_COMPUTE
#define EIGENID_SP_REGS_COMPUTE 216
#endif
constexpr int kRegCompute = EIGENID_SP_REGS_COMPUTE;
constexpr int kRegCopy = (65536 - 32 * kCW * kRegCompute) / kPT / 8 * 8;
static_assert(kRegCopy >= 24 && kRegCompute <= 232, "setmaxnreg split");

// Warp-specialised fused pass (same mathematics and accumulation orders as
// the generic one above).  Tiles are numbered g = 0, 1, ... across the row
// blocks of the pass and live in stage g % kFS.
//   copy warps:    wait empty[g % kFS] (tile g - kFS released), issue the
//                  tile's copies, arrive on full[g % kFS] when they land; the
//                  row block's VTn[rb] rows follow its first tile, once the
//                  compute warps are done with the previous row block
//                  (rbdone), and arrive on svr_full.
//   compute warps: wait full, update, arrive cbar, row product, wait cbar,
//                  (first tile: wait svr_full), transposed product, arrive
//                  empty.  Two compute-warp barriers per row block order the
//                  X read-modify-writes.
__device__ void gemm_fused(double* A22n, int ldw, int sn, const double* W2p,
                           const double* Vp, const double* VTn, double* Xn,
                           double* sm, DevStatus* status) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* sVr = sm + kFS * kFSt;
  __shared__ alignas(8) unsigned long long bars[2 * kFS + 3];
  unsigned long long* const fullb = bars;
  unsigned long long* const emptyb = bars + kFS;
  unsigned long long* const cbar = bars + 2 * kFS;
  unsigned long long* const svr_full = cbar + 1;
  unsigned long long* const rbdone = cbar + 2;
  if (tid == 0) {
    for (int b = 0; b < kFS; ++b) {
      mbar_init(fullb + b, kPT);
      mbar_init(emptyb + b, kCW);
    }
    mbar_init(cbar, kCW);
    mbar_init(svr_full, kPT);
    mbar_init(rbdone, kCW);
  }
  __syncthreads();
  if (warp >= kCW) {
    // ------------------------------------------------------- copy warps
    reg_dec<kRegCopy>();
    const int pt = tid - 32 * kCW;
    int g = 0;
    unsigned ebits = 0, rbpar = 0;
    for (int rb = fused_rb0(sn); rb < sn; rb += kG2M) {
      const int cend = min(rb + kG2M, sn);
      const int ncb = (cend + kG2N - 1) / kG2N;
      const bool interior = rb >= 0 && rb + kG2M <= sn;
      for (int ci = 0; ci < ncb; ++ci, ++g) {
        const int sb = g % kFS;
        if (g >= kFS) {
          mbar_wait<EIGENID_SP_COPY_SLEEP_NS>(emptyb + sb, (ebits >> sb) & 1u, status, 4);
          ebits ^= 1u << sb;
        }
        double* st = sm + sb * kFSt;
        const int cb = ci * kG2N;
#ifdef EIGENID_EXP_NO_COPY
        if (false) {
        } else if (false) {
#else
        if (interior) {
#endif
          constexpr int kBopIt = kG2N * (kG2K / 2) / kPT, kBopRows = kPT / 32;
          constexpr int kCIt = kG2M * (kG2N / 2) / kPT, kCRows = kPT / 16;
          constexpr int kVIt = kB * (kB / 2) / kPT;
          static_assert(kBopRows % 2 == 0 && kCRows % 4 == 0, "swizzle terms must not change");
          const long long off = (long long)cb * kB;
#if EIGENID_SP_C_FIRST
          const int crw = pt >> 4, cc2 = (pt & 15) * 2;
          const double* csrc = A22n + (long long)(rb + crw) * ldw + cb + cc2;
          double* cdst = st + kG2N * kG2K + cswz(crw, cc2);
#pragma unroll
          for (int i = 0; i < kCIt; ++i)
            cp_async16_full(cdst + i * kCRows * kG2N, csrc + (long long)i * kCRows * ldw);
          const int brow = pt >> 5, bk2 = (pt & 31) * 2;
          const double* bsrc =
              (bk2 < kB ? Vp + bk2 : W2p + (bk2 - kB)) + off + (long long)brow * kB;
          double* bdst = st + brow * kG2K + (bk2 ^ (8 * (brow & 1)));
#pragma unroll
          for (int i = 0; i < kBopIt; ++i)
            cp_async16_full(bdst + i * kBopRows * kG2K, bsrc + i * kBopRows * kB);
#else
          const int brow = pt >> 5, bk2 = (pt & 31) * 2;
          const double* bsrc =
              (bk2 < kB ? Vp + bk2 : W2p + (bk2 - kB)) + off + (long long)brow * kB;
          double* bdst = st + brow * kG2K + (bk2 ^ (8 * (brow & 1)));
#pragma unroll
          for (int i = 0; i < kBopIt; ++i)
            cp_async16_full(bdst + i * kBopRows * kG2K, bsrc + i * kBopRows * kB);
          const int crw = pt >> 4, cc2 = (pt & 15) * 2;
          const double* csrc = A22n + (long long)(rb + crw) * ldw + cb + cc2;
          double* cdst = st + kG2N * kG2K + cswz(crw, cc2);
#pragma unroll
          for (int i = 0; i < kCIt; ++i)
            cp_async16_full(cdst + i * kCRows * kG2N, csrc + (long long)i * kCRows * ldw);
#endif
          const double* vsrc = VTn + off + (long long)crw * kB + cc2;
          double* vdst = st + kG2N * kG2K + kG2M * kG2N + crw * kFVLD + cc2;
#pragma unroll
          for (int i = 0; i < kVIt; ++i)
            cp_async16_full(vdst + i * kCRows * kFVLD, vsrc + i * kCRows * kB);
        } else
#ifdef EIGENID_EXP_NO_COPY
            if (false)
#endif
        {
          for (int t = pt; t < kG2N * (kG2K / 2); t += kPT) {
            const int row = t >> 5, k2 = (t & 31) * 2;
            const int gr = cb + row;
            const int bytes = row_ok(gr, sn) ? 16 : 0;
            const long long gg = (long long)(bytes ? gr : 0) * kB;
            const double* src = k2 < kB ? Vp + gg + k2 : W2p + gg + (k2 - kB);
            cp_async16(st + row * kG2K + (k2 ^ (8 * (row & 1))), src, bytes);
          }
          double* cs = st + kG2N * kG2K;
          for (int t = pt; t < kG2M * (kG2N / 2); t += kPT) {
            const int row = t >> 4, c2 = (t & 15) * 2;
            const int gr = rb + row, gc = cb + c2;
            int bytes = 0;
            if (row_ok(gr, sn) && gc < sn) bytes = gc + 1 < sn ? 16 : 8;
            cp_async16(cs + cswz(row, c2), bytes ? A22n + (long long)gr * ldw + gc : A22n,
                       bytes);
          }
          double* vc = cs + kG2M * kG2N;
          for (int t = pt; t < kB * (kB / 2); t += kPT) {
            const int row = t >> 4, c2 = (t & 15) * 2;
            const int gr = cb + row;
            const int bytes = row_ok(gr, sn) ? 16 : 0;
            cp_async16(vc + row * kFVLD + c2, VTn + (long long)(bytes ? gr : 0) * kB + c2,
                       bytes);
          }
        }
        cpa_mbar_arrive(fullb + sb);
        if (ci == 0) {
          // VTn[rb] rows: the compute warps must be done with the previous
          // row block's transposed products
          if (rb != fused_rb0(sn)) {
            mbar_wait<EIGENID_SP_COPY_SLEEP_NS>(rbdone, rbpar, status, 5);
            rbpar ^= 1u;
          }
          for (int t = pt; t < kG2M * (kB / 2); t += kPT) {
            const int row = t >> 4, c2 = (t & 15) * 2;
            const int gr = rb + row;
            const int bytes = row_ok(gr, sn) ? 16 : 0;
            cp_async16(sVr + row * kFVRLD + c2, VTn + (long long)(bytes ? gr : 0) * kB + c2,
                       bytes);
          }
          cpa_mbar_arrive(svr_full);
        }
      }
    }
    cpa_wait0();
  } else {
    // ---------------------------------------------------- compute warps
    reg_inc<kRegCompute>();
    const int kk = lane & 3, mm = lane >> 2;
    // 8-row group mt of this warp is group warp + kCW mt of the row block
    // (interleaved, so the dead groups of a diagonal or tail tile are spread
    // evenly over the SM sub-partitions)
    int crow[kRW];
#pragma unroll
    for (int mt = 0; mt < kRW; ++mt) crow[mt] = 8 * (warp + kCW * mt) + mm;
    int g = 0;
    unsigned fbits = 0, cphase = 0, svphase = 0;
    for (int rb = fused_rb0(sn); rb < sn; rb += kG2M) {
      double2 af[kRW][kG2K / 8];
#pragma unroll
      for (int mt = 0; mt < kRW; ++mt) {
        const int r = rb + crow[mt];
#pragma unroll
        for (int q = 0; q < kG2K / 8; ++q) {
          const int k = 8 * q + 2 * kk;
          double2 v = make_double2(0.0, 0.0);
          if (row_ok(r, sn))
            v = *reinterpret_cast<const double2*>(k < kB ? W2p + (long long)r * kB + k
                                                         : Vp + (long long)r * kB + (k - kB));
          af[mt][q] = make_double2(-v.x, -v.y);
        }
      }
      double xr[kRW][kG2N / 8][2];
#pragma unroll
      for (int mt = 0; mt < kRW; ++mt)
#pragma unroll
        for (int nt = 0; nt < kG2N / 8; ++nt) xr[mt][nt][0] = xr[mt][nt][1] = 0.0;
      const int cend = min(rb + kG2M, sn);
      const int ncb = (cend + kG2N - 1) / kG2N;
      const bool interior = rb >= 0 && rb + kG2M <= sn;
      double x2n[kXT][2];
      auto load_x2 = [&](int ci) {
        const int xr0 = ci * kG2N + 8 * (warp / (4 / kXT)) + mm;
#pragma unroll
        for (int u = 0; u < kXT; ++u) {
          const int xc = 8 * ((warp % (4 / kXT)) * kXT + u) + 2 * kk;
#if defined(EIGENID_EXP_NO_XRMW) || defined(EIGENID_EXP_NO_XLOAD)
          if (xr0 < 0) {
#else
          if (xr0 < sn) {
#endif
            double2 t;
            asm volatile("ld.global.v2.f64 {%0, %1}, [%2];\n"
                         : "=d"(t.x), "=d"(t.y)
                         : "l"(Xn + (long long)xr0 * kB + xc));
            x2n[u][0] = t.x;
            x2n[u][1] = t.y;
          } else {
            x2n[u][0] = x2n[u][1] = 0.0;
          }
        }
      };
      load_x2(0);
      // skip0: a diagonal tile whose rows 0..63 (every warp's first 8-row
      // group) lie wholly above the diagonal (d = cb - rb >= 64): that group's
      // update, row product and write-back are compiled out and the
      // transposed product starts at contraction row 64 (all exact zeros
      // otherwise) -- a compile-time variant, no per-tile liveness tests.
      auto tile = [&](int ci, auto diag_tag, auto skip0_tag) {
        constexpr bool diag = decltype(diag_tag)::value;
        constexpr bool skip0 = decltype(skip0_tag)::value;
        static_assert(!skip0 || (diag && kRW == 2 && kG2M == 128), "skip0");
        const int cb = ci * kG2N;
        const int sb = g % kFS;
        const double* b = sm + sb * kFSt;
        double* cs = const_cast<double*>(b) + kG2N * kG2K;
        const double* vc = cs + kG2M * kG2N;
        // X[cb] block of this warp for the transposed product: prefetched
        // one tile ahead (nothing else touches those rows of X during this
        // row block), the first tile's at the top of the row block
        const int mt2 = warp / (4 / kXT), nb = (warp % (4 / kXT)) * kXT;
        const int xrow = cb + 8 * mt2 + mm;
        double x2[kXT][2];
#pragma unroll
        for (int u = 0; u < kXT; ++u) {
          x2[u][0] = x2n[u][0];
          x2[u][1] = x2n[u][1];
        }
        if (ci + 1 < ncb) load_x2(ci + 1);
        mbar_wait(fullb + sb, (fbits >> sb) & 1u, status, 6);
        fbits ^= 1u << sb;
        // Slow-path tiles (diagonal-crossing, or any tile of the last partial
        // row block): an 8-row group wholly above the diagonal (tile rows < d
        // = cb - rb hold only upper-triangle elements, which nothing reads)
        // or wholly past the last row skips its update and row product
        // (exact zeros), and the transposed product runs over the contraction
        // rows [d, rows in range) only.
        const int dskip = (EIGENID_SP_SKIP && EIGENID_SP_SKIP != 3 && diag) ? max(cb - rb, 0) : 0;
        const int kend4 = (EIGENID_SP_SKIP && diag) ? (min(kG2M, sn - rb) + 3) / 4 : kG2M / 4;
        bool live[kRW];
#pragma unroll
        for (int mt = 0; mt < kRW; ++mt)
          live[mt] = !(skip0 && mt == 0) &&
                     (!(EIGENID_SP_SKIP && diag) ||
                      (8 * (warp + kCW * mt) + 7 >= dskip &&
                       row_ok(rb + 8 * (warp + kCW * mt) + 7, sn)));
        // ---- rank-2kB update of this lane's C rows
        double acc[kRW][kG2N / 8][2];
#pragma unroll
        for (int mt = 0; mt < kRW; ++mt) {
          if (skip0 && mt == 0) continue;
#pragma unroll
          for (int nt = 0; nt < kG2N / 8; ++nt) {
            const double2 x = *reinterpret_cast<const double2*>(
                cs + cswz(crow[mt], 8 * nt + 2 * kk));
            acc[mt][nt][0] = x.x;
            acc[mt][nt][1] = x.y;
          }
        }
#pragma unroll
        for (int q = 0; q < kG2K / 8; ++q) {
          const int kl = (8 * q + 2 * kk) ^ (8 * (mm & 1));
          double2 bf[kG2N / 8];
#pragma unroll
          for (int nt = 0; nt < kG2N / 8; ++nt)
            bf[nt] = *reinterpret_cast<const double2*>(b + (8 * nt + mm) * kG2K + kl);
#pragma unroll
          for (int mt = 0; mt < kRW; ++mt) {
            if (!live[mt]) continue;
#pragma unroll
            for (int nt = 0; nt < kG2N / 8; ++nt)
              dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt][q].x, bf[nt].x);
          }
#pragma unroll
          for (int mt = 0; mt < kRW; ++mt) {
            if (!live[mt]) continue;
#pragma unroll
            for (int nt = 0; nt < kG2N / 8; ++nt)
              dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt][q].y, bf[nt].y);
          }
        }
        // updated C rows to shared memory, arrive, row product, then wait
#pragma unroll
        for (int mt = 0; mt < kRW; ++mt) {
          if (skip0 && mt == 0) continue;
#pragma unroll
          for (int nt = 0; nt < kG2N / 8; ++nt)
            *reinterpret_cast<double2*>(cs + cswz(crow[mt], 8 * nt + 2 * kk)) =
                make_double2(acc[mt][nt][0], acc[mt][nt][1]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(cbar);
        // ---- X[rb] += tril(C) VTn[cb] straight from the accumulators
#pragma unroll
        for (int q = 0; q < kB / 8; ++q) {
          const int k = 8 * q + 2 * kk;
          double b0[kG2N / 8], b1[kG2N / 8];
#pragma unroll
          for (int nt = 0; nt < kG2N / 8; ++nt) {
            b0[nt] = vc[k * kFVLD + 8 * nt + mm];
            b1[nt] = vc[(k + 1) * kFVLD + 8 * nt + mm];
          }
#pragma unroll
          for (int mt = 0; mt < kRW; ++mt) {
            if (!live[mt]) continue;
            const int r = rb + crow[mt];
            const double ax = (diag && cb + k > r) ? 0.0 : acc[mt][q][0];
            const double ay = (diag && cb + k + 1 > r) ? 0.0 : acc[mt][q][1];
#pragma unroll
            for (int nt = 0; nt < kG2N / 8; ++nt)
              dmma(xr[mt][nt][0], xr[mt][nt][1], ax, b0[nt]);
#pragma unroll
            for (int nt = 0; nt < kG2N / 8; ++nt)
              dmma(xr[mt][nt][0], xr[mt][nt][1], ay, b1[nt]);
          }
        }
#ifdef EIGENID_EXP_NO_STORE
        if (sn < 0) {
#else
        if (EIGENID_FAST_STORE && interior) {  // every row and column in range
#endif
#pragma unroll
          for (int mt = 0; mt < kRW; ++mt) {
            if (skip0 && mt == 0) continue;
            double* p = A22n + (long long)(rb + crow[mt]) * ldw + cb + 2 * kk;
#pragma unroll
            for (int nt = 0; nt < kG2N / 8; ++nt)
              *reinterpret_cast<double2*>(p + 8 * nt) =
                  make_double2(acc[mt][nt][0], acc[mt][nt][1]);
          }
        } else {
#pragma unroll
          for (int mt = 0; mt < kRW; ++mt) {
            if (skip0 && mt == 0) continue;
            const int r = rb + crow[mt];
#pragma unroll
            for (int nt = 0; nt < kG2N / 8; ++nt) {
              const int col = cb + 8 * nt + 2 * kk;
              if (row_ok(r, sn)) {
                double* p = A22n + (long long)r * ldw + col;
                if (col + 1 < sn)
                  *reinterpret_cast<double2*>(p) = make_double2(acc[mt][nt][0], acc[mt][nt][1]);
                else if (col < sn)
                  p[0] = acc[mt][nt][0];
              }
            }
          }
        }
        mbar_wait(cbar, cphase, status, 7);
        cphase ^= 1u;
        if (ci == 0) {  // this row block's VTn[rb] rows have landed
          mbar_wait(svr_full, svphase, status, 8);
          svphase ^= 1u;
        }
        // ---- X[cb] += strict(C)^T VTn[rb]
        {
          const int ccol = 8 * mt2 + mm;
#pragma unroll 4
          for (int k4 = skip0 ? kG2M / 8 : dskip / 4; k4 < kend4; ++k4) {
            const int krow = 4 * k4 + kk;
            const double v = cs[cswz(krow, ccol)];
            const double a = (diag && rb + krow <= cb + ccol) ? 0.0 : v;
#pragma unroll
            for (int u = 0; u < kXT; ++u)
              dmma(x2[u][0], x2[u][1], a, sVr[krow * kFVRLD + 8 * (nb + u) + mm]);
          }
#if defined(EIGENID_EXP_NO_XRMW) || defined(EIGENID_EXP_NO_XSTORE)
          if (xrow < 0) {
#else
          if (xrow < sn) {
#endif
#pragma unroll
            for (int u = 0; u < kXT; ++u)
              *reinterpret_cast<double2*>(Xn + (long long)xrow * kB + 8 * (nb + u) + 2 * kk) =
                  make_double2(x2[u][0], x2[u][1]);
          }
        }
        __syncwarp();
#ifdef EIGENID_EXP_DROP_ARRIVE  // test hook: lose ONE arrival; the waits must time out
        if (lane == 0 && !(blockIdx.x == 3 && warp == 2 && g == 7 && sn < 3000 &&
                           atomicExch(&g_drop_once, 0)))
          mbar_arrive(emptyb + sb);
#else
        if (lane == 0) mbar_arrive(emptyb + sb);
#endif
        ++g;
      };
      for (int ci = 0; ci < ncb; ++ci) {
        // EIGENID_SP_SKIP: 1 = diagonal and tail tiles, 2 = diagonal tiles
        // only, 3 = tail row blocks only (timing experiments)
        if (EIGENID_SP_SKIP0 && ci * kG2N - rb >= kG2M / 2)
          tile(ci, std::true_type{}, std::true_type{});
        else if (ci * kG2N + kB > rb || ((EIGENID_SP_SKIP & 1) && !interior))
          tile(ci, std::true_type{}, std::false_type{});
        else
          tile(ci, std::false_type{}, std::false_type{});
      }
      // the copy warps may now overwrite VTn[rb]
      __syncwarp();
      if (lane == 0) mbar_arrive(rbdone);
      // X[rb] += the row-part accumulators, after this row block's transposed
      // contributions to the same rows and before the next row block's
      bar_compute();
#pragma unroll
      for (int mt = 0; mt < kRW; ++mt) {
        const int r = rb + crow[mt];
        if (row_ok(r, sn)) {
#pragma unroll
          for (int nt = 0; nt < kG2N / 8; ++nt) {
            double2* p = reinterpret_cast<double2*>(Xn + (long long)r * kB + 8 * nt + 2 * kk);
            double2 x = *p;
            x.x += xr[mt][nt][0];
            x.y += xr[mt][nt][1];
            *p = x;
          }
        }
      }
      bar_compute();
    }
    reg_dec<128>();
  }
  if (warp >= kCW) reg_inc<128>();
#ifndef EIGENID_SP_NO_MERGE_DEC
  reg_dec<128>();  // every warp is back at 128: tell the register allocator so
#endif
  __syncthreads();
  if (tid == 0)
    for (int b = 0; b < 2 * kFS + 3; ++b) mbar_inval(bars + b);
}
#endif  // EIGENID_STAGE1_SP

__device__ void write_band(const double* W, int ldw, int m, int c_begin,
                           int c_end, double* band) {
  for (int t = threadIdx.x; t < (c_end - c_begin) * kLDAB; t += kNT) {
    const int col = c_begin + t / kLDAB, d = t % kLDAB;
    double v = 0.0;
    if (d <= kB && col + d < m) v = W[(long long)(col + d) * ldw + col];
    band[(long long)col * kLDAB + d] = v;
  }
}

#ifdef EIGENID_PHASE_TIMING
__device__ unsigned long long g_cta_span[1536];  // per-CTA start, end, SM id
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
#define PHASE(id)                                                         \
  do {                                                                    \
    __syncthreads();                                                      \
    const long long now_ = clock64();                                     \
    if (threadIdx.x == 0)                              \
      atomicAdd(&g_phase_cycles[ph_], (unsigned long long)(now_ - t_ph_)); \
    t_ph_ = now_;                                                         \
    ph_ = (id);                                                           \
  } while (0)
#else
#define PHASE(id) \
  do {            \
  } while (0)
#endif

__global__ void __launch_bounds__(kNT, kCtasPerSm) band_reduce_kernel(Stage1Args args) {
#ifdef EIGENID_PHASE_TIMING
  long long t_ph_ = clock64();
  int ph_ = 0;
  if (threadIdx.x == 0 && blockIdx.x < 512) {
    unsigned smid;
    asm volatile("mov.u32 %0, %smid;" : "=r"(smid));
    g_cta_span[2 * blockIdx.x] = gtimer();
    g_cta_span[1024 + blockIdx.x] = smid;
  }
#endif
  extern __shared__ double smem[];
  double* sgemm = smem;
  double* sG = smem + kGemmSmem;  // G, then Y
  double* sA = sG + kSmallMat;
  double* sT = sA + kSmallMat;
  double* sM = sA;               // M = T^T Y (A is dead by then)
  double* sB = sgemm;            // only alive between gram()/GEMM calls
  double* sR = sgemm + kSmallMat;
  double* red = sT + kSmallMat;
  double* stau = red + kRed;
  double* wsm = stau + kB;
  double* sS = wsm + kB;
  int* sflag = reinterpret_cast<int*>(sS + kB);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = args.n, ldw = args.ldw;
  // slot workspace: the minor (n x ldw), then V and X (= W2) for two panels
  // and VT, n x kB each (stage1_ws_doubles)
  double* W = args.ws + (long long)(args.slot0 + blockIdx.x) * args.ws_stride;
  double* const Vg[2] = {W + (long long)n * ldw, W + (long long)n * ldw + (long long)n * kB};
  double* const Xg[2] = {W + (long long)n * ldw + 2LL * n * kB,
                         W + (long long)n * ldw + 3LL * n * kB};
  double* VTg = W + (long long)n * ldw + 4LL * n * kB;

  // Solves are pulled from a work queue: the two CTAs sharing an SM do not
  // progress at the same rate, so a static blockIdx stride leaves one of
  // them running alone at the end of every wave.
  __shared__ int s_sidx;
  if (args.running) {
    if (!args.helper) {
      if (blockIdx.x == 0 && tid == 0) atomicExch(args.running, 1);
    } else if (*(volatile int*)args.running == 0) {
      return;  // the main grid is not running beside us (serialised launches)
    }
  }
  for (;;) {
    // a failed call (non-finite input, degenerate lambda(A)) stops pulling
    if (tid == 0)
      s_sidx = *(volatile const int*)&args.status->code ? args.nsolves
                                                        : atomicAdd(args.counter, 1);
    __syncthreads();
    const int sidx = s_sidx;
    __syncthreads();
    if (sidx >= args.nsolves) break;
    const int j = args.js[sidx];
    const int m = j < 0 ? n : n - 1;
    double* band = args.band + sidx * args.band_stride;
    PHASE(1);
    // materialise the lower triangle of the minor (r' = r + (r >= j)),
    // times the exact power-of-two input scale
    const double in_sc = args.scale ? args.scale[0] : 1.0;
    for (int r = warp; r < m; r += kNT / 32) {
      const int rr = (j >= 0 && r >= j) ? r + 1 : r;
      const double* src = args.A + (long long)rr * n;
      double* dst = W + (long long)r * ldw;
      for (int c0 = lane; c0 <= r; c0 += 512) {
        double v[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int cc = c0 + 32 * u;
          v[u] = cc <= r ? src[(j >= 0 && cc >= j) ? cc + 1 : cc] * in_sc : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (c0 + 32 * u <= r) dst[c0 + 32 * u] = v[u];
      }
    }
    __syncthreads();
    // Panel factorisation of columns c..c+kB-1 (trailing size s): V (Vb),
    // T (sT), the band columns, VT = V T; Xb is scratch.
    auto factor = [&](int c, int s, double* Vb, double* Xb) {
      double* P0 = W + (long long)(c + kB) * ldw + c;
      PHASE(2);
      const bool fast = s >= 2 * kB &&
                        chol_panel(P0, ldw, s, Vb, Xb, sT, sG, sA, sB, sR, sS,
                                   sgemm, sflag);
      if (!fast) {
#ifdef EIGENID_PHASE_TIMING
        if (tid == 0) atomicAdd(&g_phase_cycles[15], 1ull);
#endif
        panel_qr(P0, ldw, s, stau, red, wsm);
        extract_v(P0, ldw, s, Vb);
        // T (dlarft, forward columnwise) from G = V^T V
        gram(Vb, kB, Vb, kB, s, sG, sgemm);
        if (warp == 0) {
          for (int t = 0; t < kB; ++t) {
            double v = 0.0;
            if (lane < t)
              for (int p = lane; p < t; ++p) v += sT[lane * kSmallLD + p] * sG[p * kSmallLD + t];
            __syncwarp();
            if (lane < t) sT[lane * kSmallLD + t] = -stau[t] * v;
            if (lane == t) sT[t * kSmallLD + t] = stau[t];
            if (lane > t) sT[lane * kSmallLD + t] = 0.0;
            __syncwarp();
          }
        }
      }
      __syncthreads();
      PHASE(3);
      write_band(W, ldw, m, c, c + kB, band);
      row_transform(Vb, kB, sT, 1.0, nullptr, VTg, s);        // VT = V T
    };
    // W2 = X - V M/2 with M = T^T (V^T X), in place in Xb.
    auto form_w2 = [&](int s, const double* Vb, double* Xb) {
      PHASE(5);
      gram(Vb, kB, Xb, kB, s, sG, sgemm);                     // Y = V^T X
      for (int t = tid; t < kB * kB; t += kNT) {              // M = T^T Y
        const int q = t / kB, p = t % kB;
        double v = 0.0;
        for (int u = 0; u <= q; ++u) v += sT[u * kSmallLD + q] * sG[u * kSmallLD + p];
        sM[q * kSmallLD + p] = v;
      }
      __syncthreads();
      row_transform(Vb, kB, sM, -0.5, Xb, Xb, s);
    };
    int c = 0;
#if EIGENID_STAGE1_FUSED
    // Look-ahead schedule: panel p+1's columns are updated and factored
    // first, then one fused pass applies the rest of panel p's update and
    // forms X of panel p+1 (gemm_fused).
    if (m - kB >= 2) {
      int par = 0;
      factor(0, m - kB, Vg[0], Xg[0]);
      PHASE(7);
      gemm1(W + (long long)kB * ldw + kB, ldw, m - kB, VTg, Xg[0], sgemm);
      form_w2(m - kB, Vg[0], Xg[0]);
      for (;;) {
        const int s = m - c - kB;
        double* A22 = W + (long long)(c + kB) * ldw + (c + kB);
        const int s1 = s - kB;
        PHASE(6);
        if (s1 < 2) {
          gemm2(A22, ldw, s, Xg[par], Vg[par], sgemm);         // last update
          PHASE(0);
          c += kB;
          break;
        }
#ifndef EIGENID_OLD_UPDATE_COLS
        update_cols(A22, ldw, s, Xg[par], Vg[par], sgemm);     // next panel's columns
#else
        gemm2(A22, ldw, s, Xg[par], Vg[par], sgemm, 1);
#endif
        const int nxt = par ^ 1;
        factor(c + kB, s1, Vg[nxt], Xg[nxt]);
        for (int t = tid; t < s1 * kB; t += kNT) Xg[nxt][t] = 0.0;
        __syncthreads();
        PHASE(4);
        gemm_fused(A22 + (long long)kB * ldw + kB, ldw, s1, Xg[par] + kB * kB,
                   Vg[par] + kB * kB, VTg, Xg[nxt], sgemm, args.status);
        form_w2(s1, Vg[nxt], Xg[nxt]);
        c += kB;
        par = nxt;
      }
    }
#else
    for (; c < m; c += kB) {
      const int s = m - c - kB;
      if (s < 2) break;
      factor(c, s, Vg[0], Xg[0]);
      double* A22 = W + (long long)(c + kB) * ldw + (c + kB);
      PHASE(4);
      gemm1(A22, ldw, s, VTg, Xg[0], sgemm);                   // X = A22 VT
      form_w2(s, Vg[0], Xg[0]);
      PHASE(6);
      gemm2(A22, ldw, s, Xg[0], Vg[0], sgemm);                 // A22 -= W2V^T+VW2^T
      PHASE(7);
    }
#endif
    write_band(W, ldw, m, c, m, band);
    __syncthreads();
  }
  PHASE(0);
#ifdef EIGENID_PHASE_TIMING
  if (threadIdx.x == 0 && blockIdx.x < 512) g_cta_span[2 * blockIdx.x + 1] = gtimer();
#endif
}

#if defined(EIGENID_PHASE_TIMING) && defined(EIGENID_STAGE1_PRIMARY)
extern "C" void eigenid_debug_phase_cycles(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_phase_cycles, sizeof(g_phase_cycles));
}
extern "C" void eigenid_debug_cta_span(unsigned long long* out) {
  cudaMemcpyFromSymbol(out, g_cta_span, sizeof(g_cta_span));
}
#endif

size_t stage1_smem_bytes() { return sizeof(double) * (size_t)kStage1SmemDoubles; }
int stage1_ctas_per_sm() { return kCtasPerSm; }

cudaError_t launch_stage1(const Stage1Args& a, int grid, cudaStream_t st,
                          bool reset) {
  const size_t smem = stage1_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(
      band_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  if (reset) {
    e = cudaMemsetAsync(a.counter, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
  }
  band_reduce_kernel<<<grid, kNT, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace EIGENID_STAGE1_NS

#ifdef EIGENID_STAGE1_PRIMARY
// layout-independent band / workspace geometry
int stage1_band_ld() { return EIGENID_STAGE1_NS::kLDAB; }
int stage1_bandwidth() { return EIGENID_STAGE1_NS::kB; }
long long stage1_ws_doubles(int n, int ldw) {
  return (long long)n * ldw + 5LL * n * EIGENID_STAGE1_NS::kB;
}

#endif

}  // namespace eigenid_b200
