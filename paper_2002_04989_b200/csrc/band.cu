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
#include "common.cuh"

namespace eigenid_b200 {

constexpr int kB = 32;      // bandwidth / panel width
constexpr int kNT = 256;    // threads per CTA (8 warps)
constexpr int kLDAB = 2 * kB + 1;  // band storage: diagonals 0..2kB per column

// Shared-memory layout (doubles).
constexpr int kG1_LDA = 36, kG1_LDB = 36;            // GEMM1 tiles
constexpr int kG1_A = 64 * kG1_LDA, kG1_B = 32 * kG1_LDB;
constexpr int kG2_LD = 68;                            // GEMM2 operand tiles
constexpr int kG2_OP = 64 * kG2_LD;
constexpr int kGemmSmem = (2 * kG1_A + 2 * kG1_B) > (3 * kG2_OP)
                              ? (2 * kG1_A + 2 * kG1_B)
                              : (3 * kG2_OP);
constexpr int kSmallLD = kB + 1;
constexpr int kSmallMat = kB * kSmallLD;  // T, G/Y, M
constexpr int kStage1SmemDoubles = kGemmSmem + 3 * kSmallMat + 8 * kB + 4 * kB;

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
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cpa_wait1() { asm volatile("cp.async.wait_group 1;\n" ::); }
__device__ __forceinline__ void cpa_wait0() { asm volatile("cp.async.wait_group 0;\n" ::); }

// Reduce-scatter of 32 per-lane values: afterwards lane l holds the warp sum
// of vals[l] in vals[0].
__device__ __forceinline__ void warp_reduce_scatter32(double (&v)[kB]) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) {
    const bool up = (lane & o) != 0;
#pragma unroll
    for (int q = 0; q < o; ++q) {
      const double send = up ? v[q] : v[q + o];
      const double keep = up ? v[q + o] : v[q];
      v[q] = keep + __shfl_xor_sync(0xffffffffu, send, o);
    }
  }
}

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
};

// ---- panel QR ----------------------------------------------------------
// Householder QR of the s x kB panel P(r,t) = W[(c0+r)*ldw + cp + t]
// (LAPACK dgeqr2 / dlarfg convention: H = I - tau v v^T, v_0 = 1).
// R overwrites the panel's upper triangle, zeros below; V (s x kB,
// row-major, unit lower trapezoidal, zero above) goes to Vg; tau to stau.
__device__ void panel_qr(double* W, int ldw, int c0, int cp, int s, double* Vg,
                         double* stau, double* red, double* wsm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kr = min(kB, s - 1);
  auto P = [&](int r, int t) -> double& {
    return W[(long long)(c0 + r) * ldw + cp + t];
  };
  // sigma for column 0
  double loc = 0.0;
  for (int r = 1 + tid; r < s; r += kNT) {
    const double x = P(r, 0);
    loc += x * x;
  }
  double sigma = block_sum(loc, red);
  for (int t = 0; t < kr; ++t) {
    const double alpha = P(t, t);
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
    // v below the diagonal; w_q = P(t,q) + sum_{r>t} v_r P(r,q), q > t
    double acc[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) acc[q] = 0.0;
    for (int r = t + 1 + tid; r < s; r += kNT) {
      double* prow = &P(r, 0);
      const double v = prow[t] * scal;
      Vg[(long long)r * kB + t] = v;
      prow[t] = 0.0;
#pragma unroll
      for (int q = 0; q < kB; ++q)
        if (q > t) acc[q] += v * prow[q];
    }
    warp_reduce_scatter32(acc);
    __syncthreads();
    red[8 + warp * kB + lane] = acc[0];
    __syncthreads();
    if (tid < kB) {
      double w = 0.0;
#pragma unroll
      for (int ww = 0; ww < kNT / 32; ++ww) w += red[8 + ww * kB + tid];
      wsm[tid] = (tid > t) ? tau * (w + P(t, tid)) : 0.0;
    }
    __syncthreads();
    // apply: P(r,q) -= tau w_q v_r (r >= t, q > t); accumulate next sigma
    loc = 0.0;
    for (int r = t + tid; r < s; r += kNT) {
      double* prow = &P(r, 0);
      const double v = (r == t) ? 1.0 : Vg[(long long)r * kB + t];
#pragma unroll
      for (int q = 0; q < kB; ++q)
        if (q > t) prow[q] -= wsm[q] * v;
      if (t + 1 < kB && r > t + 1) loc += prow[t + 1] * prow[t + 1];
    }
    if (tid == 0) {
      P(t, t) = beta;
      stau[t] = tau;
      Vg[(long long)t * kB + t] = 1.0;
    }
    for (int r = tid; r < t; r += kNT) Vg[(long long)r * kB + t] = 0.0;
    sigma = block_sum(loc, red);
  }
  // columns with no reflector (s - 1 < kB)
  for (int t = kr; t < kB; ++t) {
    for (int r = tid; r < s; r += kNT) Vg[(long long)r * kB + t] = 0.0;
    if (tid == 0) stau[t] = 0.0;
  }
  __syncthreads();
}

// out[q][p] = sum_r L(r,q) R(r,p) over r in [0,s); L, R row-major s x kB.
// Staged through shared memory in 64-row chunks (stg needs 2*64*(kB+1)).
__device__ void gram(const double* Lg, const double* Rg, int s, double* out,
                     double* stg) {
  const int tid = threadIdx.x;
  double* sL = stg;
  double* sR = stg + 64 * kSmallLD;
  const int p = tid & 31, q0 = tid >> 5;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};
  for (int r0 = 0; r0 < s; r0 += 64) {
    __syncthreads();
    for (int t = tid; t < 64 * kB; t += kNT) {
      const int r = t / kB, c = t % kB;
      const bool ok = r0 + r < s;
      sL[r * kSmallLD + c] = ok ? Lg[(long long)(r0 + r) * kB + c] : 0.0;
      sR[r * kSmallLD + c] = ok ? Rg[(long long)(r0 + r) * kB + c] : 0.0;
    }
    __syncthreads();
    const int rr = min(64, s - r0);
    for (int r = 0; r < rr; ++r) {
      const double rv = sR[r * kSmallLD + p];
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[u] += sL[r * kSmallLD + q0 + 8 * u] * rv;
    }
  }
  __syncthreads();
#pragma unroll
  for (int u = 0; u < 4; ++u) out[(q0 + 8 * u) * kSmallLD + p] = acc[u];
  __syncthreads();
}

// Y(r,:) = alpha * L(r,:) * Mt + (addg ? Add(r,:) : 0) for r in [0,s).
// Mt is kB x kB in shared memory (ld kSmallLD).
__device__ void row_transform(const double* Lg, const double* Mt, double alpha,
                              const double* Add, double* Yg, int s) {
  for (int r = threadIdx.x; r < s; r += kNT) {
    double y[kB];
#pragma unroll
    for (int q = 0; q < kB; ++q) y[q] = 0.0;
    const double* lr = Lg + (long long)r * kB;
#pragma unroll 2
    for (int p = 0; p < kB; ++p) {
      const double lp = lr[p];
#pragma unroll
      for (int q = 0; q < kB; ++q) y[q] += lp * Mt[p * kSmallLD + q];
    }
    double* yr = Yg + (long long)r * kB;
    const double* ar = Add ? Add + (long long)r * kB : nullptr;
#pragma unroll
    for (int q = 0; q < kB; ++q) yr[q] = (ar ? ar[q] : 0.0) + alpha * y[q];
  }
  __syncthreads();
}

// ---- GEMM 1: X(s x kB) = A22(s x s) * VT(s x kB) --------------------------
__device__ void gemm1(const double* A22, int ldw, int s, const double* VTg,
                      double* Xg, double* sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;
  double* sA[2] = {sm, sm + kG1_A};
  double* sB[2] = {sm + 2 * kG1_A, sm + 2 * kG1_A + kG1_B};
  const int nk = (s + 31) / 32;
  for (int rb = 0; rb < s; rb += 64) {
    double acc[2][2][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
    auto stage = [&](int kb, int buf) {
      // A tile 64 x 32: 1024 16-byte chunks
      for (int t = tid; t < 64 * 16; t += kNT) {
        const int r = t >> 4, c2 = (t & 15) * 2;
        const int gr = rb + r, gc = kb + c2;
        int bytes = 0;
        if (gr < s && gc < s) bytes = (gc + 1 < s) ? 16 : 8;
        const double* src = bytes ? A22 + (long long)gr * ldw + gc : A22;
        cp_async16(sA[buf] + r * kG1_LDA + c2, src, bytes);
      }
      // VT tile 32 x 32: 512 chunks
      for (int t = tid; t < 32 * 16; t += kNT) {
        const int r = t >> 4, c2 = (t & 15) * 2;
        const int gr = kb + r;
        const int bytes = gr < s ? 16 : 0;
        const double* src = bytes ? VTg + (long long)gr * kB + c2 : VTg;
        cp_async16(sB[buf] + r * kG1_LDB + c2, src, bytes);
      }
      cpa_commit();
    };
    __syncthreads();
    stage(0, 0);
    for (int ki = 0; ki < nk; ++ki) {
      if (ki + 1 < nk) {
        stage((ki + 1) * 32, (ki + 1) & 1);
        cpa_wait1();
      } else {
        cpa_wait0();
      }
      __syncthreads();
      const double* a = sA[ki & 1];
      const double* b = sB[ki & 1];
#pragma unroll
      for (int k4 = 0; k4 < 8; ++k4) {
        const int kk = 4 * k4 + (lane & 3);
        const double a0 = a[(16 * wm + (lane >> 2)) * kG1_LDA + kk];
        const double a1 = a[(16 * wm + 8 + (lane >> 2)) * kG1_LDA + kk];
        const double b0 = b[kk * kG1_LDB + 16 * wn + (lane >> 2)];
        const double b1 = b[kk * kG1_LDB + 16 * wn + 8 + (lane >> 2)];
        dmma(acc[0][0][0], acc[0][0][1], a0, b0);
        dmma(acc[0][1][0], acc[0][1][1], a0, b1);
        dmma(acc[1][0][0], acc[1][0][1], a1, b0);
        dmma(acc[1][1][0], acc[1][1][1], a1, b1);
      }
      __syncthreads();
    }
#pragma unroll
    for (int mt = 0; mt < 2; ++mt) {
      const int r = rb + 16 * wm + 8 * mt + (lane >> 2);
      if (r >= s) continue;
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) {
        const int c = 16 * wn + 8 * nt + 2 * (lane & 3);
        *reinterpret_cast<double2*>(Xg + (long long)r * kB + c) =
            make_double2(acc[mt][nt][0], acc[mt][nt][1]);
      }
    }
  }
  __syncthreads();
}

// ---- GEMM 2: A22 -= W2 V^T + V W2^T  (full symmetric storage) ------------
// As A22 += Aop * Bop^T with Aop = -[W2 | V], Bop = [V | W2] (s x 2kB).
__device__ void gemm2(double* A22, int ldw, int s, const double* W2g,
                      const double* Vg, double* sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 2, wn = warp & 3;
  double* sOA = sm;
  double* sOB[2] = {sm + kG2_OP, sm + 2 * kG2_OP};
  const int ncb = (s + 63) / 64;
  for (int rb = 0; rb < s; rb += 64) {
    __syncthreads();
    for (int t = tid; t < 64 * 2 * kB; t += kNT) {
      const int r = t / (2 * kB), k = t % (2 * kB);
      const int gr = rb + r;
      double v = 0.0;
      if (gr < s)
        v = k < kB ? W2g[(long long)gr * kB + k] : Vg[(long long)gr * kB + k - kB];
      sOA[r * kG2_LD + k] = -v;
    }
    auto stage = [&](int cb, int buf) {
      for (int t = tid; t < 64 * 32; t += kNT) {
        const int r = t >> 5, k2 = (t & 31) * 2;
        const int gr = cb + r;
        const int bytes = gr < s ? 16 : 0;
        const double* src =
            k2 < kB ? Vg + (long long)(bytes ? gr : 0) * kB + k2
                    : W2g + (long long)(bytes ? gr : 0) * kB + (k2 - kB);
        cp_async16(sOB[buf] + r * kG2_LD + k2, src, bytes);
      }
      cpa_commit();
    };
    stage(0, 0);
    for (int ci = 0; ci < ncb; ++ci) {
      const int cb = ci * 64;
      // C fragments straight from global (issued before the wait)
      double acc[4][2][2];
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int r = rb + 32 * wm + 8 * mt + (lane >> 2);
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int c = cb + 16 * wn + 8 * nt + 2 * (lane & 3);
          if (r < s && c < s) {
            const double* p = A22 + (long long)r * ldw + c;
            acc[mt][nt][0] = p[0];
            acc[mt][nt][1] = (c + 1 < s) ? p[1] : 0.0;
          } else {
            acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
          }
        }
      }
      if (ci + 1 < ncb) {
        stage(cb + 64, (ci + 1) & 1);
        cpa_wait1();
      } else {
        cpa_wait0();
      }
      __syncthreads();
      const double* b = sOB[ci & 1];
#pragma unroll 4
      for (int k4 = 0; k4 < 2 * kB / 4; ++k4) {
        const int kk = 4 * k4 + (lane & 3);
        double af[4], bf[2];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
          af[mt] = sOA[(32 * wm + 8 * mt + (lane >> 2)) * kG2_LD + kk];
#pragma unroll
        for (int nt = 0; nt < 2; ++nt)
          bf[nt] = b[(16 * wn + 8 * nt + (lane >> 2)) * kG2_LD + kk];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
          for (int nt = 0; nt < 2; ++nt)
            dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
      }
#pragma unroll
      for (int mt = 0; mt < 4; ++mt) {
        const int r = rb + 32 * wm + 8 * mt + (lane >> 2);
        if (r >= s) continue;
#pragma unroll
        for (int nt = 0; nt < 2; ++nt) {
          const int c = cb + 16 * wn + 8 * nt + 2 * (lane & 3);
          if (c >= s) continue;
          double* p = A22 + (long long)r * ldw + c;
          p[0] = acc[mt][nt][0];
          if (c + 1 < s) p[1] = acc[mt][nt][1];
        }
      }
      __syncthreads();
    }
  }
  __syncthreads();
}

__device__ void write_band(const double* W, int ldw, int m, int c_begin,
                           int c_end, double* band) {
  for (int t = threadIdx.x; t < (c_end - c_begin) * kLDAB; t += kNT) {
    const int col = c_begin + t / kLDAB, d = t % kLDAB;
    double v = 0.0;
    if (d <= kB && col + d < m) v = W[(long long)(col + d) * ldw + col];
    band[(long long)col * kLDAB + d] = v;
  }
}

__global__ void __launch_bounds__(kNT, 1) band_reduce_kernel(Stage1Args args) {
  extern __shared__ double smem[];
  double* sgemm = smem;
  double* sT = smem + kGemmSmem;
  double* sG = sT + kSmallMat;   // G, then Y
  double* sM = sG + kSmallMat;
  double* red = sM + kSmallMat;  // 8 + 8*kB
  double* stau = red + 8 + 8 * kB;
  double* wsm = stau + kB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int n = args.n, ldw = args.ldw;
  double* W = args.ws + blockIdx.x * args.ws_stride;
  double* Vg = W + (long long)n * ldw;
  double* VTg = Vg + (long long)n * kB;
  double* Xg = VTg + (long long)n * kB;

  for (int sidx = blockIdx.x; sidx < args.nsolves; sidx += gridDim.x) {
    const int j = args.js[sidx];
    const int m = j < 0 ? n : n - 1;
    double* band = args.band + sidx * args.band_stride;
    // materialise the minor (index remap r' = r + (r >= j)), full storage
    for (int r = warp; r < m; r += kNT / 32) {
      const int rr = (j >= 0 && r >= j) ? r + 1 : r;
      const double* src = args.A + (long long)rr * n;
      double* dst = W + (long long)r * ldw;
      for (int c = lane; c < m; c += 32) dst[c] = src[(j >= 0 && c >= j) ? c + 1 : c];
    }
    __syncthreads();
    int c = 0;
    for (; c < m; c += kB) {
      const int s = m - c - kB;
      if (s < 2) break;
      const int c0 = c + kB;
      panel_qr(W, ldw, c0, c, s, Vg, stau, red, wsm);
      write_band(W, ldw, m, c, c + kB, band);
      // T (dlarft, forward columnwise) from G = V^T V
      gram(Vg, Vg, s, sG, sgemm);
      if (warp == 0) {
        for (int t = 0; t < kB; ++t) {
          // column t: T[q][t] = -tau_t * sum_{p=q}^{t-1} T[q][p] G[p][t]
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
      __syncthreads();
      row_transform(Vg, sT, 1.0, nullptr, VTg, s);           // VT = V T
      double* A22 = W + (long long)c0 * ldw + c0;
      gemm1(A22, ldw, s, VTg, Xg, sgemm);                     // X = A22 VT
      gram(Vg, Xg, s, sG, sgemm);                             // Y = V^T X
      // M = T^T Y
      for (int t = tid; t < kB * kB; t += kNT) {
        const int q = t / kB, p = t % kB;
        double v = 0.0;
        for (int u = 0; u <= q; ++u) v += sT[u * kSmallLD + q] * sG[u * kSmallLD + p];
        sM[q * kSmallLD + p] = v;
      }
      __syncthreads();
      row_transform(Vg, sM, -0.5, Xg, Xg, s);                 // W2 = X - V M/2
      gemm2(A22, ldw, s, Xg, Vg, sgemm);                      // A22 -= W2V^T+VW2^T
    }
    write_band(W, ldw, m, c, m, band);
    __syncthreads();
  }
}

size_t stage1_smem_bytes() { return sizeof(double) * (size_t)kStage1SmemDoubles; }
int stage1_band_ld() { return kLDAB; }
int stage1_bandwidth() { return kB; }

cudaError_t launch_stage1(const Stage1Args& a, int grid, cudaStream_t st) {
  const size_t smem = stage1_smem_bytes();
  cudaError_t e = cudaFuncSetAttribute(
      band_reduce_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  band_reduce_kernel<<<grid, kNT, smem, st>>>(a);
  return cudaGetLastError();
}

}  // namespace eigenid_b200
