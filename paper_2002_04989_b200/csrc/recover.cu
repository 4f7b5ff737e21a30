// recover.cu — §8 f4: sign recovery, recover_signs (signs.cpp:48-120).
//
// Given the squared magnitudes of eigenvector i (from all_magnitudes /
// vector_magnitudes) and lambda_i, the largest component (first on ties) is
// anchored and the other n-1 row equations of (A - lambda I) v = 0 are solved
// for the remaining components; only their signs are kept, the first
// component above sign_tol is made positive, and the residual
// ||(A - lambda I) v|| is checked against 1e-6 ||A||_F.
//
// The reference solves the (n-1) x (n-1) system by unblocked Gaussian
// elimination with partial pivoting (solve_linear, signs.cpp:13-44).  Here it
// is a right-looking blocked LU with partial pivoting on the augmented matrix
// [B | rhs] (B = A - lambda I without the anchor row/column), panels of 32
// columns:
//   panel kernel   one CTA factors the s x 32 panel (pivot search, row swap
//                  inside the panel, L column, rank-1 update of the panel);
//   swap_trsm      every 32-column block right of the panel (and the rhs)
//                  applies the panel's row swaps and U12 = L11^-1 A12;
//   update         A22 -= L21 U12 on the DMMA path (64 x 64 tiles, k = 32);
// then a blocked back substitution U x = y and the sign/residual epilogue.
// The pivot choice (largest |entry|, first on ties) is the reference's; the
// elimination order differs, so the solved values agree to rounding and the
// signs agree wherever they are not noise (|x| above the solve's error).
#include "kernels.cuh"

namespace eigenid_b200 {

constexpr int kRB = 32;       // panel width
constexpr int kRNT = 1024;    // panel / back-substitution CTA size

struct RecoverState {
  int anchor;        // anchored component
  int singular;      // zero pivot met (SignRecoveryFailure)
  double va;         // sqrt(clamp(mags[anchor]))
  double res2, fro2; // ||(A - lambda I) v||^2, ||A||_F^2
};

__device__ __forceinline__ double clamp01d(double x) { return fmin(fmax(x, 0.0), 1.0); }

// anchor = argmax mags exactly as signs.cpp:68-70 scans it: start at 0 and
// move on a strict '>' only, so ties keep the first index and a NaN at 0 (or
// anywhere) never wins or loses a comparison the reference would not.  One
// thread: n <= 14000 comparisons, negligible next to the LU.
__global__ void rs_anchor_kernel(const double* mags, int n, RecoverState* st) {
  if (threadIdx.x != 0) return;
  int bi = 0;
  for (int j = 1; j < n; ++j)
    if (mags[j] > mags[bi]) bi = j;
  st->anchor = bi;
  st->singular = 0;
  st->va = sqrt(clamp01d(mags[bi]));
  st->res2 = 0.0;
  st->fro2 = 0.0;
}

// W (m x (m+1), ld ldw): B without the anchor row/column | rhs
__global__ void rs_build_kernel(const double* A, int n, double lambda,
                                const RecoverState* st, double* W, long long ldw) {
  const int m = n - 1;
  const int anchor = st->anchor;
  const double va = st->va;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)m * (m + 1);
       t += (long long)gridDim.x * blockDim.x) {
    const int rr = (int)(t / (m + 1)), cc = (int)(t % (m + 1));
    const int r = rr + (rr >= anchor);
    double v;
    if (cc < m) {
      const int c = cc + (cc >= anchor);
      v = A[(long long)r * n + c] - (r == c ? lambda : 0.0);
    } else {
      v = -A[(long long)r * n + anchor] * va;  // r != anchor
    }
    W[(long long)rr * ldw + cc] = v;
  }
}

// Factor columns c0..c0+w-1 of W (rows c0..m-1): partial pivoting with the
// reference's rule, swaps applied inside the panel only (recorded in ipiv),
// L stored below the diagonal.
__global__ void __launch_bounds__(kRNT) rs_panel_kernel(double* W, long long ldw, int m,
                                                        int c0, int* ipiv,
                                                        RecoverState* st) {
  __shared__ double rv[kRNT / 32];
  __shared__ int ri[kRNT / 32];
  __shared__ int s_piv;
  __shared__ double s_inv;
  __shared__ double s_prow[kRB];
  if (st->singular) return;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int w = min(kRB, m - c0);
  for (int col = c0; col < c0 + w; ++col) {
    // pivot: largest |W[r][col]|, r >= col, smallest r on ties
    double best = -1.0;
    int bi = 0x7fffffff;
    for (int r = col + tid; r < m; r += kRNT) {
      const double v = fabs(W[(long long)r * ldw + col]);
      if (v > best) {
        best = v;
        bi = r;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) {
        best = ov;
        bi = oi;
      }
    }
    if (lane == 0) {
      rv[warp] = best;
      ri[warp] = bi;
    }
    __syncthreads();
    if (tid == 0) {
      for (int q = 1; q < kRNT / 32; ++q)
        if (rv[q] > best || (rv[q] == best && ri[q] < bi)) {
          best = rv[q];
          bi = ri[q];
        }
      s_piv = bi;
      ipiv[col - c0] = bi;
      const double p = W[(long long)bi * ldw + col];
      if (p == 0.0) st->singular = 1;
      s_inv = 1.0 / p;
    }
    __syncthreads();
    if (st->singular) return;
    const int piv = s_piv;
    // swap rows col <-> piv inside the panel; keep the pivot row in smem
    if (tid < w) {
      const int c = c0 + tid;
      const double a = W[(long long)col * ldw + c], b = W[(long long)piv * ldw + c];
      W[(long long)col * ldw + c] = b;
      W[(long long)piv * ldw + c] = a;
      s_prow[tid] = b;
    }
    __syncthreads();
    const double inv = s_inv;
    // L column and rank-1 update of the remaining panel columns
    for (int r = col + 1 + tid; r < m; r += kRNT) {
      double* row = W + (long long)r * ldw;
      const double f = row[col] * inv;
      row[col] = f;
      if (f != 0.0)
        for (int c = col + 1; c < c0 + w; ++c) row[c] -= f * s_prow[c - c0];
    }
    __syncthreads();
  }
}

// Columns [cs, m] (incl. the rhs column m), 32 per CTA, thread per column:
// apply the panel's swaps in order, then U12 = L11^-1 A12.
__global__ void rs_swap_trsm_kernel(double* W, long long ldw, int m, int c0,
                                    const int* ipiv, const RecoverState* st) {
  if (st->singular) return;
  __shared__ double sL[kRB][kRB + 1];
  __shared__ int sp[kRB];
  const int w = min(kRB, m - c0);
  for (int t = threadIdx.x; t < w * w; t += blockDim.x) {
    const int i = t / w, k = t % w;
    sL[i][k] = W[(long long)(c0 + i) * ldw + c0 + k];
  }
  if (threadIdx.x < w) sp[threadIdx.x] = ipiv[threadIdx.x];
  __syncthreads();
  const int c = c0 + w + blockIdx.x * blockDim.x + threadIdx.x;
  if (c > m) return;
  double u[kRB];
#pragma unroll
  for (int i = 0; i < kRB; ++i) u[i] = 0.0;
  for (int i = 0; i < w; ++i) {
    const int p = sp[i];
    const int r = c0 + i;
    if (p != r) {
      const double a = W[(long long)r * ldw + c], b = W[(long long)p * ldw + c];
      W[(long long)r * ldw + c] = b;
      W[(long long)p * ldw + c] = a;
    }
  }
#pragma unroll
  for (int i = 0; i < kRB; ++i) {
    if (i < w) {
      double x = W[(long long)(c0 + i) * ldw + c];
#pragma unroll
      for (int k = 0; k < kRB; ++k)
        if (k < i) x -= sL[i][k] * u[k];
      u[i] = x;
      W[(long long)(c0 + i) * ldw + c] = x;
    }
  }
}

__device__ __forceinline__ void rs_dmma(double& c0, double& c1, double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c0), "+d"(c1)
      : "d"(a), "d"(b));
}

// A22 -= L21 U12 for rows/cols >= c0 + w (cols up to the rhs column m):
// 64 x 64 tiles, 8 warps of 32 x 16, operands staged in shared memory.
__global__ void __launch_bounds__(256) rs_update_kernel(double* W, long long ldw, int m,
                                                        int c0, const RecoverState* st) {
  if (st->singular) return;
  __shared__ double sA[64][kRB + 4];
  __shared__ double sB[kRB][64 + 4];
  const int w = min(kRB, m - c0);
  const int r0 = c0 + w + 64 * blockIdx.y, q0 = c0 + w + 64 * blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int kk = lane & 3, mm = lane >> 2;
  for (int t = tid; t < 64 * kRB; t += 256) {
    const int i = t / kRB, k = t % kRB;
    const int r = r0 + i;
    sA[i][k] = (r < m && k < w) ? W[(long long)r * ldw + c0 + k] : 0.0;
  }
  for (int t = tid; t < kRB * 64; t += 256) {
    const int k = t / 64, j = t % 64;
    const int q = q0 + j;
    sB[k][j] = (q <= m && k < w) ? W[(long long)(c0 + k) * ldw + q] : 0.0;
  }
  __syncthreads();
  const int wm = warp >> 2, wn = warp & 3;  // 2 x 4 warps: 32 rows x 16 cols each
  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
  for (int k4 = 0; k4 < kRB / 4; ++k4) {
    const int k = 4 * k4 + kk;
    double af[4], bf[2];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt) af[mt] = sA[32 * wm + 8 * mt + mm][k];
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) bf[nt] = sB[k][16 * wn + 8 * nt + mm];
#pragma unroll
    for (int mt = 0; mt < 4; ++mt)
#pragma unroll
      for (int nt = 0; nt < 2; ++nt) rs_dmma(acc[mt][nt][0], acc[mt][nt][1], af[mt], bf[nt]);
  }
#pragma unroll
  for (int mt = 0; mt < 4; ++mt) {
    const int r = r0 + 32 * wm + 8 * mt + mm;
    if (r >= m) continue;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
      const int q = q0 + 16 * wn + 8 * nt + 2 * kk;
      double* p = W + (long long)r * ldw + q;
      if (q <= m) p[0] -= acc[mt][nt][0];
      if (q + 1 <= m) p[1] -= acc[mt][nt][1];
    }
  }
}

// U x = y (y = rhs column, overwritten by x), 32-row blocks from the bottom:
// warp per row for the dot with the solved part, then a warp-level triangular
// solve of the diagonal block.
__global__ void __launch_bounds__(kRNT) rs_backsub_kernel(double* W, long long ldw, int m,
                                                          const RecoverState* st) {
  if (st->singular) return;
  __shared__ double sdot[kRB];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = (m + kRB - 1) / kRB;
  for (int b = nb - 1; b >= 0; --b) {
    const int R0 = b * kRB, R1 = min(m, R0 + kRB);
    const int r = R0 + warp;
    if (warp < kRB) {
      double d = 0.0;
      if (r < R1) {
        const double* row = W + (long long)r * ldw;
        for (int c = R1 + lane; c < m; c += 32) d += row[c] * W[(long long)c * ldw + m];
      }
      d = warp_sum(d);
      if (lane == 0) sdot[warp] = d;
    }
    __syncthreads();
    if (warp == 0) {
      // lane i owns row R0 + i; sequential over the block's columns
      const int i = lane;
      const int ri = R0 + i;
      double y = ri < R1 ? W[(long long)ri * ldw + m] - sdot[i] : 0.0;
      for (int k = R1 - R0 - 1; k >= 0; --k) {
        double xk = 0.0;
        if (i == k) xk = y / W[(long long)ri * ldw + ri];
        xk = __shfl_sync(0xffffffffu, xk, k);
        if (i == k && ri < R1) W[(long long)ri * ldw + m] = xk;
        if (i < k && ri < R1) y -= W[(long long)ri * ldw + R0 + k] * xk;
      }
    }
    __syncthreads();
  }
}

// Signs from the solve, sign convention, then the residual partial sums.
__global__ void rs_finish_kernel(const double* mags, int n, double sign_tol,
                                 const double* W, long long ldw, RecoverState* st,
                                 double* v) {
  __shared__ int s_first;
  const int anchor = n > 1 ? st->anchor : 0;
  for (int j = threadIdx.x; j < n; j += blockDim.x) {
    double x = sqrt(clamp01d(mags[j]));
    if (n > 1 && j != anchor) {
      const int jj = j - (j > anchor);
      if (mags[j] > sign_tol && W[(long long)jj * ldw + (n - 1)] < 0.0) x = -x;
    }
    v[j] = x;
  }
  if (threadIdx.x == 0) s_first = 0x7fffffff;
  __syncthreads();
  for (int j = threadIdx.x; j < n; j += blockDim.x)
    if (mags[j] > sign_tol) atomicMin(&s_first, j);
  __syncthreads();
  const int f = s_first;
  const bool flip = f < n && v[f] < 0.0;
  __syncthreads();
  if (flip)
    for (int j = threadIdx.x; j < n; j += blockDim.x) v[j] = -v[j];
}

// res2 = sum_r ((A - lambda I) v)_r^2 and fro2 = ||A||_F^2, row per warp,
// per-block partials reduced in a fixed order by rs_reduce_kernel.
__global__ void rs_residual_kernel(const double* A, int n, double lambda, const double* v,
                                   double* part) {
  __shared__ double s1[8], s2[8];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double r2 = 0.0, f2 = 0.0;
  for (int r = blockIdx.x * 8 + warp; r < n; r += gridDim.x * 8) {
    const double* row = A + (long long)r * n;
    double d = 0.0, f = 0.0;
    for (int c = lane; c < n; c += 32) {
      const double a = row[c];
      d += (a - (r == c ? lambda : 0.0)) * v[c];
      f += a * a;
    }
    d = warp_sum(d);
    f = warp_sum(f);
    r2 += d * d;
    f2 += f;
  }
  if (lane == 0) {
    s1[warp] = r2;
    s2[warp] = f2;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int q = 0; q < 8; ++q) {
      a += s1[q];
      b += s2[q];
    }
    part[2 * blockIdx.x] = a;
    part[2 * blockIdx.x + 1] = b;
  }
}

__global__ void rs_reduce_kernel(const double* part, int nparts, RecoverState* st) {
  if (threadIdx.x != 0) return;
  double a = 0.0, b = 0.0;
  for (int q = 0; q < nparts; ++q) {
    a += part[2 * q];
    b += part[2 * q + 1];
  }
  st->res2 = a;
  st->fro2 = b;
}

size_t recover_state_bytes() { return sizeof(RecoverState); }

cudaError_t recover_result(const RecoverState* st_dev, RecoverResult* out, cudaStream_t s) {
  RecoverState h;
  cudaError_t e = cudaMemcpyAsync(&h, st_dev, sizeof(h), cudaMemcpyDeviceToHost, s);
  if (e != cudaSuccess) return e;
  e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return e;
  out->singular = h.singular;
  out->res2 = h.res2;
  out->fro2 = h.fro2;
  return cudaSuccess;
}

long long recover_ws_doubles(int n) {
  const long long m = n > 1 ? n - 1 : 1;
  const long long ldw = (m + 1 + 7) & ~7LL;
  return m * ldw + 4 * 296 + 64;
}

// Enqueues the whole recovery; the state (anchor, singular flag, residual
// sums) lands in *st_dev for the host-side epilogue.
cudaError_t launch_recover_signs(const double* dA, int n, const double* dmags,
                                 double lambda, double sign_tol, double* dv,
                                 double* dws, RecoverState* st_dev, cudaStream_t s,
                                 int* launches) {
  const int m = n - 1;
  const long long ldw = ((long long)(m > 0 ? m : 1) + 1 + 7) & ~7LL;
  double* W = dws;
  int* ipiv = reinterpret_cast<int*>(dws + (long long)(m > 0 ? m : 1) * ldw);
  double* part = dws + (long long)(m > 0 ? m : 1) * ldw + 64;
  rs_anchor_kernel<<<1, kRNT, 0, s>>>(dmags, n, st_dev);
  ++*launches;
  if (n > 1) {
    rs_build_kernel<<<592, 256, 0, s>>>(dA, n, lambda, st_dev, W, ldw);
    ++*launches;
    for (int c0 = 0; c0 < m; c0 += kRB) {
      const int w = min(kRB, m - c0);
      rs_panel_kernel<<<1, kRNT, 0, s>>>(W, ldw, m, c0, ipiv, st_dev);
      const int ncols = m + 1 - (c0 + w);  // incl. the rhs column
      rs_swap_trsm_kernel<<<(ncols + kRB - 1) / kRB, kRB, 0, s>>>(W, ldw, m, c0, ipiv, st_dev);
      *launches += 2;
      const int rows = m - (c0 + w);
      if (rows > 0) {
        dim3 grid((ncols + 63) / 64, (rows + 63) / 64);
        rs_update_kernel<<<grid, 256, 0, s>>>(W, ldw, m, c0, st_dev);
        ++*launches;
      }
    }
    rs_backsub_kernel<<<1, kRNT, 0, s>>>(W, ldw, m, st_dev);
    ++*launches;
  }
  rs_finish_kernel<<<1, 1024, 0, s>>>(dmags, n, sign_tol, W, ldw, st_dev, dv);
  const int nparts = 296;
  rs_residual_kernel<<<nparts, 256, 0, s>>>(dA, n, lambda, dv, part);
  rs_reduce_kernel<<<1, 32, 0, s>>>(part, nparts, st_dev);
  *launches += 3;
  return cudaGetLastError();
}

}  // namespace eigenid_b200
