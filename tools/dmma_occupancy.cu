// DMMA (mma.sync m8n8k4 f64) throughput vs. warps per SM and independent
// accumulator chains per warp, with operands from registers or from shared
// memory.  Sizes the stage-1 GEMM tiling (band.cu).
#include <cstdio>
#include <cuda_runtime.h>

template <int CH, bool SMEM>
__global__ void k(double* out, int iters) {
  __shared__ double s[2][32 * 68];
  double acc[CH][2];
  for (int t = 0; t < CH; ++t) acc[t][0] = acc[t][1] = 0;
  for (int t = threadIdx.x; t < 32 * 68; t += blockDim.x) { s[0][t] = t * 1e-6; s[1][t] = t * 2e-6; }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double a = lane * 1e-3, b = 1.0 + lane * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < CH; ++t) {
      double aa = a, bb = b;
      if (SMEM) { aa = s[0][((t & 3) * 8 + (lane >> 2)) * 68 + (it & 15) * 4 + (lane & 3)];
                  bb = s[1][((t >> 2) * 8 + (lane >> 2)) * 68 + (it & 15) * 4 + (lane & 3)]; }
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(acc[t][0]), "+d"(acc[t][1]) : "d"(aa), "d"(bb));
    }
  }
  double r = 0;
  for (int t = 0; t < CH; ++t) r += acc[t][0] + acc[t][1];
  if (r == 12345.678) out[0] = r;
}

template <int CH, bool SMEM>
void run(int warps_per_sm, double* d) {
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int iters = 2048;
  int threads = warps_per_sm * 32; int blocks = 148;
  if (threads > 1024) { threads = 1024; blocks = 148 * (warps_per_sm / 32); }
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    k<CH, SMEM><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fma = (double)iters * CH * 256.0 * (blocks * threads / 32);
    if (rep) printf("{\"warps_per_sm\": %d, \"chains\": %d, \"smem\": %d, \"tflops\": %.2f}\n",
                    warps_per_sm, CH, (int)SMEM, 2 * fma / (ms * 1e-3) / 1e12);
  }
}

int main() {
  double* d; cudaMalloc(&d, 8);
  for (int w : {4, 8, 16, 32}) {
    run<4, false>(w, d); run<8, false>(w, d); run<16, false>(w, d);
    run<8, true>(w, d); run<16, true>(w, d);
  }
  return 0;
}
