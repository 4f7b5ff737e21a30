// FP64 pipe microbenchmark for B200 (sm_100a): DFMA, DADD, DMUL, DDIV and
// DMMA (mma.sync m8n8k4 f64) throughput, timed with CUDA events. Prints one
// JSON line. Used to pin P_fp64 for the roofline.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

template <int OP>
__global__ void fp_kernel(double* out, int iters, double s) {
  double a[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) a[q] = threadIdx.x * 1e-3 + q;
  const double b = s, c = 1.0 - s;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (OP == 0) a[q] = fma(a[q], b, c);
      if (OP == 1) a[q] = a[q] + b;
      if (OP == 2) a[q] = a[q] * b;
      if (OP == 3) a[q] = c / a[q];
    }
  }
  double r = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) r += a[q];
  if (r == 12345.678) out[0] = r;
}

__global__ void dmma_kernel(double* out, int iters) {
  double acc[4][2];
  for (int t = 0; t < 4; ++t) { acc[t][0] = 0; acc[t][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(acc[t][0]), "+d"(acc[t][1]) : "d"(a), "d"(b));
    }
  }
  double r = 0;
  for (int t = 0; t < 4; ++t) r += acc[t][0] + acc[t][1];
  if (r == 12345.678) out[0] = r;
}

// Sustained DMMA: random operands (8 distinct A and B values per lane, cycled
// across the unrolled instructions so the operand bits toggle as in a real
// product), back-to-back launches for SECONDS; reports the rate over the
// whole interval, i.e. under the board's power cap.
__global__ void dmma_rand_kernel(double* out, int iters, unsigned seed) {
  double acc[4][2], a[8], b[8];
  unsigned x = seed ^ (blockIdx.x * 7919u + threadIdx.x * 104729u);
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    x ^= x << 13; x ^= x >> 17; x ^= x << 5;
    a[q] = (double)(int)x * 4.656612873077393e-10;
    x ^= x << 13; x ^= x >> 17; x ^= x << 5;
    b[q] = (double)(int)x * 4.656612873077393e-10;
  }
  for (int t = 0; t < 4; ++t) { acc[t][0] = a[t]; acc[t][1] = b[t]; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      asm volatile(
          "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
          : "+d"(acc[q & 3][0]), "+d"(acc[q & 3][1]) : "d"(a[q]), "d"(b[7 - q]));
    }
  }
  double r = 0;
  for (int t = 0; t < 4; ++t) r += acc[t][0] + acc[t][1];
  if (r == 12345.678) out[0] = r;
}

int sustained(double seconds) {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = p.multiProcessorCount * 4, threads = 256, iters = 1 << 14;
  dmma_rand_kernel<<<blocks, threads>>>(d, iters, 1u);  // warm-up
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  long long launches = 0;
  float ms = 0;
  while (ms < seconds * 1e3) {
    for (int k = 0; k < 8; ++k, ++launches)
      dmma_rand_kernel<<<blocks, threads>>>(d, iters, (unsigned)launches + 2u);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
  }
  CK(cudaGetLastError());
  const double fma = (double)launches * iters * 8.0 * (blocks * threads / 32) * 256.0;
  printf("{\"gpu\": \"%s\", \"dmma_sustained_tflops\": %.3f, \"seconds\": %.2f, "
         "\"operands\": \"random\"}\n", p.name, 2 * fma / (ms * 1e-3) / 1e12, ms / 1e3);
  return 0;
}

int main(int argc, char** argv) {
  if (argc > 1) return sustained(atof(argv[1]));
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  double* d; CK(cudaMalloc(&d, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int sms = p.multiProcessorCount;
  const int blocks = sms * 8, threads = 256, iters = 4096;
  double res[5];
  for (int op = 0; op < 5; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(e0);
      if (op == 0) fp_kernel<0><<<blocks, threads>>>(d, iters, 0.999);
      if (op == 1) fp_kernel<1><<<blocks, threads>>>(d, iters, 0.999);
      if (op == 2) fp_kernel<2><<<blocks, threads>>>(d, iters, 0.999);
      if (op == 3) fp_kernel<3><<<blocks, threads>>>(d, iters / 8, 0.999);
      if (op == 4) dmma_kernel<<<blocks, threads>>>(d, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double ops;
      if (op < 3) ops = 8.0 * iters * blocks * threads;           // per-lane ops
      else if (op == 3) ops = 8.0 * (iters / 8) * blocks * threads;
      else ops = 4.0 * iters * (blocks * threads / 32) * 256.0;   // FMAs
      res[op] = ops / (ms * 1e-3);
    }
  }
  CK(cudaGetLastError());
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"clock_khz\": %d, "
         "\"dfma_tflops\": %.3f, \"dadd_gops\": %.1f, \"dmul_gops\": %.1f, "
         "\"ddiv_gops\": %.1f, \"dmma_tflops\": %.3f}\n",
         p.name, sms, clk, 2 * res[0] / 1e12, res[1] / 1e9, res[2] / 1e9,
         res[3] / 1e9, 2 * res[4] / 1e12);
  return 0;
}
