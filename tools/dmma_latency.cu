// DMMA (mma.sync m8n8k4 f64) dependent-chain latency and per-SM-subpartition
// throughput versus warps x independent chains (development aid for the
// stage-1 transposed product).  usage: ./dmma_latency
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

template <int C>
__global__ void chain(double* out, long long* cyc, int iters) {
  double c[C][2];
  for (int k = 0; k < C; ++k) c[k][0] = c[k][1] = threadIdx.x * 1e-9;
  const double a = 1.0 + 1e-12 * threadIdx.x, b = 1.0 - 1e-12 * threadIdx.x;
  __syncthreads();
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < C; ++k) dmma(c[k][0], c[k][1], a, b);
  const long long t1 = clock64();
  double s = 0;
  for (int k = 0; k < C; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
  if (threadIdx.x == 0 && blockIdx.x == 0) *cyc = t1 - t0;
}

template <int C>
void run(int warps) {
  double* out;
  long long* cyc;
  cudaMalloc(&out, sizeof(double) * 148 * 1024);
  cudaMalloc(&cyc, sizeof(long long));
  const int iters = 4096;
  chain<C><<<148, 32 * warps>>>(out, cyc, iters);
  cudaDeviceSynchronize();
  long long h;
  cudaMemcpy(&h, cyc, sizeof h, cudaMemcpyDeviceToHost);
  const double per_dmma_warp = (double)h / (iters * C);
  // SM-level DMMA issue interval: cycles / (dmmas issued by the whole CTA)
  std::printf("chains=%d warps=%2d  cycles/dmma/warp=%6.2f  cycles per DMMA per SM=%6.2f\n",
              C, warps, per_dmma_warp * C / C, (double)h / ((double)iters * C * warps));
  cudaFree(out);
  cudaFree(cyc);
}

int main() {
  for (int w : {1, 4, 8, 16}) {
    run<1>(w);
    run<2>(w);
    run<4>(w);
    run<8>(w);
  }
  return 0;
}
