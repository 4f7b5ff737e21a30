// api.cu — the extern "C" boundary (include/eigenid_b200.h) and the device
// pipeline behind it.
//
// all_magnitudes (identity.cpp:294-316) becomes, per call:
//   n <= 64 : one fused kernel (small.cu), one CTA per matrix;
//   n  > 64 : stage 1 dense->band (band.cu) for A and every minor in the
//             shard, stage 2 band->tridiagonal (bulge.cu), Sturm bisection of
//             lambda(A) (bisect.cu, Gershgorin brackets), the degeneracy check
//             (identity.cpp:141-149), bisection of the minors inside the
//             interlacing brackets, then the identity kernel (identity.cu).
// Everything is enqueued on the context's stream with no host round trip;
// host-pointer entry points copy in/out around it and translate the device
// status record into the reference's typed errors.  There is no CPU
// fallback: without a device every entry point returns EIGENID_E_DEVICE.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: NCCL is loaded on demand (see NcclApi)

#include <algorithm>
#include <atomic>
#include <cmath>
#include <random>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/eigenid_b200.h"
#include "kernels.cuh"

namespace eigenid_b200 {
__global__ void init_status_kernel(DevStatus* st) {
  st[0].code = 0;
  st[0].phase = 0;
  st[0].index = -1;
  st[0].gap = 0.0;
  st[0].aux = -1;
  st[1].code = 0;
  st[1].phase = 0;
  st[1].index = -1;  // == ULLONG_MAX for the atomicMin in degeneracy_kernel
  st[1].gap = 0.0;
  st[1].aux = -1;
}

// Solve list of one chunk of minors: js[t] = j0 + g0 + t.
__global__ void solve_list_kernel(int* js, int j0, int g0, int count) {
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < count;
       t += gridDim.x * blockDim.x)
    js[t] = j0 + g0 + t;
}

// SymmetricMatrix::build rejects non-finite entries before anything is
// solved (matrix.cpp:17-18 -> NonFiniteEntry); the raw C-ABI takes plain
// pointers, so the check runs on the device as the first kernel of a call
// (every later stage aborts on the sticky status).  aux = matrix index.
__global__ void nonfinite_kernel(const double* __restrict__ a, long long per,
                                 long long total, DevStatus* st) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x)
    if (!isfinite(a[t])) set_status(st, EIGENID_E_NONFINITE_ENTRY, t % per, 0.0, t / per);
}

}  // namespace eigenid_b200

using namespace eigenid_b200;

namespace {

constexpr int kSmallMax = 64;
constexpr int kLargeMax = 14000;  // bisection stages (d, e^2) in shared memory

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
};

// Pinned host staging buffer, grown on demand and kept by the context.
struct HostBuf {
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMallocHost(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  template <class T>
  T* as() const { return static_cast<T*>(p); }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
};

}  // namespace

struct eigenid_gpu_ctx {
  bool wait_timed_out = false;  // finish(): a bounded device wait ran out (retried once)
  int device = 0;
  cudaStream_t stream = nullptr;
  cudaStream_t side = nullptr;  // lambda(A)'s solve, beside the minors
  cudaEvent_t ev_start = nullptr, ev_a = nullptr, ev_a0 = nullptr, ev_a1 = nullptr;
  std::mutex mu;
  DevStatus* dstatus = nullptr;
  DevStatus* hstatus = nullptr;  // pinned
  // A *_device call enqueued work whose status nobody has read yet: the
  // status stays sticky (not re-initialised) until eigenid_gpu_sync or the
  // next host-pointer call reads it.
  bool pending = false;
  DevBuf bA, bOut, bLam, bMu, bDen, bRcp, bFlags, bFlagCount, bWs, bBand, bD,
      bE2, bAe, bJs, bTmpOut, bTmpMu, bCounter, bBandA, bDeA, bJsA, bScale;
  std::atomic<size_t> solves{0};
  std::atomic<uint64_t> launches{0};
  bool profiling = false;
  double stage_ms[5] = {0, 0, 0, 0, 0};
  // multi-device context (eigenid_gpu_create_multi): peer[0] == this, one
  // single-device context per further GPU, one NCCL communicator per GPU
  int ngpu = 1;
  bool multi = false;  // created by eigenid_gpu_create_multi (NCCL path, any P)
  HostBuf hIn, hOut;   // pinned staging of the streamed host-pointer identity
  cudaEvent_t ev_io[4] = {};
  eigenid_gpu_ctx* peer[8] = {};
  ncclComm_t comm[8] = {};
};

namespace {

void set_err(eigenid_gpu_err* err, int code, long long index, double gap,
             int cuda_error, const std::string& msg) {
  if (!err) return;
  err->code = code;
  err->index = index;
  err->gap = gap;
  err->cuda_error = cuda_error;
  std::snprintf(err->msg, sizeof(err->msg), "%s", msg.c_str());
}

int cuda_fail(eigenid_gpu_err* err, cudaError_t e, const char* where) {
  const int code = (e == cudaErrorMemoryAllocation) ? EIGENID_E_ALLOC
                                                    : EIGENID_E_DEVICE;
  set_err(err, code, -1, 0.0, (int)e,
          std::string(where) + ": " + cudaGetErrorString(e));
  return code;
}

#define EID_CUDA(call, where)                          \
  do {                                                 \
    cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return cuda_fail(err, e_, where); \
  } while (0)

int check_cfg(const eigenid_gpu_config* cfg, eigenid_gpu_err* err) {
  if (!cfg) {
    set_err(err, EIGENID_E_CONFIG, -1, 0.0, 0, "null config");
    return EIGENID_E_CONFIG;
  }
  if (cfg->batch_size < 1) {  // identity.cpp:126
    set_err(err, EIGENID_E_CONFIG, -1, 0.0, 0, "batch size must be >= 1");
    return EIGENID_E_CONFIG;
  }
  if (!(cfg->degeneracy_tol >= 0.0)) {  // identity.cpp:127-128
    set_err(err, EIGENID_E_CONFIG, -1, 0.0, 0,
            "degeneracy tolerance must be >= 0");
    return EIGENID_E_CONFIG;
  }
  return EIGENID_OK;
}

int batch_of(const eigenid_gpu_config* cfg, int n) {
  // batch sizes beyond n-1 behave like a single batch (prepare_batches)
  return cfg->batch_size > (size_t)n ? n : (int)cfg->batch_size;
}

// Reads the device status (synchronising) and maps it to the C-ABI codes.
int finish(eigenid_gpu_ctx* c, eigenid_gpu_err* err, bool* degenerate) {
  EID_CUDA(cudaMemcpyAsync(c->hstatus, c->dstatus, 2 * sizeof(DevStatus),
                           cudaMemcpyDeviceToHost, c->stream),
           "status copy");
  EID_CUDA(cudaStreamSynchronize(c->stream), "stream sync");
  EID_CUDA(cudaGetLastError(), "kernel launch");
  c->pending = false;
  const DevStatus s = c->hstatus[0];
  if (degenerate) *degenerate = false;
  if (s.code == 0) return EIGENID_OK;
  char buf[200];
  switch (s.code) {
    case EIGENID_E_DEGENERATE:
      if (s.phase == 1 && degenerate) *degenerate = true;
      if (s.aux >= 0)
        std::snprintf(buf, sizeof buf,
                      "spectrum is degenerate between eigenvalues %lld and %lld"
                      " (matrix/row %lld)",
                      s.index, s.index + 1, s.aux);
      else
        std::snprintf(buf, sizeof buf,
                      "spectrum is degenerate between eigenvalues %lld and %lld",
                      s.index, s.index + 1);
      break;
    case EIGENID_E_INTERNAL:
      std::snprintf(buf, sizeof buf,
                    "reconstructed squared magnitude is negative; eigenvalue "
                    "ordering is inconsistent (i=%lld)", s.index);
      break;
    case EIGENID_E_CONVERGENCE:
      std::snprintf(buf, sizeof buf,
                    "eigenvalue solve did not converge (eigenvalue %lld of solve %lld)",
                    s.index, s.aux);
      break;
    case EIGENID_E_NONFINITE_ENTRY:
      std::snprintf(buf, sizeof buf, "matrix entry is not finite (entry %lld, matrix %lld)",
                    s.index, s.aux);
      break;
    case 30:  // kWaitTimeoutCode (band.cu, bulge.cu)
      c->wait_timed_out = true;
      std::snprintf(buf, sizeof buf,
                    "device-side wait timed out (site %lld, CTA*1000+warp %lld); "
                    "the call was abandoned", s.index, s.aux);
      set_err(err, EIGENID_E_DEVICE, s.index, 0.0, 0, buf);
      return EIGENID_E_DEVICE;
    default:
      std::snprintf(buf, sizeof buf, "device error code %d", s.code);
  }
  set_err(err, s.code, s.index, s.gap, 0, buf);
  return s.code;
}

int begin(eigenid_gpu_ctx* c, eigenid_gpu_err* err) {
  EID_CUDA(cudaSetDevice(c->device), "cudaSetDevice");
  if (c->pending) return EIGENID_OK;  // an unread device-call status is sticky
  init_status_kernel<<<1, 1, 0, c->stream>>>(c->dstatus);
  EID_CUDA(cudaGetLastError(), "init_status");
  c->launches += 1;
  return EIGENID_OK;
}

int check_finite(eigenid_gpu_ctx* c, const double* dA, size_t per, size_t count,
                 eigenid_gpu_err* err) {
  const long long total = (long long)(per * count);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  long long blocks = (total + 255) / 256;
  if (blocks > 8LL * sms) blocks = 8LL * sms;
  nonfinite_kernel<<<(unsigned)blocks, 256, 0, c->stream>>>(dA, (long long)per, total,
                                                           c->dstatus);
  EID_CUDA(cudaGetLastError(), "nonfinite check");
  c->launches += 1;
  return EIGENID_OK;
}

// NCCL, resolved at run time: the process may already hold the NCCL that
// PyTorch ships (libnccl.so.2 of nvidia-nccl), which is then reused
// (RTLD_NOLOAD); otherwise the system libnccl.so.2 is loaded.  Only
// multi-device contexts need it, so single-GPU users never load NCCL.
struct NcclApi {
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.comm_init_all = reinterpret_cast<decltype(a.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.broadcast = reinterpret_cast<decltype(a.broadcast)>(dlsym(h, "ncclBroadcast"));
    a.group_start = reinterpret_cast<decltype(a.group_start)>(dlsym(h, "ncclGroupStart"));
    a.group_end = reinterpret_cast<decltype(a.group_end)>(dlsym(h, "ncclGroupEnd"));
    a.error_string = reinterpret_cast<decltype(a.error_string)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.comm_init_all && a.comm_destroy && a.all_gather && a.broadcast &&
           a.group_start && a.group_end && a.error_string;
    return a;
  }();
  return api;
}

int nccl_fail(eigenid_gpu_err* err, ncclResult_t r, const char* where) {
  set_err(err, EIGENID_E_DEVICE, -1, 0.0, 0,
          std::string(where) + ": " + (nccl().error_string ? nccl().error_string(r) : "?"));
  return EIGENID_E_DEVICE;
}

// Per-stage device timing of run_large: enabled per context through
// eigenid_gpu_set_profiling (bench.py reads it to time the stage-1 kernel on
// its own stream) or EIGENID_PROFILE=1 (also printed to stderr).
// Same-box A/B: narrow wins at n = 1024 (89 ms vs 107 ms for the
// 1023 minors), widesp at n = 2048 (1127 vs 1161 ms) and n = 4096.
constexpr int kStage1WideMinN = 2048;
#ifndef EIGENID_STAGE1_LARGE_LAYOUT
#define EIGENID_STAGE1_LARGE_LAYOUT kWideSp
#endif
#define kStage1LargeLayout EIGENID_STAGE1_LARGE_LAYOUT
constexpr int kStages = 5;  // stage1, stage2, lambda_A (side), bisect_minors, identity
struct StageTimer {
  bool on = false, print = false;
  cudaStream_t st = nullptr;
  cudaEvent_t ev[4 * kStages + 1];
  int slot[4 * kStages + 1];
  int count = 0;
  double* sink = nullptr;  // ctx->stage_ms
  double side_ms = 0.0;     // A's pipeline on the side stream (slot 2)
  StageTimer(cudaStream_t s, bool enabled, double* out) : st(s), sink(out) {
    const char* e = std::getenv("EIGENID_PROFILE");
    print = e && e[0] == '1';
    on = enabled || print;
    mark(-1);
  }
  void mark(int stage) {
    if (!on || count > 4 * kStages) return;
    cudaEventCreate(&ev[count]);
    cudaEventRecord(ev[count], st);
    slot[count++] = stage;
  }
  ~StageTimer() {
    if (!on) return;
    if (print) std::fprintf(stderr, "[eigenid] %-14s %10.3f ms (side stream)\n", "lambda(A)", side_ms);
    static const char* names[kStages] = {"stage1", "stage2", "lambda_A",
                                         "bisect_minors", "identity"};
    cudaEventSynchronize(ev[count - 1]);
    for (int t = 0; t < kStages; ++t) sink[t] = 0.0;
    sink[2] = side_ms;
    for (int t = 1; t < count; ++t) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, ev[t - 1], ev[t]);
      sink[slot[t]] += ms;
      if (print) std::fprintf(stderr, "[eigenid] %-14s %10.3f ms\n", names[slot[t]], ms);
    }
    for (int t = 0; t < count; ++t) cudaEventDestroy(ev[t]);
  }
};

// Large-n pipeline for minor rows [j0, j1) of a device matrix.
//
// lambda(A) is solved on the context's side stream while the minors run on
// the main stream: A's stage 1 takes the SM the minors' persistent stage-1
// grid leaves free, then its chase, bisection and the degeneracy check
// (identity.cpp:299-300) run there too, and only then does that SM join the
// minors' work queue (the "helper" launch).  A degenerate lambda(A) sets the
// sticky status, so every stage's work queue stops pulling minors about one
// A-solve after the call started instead of after all n minor solves — the
// reference throws before it solves any minor.
int run_large(eigenid_gpu_ctx* c, const double* dA, int n, int j0, int j1,
              const eigenid_gpu_config* cfg, double* dout, double* dlam,
              double* dmu, bool identity, eigenid_gpu_err* err) {
  cudaStream_t st = c->stream, sa = c->side;
  const int rows = j1 - j0;  // minors; A is solved separately
  const int kB = stage1_bandwidth();
  const int ldab = stage1_band_ld();
  const int ldw = (n + 7) & ~7;
  const long long ws_stride = stage1_ws_doubles(n, ldw);
  const long long band_stride = (long long)n * ldab;
  (void)kB;
  // Memory plan: stage-1 workspace slots and the number of minors whose band
  // and tridiagonal are resident at once, sized to the free device memory
  // (large n is processed in chunks of minors).
  size_t free_b = 0, total_b = 0;
  EID_CUDA(cudaMemGetInfo(&free_b, &total_b), "cudaMemGetInfo");
  const double held = (double)(c->bWs.bytes + c->bBand.bytes + c->bD.bytes +
                               c->bE2.bytes + c->bAe.bytes);
  double budget = (double)free_b + held - 4.0e9;
  // EIGENID_MEM_BUDGET (bytes) caps the plan; the tests use it to force the
  // chunked schedule at small n.
  if (const char* mb = std::getenv("EIGENID_MEM_BUDGET")) {
    const double cap = std::atof(mb);
    if (cap > 0 && cap < budget) budget = cap;
  }
  const double ws_bytes = 8.0 * ws_stride;
  const double solve_bytes = 8.0 * (band_stride + 3.0 * n);
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c->device);
  // Stage-1 layout (band.cu): wide (one 16-warp CTA per SM) for large n,
  // narrow (two 8-warp CTAs per SM) where the panel phases weigh more.
  // wide8 (8 warps x 16 rows, one CTA per SM, 255 registers) replaces wide
  // where it measured faster.
  enum { kWide, kNarrow, kWide8, kWideSp } layout = n >= kStage1WideMinN ? kStage1LargeLayout : kNarrow;
  // EIGENID_STAGE1_LAYOUT=wide|narrow|wide8 overrides the choice (tests, A/B).
  if (const char* lay = std::getenv("EIGENID_STAGE1_LAYOUT")) {
    if (std::strcmp(lay, "wide") == 0) layout = kWide;
    if (std::strcmp(lay, "narrow") == 0) layout = kNarrow;
    if (std::strcmp(lay, "wide8") == 0) layout = kWide8;
    if (std::strcmp(lay, "widesp") == 0) layout = kWideSp;
  }
  const int cps = layout == kWide     ? wide::stage1_ctas_per_sm()
                  : layout == kWide8  ? wide8::stage1_ctas_per_sm()
                  : layout == kWideSp ? widesp::stage1_ctas_per_sm()
                                      : narrow::stage1_ctas_per_sm();
  auto launch1 = [&](const Stage1Args& a, int grid, cudaStream_t s, bool reset) {
    return layout == kWide     ? wide::launch_stage1(a, grid, s, reset)
           : layout == kWide8  ? wide8::launch_stage1(a, grid, s, reset)
           : layout == kWideSp ? widesp::launch_stage1(a, grid, s, reset)
                               : narrow::launch_stage1(a, grid, s, reset);
  };
  const int max_slots = sms * cps;
  // one SM's worth of slots is reserved for A's pipeline (then the helper)
  int slots = rows + cps < max_slots ? rows + cps : max_slots;
  while (slots > 1 && slots * ws_bytes > 0.7 * budget) slots = (slots + 1) / 2;
  long long chunk = (long long)((budget - slots * ws_bytes - solve_bytes) / solve_bytes);
  if (chunk > rows) chunk = rows;
  if (chunk < slots) chunk = slots;
  if (chunk < 1) chunk = 1;
  const bool side_ok = slots > cps;   // else A runs first, alone
  const int slot_a = side_ok ? slots - cps : 0;
  int launches = 0;
  EID_CUDA(c->bJs.ensure(sizeof(int) * (size_t)chunk), "alloc js");
  EID_CUDA(c->bJsA.ensure(sizeof(int)), "alloc jsA");
  EID_CUDA(c->bWs.ensure(sizeof(double) * (size_t)slots * ws_stride), "alloc ws");
  EID_CUDA(c->bBand.ensure(sizeof(double) * (size_t)chunk * band_stride), "alloc band");
  EID_CUDA(c->bBandA.ensure(sizeof(double) * (size_t)band_stride), "alloc bandA");
  EID_CUDA(c->bD.ensure(sizeof(double) * (size_t)chunk * n), "alloc d");
  EID_CUDA(c->bE2.ensure(sizeof(double) * (size_t)chunk * n), "alloc e2");
  EID_CUDA(c->bAe.ensure(sizeof(double) * (size_t)chunk * n), "alloc ae");
  EID_CUDA(c->bDeA.ensure(sizeof(double) * 3 * (size_t)n), "alloc deA");
  EID_CUDA(c->bCounter.ensure(sizeof(int) * 8), "alloc counter");
  int* djs = c->bJs.as<int>();
  int* djsA = c->bJsA.as<int>();
  int* ctr = c->bCounter.as<int>();  // [0] chase, [1] stage 1, [2] A stage 1, [3] A chase
  double* dA_d = c->bDeA.as<double>();

  StageTimer timer(st, c->profiling, c->stage_ms);
  // first chunk's solve list and queue, before A's pipeline forks off
  const int cnt0 = (int)(rows < chunk ? rows : chunk);
  EID_CUDA(cudaMemsetAsync(djsA, 0xff, sizeof(int), st), "jsA");  // -1 = A itself
  if (cnt0 > 0) {
    solve_list_kernel<<<(cnt0 + 255) / 256, 256, 0, st>>>(djs, j0, 0, cnt0);
    ++launches;
    EID_CUDA(cudaMemsetAsync(ctr + 1, 0, sizeof(int), st), "counter");
    EID_CUDA(cudaMemsetAsync(ctr + 4, 0, sizeof(int), st), "running flag");
  }
  EID_CUDA(c->bScale.ensure(sizeof(double) * 4), "alloc scale");
  double* dscale = c->bScale.as<double>();
  EID_CUDA(launch_input_scale(dA, (long long)n * n, dscale, st, &launches), "input scale");
  // EIGENID_BISECT_MAX_IT lowers the per-eigenvalue iteration budget (tests
  // drive the ConvergenceFailure path with it)
  int max_it = 300;
  if (const char* mi = std::getenv("EIGENID_BISECT_MAX_IT")) max_it = std::atoi(mi);
  EID_CUDA(cudaEventRecord(c->ev_start, st), "event");
  EID_CUDA(cudaStreamWaitEvent(sa, c->ev_start, 0), "event wait");
  // ---- side stream: lambda(A), the degeneracy check, then the helper
  EID_CUDA(cudaEventRecord(c->ev_a0, sa), "event");
  Stage1Args s1a{dA, n, djsA, 1, c->bWs.as<double>(), ws_stride, ldw,
                 c->bBandA.as<double>(), band_stride, ctr + 2, c->dstatus, slot_a,
                 dscale, nullptr, 0};
  EID_CUDA(launch1(s1a, 1, sa, true), "stage1 A");
  Stage2Args s2a{c->bBandA.as<double>(), band_stride, djsA, 1, n, dA_d, dA_d + n,
                 dA_d + 2 * n, n, ctr + 3, c->dstatus, c->device, cps > 1 ? 1 : 0};
  EID_CUDA(launch_stage2(s2a, sa), "stage2 A");
  BisectArgs ba{dA_d, dA_d + n, dA_d + 2 * n, n, djsA, 1, 0, n, nullptr, dlam, n,
                (n + 255) / 256, c->dstatus, dscale, max_it};
  EID_CUDA(launch_bisect(ba, 1, n, sa, &launches), "bisect A");
  launches += 2;
  if (identity)
    EID_CUDA(launch_degeneracy(dlam, n, cfg->degeneracy_tol, c->dstatus, sa, &launches),
             "degeneracy");
  EID_CUDA(cudaEventRecord(c->ev_a1, sa), "event");  // lambda(A) + degeneracy done
  Stage1Args s1{dA, n, djs, cnt0, c->bWs.as<double>(), ws_stride, ldw,
                c->bBand.as<double>(), band_stride, ctr + 1, c->dstatus, 0, dscale,
                ctr + 4, 0};
  const int grid_main = side_ok ? (cnt0 < slot_a ? cnt0 : slot_a) : (cnt0 < slots ? cnt0 : slots);
  if (side_ok && cnt0 > grid_main) {
    Stage1Args h = s1;
    h.slot0 = slot_a;
    h.helper = 1;
    const int hg = cnt0 - grid_main < cps ? cnt0 - grid_main : cps;
    EID_CUDA(launch1(h, hg, sa, false), "stage1 helper");
    ++launches;
  }
  EID_CUDA(cudaEventRecord(c->ev_a, sa), "event");

  // ---- main stream: the minors, chunk by chunk
  if (!side_ok) EID_CUDA(cudaStreamWaitEvent(st, c->ev_a, 0), "event wait");
  for (long long g0 = 0; g0 < rows; g0 += chunk) {
    const int cnt = (int)((rows - g0) < chunk ? (rows - g0) : chunk);
    if (g0 == 0) {
      EID_CUDA(launch1(s1, grid_main, st, false), "stage1");
      EID_CUDA(cudaStreamWaitEvent(st, c->ev_a, 0), "event wait");
    } else {
      solve_list_kernel<<<(cnt + 255) / 256, 256, 0, st>>>(djs, j0, (int)g0, cnt);
      ++launches;
      s1.nsolves = cnt;
      s1.running = nullptr;  // no helper for the later chunks
      EID_CUDA(launch1(s1, cnt < slots ? cnt : slots, st, true), "stage1");
    }
    ++launches;
    timer.mark(0);
    Stage2Args s2{c->bBand.as<double>(), band_stride, djs, cnt, n,
                  c->bD.as<double>(), c->bE2.as<double>(), c->bAe.as<double>(),
                  n, ctr, c->dstatus, c->device};
    EID_CUDA(launch_stage2(s2, st), "stage2");
    ++launches;
    timer.mark(1);
    BisectArgs bm{c->bD.as<double>(), c->bE2.as<double>(), c->bAe.as<double>(),
                  n, djs, cnt, 0, n, dlam, dmu + (size_t)g0 * (n - 1), n - 1, 1,
                  c->dstatus, dscale, max_it};
    EID_CUDA(launch_bisect(bm, cnt, n - 1, st, &launches), "bisect minors");
    timer.mark(3);
  }
  if (rows == 0) EID_CUDA(cudaStreamWaitEvent(st, c->ev_a, 0), "event wait");
  if (identity && rows > 0) {
    const int batch = batch_of(cfg, n);
    const int nb = identity_nb(n, batch);
    EID_CUDA(c->bDen.ensure(sizeof(double) * (size_t)n * nb), "alloc den");
    EID_CUDA(c->bRcp.ensure(sizeof(double) * (size_t)n * nb), "alloc rcp");
    const long long cap = 1 << 20;
    EID_CUDA(c->bFlags.ensure(sizeof(long long) * cap), "alloc flags");
    EID_CUDA(c->bFlagCount.ensure(sizeof(unsigned long long)), "alloc flagc");
    EID_CUDA(launch_identity(dlam, dmu, n, rows, batch, c->bDen.as<double>(),
                             c->bRcp.as<double>(), dout,
                             c->bFlagCount.as<unsigned long long>(),
                             c->bFlags.as<long long>(), cap, c->dstatus,
                             cfg->log_domain, st, &launches),
             "identity");
    timer.mark(4);
  }
  if (timer.on) {  // A's pipeline on the side stream (stage slot 2)
    float ms = 0.f;
    cudaEventSynchronize(c->ev_a);
    cudaEventElapsedTime(&ms, c->ev_a0, c->ev_a1);
    timer.side_ms = ms;
  }
  c->launches += launches;
  return EIGENID_OK;
}

// Full pipeline for rows [j0, j1) of a device matrix; dlam/dmu may be
// null (scratch is used).
int run_all(eigenid_gpu_ctx* c, const double* dA, int n, int j0, int j1,
            const eigenid_gpu_config* cfg, double* dout, double* dlam,
            double* dmu, eigenid_gpu_err* err) {
  const int rows = j1 - j0;
  if (!dlam) {
    EID_CUDA(c->bLam.ensure(sizeof(double) * n), "alloc lam");
    dlam = c->bLam.as<double>();
  }
  if (n <= kSmallMax) {
    const bool whole = (j0 == 0 && j1 == n);
    double* o = dout;
    double* mu = dmu;
    if (!whole) {
      EID_CUDA(c->bTmpOut.ensure(sizeof(double) * (size_t)n * n), "alloc tmp");
      EID_CUDA(c->bTmpMu.ensure(sizeof(double) * (size_t)n * (n - 1)), "alloc tmp");
      o = c->bTmpOut.as<double>();
      mu = c->bTmpMu.as<double>();
    }
    EID_CUDA(launch_small_all(dA, 1, n, batch_of(cfg, n), cfg->degeneracy_tol,
                              cfg->log_domain, o, dlam, mu, c->dstatus,
                              c->stream),
             "small");
    c->launches += 1;
    if (!whole) {
      EID_CUDA(cudaMemcpyAsync(dout, o + (size_t)j0 * n,
                               sizeof(double) * (size_t)rows * n,
                               cudaMemcpyDeviceToDevice, c->stream),
               "row copy");
      if (dmu)
        EID_CUDA(cudaMemcpyAsync(dmu, mu + (size_t)j0 * (n - 1),
                                 sizeof(double) * (size_t)rows * (n - 1),
                                 cudaMemcpyDeviceToDevice, c->stream),
                 "mu copy");
    }
    return EIGENID_OK;
  }
  if (!dmu) {
    EID_CUDA(c->bMu.ensure(sizeof(double) * (size_t)rows * (n - 1)), "alloc mu");
    dmu = c->bMu.as<double>();
  }
  return run_large(c, dA, n, j0, j1, cfg, dout, dlam, dmu, true, err);
}

int identity_impl(eigenid_gpu_ctx* c, const double* d_lambda,
                  const double* d_mu, size_t n, size_t j0, size_t j1,
                  const eigenid_gpu_config* cfg, double* d_out,
                  eigenid_gpu_err* err);

// Minor index j sharded over the devices of a multi-device context
// (SURVEY §8 e): device d owns the contiguous rows [d n / P, (d+1) n / P) of
// out[j*n+i], recomputes lambda(A) (1/n of the work) and writes its rows into
// its own full n x n buffer; one NCCL all-gather (in place; per-root
// broadcasts when P does not divide n) then leaves the whole matrix on every
// device.  Each (i, j) is computed by the same per-solve kernels whatever P
// is, so the result is bit-identical for every device count.
void shard_of(size_t n, int P, int d, size_t* j0, size_t* j1) {
  *j0 = n * (size_t)d / (size_t)P;
  *j1 = n * (size_t)(d + 1) / (size_t)P;
}

int multi_enqueue(eigenid_gpu_ctx* c, const double* const* dA, size_t n,
                  const eigenid_gpu_config* cfg, double* const* dfull,
                  double* const* dlam, double* const* dmu, eigenid_gpu_err* err) {
  const int P = c->ngpu;
  for (int d = 0; d < P; ++d) {
    eigenid_gpu_ctx* p = c->peer[d];
    size_t j0, j1;
    shard_of(n, P, d, &j0, &j1);
    int st;
    if ((st = begin(p, err))) return st;
    p->pending = true;
    if ((st = check_finite(p, dA[d], n * n, 1, err))) return st;
    if ((st = run_all(p, dA[d], (int)n, (int)j0, (int)j1, cfg, dfull[d] + j0 * n, dlam[d],
                      dmu[d], err)))
      return st;
  }
  if (!c->multi) return EIGENID_OK;  // a single-device context: nothing to gather
  const NcclApi& api = nccl();
  ncclResult_t r = api.group_start();
  if (r != ncclSuccess) return nccl_fail(err, r, "ncclGroupStart");
  if (n % (size_t)P == 0) {
    const size_t cnt = n / P * n;
    for (int d = 0; d < P; ++d) {
      EID_CUDA(cudaSetDevice(c->peer[d]->device), "cudaSetDevice");
      r = api.all_gather(dfull[d] + (size_t)d * cnt, dfull[d], cnt, ncclFloat64, c->comm[d],
                         c->peer[d]->stream);
      if (r != ncclSuccess) {
        api.group_end();
        return nccl_fail(err, r, "ncclAllGather");
      }
    }
  } else {
    for (int root = 0; root < P; ++root) {
      size_t j0, j1;
      shard_of(n, P, root, &j0, &j1);
      for (int d = 0; d < P; ++d) {
        EID_CUDA(cudaSetDevice(c->peer[d]->device), "cudaSetDevice");
        r = api.broadcast(dfull[d] + j0 * n, dfull[d] + j0 * n, (j1 - j0) * n, ncclFloat64,
                          root, c->comm[d], c->peer[d]->stream);
        if (r != ncclSuccess) {
          api.group_end();
          return nccl_fail(err, r, "ncclBroadcast");
        }
      }
    }
  }
  r = api.group_end();
  if (r != ncclSuccess) return nccl_fail(err, r, "ncclGroupEnd");
  return EIGENID_OK;
}

// Reads every device's status (first failing device wins).
int multi_finish(eigenid_gpu_ctx* c, eigenid_gpu_err* err, bool* degenerate) {
  int first = EIGENID_OK;
  for (int d = 0; d < c->ngpu; ++d) {
    eigenid_gpu_err e{};
    bool dg = false;
    EID_CUDA(cudaSetDevice(c->peer[d]->device), "cudaSetDevice");
    const int st = finish(c->peer[d], &e, &dg);
    if (st && first == EIGENID_OK) {
      first = st;
      if (err) *err = e;
      if (degenerate) *degenerate = dg;
    }
  }
  return first;
}

int all_magnitudes_multi(eigenid_gpu_ctx* c, const double* a, size_t n,
                         const eigenid_gpu_config* cfg, double* out, double* lambda_out,
                         double* mu_out, eigenid_gpu_err* err) {
  const int P = c->ngpu;
  const double* dA[8];
  double* dfull[8];
  double* dlam[8];
  double* dmu[8];
  for (int d = 0; d < P; ++d) {
    eigenid_gpu_ctx* p = c->peer[d];
    size_t j0, j1;
    shard_of(n, P, d, &j0, &j1);
    EID_CUDA(cudaSetDevice(p->device), "cudaSetDevice");
    EID_CUDA(p->bA.ensure(sizeof(double) * n * n), "alloc A");
    EID_CUDA(p->bOut.ensure(sizeof(double) * n * n), "alloc out");
    EID_CUDA(p->bLam.ensure(sizeof(double) * n), "alloc lam");
    EID_CUDA(p->bMu.ensure(sizeof(double) * (j1 > j0 ? j1 - j0 : 1) * (n - 1)), "alloc mu");
    EID_CUDA(cudaMemcpyAsync(p->bA.p, a, sizeof(double) * n * n, cudaMemcpyHostToDevice,
                             p->stream), "H2D A");
    dA[d] = p->bA.as<double>();
    dfull[d] = p->bOut.as<double>();
    dlam[d] = p->bLam.as<double>();
    dmu[d] = p->bMu.as<double>();
  }
  int st = multi_enqueue(c, dA, n, cfg, dfull, dlam, dmu, err);
  if (st) return st;
  EID_CUDA(cudaSetDevice(c->device), "cudaSetDevice");
  EID_CUDA(cudaMemcpyAsync(out, dfull[0], sizeof(double) * n * n, cudaMemcpyDeviceToHost,
                           c->stream), "D2H out");
  if (lambda_out)
    EID_CUDA(cudaMemcpyAsync(lambda_out, dlam[0], sizeof(double) * n,
                             cudaMemcpyDeviceToHost, c->stream), "D2H lambda");
  if (mu_out)
    for (int d = 0; d < P; ++d) {
      size_t j0, j1;
      shard_of(n, P, d, &j0, &j1);
      if (j1 == j0) continue;
      EID_CUDA(cudaSetDevice(c->peer[d]->device), "cudaSetDevice");
      EID_CUDA(cudaMemcpyAsync(mu_out + j0 * (n - 1), dmu[d],
                               sizeof(double) * (j1 - j0) * (n - 1), cudaMemcpyDeviceToHost,
                               c->peer[d]->stream), "D2H mu");
    }
  bool degenerate = false;
  st = multi_finish(c, err, &degenerate);
  c->solves += st == EIGENID_E_NONFINITE_ENTRY
                   ? 0
                   : ((st == EIGENID_E_DEGENERATE && degenerate) ? 1 : n + 1);
  return st;
}

int check_n(size_t n, eigenid_gpu_err* err) {
  if (n < 2) {  // identity.cpp:296-297
    set_err(err, EIGENID_E_MATRIX_TOO_SMALL, -1, 0.0, 0,
            "component magnitudes need n >= 2");
    return EIGENID_E_MATRIX_TOO_SMALL;
  }
  if (n > (size_t)kLargeMax) {
    set_err(err, EIGENID_E_CONFIG, -1, 0.0, 0,
            "n exceeds the eigensolver's supported size (14000)");
    return EIGENID_E_CONFIG;
  }
  return EIGENID_OK;
}

}  // namespace

namespace {
// SeededDraws (matrix_io.cpp:39-71): std::mt19937_64 and the hand-written
// variate transforms, so inputs are bit-identical to the reference's.
struct SeededDraws {
  std::mt19937_64 gen;
  bool have_spare = false;
  double spare = 0.0;
  explicit SeededDraws(uint64_t seed) : gen(seed) {}
  double unit() { return static_cast<double>(gen() >> 11) * 0x1.0p-53; }
  double uniform_open() {
    for (;;) {
      const double v = 2.0 * unit() - 1.0;
      if (v > -1.0) return v;
    }
  }
  double gaussian() {
    if (have_spare) {
      have_spare = false;
      return spare;
    }
    double u1 = unit();
    const double u2 = unit();
    while (u1 <= 0.0) u1 = unit();
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double theta = 2.0 * M_PI * u2;
    spare = r * std::sin(theta);
    have_spare = true;
    return r * std::cos(theta);
  }
};
}  // namespace

extern "C" {

void eigenid_random_symmetric(uint64_t seed, size_t n, int uniform, double* e) {
  SeededDraws d(seed);
  for (size_t t = 0; t < n * n; ++t) e[t] = uniform ? d.uniform_open() : d.gaussian();
  double asym = 0.0;  // build(kSymmetrize), matrix.cpp:20-36
  for (size_t r = 0; r < n; ++r)
    for (size_t c = r + 1; c < n; ++c) asym = std::fmax(asym, std::fabs(e[r * n + c] - e[c * n + r]));
  if (asym > 0.0)
    for (size_t r = 0; r < n; ++r)
      for (size_t c = r + 1; c < n; ++c) {
        const double m = 0.5 * (e[r * n + c] + e[c * n + r]);
        e[r * n + c] = m;
        e[c * n + r] = m;
      }
}

// C3 input: Householder QR of the seeded Gaussian G
// (row-major draws), Q sign-fixed by diag(R), A = Q diag(linspace(-1,1)) Q^T,
// build(kSymmetrize).  Plain loops in a fixed order, no BLAS, so every host
// produces the same bytes (a LAPACK QR differs across CPU kernels).
void eigenid_c3_matrix(uint64_t seed, size_t n, double* out) {
  std::vector<double> g(n * n), w(n * n), p(n * n, 0.0), beta(n), rdiag(n);
  eigenid_seeded_draws(seed, n * n, 0, g.data());
  for (size_t r = 0; r < n; ++r)
    for (size_t c = 0; c < n; ++c) w[c * n + r] = g[r * n + c];
  for (size_t k = 0; k < n; ++k) {  // W = G^T; row k holds column k
    double* x = w.data() + k * n;
    double ss = 0.0;
    for (size_t t = k; t < n; ++t) ss += x[t] * x[t];
    const double nrm = std::sqrt(ss);
    const double alpha = x[k] >= 0.0 ? -nrm : nrm;
    rdiag[k] = alpha;
    if (nrm == 0.0) {
      beta[k] = 0.0;
      continue;
    }
    x[k] -= alpha;  // Householder vector v = x - alpha e_k, in place
    double vv = 0.0;
    for (size_t t = k; t < n; ++t) vv += x[t] * x[t];
    beta[k] = 2.0 / vv;
    for (size_t j = k + 1; j < n; ++j) {
      double* y = w.data() + j * n;
      double d = 0.0;
      for (size_t t = k; t < n; ++t) d += x[t] * y[t];
      const double sc = beta[k] * d;
      for (size_t t = k; t < n; ++t) y[t] -= sc * x[t];
    }
  }
  for (size_t t = 0; t < n; ++t) p[t * n + t] = 1.0;  // P = Q^T, backward accumulation
  for (size_t k = n; k-- > 0;) {
    if (beta[k] == 0.0) continue;
    const double* v = w.data() + k * n;
    for (size_t r = k; r < n; ++r) {
      double* pr = p.data() + r * n;
      double d = 0.0;
      for (size_t t = k; t < n; ++t) d += pr[t] * v[t];
      const double sc = beta[k] * d;
      for (size_t t = k; t < n; ++t) pr[t] -= sc * v[t];
    }
  }
  for (size_t k = 0; k < n; ++k)
    if (rdiag[k] < 0.0)
      for (size_t t = 0; t < n; ++t) p[k * n + t] = -p[k * n + t];
  for (size_t t = 0; t < n * n; ++t) out[t] = 0.0;
  for (size_t k = 0; k < n; ++k) {  // A = sum_k lambda_k q_k q_k^T
    const double lk = -1.0 + 2.0 * (double)k / (double)(n - 1);
    const double* q = p.data() + k * n;
    for (size_t r = 0; r < n; ++r) {
      const double sc = lk * q[r];
      double* ar = out + r * n;
      for (size_t c = 0; c < n; ++c) ar[c] += sc * q[c];
    }
  }
  for (size_t r = 0; r < n; ++r)
    for (size_t c = r + 1; c < n; ++c) {
      const double m = 0.5 * (out[r * n + c] + out[c * n + r]);
      out[r * n + c] = m;
      out[c * n + r] = m;
    }
}

void eigenid_seeded_draws(uint64_t seed, size_t count, int kind, double* out) {
  SeededDraws d(seed);
  for (size_t t = 0; t < count; ++t) out[t] = kind ? d.uniform_open() : d.gaussian();
}

int eigenid_gpu_abi_version(void) { return EIGENID_B200_ABI_VERSION; }

int eigenid_gpu_device_count(void) {
  int c = 0;
  if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
  return c;
}

int eigenid_gpu_create(eigenid_gpu_ctx** out, int device, eigenid_gpu_err* err) {
  if (!out) {
    set_err(err, EIGENID_E_CONFIG, -1, 0.0, 0, "null ctx pointer");
    return EIGENID_E_CONFIG;
  }
  *out = nullptr;
  int count = 0;
  cudaError_t e = cudaGetDeviceCount(&count);
  if (e != cudaSuccess || count <= device || device < 0) {
    set_err(err, EIGENID_E_DEVICE, -1, 0.0, (int)e,
            "no CUDA device available (the B200 path has no CPU fallback)");
    return EIGENID_E_DEVICE;
  }
  auto* c = new (std::nothrow) eigenid_gpu_ctx();
  if (!c) {
    set_err(err, EIGENID_E_ALLOC, -1, 0.0, 0, "host allocation failed");
    return EIGENID_E_ALLOC;
  }
  c->device = device;
  c->peer[0] = c;
  if ((e = cudaSetDevice(device)) != cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking)) !=
          cudaSuccess ||
      (e = cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking)) != cudaSuccess ||
      (e = cudaEventCreateWithFlags(&c->ev_start, cudaEventDisableTiming)) != cudaSuccess ||
      (e = cudaEventCreate(&c->ev_a)) != cudaSuccess ||
      (e = cudaEventCreate(&c->ev_a0)) != cudaSuccess ||
      (e = cudaEventCreate(&c->ev_a1)) != cudaSuccess ||
      (e = cudaMalloc(&c->dstatus, 2 * sizeof(DevStatus))) != cudaSuccess ||
      (e = cudaMallocHost(&c->hstatus, 2 * sizeof(DevStatus))) != cudaSuccess) {
    delete c;
    return cuda_fail(err, e, "context creation");
  }
  *out = c;
  return EIGENID_OK;
}

int eigenid_gpu_create_multi(eigenid_gpu_ctx** out, int first_device, int num_gpus,
                             eigenid_gpu_err* err) {
  if (!out) {
    set_err(err, EIGENID_E_CONFIG, -1, 0.0, 0, "null ctx pointer");
    return EIGENID_E_CONFIG;
  }
  *out = nullptr;
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
  if (num_gpus < 1 || num_gpus > 8 || first_device < 0 || first_device + num_gpus > count) {
    set_err(err, num_gpus < 1 || num_gpus > 8 ? EIGENID_E_CONFIG : EIGENID_E_DEVICE, -1, 0.0,
            0, "num_gpus must be 1..8 and every device must exist");
    return num_gpus < 1 || num_gpus > 8 ? EIGENID_E_CONFIG : EIGENID_E_DEVICE;
  }
  if (!nccl().ok) {
    set_err(err, EIGENID_E_DEVICE, -1, 0.0, 0, "libnccl.so.2 could not be loaded");
    return EIGENID_E_DEVICE;
  }
  eigenid_gpu_ctx* c = nullptr;
  int st = eigenid_gpu_create(&c, first_device, err);
  if (st) return st;
  c->ngpu = num_gpus;
  c->multi = true;
  c->peer[0] = c;
  for (int d = 1; d < num_gpus; ++d) {
    if ((st = eigenid_gpu_create(&c->peer[d], first_device + d, err))) {
      eigenid_gpu_destroy(c);
      return st;
    }
  }
  int devs[8];
  for (int d = 0; d < num_gpus; ++d) devs[d] = first_device + d;
  const ncclResult_t r = nccl().comm_init_all(c->comm, num_gpus, devs);
  if (r != ncclSuccess) {
    for (int d = 0; d < 8; ++d) c->comm[d] = nullptr;
    eigenid_gpu_destroy(c);
    return nccl_fail(err, r, "ncclCommInitAll");
  }
  *out = c;
  return EIGENID_OK;
}

int eigenid_gpu_num_devices(eigenid_gpu_ctx* c) { return c ? c->ngpu : 0; }

void* eigenid_gpu_device_stream(eigenid_gpu_ctx* c, int d) {
  if (!c || d < 0 || d >= c->ngpu) return nullptr;
  return (void*)c->peer[d]->stream;
}

int eigenid_gpu_destroy(eigenid_gpu_ctx* c) {
  if (!c) return EIGENID_OK;
  if (c->multi) {
    for (int d = 0; d < c->ngpu; ++d) {
      if (c->comm[d]) nccl().comm_destroy(c->comm[d]);
      c->comm[d] = nullptr;
    }
    for (int d = 1; d < c->ngpu; ++d) eigenid_gpu_destroy(c->peer[d]);
    c->ngpu = 1;
  }
  cudaSetDevice(c->device);
  cudaStreamSynchronize(c->stream);
  for (DevBuf* b : {&c->bA, &c->bOut, &c->bLam, &c->bMu, &c->bDen, &c->bRcp,
                    &c->bFlags, &c->bFlagCount, &c->bWs, &c->bBand, &c->bD,
                    &c->bE2, &c->bAe, &c->bJs, &c->bTmpOut, &c->bTmpMu,
                    &c->bCounter, &c->bBandA, &c->bDeA, &c->bJsA, &c->bScale})
    b->release();
  cudaFree(c->dstatus);
  cudaFreeHost(c->hstatus);
  c->hIn.release();
  c->hOut.release();
  for (cudaEvent_t& ev : c->ev_io)
    if (ev) cudaEventDestroy(ev);
  cudaEventDestroy(c->ev_start);
  cudaEventDestroy(c->ev_a);
  cudaEventDestroy(c->ev_a0);
  cudaEventDestroy(c->ev_a1);
  cudaStreamDestroy(c->side);
  cudaStreamDestroy(c->stream);
  delete c;
  return EIGENID_OK;
}

void* eigenid_gpu_stream(eigenid_gpu_ctx* c) { return c ? (void*)c->stream : nullptr; }

int eigenid_gpu_sync(eigenid_gpu_ctx* c, eigenid_gpu_err* err) {
  std::lock_guard<std::mutex> g(c->mu);
  if (c->multi) return multi_finish(c, err, nullptr);
  return finish(c, err, nullptr);
}

int eigenid_gpu_all_magnitudes_multi_device(eigenid_gpu_ctx* c, const double* const* d_a,
                                            size_t n, const eigenid_gpu_config* cfg,
                                            double* const* d_out, eigenid_gpu_err* err) {
  int st = check_n(n, err);
  if (st) return st;
  if ((st = check_cfg(cfg, err))) return st;
  std::lock_guard<std::mutex> g(c->mu);
  const int P = c->ngpu;
  double* dlam[8];
  double* dmu[8];
  for (int d = 0; d < P; ++d) {
    eigenid_gpu_ctx* p = c->peer[d];
    size_t j0, j1;
    shard_of(n, P, d, &j0, &j1);
    EID_CUDA(cudaSetDevice(p->device), "cudaSetDevice");
    EID_CUDA(p->bLam.ensure(sizeof(double) * n), "alloc lam");
    EID_CUDA(p->bMu.ensure(sizeof(double) * (j1 > j0 ? j1 - j0 : 1) * (n - 1)), "alloc mu");
    dlam[d] = p->bLam.as<double>();
    dmu[d] = p->bMu.as<double>();
  }
  st = multi_enqueue(c, d_a, n, cfg, d_out, dlam, dmu, err);
  if (st == EIGENID_OK) c->solves += n + 1;
  return st;
}

size_t eigenid_gpu_solve_count(eigenid_gpu_ctx* c) { return c->solves.load(); }
void eigenid_gpu_reset_solve_count(eigenid_gpu_ctx* c) { c->solves.store(0); }
uint64_t eigenid_gpu_launch_count(eigenid_gpu_ctx* c) {
  uint64_t t = c->launches.load();
  for (int d = 1; d < c->ngpu; ++d) t += c->peer[d]->launches.load();
  return t;
}

void eigenid_gpu_set_profiling(eigenid_gpu_ctx* c, int on) { c->profiling = on != 0; }

int eigenid_gpu_stage_times(eigenid_gpu_ctx* c, double* ms, int cap) {
  std::lock_guard<std::mutex> g(c->mu);
  const int k = cap < 5 ? cap : 5;
  for (int t = 0; t < k; ++t) ms[t] = c->stage_ms[t];
  return k;
}

int eigenid_gpu_eigenvalues(eigenid_gpu_ctx* c, const double* a, size_t n,
                            double* out, eigenid_gpu_err* err) {
  if (n < 1) {
    set_err(err, EIGENID_E_CONFIG, -1, 0.0, 0, "matrix dimension must be >= 1");
    return EIGENID_E_CONFIG;
  }
  if (n > (size_t)kLargeMax) return check_n(n, err);
  std::lock_guard<std::mutex> g(c->mu);
  c->solves += 1;
  if (n == 1) {  // tridiagonalize + QL of a 1x1 is the entry itself
    out[0] = a[0];
    return EIGENID_OK;
  }
  int st = begin(c, err);
  if (st) return st;
  EID_CUDA(c->bA.ensure(sizeof(double) * n * n), "alloc A");
  EID_CUDA(c->bLam.ensure(sizeof(double) * n), "alloc lam");
  EID_CUDA(cudaMemcpyAsync(c->bA.p, a, sizeof(double) * n * n,
                           cudaMemcpyHostToDevice, c->stream),
           "H2D A");
  if ((st = check_finite(c, c->bA.as<double>(), n * n, 1, err))) return st;
  eigenid_gpu_config cfg{64, 0.0, 0};
  st = run_large(c, c->bA.as<double>(), (int)n, 0, 0, &cfg, nullptr,
                 c->bLam.as<double>(), nullptr, false, err);
  if (st) return st;
  EID_CUDA(cudaMemcpyAsync(out, c->bLam.p, sizeof(double) * n,
                           cudaMemcpyDeviceToHost, c->stream),
           "D2H lambda");
  return finish(c, err, nullptr);
}

static int all_magnitudes_once(eigenid_gpu_ctx* c, const double* a, size_t n,
                               const eigenid_gpu_config* cfg, double* out,
                               double* lambda_out, double* mu_out,
                               eigenid_gpu_err* err, bool* degenerate_out) {
  int st;
  if ((st = begin(c, err))) return st;
  const size_t nn = n * n;
  EID_CUDA(c->bA.ensure(sizeof(double) * nn), "alloc A");
  EID_CUDA(c->bOut.ensure(sizeof(double) * nn), "alloc out");
  EID_CUDA(c->bLam.ensure(sizeof(double) * n), "alloc lam");
  EID_CUDA(c->bMu.ensure(sizeof(double) * n * (n - 1)), "alloc mu");
  EID_CUDA(cudaMemcpyAsync(c->bA.p, a, sizeof(double) * nn,
                           cudaMemcpyHostToDevice, c->stream),
           "H2D A");
  if ((st = check_finite(c, c->bA.as<double>(), nn, 1, err))) return st;
  st = run_all(c, c->bA.as<double>(), (int)n, 0, (int)n, cfg,
               c->bOut.as<double>(), c->bLam.as<double>(), c->bMu.as<double>(),
               err);
  if (st) return st;
  EID_CUDA(cudaMemcpyAsync(out, c->bOut.p, sizeof(double) * nn,
                           cudaMemcpyDeviceToHost, c->stream),
           "D2H out");
  if (lambda_out)
    EID_CUDA(cudaMemcpyAsync(lambda_out, c->bLam.p, sizeof(double) * n,
                             cudaMemcpyDeviceToHost, c->stream),
             "D2H lambda");
  if (mu_out)
    EID_CUDA(cudaMemcpyAsync(mu_out, c->bMu.p, sizeof(double) * n * (n - 1),
                             cudaMemcpyDeviceToHost, c->stream),
             "D2H mu");
  return finish(c, err, degenerate_out);
}

int eigenid_gpu_all_magnitudes(eigenid_gpu_ctx* c, const double* a, size_t n,
                               const eigenid_gpu_config* cfg, double* out,
                               double* lambda_out, double* mu_out,
                               eigenid_gpu_err* err) {
  int st = check_n(n, err);
  if (st) return st;
  if ((st = check_cfg(cfg, err))) return st;
  std::lock_guard<std::mutex> g(c->mu);
  if (c->multi) return all_magnitudes_multi(c, a, n, cfg, out, lambda_out, mu_out, err);
  bool degenerate = false;
  c->wait_timed_out = false;
  st = all_magnitudes_once(c, a, n, cfg, out, lambda_out, mu_out, err, &degenerate);
  if (c->wait_timed_out) {
    // A bounded device-side wait ran out (band.cu kWaitTimeoutCode): the
    // kernels have unwound and the context is healthy; the pipeline is
    // idempotent, so the call is repeated once before the error is reported.
    std::fprintf(stderr, "[eigenid] %s -- retrying the call once\n", err ? err->msg : "");
    c->wait_timed_out = false;
    degenerate = false;
    if (err) std::memset(err, 0, sizeof *err);
    st = all_magnitudes_once(c, a, n, cfg, out, lambda_out, mu_out, err, &degenerate);
  }
  // identity.cpp:299-306: lambda(A) is solved, then the degeneracy check
  // throws before the n minor solves.
  // NonFiniteEntry: build() throws before any solve (matrix.cpp:17-18)
  c->solves += st == EIGENID_E_NONFINITE_ENTRY
                   ? 0
                   : ((st == EIGENID_E_DEGENERATE && degenerate) ? 1 : n + 1);
  return st;
}

int eigenid_gpu_all_magnitudes_batched(eigenid_gpu_ctx* c, const double* a,
                                       size_t count, size_t n,
                                       const eigenid_gpu_config* cfg,
                                       double* out, eigenid_gpu_err* err) {
  int st = check_n(n, err);
  if (st) return st;
  if ((st = check_cfg(cfg, err))) return st;
  if (count == 0) return EIGENID_OK;
  std::lock_guard<std::mutex> g(c->mu);
  if ((st = begin(c, err))) return st;
  const size_t tot = count * n * n;
  EID_CUDA(c->bA.ensure(sizeof(double) * tot), "alloc A");
  EID_CUDA(c->bOut.ensure(sizeof(double) * tot), "alloc out");
  EID_CUDA(cudaMemcpyAsync(c->bA.p, a, sizeof(double) * tot,
                           cudaMemcpyHostToDevice, c->stream),
           "H2D A");
  if ((st = check_finite(c, c->bA.as<double>(), n * n, count, err))) return st;
  if (n <= (size_t)kSmallMax) {
    EID_CUDA(launch_small_all(c->bA.as<double>(), count, (int)n,
                              batch_of(cfg, (int)n), cfg->degeneracy_tol,
                              cfg->log_domain, c->bOut.as<double>(), nullptr,
                              nullptr, c->dstatus, c->stream),
             "small batched");
    c->launches += 1;
  } else {
    EID_CUDA(c->bLam.ensure(sizeof(double) * n), "alloc lam");
    EID_CUDA(c->bMu.ensure(sizeof(double) * n * (n - 1)), "alloc mu");
    for (size_t t = 0; t < count; ++t) {
      st = run_all(c, c->bA.as<double>() + t * n * n, (int)n, 0, (int)n, cfg,
                   c->bOut.as<double>() + t * n * n, c->bLam.as<double>(),
                   c->bMu.as<double>(), err);
      if (st) return st;
    }
  }
  EID_CUDA(cudaMemcpyAsync(out, c->bOut.p, sizeof(double) * tot,
                           cudaMemcpyDeviceToHost, c->stream),
           "D2H out");
  st = finish(c, err, nullptr);
  if (st == EIGENID_OK) c->solves += count * (n + 1);
  return st;
}

int eigenid_gpu_minor_spectra(eigenid_gpu_ctx* c, const double* a, size_t n,
                              size_t j0, size_t j1, double* lambda, double* mu,
                              eigenid_gpu_err* err) {
  int st = check_n(n, err);
  if (st) return st;
  if (j0 > j1 || j1 > n) {
    set_err(err, EIGENID_E_INDEX, -1, 0.0, 0, "minor range out of bounds");
    return EIGENID_E_INDEX;
  }
  std::lock_guard<std::mutex> g(c->mu);
  if ((st = begin(c, err))) return st;
  const size_t rows = j1 - j0;
  EID_CUDA(c->bA.ensure(sizeof(double) * n * n), "alloc A");
  EID_CUDA(c->bLam.ensure(sizeof(double) * n), "alloc lam");
  EID_CUDA(c->bMu.ensure(sizeof(double) * (rows ? rows : 1) * (n - 1)), "alloc mu");
  EID_CUDA(cudaMemcpyAsync(c->bA.p, a, sizeof(double) * n * n,
                           cudaMemcpyHostToDevice, c->stream),
           "H2D A");
  if ((st = check_finite(c, c->bA.as<double>(), n * n, 1, err))) return st;
  eigenid_gpu_config cfg{64, 0.0, 0};
  st = run_large(c, c->bA.as<double>(), (int)n, (int)j0, (int)j1, &cfg, nullptr,
                 c->bLam.as<double>(), c->bMu.as<double>(), false, err);
  if (st) return st;
  if (lambda)
    EID_CUDA(cudaMemcpyAsync(lambda, c->bLam.p, sizeof(double) * n,
                             cudaMemcpyDeviceToHost, c->stream),
             "D2H lambda");
  if (rows)
    EID_CUDA(cudaMemcpyAsync(mu, c->bMu.p, sizeof(double) * rows * (n - 1),
                             cudaMemcpyDeviceToHost, c->stream),
             "D2H mu");
  st = finish(c, err, nullptr);
  if (st == EIGENID_OK) c->solves += 1 + rows;
  return st;
}

}  // extern "C"

namespace {
// Host-pointer identity stage for inputs larger than one staging chunk
// (C5: 8.6 GB of mu in, 8.6 GB of |v|^2 out): rows stream through two pinned
// buffers each way, so the host copies of chunk c+1 / c-1 and the transfers
// overlap the identity kernel of chunk c.  Every row is computed by the same
// kernel whatever the chunking, so the bits are those of the one-shot path.
int identity_streamed(eigenid_gpu_ctx* c, const double* lambda, const double* mu,
                      size_t n, size_t rows, size_t chunk,
                      const eigenid_gpu_config* cfg, double* out, eigenid_gpu_err* err) {
  const size_t nch = (rows + chunk - 1) / chunk;
  const size_t in_row = n - 1, out_row = n;
  EID_CUDA(c->hIn.ensure(sizeof(double) * 2 * chunk * in_row), "pinned in");
  EID_CUDA(c->hOut.ensure(sizeof(double) * 2 * chunk * out_row), "pinned out");
  EID_CUDA(c->bMu.ensure(sizeof(double) * 2 * chunk * in_row), "alloc mu");
  EID_CUDA(c->bOut.ensure(sizeof(double) * 2 * chunk * out_row), "alloc out");
  for (cudaEvent_t& ev : c->ev_io)
    if (!ev) EID_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming), "event");
  int launches = 0;
  EID_CUDA(launch_degeneracy(c->bLam.as<double>(), (int)n, cfg->degeneracy_tol, c->dstatus,
                             c->stream, &launches), "degeneracy");
  const int batch = batch_of(cfg, (int)n);
  const int nb = identity_nb((int)n, batch);
  EID_CUDA(c->bDen.ensure(sizeof(double) * n * nb), "alloc den");
  EID_CUDA(c->bRcp.ensure(sizeof(double) * n * nb), "alloc rcp");
  const long long cap = 1 << 20;
  EID_CUDA(c->bFlags.ensure(sizeof(long long) * cap), "alloc flags");
  EID_CUDA(c->bFlagCount.ensure(sizeof(unsigned long long)), "alloc flagc");
  auto rows_of = [&](size_t k) { return std::min(chunk, rows - k * chunk); };
  for (size_t k = 0; k <= nch; ++k) {
    if (k < nch) {
      const int s = (int)(k & 1);
      double* hin = c->hIn.as<double>() + s * chunk * in_row;
      if (k >= 2) EID_CUDA(cudaEventSynchronize(c->ev_io[s]), "in slot");
      std::memcpy(hin, mu + k * chunk * in_row, sizeof(double) * rows_of(k) * in_row);
      double* dmu = c->bMu.as<double>() + s * chunk * in_row;
      double* dout = c->bOut.as<double>() + s * chunk * out_row;
      EID_CUDA(cudaMemcpyAsync(dmu, hin, sizeof(double) * rows_of(k) * in_row,
                               cudaMemcpyHostToDevice, c->stream), "H2D mu");
      EID_CUDA(cudaEventRecord(c->ev_io[s], c->stream), "event");
      EID_CUDA(launch_identity(c->bLam.as<double>(), dmu, (int)n, (int)rows_of(k), batch,
                               c->bDen.as<double>(), c->bRcp.as<double>(), dout,
                               c->bFlagCount.as<unsigned long long>(),
                               c->bFlags.as<long long>(), cap, c->dstatus, cfg->log_domain,
                               c->stream, &launches), "identity");
      EID_CUDA(cudaMemcpyAsync(c->hOut.as<double>() + s * chunk * out_row, dout,
                               sizeof(double) * rows_of(k) * out_row, cudaMemcpyDeviceToHost,
                               c->stream), "D2H out");
      EID_CUDA(cudaEventRecord(c->ev_io[2 + s], c->stream), "event");
    }
    if (k >= 1) {  // chunk k-1's rows, while the device works on chunk k
      const int s = (int)((k - 1) & 1);
      EID_CUDA(cudaEventSynchronize(c->ev_io[2 + s]), "out slot");
      std::memcpy(out + (k - 1) * chunk * out_row, c->hOut.as<double>() + s * chunk * out_row,
                  sizeof(double) * rows_of(k - 1) * out_row);
    }
  }
  c->launches += launches;
  return EIGENID_OK;
}
}  // namespace

extern "C" {

int eigenid_gpu_identity(eigenid_gpu_ctx* c, const double* lambda,
                         const double* mu, size_t n, size_t j0, size_t j1,
                         const eigenid_gpu_config* cfg, double* out,
                         eigenid_gpu_err* err) {
  if (n < 2) return check_n(n, err);
  int st = check_cfg(cfg, err);
  if (st) return st;
  if (j0 > j1 || j1 > n) {
    set_err(err, EIGENID_E_INDEX, -1, 0.0, 0, "row range out of bounds");
    return EIGENID_E_INDEX;
  }
  const size_t rows = j1 - j0;
  if (rows == 0) return EIGENID_OK;
  std::lock_guard<std::mutex> g(c->mu);
  if ((st = begin(c, err))) return st;
  EID_CUDA(c->bLam.ensure(sizeof(double) * n), "alloc lam");
  // more than ~4 chunks of 256 MB of output: stream the rows
  size_t chunk = ((size_t)(256u << 20) / (sizeof(double) * n)) & ~(size_t)31;
  if (chunk < 32) chunk = 32;
  if (!cfg->log_domain && rows >= 4 * chunk) {
    EID_CUDA(cudaMemcpyAsync(c->bLam.p, lambda, sizeof(double) * n, cudaMemcpyHostToDevice,
                             c->stream), "H2D lambda");
    if ((st = identity_streamed(c, lambda, mu, n, rows, chunk, cfg, out, err))) return st;
    return finish(c, err, nullptr);
  }
  EID_CUDA(c->bMu.ensure(sizeof(double) * rows * (n - 1)), "alloc mu");
  EID_CUDA(c->bOut.ensure(sizeof(double) * rows * n), "alloc out");
  EID_CUDA(cudaMemcpyAsync(c->bLam.p, lambda, sizeof(double) * n,
                           cudaMemcpyHostToDevice, c->stream),
           "H2D lambda");
  EID_CUDA(cudaMemcpyAsync(c->bMu.p, mu, sizeof(double) * rows * (n - 1),
                           cudaMemcpyHostToDevice, c->stream),
           "H2D mu");
  st = identity_impl(c, c->bLam.as<double>(), c->bMu.as<double>(), n, j0, j1,
                     cfg, c->bOut.as<double>(), err);
  if (st) return st;
  EID_CUDA(cudaMemcpyAsync(out, c->bOut.p, sizeof(double) * rows * n,
                           cudaMemcpyDeviceToHost, c->stream),
           "D2H out");
  return finish(c, err, nullptr);
}

int eigenid_gpu_identity_device(eigenid_gpu_ctx* c, const double* d_lambda,
                                const double* d_mu, size_t n, size_t j0,
                                size_t j1, const eigenid_gpu_config* cfg,
                                double* d_out, eigenid_gpu_err* err) {
  if (n < 2) return check_n(n, err);
  int st = check_cfg(cfg, err);
  if (st) return st;
  if (j0 > j1 || j1 > n) {
    set_err(err, EIGENID_E_INDEX, -1, 0.0, 0, "row range out of bounds");
    return EIGENID_E_INDEX;
  }
  std::lock_guard<std::mutex> g(c->mu);
  if ((st = begin(c, err))) return st;
  st = identity_impl(c, d_lambda, d_mu, n, j0, j1, cfg, d_out, err);
  c->pending = true;
  return st;
}

}  // extern "C"

namespace {
int identity_impl(eigenid_gpu_ctx* c, const double* d_lambda,
                  const double* d_mu, size_t n, size_t j0, size_t j1,
                  const eigenid_gpu_config* cfg, double* d_out,
                  eigenid_gpu_err* err) {
  const int rows = (int)(j1 - j0);
  if (rows <= 0) return EIGENID_OK;
  int launches = 0;
  const int batch = batch_of(cfg, (int)n);
  const int nb = identity_nb((int)n, batch);
  EID_CUDA(c->bDen.ensure(sizeof(double) * n * nb), "alloc den");
  EID_CUDA(c->bRcp.ensure(sizeof(double) * n * nb), "alloc rcp");
  const long long cap = 1 << 20;
  EID_CUDA(c->bFlags.ensure(sizeof(long long) * cap), "alloc flags");
  EID_CUDA(c->bFlagCount.ensure(sizeof(unsigned long long)), "alloc flagc");
  EID_CUDA(launch_degeneracy(d_lambda, (int)n, cfg->degeneracy_tol, c->dstatus,
                             c->stream, &launches),
           "degeneracy");
  EID_CUDA(launch_identity(d_lambda, d_mu, (int)n, rows, batch,
                           c->bDen.as<double>(), c->bRcp.as<double>(), d_out,
                           c->bFlagCount.as<unsigned long long>(),
                           c->bFlags.as<long long>(), cap, c->dstatus,
                           cfg->log_domain, c->stream, &launches),
           "identity");
  c->launches += launches;
  return EIGENID_OK;
}
}  // namespace

extern "C" {

int eigenid_gpu_all_magnitudes_device(eigenid_gpu_ctx* c, const double* d_a,
                                      size_t n, size_t j0, size_t j1,
                                      const eigenid_gpu_config* cfg,
                                      double* d_out, double* d_lambda,
                                      double* d_mu, eigenid_gpu_err* err) {
  int st = check_n(n, err);
  if (st) return st;
  if ((st = check_cfg(cfg, err))) return st;
  if (j0 > j1 || j1 > n) {
    set_err(err, EIGENID_E_INDEX, -1, 0.0, 0, "row range out of bounds");
    return EIGENID_E_INDEX;
  }
  std::lock_guard<std::mutex> g(c->mu);
  if ((st = begin(c, err))) return st;
  c->pending = true;
  if ((st = check_finite(c, d_a, n * n, 1, err))) return st;
  st = run_all(c, d_a, (int)n, (int)j0, (int)j1, cfg, d_out, d_lambda, d_mu, err);
  if (st == EIGENID_OK) c->solves += 1 + (j1 - j0);
  return st;
}

int eigenid_gpu_all_magnitudes_batched_device(eigenid_gpu_ctx* c,
                                              const double* d_a, size_t count,
                                              size_t n,
                                              const eigenid_gpu_config* cfg,
                                              double* d_out,
                                              eigenid_gpu_err* err) {
  int st = check_n(n, err);
  if (st) return st;
  if ((st = check_cfg(cfg, err))) return st;
  if (n > (size_t)kSmallMax) {
    set_err(err, EIGENID_E_CONFIG, -1, 0.0, 0,
            "batched device entry supports n <= 64");
    return EIGENID_E_CONFIG;
  }
  std::lock_guard<std::mutex> g(c->mu);
  if ((st = begin(c, err))) return st;
  c->pending = true;
  if ((st = check_finite(c, d_a, n * n, count, err))) return st;
  EID_CUDA(launch_small_all(d_a, count, (int)n, batch_of(cfg, (int)n),
                            cfg->degeneracy_tol, cfg->log_domain, d_out,
                            nullptr, nullptr, c->dstatus, c->stream),
           "small batched");
  c->launches += 1;
  c->solves += count * (n + 1);
  return EIGENID_OK;
}

}  // extern "C"

namespace {
// vector_magnitudes (identity.cpp:276-292): lambda(A), the n minor spectra,
// check_nondegenerate(i), then evaluate() for every j.  raw / method (n
// each) and the condition flag of eigenvalue i.
int vector_impl(eigenid_gpu_ctx* c, const double* a, size_t n, size_t i,
                const eigenid_gpu_config* cfg, std::vector<double>& raw,
                std::vector<double>& method, double* cond, eigenid_gpu_err* err) {
  int st = check_n(n, err);
  if (st) return st;
  if ((st = check_cfg(cfg, err))) return st;
  if (i >= n) {  // check_component_indices(a, i, 0), identity.cpp:28-36
    set_err(err, EIGENID_E_INDEX, (long long)i, 0.0, 0, "component index out of range");
    return EIGENID_E_INDEX;
  }
  std::lock_guard<std::mutex> g(c->mu);
  if ((st = begin(c, err))) return st;
  EID_CUDA(c->bA.ensure(sizeof(double) * n * n), "alloc A");
  EID_CUDA(c->bLam.ensure(sizeof(double) * n), "alloc lam");
  EID_CUDA(c->bMu.ensure(sizeof(double) * n * (n - 1)), "alloc mu");
  EID_CUDA(c->bOut.ensure(sizeof(double) * (2 * n + 4)), "alloc out");
  EID_CUDA(cudaMemcpyAsync(c->bA.p, a, sizeof(double) * n * n,
                           cudaMemcpyHostToDevice, c->stream), "H2D A");
  if ((st = check_finite(c, c->bA.as<double>(), n * n, 1, err))) return st;
  eigenid_gpu_config scfg{64, 0.0, 0};
  st = run_large(c, c->bA.as<double>(), (int)n, 0, (int)n, &scfg, nullptr,
                 c->bLam.as<double>(), c->bMu.as<double>(), false, err);
  if (st) return st;
  int launches = 0;
  double* dout = c->bOut.as<double>();
  // check_nondegenerate for eigenvalue i (identity.cpp:137-139, :281) and
  // its condition flag (component (i, 0) evaluated into the tail)
  EID_CUDA(launch_component(c->bLam.as<double>(), c->bMu.as<double>(), (int)n,
                            (int)i, batch_of(cfg, (int)n), cfg->degeneracy_tol,
                            cfg->log_domain, 0, dout + 2 * n, c->dstatus,
                            c->stream, &launches), "gap check");
  EID_CUDA(launch_vector(c->bLam.as<double>(), c->bMu.as<double>(), (int)n,
                         (int)i, batch_of(cfg, (int)n), cfg->log_domain, dout, dout + n,
                         c->dstatus, c->stream, &launches), "vector");
  c->launches += launches;
  std::vector<double> h(2 * n + 4);
  EID_CUDA(cudaMemcpyAsync(h.data(), dout, sizeof(double) * (2 * n + 4),
                           cudaMemcpyDeviceToHost, c->stream), "D2H");
  bool degenerate = false;
  st = finish(c, err, &degenerate);
  c->solves += st == EIGENID_E_NONFINITE_ENTRY
                   ? 0
                   : ((st == EIGENID_E_DEGENERATE && degenerate) ? 1 : n + 1);
  if (st) return st;
  raw.assign(h.begin(), h.begin() + n);
  method.assign(h.begin() + n, h.begin() + 2 * n);
  *cond = h[2 * n + 3];
  return EIGENID_OK;
}

inline double clamp01h(double x) { return x < 0.0 ? 0.0 : (1.0 < x ? 1.0 : x); }
}  // namespace

extern "C" {

int eigenid_gpu_vector_magnitudes(eigenid_gpu_ctx* c, const double* a,
                                  size_t n, size_t i,
                                  const eigenid_gpu_config* cfg, double* out,
                                  double* out_raw, eigenid_gpu_err* err) {
  std::vector<double> raw, method;
  double cond = 0.0;
  const int st = vector_impl(c, a, n, i, cfg, raw, method, &cond, err);
  if (st) return st;
  for (size_t t = 0; t < n; ++t) {
    out[t] = clamp01h(raw[t]);
    if (out_raw) out_raw[t] = raw[t];
  }
  return EIGENID_OK;
}

int eigenid_gpu_vector(eigenid_gpu_ctx* c, const double* a, size_t n, size_t i,
                       const eigenid_gpu_config* cfg, eigenid_gpu_magnitude* out,
                       eigenid_gpu_err* err) {
  std::vector<double> raw, method;
  double cond = 0.0;
  const int st = vector_impl(c, a, n, i, cfg, raw, method, &cond, err);
  if (st) return st;
  for (size_t t = 0; t < n; ++t) {
    out[t].value = clamp01h(raw[t]);
    out[t].raw_value = raw[t];
    out[t].i = i;
    out[t].j = t;
    out[t].method = (int)method[t];
    out[t].condition_flag = cond;
  }
  return EIGENID_OK;
}

int eigenid_gpu_log_domain_product(eigenid_gpu_ctx* c, const double* num,
                                   const double* den, size_t len, double* out,
                                   eigenid_gpu_err* err) {
  std::lock_guard<std::mutex> g(c->mu);
  int st;
  if ((st = begin(c, err))) return st;
  EID_CUDA(c->bOut.ensure(sizeof(double) * (2 * len + 2)), "alloc factors");
  double* d = c->bOut.as<double>();
  if (len) {
    EID_CUDA(cudaMemcpyAsync(d, num, sizeof(double) * len, cudaMemcpyHostToDevice,
                             c->stream), "H2D num");
    EID_CUDA(cudaMemcpyAsync(d + len, den, sizeof(double) * len,
                             cudaMemcpyHostToDevice, c->stream), "H2D den");
  }
  int launches = 0;
  EID_CUDA(launch_log_product(d, d + len, (long long)len, d + 2 * len, c->dstatus,
                              c->stream, &launches), "log product");
  c->launches += launches;
  double h = 0.0;
  EID_CUDA(cudaMemcpyAsync(&h, d + 2 * len, sizeof(double), cudaMemcpyDeviceToHost,
                           c->stream), "D2H");
  if ((st = finish(c, err, nullptr))) {
    if (st == EIGENID_E_DEGENERATE)
      set_err(err, st, -1, 0.0, 0, "zero denominator factor");  // identity.cpp:110
    return st;
  }
  *out = h;
  return EIGENID_OK;
}

// tridiagonalize (eigensolve.hpp:41): the device reduction (dense -> band ->
// tridiagonal) of A; an orthogonally similar tridiagonal, not tred1's own.
int eigenid_gpu_tridiagonalize(eigenid_gpu_ctx* c, const double* a, size_t n,
                               double* diag, double* offdiag, eigenid_gpu_err* err) {
  if (n < 1) {
    set_err(err, EIGENID_E_DIMENSION, -1, 0.0, 0, "matrix dimension must be >= 1");
    return EIGENID_E_DIMENSION;
  }
  if (n > (size_t)kLargeMax) return check_n(n, err);
  if (n == 1) {
    diag[0] = a[0];
    return EIGENID_OK;
  }
  std::lock_guard<std::mutex> g(c->mu);
  int st;
  if ((st = begin(c, err))) return st;
  EID_CUDA(c->bA.ensure(sizeof(double) * n * n), "alloc A");
  EID_CUDA(c->bLam.ensure(sizeof(double) * n), "alloc lam");
  EID_CUDA(c->bOut.ensure(sizeof(double) * 2 * n), "alloc out");
  EID_CUDA(cudaMemcpyAsync(c->bA.p, a, sizeof(double) * n * n, cudaMemcpyHostToDevice,
                           c->stream), "H2D A");
  if ((st = check_finite(c, c->bA.as<double>(), n * n, 1, err))) return st;
  eigenid_gpu_config cfg{64, 0.0, 0};
  st = run_large(c, c->bA.as<double>(), (int)n, 0, 0, &cfg, nullptr,
                 c->bLam.as<double>(), nullptr, false, err);
  if (st) return st;
  int launches = 0;
  // the chased band of A holds (d, e) scaled by the exact input scale
  EID_CUDA(launch_band_tridiag(c->bBandA.as<double>(), stage1_band_ld(), (int)n,
                               c->bOut.as<double>(), c->bOut.as<double>() + n, c->stream,
                               &launches), "band tridiag");
  c->launches += launches;
  std::vector<double> h(2 * n), sc(2);
  EID_CUDA(cudaMemcpyAsync(h.data(), c->bOut.p, sizeof(double) * 2 * n,
                           cudaMemcpyDeviceToHost, c->stream), "D2H");
  EID_CUDA(cudaMemcpyAsync(sc.data(), c->bScale.p, sizeof(double) * 2,
                           cudaMemcpyDeviceToHost, c->stream), "D2H scale");
  if ((st = finish(c, err, nullptr))) return st;
  for (size_t k = 0; k < n; ++k) diag[k] = h[k] * sc[1];
  for (size_t k = 0; k + 1 < n; ++k) offdiag[k] = h[n + k] * sc[1];
  return EIGENID_OK;
}

// eigenvalues(TridiagonalForm) (eigensolve.cpp:72-128): Sturm bisection of
// the given (diag, offdiag) on the device, ascending.
int eigenid_gpu_tridiagonal_eigenvalues(eigenid_gpu_ctx* c, const double* diag,
                                        const double* offdiag, size_t n, double* out,
                                        eigenid_gpu_err* err) {
  if (n == 0) return EIGENID_OK;
  if (n > (size_t)kLargeMax) return check_n(n, err);
  if (n == 1) {
    out[0] = diag[0];
    return EIGENID_OK;
  }
  std::lock_guard<std::mutex> g(c->mu);
  int st;
  if ((st = begin(c, err))) return st;
  EID_CUDA(c->bOut.ensure(sizeof(double) * 2 * n), "alloc de");
  EID_CUDA(c->bDeA.ensure(sizeof(double) * 3 * n), "alloc deA");
  EID_CUDA(c->bLam.ensure(sizeof(double) * n), "alloc out");
  EID_CUDA(c->bJsA.ensure(sizeof(int)), "alloc js");
  EID_CUDA(c->bScale.ensure(sizeof(double) * 4), "alloc scale");
  double* de = c->bOut.as<double>();
  EID_CUDA(cudaMemcpyAsync(de, diag, sizeof(double) * n, cudaMemcpyHostToDevice,
                           c->stream), "H2D d");
  EID_CUDA(cudaMemcpyAsync(de + n, offdiag, sizeof(double) * (n - 1),
                           cudaMemcpyHostToDevice, c->stream), "H2D e");
  EID_CUDA(cudaMemsetAsync(c->bJsA.p, 0xff, sizeof(int), c->stream), "js");
  int launches = 0;
  double* dscale = c->bScale.as<double>();
  EID_CUDA(launch_input_scale(de, 2LL * n - 1, dscale, c->stream, &launches), "scale");
  double* d3 = c->bDeA.as<double>();
  EID_CUDA(launch_tridiag_prepare(de, (int)n, dscale, d3, d3 + n, d3 + 2 * n, c->stream,
                                  &launches), "prepare");
  int max_it = 300;
  if (const char* mi = std::getenv("EIGENID_BISECT_MAX_IT")) max_it = std::atoi(mi);
  BisectArgs ba{d3, d3 + n, d3 + 2 * n, (long long)n, c->bJsA.as<int>(), 1, 0, (int)n,
                nullptr, c->bLam.as<double>(), (long long)n, (int)((n + 255) / 256),
                c->dstatus, dscale, max_it};
  EID_CUDA(launch_bisect(ba, 1, (int)n, c->stream, &launches), "bisect");
  c->launches += launches;
  EID_CUDA(cudaMemcpyAsync(out, c->bLam.p, sizeof(double) * n, cudaMemcpyDeviceToHost,
                           c->stream), "D2H");
  return finish(c, err, nullptr);
}

// ---- sign recovery (signs.cpp:48-120) ------------------------------------
namespace {
int recover_impl(eigenid_gpu_ctx* c, const double* dA, size_t n, const double* dm,
                 double lambda_i, double sign_tol, double* dv, eigenid_gpu_err* err) {
  EID_CUDA(c->bWs.ensure(sizeof(double) * (size_t)recover_ws_doubles((int)n)), "alloc ws");
  EID_CUDA(c->bCounter.ensure(recover_state_bytes() > 16 ? recover_state_bytes() : 16),
           "alloc state");
  auto* stp = reinterpret_cast<RecoverState*>(c->bCounter.p);
  int launches = 0;
  EID_CUDA(launch_recover_signs(dA, (int)n, dm, lambda_i, sign_tol, dv, c->bWs.as<double>(),
                                stp, c->stream, &launches),
           "recover_signs");
  c->launches += launches;
  RecoverResult r;
  EID_CUDA(recover_result(stp, &r, c->stream), "recover state");
  if (r.singular) {
    set_err(err, EIGENID_E_SIGN_RECOVERY, -1, 0.0, 0,
            "row equations are singular at the anchor");
    return EIGENID_E_SIGN_RECOVERY;
  }
  const double res = std::sqrt(r.res2), bound = 1e-6 * std::sqrt(r.fro2);
  if (res > bound) {  // signs.cpp:113-118 (std::to_string formatting)
    char buf[160];
    std::snprintf(buf, sizeof buf, "sign recovery residual %f exceeds %f", res, bound);
    set_err(err, EIGENID_E_SIGN_RECOVERY, -1, 0.0, 0, buf);
    return EIGENID_E_SIGN_RECOVERY;
  }
  return EIGENID_OK;
}
}  // namespace

int eigenid_gpu_recover_signs(eigenid_gpu_ctx* c, const double* a, size_t n, size_t i,
                              const double* magnitudes, size_t n_magnitudes,
                              double lambda_i, double sign_tol, double* out_v,
                              eigenid_gpu_err* err) {
  (void)i;  // unused by the reference too (signs.cpp:54)
  if (n_magnitudes != n) {
    set_err(err, EIGENID_E_DIMENSION, -1, 0.0, 0, "magnitude vector length does not match n");
    return EIGENID_E_DIMENSION;
  }
  if (n == 0) return EIGENID_OK;
  if (n > 14000) {
    set_err(err, EIGENID_E_CONFIG, -1, 0.0, 0, "n exceeds the device limit (14000)");
    return EIGENID_E_CONFIG;
  }
  std::lock_guard<std::mutex> g(c->mu);
  int st;
  if ((st = begin(c, err))) return st;
  EID_CUDA(c->bA.ensure(sizeof(double) * n * n), "alloc A");
  EID_CUDA(c->bLam.ensure(sizeof(double) * n), "alloc mags");
  EID_CUDA(c->bOut.ensure(sizeof(double) * n), "alloc out");
  EID_CUDA(cudaMemcpyAsync(c->bA.p, a, sizeof(double) * n * n, cudaMemcpyHostToDevice,
                           c->stream), "H2D A");
  EID_CUDA(cudaMemcpyAsync(c->bLam.p, magnitudes, sizeof(double) * n, cudaMemcpyHostToDevice,
                           c->stream), "H2D mags");
  st = recover_impl(c, c->bA.as<double>(), n, c->bLam.as<double>(), lambda_i, sign_tol,
                    c->bOut.as<double>(), err);
  if (st) return st;
  EID_CUDA(cudaMemcpyAsync(out_v, c->bOut.p, sizeof(double) * n, cudaMemcpyDeviceToHost,
                           c->stream), "D2H v");
  EID_CUDA(cudaStreamSynchronize(c->stream), "sync");
  return EIGENID_OK;
}

int eigenid_gpu_recover_signs_device(eigenid_gpu_ctx* c, const double* d_a, size_t n,
                                     const double* d_magnitudes, double lambda_i,
                                     double sign_tol, double* d_out, eigenid_gpu_err* err) {
  if (n == 0) return EIGENID_OK;
  if (n > 14000) {
    set_err(err, EIGENID_E_CONFIG, -1, 0.0, 0, "n exceeds the device limit (14000)");
    return EIGENID_E_CONFIG;
  }
  std::lock_guard<std::mutex> g(c->mu);
  int st;
  if ((st = begin(c, err))) return st;
  return recover_impl(c, d_a, n, d_magnitudes, lambda_i, sign_tol, d_out, err);
}

}  // extern "C"

namespace {
// One component through the reference's per-component entries
// (identity.cpp:151-183 baseline, :240-251 component_magnitude, :253-274
// log_domain_magnitude).  Cached spectra (lambda and mu_j both given) skip
// the two solves; the baseline always solves, as the reference's does.
// out4 = {value, raw, method, condition_flag}.
int component_impl(eigenid_gpu_ctx* c, const double* a, size_t n, size_t i,
                   size_t j, const double* lambda, const double* mu_j,
                   const eigenid_gpu_config* cfg, int variant, double* out4,
                   eigenid_gpu_err* err) {
  if (n < 2) return check_n(n, err);
  int st = check_cfg(cfg, err);
  if (st) return st;
  if (i >= n || j >= n) {  // check_component_indices, identity.cpp:28-36
    char buf[160];
    std::snprintf(buf, sizeof buf, "component index (i=%zu, j=%zu) out of range for n = %zu",
                  i, j, n);
    set_err(err, EIGENID_E_INDEX, -1, 0.0, 0, buf);
    return EIGENID_E_INDEX;
  }
  const bool cached = lambda && mu_j && variant != 2;
  std::lock_guard<std::mutex> g(c->mu);
  if ((st = begin(c, err))) return st;
  EID_CUDA(c->bLam.ensure(sizeof(double) * n), "alloc lam");
  EID_CUDA(c->bMu.ensure(sizeof(double) * n), "alloc mu");
  EID_CUDA(c->bOut.ensure(sizeof(double) * 4), "alloc out");
  size_t solves = 0;
  if (cached) {
    EID_CUDA(cudaMemcpyAsync(c->bLam.p, lambda, sizeof(double) * n,
                             cudaMemcpyHostToDevice, c->stream), "H2D lambda");
    EID_CUDA(cudaMemcpyAsync(c->bMu.p, mu_j, sizeof(double) * (n - 1),
                             cudaMemcpyHostToDevice, c->stream), "H2D mu");
  } else {
    if (n > (size_t)kLargeMax) return check_n(n, err);
    EID_CUDA(c->bA.ensure(sizeof(double) * n * n), "alloc A");
    EID_CUDA(cudaMemcpyAsync(c->bA.p, a, sizeof(double) * n * n,
                             cudaMemcpyHostToDevice, c->stream), "H2D A");
    if ((st = check_finite(c, c->bA.as<double>(), n * n, 1, err))) return st;
    eigenid_gpu_config scfg{64, 0.0, 0};
    st = run_large(c, c->bA.as<double>(), (int)n, (int)j, (int)j + 1, &scfg,
                   nullptr, c->bLam.as<double>(), c->bMu.as<double>(), false,
                   err);
    if (st) return st;
    solves = 2;
  }
  int launches = 0;
  const int logd = variant == 1 ? 1 : cfg->log_domain;
  EID_CUDA(launch_component(c->bLam.as<double>(), c->bMu.as<double>(), (int)n,
                            (int)i, batch_of(cfg, (int)n), cfg->degeneracy_tol,
                            logd, variant, c->bOut.as<double>(), c->dstatus,
                            c->stream, &launches), "component");
  c->launches += launches;
  EID_CUDA(cudaMemcpyAsync(out4, c->bOut.p, sizeof(double) * 4,
                           cudaMemcpyDeviceToHost, c->stream), "D2H");
  st = finish(c, err, nullptr);
  c->solves += st == EIGENID_E_NONFINITE_ENTRY ? 0 : solves;
  if (st == EIGENID_E_NONFINITE) {
    static const char* what[4] = {"", "numerator product left the finite range",
                                  "denominator product left the finite range",
                                  "factor ratio is not finite"};  // identity.cpp:163-174
    const long long k = c->hstatus[0].aux;
    set_err(err, st, -1, 0.0, 0, what[k >= 1 && k <= 3 ? k : 3]);
  }
  return st;
}
}  // namespace

extern "C" {

int eigenid_gpu_component_magnitude(eigenid_gpu_ctx* c, const double* a,
                                    size_t n, size_t i, size_t j,
                                    const double* lambda, const double* mu_j,
                                    const eigenid_gpu_config* cfg,
                                    double* value, double* raw, int* method,
                                    eigenid_gpu_err* err) {
  double h[4];
  const int st = component_impl(c, a, n, i, j, lambda, mu_j, cfg, 0, h, err);
  if (st) return st;
  *value = h[0];
  if (raw) *raw = h[1];
  if (method) *method = (int)h[2];
  return EIGENID_OK;
}

int eigenid_gpu_component(eigenid_gpu_ctx* c, const double* a, size_t n, size_t i,
                          size_t j, const double* lambda, const double* mu_j,
                          const eigenid_gpu_config* cfg, int variant,
                          eigenid_gpu_magnitude* out, eigenid_gpu_err* err) {
  if (variant < 0 || variant > 2) {
    set_err(err, EIGENID_E_CONFIG, -1, 0.0, 0, "unknown component variant");
    return EIGENID_E_CONFIG;
  }
  double h[4];
  const int st = component_impl(c, a, n, i, j, lambda, mu_j, cfg, variant, h, err);
  if (st) return st;
  out->value = h[0];
  out->raw_value = h[1];
  out->i = i;
  out->j = j;
  out->method = (int)h[2];
  out->condition_flag = h[3];
  return EIGENID_OK;
}

int eigenid_gpu_c5_mu_device(eigenid_gpu_ctx* c, uint64_t seed,
                             const double* d_lambda, size_t n, size_t j0,
                             size_t j1, double* d_mu, eigenid_gpu_err* err) {
  if (n < 2) return check_n(n, err);
  std::lock_guard<std::mutex> g(c->mu);
  int launches = 0;
  EID_CUDA(launch_c5_mu(seed, d_lambda, (int)n, (int)j0, (int)(j1 - j0), d_mu,
                        c->stream, &launches),
           "c5 mu");
  c->launches += launches;
  return EIGENID_OK;
}

}  // extern "C"
