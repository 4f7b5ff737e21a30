"""cuBLAS FP64 GEMM throughput on the shapes of the stage-1 updates
(calibration only — not used by the product)."""
import torch
torch.backends.cuda.matmul.allow_tf32 = False
dev = "cuda"
def bench(m, n, k, reps=10):
    a = torch.randn(m, k, dtype=torch.float64, device=dev)
    b = torch.randn(k, n, dtype=torch.float64, device=dev)
    c = torch.randn(m, n, dtype=torch.float64, device=dev)
    for _ in range(3):
        c.addmm_(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        c.addmm_(a, b)
    e1.record(); e1.synchronize()
    t = e0.elapsed_time(e1) / 1e3 / reps
    return 2.0 * m * n * k / t / 1e12
for (m, n, k) in [(8192, 8192, 8192), (4096, 4096, 4096), (4095, 4095, 64), (4095, 4095, 32),
                  (4095, 32, 4095), (16384, 16384, 64), (1023, 1023, 64)]:
    print(f"dgemm m={m} n={n} k={k}: {bench(m, n, k):.2f} TFLOP/s", flush=True)
# batched: 148 independent rank-64 updates of 4095^2 (the stage-1 GEMM2 shape per SM)
a = torch.randn(148, 4095, 64, dtype=torch.float64, device=dev)
b = torch.randn(148, 64, 4095, dtype=torch.float64, device=dev)
c = torch.randn(148, 4095, 4095, dtype=torch.float64, device=dev)
for _ in range(2): c.baddbmm_(a, b)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); c.baddbmm_(a, b); e1.record(); e1.synchronize()
t = e0.elapsed_time(e1) / 1e3
print(f"batched 148 x (4095^2 += 4095x64 . 64x4095): {2*148*4095*4095*64/t/1e12:.2f} TFLOP/s")
for (m, n, k) in [(4095, 4095, 128), (4095, 64, 4095), (4095, 4095, 256), (4095, 128, 4095)]:
    print(f"dgemm m={m} n={n} k={k}: {bench(m, n, k):.2f} TFLOP/s", flush=True)
