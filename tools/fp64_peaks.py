"""Measure FP64 / complex128 GEMM peaks with cuBLAS via torch (yardstick only)."""
import json, torch
def bench(dtype, n, reps=10):
    a = torch.randn(n, n, dtype=dtype, device="cuda"); b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(3): a @ b
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); a @ b; e1.record(); e1.synchronize(); best = min(best, e0.elapsed_time(e1))
    mult = 8 if dtype.is_complex else 2
    return mult * n**3 / best / 1e9
out = {"dgemm_tflops_8192": bench(torch.float64, 8192), "zgemm_tflops_4096": bench(torch.complex128, 4096),
       "dgemm_tflops_512": bench(torch.float64, 512, 50), "zgemm_tflops_512": bench(torch.complex128, 512, 50)}
print(json.dumps(out))
