"""cuBLAS FP64 / complex128 GEMM throughput on the local GPU (library reference
point for the FP64 roofline; our own kernels never call cuBLAS)."""
import json
import torch

def bench(dtype, n, reps=10):
    a = torch.randn(n, n, dtype=dtype, device="cuda")
    b = torch.randn(n, n, dtype=dtype, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    mult = 8 if dtype.is_complex else 2
    return mult * n ** 3 / (best * 1e-3) / 1e12

out = {}
for n in (1024, 4096, 8192):
    out[f"dgemm_{n}_tflops"] = bench(torch.float64, n)
for n in (256, 1024, 4096):
    out[f"zgemm_{n}_tflops"] = bench(torch.complex128, n)
print(json.dumps(out))
