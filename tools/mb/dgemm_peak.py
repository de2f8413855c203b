"""Development aid: cuBLAS fp64 GEMM throughput on this GPU (the DMMA roofline reference for the
Gram / Cholesky kernels). Prints TFLOP/s for a few square sizes (best of 5, CUDA events)."""
import torch
for n in (4096, 8192, 16384):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b)
    best = 1e9
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"DGEMM n={n}: {2 * n ** 3 / best / 1e9:.1f} TFLOP/s ({best:.2f} ms)", flush=True)
