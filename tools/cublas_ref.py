"""cuBLAS (torch.matmul) timing of the predictor's layer-1/2 shapes, for context only."""
import torch

for (M, K, N) in [(2048, 4096, 2048), (512, 4096, 2048), (4096, 4096, 2048), (4096, 5120, 2048), (2048, 2048, 512),
                  (8192, 8192, 8192)]:
    a = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
    b = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
    for _ in range(10):
        c = a @ b.t()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 50
    e0.record()
    for _ in range(n):
        c = a @ b.t()
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) / n * 1e3
    print(f"cuBLAS M={M} K={K} N={N}: {t:8.2f} us  {2 * M * N * K / t / 1e6:8.1f} TFLOP/s")
