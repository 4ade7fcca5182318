"""Library context: cuBLAS DGEMM throughput via torch.matmul(float64) on this B200."""
import torch, time
for n in (4096, 8192, 16384):
    a = torch.rand(n, n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3): c = a @ b
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5 if n < 16384 else 2
    e0.record()
    for _ in range(reps): c = a @ b
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print(f"cublas dgemm n={n}: {ms:.3f} ms {2*n**3/ms/1e9:.2f} TFLOP/s")
