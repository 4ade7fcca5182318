"""One cuBLAS FP64 GEMM (torch.matmul, column-major view) at 16384^3 after a warm-up, for an
ncu DRAM-traffic comparison with gemm_kernel (context only)."""
import torch
n = 16384
A = torch.randn(n, n, dtype=torch.float64, device="cuda"); B = torch.randn(n, n, dtype=torch.float64, device="cuda")
C = torch.matmul(A, B); torch.cuda.synchronize()
C = torch.matmul(A, B); torch.cuda.synchronize()
print("ok")
