"""c2-shaped calls (16384 x 16384 x 256, NN, alpha=-1, beta=1) for ncu: warm-up, then one noft
and one FT (checksum-GEMM mode) call."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_02444_b200 import ftblas as fb
fb.ftblas_set_stream(torch.cuda.current_stream())
M = N = 16384; K = int(sys.argv[1]) if len(sys.argv) > 1 else 256
A = torch.rand(M * K, dtype=torch.float64, device="cuda"); B = torch.rand(K * N, dtype=torch.float64, device="cuda")
C = torch.rand(M * N, dtype=torch.float64, device="cuda")
for _ in range(2):
    fb.ftblas_dgemm_noft("N", "N", M, N, K, -1.0, A, M, B, K, 1.0, C, M)
    fb.ftblas_dgemm("N", "N", M, N, K, -1.0, A, M, B, K, 1.0, C, M)
torch.cuda.synchronize()
print("ok")
