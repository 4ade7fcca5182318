"""One noft + one FT call at a given size (for ncu captures)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_02444_b200 import ftblas as fb
M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
ta, tb = (sys.argv[2] if len(sys.argv) > 2 else "NN")
A = torch.rand(M * K, dtype=torch.float64, device="cuda"); B = torch.rand(K * N, dtype=torch.float64, device="cuda")
C = torch.rand(M * N, dtype=torch.float64, device="cuda")
lda = M if ta == "N" else K; ldb = K if tb == "N" else N
fb.ftblas_set_stream(torch.cuda.current_stream())
for _ in range(2):
    fb.ftblas_dgemm_noft(ta, tb, M, N, K, 1.0, A, lda, B, ldb, 0.5, C, M)
    fb.ftblas_dgemm(ta, tb, M, N, K, 1.0, A, lda, B, ldb, 0.5, C, M)
torch.cuda.synchronize()
print("ok")
