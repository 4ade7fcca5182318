"""One noft + one FT (checksum-GEMM mode) call per shape, after a warm-up (for ncu launch lists)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2305_02444_b200 import ftblas as fb
fb.ftblas_set_stream(torch.cuda.current_stream())
for M, N, K, ta, tb in [(4096, 4096, 4096, "N", "T"), (16384, 16384, 256, "N", "N"), (2048, 16384, 16384, "N", "N")]:
    lda = M if ta == "N" else K; ldb = K if tb == "N" else N
    A = torch.rand(M * K, dtype=torch.float64, device="cuda"); B = torch.rand(K * N, dtype=torch.float64, device="cuda")
    C = torch.rand(M * N, dtype=torch.float64, device="cuda")
    for _ in range(2):
        fb.ftblas_dgemm_noft(ta, tb, M, N, K, 1.0, A, lda, B, ldb, 0.5, C, M)
        fb.ftblas_dgemm(ta, tb, M, N, K, 1.0, A, lda, B, ldb, 0.5, C, M)
    torch.cuda.synchronize()
    del A, B, C
print("ok")
