"""c1-shaped calls (4096^3, NT, alpha 1.5, beta -0.5; or another transB) through a library build
for ncu launch lists: warm-up, then one noft and one FT call.
Usage: python tools/prof_c1_lib.py LIB.so [transB]"""
import ctypes as ct, os, sys
import torch
L = ct.CDLL(os.path.abspath(sys.argv[1]))
P, I, D = ct.c_void_p, ct.c_int64, ct.c_double
common = [ct.c_char, ct.c_char, I, I, I, D, P, I, P, I, D, P, I]
L.ftblas_dgemm.argtypes = common + [P]; L.ftblas_dgemm_noft.argtypes = common
L.ftblas_set_stream.argtypes = [P]
L.ftblas_set_stream(ct.c_void_p(torch.cuda.current_stream().cuda_stream))
M = N = K = 4096
A = torch.rand(M * K, dtype=torch.float64, device="cuda"); B = torch.rand(K * N, dtype=torch.float64, device="cuda")
C = torch.rand(M * N, dtype=torch.float64, device="cuda")
tb = (sys.argv[2] if len(sys.argv) > 2 else "T").encode()
args = (b"N", tb, M, N, K, 1.5, A.data_ptr(), M, B.data_ptr(), N if tb == b"T" else K, -0.5, C.data_ptr(), M)
for _ in range(3):
    L.ftblas_dgemm_noft(*args)
    L.ftblas_dgemm(*args, None)
torch.cuda.synchronize()
print("ok")
