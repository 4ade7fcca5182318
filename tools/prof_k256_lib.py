"""c2-shaped calls (16384 x 16384 x 256, NN, alpha=-1, beta=1) through a given libftblas build
(tools/exp/*.so, private ctypes handle) for ncu launch lists: warm-up, then noft + FT."""
import ctypes as ct, os, sys
import torch
lib = sys.argv[1]
L = ct.CDLL(os.path.abspath(lib))
P, I, D = ct.c_void_p, ct.c_int64, ct.c_double
common = [ct.c_char, ct.c_char, I, I, I, D, P, I, P, I, D, P, I]
L.ftblas_dgemm.argtypes = common + [P]; L.ftblas_dgemm_noft.argtypes = common
L.ftblas_set_stream.argtypes = [P]
L.ftblas_set_stream(ct.c_void_p(torch.cuda.current_stream().cuda_stream))
M = N = 16384; K = int(sys.argv[2]) if len(sys.argv) > 2 else 256
A = torch.rand(M * K, dtype=torch.float64, device="cuda"); B = torch.rand(K * N, dtype=torch.float64, device="cuda")
C = torch.rand(M * N, dtype=torch.float64, device="cuda")
args = (b"N", b"N", M, N, K, -1.0, A.data_ptr(), M, B.data_ptr(), K, 1.0, C.data_ptr(), M)
for _ in range(2):
    L.ftblas_dgemm_noft(*args)
    L.ftblas_dgemm(*args, None)
torch.cuda.synchronize()
print("ok")
