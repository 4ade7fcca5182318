"""One FT call (checksum-GEMM mode) at 16384^3 NN beta=0 per library build given on the command
line (for ncu DRAM-traffic comparisons of rasterizations)."""
import ctypes as ct, os, sys, shutil, tempfile
import torch
n = 16384
A = torch.randn(n * n, dtype=torch.float64, device="cuda"); B = torch.randn(n * n, dtype=torch.float64, device="cuda")
C = torch.zeros(n * n, dtype=torch.float64, device="cuda")
P, I, D = ct.c_void_p, ct.c_int64, ct.c_double
for path in sys.argv[1:]:
    tmp = os.path.join(tempfile.mkdtemp(), os.path.basename(path)); shutil.copy(path, tmp)
    L = ct.CDLL(tmp)
    L.ftblas_dgemm_noft.argtypes = [ct.c_char, ct.c_char, I, I, I, D, P, I, P, I, D, P, I]
    L.ftblas_set_stream.argtypes = [P]
    L.ftblas_set_stream(ct.c_void_p(torch.cuda.current_stream().cuda_stream))
    L.ftblas_dgemm_noft(b"N", b"N", n, n, n, 1.0, A.data_ptr(), n, B.data_ptr(), n, 0.0, C.data_ptr(), n)
    torch.cuda.synchronize()
    print(os.path.basename(path), "ok", flush=True)
