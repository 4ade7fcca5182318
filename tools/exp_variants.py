"""Time experimental builds of libftblas (tools/exp/*.so) on one shape (development aid)."""
import ctypes as ct, glob, os, sys
import torch
M = N = K = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
TB = os.environ.get("TRANSB", "N").encode()
libs = sys.argv[2:] or sorted(glob.glob(os.path.join(os.path.dirname(__file__), "exp", "*.so")))
A = torch.rand(M * K, dtype=torch.float64, device="cuda"); B = torch.rand(K * N, dtype=torch.float64, device="cuda")
C = torch.rand(M * N, dtype=torch.float64, device="cuda")
for path in libs:
    L = ct.CDLL(path)
    P, I, D = ct.c_void_p, ct.c_int64, ct.c_double
    common = [ct.c_char, ct.c_char, I, I, I, D, P, I, P, I, D, P, I]
    L.ftblas_dgemm.argtypes = common + [P]; L.ftblas_dgemm_noft.argtypes = common
    L.ftblas_set_stream.argtypes = [P]
    L.ftblas_set_stream(ct.c_void_p(torch.cuda.current_stream().cuda_stream))
    for name, fn in (("noft", lambda: L.ftblas_dgemm_noft(b"N", TB, M, N, K, 1.0, A.data_ptr(), M, B.data_ptr(), K if TB == b"N" else N, 0.0, C.data_ptr(), M)),
                     ("ft", lambda: L.ftblas_dgemm(b"N", TB, M, N, K, 1.0, A.data_ptr(), M, B.data_ptr(), K if TB == b"N" else N, 0.0, C.data_ptr(), M, None))):
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 5
        e0.record()
        for _ in range(reps): fn()
        e1.record(); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"{os.path.basename(path):28s} {TB.decode()} {name:5s} {M}^3 {ms:8.3f} ms {2.0*M*N*K/ms/1e9:6.2f} TF", flush=True)
