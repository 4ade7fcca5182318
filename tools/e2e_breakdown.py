"""Where the e2e time of ftblas_dgemm_host goes at c3: device-side sums of the checksum stage
and main-kernel time over the pipeline's block calls (ftblas_profile) vs the wall time of the
call and of the single device call on resident inputs.  Development aid."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2305_02444_b200 import ftblas as fb
M = N = K = 16384
g = torch.Generator().manual_seed(0)
hA = torch.randn(M * K, dtype=torch.float64, generator=g).pin_memory()
hB = torch.randn(K * N, dtype=torch.float64, generator=g).pin_memory()
hC = torch.zeros(M * N, dtype=torch.float64).pin_memory()
fb.ftblas_set_stream(torch.cuda.current_stream())
dA, dB, dC = hA.cuda(), hB.cuda(), hC.cuda()
for name, fn in (("device", lambda: fb.ftblas_dgemm("N", "N", M, N, K, 1.0, dA, M, dB, K, 0.0, dC, M)),
                 ("host", lambda: fb.ftblas_dgemm_host("N", "N", M, N, K, 1.0, hA, M, hB, K, 0.0, hC, M))):
    fn(); torch.cuda.synchronize()
    fb.ftblas_profile(True); fb.ftblas_profile_read()
    t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); wall = (time.perf_counter() - t0) * 1e3
    fb.ftblas_profile(False)
    enc, gemm, n = fb.ftblas_profile_read()
    print(f"{name:6s} wall {wall:7.1f} ms  checksum stage {enc:6.2f} ms  main kernels {gemm:7.2f} ms  calls {n}")
