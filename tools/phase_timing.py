"""Per-CTA phase durations of the GEMM kernel (non-FT and FT) from the globaltimer stamps of
the `phases` variant (python tools/variant_build.py phases), plus the share of SM time with
0 / 1 / 2 CTAs in their mainloop.  Usage: python tools/phase_timing.py [M=N] [K]   (NN, alpha=-1,
beta=1, uniform data).  Development aid; timing-only build."""
import ctypes as ct
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L = ct.CDLL(os.path.join(ROOT, "tools", "var", "phases.so"))
P, I, D = ct.c_void_p, ct.c_int64, ct.c_double
common = [ct.c_char, ct.c_char, I, I, I, D, P, I, P, I, D, P, I]
L.ftblas_dgemm.argtypes = common + [P]
L.ftblas_dgemm_noft.argtypes = common
L.ftblas_set_stream.argtypes = [P]
L.ftblas_debug_times.argtypes = [P]
L.ftblas_set_stream(ct.c_void_p(torch.cuda.current_stream().cuda_stream))
M = N = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
K = int(sys.argv[2]) if len(sys.argv) > 2 else 256
A = torch.rand(M * K, dtype=torch.float64, device="cuda")
B = torch.rand(K * N, dtype=torch.float64, device="cuda")
C = torch.rand(M * N, dtype=torch.float64, device="cuda")
args = (b"N", b"N", M, N, K, -1.0, A.data_ptr(), M, B.data_ptr(), K, 1.0, C.data_ptr(), M)
buf = np.zeros(65536 * 8, dtype=np.uint64)
for name, fn in (("noft", lambda: L.ftblas_dgemm_noft(*args)), ("ft", lambda: L.ftblas_dgemm(*args, None))):
    for _ in range(2):
        fn()
        torch.cuda.synchronize()
    L.ftblas_debug_times(buf.ctypes.data)
    n = min(65536, 2 * (M // 128) * (N // 128)) if K <= 2048 else (M // 128) * (N // 128)
    t = buf.reshape(-1, 8)[:n].astype(np.int64)
    d = lambda a, b: (t[:, b] - t[:, a]) / 1e3  # noqa: E731
    if name == "noft":
        print(f"{name}: mainloop {d(0, 1).mean():.2f}  C0 {d(1, 2).mean():.2f}  form {d(2, 3).mean():.2f}  "
              f"store {d(3, 5).mean():.2f}  epilogue {d(1, 5).mean():.2f} us")
    else:
        print(f"{name}: mainloop {d(0, 1).mean():.2f}  C0 {d(1, 2).mean():.2f}  sums {d(2, 3).mean():.2f}  "
              f"verify+exchange {d(3, 4).mean():.2f}  store {d(4, 5).mean():.2f}  epilogue {d(1, 5).mean():.2f} us")
    t0 = t[:, 0].min()
    s, ml, e, sm = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3, (t[:, 5] - t0) / 1e3, t[:, 7]
    span = e.max()
    res = []
    for q in np.unique(sm):
        ev = sorted([(s[i], 1) for i in np.where(sm == q)[0]] + [(ml[i], -1) for i in np.where(sm == q)[0]])
        cur, last, acc = 0, 0.0, [0.0, 0.0, 0.0]
        for tt, dd in ev:
            acc[min(cur, 2)] += tt - last
            last, cur = tt, cur + dd
        acc[0] += span - last
        res.append([x / span for x in acc])
    r = np.mean(res, axis=0) * 100
    print(f"   SM time with 0 / 1 / 2 CTAs in mainloop: {r[0]:.1f} / {r[1]:.1f} / {r[2]:.1f} %")
