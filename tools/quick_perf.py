"""Quick FT / non-FT / cuBLAS timing (development aid, not the bench contract)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2305_02444_b200 import ftblas as fb
import synthetic as syn

def timeit(fn, reps):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

fb.ftblas_set_stream(torch.cuda.current_stream())
for name, M, N, K, ta, tb in [("4096 NT", 4096, 4096, 4096, "N", "T"), ("4096 NN", 4096, 4096, 4096, "N", "N"),
                              ("16384x16384x256", 16384, 16384, 256, "N", "N"), ("8192 NN", 8192, 8192, 8192, "N", "N"),
                              ("16384 NN", 16384, 16384, 16384, "N", "N")]:
    A = torch.rand(M * K, dtype=torch.float64, device="cuda") * 2 - 1
    B = torch.rand(K * N, dtype=torch.float64, device="cuda") * 2 - 1
    C = torch.rand(M * N, dtype=torch.float64, device="cuda") * 2 - 1
    lda = M if ta == "N" else K
    ldb = K if tb == "N" else N
    reps = 3 if M * N * K > 1e12 else 10
    fl = 2.0 * M * N * K
    t_nf = timeit(lambda: fb.ftblas_dgemm_noft(ta, tb, M, N, K, 1.0, A, lda, B, ldb, 0.5, C, M), reps)
    fb.ftblas_set_checksum_mode("fused")
    t_fu = timeit(lambda: fb.ftblas_dgemm(ta, tb, M, N, K, 1.0, A, lda, B, ldb, 0.5, C, M), reps)
    fb.ftblas_set_checksum_mode("gemm")
    t_ft = timeit(lambda: fb.ftblas_dgemm(ta, tb, M, N, K, 1.0, A, lda, B, ldb, 0.5, C, M), reps)
    Am = A.view(K, M).t() if ta == "N" else A.view(M, K)
    Bm = B.view(N, K).t() if tb == "N" else B.view(K, N)
    t_cb = timeit(lambda: torch.matmul(Am, Bm), reps)
    print(f"{name:18s} noft {t_nf:8.3f} ms {fl/t_nf/1e9:6.2f} TF | ft {t_ft:8.3f} ms {fl/t_ft/1e9:6.2f} TF "
          f"ovh {100*(t_ft/t_nf-1):5.2f}% | fused {fl/t_fu/1e9:6.2f} TF ovh {100*(t_fu/t_nf-1):5.2f}% | cublas {t_cb:8.3f} ms {fl/t_cb/1e9:6.2f} TF", flush=True)
    rep = fb.Report(16); fb.ftblas_dgemm(ta, tb, M, N, K, 1.0, A, lda, B, ldb, 0.5, C, M, rep)
    print("   fault-free report count", rep.count, "tiles flagged", rep.tiles_flagged, flush=True)
    del A, B, C
