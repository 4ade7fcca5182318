"""Development aid: per FT call, the checksum-stage and main-kernel device times (ftblas_profile)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synthetic as syn
from tests._util import to_dev
from paper_2305_02444_b200 import ftblas as ft
w = syn.CONFIG_BY_NAME[sys.argv[1]]
tiles = sys.argv[2] if len(sys.argv) > 2 else "auto"
d = syn.make_inputs(w)
ft.ftblas_set_stream(torch.cuda.current_stream()); ft.ftblas_set_tile_policy(tiles)
A_t, pA = to_dev(d["A"]); B_t, pB = to_dev(d["B"]); C_t, pC = to_dev(d["C"])
call = lambda: ft.ftblas_dgemm(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"], w.beta, pC, d["ldc"], None)
for _ in range(3): call()
torch.cuda.synchronize()
ft.ftblas_profile(True)
n = 10
for _ in range(n): call()
torch.cuda.synchronize()
st, gm, nl = ft.ftblas_profile_read()
ft.ftblas_profile(False)
print(f"{w.name} {tiles}: stage {st / n * 1e3:.1f} us, main kernel {gm / n:.4f} ms per call ({nl} launches)")
