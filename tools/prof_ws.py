"""Development aid: run <calls> FT (or non-FT) calls of a workload with the ws tile policy (for ncu)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synthetic as syn
from tests._util import to_dev
from paper_2305_02444_b200 import ftblas as ft
w = syn.CONFIG_BY_NAME[sys.argv[1]]
mode = sys.argv[2] if len(sys.argv) > 2 else "ft"
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 2
tiles = sys.argv[4] if len(sys.argv) > 4 else "ws"
d = syn.make_inputs(w)
ft.ftblas_set_stream(None); ft.ftblas_set_tile_policy(tiles)
A_t, pA = to_dev(d["A"]); B_t, pB = to_dev(d["B"]); C_t, pC = to_dev(d["C"])
for _ in range(calls):
    if mode == "ft":
        ft.ftblas_dgemm(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"], w.beta, pC, d["ldc"], None)
    else:
        ft.ftblas_dgemm_noft(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"], w.beta, pC, d["ldc"])
torch.cuda.synchronize()
print("ok")
