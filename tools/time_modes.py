"""Development aid: per-call time of FT calls under each checksum mode / tile policy (small shapes)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synthetic as syn
from tests._util import to_dev
from paper_2305_02444_b200 import ftblas as ft
w = syn.CONFIG_BY_NAME[sys.argv[1]]
d = syn.make_inputs(w)
ft.ftblas_set_stream(torch.cuda.current_stream())
A_t, pA = to_dev(d["A"]); B_t, pB = to_dev(d["B"]); C_t, pC = to_dev(d["C"])
def run(n, noft=False):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        if noft:
            ft.ftblas_dgemm_noft(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"], w.beta, pC, d["ldc"])
        else:
            ft.ftblas_dgemm(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"], w.beta, pC, d["ldc"], None)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3
for mode in ("gemm", "fused"):
    ft.ftblas_set_checksum_mode(mode)
    for tiles in ("auto", "full", "pair"):
        ft.ftblas_set_tile_policy(tiles)
        run(20); print(f"{w.name} {mode} {tiles}: FT {run(200):.1f} us/call")
ft.ftblas_set_checksum_mode("gemm")
for tiles in ("auto", "full", "pair"):
    ft.ftblas_set_tile_policy(tiles)
    run(20, True); print(f"{w.name} noft {tiles}: {run(200, True):.1f} us/call")
