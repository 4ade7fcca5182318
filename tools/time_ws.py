"""Development aid: per-call CUDA-event times of FT / non-FT calls (back to back) for a workload."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synthetic as syn
from tests._util import to_dev
from paper_2305_02444_b200 import ftblas as ft
w = syn.CONFIG_BY_NAME[sys.argv[1]]
if os.environ.get("BETA") is not None:  # override beta (development: the C0 traffic's share)
    import dataclasses
    w = dataclasses.replace(w, beta=float(os.environ["BETA"]))
tiles = sys.argv[2] if len(sys.argv) > 2 else "ws"
d = syn.make_inputs(w)
ft.ftblas_set_stream(torch.cuda.current_stream()); ft.ftblas_set_tile_policy(tiles)
A_t, pA = to_dev(d["A"]); B_t, pB = to_dev(d["B"]); C_t, pC = to_dev(d["C"])
flops = 2.0 * w.M * w.N * w.K
def run(mode, n):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(n + 1)]
    ev[0].record()
    for i in range(n):
        if mode == "ft":
            ft.ftblas_dgemm(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"], w.beta, pC, d["ldc"], None)
        else:
            ft.ftblas_dgemm_noft(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"], w.beta, pC, d["ldc"])
        ev[i + 1].record()
    torch.cuda.synchronize()
    ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(n)]
    return ms
for mode in ["noft", "ft", "noft", "ft"]:
    run(mode, 3)
    ms = run(mode, 10)
    print(f"{w.name} {tiles} {mode}: " + " ".join(f"{x:.3f}" for x in ms) + f"  median {sorted(ms)[5]:.3f} ms = {flops / sorted(ms)[5] / 1e9:.2f} TF")
