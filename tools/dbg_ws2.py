"""Debug aid: compare the ws policy against the full policy at 4096^3 NT with 100 flips."""
import os, shutil, sys
variant = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if variant != "base":
    shutil.copy(os.path.join(ROOT, "tools", "dbg", variant + ".so"), os.path.join(ROOT, "paper_2305_02444_b200", "lib", "libftblas.so"))
sys.path.insert(0, ROOT)
import numpy as np, torch
import synthetic as syn
from tests._util import to_dev, from_dev
from paper_2305_02444_b200 import ftblas as ft
ft.ftblas_set_stream(None); ft.ftblas_set_checksum_mode("gemm")
M = N = K = 4096
w = syn.Workload("t", M, N, K, "N", "T", 1.5, -0.5, "uniform", True, seed=5)
d = syn.make_inputs(w)
plan = syn.fault_plan(M, N, 100, 17)
out = {}
for pol in ["full", "ws"]:
    ft.ftblas_set_tile_policy(pol)
    A_t, pA = to_dev(d["A"]); B_t, pB = to_dev(d["B"]); C_t, pC = to_dev(d["C"])
    ft.ftblas_set_fault_plan(*plan)
    rep = ft.Report(20000)
    ft.ftblas_dgemm("N", "T", M, N, K, 1.5, pA, d["lda"], pB, d["ldb"], -0.5, pC, d["ldc"], rep)
    torch.cuda.synchronize()
    out[pol] = (from_dev(C_t, d["C"]), rep.count, rep.tiles_flagged, rep.rows_flagged, rep.cols_flagged)
    ft.ftblas_clear_fault_plan()
print(variant, "full", out["full"][1:], "ws", out["ws"][1:])
Cf, Cw = out["full"][0], out["ws"][0]
bad = np.argwhere(~np.isclose(Cf, Cw, rtol=1e-12, atol=1e-9))
tiles = {}
for i, j in bad:
    tiles.setdefault((i // 128, j // 128), []).append((i % 128, j % 128))
print(variant, "wrong elements", len(bad), "tiles", len(tiles))
for t, el in list(tiles.items())[:6]:
    rows = sorted({r for r, c in el}); cols = sorted({c for r, c in el})
    print("  tile", t, "n", len(el), "rows", rows[:20], "cols", cols[:40])
