"""Development aid: SM clock / power sampled by nvidia-smi while FT or non-FT calls of a workload run
back to back (is a time difference a clock difference?).  Usage: clock_probe.py <workload> [tiles]"""
import os, subprocess, sys, time, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import synthetic as syn
from tests._util import to_dev
from paper_2305_02444_b200 import ftblas as ft
w = syn.CONFIG_BY_NAME[sys.argv[1]]
tiles = sys.argv[2] if len(sys.argv) > 2 else "ws"
d = syn.make_inputs(w)
ft.ftblas_set_stream(torch.cuda.current_stream()); ft.ftblas_set_tile_policy(tiles)
A_t, pA = to_dev(d["A"]); B_t, pB = to_dev(d["B"]); C_t, pC = to_dev(d["C"])
def call(mode):
    if mode == "ft":
        ft.ftblas_dgemm(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"], w.beta, pC, d["ldc"], None)
    else:
        ft.ftblas_dgemm_noft(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"], w.beta, pC, d["ldc"])
for mode in ["noft", "ft", "noft", "ft"]:
    for _ in range(20): call(mode)
    torch.cuda.synchronize()
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active,temperature.gpu",
                          "--format=csv,noheader,nounits", "-lms", "20"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.3)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 600
    e0.record()
    for _ in range(n): call(mode)
    e1.record(); torch.cuda.synchronize()
    p.terminate()
    rows = [r.split(",") for r in p.stdout.read().strip().splitlines()]
    rows = rows[len(rows) // 4:]  # under load
    clk = [float(r[0]) for r in rows]; pw = [float(r[1]) for r in rows]
    print(f"{w.name} {tiles} {mode}: {e0.elapsed_time(e1) / n:.4f} ms/call; SM MHz median {statistics.median(clk)} min {min(clk)} "
          f"max {max(clk)}; power median {statistics.median(pw):.0f} W max {max(pw):.0f}; reasons {sorted({r[2].strip() for r in rows})}; n={len(rows)}")
