"""Development aid: phase breakdown of gemm_ws_kernel from a -DFTB_WS_PROF build
(tools/dbg/ws_prof.so copied over the library).  Usage: python tools/ws_phases.py <workload> [ft|noft]"""
import ctypes as ct, os, shutil, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
shutil.copy(os.path.join(ROOT, "tools", "dbg", os.environ.get("WS_PROF_SO", "ws_prof.so")), os.path.join(ROOT, "paper_2305_02444_b200", "lib", "libftblas.so"))
sys.path.insert(0, ROOT)
import numpy as np, torch
import synthetic as syn
from tests._util import to_dev
from paper_2305_02444_b200 import ftblas as ft
names = ["mma_wait_full", "mma_wait_buf", "mma_tail", "epi_wait_acc", "epi_c0load", "mma_kloop", "epi_verify",
         "epi_locate", "epi_store", "prod_wait_empty", "epi_total", "mma_total"]
w = syn.CONFIG_BY_NAME[sys.argv[1]]
mode = sys.argv[2] if len(sys.argv) > 2 else "ft"
d = syn.make_inputs(w)
nfl = int(os.environ.get("FLIPS", "0"))  # FLIPS=n: a seeded fault plan of n flips (development: which phase the flagged tiles stretch)
ft.ftblas_set_stream(None); ft.ftblas_set_tile_policy("ws")
A_t, pA = to_dev(d["A"]); B_t, pB = to_dev(d["B"]); C_t, pC = to_dev(d["C"])
L = ft.lib
if nfl:
    ft.ftblas_set_fault_plan(*syn.fault_plan(w.M, w.N, nfl, w.seed))
rep = ft.Report(4 * nfl + 16)
L.ftblas_ws_prof_read.argtypes = [ct.POINTER(ct.c_ulonglong), ct.c_int]
buf = (ct.c_ulonglong * (1024 * 16))()
def call():
    if mode == "ft":
        ft.ftblas_dgemm(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"], w.beta, pC, d["ldc"], rep if nfl else None)
    else:
        ft.ftblas_dgemm_noft(w.transA, w.transB, w.M, w.N, w.K, w.alpha, pA, d["lda"], pB, d["ldb"], w.beta, pC, d["ldc"])
for _ in range(3): call()
torch.cuda.synchronize(); L.ftblas_ws_prof_read(buf, 1024 * 16)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); call(); e1.record(); torch.cuda.synchronize()
L.ftblas_ws_prof_read(buf, 1024 * 16)
a = np.array(buf[:148 * 16], dtype=np.float64).reshape(148, 16) / 1e3  # us
print(f"{w.name} {mode}: call {e0.elapsed_time(e1):.3f} ms; per-CTA phase sums (us): mean / max")
for k, n in enumerate(names):
    print(f"  {n:18s} {a[:, k].mean():10.1f} {a[:, k].max():10.1f}")
if nfl:
    print("  located", rep.count, "of", nfl, "; CTAs by mma_total:", np.argsort(-a[:, 11])[:6], np.sort(-a[:, 11])[:6] * -1)
