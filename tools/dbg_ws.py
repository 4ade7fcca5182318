import sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import synthetic as syn
from tests._util import to_dev, from_dev
from paper_2305_02444_b200 import ftblas as ft
ft.ftblas_set_stream(None); ft.ftblas_set_checksum_mode("gemm")
for (M, N, K, tA, tB, al, be, nfl) in [(2048, 2048, 2048, "N", "T", 1.5, -0.5, 100), (4096, 4096, 4096, "N", "T", 1.5, -0.5, 100), (4096,4096,512,"N","N",1.0,0.0,100), (4096,4096,512,"N","T",1.0,0.0,100), (4096,4096,512,"N","N",1.5,-0.5,100)]:
    w = syn.Workload("t", M, N, K, tA, tB, al, be, "uniform", True, seed=5)
    d = syn.make_inputs(w)
    plan = syn.fault_plan(M, N, nfl, 17)
    for pol in ["full", "ws"]:
        ft.ftblas_set_tile_policy(pol)
        A_t, pA = to_dev(d["A"]); B_t, pB = to_dev(d["B"]); C_t, pC = to_dev(d["C"])
        ft.ftblas_set_fault_plan(*plan)
        rep = ft.Report(20000)
        ft.ftblas_dgemm(tA, tB, M, N, K, al, pA, d["lda"], pB, d["ldb"], be, pC, d["ldc"], rep)
        torch.cuda.synchronize()
        ents = rep.entries()
        want = set(zip(plan[0].tolist(), plan[1].tolist()))
        got = [(e["i"], e["j"]) for e in ents]
        extra = [e for e in ents if (e["i"], e["j"]) not in want]
        print(M, N, K, tA, tB, pol, "count", rep.count, "tiles", rep.tiles_flagged, "rows", rep.rows_flagged, "cols", rep.cols_flagged, "missing", len(want - set(got)), "extra", len(extra), flush=True)
        if extra[:3]: print("   extra sample", extra[:3])
        ft.ftblas_clear_fault_plan()
        C_t2, pC2 = to_dev(d["C"])
        rep2 = ft.Report(20000)
        ft.ftblas_dgemm(tA, tB, M, N, K, al, pA, d["lda"], pB, d["ldb"], be, pC2, d["ldc"], rep2)
        torch.cuda.synchronize()
        print("   fault-free count", rep2.count, "tiles", rep2.tiles_flagged, flush=True)
