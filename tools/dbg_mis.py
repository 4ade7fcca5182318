import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import synthetic as syn
import tests.test_gpu_parity as T
ft = T._lib("gemm", sys.argv[1] if len(sys.argv) > 1 else "pair")
w = syn.Workload("t", 201, 150, 45, "N", "T", 1.25, -1.0, "uniform", True, seed=5)
d = syn.make_inputs(w, pad=1)
plan = syn.fault_plan(w.M, w.N, 2, 9)
print("plan", plan)
for off in [(1, 0, 0), (0, 0, 0), (0, 1, 1)]:
    C_gpu, rep = T.run_gpu(ft, w, d, plan=plan, offsets=off)
    C_ref, orep, _ = T.run_oracle(w, d, plan)
    bad = np.argwhere(~(np.abs(C_gpu - C_ref) <= 1e-9 * (1 + np.abs(C_ref))))
    print(off, "report", [(e["i"], e["j"], e["kind"]) for e in rep.entries()], "bad", bad[:5].tolist(), [C_gpu[i, j] for i, j in bad[:3]], [C_ref[i, j] for i, j in bad[:3]])
