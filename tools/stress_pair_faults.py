"""Report counts of a c1-shaped run (4096^2, NT, alpha 1.5, beta -0.5) with 100 injected flips at
K = 4096 / 2048 / 1024, through given library builds and tile policies (LIB[:auto|full|pair]).
Correct output: count = tiles = rows = cols = 100.  The regression behind
tests/test_gpu_parity.py::test_many_faulted_tiles_leave_neighbours_clean.
Usage: python tools/stress_pair_faults.py paper_2305_02444_b200/lib/libftblas.so:pair ..."""
import ctypes as ct, os, sys, shutil, tempfile
import numpy as np, torch
sys.path.insert(0, os.getcwd())
import synthetic as syn
w = syn.CONFIGS[1]
d = syn.make_inputs(w)
plan = syn.fault_plan(w.M, w.N, w.n_flips, w.seed)
A = torch.from_numpy(np.asfortranarray(d["A"]).reshape(-1, order="F").copy()).cuda()
B = torch.from_numpy(np.asfortranarray(d["B"]).reshape(-1, order="F").copy()).cuda()
C0 = torch.from_numpy(np.asfortranarray(d["C"]).reshape(-1, order="F").copy()).cuda()
P, I, D = ct.c_void_p, ct.c_int64, ct.c_double
for spec in sys.argv[1:]:
    path, _, pol = spec.partition(":")
    tmp = os.path.join(tempfile.mkdtemp(), os.path.basename(path)); shutil.copy(path, tmp)
    L = ct.CDLL(tmp)
    common = [ct.c_char, ct.c_char, I, I, I, D, P, I, P, I, D, P, I]
    L.ftblas_dgemm.argtypes = common + [P]
    L.ftblas_set_stream.argtypes = [P]; L.ftblas_set_stream(ct.c_void_p(torch.cuda.current_stream().cuda_stream))
    L.ftblas_set_tile_policy.argtypes = [ct.c_int]; L.ftblas_set_tile_policy({"auto": 0, "full": 1, "pair": 2}[pol or "auto"])
    L.ftblas_set_fault_plan.argtypes = [I, P, P, P]
    pi, pj, pb = (np.ascontiguousarray(x) for x in plan)
    pi = pi.astype(np.int64); pj = pj.astype(np.int64); pb = pb.astype(np.int32)
    L.ftblas_set_fault_plan(len(pi), pi.ctypes.data, pj.ctypes.data, pb.ctypes.data)
    class Rep(ct.Structure):
        _fields_ = [("entries", P), ("capacity", ct.c_int64), ("count", ct.c_int64), ("tiles_flagged", ct.c_int64), ("rows_flagged", ct.c_int64), ("cols_flagged", ct.c_int64)]
    for Kx in (4096, 2048, 1024):
        C = C0.clone()
        r = Rep(); r.capacity = 0; r.entries = None
        rc = L.ftblas_dgemm(w.transA.encode(), w.transB.encode(), w.M, w.N, Kx, w.alpha, A.data_ptr(), d["lda"], B.data_ptr(), d["ldb"], w.beta, C.data_ptr(), d["ldc"], ct.byref(r))
        torch.cuda.synchronize()
        print(f"{spec:24s} K={Kx} rc={rc} count={r.count} tiles={r.tiles_flagged} rows={r.rows_flagged} cols={r.cols_flagged}", flush=True)
