"""A/B timing of library builds (tools/exp/*.so) on the BASELINE config shapes (alpha, beta,
transposes as in synthetic.CONFIGS; uniform random data).  Development aid."""
import ctypes as ct, glob, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synthetic as syn
libs = sys.argv[1:] or sorted(glob.glob(os.path.join(os.path.dirname(__file__), "exp", "*.so")))
P, I, D = ct.c_void_p, ct.c_int64, ct.c_double
common = [ct.c_char, ct.c_char, I, I, I, D, P, I, P, I, D, P, I]
Ls = []
import shutil, tempfile
for spec in libs:
    path, _, policy = spec.partition(":")
    if policy:  # a private copy: ctypes would share one handle (and its state) per path
        tmp = os.path.join(tempfile.mkdtemp(), policy + "_" + os.path.basename(path))
        shutil.copy(path, tmp)
        L = ct.CDLL(tmp)
    else:
        L = ct.CDLL(path)
    L.ftblas_dgemm.argtypes = common + [P]; L.ftblas_dgemm_noft.argtypes = common
    L.ftblas_set_stream.argtypes = [P]
    L.ftblas_set_stream(ct.c_void_p(torch.cuda.current_stream().cuda_stream))
    if policy:
        L.ftblas_set_tile_policy.argtypes = [ct.c_int]
        L.ftblas_set_tile_policy({"auto": 0, "full": 1, "pair": 2}[policy])
    Ls.append((os.path.basename(path) + (":" + policy if policy else ""), L))
SEL = os.environ.get("CONFIGS")
for w in [c for c in syn.CONFIGS[:4] if not SEL or c.name.split("_")[0] in SEL.split(",")]:
    M, N, K = w.M, w.N, w.K
    lda = M if w.transA == "N" else K; ldb = K if w.transB == "N" else N
    A = torch.rand(M * K, dtype=torch.float64, device="cuda") * 2 - 1
    B = torch.rand(K * N, dtype=torch.float64, device="cuda") * 2 - 1
    C = torch.rand(M * N, dtype=torch.float64, device="cuda") * 2 - 1
    reps = 3 if M * N * K > 1e12 else 10
    for name, L in Ls:
        args = (w.transA.encode(), w.transB.encode(), M, N, K, w.alpha, A.data_ptr(), lda, B.data_ptr(), ldb, w.beta, C.data_ptr(), M)
        res = []
        for fn, extra in ((L.ftblas_dgemm_noft, ()), (L.ftblas_dgemm, (None,))):
            fn(*args, *extra); torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(reps): fn(*args, *extra)
            e1.record(); torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) / reps)
        fl = 2.0 * M * N * K
        print(f"{w.name:22s} {name:20s} noft {res[0]:8.3f} ms {fl/res[0]/1e9:6.2f} TF | ft {res[1]:8.3f} ms {fl/res[1]/1e9:6.2f} TF ovh {100*(res[1]/res[0]-1):5.2f}%", flush=True)
    del A, B, C
