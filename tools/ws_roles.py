"""Development aid: build gemm_ws_kernel warp-role variants (-DFTB_WS_EPI_WG / -DFTB_WS_PROD_WG)
into tools/var/ws_e<E>p<P>.so (parallel nvcc), and run tools/time_ws.py with each copied over
the library.  Usage: python tools/ws_roles.py build E:P [E:P ...]
                     python tools/ws_roles.py run WORKLOAD TILES E:P [E:P ...]"""
import os, shutil, subprocess, sys
from concurrent.futures import ThreadPoolExecutor
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2305_02444_b200", "lib", "libftblas.so")
SRC = os.path.join(ROOT, "paper_2305_02444_b200", "csrc", "ftblas.cu")


def so(v):
    e, p = v.split(":")[:2]
    extra = "_".join(v.split(":")[2:])
    return os.path.join(ROOT, "tools", "var", f"ws_e{e}p{p}{('_' + extra) if extra else ''}.so")


def build(v):
    e, p = v.split(":")[:2]
    defs = [f"-DFTB_WS_EPI_WG={e}", f"-DFTB_WS_PROD_WG={p}"] + [f"-D{d}" for d in v.split(":")[2:]]
    cmd = ["/usr/local/cuda/bin/nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-Xcompiler", "-fPIC", "-shared", *defs, "-o", so(v), SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    return v, r.returncode, r.stderr[-1500:]


if __name__ == "__main__":
    os.makedirs(os.path.join(ROOT, "tools", "var"), exist_ok=True)
    if sys.argv[1] == "build":
        with ThreadPoolExecutor(8) as ex:
            for v, rc, err in ex.map(build, sys.argv[2:]):
                print(v, "rc", rc, err if rc else "")
    else:
        wl, tiles = sys.argv[2], sys.argv[3]
        keep = LIB + ".orig"
        shutil.copy(LIB, keep)
        try:
            for v in sys.argv[4:]:
                shutil.copy(so(v), LIB)
                print(f"== variant {v}", flush=True)
                subprocess.run([sys.executable, os.path.join(ROOT, "tools", "time_ws.py"), wl, tiles], timeout=600)
        finally:
            shutil.copy(keep, LIB)
