"""Build experimental variants of libftblas.so into tools/exp/<name>.so (development aid).

A variant is the current csrc/ with text patches applied (timing-only instrumentation or
ablations); nothing here is used by the library, tests or bench.  Usage:
    python tools/variant_build.py phases        # per-CTA globaltimer stamps (tools/phase_timing.py)
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "paper_2305_02444_b200", "csrc")


def read():
    return (open(os.path.join(SRC, "ftblas_kernels.cuh")).read(),
            open(os.path.join(SRC, "ftblas.cu")).read())


def patch(text, old, new):
    assert text.count(old) == 1, f"patch anchor not unique / missing: {old[:60]!r}"
    return text.replace(old, new)


def build(name, kern, cu, extra=()):
    base = f"/tmp/ftblas_variant/{name}"
    d = os.path.join(base, "p", "c")  # csrc/ftblas.cu includes ../../include/ftblas.h
    os.makedirs(d, exist_ok=True)
    if not os.path.exists(os.path.join(base, "include")):
        os.symlink(os.path.join(ROOT, "include"), os.path.join(base, "include"))
    open(os.path.join(d, "ftblas_kernels.cuh"), "w").write(kern)
    open(os.path.join(d, "ftblas.cu"), "w").write(cu)
    open(os.path.join(d, "ftblas_ws.cuh"), "w").write(open(os.path.join(SRC, "ftblas_ws.cuh")).read())
    os.makedirs(os.path.join(ROOT, "tools", "var"), exist_ok=True)
    out = os.path.join(ROOT, "tools", "var", name + ".so")
    cmd = ["/usr/local/cuda/bin/nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a",
           "-lineinfo", "-Xcompiler", "-fPIC", "-shared", *extra, "-o", out, os.path.join(d, "ftblas.cu")]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode:
        sys.exit(r.stderr[-2000:])
    return out


def phases():
    """globaltimer stamps per CTA: 0 start, 1 mainloop end, 2 C0 staged, 3 sums / form done,
    4 verification + exchange done (FT), 5 stored; 7 = SM id.  Read by ftblas_debug_times."""
    k, cu = read()
    k = patch(k, "namespace ftb {\n", "namespace ftb {\n__device__ unsigned long long dbg_t[65536 * 8];\n"
              "__device__ __forceinline__ unsigned long long gtime() { unsigned long long t; "
              "asm volatile(\"mov.u64 %0, %%globaltimer;\" : \"=l\"(t)); return t; }\n")
    T = lambda s: f"if (MODE != MODE_FT_FUSED && tid == 0 && blockIdx.x < 65536) dbg_t[blockIdx.x * 8 + {s}] = gtime();"  # noqa: E731
    k = patch(k, "    const int wm = warp % NWM, wn = warp / NWM;",
              "    const int wm = warp % NWM, wn = warp / NWM;\n    if (MODE != MODE_FT_FUSED && tid == 0 && blockIdx.x < 65536) "
              "{ unsigned s; asm volatile(\"mov.u32 %0, %%smid;\" : \"=r\"(s)); dbg_t[blockIdx.x * 8 + 7] = s; }\n    " + T(0))
    k = patch(k, "    bar_mma();  // all MMA warps done with the pipeline smem (every issued copy was consumed)",
              "    bar_mma();  // all MMA warps done with the pipeline smem (every issued copy was consumed)\n    " + T(1))
    k = patch(k, "        if (!beta0) {\n            stage_c0();\n            bar_mma();\n        }\n        form_out();\n        bar_mma();\n        store_tile();",
              "        if (!beta0) {\n            stage_c0();\n            bar_mma();\n        }\n        " + T(2) +
              "\n        form_out();\n        bar_mma();\n        " + T(3) + "\n        store_tile();\n        bar_mma();\n        " + T(5))
    k = patch(k, "    if (!beta0) {\n        stage_c0();\n        bar_mma();\n    }\n    // fault injection",
              "    if (!beta0) {\n        stage_c0();\n        bar_mma();\n    }\n    " + T(2) + "\n    // fault injection")
    k = patch(k, "    if (PAIR) cp_wait<0>();  // this thread's side-data copies (beta = 0 has no C0 staging wait)\n    bar_mma();",
              "    if (PAIR) cp_wait<0>();  // this thread's side-data copies (beta = 0 has no C0 staging wait)\n    bar_mma();\n    " + T(3))
    k = patch(k, "    const int nct = PAIR ? nc + peer_nc : nc;", "    const int nct = PAIR ? nc + peer_nc : nc;\n    " + T(4))
    k = patch(k, "    // coalesced store of the verified tile\n    store_tile();\n}",
              "    // coalesced store of the verified tile\n    store_tile();\n    bar_mma();\n    " + T(5) + "\n}")
    cu += ('\nextern "C" int ftblas_debug_times(void *dst) {\n'
           '    return (int)cudaMemcpyFromSymbol(dst, ftb::dbg_t, sizeof(unsigned long long) * 65536 * 8);\n}\n')
    return build("phases", k, cu)



def loader_encode():
    """Timing-only experiment: producer warps 1..3 of the 128 x 128 FT kernel
    form e^T op(A) and op(B) e of every staged k-tile from shared memory (warp 1: the 32 column
    sums of the A stage, warp 2: of the B stage, lane = k, 4 partial chains) as the paper's
    packing-fused encoding would, consuming each stage like an MMA warp.  The sums go to a dummy
    global so they are not eliminated; the regular encode pass still runs (results unchanged)."""
    k, cu = read()
    k = patch(k, "namespace ftb {\n", "namespace ftb {\n__device__ double dbg_loader_sink[1024];\n")
    k = patch(k, "            mbar_init(&empty_bar[s], NT / 32);  // one arrival per MMA warp",
              "            mbar_init(&empty_bar[s], NT / 32 + ((FT && NWN == 4) ? 2 : 0));")
    k = patch(k, "            mbar_arrive(&norm_bar);\n        }\n",
              "            mbar_arrive(&norm_bar);\n"
              "            if (pt < 96) {\n"
              "                const int wsel = (pt - 32) >> 5, kq = pt & 31;\n"
              "                double acc4[4] = {0.0, 0.0, 0.0, 0.0};\n"
              "                for (int kt = 0; kt < ktiles; kt++) {\n"
              "                    const int st = kt % NS;\n"
              "                    mbar_wait(&full_bar[st], (kt / NS) & 1);\n"
              "                    const double *ts = wsel == 0 ? sA(st) : sB(st);\n"
              "                    double s4[4] = {0.0, 0.0, 0.0, 0.0};\n"
              "                    if (wsel == 0) {\n"
              "#pragma unroll 8\n"
              "                        for (int mn = 0; mn < 128; mn++) s4[mn & 3] += ts[Tile<KCA>::idx(mn, kq)];\n"
              "                    } else {\n"
              "#pragma unroll 8\n"
              "                        for (int mn = 0; mn < BNT; mn++) s4[mn & 3] += ts[Tile<KCB, BNT>::idx(mn, kq)];\n"
              "                    }\n"
              "                    __syncwarp();\n"
              "                    if ((pt & 31) == 0) mbar_arrive(&empty_bar[st]);\n"
              "                    for (int u = 0; u < 4; u++) acc4[u] += s4[u];\n"
              "                }\n"
              "                dbg_loader_sink[(blockIdx.x * 64 + pt) & 1023] = (acc4[0] + acc4[1]) + (acc4[2] + acc4[3]);\n"
              "            }\n"
              "        }\n")
    return build("loader_encode", k, cu)


if __name__ == "__main__":
    for v in sys.argv[1:] or ["phases"]:
        print(globals()[v]())
