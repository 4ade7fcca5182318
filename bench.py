#!/usr/bin/env python
"""bench.py -- ABFT DGEMM (FP64, Huang-Abraham checksums fused) throughput on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one full hot-path pass over the workload: the checksum-encode kernel, the
DMMA GEMM kernel with fused checksum accumulation and the verify/locate/correct
epilogue, with the workload's seeded bit flips injected (and, for N > 1, the NCCL
broadcast of op(B) to the row-block shards).  Prints ONE JSON line on rank 0.
Launch for N > 1:  python -m torch.distributed.run --nproc-per-node N --master-addr
127.0.0.1 --master-port P bench.py --gpus N ...
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synthetic as syn  # noqa: E402

METRIC = "ABFT DGEMM FP64 TFLOP/s at 1/2/4/8 B200; FT overhead % vs non-FT; % FP64 peak"
DEFAULT_WORKLOAD = "c3_16384_sharded"
# FP64 DMMA peak of B200: 148 SMs x 64 FP64 FMA/clk/SM (DMMA.8x8x4 = 256 FMA per 4 clk per SM)
# x 2 FLOP x 1.965 GHz max SM clock = 37.23 TFLOP/s; the DMMA microbenchmark reached 37.15
# (profiles/r01_fp64_pipes.txt).  See DESIGN.md section 5 for why this, not bf16 x ratio.
FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12


def base_config(w) -> dict:
    """The workload keys both arms (ours and --impl reference) report."""
    return {"workload": w.name, "M": w.M, "N": w.N, "K": w.K, "transA": w.transA,
            "transB": w.transB, "alpha": w.alpha, "beta": w.beta,
            "dist": {"uniform": "U[-1,1]", "normal": "N(0,1)"}[w.dist], "seed": w.seed,
            "injected_flips": w.n_flips, "flip_bits": [syn.BIT_LO, syn.BIT_HI],
            "verification_tile": [syn.TILE_M, syn.TILE_N]}


def ratio_rule(achieved: float) -> dict:
    """The contraction peak by the task's ratio rule: measured bf16 (MEASURED_PEAKS.json) x the
    nominal FP64 / bf16 ratio of B200 (45 / 2250 TFLOP/s).  Reported beside the DMMA-measured
    peak used for `frac` (the rule's figure is below what cuBLAS DGEMM reaches on these GPUs)."""
    try:
        bf16 = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"])
        src = "MEASURED_PEAKS.json bf16_tflops"
    except (OSError, ValueError, KeyError):
        bf16, src = 1590.0, "fallback 1.59 PFLOP/s (B200_PROFILING.md)"
    peak = bf16 * 45.0 / 2250.0
    return {"peak": peak, "frac": achieved / peak, "how": f"{src} {bf16:.1f} x 45/2250"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.proc, self.lines = gpu, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            p = [x.strip() for x in ln.split(",")]
            if len(p) < 9:
                continue
            try:
                sm.append(float(p[1]))
                smax.append(float(p[2]))
            except ValueError:
                continue
            for n, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(smax), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- helpers
def col_major_rows(x: np.ndarray, r0: int, r1: int) -> np.ndarray:
    return np.asfortranarray(x[r0:r1, :])


def flat_f(x: np.ndarray) -> np.ndarray:
    return np.asfortranarray(x).reshape(-1, order="F")


_OS = {}  # state inherited by the forked oracle workers (inputs are shared copy-on-write)


def _oracle_worker(rank: int):
    import oracle
    w, d, plan, order, faulty, procs, deadline, C = (_OS[k] for k in
                                                     ("w", "d", "plan", "order", "faulty", "procs", "deadline", "C"))
    ntm, ntn = -(-w.M // 128), -(-w.N // 128)
    done, flops, nf = 0, 0.0, 0
    t0 = time.perf_counter()  # the worker's own clock: process start-up (fork of a large parent) is not oracle time
    deadline += t0
    for t in order[rank::procs]:
        mask = np.zeros(ntm * ntn, np.uint8)
        mask[t] = 1
        oracle.abft_dgemm(w.transA, w.transB, w.M, w.N, w.K, w.alpha, d["A"], d["lda"], d["B"],
                          d["ldb"], w.beta, C, w.M, faults=plan, tiles_only=mask)
        tm, tn = t % ntm, t // ntm
        flops += 2.0 * min(128, w.M - tm * 128) * min(128, w.N - tn * 128) * w.K
        done += 1
        nf += t in faulty
        if time.perf_counter() >= deadline:
            break
    return done, flops, nf, time.perf_counter() - t0


def oracle_sample(w, d, plan, seconds: float, procs: int | None = None):
    """Time the CPU oracle, as it stands, on whole verification tiles for about `seconds`: one
    single-threaded oracle process per host core (bounded at 32), each working through its share of
    a fixed tile sample (the first faulty tiles, then seeded random ones) until the deadline."""
    import multiprocessing as mp
    ntm, ntn = -(-w.M // 128), -(-w.N // 128)
    if procs is None:
        procs = max(1, min(len(os.sched_getaffinity(0)), 32, ntm * ntn))
    faulty = sorted({(int(j) // 128) * ntm + int(i) // 128 for i, j in zip(plan[0], plan[1])})
    rng = np.random.default_rng(12345)
    order = faulty[:procs] + [int(t) for t in rng.permutation(ntm * ntn)[:64 * procs]]
    order = list(dict.fromkeys(order))
    _OS.update(w=w, d=d, plan=plan, order=order, faulty=set(faulty), procs=procs,
               deadline=seconds, C=np.asfortranarray(d["C"].copy()))
    if procs == 1:
        res = [_oracle_worker(0)]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_oracle_worker, range(procs), chunksize=1)
    el = max(r[3] for r in res)  # the slowest worker's loop (all run concurrently)
    _OS.clear()
    done, flops, nf = (sum(r[i] for r in res) for i in range(3))
    return {"value": flops / el / 1e12, "unit": "TFLOP/s", "cores": procs, "kind": "oracle",
            "sample": f"{done} of {ntm * ntn} verification tiles (128x128, K={w.K}) of {w.name}, "
                      f"{nf} with injected flips; oracle/ftblas_oracle.c, {procs} single-threaded "
                      f"processes (one per host core), {el:.1f} s (slowest worker's loop)"}


# ----------------------------------------------------------------------------- reference arm
def run_reference(args, w):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    log(f"[reference] generating {w.name} inputs")
    d = syn.make_inputs(w)
    plan = syn.fault_plan(w.M, w.N, w.n_flips, w.seed)
    step_s = max(1.0, min(20.0, 120.0 / max(1, args.steps + args.warmup)))
    for _ in range(args.warmup):
        oracle_sample(w, d, plan, step_s / 4)
    vals = []
    for _ in range(args.steps):
        vals.append(oracle_sample(w, d, plan, step_s))
    v = statistics.median(x["value"] for x in vals)
    cb = dict(vals[-1])
    cb["value"] = v
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "TFLOP/s", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "ms_per_step": 1e3 * step_s,
           "config": dict(base_config(w), parallelism=f"CPU oracle, {cb['cores']} processes, bounded tile sample per step",
                          l2="n/a (host)"),
           "cpu_baseline": cb,
           "e2e": {"value": v, "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


# ----------------------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=DEFAULT_WORKLOAD, choices=list(syn.CONFIG_BY_NAME))
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N > 1 (gloo: functional check of the multi-rank "
                         "path on fewer GPUs than ranks; not a performance configuration)")
    ap.add_argument("--tiles", default="auto", choices=["auto", "full", "pair", "ws"],
                    help="CTA tiling policy of the GEMM kernels (ftblas_set_tile_policy)")
    ap.add_argument("--no-share-b-encoding", action="store_true",
                    help="N > 1: every rank encodes all of op(B) (default: each rank encodes 1/N of its "
                         "column tiles, all-gathered; shard.shared_b_encoding)")
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-configs", action="store_true",
                    help="do not time BASELINE configs[0..2] beside the headline workload")
    ap.add_argument("--skip-cpu", action="store_true")
    args = ap.parse_args()
    w = syn.CONFIG_BY_NAME[args.workload]
    if args.impl == "reference":
        return run_reference(args, w)
    args.warmup = max(3, args.warmup)

    import torch
    import torch.distributed as dist
    from paper_2305_02444_b200 import ftblas as fb
    from paper_2305_02444_b200 import shard

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local % max(1, torch.cuda.device_count()))
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    stream = torch.cuda.current_stream()
    fb.ftblas_set_stream(stream)
    fb.ftblas_set_checksum_mode("gemm")
    fb.ftblas_set_tile_policy(args.tiles)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if args.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda" if args.backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---------------------------------------------------------------- inputs
    t0 = time.perf_counter()
    d = syn.make_inputs(w)
    plan = syn.fault_plan(w.M, w.N, w.n_flips, w.seed)
    r0, r1 = shard.shard_rows(w.M, world, rank)
    m = r1 - r0
    if w.transA == "N":
        A_loc = col_major_rows(d["A"], r0, r1)
        lda = max(1, m)
    else:
        A_loc = np.asfortranarray(d["A"][:, r0:r1])
        lda = d["lda"]
    C_loc = col_major_rows(d["C"], r0, r1)
    ldc = max(1, m)
    plan_loc = shard.shard_plan(plan, r0, r1)
    A_dev = torch.from_numpy(flat_f(A_loc)).cuda()
    B_dev = (torch.from_numpy(flat_f(d["B"])).cuda() if rank == 0
             else torch.empty(d["B"].size, dtype=torch.float64, device="cuda"))
    C0_dev = torch.from_numpy(flat_f(C_loc)).cuda()
    C_dev = C0_dev.clone()
    log(f"[rank {rank}] inputs ready in {time.perf_counter() - t0:.1f} s; rows [{r0},{r1})")
    flops_total = 2.0 * w.M * w.N * w.K
    flops_local = 2.0 * m * w.N * w.K

    keep = []  # op(B) encodings of the current step (the kernels read them asynchronously)

    def gemm_ft(ta, tb, M_, N_, K_, al, A_, lda_, B_, ldb_, be, C_, ldc_, col_offset, append, b_enc=None):
        # blocks after the first reuse the checksum encoding of this rank's A (unchanged); with
        # b_enc the block's op(B) encoding was computed once across the ranks (shard.shared_b_encoding)
        if b_enc is not None:
            b_enc = b_enc if b_enc.is_cuda else b_enc.cuda()
            keep.append(b_enc)
            fb.ftblas_set_b_encoding(b_enc, N_, K_)
        fb.ftblas_dgemm_ex(ta, tb, M_, N_, K_, al, A_, lda_, B_, ldb_, be, C_, ldc_, 0, col_offset, append,
                           reuse_a=append, b_encoded=b_enc is not None)
        if b_enc is not None:
            fb.ftblas_set_b_encoding(None)

    class Encoder:
        """ftblas_encode_b for shard.shared_b_encoding; gloo collectives run on host copies."""
        layout = staticmethod(fb.ftblas_b_encoding_layout)

        @staticmethod
        def empty(n):
            return torch.empty(n, dtype=torch.float64, device="cuda" if args.backend == "nccl" else "cpu")

        @staticmethod
        def encode(tb, n, K_, B_, ldb_, out):
            dst = out if out.is_cuda else torch.empty(out.numel(), dtype=torch.float64, device="cuda")
            fb.ftblas_encode_b(tb, n, K_, B_, ldb_, dst)
            if dst is not out:
                out.copy_(dst)
    encoder = Encoder() if (world > 1 and not args.no_share_b_encoding) else None

    def gemm_noft(ta, tb, M_, N_, K_, al, A_, lda_, B_, ldb_, be, C_, ldc_, col_offset, append):
        fb.ftblas_dgemm_noft(ta, tb, M_, N_, K_, al, A_, lda_, B_, ldb_, be, C_, ldc_)

    # N > 1: op(B) is broadcast in column chunks of whole tiles, the GEMM of chunk c overlapping
    # the broadcast of chunks > c (shard.sharded_dgemm); N = 1: one call, no exchange.
    # the chunk bounds must be identical on every rank (each chunk is one collective):
    # computed from rank 0's row count, the largest shard
    m_ref = shard.shard_rows(w.M, world, 0)[1] - shard.shard_rows(w.M, world, 0)[0]
    chunks = shard.broadcast_chunk_bounds(m_ref, w.N) if (world > 1 and w.transB == "N") else 1

    def step(gemm, broadcast):
        # C := alpha AB + beta C accumulates into C; the value drifts but the work is identical
        keep.clear()
        shard.sharded_dgemm(gemm, w.transA, w.transB, w.M, w.N, w.K, w.alpha, A_dev, lda, B_dev,
                            d["ldb"], w.beta, C_dev, ldc, rank=rank, world=world,
                            broadcast=broadcast and world > 1, chunks=chunks if broadcast else 1,
                            encoder=encoder if gemm is gemm_ft else None)

    def timed(fn, steps, warm=1):
        for _ in range(warm):  # first launches of a kernel instantiation load its module
            fn()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        return max_over_ranks(e0.elapsed_time(e1)) / steps

    K, W = args.steps, args.warmup
    if plan_loc is not None and len(plan_loc[0]):
        fb.ftblas_set_fault_plan(*plan_loc)
    else:
        fb.ftblas_clear_fault_plan()
    for _ in range(W):
        step(gemm_ft, True)
    torch.cuda.synchronize()

    # ---------------------------------------------------------------- headline: FT + flips
    clk = ClockSampler(local)
    with clk:
        time.sleep(0.4)
        fb.ftblas_profile(True)
        fb.ftblas_profile_read()
        n0 = fb.ftblas_launch_count()
        ms_step = timed(lambda: step(gemm_ft, True), K, warm=0)  # warmed above; profiled: exactly K steps
        launches = fb.ftblas_launch_count() - n0
        fb.ftblas_profile(False)
        enc_ms, gemm_ms, n_g = fb.ftblas_profile_read()
        rep = fb.ftblas_report_fetch(fb.Report(max(16, 2 * len(plan_loc[0]))))
        # overhead comparisons on the local GEMM call (no broadcast), same inputs
        ms_ft_err = timed(lambda: step(gemm_ft, False), K)
        fb.ftblas_clear_fault_plan()
        ms_ft0 = timed(lambda: step(gemm_ft, False), K)
        ms_noft = timed(lambda: step(gemm_noft, False), K)
        # the non-FT baseline under every CTA tiling (the overhead is also given against the
        # fastest of them, not only against the same tiling)
        noft_by_tiles = {}
        for tl in ("full", "pair", "ws"):
            fb.ftblas_set_tile_policy(tl)
            noft_by_tiles[tl] = timed(lambda: step(gemm_noft, False), max(2, min(K, 5)))
        fb.ftblas_set_tile_policy(args.tiles)
        ms_noft_best = min([ms_noft] + list(noft_by_tiles.values()))
        # the same FT call with the checksum row/column accumulated in the main mainloop
        # (FTBLAS_CHECKSUM_FUSED) instead of the checksum GEMMs, for comparison
        fb.ftblas_set_checksum_mode("fused")
        ms_fused0 = timed(lambda: step(gemm_ft, False), max(1, min(K, 3)))
        fb.ftblas_set_checksum_mode("gemm")
        for _ in range(2):  # keep the GPU loaded until the sampler stops
            step(gemm_ft, False)
        torch.cuda.synchronize()
    clocks = clk.summary()
    planned_local = len(plan_loc[0])
    entries = shard.globalize(rep.entries(), r0)
    located = sorted((e["i"], e["j"]) for e in entries)
    want = sorted(zip((plan_loc[0] + r0).tolist(), plan_loc[1].tolist()))
    ok_local = (rep.count == planned_local) and located == want
    ok_all = sum_over_ranks(0.0 if ok_local else 1.0) == 0.0
    reported = int(sum_over_ranks(float(rep.count)))
    launches_all = int(sum_over_ranks(float(launches)))
    # per step: a step of a chunked multi-GPU run is several main-kernel launches (one per
    # op(B) column chunk); the roofline counts the step's algorithmic FLOPs on this rank over
    # the summed device time of those launches
    gemm_step_ms = gemm_ms / max(1, K)
    enc_step_ms = enc_ms / max(1, K)
    gemm_launches_per_step = n_g / max(1, K)

    # ---------------------------------------------------------------- e2e: host buffers
    e2e = None
    if not args.skip_e2e:
        if plan_loc is not None and len(plan_loc[0]):
            fb.ftblas_set_fault_plan(*plan_loc)

        def pinned(x: np.ndarray):
            t = torch.empty(x.size, dtype=torch.float64, pin_memory=True)
            t.numpy()[:] = flat_f(x)
            return t

        hA, hB, hC = pinned(A_loc), pinned(d["B"]), pinned(C_loc)
        h2d = A_loc.nbytes + d["B"].nbytes + (C_loc.nbytes if w.beta != 0.0 else 0)
        d2h = C_loc.nbytes

        def e2e_step():
            fb.ftblas_dgemm_host(w.transA, w.transB, m, w.N, w.K, w.alpha, hA.data_ptr(), lda,
                                 hB.data_ptr(), d["ldb"], w.beta, hC.data_ptr(), ldc, None)

        e2e_step()
        ms_e2e = timed(e2e_step, max(2, min(K, 3)))
        # the last step's report (accumulated over the pipeline's blocks): every flip located
        n_loc = 0 if plan_loc is None else len(plan_loc[0])
        rep_e2e = fb.ftblas_report_fetch(fb.Report(max(16, 2 * n_loc)))
        got_e2e = sorted((e["i"], e["j"]) for e in rep_e2e.entries())
        want_e2e = [] if plan_loc is None else sorted(zip(plan_loc[0].tolist(), plan_loc[1].tolist()))
        e2e_ok = sum_over_ranks(0.0 if (rep_e2e.count == len(want_e2e) and got_e2e == want_e2e) else 1.0) == 0.0
        fb.ftblas_clear_fault_plan()
        e2e = {"value": flops_total / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOP/s",
               "h2d_bytes_per_step": int(sum_over_ranks(float(h2d))),
               "d2h_bytes_per_step": int(sum_over_ranks(float(d2h))),
               "ms_per_step": ms_e2e,
               "all_located_and_corrected": bool(e2e_ok),
               "path": "ftblas_dgemm_host (pinned host A,B,C -> device, ABFT DGEMM, C -> host)"}
        del hA, hB, hC

    # ---------------------------------------------------------------- traffic (ncu capture)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath))
            key = f"{w.name}/world{world}"
            if key in tj:
                traffic = tj[key]["dram_bytes_per_launch"]
        except (ValueError, KeyError):
            traffic = None

    # ---------------------------------------------------------------- the other 1-GPU configs
    # BASELINE configs[0..2] (each under 10 ms per call) in the same driver-timed run: FT with
    # and without the config's flips, the non-FT baseline under every CTA tiling, located vs
    # planned flips, the main kernel's roofline fraction.  configs[4] (17 GB, quoted for an
    # 8-GPU shard) is left to --workload.
    configs = None
    if world == 1 and not args.skip_configs:
        configs = {}
        for wn in ("c0_256_ft", "c1_4096_tn", "c2_rankk_16384x256"):
            if wn == w.name:
                continue
            cw = syn.CONFIG_BY_NAME[wn]
            log(f"[bench] config {wn}")
            cd = syn.make_inputs(cw)
            cplan = syn.fault_plan(cw.M, cw.N, cw.n_flips, cw.seed)
            cA = torch.from_numpy(flat_f(cd["A"])).cuda()
            cB = torch.from_numpy(flat_f(cd["B"])).cuda()
            cC = torch.from_numpy(flat_f(cd["C"])).cuda()

            def cft():
                fb.ftblas_dgemm(cw.transA, cw.transB, cw.M, cw.N, cw.K, cw.alpha, cA, cd["lda"], cB, cd["ldb"],
                                cw.beta, cC, cd["ldc"])

            def cnoft():
                fb.ftblas_dgemm_noft(cw.transA, cw.transB, cw.M, cw.N, cw.K, cw.alpha, cA, cd["lda"], cB,
                                     cd["ldb"], cw.beta, cC, cd["ldc"])
            cflops = 2.0 * cw.M * cw.N * cw.K
            ctf = lambda ms: cflops / (ms * 1e-3) / 1e12  # noqa: E731
            fb.ftblas_set_fault_plan(*cplan)
            for _ in range(W):
                cft()
            fb.ftblas_profile(True)
            fb.ftblas_profile_read()
            c_err = timed(cft, K, warm=0)
            fb.ftblas_profile(False)
            _, c_gemm_ms, c_n = fb.ftblas_profile_read()
            crep = fb.ftblas_report_fetch(fb.Report(max(16, 2 * cw.n_flips)))
            got = sorted((e["i"], e["j"]) for e in crep.entries())
            want = sorted(zip(cplan[0].tolist(), cplan[1].tolist()))
            fb.ftblas_clear_fault_plan()
            c_ft0 = timed(cft, K, warm=1)
            c_noft = timed(cnoft, K, warm=W)
            c_noft_t = {}
            for tl in ("full", "pair", "ws"):
                fb.ftblas_set_tile_policy(tl)
                c_noft_t[tl] = timed(cnoft, K, warm=2)
            fb.ftblas_set_tile_policy(args.tiles)
            c_best = min(list(c_noft_t.values()) + [c_noft])
            k_ms = c_gemm_ms / max(1, c_n)
            configs[wn] = {
                "M": cw.M, "N": cw.N, "K": cw.K, "transA": cw.transA, "transB": cw.transB,
                "alpha": cw.alpha, "beta": cw.beta, "injected_flips": cw.n_flips,
                "ft_flips_tflops": ctf(c_err), "ft_0err_tflops": ctf(c_ft0), "noft_tflops": ctf(c_noft),
                "ms_per_call": {"ft_flips": c_err, "ft_0err": c_ft0, "noft": c_noft},
                "ft_overhead_pct": {"errors_0": 100.0 * (c_ft0 / c_noft - 1.0),
                                    f"errors_{cw.n_flips}": 100.0 * (c_err / c_noft - 1.0)},
                "ft_overhead_vs_best_noft_pct": {"errors_0": 100.0 * (c_ft0 / c_best - 1.0),
                                                 f"errors_{cw.n_flips}": 100.0 * (c_err / c_best - 1.0)},
                "noft_tflops_by_tiling": {k: ctf(v) for k, v in c_noft_t.items()},
                "corrections": {"planned": len(want), "reported": int(crep.count),
                                "all_located_and_corrected": bool(crep.count == len(want) and got == want)},
                "roofline": {"bound": "tensor", "kernel_ms": k_ms, "achieved": cflops / (k_ms * 1e-3) / 1e12,
                             "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
                             "frac": cflops / (k_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS},
            }
            del cA, cB, cC, cd
            torch.cuda.empty_cache()

    cpu = None
    if rank == 0 and world == 1 and not args.skip_cpu:
        log("[bench] timing the CPU oracle on a bounded sample")
        cpu = oracle_sample(w, d, plan, args.cpu_seconds)

    if rank == 0:
        value = flops_total / (ms_step * 1e-3) / 1e12
        achieved = flops_local / (gemm_step_ms * 1e-3) / 1e12
        tf = lambda ms: flops_total / (ms * 1e-3) / 1e12  # noqa: E731
        out = {
            "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "strong", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": dict(base_config(w),
                       parallelism= f"row-block x{world}" + (
                           (f", op(B) {args.backend.upper()} broadcast per step in {len(chunks)} column chunks "
                            f"{[c1 - c0 for c0, c1 in chunks]} overlapped with the GEMM"
                            if isinstance(chunks, list) else f", op(B) {args.backend.upper()} broadcast per step")
                           + (f"; op(B) encoding shared: each rank encodes 1/{world} of each chunk's column tiles, "
                              "all-gathered" if encoder is not None else "; op(B) encoded on every rank")
                           if world > 1 else ""),
                       l2="no flush: operands (%.1f GiB) >> 126 MB L2" % ((d["A"].nbytes + d["B"].nbytes + d["C"].nbytes) / 2**30)),
            "fp64_peak_tflops": FP64_PEAK_TFLOPS,
            "pct_fp64_peak": 100.0 * value / (FP64_PEAK_TFLOPS * world),
            "noft_tflops": tf(ms_noft), "ft_0err_tflops": tf(ms_ft0), "ft_flips_tflops": tf(ms_ft_err),
            "ft_overhead_pct": {"errors_0": 100.0 * (ms_ft0 / ms_noft - 1.0),
                                f"errors_{w.n_flips}": 100.0 * (ms_ft_err / ms_noft - 1.0)},
            "ft_overhead_vs_best_noft_pct": {"errors_0": 100.0 * (ms_ft0 / ms_noft_best - 1.0),
                                             f"errors_{w.n_flips}": 100.0 * (ms_ft_err / ms_noft_best - 1.0),
                                             "noft_tflops_by_tiling": {k: tf(v) for k, v in noft_by_tiles.items()}},
            "tiles": args.tiles,
            "checksum_mode": "gemm (checksum row/column by split-K DMMA GEMMs before the main GEMM)",
            "fused_mode": {"ft_0err_tflops": tf(ms_fused0), "ft_overhead_pct": 100.0 * (ms_fused0 / ms_noft - 1.0),
                           "note": "checksums accumulated in the main mainloop (DFMA beside DMMA)"},
            "corrections": {"planned": int(len(plan[0])), "reported": reported, "all_located_and_corrected": bool(ok_all)},
            "gpu_launches": launches_all,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": FP64_PEAK_TFLOPS,
                         "unit": "TFLOP/s", "frac": achieved / FP64_PEAK_TFLOPS, "traffic": traffic,
                         "kernel": "gemm_kernel<FT_PRE> (TMA + DMMA mainloop, verify/locate/correct epilogue)",
                         "kernel_ms": gemm_step_ms,
                         "kernel_launches_per_step": gemm_launches_per_step,
                         "checksum_stage_ms": enc_step_ms,
                         "peak_source": "148 SM x 64 FP64 FMA/clk x 2 x 1.965 GHz (DMMA microbench 37.15, profiles/r01_fp64_pipes.txt)",
                         "peak_ratio_rule": ratio_rule(achieved)},
            "clocks": clocks,
            "e2e": e2e,
            "configs": configs,
            "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
