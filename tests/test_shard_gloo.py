"""Multi-process (world_size 2, gloo, CPU) test of the row-block sharding host logic:
ranges, fault-plan slicing, the op(B) broadcast, report globalization and gathering.
The single-device GEMM is the CPU oracle here (tests may use it); on GPUs it is
ftblas_dgemm.  The sharded result must equal the unsharded oracle run exactly."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synthetic as syn
from paper_2305_02444_b200 import shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, tA, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = syn.Workload("shard", 300, 140, 50, tA, "N", 1.5, -0.5, "uniform", True, seed=17)
        d = syn.make_inputs(w)
        plan = syn.fault_plan(w.M, w.N, 3, 4)
        r0, r1 = shard.shard_rows(w.M, world, rank)
        m = r1 - r0
        if tA == "N":
            A_loc = np.asfortranarray(d["A"][r0:r1, :]); lda = max(1, m)
        else:
            A_loc = np.asfortranarray(d["A"][:, r0:r1]); lda = d["lda"]
        C_loc = np.asfortranarray(d["C"][r0:r1, :])
        # B only exists on rank 0 before the broadcast
        B_t = torch.from_numpy(np.asfortranarray(d["B"]).reshape(-1, order="F").copy()) if rank == 0 \
            else torch.zeros(d["B"].size, dtype=torch.float64)
        pl = shard.shard_plan(plan, r0, r1)
        captured = {}

        def cpu_gemm(ta, tb, M_, N_, K_, al, A_, lda_, B_, ldb_, be, C_, ldc_, rep):
            Bm = B_.numpy().reshape((ldb_, -1), order="F")
            entries, st = oracle.abft_dgemm(ta, tb, M_, N_, K_, al, A_, lda_, Bm, ldb_, be, C_, ldc_,
                                            faults=pl)
            captured["entries"] = entries

        shard.sharded_dgemm(cpu_gemm, tA, "N", w.M, w.N, w.K, w.alpha, A_loc, lda, B_t, d["ldb"],
                            w.beta, C_loc, max(1, m), rank=rank, world=world)
        ents = shard.gather_reports(shard.globalize(captured["entries"], r0))
        parts = [None] * world
        dist.all_gather_object(parts, (r0, r1, C_loc))
        if rank == 0:
            q.put((ents, parts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tA", ["N", "T"])
def test_sharded_equals_unsharded(tA):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, tA, q)) for r in range(world)]
    for p in procs:
        p.start()
    ents, parts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = syn.Workload("shard", 300, 140, 50, tA, "N", 1.5, -0.5, "uniform", True, seed=17)
    d = syn.make_inputs(w)
    plan = syn.fault_plan(w.M, w.N, 3, 4)
    C = np.asfortranarray(d["C"].copy())
    full, _ = oracle.abft_dgemm(tA, "N", w.M, w.N, w.K, w.alpha, d["A"], d["lda"], d["B"], d["ldb"],
                                w.beta, C, w.M, faults=plan)
    key = lambda es: sorted((e["tile_m"], e["tile_n"], e["i"], e["j"], e["kind"]) for e in es)
    assert key(ents) == key(full) and len(full) == 3
    stitched = np.vstack([c for (_, _, c) in sorted(parts, key=lambda t: t[0])])
    assert np.array_equal(stitched, C)


def test_shard_rows_cover_whole_tiles():
    for M in (1, 127, 128, 300, 16384):
        for world in (1, 2, 3, 4, 8):
            rs = [shard.shard_rows(M, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == M
            for (a, b), (c, _) in zip(rs, rs[1:]):
                assert b == c and (a % 128 == 0 or a == b)
    plan = (np.array([5, 130, 260]), np.array([1, 2, 3]), np.array([40, 50, 60]))
    i, j, b = shard.shard_plan(plan, 128, 256)
    assert i.tolist() == [2] and j.tolist() == [2] and b.tolist() == [50]
