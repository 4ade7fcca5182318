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


def _worker(rank, world, port, tA, chunks, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        w = syn.Workload("shard", 300, 300, 50, tA, "N", 1.5, -0.5, "uniform", True, seed=17)
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
        captured = {"entries": []}
        C_flat = torch.from_numpy(C_loc.reshape(-1, order="F").copy())

        def cpu_gemm(ta, tb, M_, N_, K_, al, A_, lda_, B_, ldb_, be, C_, ldc_, col_offset, append):
            # the oracle on the column block [col_offset, col_offset + N_) of this rank's C
            Bm = B_.numpy()[: ldb_ * N_].reshape((ldb_, N_), order="F")
            Cm = C_.numpy()[: ldc_ * N_].reshape((ldc_, N_), order="F")
            plj = None
            if pl is not None:
                sel = (pl[1] >= col_offset) & (pl[1] < col_offset + N_)
                plj = (pl[0][sel], pl[1][sel] - col_offset, pl[2][sel])
            entries, st = oracle.abft_dgemm(ta, tb, M_, N_, K_, al, A_, lda_, Bm, ldb_, be, Cm, ldc_,
                                            faults=plj)
            for e in entries:  # block-global columns, as ftblas_dgemm_ex reports them
                e = dict(e)
                e["j"] = int(e["j"]) + col_offset
                e["tile_n"] = int(e["tile_n"]) + col_offset // 128
                captured["entries"].append(e)

        if chunks == "geo":  # explicit geometric bounds, from rank 0's (largest) shard on every rank
            m_ref = shard.shard_rows(w.M, world, 0)[1] - shard.shard_rows(w.M, world, 0)[0]
            chunks = shard.broadcast_chunk_bounds(m_ref, w.N, sms=2)
            assert len(chunks) == 2
        shard.sharded_dgemm(cpu_gemm, tA, "N", w.M, w.N, w.K, w.alpha, A_loc, lda, B_t, d["ldb"],
                            w.beta, C_flat, max(1, m), rank=rank, world=world, chunks=chunks)
        C_loc = C_flat.numpy().reshape((max(1, m), w.N), order="F")[:m]
        ents = shard.gather_reports(shard.globalize(captured["entries"], r0))
        parts = [None] * world
        dist.all_gather_object(parts, (r0, r1, C_loc))
        if rank == 0:
            q.put((ents, parts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tA,chunks", [("N", 1), ("T", 1), ("N", 2), ("T", 3), ("N", "geo")])
def test_sharded_equals_unsharded(tA, chunks):
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, tA, chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    ents, parts = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = syn.Workload("shard", 300, 300, 50, tA, "N", 1.5, -0.5, "uniform", True, seed=17)
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


def test_chunk_bounds_whole_tiles():
    assert shard.chunk_bounds(300, 2) == [(0, 256), (256, 300)]
    assert shard.chunk_bounds(300, 8) == [(0, 128), (128, 256), (256, 300)]
    for N in (1, 128, 129, 16384, 16500):
        for ch in (1, 2, 3, 8):
            b = shard.chunk_bounds(N, ch)
            assert b[0][0] == 0 and b[-1][1] == N
            assert all(c0 % 128 == 0 and c0 < c1 for c0, c1 in b)
            assert all(p[1] == q[0] for p, q in zip(b, b[1:]))


def test_broadcast_chunk_bounds_geometric_whole_waves():
    import math
    for m, N in [(2048, 16384), (4096, 16384), (8192, 16384), (4096, 32768), (300, 300), (16384, 256)]:
        b = shard.broadcast_chunk_bounds(m, N)
        assert b[0][0] == 0 and b[-1][1] == N
        assert all(c0 % 128 == 0 and c0 < c1 for c0, c1 in b)
        assert all(p[1] == q[0] for p, q in zip(b, b[1:]))
        rows = -(-m // 128)
        waves = [math.ceil(rows * -(-(c1 - c0) // 128) / 148) for c0, c1 in b]
        ideal = rows * -(-N // 128) / 148
        assert sum(waves) <= math.ceil(ideal) + 1, (m, N, b, waves, ideal)
    # c3 at 8 GPUs: 9 / 18 / 37 tile-columns (1, 2, 4 waves), then the rest
    assert [(c1 - c0) // 128 for c0, c1 in shard.broadcast_chunk_bounds(2048, 16384)] == [9, 18, 37, 64]


class _NumpyEncoder:
    """Test stand-in for ftblas_encode_b on CPU tensors: the definitions of the B-side encoding
    (w_J = sum of the tile's columns, column 1-norms, tile maxima of the row |.| sums) written into
    the library's section layout (ftblas_b_encoding_layout, which needs no GPU)."""

    def __init__(self):
        from paper_2305_02444_b200 import ftblas
        self.layout = ftblas.ftblas_b_encoding_layout

    def empty(self, n):
        return torch.empty(n, dtype=torch.float64)

    def encode(self, transB, n, K, B, ldb, out):
        Bv = B.numpy()
        if transB in ("N", "n"):
            P = np.stack([Bv[j * ldb: j * ldb + K] for j in range(n)], axis=1)          # K x n
        else:
            P = np.stack([Bv[k * ldb: k * ldb + n] for k in range(K)], axis=0)          # K x n
        o_n, o_m, tot = self.layout(n, K)
        kp = self.layout(128, K)[0]
        e = np.zeros(tot)
        for t in range(-(-n // 128)):
            blk = P[:, t * 128:(t + 1) * 128]
            e[t * kp: t * kp + K] = blk.sum(axis=1)
            e[o_m + t] = np.abs(blk).sum(axis=1).max() if K else 0.0
        e[o_n: o_n + n] = np.abs(P).sum(axis=0)
        out[:tot] = torch.from_numpy(e)


def _enc_worker(rank, world, port, tB, chunks, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        M, N, K = 256, 700, 70
        rng = np.random.default_rng(5)
        Bm = rng.uniform(-1, 1, (K, N) if tB == "N" else (N, K))
        ldb = Bm.shape[0]
        B_t = torch.from_numpy(np.asfortranarray(Bm).reshape(-1, order="F").copy()) if rank == 0 \
            else torch.zeros(Bm.size, dtype=torch.float64)
        enc = _NumpyEncoder()
        seen = []

        def gemm(ta, tb, m, n, K_, al, A_, lda_, B_, ldb_, be, C_, ldc_, col_offset, append, b_enc=None):
            ref = enc.empty(enc.layout(n, K_)[2])
            enc.encode(tb, n, K_, B_, ldb_, ref)
            seen.append((col_offset, n, bool(torch.equal(b_enc, ref))))

        A = np.zeros((M, K))
        C = torch.zeros(M * N, dtype=torch.float64)
        shard.sharded_dgemm(gemm, "N", tB, M, N, K, 1.0, A, M, B_t, ldb, 0.0, C, M, rank=rank, world=world,
                            chunks=chunks, encoder=enc)
        q.put((rank, seen))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("tB,chunks", [("N", 1), ("N", 3), ("T", 1)])
def test_shared_b_encoding_equals_whole_encoding(tB, chunks):
    """Every rank's assembled op(B) encoding (slices encoded by the ranks, all-gathered) equals the
    encoding of the whole block, for every column block of the chunked broadcast."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_enc_worker, args=(r, world, port, tB, chunks, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for _, seen in res:
        assert seen and all(ok for _, _, ok in seen), seen
        assert sum(n for _, n, _ in seen) == 700


def test_b_encoding_slices_cover_tiles():
    for n in (1, 128, 300, 700, 16384):
        for world in (1, 2, 3, 8):
            sl = shard.b_encoding_slices(n, world)
            assert sl[0][0] == 0 and sl[-1][1] == -(-n // 128)
            assert sum(nr for _, _, nr in sl) == n
            assert all(a[1] == b[0] for a, b in zip(sl, sl[1:]))
