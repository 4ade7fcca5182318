// ftblas_ws.cuh -- persistent, warp-specialized ABFT DGEMM with the epilogue staged in TMEM.
//
// One CTA per SM walks its share of the 128 x 128 tiles of C (tile x = blockIdx.x + i gridDim.x,
// rasterized by tile_coords).  Three roles run concurrently:
//   producer  (warp 12, one thread; all of warpgroup 3 for the cp.async fallback): streams the
//             operand tiles of every k-tile of every tile of the CTA through a STAGES-deep TMA /
//             mbarrier ring (the ring runs across tile boundaries) and prefetches each tile's C0
//             into L2 near the end of its mainloop;
//   MMA       (warps 0..7, 64 x 32 warp tiles, the mainloop of gemm_kernel<NWN = 4>): DMMA into
//             registers; at the end of a tile the accumulators are injected with the planned
//             flips (test harness), written to one of two TMEM buffers (tcgen05.st) and handed
//             over with an mbarrier -- the warps start the next tile's mainloop at once;
//   epilogue  (warps 8..11): per tile, read the accumulators back from TMEM (tcgen05.ld), form
//             out = alpha acc + beta C0 with the row / column sums of d = out - beta C0 and the
//             |C0| maxima (reading R4k), verify every row and column against the checksum-GEMM
//             references, locate and correct (lines 540, 521; readings
//             R5-R7), and store the verified tile -- all while the MMA warps run the next tile.
// TMEM is used as the accumulator hand-over buffer the DMMA path (FP64 tensor cores have no
// tcgen05.mma kind) otherwise lacks: 2 buffers x 256 columns x 128 lanes x 32 bit = all 512
// columns.  MMA warp w writes lanes 32 (w % 4) .. +31 (its TMEM sub-partition), columns
// buf * 256 + (w / 4) * 128 + [0, 128): the 64 doubles of its accumulator in fragment order
// (element (a, b, e) at words 16 a + 4 b + 2 e).  Epilogue warp ew (= warp % 4) reads the
// same lanes, i.e. exactly the fragments of MMA warps ew and ew + 4 ("twins"), so the
// epilogue reuses the fragment row / column maps of the mainloop.  DESIGN.md section 5.
#pragma once
#include "ftblas_kernels.cuh"

namespace ftb {

constexpr int WS_THREADS = 512;                 // 8 MMA + 4 epilogue + 4 producer-group warps
constexpr int WS_STAGES = 3;
constexpr int WS_STAGE_EL = 2 * TILE_EL;        // A 128 x BK | B 128 x BK
constexpr int WS_SMEM = WS_STAGES * WS_STAGE_EL * 8 + 1024;
// setmaxnreg split of the 64 K registers (one CTA per SM): the MMA warps hold 64 accumulators
// + two sets of fragments; the non-FT epilogue needs fewer registers than the FT one
template <bool FT>
struct WsRegs {
    static constexpr int MMA = FT ? 184 : 192, EPI = FT ? 104 : 88, PROD = FT ? 40 : 32;
    static_assert(256 * MMA + 128 * EPI + 128 * PROD <= 65536,
                  "setmaxnreg budget exceeds the register file of one CTA per SM");
};
constexpr int WS_CAND = 256;                    // candidates per recompute batch (rare path)

// ------------------------------------------------------------------ TMEM primitives
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// 16 consecutive 32-bit TMEM columns of this thread's lane <- 8 doubles (lo, hi word pairs);
// the store is waited for inside the same asm statement, so the source registers are free
// afterwards whatever the compiler schedules next
__device__ __forceinline__ void tmem_st8d(unsigned taddr, const double *v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};\n"
        "tcgen05.wait::st.sync.aligned;\n" ::"r"(taddr),
        "r"(__double2loint(v[0])), "r"(__double2hiint(v[0])), "r"(__double2loint(v[1])), "r"(__double2hiint(v[1])),
        "r"(__double2loint(v[2])), "r"(__double2hiint(v[2])), "r"(__double2loint(v[3])), "r"(__double2hiint(v[3])),
        "r"(__double2loint(v[4])), "r"(__double2hiint(v[4])), "r"(__double2loint(v[5])), "r"(__double2hiint(v[5])),
        "r"(__double2loint(v[6])), "r"(__double2hiint(v[6])), "r"(__double2loint(v[7])), "r"(__double2hiint(v[7]))
        : "memory");
}
// 8 doubles <- 16 consecutive TMEM columns (load and wait in one statement: the registers
// are valid when it returns)
__device__ __forceinline__ void tmem_ld8d(unsigned taddr, double *v) {
    int w[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];\n"
        "tcgen05.wait::ld.sync.aligned;\n"
        : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7]),
          "=r"(w[8]), "=r"(w[9]), "=r"(w[10]), "=r"(w[11]), "=r"(w[12]), "=r"(w[13]), "=r"(w[14]), "=r"(w[15])
        : "r"(taddr)
        : "memory");
#pragma unroll
    for (int q = 0; q < 8; q++) v[q] = __hiloint2double(w[2 * q + 1], w[2 * q]);
}

// verification tile references of tile (tm, tn) -> smem (FT): finalized norms and checksum-GEMM
// slices (side_finalize_kernel / single-split R, S read in place), one row and one column per
// epilogue thread
struct WsSide {
    double nrm_row[BM], nrm_col[BN], pre_r[BM], pre_s[BN], nrm_max[2];
};

template <bool KCA, bool KCB, bool TMA, bool FT>
__global__ void __launch_bounds__(WS_THREADS, 1)
    gemm_ws_kernel(const __grid_constant__ GemmArgs g, const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB) {
    extern __shared__ __align__(1024) double smem_raw[];
    __shared__ __align__(8) unsigned long long full_bar[WS_STAGES], empty_bar[WS_STAGES], acc_full[2], acc_empty[2];
    __shared__ unsigned tmem_base_sh;
    __shared__ WsSide side;
    __shared__ double red_r[4][BM], red_c[2][BN], dres[BM];  // row partials per warp column
    __shared__ unsigned redm_r[4][BM], redm_c[2][BN];
    __shared__ int flags[2 + BM + BN];
    __shared__ int rrank[BM], crank[BN];
    __shared__ double cand_y[FT ? WS_CAND : 1], cand_eb[FT ? WS_CAND : 1];
    double *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) / 8u;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long ntm = (g.M + BM - 1) / BM, ntn = (g.N + BN - 1) / BN, ntiles = ntm * ntn;
    const int ktiles = (g.alpha == 0.0) ? 0 : (int)((g.K + BK - 1) / BK);
    constexpr int PT = 128;  // producer-group threads

    if (tid == 0) {
        for (int s = 0; s < WS_STAGES; s++) {
            mbar_init(&full_bar[s], 1 + (TMA ? 0 : PT));
            mbar_init(&empty_bar[s], 8);     // one arrival per MMA warp
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&acc_full[b], 8);      // MMA warps: accumulators in TMEM
            mbar_init(&acc_empty[b], 4);     // epilogue warps: buffer read
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    if (warp == 13) {  // TMEM: all 512 columns (two accumulator buffers); one CTA per SM
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tmem_base_sh))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const unsigned tbase = tmem_base_sh;

    if (warp >= 12) {
        // ------------------------------------------------------------------ producer group
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(WsRegs<FT>::PROD));
        const int pt = tid - 384;
        if (TMA ? pt == 0 : true) {
            constexpr unsigned TX = TMA ? 2u * TILE_EL * 8u : 0u;
            unsigned kg = 0;
            for (long long x = blockIdx.x; x < ntiles; x += gridDim.x) {
                long long tm, tn;
                tile_coords(x, ntm, ntn, tm, tn);
                const long long m0 = tm * BM, n0 = tn * BN;
                const int pf_kt = max(0, ktiles - WS_STAGES - 1);
                for (int kt = 0; kt < ktiles; kt++, kg++) {
                    const int st = (int)(kg % WS_STAGES);
                    if (kg >= WS_STAGES) mbar_wait(&empty_bar[st], ((kg / WS_STAGES) - 1) & 1);
                    double *sa = smem + st * WS_STAGE_EL;
                    if (pt == 0) mbar_arrive_expect_tx(&full_bar[st], TX);
                    produce_tile<KCA, TMA, 128, PT>(sa, &tmA, &full_bar[st], g.A, g.lda, m0, (long long)kt * BK, g.M, g.K, pt);
                    produce_tile<KCB, TMA, 128, PT>(sa + TILE_EL, &tmB, &full_bar[st], g.B, g.ldb, n0, (long long)kt * BK,
                                                    g.N, g.K, pt);
                    if (!TMA) cp_async_mbar_arrive(&full_bar[st]);
                    if (pt == 0 && kt == pf_kt && g.beta != 0.0 && g.vecC) {
                        // C0 of this tile -> L2 shortly before its epilogue reads it
                        const unsigned bytes = (unsigned)(min((long long)BM, g.M - m0) * 8) & ~15u;
                        const long long nv = min((long long)BN, g.N - n0);
                        if (bytes)
                            for (int c = 0; c < nv; c++) bulk_prefetch_l2(g.C + m0 + (n0 + c) * g.ldc, bytes);
                    }
                }
            }
            if (!TMA) cp_wait<0>();
        }
    } else if (warp >= 8) {
        // ------------------------------------------------------------------ epilogue
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(WsRegs<FT>::EPI));
        const int ew = warp - 8, et = tid - 256;  // epilogue warp (= TMEM sub-partition), thread
        const int wm = ew & 1, wn0 = ew >> 1;     // twins: MMA warps ew (wn0) and ew + 4 (wn0 + 2)
        auto epi_bar = [&]() { asm volatile("bar.sync 2, 128;\n" ::: "memory"); };
        const bool beta0 = g.beta == 0.0, beta1 = g.beta == 1.0;
        const double aa = fabs(g.alpha), ab = fabs(g.beta);
        auto row_of = [&](int a) { return frag_mn<KCA>(wm * 64, a, lane >> 2); };
        auto col_of = [&](int t, int b, int e) { return frag_mn<KCB>((wn0 + 2 * t) * 32, b, 2 * (lane & 3) + e); };
        int it = 0;
        for (long long x = blockIdx.x; x < ntiles; x += gridDim.x, it++) {
            long long tm, tn;
            tile_coords(x, ntm, ntn, tm, tn);
            const long long m0 = tm * BM, n0 = tn * BN;
            const long long mvalid = min((long long)BM, g.M - m0), nvalid = min((long long)BN, g.N - n0);
            if (FT) {  // side data of this tile (loads overlap the wait for the accumulators)
                const long long gi = m0 + et, gj = n0 + et;
                side.nrm_row[et] = et < mvalid ? g.fin_nrmA[gi] : 0.0;
                side.pre_r[et] = et < mvalid ? g.fin_R[tn * g.M + gi] : 0.0;
                side.nrm_col[et] = et < nvalid ? g.fin_nrmB[gj] : 0.0;
                side.pre_s[et] = et < nvalid ? g.fin_S[tm * g.N + gj] : 0.0;
                if (et == 0) {
                    side.nrm_max[0] = g.fin_maxA[tm];
                    side.nrm_max[1] = g.fin_maxB[tn];
                    flags[0] = 0;
                    flags[1] = 0;
                }
            }
            const int buf = it & 1;
            mbar_wait(&acc_full[buf], (unsigned)((it >> 1) & 1));
            tc_fence_after();
            const unsigned tb = tbase + ((unsigned)(32 * ew) << 16) + (unsigned)(buf * 256);
            // ---- pass 1: out, sums, maxima (FT: out back into TMEM in place; non-FT: stored).
            // Twin t (MMA warp ew + 4 t, warp column wn0 + 2 t) row by row: the row partial of a
            // fragment row over this twin's 32 columns (8 elements per lane, 4 lanes per row), the
            // column partials over this warp's 64 rows carried across the rows.
#pragma unroll 1
            for (int t = 0; t < 2; t++) {
                double cs[8];
                unsigned cm[8];
#pragma unroll
                for (int q = 0; q < 8; q++) { cs[q] = 0.0; cm[q] = 0u; }
#pragma unroll 1
                for (int a = 0; a < 8; a++) {
                    double v[8];
                    tmem_ld8d(tb + t * 128 + 16 * a, v);
                    const int row = row_of(a);
                    const long long gi = m0 + row;
                    double rsa = 0.0;
                    unsigned rma = 0u;
#pragma unroll
                    for (int q = 0; q < 8; q++) {
                        const int col = col_of(t, q >> 1, q & 1);
                        const bool ok = row < mvalid && col < nvalid;
                        const long long off = gi + (n0 + col) * g.ldc;
                        double o, d;
                        if (beta0) {
                            o = g.alpha * v[q];
                            d = o;
                        } else {
                            const double c0 = ok ? g.C[off] : 0.0;
                            const double tt = beta1 ? c0 : g.beta * c0;
                            o = fma(g.alpha, v[q], tt);
                            d = o - tt;
                            if (FT) {
                                const unsigned h = (unsigned)__double2hiint(c0) & 0x7fffffffu;
                                rma = max(rma, h);
                                cm[q] = max(cm[q], h);
                            }
                        }
                        if (FT) {
                            d = ok ? d : 0.0;
                            rsa += d;
                            cs[q] += d;
                            v[q] = o;
                        } else if (ok) {
                            g.C[off] = o;
                        }
                    }
                    if (FT) {
                        tmem_st8d(tb + t * 128 + 16 * a, v);
                        // the row's 4 lanes (lane bits 0, 1)
                        rsa += __shfl_xor_sync(0xffffffffu, rsa, 1);
                        rsa += __shfl_xor_sync(0xffffffffu, rsa, 2);
                        rma = max(rma, __shfl_xor_sync(0xffffffffu, rma, 1));
                        rma = max(rma, __shfl_xor_sync(0xffffffffu, rma, 2));
                        if ((lane & 3) == 0) {
                            red_r[wn0 + 2 * t][row] = rsa;
                            redm_r[wn0 + 2 * t][row] = rma;
                        }
                    }
                }
                if (FT) {
                    // column sums over this warp's 64 rows: 8 (b, e) values per lane over the 8
                    // lanes of a column (lane bits 2..4), transposing butterfly -> one column per lane
#pragma unroll
                    for (int off = 4; off <= 16; off <<= 1) {
                        const bool up = (lane & off) != 0;
                        const int h = 8 * 4 / (2 * off);  // 4, 2, 1 values kept
#pragma unroll
                        for (int j = 0; j < 4; j++) {
                            if (j < h) {
                                const double send = up ? cs[j] : cs[j + h];
                                const double keep = up ? cs[j + h] : cs[j];
                                cs[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
                                const unsigned msend = up ? cm[j] : cm[j + h];
                                const unsigned mkeep = up ? cm[j + h] : cm[j];
                                cm[j] = max(mkeep, __shfl_xor_sync(0xffffffffu, msend, off));
                            }
                        }
                    }
                    const int q = ((lane >> 2) & 1) * 4 + ((lane >> 3) & 1) * 2 + ((lane >> 4) & 1);
                    const int col = col_of(t, q >> 1, q & 1);
                    red_c[wm][col] = cs[0];
                    redm_c[wm][col] = cm[0];
                }
            }
            if (FT) {
                epi_bar();
                // ---- verification (readings R3, R4, R4k): thread et checks
                // row et and column et
                auto c0_bound = [&](unsigned h, long long n) {
                    if (h >= 0x7ff00000u) return __longlong_as_double(0x7ff0000000000000ll);
                    return (double)n * __hiloint2double((int)(h + 1u), 0);
                };
                if (et < mvalid) {
                    const double sum = (red_r[0][et] + red_r[1][et]) + (red_r[2][et] + red_r[3][et]);
                    const double c0a = beta0 ? 0.0 : c0_bound(max(max(redm_r[0][et], redm_r[1][et]),
                                                                  max(redm_r[2][et], redm_r[3][et])), nvalid);
                    const double tau = 4.0 * U_ROUND * (double)(g.K + nvalid + 3) *
                                       (aa * side.nrm_row[et] * side.nrm_max[1] + ab * c0a);
                    const double d = sum - g.alpha * side.pre_r[et];
                    dres[et] = d;
                    if (!(fabs(d) <= tau)) flags[2 + atomicAdd(&flags[0], 1)] = et;
                }
                if (et < nvalid) {
                    const double sum = red_c[0][et] + red_c[1][et];
                    const double c0a = beta0 ? 0.0 : c0_bound(max(redm_c[0][et], redm_c[1][et]), mvalid);
                    const double tau = 4.0 * U_ROUND * (double)(g.K + mvalid + 3) *
                                       (aa * side.nrm_max[0] * side.nrm_col[et] + ab * c0a);
                    const double d = sum - g.alpha * side.pre_s[et];
                    if (!(fabs(d) <= tau)) flags[2 + BM + atomicAdd(&flags[1], 1)] = et;
                }
                epi_bar();
                const int nr = flags[0], nc = flags[1];
                if (nr != 0 || nc != 0) {
                    // ---- locate + correct (rare): candidates = (flagged rows, or all rows) x
                    // (flagged columns, or all columns) (readings R5, R7), recomputed from the
                    // definition by the 4 epilogue warps (reading R6), decided by the owner of
                    // the element in TMEM
                    if (et == 0) {
                        atomicAdd(&g.rep->tiles_flagged, 1ull);
                        atomicAdd(&g.rep->rows_flagged, (unsigned long long)nr);
                        atomicAdd(&g.rep->cols_flagged, (unsigned long long)nc);
                        for (int x1 = 1; x1 < nr; x1++)
                            for (int y = x1; y > 0 && flags[2 + y - 1] > flags[2 + y]; y--) {
                                const int tt = flags[2 + y]; flags[2 + y] = flags[2 + y - 1]; flags[2 + y - 1] = tt;
                            }
                        for (int x1 = 1; x1 < nc; x1++)
                            for (int y = x1; y > 0 && flags[2 + BM + y - 1] > flags[2 + BM + y]; y--) {
                                const int tt = flags[2 + BM + y];
                                flags[2 + BM + y] = flags[2 + BM + y - 1];
                                flags[2 + BM + y - 1] = tt;
                            }
                    }
                    rrank[et] = (nr == 0 && et < mvalid) ? et : -1;
                    crank[et] = (nc == 0 && et < nvalid) ? et : -1;
                    epi_bar();
                    if (et < nr) rrank[flags[2 + et]] = et;
                    if (et < nc) crank[flags[2 + BM + et]] = et;
                    epi_bar();
                    const bool single = nr == 1 && nc == 1;  // Huang-Abraham location (line 540)
                    const long long ncr = nr ? nr : mvalid, ncc = nc ? nc : nvalid, ncand = ncr * ncc;
                    for (long long base = 0; base < ncand; base += WS_CAND) {
                        const long long nb = min((long long)WS_CAND, ncand - base);
                        for (long long q = ew; q < nb; q += 4) {
                            const long long idx = base + q;
                            const int rr = (int)(idx % ncr), cc = (int)(idx / ncr);
                            const int r = nr ? flags[2 + rr] : rr, c = nc ? flags[2 + BM + cc] : cc;
                            const long long gi = m0 + r, gj = n0 + c;
                            double s, sa;
                            warp_recompute<KCA, KCB>(g, gi, gj, s, sa);
                            if (lane == 0) {
                                const double c0 = beta0 ? 0.0 : g.C[gi + gj * g.ldc];  // C not yet stored
                                cand_y[q] = beta0 ? g.alpha * s : fma(g.alpha, s, g.beta * c0);
                                cand_eb[q] = 4.0 * U_ROUND * (double)(g.K + 3) * (aa * sa + ab * fabs(c0));
                            }
                        }
                        epi_bar();
#pragma unroll 1
                        for (int t = 0; t < 2; t++)
#pragma unroll 1
                            for (int a = 0; a < 8; a++) {
                                double v[8];
                                tmem_ld8d(tb + t * 128 + 16 * a, v);
                                const int row = row_of(a), rr = rrank[row];
                                bool changed = false;
#pragma unroll
                                for (int q = 0; q < 8; q++) {
                                    const int col = col_of(t, q >> 1, q & 1), cc = crank[col];
                                    if (rr < 0 || cc < 0) continue;
                                    const long long idx = (long long)cc * ncr + rr - base;
                                    if (idx < 0 || idx >= nb) continue;
                                    const double y = cand_y[idx];
                                    if (single || !(fabs(v[q] - y) <= cand_eb[idx])) {
                                        v[q] = y;  // correction (reading R6: the recomputed element)
                                        changed = true;
                                        const unsigned long long p = atomicAdd(&g.rep->count, 1ull);
                                        if ((long long)p < g.rep_cap) {
                                            Correction cr;
                                            cr.tile_m = tm + g.off_i / BM; cr.tile_n = tn + g.off_j / BN;
                                            cr.i = m0 + row + g.off_i; cr.j = n0 + col + g.off_j;
                                            cr.residual = dres[row];
                                            cr.kind = single ? 1 : 2; cr.pad = 0;
                                            g.rep_entries[p] = cr;
                                        }
                                    }
                                }
                                if (__any_sync(0xffffffffu, changed)) tmem_st8d(tb + t * 128 + 16 * a, v);
                            }
                        epi_bar();
                    }
                }
                // ---- pass 2: store the verified tile
#pragma unroll 1
                for (int t = 0; t < 2; t++)
#pragma unroll 2
                    for (int a = 0; a < 8; a++) {
                        double v[8];
                        tmem_ld8d(tb + t * 128 + 16 * a, v);
                        const int row = row_of(a);
#pragma unroll
                        for (int q = 0; q < 8; q++) {
                            const int col = col_of(t, q >> 1, q & 1);
                            if (row < mvalid && col < nvalid) g.C[(m0 + row) + (n0 + col) * g.ldc] = v[q];
                        }
                    }
            }
            // buffer read: hand it back to the MMA warps
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
            epi_bar();  // side data / flags / reductions of this tile consumed by every thread
        }
    } else {
        // ------------------------------------------------------------------ MMA warps
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(WsRegs<FT>::MMA));
        const int wm = warp % 2, wn = warp / 2;
        const FragAddr<KCA> fA(wm * 64, lane);
        const FragAddr<KCB> fB(wn * 32, lane);
        auto row_of = [&](int a) { return frag_mn<KCA>(wm * 64, a, lane >> 2); };
        auto col_of = [&](int b, int e) { return frag_mn<KCB>(wn * 32, b, 2 * (lane & 3) + e); };
        double acc[8][4][2];
        auto zero_acc = [&]() {
#pragma unroll
            for (int a = 0; a < 8; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
        };
        // end of tile x (the it-th of this CTA): planned flips (test harness), then the
        // accumulators go to TMEM buffer it & 1 and the epilogue is signalled
        auto finish_tile = [&](long long x, int it) {
            if (FT && g.plan_ptr) {
                long long tm, tn;
                tile_coords(x, ntm, ntn, tm, tn);
                const long long gtm = tm + g.off_i / BM, gtn = tn + g.off_j / BN;
                if (gtm < g.plan_ntm && gtn < g.plan_ntn) {
                    const long long tix = gtn * g.plan_ntm + gtm;
                    const int lo = g.plan_ptr[tix], hi = g.plan_ptr[tix + 1];
                    for (int f = lo; f < hi; f++) {
                        const long long li = g.plan_i[f] - g.off_i - tm * BM, lj = g.plan_j[f] - g.off_j - tn * BN;
                        const int bit = g.plan_bit[f];
#pragma unroll
                        for (int a = 0; a < 8; a++)
#pragma unroll
                            for (int b = 0; b < 4; b++)
#pragma unroll
                                for (int e = 0; e < 2; e++)
                                    if (row_of(a) == li && col_of(b, e) == lj) acc[a][b][e] = flip_bit(acc[a][b][e], bit);
                    }
                }
            }
            const int buf = it & 1;
            if (it >= 2) mbar_wait(&acc_empty[buf], (unsigned)(((it >> 1) - 1) & 1));
            tc_fence_after();
            const unsigned tb = tbase + ((unsigned)(32 * (warp & 3)) << 16) + (unsigned)(buf * 256 + (warp >> 2) * 128);
#pragma unroll
            for (int a = 0; a < 8; a++) tmem_st8d(tb + 16 * a, &acc[a][0][0]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_full[buf]);
        };
        if (ktiles == 0) {  // alpha == 0 or K == 0: zero accumulators, epilogue only
            int it = 0;
            for (long long x = blockIdx.x; x < ntiles; x += gridDim.x, it++) {
                zero_acc();
                finish_tile(x, it);
            }
        } else {
            // The ring of operand stages runs across tile boundaries: slot st of round `phase`
            // holds the next k-tile.  The loop is unrolled over the slots so every fragment
            // address is one of the 8 FragAddr offsets plus an immediate (as in gemm_kernel).
            long long x = blockIdx.x;
            int it = 0, kt = 0;
            unsigned phase = 0;
            bool done = x >= ntiles;
            zero_acc();
            while (!done) {
#pragma unroll
                for (int st = 0; st < WS_STAGES; st++) {
                    if (!done) {
                        mbar_wait(&full_bar[st], phase);
                        const double *a_s = smem + st * WS_STAGE_EL, *b_s = a_s + TILE_EL;
#pragma unroll
                        for (int kk = 0; kk < BK / 4; kk++) {
                            double af[8], bf[4];
#pragma unroll
                            for (int f = 0; f < 8; f++) af[f] = a_s[fA(f, kk)];
#pragma unroll
                            for (int f = 0; f < 4; f++) bf[f] = b_s[fB(f, kk)];
#pragma unroll
                            for (int a = 0; a < 8; a++)
#pragma unroll
                                for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
                        }
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&empty_bar[st]);
                        if (++kt == ktiles) {
                            finish_tile(x, it);
                            it++;
                            kt = 0;
                            x += gridDim.x;
                            done = x >= ntiles;
                            zero_acc();
                        }
                    }
                }
                phase ^= 1u;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 13) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase) : "memory");
    }
}

}  // namespace ftb
