// ftblas_ws.cuh -- persistent, warp-specialized ABFT DGEMM with the epilogue staged in TMEM.
//
// One CTA per SM walks its share of the 128 x 128 tiles of C (tile x = blockIdx.x + i gridDim.x,
// rasterized by tile_coords).  Three roles run concurrently:
//   producer  (warp 12, one thread; all of warpgroup 3 for the non-TMA fallback): streams the
//             operand tiles of every k-tile of every tile of the CTA through a WS_STAGES-deep
//             TMA / mbarrier ring that runs across tile boundaries, and prefetches each tile's
//             C0 into L2 near the end of its mainloop;
//   MMA       (warps 0..7, 32 x 64 warp tiles: warp w owns rows 32 (w % 4) .. +31, columns
//             64 (w / 4) .. +63): DMMA into registers; at the end of a tile the accumulators get
//             the planned flips (test harness) and go to one of two TMEM buffers (tcgen05.st),
//             handed over with an mbarrier -- the warps start the next tile's mainloop at once;
//   epilogue  (warps 8..11): per tile, read the accumulators back from TMEM (tcgen05.ld), form
//             out = alpha acc + beta C0 with the row / column sums of d = out - beta C0 and the
//             |C0| maxima (readings R3, R4k), verify every row and column against the checksum-
//             GEMM references, locate and correct (lines 540, 521; readings
//             R5-R7) and store the verified tile -- while the MMA warps run the next tile.
// TMEM is the accumulator hand-over buffer the DMMA path (FP64 tensor cores have no tcgen05.mma
// kind) otherwise lacks: 2 buffers x 256 columns x 128 lanes x 32 bit = all 512 columns, TMEM
// lane = tile row.  MMA warp w stores with the 16x256b shape (a thread of fragment row g writes
// lanes g and g + 8, the mma.sync accumulator layout), so fragments a = 2p, 2p + 1 land in lanes
// 32 (w % 4) + 16 p + [0, 16) and a row's 64 doubles of warp column w / 4 fill TMEM columns
// buf * 256 + (w / 4) * 128 + [0, 128).  Epilogue warp ew (= its TMEM sub-partition) therefore
// owns rows 32 ew .. +31, one row per thread, and reads its row 8 columns at a time.
// With the lane = row layout a warp's C0 load / C store of one column covers 32 consecutive
// rows (256 contiguous bytes), so the epilogue moves C with plain coalesced L2-only accesses
// (ld/st.global.cg) and all shared memory goes to a 3-stage operand ring.  No L1-allocating
// loads and no K-long recomputation run beside the DMMA mainloop (corrections are deferred to
// correct_kernel): with ~200 KB of shared memory in use, long streams of L1-allocating loads
// beside the mainloop corrupted accumulators.
#pragma once
#include "ftblas_kernels.cuh"
#ifdef FTB_DBG_CORR
#include <cstdio>
#endif

namespace ftb {

constexpr int WS_THREADS = 512;                 // 8 MMA + 4 epilogue + 4 producer-group warps
// Warp roles: warps 12..15 producer group; the epilogue warpgroup first (warps 0..3) and the MMA
// warps 4..11 by default (-DFTB_WS_EPI_LAST: MMA 0..7, epilogue 8..11).  A warp's TMEM
// sub-partition is warp % 4 either way.
#ifdef FTB_WS_EPI_LAST
#define WS_IS_EPI(w) ((w) >= 8)
#define WS_MMA_IDX(w) (w)
#else
#define WS_IS_EPI(w) ((w) < 4)
#define WS_MMA_IDX(w) ((w) - 4)
#endif
#ifndef FTB_WS_STAGES
#define FTB_WS_STAGES 2
#endif
constexpr int WS_STAGES = FTB_WS_STAGES;
constexpr int WS_STAGE_EL = 2 * TILE_EL;        // A 128 x BK | B 128 x BK
constexpr int WS_QCOLS = 32;                     // C staging: quarter tiles of 32 columns x 128 rows,
constexpr int WS_CBUF_EL = WS_QCOLS * BM;        // double-buffered (TMA load / store)
constexpr int WS_SMEM = (WS_STAGES * WS_STAGE_EL + 2 * WS_CBUF_EL) * 8 + 1024;

// setmaxnreg split of the 64 K registers (one CTA per SM)
template <bool FT>
struct WsRegs {
    static constexpr int MMA = FT ? 192 : 200, EPI = FT ? 104 : 72, PROD = FT ? 24 : 32;
    static_assert(256 * MMA + 128 * EPI + 128 * PROD <= 65536,
                  "setmaxnreg budget exceeds the register file of one CTA per SM");
};

// ------------------------------------------------------------------ phase timing (development)
// -DFTB_WS_PROF: per-CTA globaltimer sums of the phases below (read by ftblas_ws_prof_read);
// compiled out otherwise.
#ifdef FTB_WS_PROF
__device__ unsigned long long ws_prof[1024][16];
__device__ __forceinline__ unsigned long long ws_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define WS_T(v) const unsigned long long v = ws_now()
#define WS_ADD(slot, t0) ws_prof[blockIdx.x][slot] += ws_now() - (t0)
#else
#define WS_T(v)
#define WS_ADD(slot, t0)
#endif
enum { WP_MMA_WAIT_FULL = 0, WP_MMA_WAIT_EMPTYACC, WP_MMA_TMEMST, WP_EPI_WAIT_ACC, WP_EPI_WAIT_C0, WP_EPI_PASS1,
       WP_EPI_VERIFY, WP_EPI_PASS2, WP_EPI_STORE, WP_PROD_WAIT_EMPTY, WP_EPI_TOTAL, WP_MMA_TOTAL };

// ------------------------------------------------------------------ primitives
// mbarrier wait as a C loop (not a branch inside inline asm) so the compiler reconverges the warp
// after it: the tcgen05.ld / st that follow are .sync.aligned (every lane of the warp executes
// them together).
__device__ __forceinline__ void ws_wait(unsigned long long *b, unsigned parity) {
    unsigned ok = 0;
    do {
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
                     : "=r"(ok) : "r"(smem_u32(b)), "r"(parity) : "memory");
    } while (!ok);
}
// A per-lane condition the compiler cannot treat as loop-invariant: loops that contain
// tcgen05.ld / st must not be unswitched on a lane-dependent condition, which would put the
// lanes of a warp into two copies of the loop.
__device__ __forceinline__ bool lane_opaque(bool b) {
    unsigned r;
    asm volatile("mov.b32 %0, %1;\n" : "=r"(r) : "r"((unsigned)b));
    return r != 0;
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

// read-only global data (operands, finalized side data, fault plan) without L1 allocation
__device__ __forceinline__ double ld_ro(const double *p) {
    double v;
    asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ long long ld_ro(const long long *p) {
    long long v;
    asm volatile("ld.global.nc.L1::no_allocate.s64 %0, [%1];\n" : "=l"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ int ld_ro(const int *p) {
    int v;
    asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];\n" : "=r"(v) : "l"(p));
    return v;
}

// Accumulator fragments a = 2p, 2p+1 (8 b x 2 e each) of an MMA thread -> TMEM lanes 16 p + g
// and 16 p + 8 + g of its warp's sub-partition, 16x256b shape: repetition r = 2 b + e carries
// {acc[2p][b][e], acc[2p+1][b][e]} into columns 8 r + 2 t of those two lanes.  8 repetitions per
// instruction; the wait is inside the statement so the registers are free afterwards.
__device__ __forceinline__ void tmem_st_pair8(unsigned taddr, const double *lo_row, const double *hi_row) {
    __syncwarp();  // .sync.aligned: the warp arrives converged
    asm volatile(
        "tcgen05.st.sync.aligned.16x256b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16, "
        "%17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31, %32};\n"
        "tcgen05.wait::st.sync.aligned;\n" ::"r"(taddr),
        "r"(__double2loint(lo_row[0])), "r"(__double2hiint(lo_row[0])), "r"(__double2loint(hi_row[0])), "r"(__double2hiint(hi_row[0])),
        "r"(__double2loint(lo_row[1])), "r"(__double2hiint(lo_row[1])), "r"(__double2loint(hi_row[1])), "r"(__double2hiint(hi_row[1])),
        "r"(__double2loint(lo_row[2])), "r"(__double2hiint(lo_row[2])), "r"(__double2loint(hi_row[2])), "r"(__double2hiint(hi_row[2])),
        "r"(__double2loint(lo_row[3])), "r"(__double2hiint(lo_row[3])), "r"(__double2loint(hi_row[3])), "r"(__double2hiint(hi_row[3])),
        "r"(__double2loint(lo_row[4])), "r"(__double2hiint(lo_row[4])), "r"(__double2loint(hi_row[4])), "r"(__double2hiint(hi_row[4])),
        "r"(__double2loint(lo_row[5])), "r"(__double2hiint(lo_row[5])), "r"(__double2loint(hi_row[5])), "r"(__double2hiint(hi_row[5])),
        "r"(__double2loint(lo_row[6])), "r"(__double2hiint(lo_row[6])), "r"(__double2loint(hi_row[6])), "r"(__double2hiint(hi_row[6])),
        "r"(__double2loint(lo_row[7])), "r"(__double2hiint(lo_row[7])), "r"(__double2loint(hi_row[7])), "r"(__double2hiint(hi_row[7]))
        : "memory");
}
// 8 doubles of this thread's TMEM lane <-> 16 consecutive columns (32x32b shape)
__device__ __forceinline__ void tmem_st8d(unsigned taddr, const double *v) {
    __syncwarp();  // .sync.aligned: the warp arrives converged
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, %16};\n"
        "tcgen05.wait::st.sync.aligned;\n" ::"r"(taddr),
        "r"(__double2loint(v[0])), "r"(__double2hiint(v[0])), "r"(__double2loint(v[1])), "r"(__double2hiint(v[1])),
        "r"(__double2loint(v[2])), "r"(__double2hiint(v[2])), "r"(__double2loint(v[3])), "r"(__double2hiint(v[3])),
        "r"(__double2loint(v[4])), "r"(__double2hiint(v[4])), "r"(__double2loint(v[5])), "r"(__double2hiint(v[5])),
        "r"(__double2loint(v[6])), "r"(__double2hiint(v[6])), "r"(__double2loint(v[7])), "r"(__double2hiint(v[7]))
        : "memory");
}
__device__ __forceinline__ void tmem_ld8d(unsigned taddr, double *v) {
    __syncwarp();  // .sync.aligned: the warp arrives converged
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

// C0 / C of the epilogue: TMA of quarter tiles (box {128 rows, 32 columns}, dense
// [column][row] in shared memory); fallback (C not 16-byte aligned or odd ldc): L2-only loads
// and stores (no L1 allocation, see the file comment).
__device__ __forceinline__ double ld_c(const double *p) {
    double v;
    asm volatile("ld.global.cg.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_c(double *p, double v) {
    asm volatile("st.global.cg.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ void tma_load_c(double *dst, const CUtensorMap *map, unsigned long long *bar, int row0,
                                           int col0) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::
            "r"(smem_u32(dst)), "l"(map), "r"(smem_u32(bar)), "r"(row0), "r"(col0)
        : "memory");
}
__device__ __forceinline__ void tma_store_c(const CUtensorMap *map, const double *src, int row0, int col0) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];\n" ::"l"(map),
                 "r"(smem_u32(src)), "r"(row0), "r"(col0)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
}
__device__ __forceinline__ void tma_store_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() { asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory"); }

// Non-TMA operand staging (pointer not 16-byte aligned or odd ld): the producer group copies
// the tile element by element through registers, read-only loads that bypass L1 (see above),
// zero-fill outside [0, MNd) x [0, Kd); the caller arrives on the stage barrier afterwards.
template <bool KC, int ROWS, int NTP>
__device__ __forceinline__ void produce_tile_ro(double *s, const double *X, long long ld, long long mn0, long long k0,
                                                long long MNd, long long Kd, int pt) {
#pragma unroll 4
    for (int c = pt; c < ROWS * BK; c += NTP) {
        int mn, k;
        if (KC) { mn = c / BK; k = c % BK; }
        else    { k = c / ROWS; mn = c % ROWS; }
        const long long gmn = mn0 + mn, gk = k0 + k;
        s[Tile<KC, ROWS>::idx(mn, k)] = (gmn < MNd && gk < Kd) ? ld_ro(gaddr<KC>(X, ld, gmn, gk)) : 0.0;
    }
}

template <int V>
struct IntC {
    static constexpr int value = V;
};

// verification references of one tile (FT): finalized norms and checksum-GEMM slices
struct WsSide {
    double nrm_row[BM], nrm_col[BN], pre_r[BM], pre_s[BN], nrm_max[2];
};

template <bool KCA, bool KCB, bool TMA, bool FT>
__global__ void __launch_bounds__(WS_THREADS, 1)
    gemm_ws_kernel(const __grid_constant__ GemmArgs g, const __grid_constant__ CUtensorMap tmA,
                   const __grid_constant__ CUtensorMap tmB, const __grid_constant__ CUtensorMap tmC) {
    extern __shared__ __align__(1024) double smem_raw[];
    __shared__ __align__(8) unsigned long long full_bar[WS_STAGES], empty_bar[WS_STAGES], acc_full[2], acc_empty[2],
        c0_full[2];
    __shared__ unsigned tmem_base_sh;
    __shared__ WsSide side;
    __shared__ double red_c[4][BN], dres[BM];  // column partials per epilogue warp (32 rows each)
    __shared__ unsigned redm_c[4][BN];
    __shared__ int flags[2 + BM + BN];
    __shared__ int rflag[BM], cflag[BN];
    double *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) / 8u;
    double *cbuf = smem + WS_STAGES * WS_STAGE_EL;  // 2 x [32 columns][128 rows]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long ntm = (g.M + BM - 1) / BM, ntn = (g.N + BN - 1) / BN, ntiles = ntm * ntn;
    const int ktiles = (g.alpha == 0.0) ? 0 : (int)((g.K + BK - 1) / BK);
    constexpr int PT = 128;  // producer-group threads

    if (tid == 0) {
        for (int s = 0; s < WS_STAGES; s++) {
            mbar_init(&full_bar[s], TMA ? 1 : PT);
            mbar_init(&empty_bar[s], 8);     // one arrival per MMA warp
        }
        for (int b = 0; b < 2; b++) {
            mbar_init(&acc_full[b], 8);      // MMA warps: accumulators in TMEM
            mbar_init(&acc_empty[b], 4);     // epilogue warps: buffer read
            mbar_init(&c0_full[b], 1);       // C0 quarter tile in cbuf[b] (TMA, expect_tx)
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
            constexpr unsigned TX = 2u * TILE_EL * 8u;
            unsigned kg = 0;
            for (long long x = blockIdx.x; x < ntiles; x += gridDim.x) {
                long long tm, tn;
                tile_coords(x, ntm, ntn, tm, tn);
                const long long m0 = tm * BM, n0 = tn * BN;
                const int pf_kt = max(0, ktiles - WS_STAGES - 2);
                for (int kt = 0; kt < ktiles; kt++, kg++) {
                    const int st = (int)(kg % WS_STAGES);
                    if (kg >= WS_STAGES) {
                        WS_T(t0);
                        ws_wait(&empty_bar[st], ((kg / WS_STAGES) - 1) & 1);
                        if (pt == 0) WS_ADD(WP_PROD_WAIT_EMPTY, t0);
                    }
                    double *sa = smem + st * WS_STAGE_EL;
                    const long long k0 = (long long)kt * BK;
                    if (TMA) {
                        mbar_arrive_expect_tx(&full_bar[st], TX);
                        produce_tile<KCA, true, 128, PT>(sa, &tmA, &full_bar[st], g.A, g.lda, m0, k0, g.M, g.K, 0);
                        produce_tile<KCB, true, 128, PT>(sa + TILE_EL, &tmB, &full_bar[st], g.B, g.ldb, n0, k0, g.N, g.K, 0);
                    } else {
                        produce_tile_ro<KCA, 128, PT>(sa, g.A, g.lda, m0, k0, g.M, g.K, pt);
                        produce_tile_ro<KCB, 128, PT>(sa + TILE_EL, g.B, g.ldb, n0, k0, g.N, g.K, pt);
                        mbar_arrive(&full_bar[st]);  // release: this thread's smem writes
                    }
                    if (pt == 0 && kt == pf_kt && g.beta != 0.0 && g.vecC) {
                        // C0 of this tile -> L2 shortly before its epilogue loads it
                        const unsigned bytes = (unsigned)(min((long long)BM, g.M - m0) * 8) & ~15u;
                        const long long nv = min((long long)BN, g.N - n0);
                        if (bytes)
                            for (int c = 0; c < nv; c++) bulk_prefetch_l2(g.C + m0 + (n0 + c) * g.ldc, bytes);
                    }
                }
            }
        }
    } else if (WS_IS_EPI(warp)) {
        // ------------------------------------------------------------------ epilogue
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(WsRegs<FT>::EPI));
        const int ew = warp & 3, et = 32 * ew + lane;  // epilogue warp (= TMEM sub-partition), thread
        auto epi_bar = [&]() {  // bar.sync is .aligned: reconverge the warp first
            __syncwarp();
            asm volatile("bar.sync 2, 128;\n" ::: "memory");
        };
        // beta classes decided once on the integer pipe (FP64 instructions beside the DMMA stream
        // wait for the tensor pipe: every one in the per-element code costs)
        const long long bbits = __double_as_longlong(g.beta);
        const bool beta0 = (bbits << 1) == 0, beta1 = bbits == 0x3ff0000000000000ll;
        const int bmode = beta0 ? 0 : (beta1 ? 1 : 2);
        const double aa = fabs(g.alpha), ab = fabs(g.beta);
        // this thread's row of every tile (TMEM lane 32 ew + lane) and the columns of the 8
        // doubles of TMEM chunk j of warp column wn (q = 4 e + t)
        const int row = frag_mn<KCA>(32 * ew, lane >> 3, lane & 7);
        auto col_of = [&](int wn, int j, int q) { return frag_mn<KCB>(64 * wn, j, 2 * (q & 3) + (q >> 2)); };
        // C staging: quarter q of a tile = columns 32 q .. +31 = TMEM chunks (h = q / 2, j = 4 (q % 2)
        // .. +3) of every row (both column layouts), in cbuf[slot] ([32 columns][128 rows]).  The
        // loads / stores are TMA (thread 0) when C has a tensor map, else L2-only copies.
        const bool tma_c = g.vecC != 0;
        const bool need_c0 = !beta0;
        unsigned c0_phase[2] = {0u, 0u};
        auto qbuf = [&](int slot) { return cbuf + slot * WS_CBUF_EL; };
        auto load_c0 = [&](long long m0, long long n0, int q, int slot) {  // issue (TMA) / copy
            if (tma_c) {
                if (et == 0) {
                    mbar_arrive_expect_tx(&c0_full[slot], (unsigned)(WS_CBUF_EL * 8));
                    tma_load_c(qbuf(slot), &tmC, &c0_full[slot], (int)m0, (int)(n0 + WS_QCOLS * q));
                }
            } else {
                const long long gi = m0 + et;
                for (int c = 0; c < WS_QCOLS; c++) {
                    const long long gj = n0 + WS_QCOLS * q + c;
                    qbuf(slot)[c * BM + et] = (gi < g.M && gj < g.N) ? ld_c(g.C + gi + gj * g.ldc) : 0.0;
                }
            }
        };
        auto wait_c0 = [&](int slot) {
            if (tma_c) {
                ws_wait(&c0_full[slot], c0_phase[slot]);
                c0_phase[slot] ^= 1u;
            } else {
                epi_bar();
            }
        };
        // cbuf[slot] -> quarter q of C; the slot can be refilled once this returns (thread 0 waits
        // for the TMA to have read it; the barrier publishes that to the other threads)
        auto store_q = [&](long long m0, long long n0, int q, int slot, long long mvalid, long long nvalid) {
            if (tma_c) {
                fence_proxy_async_smem();  // generic-proxy writes of cbuf -> visible to the TMA
                epi_bar();
                if (et == 0) {
                    tma_store_c(&tmC, qbuf(slot), (int)m0, (int)(n0 + WS_QCOLS * q));
                    tma_store_wait_read();
                }
                epi_bar();
            } else {
                epi_bar();
                if (et < mvalid)
                    for (int c = 0; c < WS_QCOLS && WS_QCOLS * q + c < nvalid; c++)
                        st_c(g.C + (m0 + et) + (n0 + WS_QCOLS * q + c) * g.ldc, qbuf(slot)[c * BM + et]);
                epi_bar();
            }
        };
        int it = 0;
        if (blockIdx.x < ntiles && need_c0) {  // C0 quarters 0, 1 of the first tile
            long long tm, tn;
            tile_coords(blockIdx.x, ntm, ntn, tm, tn);
            load_c0(tm * BM, tn * BN, 0, 0);
            load_c0(tm * BM, tn * BN, 1, 1);
        }
        for (long long x = blockIdx.x; x < ntiles; x += gridDim.x, it++) {
            long long tm, tn;
            tile_coords(x, ntm, ntn, tm, tn);
            const long long m0 = tm * BM, n0 = tn * BN;
            const long long mvalid = min((long long)BM, g.M - m0), nvalid = min((long long)BN, g.N - n0);
            const bool rowok = row < mvalid;
            const bool has_next = x + gridDim.x < ntiles;
            long long m0n = 0, n0n = 0;
            if (has_next) {
                long long tm2, tn2;
                tile_coords(x + gridDim.x, ntm, ntn, tm2, tn2);
                m0n = tm2 * BM; n0n = tn2 * BN;
            }
            if (FT) {  // side data of this tile (loads overlap the wait for the accumulators)
                const long long gi = m0 + et, gj = n0 + et;
                side.nrm_row[et] = et < mvalid ? ld_ro(g.fin_nrmA + gi) : 0.0;
                side.pre_r[et] = et < mvalid ? ld_ro(g.fin_R + tn * g.M + gi) : 0.0;
                side.nrm_col[et] = et < nvalid ? ld_ro(g.fin_nrmB + gj) : 0.0;
                side.pre_s[et] = et < nvalid ? ld_ro(g.fin_S + tm * g.N + gj) : 0.0;
                if (et == 0) {
                    side.nrm_max[0] = ld_ro(g.fin_maxA + tm);
                    side.nrm_max[1] = ld_ro(g.fin_maxB + tn);
                    flags[0] = 0;
                    flags[1] = 0;
                }
            }
            const int buf = it & 1;
            WS_T(tw0);
            ws_wait(&acc_full[buf], (unsigned)((it >> 1) & 1));
            if (et == 0) WS_ADD(WP_EPI_WAIT_ACC, tw0);
            WS_T(tp1);
            tc_fence_after();
            const unsigned tb = tbase + ((unsigned)(32 * ew) << 16) + (unsigned)(buf * 256);
            // ---- pass 1, quarter by quarter, chunk = 8 doubles of this thread's row: out, the row
            // sum (8 independent partials, one per chunk position q, combined in fixed order after
            // the tile, so the FP64 adds do not form one 128-long dependency chain) and the column
            // partials.  FT: out goes back into TMEM; non-FT: into cbuf, stored per quarter.
            double rsq[8];
#pragma unroll
            for (int q = 0; q < 8; q++) rsq[q] = 0.0;
            unsigned rm = 0u;
            auto pass1 = [&](auto mode_c) {
                constexpr int MODE = decltype(mode_c)::value;  // 0: beta = 0, 1: beta = 1, 2: other
#pragma unroll 1
                for (int qq = 0; qq < 4; qq++) {
                    const int slot = qq & 1;
                    double *cb = qbuf(slot);
                    if (MODE != 0) {
                        WS_T(tc0);
                        wait_c0(slot);
                        if (et == 0) WS_ADD(WP_EPI_WAIT_C0, tc0);
                    }
                    // FT, column pass view of the quarter: this thread = column 32 qq + lane over its
                    // warp's 32 rows, visited in a lane-skewed order (row 32 ew + (i + lane) % 32) so
                    // the half-warps' 64-bit shared loads hit distinct banks
                    const int r0 = 32 * ew, cq = lane;
                    if (FT && MODE != 0) {  // column maxima of |C0| (high words, integer pipe)
                        unsigned m = 0u;
#pragma unroll 8
                        for (int i = 0; i < 32; i++)
                            m = max(m, (unsigned)__double2hiint(cb[cq * BM + r0 + ((i + lane) & 31)]) & 0x7fffffffu);
                        redm_c[ew][WS_QCOLS * qq + cq] = m;
                        __syncwarp();  // the warp's C0 reads before its rows are overwritten with d
                    }
                    // two chunks at a time: the FP64 instructions wait for the DMMA stream of the MMA
                    // warps, so independent ones are issued together (16 per level)
#pragma unroll 1
                    for (int jj = 0; jj < 4; jj += 2) {
                        const int h = qq >> 1, j = 4 * (qq & 1) + jj;
                        double v[2][8];
                        tmem_ld8d(tb + h * 128 + 16 * j, v[0]);
                        tmem_ld8d(tb + h * 128 + 16 * (j + 1), v[1]);
                        const bool rk = lane_opaque(rowok);
#pragma unroll
                        for (int u = 0; u < 2; u++)
#pragma unroll
                            for (int q = 0; q < 8; q++) {
                                const int col = col_of(h, j + u, q);
                                const int cl = col - WS_QCOLS * qq;  // column in the quarter
                                double o, d;
                                if (MODE == 0) {
                                    o = g.alpha * v[u][q];
                                    d = o;
                                } else {
                                    const double c0 = cb[cl * BM + row];  // 0 outside M x N (zero fill)
                                    const double tt = MODE == 1 ? c0 : g.beta * c0;
                                    o = fma(g.alpha, v[u][q], tt);
                                    d = o - tt;
                                    if (FT) rm = max(rm, (unsigned)__double2hiint(c0) & 0x7fffffffu);
                                }
                                if (FT) {
                                    d = (rk && col < nvalid) ? d : 0.0;
                                    rsq[q] += d;
                                    cb[cl * BM + row] = d;  // for the column pass (in place of C0)
                                    v[u][q] = o;
                                } else {
                                    cb[cl * BM + row] = o;
                                }
                            }
                        if (FT) {
                            tmem_st8d(tb + h * 128 + 16 * j, v[0]);
                            tmem_st8d(tb + h * 128 + 16 * (j + 1), v[1]);
                        }
                    }
                    if (FT) {
                        // column sums of d over the warp's 32 rows: 8 independent partial sums
                        __syncwarp();
                        double sp[8];
                        const double *cc = cb + cq * BM + r0;
#pragma unroll
                        for (int u = 0; u < 8; u++) sp[u] = cc[(u + lane) & 31];
#pragma unroll
                        for (int i = 8; i < 32; i += 8)
#pragma unroll
                            for (int u = 0; u < 8; u++) sp[u] += cc[(i + u + lane) & 31];
                        red_c[ew][WS_QCOLS * qq + cq] = ((sp[0] + sp[1]) + (sp[2] + sp[3])) + ((sp[4] + sp[5]) + (sp[6] + sp[7]));
                        if (MODE == 0) redm_c[ew][WS_QCOLS * qq + cq] = 0u;
                        __syncwarp();  // column reads done before the slot is rewritten
                    }
                    if (!FT) {
                        store_q(m0, n0, qq, slot, mvalid, nvalid);  // the slot is free afterwards
                    } else if (MODE != 0) {
                        epi_bar();  // every thread done reading this C0 quarter
                    }
                    // refill the slot: quarter qq + 2 of this tile, or (non-FT) quarter qq - 2 of the
                    // next one (FT: the next tile's C0 waits until pass 2 has used the slots)
                    if (MODE != 0) {
                        if (qq < 2) load_c0(m0, n0, qq + 2, slot);
                        else if (!FT && has_next) load_c0(m0n, n0n, qq - 2, slot);
                    }
                }
            };
            if (bmode == 0) pass1(IntC<0>{});
            else if (bmode == 1) pass1(IntC<1>{});
            else pass1(IntC<2>{});
            if (et == 0) WS_ADD(WP_EPI_PASS1, tp1);
            WS_T(tv0);
            if (FT) {
                epi_bar();
                // ---- verification (readings R3, R4, R4k): each thread checks
                // its own row (the whole row sum is in-thread) and column et
                auto c0_bound = [&](unsigned hw, long long n) {
                    if (hw >= 0x7ff00000u) return __longlong_as_double(0x7ff0000000000000ll);
                    return (double)n * __hiloint2double((int)(hw + 1u), 0);
                };
                if (rowok) {
                    const double rs = ((rsq[0] + rsq[1]) + (rsq[2] + rsq[3])) + ((rsq[4] + rsq[5]) + (rsq[6] + rsq[7]));
                    const double c0a = beta0 ? 0.0 : c0_bound(rm, nvalid);
                    const double tau = 4.0 * U_ROUND * (double)(g.K + nvalid + 3) *
                                       (aa * side.nrm_row[row] * side.nrm_max[1] + ab * c0a);
                    const double d = rs - g.alpha * side.pre_r[row];
                    dres[row] = d;
                    if (!(fabs(d) <= tau)) flags[2 + atomicAdd(&flags[0], 1)] = row;
                }
                if (et < nvalid) {
                    const double sum = (red_c[0][et] + red_c[1][et]) + (red_c[2][et] + red_c[3][et]);
                    const unsigned mx = max(max(redm_c[0][et], redm_c[1][et]), max(redm_c[2][et], redm_c[3][et]));
                    const double c0a = beta0 ? 0.0 : c0_bound(mx, mvalid);
                    const double tau = 4.0 * U_ROUND * (double)(g.K + mvalid + 3) *
                                       (aa * side.nrm_max[0] * side.nrm_col[et] + ab * c0a);
                    const double d = sum - g.alpha * side.pre_s[et];
                    if (!(fabs(d) <= tau)) flags[2 + BM + atomicAdd(&flags[1], 1)] = et;
                }
                epi_bar();
                const int nr = flags[0], nc = flags[1];
                if (nr != 0 || nc != 0) {
                    // ---- locate (rare): candidates = (flagged rows, or all rows) x (flagged
                    // columns, or all columns) (readings R5, R7).  Each row owner lists its
                    // candidates with their stored value and C0 (C is not yet overwritten); the
                    // K-long recomputation and the correction (reading R6) run after the GEMM in
                    // correct_kernel, so no long phase runs beside the DMMA mainloop.
                    if (et == 0) {
                        atomicAdd(&g.rep->tiles_flagged, 1ull);
                        atomicAdd(&g.rep->rows_flagged, (unsigned long long)nr);
                        atomicAdd(&g.rep->cols_flagged, (unsigned long long)nc);
                    }
                    rflag[et] = (nr == 0 && et < mvalid) ? 1 : 0;
                    cflag[et] = (nc == 0 && et < nvalid) ? 1 : 0;
                    epi_bar();
                    if (et < nr) rflag[flags[2 + et]] = 1;
                    if (et < nc) cflag[flags[2 + BM + et]] = 1;
                    epi_bar();
                    const bool single = nr == 1 && nc == 1;  // Huang-Abraham location (line 540)
                    const bool mine = rflag[row] != 0;
                    if (__any_sync(0xffffffffu, mine)) {
#pragma unroll 1
                        for (int h = 0; h < 2; h++)
#pragma unroll 1
                            for (int j = 0; j < 8; j++) {
                                double v[8];
                                tmem_ld8d(tb + h * 128 + 16 * j, v);
                                const bool mn = lane_opaque(mine);
#pragma unroll
                                for (int q = 0; q < 8; q++) {
                                    const int col = col_of(h, j, q);
                                    if (!mn || !cflag[col]) continue;
                                    const unsigned long long p = atomicAdd(&g.pend->count, 1ull);
                                    if ((long long)p < g.pend_cap) {
                                        Pending pe;
                                        pe.i = m0 + row; pe.j = n0 + col;
                                        pe.cur = v[q];
                                        pe.c0 = beta0 ? 0.0 : ld_c(g.C + (m0 + row) + (n0 + col) * g.ldc);
                                        pe.residual = dres[row];
                                        pe.single = single ? 1 : 0; pe.pad = 0;
                                        g.pend_entries[p] = pe;
                                    }
                                }
                            }
                    }
                }
                if (et == 0) WS_ADD(WP_EPI_VERIFY, tv0);
                WS_T(tq0);
                // ---- pass 2: the verified tile -> cbuf -> C, quarter by quarter (double-buffered);
                // then C0 quarters 0, 1 of the next tile
#pragma unroll 1
                for (int qq = 0; qq < 4; qq++) {
                    const int slot = qq & 1;
                    double *cb = qbuf(slot);
#pragma unroll 1
                    for (int jj = 0; jj < 4; jj++) {
                        const int h = qq >> 1, j = 4 * (qq & 1) + jj;
                        double v[8];
                        tmem_ld8d(tb + h * 128 + 16 * j, v);
#pragma unroll
                        for (int q = 0; q < 8; q++) cb[(col_of(h, j, q) - WS_QCOLS * qq) * BM + row] = v[q];
                    }
                    WS_T(ts1);
                    store_q(m0, n0, qq, slot, mvalid, nvalid);
                    if (et == 0) WS_ADD(WP_EPI_STORE, ts1);
                }
                if (need_c0 && has_next) {
                    load_c0(m0n, n0n, 0, 0);
                    load_c0(m0n, n0n, 1, 1);
                }
                if (et == 0) WS_ADD(WP_EPI_PASS2, tq0);
            }
            // accumulator buffer read: hand it back to the MMA warps
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_empty[buf]);
            epi_bar();  // side data / flags / reductions of this tile consumed by every thread
            if (et == 0) WS_ADD(WP_EPI_TOTAL, tw0);
        }
        if (tma_c && et == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");  // stores done
    } else {
        // ------------------------------------------------------------------ MMA warps
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(WsRegs<FT>::MMA));
        const int mw = WS_MMA_IDX(warp);           // MMA warp index 0..7
        const int wm = mw & 3, wn = mw >> 2;       // rows 32 wm, columns 64 wn of the tile
        const FragAddr<KCA> fA(wm * 32, lane);
        const FragAddr<KCB> fB(wn * 64, lane);
        auto row_of = [&](int a) { return frag_mn<KCA>(wm * 32, a, lane >> 2); };
        auto col_of = [&](int b, int e) { return frag_mn<KCB>(wn * 64, b, 2 * (lane & 3) + e); };
        double acc[4][8][2];
        auto zero_acc = [&]() {
#pragma unroll
            for (int a = 0; a < 4; a++)
#pragma unroll
                for (int b = 0; b < 8; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
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
                    const int lo = ld_ro(g.plan_ptr + tix), hi = ld_ro(g.plan_ptr + tix + 1);
                    for (int f = lo; f < hi; f++) {
                        const long long li = ld_ro(g.plan_i + f) - g.off_i - tm * BM;
                        const long long lj = ld_ro(g.plan_j + f) - g.off_j - tn * BN;
                        const int bit = ld_ro(g.plan_bit + f);
#pragma unroll
                        for (int a = 0; a < 4; a++)
#pragma unroll
                            for (int b = 0; b < 8; b++)
#pragma unroll
                                for (int e = 0; e < 2; e++)
                                    if (row_of(a) == li && col_of(b, e) == lj) acc[a][b][e] = flip_bit(acc[a][b][e], bit);
                    }
                }
            }
            const int buf = it & 1;
            WS_T(te0);
            if (it >= 2) ws_wait(&acc_empty[buf], (unsigned)(((it >> 1) - 1) & 1));
            if (mw == 0 && lane == 0) WS_ADD(WP_MMA_WAIT_EMPTYACC, te0);
            WS_T(ts0);
            tc_fence_after();
            const unsigned tb = tbase + ((unsigned)(32 * wm) << 16) + (unsigned)(buf * 256 + wn * 128);
#pragma unroll
            for (int p = 0; p < 2; p++) {
                // repetitions r = 2 b + e: 0..7 (b < 4) and 8..15 (b >= 4)
                double lo0[8], hi0[8], lo1[8], hi1[8];
#pragma unroll
                for (int r = 0; r < 8; r++) {
                    lo0[r] = acc[2 * p][r >> 1][r & 1];
                    hi0[r] = acc[2 * p + 1][r >> 1][r & 1];
                    lo1[r] = acc[2 * p][4 + (r >> 1)][r & 1];
                    hi1[r] = acc[2 * p + 1][4 + (r >> 1)][r & 1];
                }
                tmem_st_pair8(tb + ((unsigned)(16 * p) << 16), lo0, hi0);
                tmem_st_pair8(tb + ((unsigned)(16 * p) << 16) + 64, lo1, hi1);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&acc_full[buf]);
            if (mw == 0 && lane == 0) WS_ADD(WP_MMA_TMEMST, ts0);
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
            WS_T(tm0);
            long long x = blockIdx.x;
            int it = 0, kt = 0;
            unsigned phase = 0;
            bool done = x >= ntiles;
            zero_acc();
            while (!done) {
#pragma unroll
                for (int st = 0; st < WS_STAGES; st++) {
                    if (!done) {
                        WS_T(tf0);
                        ws_wait(&full_bar[st], phase);
                        if (mw == 0 && lane == 0) WS_ADD(WP_MMA_WAIT_FULL, tf0);
                        const double *a_s = smem + st * WS_STAGE_EL, *b_s = a_s + TILE_EL;
#pragma unroll
                        for (int kk = 0; kk < BK / 4; kk++) {
                            double af[4], bf[8];
#pragma unroll
                            for (int f = 0; f < 4; f++) af[f] = a_s[fA(f, kk)];
#pragma unroll
                            for (int f = 0; f < 8; f++) bf[f] = b_s[fB(f, kk)];
#pragma unroll
                            for (int a = 0; a < 4; a++)
#pragma unroll
                                for (int b = 0; b < 8; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
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
            if (mw == 0 && lane == 0) WS_ADD(WP_MMA_TOTAL, tm0);
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 13) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tbase) : "memory");
    }
}

// ------------------------------------------------------------------ deferred correction
// After gemm_ws_kernel<FT>: every located candidate (i, j) is recomputed from its definition,
// y = alpha sum_k op(A)(i,k) op(B)(k,j) + beta C0_ij (reading R6; one CTA per candidate, the K
// range split over its 8 warps, fixed-order combination), and replaced iff it is the single
// located error or differs from y beyond its rounding bound (reading R7); the report entry is
// written for every replacement.  Runs on the GEMM's stream, so C is final when it starts.
constexpr int CORR_THREADS = 256;
template <bool KCA, bool KCB>
__global__ void __launch_bounds__(CORR_THREADS) correct_kernel(const __grid_constant__ GemmArgs g) {
    __shared__ double ps[CORR_THREADS / 32], psa[CORR_THREADS / 32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long n = min((long long)g.pend->count, g.pend_cap);
    const double aa = fabs(g.alpha), ab = fabs(g.beta);
    for (long long q = blockIdx.x; q < n; q += gridDim.x) {
        const Pending pe = g.pend_entries[q];
        double s = 0.0, sa = 0.0;
        for (long long k = tid; k < g.K; k += CORR_THREADS) {
            const double a = ld_ro(gaddr<KCA>(g.A, g.lda, pe.i, k));
            const double b = ld_ro(gaddr<KCB>(g.B, g.ldb, pe.j, k));
            s = fma(a, b, s);
            sa = fma(fabs(a), fabs(b), sa);
        }
#pragma unroll
        for (int off = 16; off; off >>= 1) {
            s += __shfl_xor_sync(0xffffffffu, s, off);
            sa += __shfl_xor_sync(0xffffffffu, sa, off);
        }
        if (lane == 0) { ps[warp] = s; psa[warp] = sa; }
        __syncthreads();
        if (tid == 0) {
            s = 0.0; sa = 0.0;
            for (int w = 0; w < CORR_THREADS / 32; w++) { s += ps[w]; sa += psa[w]; }
            const double y = g.beta == 0.0 ? g.alpha * s : fma(g.alpha, s, g.beta * pe.c0);
            const double eb = 4.0 * U_ROUND * (double)(g.K + 3) * (aa * sa + ab * fabs(pe.c0));
#ifdef FTB_DBG_CORR
            printf("corr q %lld i %lld j %lld cur %g c0 %g y %g single %d ldc %lld C %p K %lld\n", q, pe.i, pe.j, pe.cur, pe.c0, y,
                   pe.single, g.ldc, (void *)g.C, g.K);
#endif
            if (pe.single || !(fabs(pe.cur - y) <= eb)) {
                g.C[pe.i + pe.j * g.ldc] = y;  // correction (reading R6: the recomputed element)
                const unsigned long long p = atomicAdd(&g.rep->count, 1ull);
                if ((long long)p < g.rep_cap) {
                    Correction cr;
                    cr.tile_m = (pe.i + g.off_i) / BM; cr.tile_n = (pe.j + g.off_j) / BN;
                    cr.i = pe.i + g.off_i; cr.j = pe.j + g.off_j;
                    cr.residual = pe.residual;
                    cr.kind = pe.single ? 1 : 2; cr.pad = 0;
                    g.rep_entries[p] = cr;
                }
            }
        }
        __syncthreads();
    }
}

}  // namespace ftb
