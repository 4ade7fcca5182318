// ftblas_kernels.cuh -- sm_100a kernels of the ABFT DGEMM hot path.
//
//   encode_kernel : Huang-Abraham checksum encoding of op(A) and op(B) per
//                   verification tile (section II.A:
//                   A^c = [A; e^T A], B^r = [B, B e]) plus the norms used by the
//                   round-off threshold (reading R4).
//   gemm_kernel   : C := alpha op(A) op(B) + beta C on FP64 tensor cores
//                   (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4), cp.async multi-stage
//                   smem pipeline; with FT=true it also accumulates the checksum
//                   column C e = A (B e) and row e^T C = (e^T A) B of the tile in the
//                   same mainloop (line 516, "C^f = A^c B^r"), and its epilogue
//                   verifies, locates and corrects (lines 517, 540, 521) before the
//                   store.  FT=false is the non-FT baseline (same tiles/mainloop).
//
// Layout of one CTA: 256 threads = 8 warps in a 2 (M) x 4 (N) grid, warp tile
// 64 x 32 = 8 x 4 DMMA fragments of 8x8, CTA tile 128 x 128, BK = 16,
// STAGES-deep cp.async ring.  See DESIGN.md section 4 for the roofline.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace ftb {

constexpr int BM = 128, BN = 128, BK = 32, STAGES = 3, NTHREADS = 256;
constexpr int WM = 64, WN = 32, FM = WM / 8, FN = WN / 8;
// Padded smem strides chosen so that a DMMA fragment load (a half-warp reads 4 mn x 4 k
// doubles) touches 16 distinct 8-byte bank pairs: row strides == 32 (mod 128) bytes.
constexpr int LD_MN = 128 + 4;  // doubles per k-row when the mn index is contiguous (1056 B)
constexpr int LD_K = BK + 4;    // doubles per mn-row when k is contiguous (288 B)
constexpr double U_ROUND = 1.0 / 9007199254740992.0;  // 2^-53

// smem doubles of one operand tile (one stage)
template <bool KC>
struct Tile {
    static constexpr int ELEMS = KC ? 128 * LD_K : BK * LD_MN;
    __device__ __forceinline__ static int idx(int mn, int k) { return KC ? mn * LD_K + k : k * LD_MN + mn; }
};

struct Correction {  // == ftblas_correction (48 bytes)
    long long tile_m, tile_n, i, j;
    double residual;
    int kind, pad;
};
struct ReportHdr {  // device-side counters
    unsigned long long count, tiles_flagged, rows_flagged, cols_flagged;
};

struct GemmArgs {
    const double *A, *B;
    double *C;
    long long lda, ldb, ldc;
    long long M, N, K;
    double alpha, beta;
    // FT workspace (encode outputs)
    const double *VA;      // ntm x Kp: e^T op(A) per row tile
    const double *WB;      // ntn x Kp: op(B) e per column tile
    const double *lineA;   // kch x M : partial sum_k |op(A)(i,k)|
    const double *lineB;   // kch x N : partial sum_k |op(B)(k,j)|
    const double *tmaxA;   // kch x ntm: partial max_k sum_i |op(A)(i,k)|
    const double *tmaxB;   // kch x ntn
    int kch;
    long long Kp;
    // fault plan (CSR by tile, tile index = tn * ntm + tm)
    const int *plan_ptr;   // ntm*ntn + 1 or nullptr
    const long long *plan_i, *plan_j;
    const int *plan_bit;
    // report
    ReportHdr *rep;
    Correction *rep_entries;
    long long rep_cap;
};

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ unsigned smem_u32(const void *p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void *dst, const void *src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_async8(void *dst, const void *src, int bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// mbarrier primitives (producer/consumer pipeline between the load warp and the MMA warps)
__device__ __forceinline__ void mbar_init(unsigned long long *b, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.shared::cta.b64 st, [%0];\n\t}\n" ::"r"(smem_u32(b))
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long *b, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tLAB_WAIT:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra LAB_WAIT;\n\t}\n" ::"r"(smem_u32(b)), "r"(parity)
        : "memory");
}
// arrive on b when all prior cp.async of this thread have landed (count pre-set at init)
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long *b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void bar_mma() {  // named barrier over the NTHREADS MMA threads only
    asm volatile("bar.sync 1, %0;\n" ::"n"(NTHREADS) : "memory");
}

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ double flip_bit(double x, int bit) {
    return __longlong_as_double(__double_as_longlong(x) ^ (1ll << bit));
}

// Element (mn, k) of an operand tile source.  KC: k contiguous in global memory.
// op(A)(m,k): 'N' -> A[m + k lda] (KC=false), 'T' -> A[k + m lda] (KC=true)
// op(B)(k,n): 'N' -> B[k + n ldb] (KC=true),  'T' -> B[n + k ldb] (KC=false)
template <bool KC>
__device__ __forceinline__ const double *gaddr(const double *X, long long ld, long long mn, long long k) {
    return KC ? X + k + mn * ld : X + mn + k * ld;
}

// Stage one 128 x BK operand tile into smem with cp.async (zero-fill outside [0,MNd) x [0,Kd)).
template <bool KC, bool VEC, int NT = NTHREADS>
__device__ __forceinline__ void load_tile(double *s, const double *X, long long ld, long long mn0,
                                          long long k0, long long MNd, long long Kd, int tid) {
    if (VEC) {  // 16-byte chunks along the contiguous dimension (needs 16B-aligned X, even ld)
#pragma unroll
        for (int q = 0; q < (128 * BK / 2) / NT; q++) {
            int c = tid + q * NT;
            int mn, k;
            if (KC) { mn = c / (BK / 2); k = (c % (BK / 2)) * 2; }
            else    { k = c >> 6;  mn = (c & 63) * 2; }
            long long gmn = mn0 + mn, gk = k0 + k;
            int nvalid;
            if (KC) nvalid = (gmn < MNd) ? (int)min(2ll, max(0ll, Kd - gk)) : 0;
            else    nvalid = (gk < Kd) ? (int)min(2ll, max(0ll, MNd - gmn)) : 0;
            const double *src = nvalid ? gaddr<KC>(X, ld, gmn, gk) : X;
            cp_async16(s + Tile<KC>::idx(mn, k), src, nvalid * 8);
        }
    } else {  // 8-byte elements: any alignment / odd ld
#pragma unroll
        for (int q = 0; q < (128 * BK) / NT; q++) {
            int c = tid + q * NT;
            int mn, k;
            if (KC) { mn = c / BK; k = c % BK; }
            else    { k = c >> 7;  mn = c & 127; }
            long long gmn = mn0 + mn, gk = k0 + k;
            bool ok = gmn < MNd && gk < Kd;
            cp_async8(s + Tile<KC>::idx(mn, k), ok ? gaddr<KC>(X, ld, gmn, gk) : X, ok ? 8 : 0);
        }
    }
}

// Producer-side staging of one 128 x BK operand tile by the PRODUCER_THREADS threads of the
// load warpgroup: one base pointer + a constant stride per thread (low register footprint,
// the producer runs with PRODUCER_REGS registers after setmaxnreg.dec).
constexpr int PRODUCER_THREADS_ = 128;
template <bool KC, bool VEC>
__device__ __forceinline__ void produce_tile(double *s, const double *X, long long ld, long long mn0,
                                             long long k0, long long MNd, long long Kd, int pt) {
    if (VEC) {
        if (KC) {  // k contiguous: BK/2 16-byte chunks per mn row
            constexpr int CPR = BK / 2, STEP = PRODUCER_THREADS_ / CPR;
            const int k = (pt % CPR) * 2, mnb = pt / CPR;
            const long long gk = k0 + k;
            const int kval = (int)min(2ll, max(0ll, Kd - gk));
            const double *src = X + gk + (mn0 + mnb) * ld;
            double *dst = s + mnb * LD_K + k;
#pragma unroll 4
            for (int q = 0; q < 128 / STEP; q++) {
                const int nv = (mn0 + mnb + q * STEP < MNd) ? kval : 0;
                cp_async16(dst + q * STEP * LD_K, nv ? src + (long long)q * STEP * ld : X, nv * 8);
            }
        } else {   // mn contiguous: 64 chunks per k row
            constexpr int STEP = PRODUCER_THREADS_ / 64;
            const int mn = (pt % 64) * 2, kb = pt / 64;
            const long long gmn = mn0 + mn;
            const int mval = (int)min(2ll, max(0ll, MNd - gmn));
            const double *src = X + gmn + (k0 + kb) * ld;
            double *dst = s + kb * LD_MN + mn;
#pragma unroll 4
            for (int q = 0; q < BK / STEP; q++) {
                const int nv = (k0 + kb + q * STEP < Kd) ? mval : 0;
                cp_async16(dst + q * STEP * LD_MN, nv ? src + (long long)q * STEP * ld : X, nv * 8);
            }
        }
    } else {  // 8-byte elements (misaligned pointer / odd ld): correctness path
#pragma unroll 1
        for (int c = pt; c < 128 * BK; c += PRODUCER_THREADS_) {
            int mn, k;
            if (KC) { mn = c / BK; k = c % BK; }
            else    { k = c >> 7;  mn = c & 127; }
            const long long gmn = mn0 + mn, gk = k0 + k;
            const bool ok = gmn < MNd && gk < Kd;
            cp_async8(s + Tile<KC>::idx(mn, k), ok ? gaddr<KC>(X, ld, gmn, gk) : X, ok ? 8 : 0);
        }
    }
}

// ------------------------------------------------------------------ encode kernel
// P(i,k) = op(A)(i,k) (operand 0) or op(B)(k,i) (operand 1).  KC: k contiguous.
// Block (tile t, chunk ch, operand) reduces a 128 x [kbeg,kend) slab:
//   V[t*Kp + k]            = sum_{i in tile} P(i,k)         (A^c row / B^r column)
//   line[ch*MNd + i]       = sum_{k in chunk} |P(i,k)|       (row / column 1-norms)
//   tmax[ch*ntiles + t]    = max_{k in chunk} sum_i |P(i,k)|
struct EncodeOperand {
    const double *X;
    long long ld, MNd;
    int kc;
    double *V, *line, *tmax;
    int ntiles;
};
struct EncodeArgs {
    EncodeOperand op[2];
    long long K, Kp, kper;
    int kch;
    ReportHdr *rep;  // zeroed here (stream-ordered before the GEMM kernel)
};

template <bool KC>
__device__ void encode_slab(const EncodeOperand &o, const EncodeArgs &a, int t, int ch, double (*s)[33],
                            double *red) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long i0 = (long long)t * 128;
    const long long kbeg = (long long)ch * a.kper;
    const long long kend = min(kbeg + a.kper, a.Kp);
    double la = 0.0, tm = 0.0;
    for (long long kb = kbeg; kb < kend; kb += 32) {
        for (int idx = tid; idx < 128 * 32; idx += NTHREADS) {
            int i, kk;
            if (KC) { i = idx >> 5; kk = idx & 31; }
            else    { i = idx & 127; kk = idx >> 7; }
            long long gi = i0 + i, gk = kb + kk;
            double v = 0.0;
            if (gi < o.MNd && gk < a.K) v = *gaddr<KC>(o.X, o.ld, gi, gk);
            s[i][kk] = v;
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < 4; q++) {
            int kk = warp * 4 + q;
            double sum = 0.0, sa = 0.0;
#pragma unroll
            for (int r = 0; r < 4; r++) {
                double v = s[lane + 32 * r][kk];
                sum += v;
                sa += fabs(v);
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                sum += __shfl_xor_sync(0xffffffffu, sum, off);
                sa += __shfl_xor_sync(0xffffffffu, sa, off);
            }
            if (kb + kk < kend) {
                if (lane == 0) o.V[(long long)t * a.Kp + kb + kk] = sum;
                tm = fmax(tm, sa);
            }
        }
        {
            int i = tid & 127, h = tid >> 7;
#pragma unroll
            for (int kk = 0; kk < 16; kk++) la += fabs(s[i][h * 16 + kk]);
        }
        __syncthreads();
    }
    // line partials: combine the two k-halves in fixed order
    red[tid] = la;
    if (lane == 0) red[NTHREADS + warp] = tm;
    __syncthreads();
    if (tid < 128) {
        long long gi = i0 + tid;
        if (gi < o.MNd) o.line[(long long)ch * o.MNd + gi] = red[tid] + red[tid + 128];
    }
    if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < NTHREADS / 32; w++) m = fmax(m, red[NTHREADS + w]);
        o.tmax[(long long)ch * o.ntiles + t] = m;
    }
}

__global__ void __launch_bounds__(NTHREADS) encode_kernel(EncodeArgs a) {
    __shared__ double s[128][33];
    __shared__ double red[NTHREADS + NTHREADS / 32];
    const EncodeOperand &o = a.op[blockIdx.z];
    const int t = blockIdx.x, ch = blockIdx.y;
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && threadIdx.x == 0 && a.rep) {
        a.rep->count = 0; a.rep->tiles_flagged = 0; a.rep->rows_flagged = 0; a.rep->cols_flagged = 0;
    }
    if (t >= o.ntiles) return;
    if (o.kc) encode_slab<true>(o, a, t, ch, s, red);
    else      encode_slab<false>(o, a, t, ch, s, red);
}


// ------------------------------------------------------------------ GEMM kernel
constexpr int LDT = 130;  // epilogue tile leading dimension (conflict-free fragment stores)
constexpr int EPI_EL = 128 * LDT   /* tile */
                     + 6 * 128     /* rowS[2][128], rowC[2][128], rowCA[2][128] */
                     + 3 * 128     /* colS, colC, colCA */
                     + 2 * 256     /* rsp[2][128], ssp[2][128] */
                     + 128         /* row residuals */
                     + 136;        /* flags (int) */

template <bool KCA, bool KCB, bool FT>
struct SmemPlan {
    static constexpr int A_EL = Tile<KCA>::ELEMS, B_EL = Tile<KCB>::ELEMS;
    static constexpr int STAGE_EL = A_EL + B_EL + (FT ? 2 * BK : 0);
    static constexpr int PIPE_EL = STAGES * STAGE_EL;
    static constexpr int BYTES = 8 * ((FT && EPI_EL > PIPE_EL) ? EPI_EL : PIPE_EL);
};

// Tile rasterization: groups of GROUP_M tile-rows, column-major inside a group, so the
// CTAs resident at one time share a few A row panels and B column panels in L2.
constexpr int GROUP_M = 16;
__device__ __forceinline__ void tile_coords(long long x, long long ntm, long long ntn, long long &tm, long long &tn) {
    const long long gsz = (long long)GROUP_M * ntn;
    const long long grp = x / gsz, first = grp * GROUP_M;
    const long long gm = min(ntm - first, (long long)GROUP_M);
    const long long r = x % gsz;
    tm = first + r % gm;
    tn = r / gm;
}

// One warp recomputes element (i,j) of op(A) op(B) from its definition:
// s = sum_k op(A)(i,k) op(B)(k,j), sa = sum_k |op(A)(i,k)| |op(B)(k,j)|.
template <bool KCA, bool KCB>
__device__ void warp_recompute(const GemmArgs &g, long long i, long long j, double &s, double &sa) {
    const int lane = threadIdx.x & 31;
    s = 0.0; sa = 0.0;
    for (long long k = lane; k < g.K; k += 32) {
        const double a = *gaddr<KCA>(g.A, g.lda, i, k);
        const double b = *gaddr<KCB>(g.B, g.ldb, j, k);
        s = fma(a, b, s);
        sa = fma(fabs(a), fabs(b), sa);
    }
#pragma unroll
    for (int off = 16; off; off >>= 1) {
        s += __shfl_xor_sync(0xffffffffu, s, off);
        sa += __shfl_xor_sync(0xffffffffu, sa, off);
    }
}

// Block = NTHREADS MMA threads (8 warps) + 1 producer warp that stages tiles with cp.async
// and signals per-stage `full` mbarriers; MMA warps release stages through `empty` mbarriers
// (no CTA-wide barrier in the mainloop, so the two MMA warps of an SMSP drift independently).
constexpr int PRODUCER_THREADS = PRODUCER_THREADS_;  // one warpgroup; registers go to the MMA warps
constexpr int GEMM_THREADS = NTHREADS + PRODUCER_THREADS;
// setmaxnreg only moves registers inside the CTA's launch allocation: ptxas caps a
// __launch_bounds__(384, 1) kernel at 168 registers/thread (65536/384 rounded down to a
// multiple of 8), so the pool is 384 x 168 = 64512.  An .inc that asks for more than the
// pool blocks forever.
constexpr int LAUNCH_REGS = 168;
constexpr int MMA_REGS = 224, PRODUCER_REGS = 56;  // 256x224 + 128x56 = 64512
static_assert(NTHREADS * MMA_REGS + PRODUCER_THREADS * PRODUCER_REGS <= GEMM_THREADS * LAUNCH_REGS,
              "setmaxnreg budget exceeds the launch register allocation (would deadlock)");

template <bool KCA, bool KCB, bool VECA, bool VECB, bool FT>
__global__ void __launch_bounds__(GEMM_THREADS, 1) gemm_kernel(GemmArgs g) {
    extern __shared__ __align__(128) double smem[];
    __shared__ __align__(8) unsigned long long full_bar[STAGES], empty_bar[STAGES];
    using SP = SmemPlan<KCA, KCB, FT>;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;
    const long long ntm = (g.M + BM - 1) / BM, ntn = (g.N + BN - 1) / BN;
    long long tm, tn;
    tile_coords(blockIdx.x, ntm, ntn, tm, tn);
    const long long m0 = tm * BM, n0 = tn * BN;
    const int ktiles = (g.alpha == 0.0) ? 0 : (int)((g.K + BK - 1) / BK);

    auto sA = [&](int st) { return smem + st * SP::STAGE_EL; };
    auto sB = [&](int st) { return smem + st * SP::STAGE_EL + SP::A_EL; };
    auto sW = [&](int st) { return smem + st * SP::STAGE_EL + SP::A_EL + SP::B_EL; };
    auto sV = [&](int st) { return smem + st * SP::STAGE_EL + SP::A_EL + SP::B_EL + BK; };

    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&full_bar[s], PRODUCER_THREADS); // one cp.async arrival per producer thread
            mbar_init(&empty_bar[s], NTHREADS / 32);   // one arrival per MMA warp
        }
    }
    __syncthreads();

    if (warp >= NTHREADS / 32) {
        // ------------------------------------------------------------ producer warpgroup
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
        const int pt = tid - NTHREADS;
        for (int kt = 0; kt < ktiles; kt++) {
            const int st = kt % STAGES;
            if (kt >= STAGES) mbar_wait(&empty_bar[st], ((kt / STAGES) - 1) & 1);
            const long long k0 = (long long)kt * BK;
            produce_tile<KCA, VECA>(sA(st), g.A, g.lda, m0, k0, g.M, g.K, pt);
            produce_tile<KCB, VECB>(sB(st), g.B, g.ldb, n0, k0, g.N, g.K, pt);
            if (FT) {
#pragma unroll
                for (int q = pt; q < BK; q += PRODUCER_THREADS) {
                    if (q < BK / 2) cp_async16(sW(st) + q * 2, g.WB + tn * g.Kp + k0 + q * 2, 16);
                    else            cp_async16(sV(st) + (q - BK / 2) * 2, g.VA + tm * g.Kp + k0 + (q - BK / 2) * 2, 16);
                }
            }
            cp_async_mbar_arrive(&full_bar[st]);
        }
        cp_wait<0>();
        return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(MMA_REGS));

    double acc[FM][FN][2];
#pragma unroll
    for (int a = 0; a < FM; a++)
#pragma unroll
        for (int b = 0; b < FN; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
    // checksum partials.  MN-contiguous smem layout: thread owns row/col (tid&127), k-half tid>>7.
    // k-contiguous layout: warp w owns rows 16w..16w+15, lane (r=lane>>2, kk=lane&3) owns rows
    // 16w+r and 16w+8+r at k = kk, kk+4, kk+8, kk+12 (2-wavefront smem reads).
    double rp0 = 0.0, rp1 = 0.0, sp0 = 0.0, sp1 = 0.0;

    for (int kt = 0; kt < ktiles; kt++) {
        const int st = kt % STAGES;
        mbar_wait(&full_bar[st], (kt / STAGES) & 1);
        const double *a_s = sA(st), *b_s = sB(st);
#pragma unroll
        for (int kk = 0; kk < BK / 4; kk++) {
            double af[FM], bf[FN];
            const int k = kk * 4 + (lane & 3);
#pragma unroll
            for (int f = 0; f < FM; f++) af[f] = a_s[Tile<KCA>::idx(wm * WM + f * 8 + (lane >> 2), k)];
#pragma unroll
            for (int f = 0; f < FN; f++) bf[f] = b_s[Tile<KCB>::idx(wn * WN + f * 8 + (lane >> 2), k)];
#pragma unroll
            for (int a = 0; a < FM; a++)
#pragma unroll
                for (int b = 0; b < FN; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
        if (FT) {
            // checksum column r_i += sum_k op(A)(i,k) w_k  and row s_j += sum_k v_k op(B)(k,j)
            const double *w_s = sW(st), *v_s = sV(st);
            if (!KCA) {
                const int r = tid & 127, h = tid >> 7;
#pragma unroll
                for (int q = 0; q < BK / 2; q++)
                    rp0 = fma(a_s[Tile<KCA>::idx(r, h * (BK / 2) + q)], w_s[h * (BK / 2) + q], rp0);
            } else {
                const int r = warp * 16 + (lane >> 2), kk = lane & 3;
#pragma unroll
                for (int q = 0; q < BK / 4; q++) {
                    rp0 = fma(a_s[Tile<KCA>::idx(r, kk + 4 * q)], w_s[kk + 4 * q], rp0);
                    rp1 = fma(a_s[Tile<KCA>::idx(r + 8, kk + 4 * q)], w_s[kk + 4 * q], rp1);
                }
            }
            if (!KCB) {
                const int c = tid & 127, h = tid >> 7;
#pragma unroll
                for (int q = 0; q < BK / 2; q++)
                    sp0 = fma(v_s[h * (BK / 2) + q], b_s[Tile<KCB>::idx(c, h * (BK / 2) + q)], sp0);
            } else {
                const int c = warp * 16 + (lane >> 2), kk = lane & 3;
#pragma unroll
                for (int q = 0; q < BK / 4; q++) {
                    sp0 = fma(v_s[kk + 4 * q], b_s[Tile<KCB>::idx(c, kk + 4 * q)], sp0);
                    sp1 = fma(v_s[kk + 4 * q], b_s[Tile<KCB>::idx(c + 8, kk + 4 * q)], sp1);
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[st]);
    }
    bar_mma();  // all MMA warps done with the pipeline smem (the producer has no pending copies)

    const bool beta0 = (g.beta == 0.0);
    if (!FT) {
        // ---------------------------------------------------------- non-FT epilogue
#pragma unroll
        for (int a = 0; a < FM; a++)
#pragma unroll
            for (int b = 0; b < FN; b++)
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    const long long gi = m0 + wm * WM + a * 8 + (lane >> 2);
                    const long long gj = n0 + wn * WN + b * 8 + 2 * (lane & 3) + e;
                    if (gi < g.M && gj < g.N) {
                        double *p = g.C + gi + gj * g.ldc;
                        *p = beta0 ? g.alpha * acc[a][b][e] : fma(g.alpha, acc[a][b][e], g.beta * *p);
                    }
                }
        return;
    }

    // -------------------------------------------------------------- FT epilogue
    double *tileS = smem;                    // [128 cols][LDT]
    double *rowS = tileS + 128 * LDT;        // [2][128]
    double *rowC = rowS + 256, *rowCA = rowC + 256;
    double *colS = rowCA + 256, *colC = colS + 128, *colCA = colC + 128;
    double *rsp = colCA + 128, *ssp = rsp + 256, *dres = ssp + 256;
    int *flags = reinterpret_cast<int *>(dres + 128);  // [0] nrow, [1] ncol, [2..129] rows, [130..257] cols
    const long long mvalid = min((long long)BM, g.M - m0), nvalid = min((long long)BN, g.N - n0);

    // checksum partials -> rsp/ssp ([2][128]: r_i = rsp[i] + rsp[128+i])
    if (!KCA) {
        rsp[tid] = rp0;
    } else {
#pragma unroll
        for (int off = 1; off <= 2; off <<= 1) {
            rp0 += __shfl_xor_sync(0xffffffffu, rp0, off);
            rp1 += __shfl_xor_sync(0xffffffffu, rp1, off);
        }
        if ((lane & 3) == 0) {
            const int r = warp * 16 + (lane >> 2);
            rsp[r] = rp0; rsp[r + 8] = rp1; rsp[128 + r] = 0.0; rsp[128 + r + 8] = 0.0;
        }
    }
    if (!KCB) {
        ssp[tid] = sp0;
    } else {
#pragma unroll
        for (int off = 1; off <= 2; off <<= 1) {
            sp0 += __shfl_xor_sync(0xffffffffu, sp0, off);
            sp1 += __shfl_xor_sync(0xffffffffu, sp1, off);
        }
        if ((lane & 3) == 0) {
            const int c = warp * 16 + (lane >> 2);
            ssp[c] = sp0; ssp[c + 8] = sp1; ssp[128 + c] = 0.0; ssp[128 + c + 8] = 0.0;
        }
    }
    if (tid == 0) { flags[0] = 0; flags[1] = 0; }

    // C0 tile -> smem, then its row/column sums (the beta C encoding)
    const int rr = tid & 127, hh = tid >> 7;
    if (!beta0) {
        for (int idx = tid; idx < BM * BN; idx += NTHREADS) {
            const int row = idx & 127, col = idx >> 7;
            const long long gi = m0 + row, gj = n0 + col;
            tileS[row + col * LDT] = (gi < g.M && gj < g.N) ? g.C[gi + gj * g.ldc] : 0.0;
        }
        bar_mma();
        double s = 0.0, sa = 0.0;
        for (int c = hh * 64; c < hh * 64 + 64; c++) {
            const double v = tileS[rr + c * LDT];
            s += v; sa += fabs(v);
        }
        rowC[hh * 128 + rr] = s; rowCA[hh * 128 + rr] = sa;
        for (int q = 0; q < 16; q++) {
            const int c = warp * 16 + q;
            double cs = 0.0, ca = 0.0;
#pragma unroll
            for (int r4 = 0; r4 < 4; r4++) {
                const double v = tileS[lane + 32 * r4 + c * LDT];
                cs += v; ca += fabs(v);
            }
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                cs += __shfl_xor_sync(0xffffffffu, cs, off);
                ca += __shfl_xor_sync(0xffffffffu, ca, off);
            }
            if (lane == 0) { colC[c] = cs; colCA[c] = ca; }
        }
        bar_mma();
    }
    // fault injection (test harness): flip accumulator bits of planned elements of this tile
    if (g.plan_ptr) {
        const int tix = (int)(tn * ntm + tm);
        const int lo = g.plan_ptr[tix], hi = g.plan_ptr[tix + 1];
        for (int f = lo; f < hi; f++) {
            const long long li = g.plan_i[f] - m0, lj = g.plan_j[f] - n0;
            const int bit = g.plan_bit[f];
#pragma unroll
            for (int a = 0; a < FM; a++)
#pragma unroll
                for (int b = 0; b < FN; b++)
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        const int row = wm * WM + a * 8 + (lane >> 2), col = wn * WN + b * 8 + 2 * (lane & 3) + e;
                        if (row == li && col == lj) acc[a][b][e] = flip_bit(acc[a][b][e], bit);
                    }
        }
    }
    // out = alpha acc + beta c0 -> smem tile (each element read/written by its owner thread)
#pragma unroll
    for (int a = 0; a < FM; a++)
#pragma unroll
        for (int b = 0; b < FN; b++)
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const int row = wm * WM + a * 8 + (lane >> 2), col = wn * WN + b * 8 + 2 * (lane & 3) + e;
                const bool ok = row < mvalid && col < nvalid;
                double o;
                if (beta0) o = g.alpha * acc[a][b][e];
                else       o = fma(g.alpha, acc[a][b][e], g.beta * tileS[row + col * LDT]);
                tileS[row + col * LDT] = ok ? o : 0.0;
            }
    bar_mma();
    // row / column sums of the computed tile (warp-shuffle reductions for the columns)
    {
        double s = 0.0;
        for (int c = hh * 64; c < hh * 64 + 64; c++) s += tileS[rr + c * LDT];
        rowS[hh * 128 + rr] = s;
        for (int q = 0; q < 16; q++) {
            const int c = warp * 16 + q;
            double cs = 0.0;
#pragma unroll
            for (int r4 = 0; r4 < 4; r4++) cs += tileS[lane + 32 * r4 + c * LDT];
#pragma unroll
            for (int off = 16; off; off >>= 1) cs += __shfl_xor_sync(0xffffffffu, cs, off);
            if (lane == 0) colS[c] = cs;
        }
    }
    bar_mma();
    // verification: flag rows / columns beyond the round-off threshold
    const double aa = fabs(g.alpha), ab = fabs(g.beta);
    if (tid < 128) {
        const int r = tid;
        const long long gi = m0 + r;
        if (r < mvalid) {
            const double sum = rowS[r] + rowS[128 + r];
            const double rr2 = rsp[r] + rsp[128 + r];
            const double c0s = beta0 ? 0.0 : rowC[r] + rowC[128 + r];
            const double c0a = beta0 ? 0.0 : rowCA[r] + rowCA[128 + r];
            const double ref = beta0 ? g.alpha * rr2 : fma(g.alpha, rr2, g.beta * c0s);
            double rowabs = 0.0, bmax = 0.0;
            for (int c = 0; c < g.kch; c++) {
                rowabs += g.lineA[(long long)c * g.M + gi];
                bmax = fmax(bmax, g.tmaxB[(long long)c * ntn + tn]);
            }
            const double tau = 4.0 * U_ROUND * (double)(g.K + nvalid + 3) * (aa * rowabs * bmax + ab * c0a);
            const double d = sum - ref;
            dres[r] = d;
            if (!(fabs(d) <= tau)) {
                const int p = atomicAdd(&flags[0], 1);
                flags[2 + p] = r;
            }
        }
    } else {
        const int c = tid - 128;
        const long long gj = n0 + c;
        if (c < nvalid) {
            const double sum = colS[c];
            const double ss2 = ssp[c] + ssp[128 + c];
            const double c0s = beta0 ? 0.0 : colC[c];
            const double c0a = beta0 ? 0.0 : colCA[c];
            const double ref = beta0 ? g.alpha * ss2 : fma(g.alpha, ss2, g.beta * c0s);
            double colabs = 0.0, amax = 0.0;
            for (int q = 0; q < g.kch; q++) {
                colabs += g.lineB[(long long)q * g.N + gj];
                amax = fmax(amax, g.tmaxA[(long long)q * ntm + tm]);
            }
            const double tau = 4.0 * U_ROUND * (double)(g.K + mvalid + 3) * (aa * amax * colabs + ab * c0a);
            const double d = sum - ref;
            if (!(fabs(d) <= tau)) {
                const int p = atomicAdd(&flags[1], 1);
                flags[130 + p] = c;
            }
        }
    }
    bar_mma();
    const int nr = flags[0], nc = flags[1];
    if (nr != 0 || nc != 0) {
        // ---------------------------------------------------------- locate + correct (rare)
        if (tid == 0) {
            atomicAdd(&g.rep->tiles_flagged, 1ull);
            atomicAdd(&g.rep->rows_flagged, (unsigned long long)nr);
            atomicAdd(&g.rep->cols_flagged, (unsigned long long)nc);
            for (int x = 1; x < nr; x++)
                for (int y = x; y > 0 && flags[2 + y - 1] > flags[2 + y]; y--) {
                    const int t = flags[2 + y]; flags[2 + y] = flags[2 + y - 1]; flags[2 + y - 1] = t;
                }
            for (int x = 1; x < nc; x++)
                for (int y = x; y > 0 && flags[130 + y - 1] > flags[130 + y]; y--) {
                    const int t = flags[130 + y]; flags[130 + y] = flags[130 + y - 1]; flags[130 + y - 1] = t;
                }
        }
        bar_mma();
        const bool single = (nr == 1 && nc == 1);  // Huang-Abraham location (line 540)
        const long long ncr = nr ? nr : mvalid, ncc = nc ? nc : nvalid;
        for (long long q = warp; q < ncr * ncc; q += NTHREADS / 32) {
            const int r = nr ? flags[2 + (int)(q % ncr)] : (int)(q % ncr);
            const int c = nc ? flags[130 + (int)(q / ncr)] : (int)(q / ncr);
            const long long gi = m0 + r, gj = n0 + c;
            double s, sa;
            warp_recompute<KCA, KCB>(g, gi, gj, s, sa);
            const double c0 = beta0 ? 0.0 : g.C[gi + gj * g.ldc];  // C is stored after this phase
            const double y = beta0 ? g.alpha * s : fma(g.alpha, s, g.beta * c0);
            const double eb = 4.0 * U_ROUND * (double)(g.K + 3) * (aa * sa + ab * fabs(c0));
            const double cur = tileS[r + c * LDT];
            if (lane == 0 && (single || !(fabs(cur - y) <= eb))) {
                tileS[r + c * LDT] = y;  // correction (reading R6: recompute the located element)
                const unsigned long long p = atomicAdd(&g.rep->count, 1ull);
                if ((long long)p < g.rep_cap) {
                    Correction cr;
                    cr.tile_m = tm; cr.tile_n = tn; cr.i = gi; cr.j = gj;
                    cr.residual = dres[r];
                    cr.kind = single ? 1 : 2; cr.pad = 0;
                    g.rep_entries[p] = cr;
                }
            }
        }
        bar_mma();
    }
    // coalesced store of the verified tile
    for (int idx = tid; idx < BM * BN; idx += NTHREADS) {
        const int row = idx & 127, col = idx >> 7;
        if (row < mvalid && col < nvalid) g.C[(m0 + row) + (n0 + col) * g.ldc] = tileS[row + col * LDT];
    }
}

}  // namespace ftb
