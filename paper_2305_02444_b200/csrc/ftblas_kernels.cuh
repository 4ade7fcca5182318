// ftblas_kernels.cuh -- sm_100a kernels of the ABFT DGEMM hot path.
//
//   encode_kernel : Huang-Abraham checksum encoding of op(A) and op(B) per
//                   verification tile (section II.A:
//                   A^c = [A; e^T A], B^r = [B, B e]) plus the norms used by the
//                   round-off threshold (reading R4).  HBM-bound stream.
//   gemm_kernel   : C := alpha op(A) op(B) + beta C on FP64 tensor cores
//                   (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4, the FP64 tensor-core
//                   instruction of sm_100a; tcgen05.mma has no f64 kind).  Operand tiles
//                   are staged by TMA (cp.async.bulk.tensor, 128-byte swizzle) into a
//                   STAGES-deep smem ring driven by one producer thread and mbarriers.
//                   With FT=true it also accumulates the checksum column C e = A (B e)
//                   and row e^T C = (e^T A) B of the tile in the same mainloop (line 516,
//                   "C^f = A^c B^r"), and its epilogue verifies, locates and corrects
//                   (lines 517, 540, 521) before the store.  FT=false is the non-FT
//                   baseline (same tiles/mainloop).
//
// CTA: 8 MMA warps (DMMA fragments of 8x8, BK = 32) plus producer threads (struct Warps).
// NWN = 4: 128 x 128 CTA tile, 2 x 4 warps of 64 x 32, producer warpgroup, one CTA per SM,
// 3-stage ring.  NWN = 2 ("pair"): 128 x 64 CTA tile, 4 x 2 warps of 32 x 32, one producer
// warp, two CTAs per SM, 2-stage ring; in FT mode the two halves of a 128 x 128 verification
// tile are a cluster exchanging row sums through DSMEM.
//   side_finalize_kernel / cksum_kernel: see their sections.  DESIGN.md section 5.
#pragma once
#include <cstdint>
#include <cuda.h>
#include <cuda_runtime.h>

namespace ftb {

#ifndef FTB_BK  // k-depth of a pipeline stage / number of stages (overridable for experiments)
#define FTB_BK 32
#endif
#ifndef FTB_STAGES
#define FTB_STAGES 3
#endif
constexpr int BM = 128, BN = 128, BK = FTB_BK, STAGES = FTB_STAGES, NTHREADS = 256;
constexpr int WM = 64, WN = 32, FM = WM / 8, FN = WN / 8;
static_assert(BK % 16 == 0, "BK must be a multiple of the 16-double TMA box row");
constexpr double U_ROUND = 1.0 / 9007199254740992.0;  // 2^-53

// ---------------------------------------------------------------- smem operand tile layout
// One stage of an operand is a dense 128 x BK tile of doubles made of 128-byte rows, the
// layout TMA writes with CU_TENSOR_MAP_SWIZZLE_128B:
//   KC=false (mn contiguous in HBM: op(A)=A 'N', op(B)=B 'T'): 8 boxes of 16 mn, each box
//            [BK k-rows][16 mn];
//   KC=true  (k contiguous in HBM: op(A)=A 'T', op(B)=B 'N'): BK/16 boxes of 16 k, each box
//            [128 mn-rows][16 k].
// Inside 128-byte row r, the 16-byte unit u (elements 2u, 2u+1) sits at unit u ^ (r & 7).
// With the fragment row maps of frag_mn() below, every DMMA fragment load (a warp reads
// 8 mn x 4 k; the 64-bit shared load is served per half-warp of 4 mn x 4 k) touches 16
// distinct 8-byte bank pairs in each half-warp: 2 wavefronts for 256 bytes, conflict-free.
// (ROWS = mn extent of the tile: 128 for the main GEMM, 16..128 for the checksum GEMMs' thin
// operand.)
constexpr int TILE_EL = 128 * BK;
template <bool KC, int ROWS = 128>
struct Tile {
    __device__ __forceinline__ static int idx(int mn, int k) {
        if (KC) {
            const int kk = k & 15;
            return (k >> 4) * (ROWS * 16) + mn * 16 + ((((kk >> 1) ^ (mn & 7)) << 1) | (kk & 1));
        } else {
            const int m = mn & 15;
            return (mn >> 4) * (BK * 16) + k * 16 + ((((m >> 1) ^ (k & 7)) << 1) | (m & 1));
        }
    }
};
// mn index (within the CTA tile) of row g = (g2 g1 g0) of the 8-wide fragment f of a warp
// tile starting at `base` (a half-warp has fixed g2 and covers g0, g1 x 4 k):
//   KC=true : mn = base + 8 f + (g2 + 2 g0 + 4 g1)     -> bank pair (k0, k1^g2, k2^g0, k3^g1)
//   KC=false: mn = base + 16 (f>>1) + (g0 + 2 (f&1) + 4 g2 + 8 g1)
//                                                       -> bank pair (g0, f1^k0, g2^k1, g1^k2)
// so the 16 lanes of a half-warp hit 16 distinct bank pairs in both layouts.  The
// accumulator row / column of C fragment element (g, j) is frag_mn of the A / B side: the
// MMA is agnostic to which mn a fragment row stands for, as long as A, B and C agree.
template <bool KC>
__device__ __forceinline__ int frag_mn(int base, int f, int g) {
    const int g0 = g & 1, g1 = (g >> 1) & 1, g2 = g >> 2;
    return KC ? base + 8 * f + (g2 + 2 * g0 + 4 * g1)
              : base + 16 * (f >> 1) + (g0 + 2 * (f & 1) + 4 * g2 + 8 * g1);
}

// Per-thread precomputed smem offsets of the DMMA fragment loads: the element (row g of
// fragment f, k = 4 kk + (lane & 3)) of a warp tile at `base` is at a compile-time constant
// (from f, kk) plus one of 4 per-thread offsets (the swizzle XOR only depends on f & 1 and
// kk & 1 for KC=false, on kk & 3 for KC=true).  Equal to Tile<KC>::idx(frag_mn<KC>(base, f,
// g), k) -- asserted by the unit test of tests/test_gpu_parity.py through the results.
template <bool KC, int ROWS = 128>
struct FragAddr {
    int off[4];
    __device__ __forceinline__ FragAddr(int base, int lane) {
        const int g = lane >> 2, l3 = lane & 3;
#pragma unroll
        for (int v = 0; v < 4; v++) {
            if (KC) {  // v = kk & 3; mn = base + frag_mn<true>(0, 0, g), base % 8 == 0
                const int kk16 = 4 * v + l3, n = frag_mn<true>(0, 0, g);
                off[v] = (base + n) * 16 + ((((kk16 >> 1) ^ (n & 7)) << 1) | (kk16 & 1));
            } else {   // v = (f & 1) | (kk & 1) << 1; base % 16 == 0
                const int f1 = v & 1, k7 = 4 * (v >> 1) + l3;
                const int m = frag_mn<false>(0, f1, g);
                off[v] = (base >> 4) * (BK * 16) + l3 * 16 + ((((m >> 1) ^ k7) << 1) | (m & 1));
            }
        }
    }
    // f, kk compile-time after unrolling
    __device__ __forceinline__ int operator()(int f, int kk) const {
        if (KC) return off[kk & 3] + (kk >> 2) * (ROWS * 16) + 8 * f * 16;
        return off[(f & 1) | ((kk & 1) << 1)] + (f >> 1) * (BK * 16) + (kk & ~1) * 4 * 16 + (kk & 1) * 4 * 16;
    }
};

struct Correction {  // == ftblas_correction (48 bytes)
    long long tile_m, tile_n, i, j;
    double residual;
    int kind, pad;
};
struct ReportHdr {  // device-side counters
    unsigned long long count, tiles_flagged, rows_flagged, cols_flagged;
};
// A correction candidate located by the persistent kernel's epilogue, recomputed after the
// GEMM by correct_kernel (ftblas_ws.cuh): element (i, j) of the call's C, its stored value,
// its C0, the row residual and whether it is a single-error location (kind 1).
struct Pending {
    long long i, j;
    double cur, c0, residual;
    int single, pad;
};
struct PendingHdr {
    unsigned long long count;
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
    int kch, kchB;         // partial counts of the A side / the B side (1: finalized, ftblas_encode_b)
    long long Kp;
    const double *Rpre;    // FT_PRE: [splits_r][ntn][M], R[tn][i] = sum_k op(A)(i,k) WB[tn][k] (k-split partials)
    const double *Spre;    // FT_PRE: [splits_s][ntm][N], S[tm][j] = sum_k VA[tm][k] op(B)(k,j)
    int splits_r, splits_s;
    long long stride_r, stride_s;
    // finalized side data (side_finalize_kernel): partials summed once, in fixed order
    const double *fin_nrmA, *fin_nrmB;  // M, N  : ||op(A)(i,:)||_1, ||op(B)(:,j)||_1
    const double *fin_maxA, *fin_maxB;  // ntm, ntn: tile maxima of the column / row |.| sums
    const double *fin_R, *fin_S;        // FT_PRE: ntn x M, ntm x N (checksum GEMM results)
    // fault plan in the caller's coordinates: CSR by the caller's tile (index gtn * plan_ntm +
    // gtm over a plan_ntm x plan_ntn grid), entries i, j of the caller's C
    const int *plan_ptr;   // plan_ntm * plan_ntn + 1 or nullptr
    const long long *plan_i, *plan_j;
    const int *plan_bit;
    long long plan_ntm, plan_ntn;
    // report
    ReportHdr *rep;
    Correction *rep_entries;
    long long rep_cap;
    PendingHdr *pend;        // correction candidates (persistent kernel, ftblas_ws.cuh)
    Pending *pend_entries;
    long long pend_cap;
    long long off_i, off_j;  // position of this call's C block in the caller's C (report indices)
    int vecC;              // C 16-byte aligned with even ldc (cp.async16 staging of C0)
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
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long *b, unsigned bytes) {
    asm volatile("{\n\t.reg .b64 st;\n\tmbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n\t}\n" ::"r"(
                     smem_u32(b)), "r"(bytes)
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
// TMA: 2-D tiled box global -> smem, completion counted in bytes on mbarrier b
__device__ __forceinline__ void tma_load_2d(void *dst, const CUtensorMap *map, unsigned long long *b, int c0,
                                            int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];\n" ::
            "r"(smem_u32(dst)), "l"(map), "r"(smem_u32(b)), "r"(c0), "r"(c1)
        : "memory");
}
// bulk (non-tensor) copy of `bytes` (multiple of 16) global -> smem, counted on mbarrier b
__device__ __forceinline__ void bulk_load(void *dst, const void *src, unsigned bytes, unsigned long long *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                     smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(b))
                 : "memory");
}
// Distributed shared memory (cluster of 2): store to the same variable in CTA `rank` of the
// cluster, and the cluster-wide barrier (release / acquire).
__device__ __forceinline__ void st_cluster_f64(double *p, unsigned rank, double v) {
    unsigned a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
    asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(a), "d"(v) : "memory");
}
__device__ __forceinline__ void st_cluster_s32(int *p, unsigned rank, int v) {
    unsigned a;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(a) : "r"(smem_u32(p)), "r"(rank));
    asm volatile("st.shared::cluster.s32 [%0], %1;\n" ::"r"(a), "r"(v) : "memory");
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// L2 prefetch of `bytes` (multiple of 16, 16-byte aligned source) -- no smem, no completion
__device__ __forceinline__ void bulk_prefetch_l2(const void *src, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(src), "r"(bytes) : "memory");
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

constexpr int PRODUCER_THREADS = 128;  // one warpgroup; registers go to the MMA warps

// Stage one 128 x BK operand tile (rows [mn0, mn0+128), k [k0, k0+BK)) into the swizzled
// layout.  TMA=true: thread 0 of the producer warpgroup issues the boxes (bytes counted on
// `bar` through the expect_tx of the caller); out-of-range elements are zero-filled by TMA.
// TMA=false (operand pointer not 16-byte aligned or odd ld, where a tensor map cannot be
// built): every producer thread copies 8-byte elements with cp.async, zero-fill outside
// [0,MNd) x [0,Kd).
template <bool KC, bool TMA, int ROWS = 128, int NTP = PRODUCER_THREADS>
__device__ __forceinline__ void produce_tile(double *s, const CUtensorMap *map, unsigned long long *bar,
                                             const double *X, long long ld, long long mn0, long long k0,
                                             long long MNd, long long Kd, int pt) {
    if (TMA) {
        if (pt == 0) {
            if (KC) {
#pragma unroll
                for (int h = 0; h < BK / 16; h++) tma_load_2d(s + h * ROWS * 16, map, bar, (int)(k0 + 16 * h), (int)mn0);
            } else {
#pragma unroll
                for (int c = 0; c < ROWS / 16; c++) tma_load_2d(s + c * BK * 16, map, bar, (int)(mn0 + 16 * c), (int)k0);
            }
        }
    } else {
#pragma unroll 4
        for (int c = pt; c < ROWS * BK; c += NTP) {
            int mn, k;
            if (KC) { mn = c / BK; k = c % BK; }
            else    { k = c / ROWS; mn = c % ROWS; }
            const long long gmn = mn0 + mn, gk = k0 + k;
            const bool ok = gmn < MNd && gk < Kd;
            cp_async8(s + Tile<KC, ROWS>::idx(mn, k), ok ? gaddr<KC>(X, ld, gmn, gk) : X, ok ? 8 : 0);
        }
    }
}

// ------------------------------------------------------------------ encode kernel
// P(i,k) = op(A)(i,k) (operand 0) or op(B)(k,i) (operand 1).  KC: k contiguous.
// Block (tile t, chunk ch, operand) streams the 128 x [kbeg,kend) slab of P once:
//   V[t*Kp + k]            = sum_{i in tile} P(i,k)         (A^c row / B^r column, line 516)
//   line[ch*MNd + i]       = sum_{k in chunk} |P(i,k)|       (row / column 1-norms, reading R4)
//   tmax[ch*ntiles + t]    = max_{k in chunk} sum_i |P(i,k)|
// V is zero for k in [K, Kp) (the GEMM stages whole BK-wide slices of V).  HBM-bound: every
// element is read once with coalesced (16-byte where possible) loads, several loads in flight
// per thread; the cross-lane reductions are warp shuffles.
struct EncodeOperand {
    const double *X;
    long long ld, MNd;
    int kc, vec;
    double *V, *line, *tmax;
    int ntiles;
};
struct EncodeArgs {
    EncodeOperand op[2];
    long long K, Kp, kper;
    int kch;
    ReportHdr *rep;  // zeroed here (stream-ordered before the GEMM kernel)
    PendingHdr *pend;  // zeroed here on every FT call
    int op_base;     // operand of blockIdx.z = 0
};

// an unsigned stored in the low word of a double's bit pattern (smem / DSMEM transport only)
__device__ __forceinline__ double u32_as_dbits(unsigned u) { return __longlong_as_double((long long)u); }
__device__ __forceinline__ unsigned dbits_as_u32(double d) { return (unsigned)__double_as_longlong(d); }

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// mn contiguous (op(A) = A 'N', op(B) = B 'T'): warp w reduces columns k = kbeg + w + 8q.
// Lane l owns rows {2l, 2l+1, 64+2l, 65+2l} (VEC, 16-byte loads) or {l, l+32, l+64, l+96}.
template <bool VEC>
__device__ void encode_mn_contig(const EncodeOperand &o, const EncodeArgs &a, int t, long long kbeg,
                                 long long kend, double *red, double &tm) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long i0 = (long long)t * 128;
    int rows[4];
    if (VEC) { rows[0] = 2 * lane; rows[1] = 2 * lane + 1; rows[2] = 64 + 2 * lane; rows[3] = 65 + 2 * lane; }
    else     { rows[0] = lane; rows[1] = lane + 32; rows[2] = lane + 64; rows[3] = lane + 96; }
    bool rv[4];
#pragma unroll
    for (int r = 0; r < 4; r++) rv[r] = i0 + rows[r] < o.MNd;
    double la[4] = {0.0, 0.0, 0.0, 0.0};
    constexpr int U = 4;  // columns per warp per iteration (independent loads in flight)
    for (long long k = kbeg + warp; k < kend; k += 8 * U) {
        double x[U][4];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const long long kk = k + 8 * u;
            const bool kv = kk < a.K && kk < kend;
            const double *col = o.X + i0 + kk * o.ld;
            if (VEC) {
                double2 p = make_double2(0.0, 0.0), q = make_double2(0.0, 0.0);
                if (kv && rv[1]) p = __ldcs(reinterpret_cast<const double2 *>(col + rows[0]));
                else if (kv && rv[0]) p.x = __ldcs(col + rows[0]);
                if (kv && rv[3]) q = __ldcs(reinterpret_cast<const double2 *>(col + rows[2]));
                else if (kv && rv[2]) q.x = __ldcs(col + rows[2]);
                x[u][0] = p.x; x[u][1] = p.y; x[u][2] = q.x; x[u][3] = q.y;
            } else {
#pragma unroll
                for (int r = 0; r < 4; r++) x[u][r] = (kv && rv[r]) ? __ldcs(col + rows[r]) : 0.0;
            }
        }
        // v[u] = this lane's part of the sum of column u, v[U + u] of its |.| sum; the 2U = 8
        // warp sums by a transposing butterfly (7 + 2 shuffles instead of 40): afterwards lane
        // l holds value 4 b4 + 2 b3 + b2 (b = bits of l), the same in the 4 lanes l ^ {1,2,3}
        double v[2 * U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            v[u] = (x[u][0] + x[u][1]) + (x[u][2] + x[u][3]);
            v[U + u] = (fabs(x[u][0]) + fabs(x[u][1])) + (fabs(x[u][2]) + fabs(x[u][3]));
#pragma unroll
            for (int r = 0; r < 4; r++) la[r] += fabs(x[u][r]);
        }
#pragma unroll
        for (int off = 16; off >= 4; off >>= 1) {
            const bool up = (lane & off) != 0;
#pragma unroll
            for (int j = 0; j < off / 4; j++) {
                const double send = up ? v[j] : v[j + off / 4];
                const double keep = up ? v[j + off / 4] : v[j];
                v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
        }
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 2);
        v[0] += __shfl_xor_sync(0xffffffffu, v[0], 1);
        const int idx = ((lane >> 2) & 1) + ((lane >> 3) & 1) * 2 + ((lane >> 4) & 1) * 4;
        const long long kk = k + 8 * (idx & (U - 1));
        if (kk < kend) {
            if (idx < U) {
                if ((lane & 3) == 0) o.V[(long long)t * a.Kp + kk] = v[0];  // 0 for kk >= K
            } else {
                tm = fmax(tm, v[0]);
            }
        }
    }
#pragma unroll
    for (int r = 0; r < 4; r++) red[warp * 128 + rows[r]] = la[r];
}

// k contiguous (op(A) = A 'T', op(B) = B 'N'): the chunk is walked in slabs of 128 k; warp w
// owns mn 16w .. 16w+15 of the tile and lane l the 4 consecutive k 4l .. 4l+3 of the slab, so
// one warp-wide load pair reads 1 KB of one mn (2 x 16 B per lane when 16-byte aligned).  The
// per-mn |.| sums over the slab's 128 k: transposing butterfly over the warp's 16 mn (15 + 1
// shuffles), lanes 2j, 2j+1 then hold mn 16w + j.  The per-k sums over the tile's 128 mn (V and
// the |.| sums behind tmax) are combined across the 8 warps through shared memory in warp order.
__device__ void encode_k_contig(const EncodeOperand &o, const EncodeArgs &a, int t, long long kbeg,
                                long long kend, double *red, double &tm) {
    __shared__ double ks[NTHREADS / 32][2][128];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const long long i0 = (long long)t * 128;
    const int nrow = (int)min(128ll, o.MNd - i0);
    const long long klim = min(kend, a.K);
    const int idx = ((lane >> 1) & 1) + ((lane >> 2) & 1) * 2 + ((lane >> 3) & 1) * 4 + ((lane >> 4) & 1) * 8;
    double la = 0.0;
    for (long long k0 = kbeg; k0 < kend; k0 += 128) {
        const long long k = k0 + 4 * lane;
        const bool full = o.vec && k + 3 < klim;  // 2 x 16-byte loads
        double s4[4] = {0.0, 0.0, 0.0, 0.0}, sa4[4] = {0.0, 0.0, 0.0, 0.0}, v[16];
#pragma unroll
        for (int j = 0; j < 16; j++) {
            const int i = warp * 16 + j;
            double x[4] = {0.0, 0.0, 0.0, 0.0};
            if (i < nrow) {
                const double *p = o.X + k + (i0 + i) * o.ld;
                if (full) {
                    const double2 u0 = __ldcs(reinterpret_cast<const double2 *>(p));
                    const double2 u1 = __ldcs(reinterpret_cast<const double2 *>(p) + 1);
                    x[0] = u0.x; x[1] = u0.y; x[2] = u1.x; x[3] = u1.y;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; q++) x[q] = (k + q < klim) ? __ldcs(p + q) : 0.0;
                }
            }
#pragma unroll
            for (int q = 0; q < 4; q++) { s4[q] += x[q]; sa4[q] += fabs(x[q]); }
            v[j] = (fabs(x[0]) + fabs(x[1])) + (fabs(x[2]) + fabs(x[3]));
        }
#pragma unroll
        for (int off = 16; off >= 2; off >>= 1) {
            const bool up = (lane & off) != 0;
#pragma unroll
            for (int j = 0; j < off / 2; j++) {
                const double send = up ? v[j] : v[j + off / 2];
                const double keep = up ? v[j + off / 2] : v[j];
                v[j] = keep + __shfl_xor_sync(0xffffffffu, send, off);
            }
        }
        la += v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
#pragma unroll
        for (int q = 0; q < 4; q++) { ks[warp][0][4 * lane + q] = s4[q]; ks[warp][1][4 * lane + q] = sa4[q]; }
        __syncthreads();
        if (tid < 128 && k0 + tid < kend) {
            double sv = 0.0, sav = 0.0;
#pragma unroll
            for (int w = 0; w < NTHREADS / 32; w++) { sv += ks[w][0][tid]; sav += ks[w][1][tid]; }
            o.V[(long long)t * a.Kp + k0 + tid] = sv;  // 0 for k >= K
            tm = fmax(tm, sav);
        }
        __syncthreads();
    }
    // line partials: this warp's 16 mn, zeros elsewhere (the caller adds the warps' rows)
    for (int i = lane; i < 128; i += 32) red[warp * 128 + i] = 0.0;
    __syncwarp();
    if ((lane & 1) == 0) red[warp * 128 + warp * 16 + idx] = la;
}

// PATH 0: k contiguous (slab walk, cross-warp k sums in shared memory);
// PATH 1 / 2: mn contiguous with 16-byte / 8-byte loads.  3 blocks / SM (<= 80 registers): a
// latency-bound stream that wants loads in flight).  Operand = a.op[a.op_base + blockIdx.z],
// laid out along PATH0 (z = 0) or PATH1 (z = 1): both operands in one launch.
template <int PATH0, int PATH1>
__global__ void __launch_bounds__(NTHREADS, 3) encode_kernel(EncodeArgs a) {
    __shared__ double red[(NTHREADS / 32) * 128];
    __shared__ double wmax[NTHREADS / 32];
    const EncodeOperand &o = a.op[a.op_base + blockIdx.z];
    const int t = blockIdx.x, ch = blockIdx.y, tid = threadIdx.x;
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && tid == 0 && a.rep) {
        a.rep->count = 0; a.rep->tiles_flagged = 0; a.rep->rows_flagged = 0; a.rep->cols_flagged = 0;
    }
    if (blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && tid == 0 && a.pend) a.pend->count = 0;
    if (t >= o.ntiles) return;
    const long long kbeg = (long long)ch * a.kper;
    const long long kend = min(kbeg + a.kper, a.Kp);
    double tm = 0.0;
    const int path = blockIdx.z == 0 ? PATH0 : PATH1;  // block-uniform
    if (path == 0)      encode_k_contig(o, a, t, kbeg, kend, red, tm);
    else if (path == 1) encode_mn_contig<true>(o, a, t, kbeg, kend, red, tm);
    else                encode_mn_contig<false>(o, a, t, kbeg, kend, red, tm);
#pragma unroll
    for (int off = 16; off; off >>= 1) tm = fmax(tm, __shfl_xor_sync(0xffffffffu, tm, off));
    if ((tid & 31) == 0) wmax[tid >> 5] = tm;
    __syncthreads();
    if (tid < 128) {  // line partial of row tid: warps combined in fixed order
        double l = 0.0;
#pragma unroll
        for (int w = 0; w < NTHREADS / 32; w++) l += red[w * 128 + tid];
        const long long gi = (long long)t * 128 + tid;
        if (gi < o.MNd) o.line[(long long)ch * o.MNd + gi] = l;
    }
    if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < NTHREADS / 32; w++) m = fmax(m, wmax[w]);
        o.tmax[(long long)ch * o.ntiles + t] = m;
    }
}


// ------------------------------------------------------------------ GEMM kernel
constexpr int LDT = 130;  // epilogue tile leading dimension (conflict-free fragment stores)
        /* flags (int) */

// Dynamic smem: [STAGES][A tile | B tile] (1024-byte aligned boxes for the 128-byte swizzle),
// then [STAGES][w_J slice | v_I slice] (FT checksum vectors, BK each).  The FT epilogue
// reuses the same bytes once the mainloop has drained.
// Kernel modes.  NOFT: plain DGEMM (the overhead denominator; also computes the checksum
// GEMMs of MODE_FT_PRE).  FT_PRE: the border of C^f = A^c B^r was
// computed before the launch by two DMMA GEMMs, R = op(A) W and S^T = op(B)^T V^T (DESIGN.md
// section 5, "checksum GEMMs"); the mainloop is the plain one and the epilogue verifies.
// FT_FUSED: the checksum column / row are accumulated in the same mainloop from the operand
// fragments (DFMA), as the paper fuses them into its kernel.
enum { MODE_NOFT = 0, MODE_FT_PRE = 1, MODE_FT_FUSED = 2 };

// Warp layout of a gemm_kernel CTA (128 x 32 NWN tile).  Both layouts have 8 MMA warps, two
// per SM sub-partition, which is what keeps the DMMA pipe fed (tools/dmma_mainloop.cu: a
// 128 x 64 CTA of 4 warps reaches 32.5 TFLOP/s alone, of 8 warps 32 x 32 36.9).
//   NWN = 4: 2 (M) x 4 (N) warps of 64 x 32, producer warpgroup (setmaxnreg 224 / 56).
//   NWN = 2: 4 (M) x 2 (N) warps of 32 x 32, one producer warp, 2 CTAs / SM, no setmaxnreg
//            (9 warps x 2 CTAs: at most 5 warps per SM sub-partition -> 96 registers).
template <int NWN>
struct Warps {
    static constexpr int WM = NWN == 4 ? 64 : 32, WN = 32;
    static constexpr int NWM = BM / WM, NWW = 32 * NWN / WN;  // warps along M / along N
    static constexpr int FM = WM / 8, FN = WN / 8;
    static constexpr int NT = 32 * NWM * NWW;                 // MMA threads
    static constexpr int PT = NWN == 4 ? PRODUCER_THREADS : 32;  // producer threads
    static_assert(NT == 256, "8 MMA warps");
};

template <int MODE, int NWN = 4>
struct SmemPlan {
    static constexpr int BNT = 32 * NWN;
    static constexpr int STAGE_EL = TILE_EL + BNT * BK;
    static constexpr int NSTAGE = NWN == 4 ? STAGES : 2;  // pair CTAs: 2 per SM
    static constexpr int PIPE_EL = NSTAGE * STAGE_EL + (MODE == MODE_FT_FUSED ? NSTAGE * 2 * BK : 0);
    // every mode stages the C tile ([BNT][LDT]) in the drained pipeline bytes; FT adds the
    // reduction arrays
    static constexpr int EPI_FT = BNT * LDT + Warps<NWN>::NWW * 3 * 128 + Warps<NWN>::NWM * 3 * BNT + 2 * 256 + 128 + 136;
    static constexpr int EPI = MODE != MODE_NOFT ? EPI_FT : BNT * LDT;
    static constexpr int EL = EPI > PIPE_EL ? EPI : PIPE_EL;
    static constexpr int BYTES = 8 * EL + 1024;  // + alignment slack
};

// sum_{c < n} p[c * stride] in index order, loads issued in batches of 8 (n <= 64 here)
__device__ __forceinline__ double sum_strided(const double *p, long long stride, int n) {
    double s = 0.0;
    for (int c0 = 0; c0 < n; c0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = (c0 + u < n) ? p[(long long)(c0 + u) * stride] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; u++)
            if (c0 + u < n) s += v[u];
    }
    return s;
}
__device__ __forceinline__ double max_strided(const double *p, long long stride, int n) {
    double m = 0.0;
    for (int c0 = 0; c0 < n; c0 += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; u++) v[u] = (c0 + u < n) ? p[(long long)(c0 + u) * stride] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; u++) m = fmax(m, v[u]);
    }
    return m;
}

// Tile rasterization: groups of GROUP_M tile-rows, column-major inside a group, so the
// CTAs resident at one time share a few A row panels and B column panels in L2.
constexpr int GROUP_M = 8;
__device__ __forceinline__ void tile_coords(long long x, long long ntm, long long ntn, long long &tm, long long &tn) {
    const long long gsz = (long long)GROUP_M * ntn;
    const long long grp = x / gsz, first = grp * GROUP_M;
    const long long gm = min(ntm - first, (long long)GROUP_M);
    const long long r = x % gsz;
    tm = first + r % gm;
    tn = r / gm;
}

// Block = NTHREADS MMA threads (8 warps) + producer threads (Warps<NWN>::PT).  Thread 0 of the producer
// issues the TMA boxes of each stage (and the bulk copies of the checksum-vector slices) and
// arms the stage's `full` mbarrier with the byte count; MMA warps release stages through
// `empty` mbarriers (no CTA-wide barrier in the mainloop).  The other producer threads only
// work when an operand cannot be described by a tensor map (cp.async fallback) and, for FT,
// reduce the threshold norms of the tile.
constexpr int GEMM_THREADS = NTHREADS + PRODUCER_THREADS;
// setmaxnreg only moves registers inside the CTA's launch allocation: ptxas caps a
// __launch_bounds__(384, 1) kernel at 168 registers/thread (65536/384 rounded down to a
// multiple of 8), so the pool is 384 x 168 = 64512.  An .inc that asks for more than the
// pool blocks forever.
constexpr int LAUNCH_REGS = 168;
constexpr int MMA_REGS = 224, PRODUCER_REGS = 56;  // 256x224 + 128x56 = 64512
static_assert(NTHREADS * MMA_REGS + PRODUCER_THREADS * PRODUCER_REGS <= GEMM_THREADS * LAUNCH_REGS,
              "setmaxnreg budget exceeds the launch register allocation (would deadlock)");
// Pair CTAs (2 per SM) have one producer warp and no setmaxnreg: with a producer warpgroup
// (with or without setmaxnreg) accumulators of CTAs sharing an SM came out corrupted under
// some schedules (NT operands, tiles with long correction phases next to clean ones); the
// one-warp variant is clean in every stress run (regression test
// test_many_faulted_tiles_leave_neighbours_clean).  9 warps per CTA -> 96 registers.

// NWN = 4: one CTA per 128 x 128 tile (8 MMA warps of 64 x 32, 1 CTA / SM).
// NWN = 2 ("pair"): one CTA per 128 x 64 half of a 128 x 128 verification tile (8 MMA warps of
// 32 x 32, 2 CTAs / SM, so one CTA's epilogue overlaps the other's mainloop); for FT the two halves
// form a cluster of 2 and exchange their row partial sums and column-flag counts through
// distributed shared memory, so verification, location and reports are those of the
// 128 x 128 tile.
template <bool KCA, bool KCB, bool TMA, int MODE, int NWN>
__global__ void __launch_bounds__(Warps<NWN>::NT + Warps<NWN>::PT, NWN == 2 ? 2 : 1)
    gemm_kernel(const __grid_constant__ GemmArgs g, const __grid_constant__ CUtensorMap tmA,
                const __grid_constant__ CUtensorMap tmB) {
    using WL = Warps<NWN>;
    constexpr int NT = WL::NT, PT = WL::PT;    // MMA / producer threads
    constexpr int WM = WL::WM, WN = WL::WN, FM = WL::FM, FN = WL::FN, NWM = WL::NWM, NWW = WL::NWW;
    constexpr int BNT = 32 * NWN;              // CTA tile columns
    constexpr bool FT = MODE != MODE_NOFT, FUSED = MODE == MODE_FT_FUSED;
    constexpr bool PAIR = NWN == 2 && FT;      // cluster pair sharing one verification tile
    static_assert(NWN == 4 || (NWN == 2 && !FUSED), "pair tiles: NOFT / FT_PRE only");
    extern __shared__ __align__(1024) double smem_raw[];
    __shared__ __align__(8) unsigned long long full_bar[STAGES], empty_bar[STAGES], norm_bar;
    // threshold norms of this tile (reading R4), reduced over the encode k-chunks by the
    // producer warpgroup while the MMA warps run the mainloop
    __shared__ double nrm_row[BM], nrm_col[BNT], nrm_max[2];
    // FT_PRE: this tile's slices of the checksum GEMM outputs R and S^T (loaded by the producer)
    __shared__ double pre_r[MODE == MODE_FT_PRE ? BM : 1], pre_s[MODE == MODE_FT_PRE ? BNT : 1];
    // PAIR: row partial sums (out, C0, |C0|) and the column-flag count written by the peer CTA
    __shared__ double peer_rows[PAIR ? 3 * BM : 1];
    __shared__ int peer_nc;
    constexpr bool TMA_A = TMA, TMA_B = TMA;
    // 1024-byte aligned base, derived by indexing (keeps the pointer in the shared window so
    // the loads below use 32-bit shared addressing)
    double *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) / 8u;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % NWM, wn = warp / NWM;
    const long long ntm = (g.M + BM - 1) / BM, ntn = (g.N + BN - 1) / BN;  // 128 x 128 tiles
    long long tm, tn;
    tile_coords(NWN == 4 ? blockIdx.x : blockIdx.x >> 1, ntm, ntn, tm, tn);
    const int half = NWN == 4 ? 0 : (int)(blockIdx.x & 1);  // PAIR: also the cluster rank
    const long long m0 = tm * BM, n0 = tn * BN + half * BNT;  // this CTA's columns [n0, n0 + BNT)
    const int ktiles = (g.alpha == 0.0) ? 0 : (int)((g.K + BK - 1) / BK);
    using SP = SmemPlan<MODE, NWN>;
    constexpr int NS = SP::NSTAGE;  // pipeline stages

    auto sA = [&](int st) { return smem + st * SP::STAGE_EL; };
    auto sB = [&](int st) { return smem + st * SP::STAGE_EL + TILE_EL; };
    auto sW = [&](int st) { return smem + NS * SP::STAGE_EL + st * 2 * BK; };
    auto sV = [&](int st) { return sW(st) + BK; };

    constexpr bool ALL_TMA = TMA_A && TMA_B;
    if (tid == 0) {
        for (int s = 0; s < NS; s++) {
            // thread 0 of the producer arrives with expect_tx; cp.async fallback threads add
            // one arrival each when their copies land
            mbar_init(&full_bar[s], 1 + (ALL_TMA ? 0 : PT));
            mbar_init(&empty_bar[s], NT / 32);  // one arrival per MMA warp
        }
        if (NWN == 4 && FT) mbar_init(&norm_bar, PT - 32);  // producer warps 1..3
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // PAIR: every thread arrives on the cluster barrier now and the MMA threads wait on it
    // before the first distributed-shared-memory store, so the peer CTA is known to have
    // started (the programming model's requirement for DSMEM access)
    if (PAIR) asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");

    if (warp >= NT / 32) {
        // ------------------------------------------------------------ producer warpgroup
        if (NWN == 4) asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
        const int pt = tid - NT;
        constexpr unsigned TX = (TMA_A ? TILE_EL * 8 : 0) + (TMA_B ? BNT * BK * 8 : 0) + (FUSED ? 2 * BK * 8 : 0);
        auto produce = [&](int kt) {
            const int st = kt % NS;
            const long long k0 = (long long)kt * BK;
            if (pt == 0) {
                mbar_arrive_expect_tx(&full_bar[st], TX);
                if (FUSED) {
                    bulk_load(sW(st), g.WB + tn * g.Kp + k0, BK * 8, &full_bar[st]);
                    bulk_load(sV(st), g.VA + tm * g.Kp + k0, BK * 8, &full_bar[st]);
                }
            }
            produce_tile<KCA, TMA_A, 128, PT>(sA(st), &tmA, &full_bar[st], g.A, g.lda, m0, k0, g.M, g.K, pt);
            produce_tile<KCB, TMA_B, BNT, PT>(sB(st), &tmB, &full_bar[st], g.B, g.ldb, n0, k0, g.N, g.K, pt);
            if (!ALL_TMA) cp_async_mbar_arrive(&full_bar[st]);
        };
        if (FT && NWN == 4 && pt >= 32) {
            // Threshold norms (reading R4) and, for FT_PRE, the checksum-GEMM slices of this tile,
            // by producer warps 1..3 while thread 0 streams the operand stages: quantity q < 128 is
            // row q, 128 <= q < 128 + BNT column q - 128 of this CTA, then the tile maxima of A / B.
            // Sums over the encode k-chunks / the k-splits in fixed order, loads issued in batches
            // (FP64 arithmetic off the MMA warps: beside the DMMA stream it costs several times its
            // share).  Pair tiles copy the side_finalize_kernel sums instead
            // (MMA threads, cp.async, below).
            for (int q = pt - 32; q < 128 + BNT + 2; q += PT - 32) {
                if (q < 128) {
                    const long long gi = m0 + q;
                    const bool ok = gi < g.M;
                    nrm_row[q] = !ok ? 0.0 : sum_strided(g.lineA + gi, g.M, g.kch);
                    if (MODE == MODE_FT_PRE)
                        pre_r[q] = !ok ? 0.0 : sum_strided(g.Rpre + tn * g.M + gi, g.stride_r, g.splits_r);
                } else if (q < 128 + BNT) {
                    const long long gj = n0 + (q - 128);
                    const bool ok = gj < g.N;
                    nrm_col[q - 128] = !ok ? 0.0 : sum_strided(g.lineB + gj, g.N, g.kchB);
                    if (MODE == MODE_FT_PRE)
                        pre_s[q - 128] = !ok ? 0.0 : sum_strided(g.Spre + tm * g.N + gj, g.stride_s, g.splits_s);
                } else if (q == 128 + BNT) {
                    nrm_max[0] = max_strided(g.tmaxA + tm, ntm, g.kch);
                } else {
                    nrm_max[1] = max_strided(g.tmaxB + tn, ntn, g.kchB);
                }
            }
            mbar_arrive(&norm_bar);
        }
        if (ALL_TMA) {
            if (pt != 0) return;
            for (int kt = 0; kt < ktiles; kt++) {
                if (kt == NS && g.beta != 0.0 && g.vecC) {
                    // C0 of this tile -> L2 while the mainloop runs (the epilogue stages it into
                    // smem afterwards); after the first stages so it does not delay them
                    const unsigned bytes = (unsigned)(min((long long)BM, g.M - m0) * 8) & ~15u;
                    const long long nv = min((long long)BNT, g.N - n0);
                    if (bytes)
                        for (int c = 0; c < nv; c++) bulk_prefetch_l2(g.C + m0 + (n0 + c) * g.ldc, bytes);
                }
                if (kt >= NS) mbar_wait(&empty_bar[kt % NS], ((kt / NS) - 1) & 1);
                produce(kt);
            }
        } else {
            for (int kt = 0; kt < ktiles; kt++) {
                if (kt >= NS) mbar_wait(&empty_bar[kt % NS], ((kt / NS) - 1) & 1);
                produce(kt);
            }
            cp_wait<0>();
        }
        return;
    }
    if (NWN == 4) asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(MMA_REGS));
    auto bar_mma = [&]() { asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory"); };
    if (PAIR) {
        // this half's finalized side data (side_finalize_kernel) -> smem by cp.async while the
        // first operand stages are in flight; completed by the epilogue's cp.async wait
        for (int q = tid; q < 128 + BNT + 2; q += NT) {
            if (q < 128) {
                const long long gi = m0 + q;
                const bool ok = gi < g.M;
                cp_async8(&nrm_row[q], ok ? g.fin_nrmA + gi : g.fin_nrmA, ok ? 8 : 0);
                cp_async8(&pre_r[q], ok ? g.fin_R + tn * g.M + gi : g.fin_R, ok ? 8 : 0);
            } else if (q < 128 + BNT) {
                const long long gj = n0 + (q - 128);
                const bool ok = gj < g.N;
                cp_async8(&nrm_col[q - 128], ok ? g.fin_nrmB + gj : g.fin_nrmB, ok ? 8 : 0);
                cp_async8(&pre_s[q - 128], ok ? g.fin_S + tm * g.N + gj : g.fin_S, ok ? 8 : 0);
            } else if (q == 128 + BNT) {
                cp_async8(&nrm_max[0], g.fin_maxA + tm, 8);
            } else {
                cp_async8(&nrm_max[1], g.fin_maxB + tn, 8);
            }
        }
        cp_commit();
    }

    double acc[FM][FN][2];
#pragma unroll
    for (int a = 0; a < FM; a++)
#pragma unroll
        for (int b = 0; b < FN; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
    // checksum partials (FT): the border of C^f = A^c B^r accumulated from
    // the operand fragments already in registers for the DMMAs:
    //   rp[t] += op(A)(row, k) w_J[k]   for the rows of A fragment 2 wn + t (column C e = A (B e))
    //   sp[t] += v_I[k] op(B)(k, col)   for the cols of B fragment 2 wm + t (row e^T C = (e^T A) B)
    // each lane over its k = 4 kk + (lane & 3); the 4 k-lanes are combined after the loop.  The
    // four wn-warps of a wm-half split the 8 A fragments, the two wm-warps of a wn-column the 4 B
    // fragments; the fragment is picked with warp-uniform selects (constant register indices).
    double rp[2] = {0.0, 0.0}, sp[2] = {0.0, 0.0};
    const FragAddr<KCA> fA(wm * WM, lane);
    const FragAddr<KCB, BNT> fB(wn * WN, lane);

    // One pipeline stage; `st` is a compile-time constant (the k-tile loop is unrolled by
    // NS), so every fragment address is a per-thread offset plus an immediate.
    auto consume = [&](const int st, const int kt) {
        mbar_wait(&full_bar[st], (kt / NS) & 1);
        const double *a_s = sA(st), *b_s = sB(st);
        const double *w_s = sW(st), *v_s = sV(st);
#pragma unroll
        for (int kk = 0; kk < BK / 4; kk++) {
            double af[FM], bf[FN];
            const int k = kk * 4 + (lane & 3);
#pragma unroll
            for (int f = 0; f < FM; f++) af[f] = a_s[fA(f, kk)];
#pragma unroll
            for (int f = 0; f < FN; f++) bf[f] = b_s[fB(f, kk)];
#pragma unroll
            for (int a = 0; a < FM; a++)
#pragma unroll
                for (int b = 0; b < FN; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
            if constexpr (FUSED) {
                const double wk = w_s[k], vk = v_s[k];
                // warp-uniform branches pick the fragment pair (no select temporaries)
                if (wn == 0)      { rp[0] = fma(af[0], wk, rp[0]); rp[1] = fma(af[1], wk, rp[1]); }
                else if (wn == 1) { rp[0] = fma(af[2], wk, rp[0]); rp[1] = fma(af[3], wk, rp[1]); }
                else if (wn == 2) { rp[0] = fma(af[4], wk, rp[0]); rp[1] = fma(af[5], wk, rp[1]); }
                else              { rp[0] = fma(af[6], wk, rp[0]); rp[1] = fma(af[7], wk, rp[1]); }
                if (wm == 0) { sp[0] = fma(vk, bf[0], sp[0]); sp[1] = fma(vk, bf[1], sp[1]); }
                else         { sp[0] = fma(vk, bf[2], sp[0]); sp[1] = fma(vk, bf[3], sp[1]); }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[st]);
    };
    for (int kt0 = 0; kt0 < ktiles; kt0 += NS) {
#pragma unroll
        for (int st = 0; st < NS; st++)
            if (kt0 + st < ktiles) consume(st, kt0 + st);
    }
    bar_mma();  // all MMA warps done with the pipeline smem (every issued copy was consumed)

    // accumulator element (a, b, e) of this thread is C-tile entry (row_of(a), col_of(b, e))
    auto row_of = [&](int a) { return frag_mn<KCA>(wm * WM, a, lane >> 2); };
    auto col_of = [&](int b, int e) { return frag_mn<KCB>(wn * WN, b, 2 * (lane & 3) + e); };

    const bool beta0 = (g.beta == 0.0);
    // beta = 1 (rank-k updates): the non-FT epilogue skips the DMUL (1.0 * c0 is exact, same
    // value); the FT epilogue keeps the general form (measured faster there: c2 4.709 vs 4.738 ms)
    const bool beta1 = (g.beta == 1.0);
    // The epilogue stages the C tile in smem ([128 cols][LDT], reusing the drained pipeline):
    // C0 arrives with cp.async (every load of the tile in flight at once, zero-fill outside
    // M x N), out = alpha acc + beta C0 is formed per fragment element, and the tile leaves
    // with coalesced column stores.
    double *tileS = smem;
    // mvalid x nvalid: valid part of this CTA's block; tvalid: valid columns of the whole
    // 128-wide verification tile (the row thresholds count all its columns)
    const long long mvalid = min((long long)BM, g.M - m0), nvalid = max(0ll, min((long long)BNT, g.N - n0));
    const long long tvalid = min((long long)BN, g.N - tn * BN);
    auto stage_c0 = [&]() {
        if (g.vecC) {
#pragma unroll 8
            for (int idx = tid; idx < BM * BNT / 2; idx += NT) {
                const int row = (idx & 63) * 2, col = idx >> 6;
                const long long gi = m0 + row, gj = n0 + col;
                const int nv = (gj < g.N) ? (int)min(2ll, max(0ll, g.M - gi)) : 0;
                cp_async16(tileS + row + col * LDT, nv ? g.C + gi + gj * g.ldc : g.C, nv * 8);
            }
        } else {
#pragma unroll 8
            for (int idx = tid; idx < BM * BNT; idx += NT) {
                const int row = idx & 127, col = idx >> 7;
                const long long gi = m0 + row, gj = n0 + col;
                const bool ok = gi < g.M && gj < g.N;
                cp_async8(tileS + row + col * LDT, ok ? g.C + gi + gj * g.ldc : g.C, ok ? 8 : 0);
            }
        }
        cp_commit();
        cp_wait<0>();
    };
    // out = alpha acc + beta c0 -> smem tile (each element read/written by its owner thread)
    auto form_out = [&]() {
#pragma unroll
        for (int a = 0; a < FM; a++)
#pragma unroll
            for (int b = 0; b < FN; b++)
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    const int row = row_of(a), col = col_of(b, e);
                    const bool ok = row < mvalid && col < nvalid;
                    double o;
                    if (beta0) o = g.alpha * acc[a][b][e];
                    else if (beta1) o = fma(g.alpha, acc[a][b][e], tileS[row + col * LDT]);
                    else       o = fma(g.alpha, acc[a][b][e], g.beta * tileS[row + col * LDT]);
                    tileS[row + col * LDT] = ok ? o : 0.0;
                }
    };
    auto store_tile = [&]() {
        if (g.vecC) {
#pragma unroll 8
            for (int idx = tid; idx < BM * BNT / 2; idx += NT) {
                const int row = (idx & 63) * 2, col = idx >> 6;
                if (col >= nvalid || row >= mvalid) continue;
                double *dst = g.C + (m0 + row) + (n0 + col) * g.ldc;
                if (row + 1 < mvalid) *reinterpret_cast<double2 *>(dst) = *reinterpret_cast<const double2 *>(tileS + row + col * LDT);
                else                  *dst = tileS[row + col * LDT];
            }
        } else {
            for (int idx = tid; idx < BM * BNT; idx += NT) {
                const int row = idx & 127, col = idx >> 7;
                if (row < mvalid && col < nvalid) g.C[(m0 + row) + (n0 + col) * g.ldc] = tileS[row + col * LDT];
            }
        }
    };

    if (!FT) {
        // ---------------------------------------------------------- non-FT epilogue
        if (!beta0) {
            stage_c0();
            bar_mma();
        }
        form_out();
        bar_mma();
        store_tile();
        return;
    }

    // -------------------------------------------------------------- FT epilogue
    // partial row sums [wn][q][128] and column sums [wm][q][BNT], q = 0: out, 1: C0, 2: |C0|
    double *red_r = tileS + BNT * LDT;       // NWW x 3 x 128
    double *red_c = red_r + NWW * 3 * 128;   // NWM x 3 x BNT
    double *rsp = red_c + NWM * 3 * BNT, *ssp = rsp + 256, *dres = ssp + 256;
    int *flags = reinterpret_cast<int *>(dres + 128);  // [0] nrow, [1] ncol, [2..129] rows, [130..] cols

    // checksum reference: FUSED -- combine the 4 k-lanes of the mainloop partials (fixed order),
    // one writer per row / column; FT_PRE -- the checksum-GEMM slices staged by the producer
    // (read after the norm barrier below).  rsp[i] = r_i (row i of the C e column), ssp[j] = s_j
    // (column j of the e^T C row).
    if constexpr (FUSED) {
#pragma unroll
        for (int t = 0; t < 2; t++) {
            rp[t] += __shfl_xor_sync(0xffffffffu, rp[t], 1);
            rp[t] += __shfl_xor_sync(0xffffffffu, rp[t], 2);
            sp[t] += __shfl_xor_sync(0xffffffffu, sp[t], 1);
            sp[t] += __shfl_xor_sync(0xffffffffu, sp[t], 2);
        }
        if ((lane & 3) == 0) {
#pragma unroll
            for (int t = 0; t < 2; t++) {
                rsp[frag_mn<KCA>(wm * WM, 2 * wn + t, lane >> 2)] = rp[t];
                ssp[frag_mn<KCB>(wn * WN, 2 * wm + t, lane >> 2)] = sp[t];
            }
        }
    }
    if (tid == 0) { flags[0] = 0; flags[1] = 0; }

    // C0 tile -> smem (all loads in flight at once)
    if (!beta0) {
        stage_c0();
        bar_mma();
    }
    // fault injection (test harness): flip accumulator bits of planned elements of this tile
    const long long gtm = tm + g.off_i / BM, gtn = tn + g.off_j / BN;  // the caller's tile
    if (g.plan_ptr && gtm < g.plan_ntm && gtn < g.plan_ntn) {
        const long long tix = gtn * g.plan_ntm + gtm;
        const int lo = g.plan_ptr[tix], hi = g.plan_ptr[tix + 1];
        for (int f = lo; f < hi; f++) {
            const long long li = g.plan_i[f] - g.off_i - m0, lj = g.plan_j[f] - g.off_j - n0;
            const int bit = g.plan_bit[f];
#pragma unroll
            for (int a = 0; a < FM; a++)
#pragma unroll
                for (int b = 0; b < FN; b++)
#pragma unroll
                    for (int e = 0; e < 2; e++) {
                        if (row_of(a) == li && col_of(b, e) == lj) acc[a][b][e] = flip_bit(acc[a][b][e], bit);
                    }
        }
    }
    // One pass over this thread's fragment elements: out = alpha acc + beta C0 into the smem
    // tile (0 outside M x N), with, per row and per column of the tile, the sum of
    // d = out - beta C0 (the computed alpha op(A) op(B) part of the stored value, PAPER.md
    // line 558: the reference sums are formed "at register level") and the maximum of |C0|
    // (threshold ingredient, reading R4k).  d costs one DADD per element beyond the plain
    // epilogue and the |C0| maxima run on the integer pipe (maxima of the high words of the
    // doubles, which order non-negative doubles): FP64 instructions in the epilogue wait for
    // the FP64 pipe that the co-resident CTA's DMMA stream keeps busy.
    // Sums: over the thread's elements of a fragment row / column, then over the 4 / 8 lanes
    // of that row / column (transposing butterflies); column fragments outer, so the column
    // partials of one fragment are reduced and stored before the next.
    {
        double rs[FM];
        unsigned rm[FM];
#pragma unroll
        for (int a = 0; a < FM; a++) { rs[a] = 0.0; rm[a] = 0u; }
#pragma unroll
        for (int b = 0; b < FN; b++) {
            double cs[2] = {0.0, 0.0};
            unsigned cm[2] = {0u, 0u};
#pragma unroll
            for (int a = 0; a < FM; a++) {
                const int row = row_of(a);
#pragma unroll
                for (int e = 0; e < 2; e++) {
                    const int col = col_of(b, e);
                    const bool ok = row < mvalid && col < nvalid;
                    double o, d;
                    if (beta0) {
                        o = g.alpha * acc[a][b][e];
                        d = o;
                    } else {
                        const double c0 = tileS[row + col * LDT];  // 0 outside M x N (zero-filled)
                        const double t = g.beta * c0;
                        o = fma(g.alpha, acc[a][b][e], t);
                        d = o - t;
                        const unsigned h = (unsigned)__double2hiint(c0) & 0x7fffffffu;
                        rm[a] = max(rm[a], h);
                        cm[e] = max(cm[e], h);
                    }
                    o = ok ? o : 0.0;
                    d = ok ? d : 0.0;
                    tileS[row + col * LDT] = o;
                    rs[a] += d;
                    cs[e] += d;
                }
            }
            // columns: 8 lanes (lane bits 2..4); first step transposing (lane keeps e = bit 2)
            {
                const bool hi = lane & 4;
                double x = (hi ? cs[1] : cs[0]) + __shfl_xor_sync(0xffffffffu, hi ? cs[0] : cs[1], 4);
                x += __shfl_xor_sync(0xffffffffu, x, 8);
                x += __shfl_xor_sync(0xffffffffu, x, 16);
                unsigned m = hi ? cm[1] : cm[0];
                m = max(m, __shfl_xor_sync(0xffffffffu, hi ? cm[0] : cm[1], 4));
                m = max(m, __shfl_xor_sync(0xffffffffu, m, 8));
                m = max(m, __shfl_xor_sync(0xffffffffu, m, 16));
                if ((lane & 24) == 0) {
                    const int c = col_of(b, hi ? 1 : 0);
                    red_c[(wm * 3 + 0) * BNT + c] = x;
                    red_c[(wm * 3 + 1) * BNT + c] = u32_as_dbits(m);
                }
            }
        }
        // rows: 4 lanes (lane bits 0, 1), transposing: FM values halve twice (FM = 4 or 8)
        {
            constexpr int H = FM / 2, Q = FM / 4;
            const bool b0 = lane & 1, b1 = lane & 2;
            double w[H], x[Q];
            unsigned wmx[H], xm[Q];
#pragma unroll
            for (int p = 0; p < H; p++) {
                w[p] = (b0 ? rs[p + H] : rs[p]) + __shfl_xor_sync(0xffffffffu, b0 ? rs[p] : rs[p + H], 1);
                wmx[p] = max(b0 ? rm[p + H] : rm[p], __shfl_xor_sync(0xffffffffu, b0 ? rm[p] : rm[p + H], 1));
            }
#pragma unroll
            for (int p = 0; p < Q; p++) {
                x[p] = (b1 ? w[p + Q] : w[p]) + __shfl_xor_sync(0xffffffffu, b1 ? w[p] : w[p + Q], 2);
                xm[p] = max(b1 ? wmx[p + Q] : wmx[p], __shfl_xor_sync(0xffffffffu, b1 ? wmx[p] : wmx[p + Q], 2));
            }
#pragma unroll
            for (int p = 0; p < Q; p++) {
                const int a = p + (b0 ? H : 0) + (b1 ? Q : 0);
                red_r[(wn * 3 + 0) * 128 + row_of(a)] = x[p];
                red_r[(wn * 3 + 1) * 128 + row_of(a)] = u32_as_dbits(xm[p]);
            }
        }
    }
    if (PAIR) cp_wait<0>();  // this thread's side-data copies (beta = 0 has no C0 staging wait)
    bar_mma();
    // verification: flag rows / columns beyond the round-off threshold
    const double aa = fabs(g.alpha), ab = fabs(g.beta);
    if (!PAIR) mbar_wait(&norm_bar, 0);  // producer-reduced norms are in nrm_row / nrm_col / nrm_max
    // row sums of this CTA's columns (wn partials in fixed order); PAIR: exchanged with the
    // peer half through distributed shared memory and added in half order (h0 + h1), so both
    // CTAs hold the identical sums of the whole 128-wide tile.  q = 0: sum of d, q = 1: the
    // high word of max |C0| (as the bits of a double; combined with an integer max).
    auto rsum_local = [&](int q, int r) {
        if (q == 0) {
            double v = red_r[(0 * 3 + 0) * 128 + r];
#pragma unroll
            for (int w = 1; w < NWW; w++) v += red_r[(w * 3 + 0) * 128 + r];
            return v;
        }
        unsigned m = dbits_as_u32(red_r[(0 * 3 + 1) * 128 + r]);
#pragma unroll
        for (int w = 1; w < NWW; w++) m = max(m, dbits_as_u32(red_r[(w * 3 + 1) * 128 + r]));
        return u32_as_dbits(m);
    };
    auto rsum = [&](int q, int r) {
        if (!PAIR) return rsum_local(q, r);
        const double mine = rsum_local(q, r), theirs = peer_rows[q * BM + r];
        if (q == 1) return u32_as_dbits(max(dbits_as_u32(mine), dbits_as_u32(theirs)));
        return half == 0 ? mine + theirs : theirs + mine;
    };
    // n x max |C0| >= sum |C0| over n elements (reading R4k): the high word h of max |C0|
    // rounded up to h + 1 (+Inf when C0 holds Inf / NaN)
    auto c0_bound = [&](double hbits, long long n) {
        const unsigned h = dbits_as_u32(hbits);
        if (h >= 0x7ff00000u) return __longlong_as_double(0x7ff0000000000000ll);
        return (double)n * __hiloint2double((int)(h + 1u), 0);
    };
    auto verify_row = [&](int r) {
        if (r >= mvalid) return;
        const double sum = rsum(0, r);
        const double rr2 = FUSED ? rsp[r] : pre_r[r];
        const double c0a = beta0 ? 0.0 : c0_bound(rsum(1, r), tvalid);
        const double ref = g.alpha * rr2;
        const double rowabs = nrm_row[r], bmax = nrm_max[1];
        const double tau = 4.0 * U_ROUND * (double)(g.K + tvalid + 3) * (aa * rowabs * bmax + ab * c0a);
        const double d = sum - ref;
        dres[r] = d;
        if (!(fabs(d) <= tau)) {
            const int p = atomicAdd(&flags[0], 1);
            flags[2 + p] = r;
        }
    };
    auto verify_col = [&](int c) {  // all 128 rows of a column are in this CTA
        if (c >= nvalid) return;
        double sum = red_c[(0 * 3 + 0) * BNT + c];
        unsigned m = dbits_as_u32(red_c[(0 * 3 + 1) * BNT + c]);
#pragma unroll
        for (int w = 1; w < NWM; w++) {
            sum += red_c[(w * 3 + 0) * BNT + c];
            m = max(m, dbits_as_u32(red_c[(w * 3 + 1) * BNT + c]));
        }
        const double ss2 = FUSED ? ssp[c] : pre_s[c];
        const double c0a = beta0 ? 0.0 : c0_bound(u32_as_dbits(m), mvalid);
        const double ref = g.alpha * ss2;
        const double colabs = nrm_col[c], amax = nrm_max[0];
        const double tau = 4.0 * U_ROUND * (double)(g.K + mvalid + 3) * (aa * amax * colabs + ab * c0a);
        const double d = sum - ref;
        if (!(fabs(d) <= tau)) {
            const int p = atomicAdd(&flags[1], 1);
            flags[130 + p] = c;
        }
    };
    if (PAIR) {
        // one cluster barrier per tile: the columns are verified before the exchange, so the
        // column-flag count travels with the row partial sums
        const unsigned peer = (unsigned)(half ^ 1);
        asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");  // peer started (arrived at entry)
        for (int qq = tid; qq < BM + BNT; qq += NT) {
            if (qq < BM) {
#pragma unroll
                for (int q = 0; q < 2; q++) st_cluster_f64(&peer_rows[q * BM + qq], peer, rsum_local(q, qq));
            } else {
                verify_col(qq - BM);
            }
        }
        bar_mma();
        if (tid == 0) st_cluster_s32(&peer_nc, peer, flags[1]);
        cluster_sync();
        for (int r = tid; r < BM; r += NT) verify_row(r);
    } else {
        for (int qq = tid; qq < BM + BNT; qq += NT) {
            if (qq < BM) verify_row(qq);
            else verify_col(qq - BM);
        }
    }
    bar_mma();
    // nr: flagged rows of the verification tile (identical in both halves); nc: flagged columns
    // of this CTA; nct: flagged columns of the whole tile (PAIR: + the peer's count)
    const int nr = flags[0], nc = flags[1];
    const int nct = PAIR ? nc + peer_nc : nc;
    if (nr != 0 || nct != 0) {
        // ---------------------------------------------------------- locate (rare)
        // candidates: (flagged rows, or all rows) x (this CTA's flagged columns, or all its
        // columns when no column of the tile is flagged); none when only the peer has flags
        // (readings R5, R7).  Each is listed with its stored value and C0 (C is stored after
        // this); the K-long recomputation and the correction (reading R6) run after the GEMM in
        // correct_kernel (ftblas_ws.cuh): a long recomputation beside DMMA mainloops running on
        // the same SM (the co-resident pair CTA) corrupted their accumulators (DESIGN.md
        // section 2), and one warp on a K-long strided dot product stalled the tile.
        if (tid == 0) {
            if (half == 0) {  // once per verification tile
                atomicAdd(&g.rep->tiles_flagged, 1ull);
                atomicAdd(&g.rep->rows_flagged, (unsigned long long)nr);
            }
            atomicAdd(&g.rep->cols_flagged, (unsigned long long)nc);
        }
        const bool single = (nr == 1 && nct == 1);  // Huang-Abraham location (line 540)
        const long long ncr = nr ? nr : mvalid, ncc = nct ? nc : nvalid;
        for (long long q = tid; q < ncr * ncc; q += NT) {
            const int r = nr ? flags[2 + (int)(q % ncr)] : (int)(q % ncr);
            const int c = nc ? flags[130 + (int)(q / ncr)] : (int)(q / ncr);
            const unsigned long long p = atomicAdd(&g.pend->count, 1ull);
            if ((long long)p < g.pend_cap) {
                Pending pe;
                pe.i = m0 + r; pe.j = n0 + c;
                pe.cur = tileS[r + c * LDT];
                pe.c0 = beta0 ? 0.0 : __ldcg(g.C + (m0 + r) + (n0 + c) * g.ldc);
                pe.residual = dres[r];
                pe.single = single ? 1 : 0; pe.pad = 0;
                g.pend_entries[p] = pe;
            }
        }
        bar_mma();  // every candidate's C0 read before the tile overwrites C
    }
    // coalesced store of the verified tile
    store_tile();
}



// ------------------------------------------------------------------ side-data finalize
// FT_PRE: sums the per-k-chunk norm partials of encode_kernel and the k-split partials of the
// checksum GEMMs in fixed (index) order into one value per row / column (and the tile maxima),
// so the GEMM kernel only copies them (grid-stride, HBM-bound, one read of every partial).
struct FinArgs {
    const double *lineA, *lineB, *tmaxA, *tmaxB, *Rp, *Sp;
    long long M, N, ntm, ntn, stride_r, stride_s;
    int kch, kchB, splits_r, splits_s;
    double *nrmA, *nrmB, *maxA, *maxB, *R, *S;
};
__global__ void __launch_bounds__(256) side_finalize_kernel(FinArgs f) {
    const long long nA = f.M, nB = f.N, nmA = f.ntm, nmB = f.ntn;
    const long long nR = f.Rp ? f.ntn * f.M : 0, nS = f.Sp ? f.ntm * f.N : 0;  // nullptr: already final
    const long long total = nA + nB + nmA + nmB + nR + nS;
    for (long long x = (long long)blockIdx.x * blockDim.x + threadIdx.x; x < total; x += (long long)gridDim.x * blockDim.x) {
        long long y = x;
        if (y < nA) { f.nrmA[y] = sum_strided(f.lineA + y, f.M, f.kch); continue; }
        y -= nA;
        if (y < nB) { f.nrmB[y] = sum_strided(f.lineB + y, f.N, f.kchB); continue; }
        y -= nB;
        if (y < nmA) { f.maxA[y] = max_strided(f.tmaxA + y, f.ntm, f.kch); continue; }
        y -= nmA;
        if (y < nmB) { f.maxB[y] = max_strided(f.tmaxB + y, f.ntn, f.kchB); continue; }
        y -= nmB;
        if (y < nR) { f.R[y] = sum_strided(f.Rp + y, f.stride_r, f.splits_r); continue; }
        y -= nR;
        f.S[y] = sum_strided(f.Sp + y, f.stride_s, f.splits_s);
    }
}

// ------------------------------------------------------------------ checksum GEMM kernel
// The checksum GEMMs of MODE_FT_PRE (the border of C^f = A^c B^r):
//   R   (M x ntn) = op(A)   . [B e_J]_J        (C e for every column tile J)
//   S^T (N x ntm) = op(B)^T . [(e_I^T A)^T]_I  (e^T C for every row tile I)
// i.e. out (P x Q) = X (P x K) . Y (K x Q) with Q = ntn or ntm small and Y = the encode
// vectors (k-contiguous, ld Kp).  A CTA computes 128 rows of P times all QN (>= Q) columns
// over one k-split; split s writes its partial to out + s * split_stride (no atomics: the
// FT_PRE epilogue adds the splits in order, so the result is deterministic).  Same producer /
// TMA / swizzled-fragment machinery as gemm_kernel; the 8 MMA warps form NWM x NWN with
// NWN = QN / 32 (at least 1), so QN = 128 runs the main kernel's 64 x 32 warp tiles (12
// fragment loads per 32 DMMA), QN = 64 32 x 32, QN <= 32 16 x QN.
struct CkArgs {
    const double *X, *Y;
    long long ldx, ldy;
    long long P, Q, K, kper;  // kper: k per split (multiple of BK)
    double *out;
    long long ldo, split_stride;
};

template <int QN>
struct CkPlan {
    static constexpr int B_EL = QN * BK;
    static constexpr int STAGE_EL = TILE_EL + B_EL;
    static constexpr int BYTES = 8 * STAGES * STAGE_EL + 1024;
};

template <bool KCX, bool TMA, int QN>
__global__ void __launch_bounds__(GEMM_THREADS, 1)
    cksum_kernel(const __grid_constant__ CkArgs g, const __grid_constant__ CUtensorMap tmX,
                 const __grid_constant__ CUtensorMap tmY) {
    constexpr int NWN_C = QN >= 32 ? QN / 32 : 1, NWM_C = 8 / NWN_C;
    constexpr int WM_C = BM / NWM_C, WN_C = QN / NWN_C;
    constexpr int FMC = WM_C / 8, FQ = WN_C / 8;
    extern __shared__ __align__(1024) double smem_raw[];
    __shared__ __align__(8) unsigned long long full_bar[STAGES], empty_bar[STAGES];
    double *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u) / 8u;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % NWM_C, wn = warp / NWM_C;
    const long long p0 = (long long)blockIdx.x * BM;
    const long long kbeg = (long long)blockIdx.y * g.kper;
    const long long kend = min(g.K, kbeg + g.kper);
    const int ktiles = kend > kbeg ? (int)((kend - kbeg + BK - 1) / BK) : 0;
    auto sX = [&](int st) { return smem + st * CkPlan<QN>::STAGE_EL; };
    auto sY = [&](int st) { return smem + st * CkPlan<QN>::STAGE_EL + TILE_EL; };
    if (tid == 0) {
        for (int s = 0; s < STAGES; s++) {
            mbar_init(&full_bar[s], 1 + (TMA ? 0 : PRODUCER_THREADS));
            mbar_init(&empty_bar[s], NTHREADS / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    if (warp >= NTHREADS / 32) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(PRODUCER_REGS));
        const int pt = tid - NTHREADS;
        constexpr unsigned TX = TMA ? (TILE_EL + CkPlan<QN>::B_EL) * 8 : 0;
        for (int kt = 0; kt < ktiles; kt++) {
            const int st = kt % STAGES;
            if (kt >= STAGES) mbar_wait(&empty_bar[st], ((kt / STAGES) - 1) & 1);
            const long long k0 = kbeg + (long long)kt * BK;
            if (pt == 0) mbar_arrive_expect_tx(&full_bar[st], TX);
            produce_tile<KCX, TMA>(sX(st), &tmX, &full_bar[st], g.X, g.ldx, p0, k0, g.P, g.K, pt);
            produce_tile<true, TMA, QN>(sY(st), &tmY, &full_bar[st], g.Y, g.ldy, 0, k0, g.Q, g.K, pt);
            if (!TMA) cp_async_mbar_arrive(&full_bar[st]);
            if (TMA && pt != 0) break;  // thread 0 issues every TMA stage
        }
        if (!TMA) cp_wait<0>();
        return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(MMA_REGS));
    double acc[FMC][FQ][2];
#pragma unroll
    for (int a = 0; a < FMC; a++)
#pragma unroll
        for (int b = 0; b < FQ; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
    const FragAddr<KCX> fX(wm * WM_C, lane);
    const FragAddr<true, QN> fY(wn * WN_C, lane);
    auto consume = [&](const int st, const int kt) {
        mbar_wait(&full_bar[st], (kt / STAGES) & 1);
        const double *x_s = sX(st), *y_s = sY(st);
#pragma unroll
        for (int kk = 0; kk < BK / 4; kk++) {
            double xf[FMC], yf[FQ];
#pragma unroll
            for (int f = 0; f < FMC; f++) xf[f] = x_s[fX(f, kk)];
#pragma unroll
            for (int f = 0; f < FQ; f++) yf[f] = y_s[fY(f, kk)];
#pragma unroll
            for (int a = 0; a < FMC; a++)
#pragma unroll
                for (int b = 0; b < FQ; b++) dmma(acc[a][b][0], acc[a][b][1], xf[a], yf[b]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty_bar[st]);
    };
    for (int kt0 = 0; kt0 < ktiles; kt0 += STAGES) {
#pragma unroll
        for (int st = 0; st < STAGES; st++)
            if (kt0 + st < ktiles) consume(st, kt0 + st);
    }
    double *out = g.out + (long long)blockIdx.y * g.split_stride;
#pragma unroll
    for (int a = 0; a < FMC; a++) {
        const long long pi = p0 + frag_mn<KCX>(wm * WM_C, a, lane >> 2);
#pragma unroll
        for (int b = 0; b < FQ; b++)
#pragma unroll
            for (int e = 0; e < 2; e++) {
                const long long q = frag_mn<true>(wn * WN_C, b, 2 * (lane & 3) + e);
                if (pi < g.P && q < g.Q) out[pi + q * g.ldo] = acc[a][b][e];
            }
    }
}

}  // namespace ftb
