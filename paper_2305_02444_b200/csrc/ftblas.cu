// ftblas.cu -- host side of libftblas.so: the C ABI declared in include/ftblas.h.
//
// Argument checking (BLAS xerbla numbering), workspace management, fault-plan
// upload (CSR by verification tile), kernel selection by transpose/alignment,
// launches on the caller's stream, report readback.  All arithmetic of the hot
// path runs in the kernels of ftblas_kernels.cuh.
#include "ftblas_kernels.cuh"
#include "ftblas_ws.cuh"
#include "../../include/ftblas.h"

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <map>
#include <vector>

namespace {

using namespace ftb;

struct DevBuf {
    void *p = nullptr;
    size_t bytes = 0;
    cudaError_t ensure(size_t need) {
        if (need <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, need);
        if (e == cudaSuccess) bytes = need;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
    }
    template <class T> T *as() const { return static_cast<T *>(p); }
};

struct Ctx {
    cudaStream_t stream = nullptr;
    DevBuf ws;            // encode outputs
    DevBuf rep;           // ReportHdr + entries
    long long rep_cap = 1 << 16;
    DevBuf pend;          // PendingHdr + correction candidates of the persistent kernel
    DevBuf encws;         // ftblas_encode_b: per-k-chunk norm partials
    const double *b_enc = nullptr;  // ftblas_set_b_encoding (used by FTBLAS_B_ENCODED calls)
    long long b_enc_N = -1, b_enc_K = -1;
    long long pend_cap = 1 << 16;
    DevBuf plan_dev;      // fault plan: i, j (caller coordinates), bit, CSR offsets by caller tile
    long long plan_version = 0, plan_uploaded = -1;
    void *plan_host = nullptr;  // pinned staging of the plan upload
    size_t plan_host_bytes = 0;
    cudaEvent_t ev_plan = nullptr;
    std::vector<long long> plan_i, plan_j;
    std::vector<int> plan_bit;
    DevBuf hA, hB, hC;    // ftblas_dgemm_host device staging
    cudaStream_t s_up = nullptr, s_down = nullptr;  // ftblas_dgemm_host copy streams
    cudaStream_t s_side = nullptr;                   // checksum GEMM S^T (forked / joined)
    // ftblas_dgemm_host pipeline events: at most HOST_MAX_RB row blocks x HOST_MAX_CB column
    // blocks and HOST_MAX_KP k parts (checked against the block policy before any use)
    static constexpr int HOST_MAX_RB = 4, HOST_MAX_CB = 8, HOST_MAX_BLOCKS = 16, HOST_MAX_KP = 4;
    cudaEvent_t ev_entry = nullptr, ev_exit = nullptr, ev_up[HOST_MAX_CB] = {}, ev_done[HOST_MAX_BLOCKS] = {},
                ev_a[HOST_MAX_RB] = {}, ev_kp[HOST_MAX_CB * HOST_MAX_KP] = {};
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr, ev_switch = nullptr;
    // cached A-side encoding (FTBLAS_REUSE_A_ENCODE)
    struct AKey {
        const void *A; long long lda, M, K; bool kc, a0;
        bool operator==(const AKey &o) const {
            return A == o.A && lda == o.lda && M == o.M && K == o.K && kc == o.kc && a0 == o.a0;
        }
    };
    AKey a_key{};
    bool a_valid = false;
    int a_kch = 1;
    long long ws_gen = 0, a_ws_gen = -1;
    cudaError_t ensure_copy_streams() {
        if (s_up) return cudaSuccess;
        cudaError_t e = cudaStreamCreateWithFlags(&s_up, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s_down, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&s_side, cudaStreamNonBlocking);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_switch, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_entry, cudaEventDisableTiming);
        if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_exit, cudaEventDisableTiming);
        for (cudaEvent_t &x : ev_up) if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
        for (cudaEvent_t &x : ev_done) if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
        for (cudaEvent_t &x : ev_a) if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
        for (cudaEvent_t &x : ev_kp) if (e == cudaSuccess) e = cudaEventCreateWithFlags(&x, cudaEventDisableTiming);
        return e;
    }
    long long launches = 0;
    bool profiling = false, profiling_done = false;
    struct Rec { cudaEvent_t e0, e1, e2; bool ft; };
    std::vector<Rec> recs, pool;
    char err[512] = "no error";
    int checksum_mode = FTBLAS_CHECKSUM_GEMM;
    int tile_policy = FTBLAS_TILES_AUTO;
    long long pair_kmax = 2048;  // FTBLAS_TILES_AUTO: half-tile CTAs for K <= pair_kmax (c1, K = 4096: full 34.1, pair 34.0 TF FT)
    int device = -1;
};
Ctx &ctx() {
    static Ctx c;
    return c;
}

int cuda_fail(cudaError_t e, const char *what) {
    snprintf(ctx().err, sizeof(ctx().err), "%s: %s", what, cudaGetErrorString(e));
    return FTBLAS_ERR_CUDA;
}
int arg_fail(int p, const char *what) {
    snprintf(ctx().err, sizeof(ctx().err), "invalid argument %d: %s", p, what);
    return -p;
}

#define CK(call, what)                                   \
    do {                                                 \
        cudaError_t _e = (call);                         \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

bool trans_ok(char t) { return t == 'N' || t == 'n' || t == 'T' || t == 't' || t == 'C' || t == 'c'; }
bool is_t(char t) { return !(t == 'N' || t == 'n'); }

int check_args(char ta, char tb, long long M, long long N, long long K, const void *A, long long lda,
               const void *B, long long ldb, const void *C, long long ldc, double alpha, double beta) {
    if (!trans_ok(ta)) return arg_fail(1, "transA");
    if (!trans_ok(tb)) return arg_fail(2, "transB");
    if (M < 0) return arg_fail(3, "M < 0");
    if (N < 0) return arg_fail(4, "N < 0");
    if (K < 0) return arg_fail(5, "K < 0");
    const long long nrowa = is_t(ta) ? K : M, nrowb = is_t(tb) ? N : K;
    if (lda < std::max<long long>(1, nrowa)) return arg_fail(8, "lda too small");
    if (ldb < std::max<long long>(1, nrowb)) return arg_fail(10, "ldb too small");
    if (ldc < std::max<long long>(1, M)) return arg_fail(13, "ldc too small");
    if (M > 0 && N > 0 && K > 0 && alpha != 0.0) {
        if (!A) return arg_fail(7, "A is NULL");
        if (!B) return arg_fail(9, "B is NULL");
    }
    if (M > 0 && N > 0 && !C) return arg_fail(12, "C is NULL");
    (void)beta;
    return 0;
}

// tiles = number of 128 x 128 tiles.  NWN = 4: one CTA per tile.  NWN = 2: two CTAs per tile
// (128 x 64 halves, two resident per SM); for FT the halves of a tile form a cluster of 2.
template <bool KCA, bool KCB, bool TMA, int MODE, int NWN>
cudaError_t launch_gemm_t(const GemmArgs &g, const CUtensorMap &ma, const CUtensorMap &mb, long long tiles,
                          cudaStream_t s) {
    auto kern = gemm_kernel<KCA, KCB, TMA, MODE, NWN>;
    const int bytes = SmemPlan<MODE, NWN>::BYTES;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    const unsigned threads = Warps<NWN>::NT + Warps<NWN>::PT;
    if (NWN == 2) {
        e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e != cudaSuccess) return e;
    }
    if (NWN == 2 && MODE != MODE_NOFT) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3((unsigned)(2 * tiles), 1, 1);
        cfg.blockDim = dim3(threads, 1, 1);
        cfg.dynamicSmemBytes = bytes;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, g, ma, mb);
    } else {
        kern<<<(unsigned)(NWN == 2 ? 2 * tiles : tiles), threads, bytes, s>>>(g, ma, mb);
        e = cudaGetLastError();
    }
    ctx().launches++;
    return e;
}

template <int MODE, int NWN>
cudaError_t launch_gemm(bool kca, bool kcb, bool tma, const GemmArgs &g, const CUtensorMap &ma,
                        const CUtensorMap &mb, long long tiles, cudaStream_t s) {
    // 8 instantiations per mode and tile width: transpose layout x (TMA | cp.async fallback)
#define L(a, b, c) if (kca == a && kcb == b && tma == c) return launch_gemm_t<a, b, c, MODE, NWN>(g, ma, mb, tiles, s)
    L(false, true, true); L(false, false, true); L(true, true, true); L(true, false, true);
    L(false, true, false); L(false, false, false); L(true, true, false); L(true, false, false);
#undef L
    return cudaErrorInvalidValue;
}

int sm_count() {
    int dev = 0, n = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
    return n;
}

// Persistent warp-specialized kernel (ftblas_ws.cuh): one CTA per SM over all tiles.
cudaError_t launch_ws_any(const void *kern, GemmArgs g, const CUtensorMap &ma, const CUtensorMap &mb, long long tiles,
                          cudaStream_t s);

template <bool KCA, bool KCB, bool TMA, bool FT>
cudaError_t launch_ws_t(const GemmArgs &g, const CUtensorMap &ma, const CUtensorMap &mb, long long tiles,
                        cudaStream_t s) {
    return launch_ws_any(reinterpret_cast<const void *>(gemm_ws_kernel<KCA, KCB, TMA, FT>), g, ma, mb, tiles, s);
}

template <bool FT>
cudaError_t launch_ws(bool kca, bool kcb, bool tma, const GemmArgs &g, const CUtensorMap &ma, const CUtensorMap &mb,
                      long long tiles, cudaStream_t s) {
#define L(a, b, c) if (kca == a && kcb == b && tma == c) return launch_ws_t<a, b, c, FT>(g, ma, mb, tiles, s)
    L(false, true, true); L(false, false, true); L(true, true, true); L(true, false, true);
    L(false, true, false); L(false, false, false); L(true, true, false); L(true, false, false);
#undef L
    return cudaErrorInvalidValue;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda link)
using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn encode_tiled() {
    static EncodeTiledFn fn = [] {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            p = nullptr;
        return reinterpret_cast<EncodeTiledFn>(p);
    }();
    return fn;
}

// Tensor map of one operand, as gemm_kernel stages it (ftblas_kernels.cuh, Tile): KC=false
// (mn contiguous): dims {MNd, Kd}, box {16, BK}; KC=true (k contiguous): dims {Kd, MNd}, box
// {16, 128}.  128-byte swizzle, zero fill out of bounds.  Returns false when TMA cannot
// describe the operand (the kernel then stages it with cp.async).
bool make_operand_map(CUtensorMap *m, const double *X, long long ld, long long MNd, long long Kd, bool kc,
                      unsigned rows = 128) {
    std::memset(m, 0, sizeof(*m));
    EncodeTiledFn fn = encode_tiled();
    if (!fn || !X || MNd <= 0 || Kd <= 0 || (reinterpret_cast<uintptr_t>(X) & 15) || (ld & 1)) return false;
    if (MNd >= (1ll << 31) || Kd >= (1ll << 31)) return false;
    const cuuint64_t dims[2] = {(cuuint64_t)(kc ? Kd : MNd), (cuuint64_t)(kc ? MNd : Kd)};
    const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
    const cuuint32_t box[2] = {16u, kc ? (cuuint32_t)rows : (cuuint32_t)BK};
    const cuuint32_t estr[2] = {1u, 1u};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(X), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

cudaError_t launch_ws_any(const void *kern, GemmArgs g, const CUtensorMap &ma, const CUtensorMap &mb, long long tiles,
                          cudaStream_t s) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, WS_SMEM);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)std::min<long long>(tiles, sm_count());
    void *args[] = {&g, const_cast<CUtensorMap *>(&ma), const_cast<CUtensorMap *>(&mb)};
    e = cudaLaunchKernel(kern, dim3(grid), dim3(WS_THREADS), args, WS_SMEM, s);
    ctx().launches++;
    return e;
}

bool vec_ok(const void *p, long long ld) {
    return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && (ld % 2 == 0);
}

// Upload the fault plan once per plan version, in the caller's coordinates: CSR by the
// caller's 128 x 128 tile (index gtn * plan_ntm + gtm over the grid that covers every planned
// element).  A call on the block at (off_i, off_j) looks its tiles up at (tm + off_i / 128,
// tn + off_j / 128), so blocked / chunked callers share one upload.  The copy is stream-ordered
// from a pinned staging buffer (no host stall); the staging buffer is rewritten only after the
// previous upload has completed (ev_plan).
int prepare_plan(GemmArgs &g) {
    Ctx &c = ctx();
    g.plan_ptr = nullptr; g.plan_i = nullptr; g.plan_j = nullptr; g.plan_bit = nullptr;
    g.plan_ntm = 0; g.plan_ntn = 0;
    if (c.plan_i.empty()) return 0;
    const size_t n = c.plan_i.size();
    const size_t bytes_ij = n * sizeof(long long), bytes_b = (n * sizeof(int) + 15) / 16 * 16;
    long long ntm = 1, ntn = 1;
    for (size_t f = 0; f < n; f++) {
        ntm = std::max(ntm, c.plan_i[f] / BM + 1);
        ntn = std::max(ntn, c.plan_j[f] / BN + 1);
    }
    const long long nt = ntm * ntn;
    const size_t bytes_ptr = (size_t)(nt + 1) * sizeof(int);
    const size_t total = 2 * bytes_ij + bytes_b + bytes_ptr;
    if (c.plan_uploaded != c.plan_version) {
        std::vector<int> cnt(nt + 1, 0);
        for (size_t f = 0; f < n; f++) cnt[(c.plan_j[f] / BN) * ntm + c.plan_i[f] / BM + 1]++;
        for (long long t = 0; t < nt; t++) cnt[t + 1] += cnt[t];
        if (c.ev_plan) CK(cudaEventSynchronize(c.ev_plan), "plan staging reuse");
        else CK(cudaEventCreateWithFlags(&c.ev_plan, cudaEventDisableTiming), "event");
        if (c.plan_host_bytes < total) {
            if (c.plan_host) cudaFreeHost(c.plan_host);
            c.plan_host = nullptr; c.plan_host_bytes = 0;
            CK(cudaHostAlloc(&c.plan_host, total, cudaHostAllocDefault), "cudaHostAlloc(plan)");
            c.plan_host_bytes = total;
        }
        char *h = static_cast<char *>(c.plan_host);
        long long *pi = reinterpret_cast<long long *>(h), *pj = reinterpret_cast<long long *>(h + bytes_ij);
        int *pb = reinterpret_cast<int *>(h + 2 * bytes_ij);
        std::memcpy(h + 2 * bytes_ij + bytes_b, cnt.data(), bytes_ptr);
        std::vector<int> fill(cnt.begin(), cnt.end() - 1);
        for (size_t f = 0; f < n; f++) {
            const int pos = fill[(c.plan_j[f] / BN) * ntm + c.plan_i[f] / BM]++;
            pi[pos] = c.plan_i[f]; pj[pos] = c.plan_j[f]; pb[pos] = c.plan_bit[f];
        }
        CK(c.plan_dev.ensure(total), "cudaMalloc(plan)");
        CK(cudaMemcpyAsync(c.plan_dev.p, h, total, cudaMemcpyHostToDevice, c.stream), "plan upload");
        CK(cudaEventRecord(c.ev_plan, c.stream), "event");
        c.plan_uploaded = c.plan_version;
    }
    char *base = c.plan_dev.as<char>();
    g.plan_i = reinterpret_cast<const long long *>(base);
    g.plan_j = reinterpret_cast<const long long *>(base + bytes_ij);
    g.plan_bit = reinterpret_cast<const int *>(base + 2 * bytes_ij);
    g.plan_ptr = reinterpret_cast<const int *>(base + 2 * bytes_ij + bytes_b);
    g.plan_ntm = ntm; g.plan_ntn = ntn;
    return 0;
}

cudaEvent_t new_event() {
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
}
Ctx::Rec take_rec(bool ft) {
    Ctx &c = ctx();
    Ctx::Rec r;
    if (!c.pool.empty()) { r = c.pool.back(); c.pool.pop_back(); }
    else { r.e0 = new_event(); r.e1 = new_event(); r.e2 = new_event(); }
    r.ft = ft;
    return r;
}

int fetch_report(ftblas_err_report *r) {
    Ctx &c = ctx();
    CK(cudaStreamSynchronize(c.stream), "report sync");
    ReportHdr h{};
    if (c.rep.p) CK(cudaMemcpy(&h, c.rep.p, sizeof(h), cudaMemcpyDeviceToHost), "report header");
    r->count = (int64_t)h.count;
    r->tiles_flagged = (int64_t)h.tiles_flagged;
    r->rows_flagged = (int64_t)h.rows_flagged;
    r->cols_flagged = (int64_t)h.cols_flagged;
    const long long n = std::min<long long>({(long long)h.count, (long long)r->capacity, c.rep_cap});
    if (n > 0 && r->entries)
        CK(cudaMemcpy(r->entries, c.rep.as<char>() + sizeof(ReportHdr), n * sizeof(Correction),
                      cudaMemcpyDeviceToHost), "report entries");
    return 0;
}

// Operand staging for one GEMM call: tensor maps when both operands can be described by
// TMA (16-byte aligned, even ld), else the cp.async fallback for both.
struct Staging {
    CUtensorMap ma, mb;
    bool tma;
};
Staging make_staging(const double *A, long long lda, long long M, bool kca, const double *B, long long ldb,
                     long long N, bool kcb, long long K, double alpha, unsigned brows = 128) {
    Staging st;
    const bool use = K > 0 && alpha != 0.0;
    const bool ta = use && make_operand_map(&st.ma, A, lda, M, K, kca);
    const bool tb = use && make_operand_map(&st.mb, B, ldb, N, K, kcb, brows);
    st.tma = ta && tb;
    if (!st.tma) { std::memset(&st.ma, 0, sizeof(st.ma)); std::memset(&st.mb, 0, sizeof(st.mb)); }
    return st;
}

template <bool KCX, bool TMA, int QN>
cudaError_t launch_cksum_t(const CkArgs &a, const CUtensorMap &mx, const CUtensorMap &my, dim3 grid, cudaStream_t s) {
    auto kern = cksum_kernel<KCX, TMA, QN>;
    const int bytes = CkPlan<QN>::BYTES;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e != cudaSuccess) return e;
    kern<<<grid, GEMM_THREADS, bytes, s>>>(a, mx, my);
    ctx().launches++;
    return cudaGetLastError();
}

// Split count of a checksum GEMM with `tiles` 128-row tiles: about four waves of CTAs in
// total, at least one BK slice per split.
void cksum_split(long long tiles, long long K, long long Q, long long &splits, long long &kper) {
    const long long kt = std::max<long long>(1, (K + BK - 1) / BK);
    // about 4 waves of CTAs, but the k-split partials (splits x P x Q doubles, written and
    // re-read) at most 1/8 of the operand bytes (P x K): c2 (Q = 128, K = 256) -> 1 split,
    // c1 (Q = 32, K = 4096) -> 16, c3 -> 5
    const long long cap = std::max<long long>(1, K / (8 * std::max<long long>(1, Q)));
    splits = std::max<long long>(1, std::min<long long>({kt, cap, (4 * 148 + tiles - 1) / tiles}));
    kper = (kt + splits - 1) / splits * BK;
    splits = (K + kper - 1) / kper;
}

// Checksum GEMM out (P x Q, ld P, k-split partials at out + s * split_stride) = op(X) (P x K) .
// Y (K x Q; Y(k, q) = Y[q * ldy + k]) for Q <= 128 (the caller splits wider Q).
cudaError_t cksum_gemm(bool kcx, const double *X, long long ldx, long long P, const double *Y, long long ldy,
                       long long Q, long long K, long long splits, long long kper, double *out,
                       long long split_stride, cudaStream_t s) {
    CkArgs a{};
    a.X = X; a.Y = Y; a.ldx = ldx; a.ldy = ldy; a.P = P; a.Q = Q; a.K = K; a.kper = kper;
    a.out = out; a.ldo = P; a.split_stride = split_stride;
    Staging st;
    const bool tx = make_operand_map(&st.ma, X, ldx, P, K, kcx);
    const int qn = Q <= 16 ? 16 : Q <= 32 ? 32 : Q <= 64 ? 64 : 128;
    bool ty = false;
    if (tx) {  // Y: k-contiguous, box {16, QN} (rows >= Q zero-filled)
        std::memset(&st.mb, 0, sizeof(st.mb));
        EncodeTiledFn fn = encode_tiled();
        const cuuint64_t dims[2] = {(cuuint64_t)K, (cuuint64_t)Q};
        const cuuint64_t strides[1] = {(cuuint64_t)ldy * 8};
        const cuuint32_t box[2] = {16u, (cuuint32_t)qn};
        const cuuint32_t estr[2] = {1u, 1u};
        ty = fn && (reinterpret_cast<uintptr_t>(Y) & 15) == 0 && (ldy & 1) == 0 &&
             fn(&st.mb, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double *>(Y), dims, strides, box, estr,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
    }
    const bool tma = tx && ty;
    if (!tma) { std::memset(&st.ma, 0, sizeof(st.ma)); std::memset(&st.mb, 0, sizeof(st.mb)); }
    const dim3 grid((unsigned)((P + BM - 1) / BM), (unsigned)splits, 1);
#define L(x, t, q) if (kcx == x && tma == t && qn == q) return launch_cksum_t<x, t, q>(a, st.ma, st.mb, grid, s)
    L(false, true, 16); L(false, true, 32); L(false, true, 64); L(false, true, 128);
    L(true, true, 16); L(true, true, 32); L(true, true, 64); L(true, true, 128);
    L(false, false, 16); L(false, false, 32); L(false, false, 64); L(false, false, 128);
    L(true, false, 16); L(true, false, 32); L(true, false, 64); L(true, false, 128);
#undef L
    return cudaErrorInvalidValue;
}

// Layout of a finalized op(B) encoding (ftblas_encode_b; doubles, sections 16-byte aligned):
// [0, oN): WB, ceil(N/128) rows of Kp (w_J = op(B) e_J, zero for k >= K); [oN, oN + N): the
// column 1-norms ||op(B)(:, j)||_1; [oM, oM + ceil(N/128)): the tile maxima max_k sum_j |op(B)(k, j)|.
void b_layout(long long N, long long K, long long &oN, long long &oM, long long &total) {
    const long long Kp = std::max<long long>(BK, (K + BK - 1) / BK * BK), ntn = (N + BN - 1) / BN;
    auto al = [](long long n) { return (n + 1) / 2 * 2; };
    oN = al(ntn * Kp);
    oM = oN + al(N);
    total = oM + al(ntn);
}

cudaError_t launch_encode(int p0, int p1, dim3 grid, const EncodeArgs &ea, cudaStream_t s) {
#define L(x, y) if (p0 == x && p1 == y) { encode_kernel<x, y><<<grid, NTHREADS, 0, s>>>(ea); return cudaGetLastError(); }
    L(0, 0) L(0, 1) L(0, 2) L(1, 0) L(1, 1) L(1, 2) L(2, 0) L(2, 1) L(2, 2)
#undef L
    return cudaErrorInvalidValue;
}

int dgemm_impl(bool ft, char ta, char tb, long long M, long long N, long long K, double alpha,
               const double *A, long long lda, const double *B, long long ldb, double beta, double *C,
               long long ldc, ftblas_err_report *rep, long long off_i = 0, long long off_j = 0,
               bool append = false, bool reuse_a = false, bool inject = true, const double *benc = nullptr) {
    static_assert(sizeof(Correction) == sizeof(ftblas_correction), "ABI");
    Ctx &c = ctx();
    int rc = check_args(ta, tb, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta);
    if (rc) return rc;
    if (ft) {
        CK(c.rep.ensure(sizeof(ReportHdr) + c.rep_cap * sizeof(Correction)), "cudaMalloc(report)");
        CK(c.pend.ensure(sizeof(Pending) + c.pend_cap * sizeof(Pending)), "cudaMalloc(pending)");
    }
    if (M == 0 || N == 0) {
        if (ft && !append) CK(cudaMemsetAsync(c.rep.p, 0, sizeof(ReportHdr), c.stream), "report reset");
        return rep ? fetch_report(rep) : 0;
    }
    const bool kca = is_t(ta), kcb = !is_t(tb);
    const long long ntm = (M + BM - 1) / BM, ntn = (N + BN - 1) / BN;
    GemmArgs g{};
    g.A = A; g.B = B; g.C = C; g.lda = lda; g.ldb = ldb; g.ldc = ldc;
    g.M = M; g.N = N; g.K = K; g.alpha = alpha; g.beta = beta;
    const bool va = vec_ok(A, lda), vb = vec_ok(B, ldb);
    g.vecC = vec_ok(C, ldc) ? 1 : 0;  // 16-byte C0 staging / stores in every mode
    // tile policy: 128 x 64 half-tile CTAs (2 per SM, epilogue of one overlapping the mainloop of
    // the other) when the per-tile mainloop is short, 128 x 128 CTAs otherwise; the fused
    // checksum mode always uses 128 x 128
    const bool fused = ft && c.checksum_mode == FTBLAS_CHECKSUM_FUSED;
    // AUTO, FT calls with a short mainloop per tile (K <= pair_kmax): the persistent kernel, whose
    // MMA warps do the epilogue arithmetic in registers and whose epilogue warps overlap C
    // traffic and location with the next tile (c2: 4.47 ms vs 4.79 ms for pair tiles); non-FT
    // calls there keep the pair tiles (4.02 vs 4.10 ms)
    // (at least one wave of tiles: on a handful of tiles the persistent kernel's prologue is not
    // amortized, c0 256^3: 0.42 vs 0.59 TFLOP/s)
    const bool ws = !fused && (c.tile_policy == FTBLAS_TILES_WS ||
                               (ft && c.tile_policy == FTBLAS_TILES_AUTO && K <= c.pair_kmax &&
                                ntm * ntn >= sm_count()));
    const bool pair = !fused && !ws && (c.tile_policy == FTBLAS_TILES_PAIR ||
                                        (c.tile_policy == FTBLAS_TILES_AUTO && K <= c.pair_kmax));
    const Staging stg = make_staging(A, lda, M, kca, B, ldb, N, kcb, K, alpha, pair ? 64u : 128u);
    Ctx::Rec rec{};
    if (c.profiling) {
        rec = take_rec(ft);
        CK(cudaEventRecord(rec.e0, c.stream), "event");
    }
    if (ft) {
        const long long Kp = std::max<long long>(BK, (K + BK - 1) / BK * BK);
        // k-chunks of the encode pass: about eight waves of blocks (two resident per SM), so the
        // last partial wave costs little; chunks >= 128 columns; at most 32 partials per row (the
        // GEMM producer reduces them per tile)
        long long kch_l = (8 * 2 * 148 + ntm + ntn - 1) / (ntm + ntn);
        kch_l = std::min<long long>({kch_l, 32, std::max<long long>(1, Kp / 128)});
        int kch = (int)std::max<long long>(1, kch_l);
        // FTBLAS_REUSE_A_ENCODE: the caller promises op(A) is unchanged since the previous call
        // on the same A (the blocks of a chunked call); its encoding is reused when the cached
        // key matches and the workspace was not reallocated, else A is encoded as usual.
        const Ctx::AKey akey{A, lda, M, K, kca, alpha == 0.0};
        bool skip_a = reuse_a && c.a_valid && c.a_key == akey && c.a_ws_gen == c.ws_gen;
        const bool pre = c.checksum_mode == FTBLAS_CHECKSUM_GEMM;
        long long spR = 1, kpR = Kp, spS = 1, kpS = Kp;
        if (pre) {
            cksum_split(ntm * ((ntn + 127) / 128), K, std::min<long long>(ntn, 128), spR, kpR);
            cksum_split(ntn * ((ntm + 127) / 128), K, std::min<long long>(ntm, 128), spS, kpS);
        }
        // workspace: A side first (VA, lineA, tmaxA: independent of N, so a chunked caller can
        // reuse them), then the B side, then the checksum-GEMM partials
        // (every sub-array starts on a 128-byte boundary: bulk copies and TMA need >= 16 B)
        auto al = [](size_t n) { return (n + 15) / 16 * 16; };
        size_t oLA, oTA, oWB, oLB, oTB, oR, oS, oF, nF, need;
        auto layout = [&](int kc) {
            oLA = al((size_t)ntm * Kp); oTA = oLA + al((size_t)kc * M); oWB = oTA + al((size_t)kc * ntm);
            oLB = oWB + al((size_t)ntn * Kp); oTB = oLB + al((size_t)kc * N); oR = oTB + al((size_t)kc * ntn);
            oS = oR + (pre ? al((size_t)spR * ntn * M) : 0);
            oF = oS + (pre ? al((size_t)spS * ntm * N) : 0);  // finalized side data
            nF = pre ? (size_t)(M + N + ntm + ntn) + (size_t)ntn * M + (size_t)ntm * N : 0;
            need = (oF + nF) * sizeof(double);
        };
        layout(skip_a ? c.a_kch : kch);
        if (skip_a && need > c.ws.bytes) {
            // the workspace grows (free + malloc): the cached A encoding does not survive it,
            // so A is encoded again with this call's own chunk count
            skip_a = false;
            layout(kch);
        }
        if (skip_a) kch = c.a_kch;
        const long long kper = ((Kp + kch - 1) / kch + 31) / 32 * 32;
        const size_t nRS = pre ? (size_t)spR * ntn * M + (size_t)spS * ntm * N : 0;
        if (need > c.ws.bytes) c.ws_gen++;
        CK(c.ws.ensure(need), "cudaMalloc(workspace)");
        double *w = c.ws.as<double>();
        g.VA = w;
        double *lineA = w + oLA, *tmaxA = w + oTA;
        g.WB = w + oWB;
        double *lineB = w + oLB, *tmaxB = w + oTB;
        // FTBLAS_B_ENCODED: op(B)'s finalized encoding (ftblas_encode_b, e.g. assembled from the
        // slices that the ranks of a sharded product encoded) replaces the B side of the encode pass
        const bool ext_b = benc != nullptr && K > 0 && alpha != 0.0;
        int kchB = kch;
        if (ext_b) {
            long long oN, oM, tot;
            b_layout(N, K, oN, oM, tot);
            g.WB = benc;
            lineB = const_cast<double *>(benc) + oN;
            tmaxB = const_cast<double *>(benc) + oM;
            kchB = 1;
        }
        g.lineA = lineA; g.lineB = lineB; g.tmaxA = tmaxA; g.tmaxB = tmaxB;
        g.kch = kch; g.kchB = kchB; g.Kp = Kp;
        double *Rpre = w + oR, *Spre = w + oS;
        double *fin = w + oF;
        g.fin_nrmA = fin; g.fin_nrmB = fin + M; g.fin_maxA = fin + M + N; g.fin_maxB = fin + M + N + ntm;
        // one k-split each: the checksum GEMM outputs are final, the pair tiles read them in place
        const bool rs_final = spR == 1 && spS == 1;
        g.fin_R = rs_final ? Rpre : fin + M + N + ntm + ntn;
        g.fin_S = rs_final ? Spre : g.fin_R + (size_t)ntn * M;
        g.Rpre = pre ? Rpre : nullptr;
        g.Spre = pre ? Spre : nullptr;
        g.splits_r = (int)spR; g.splits_s = (int)spS;
        g.stride_r = ntn * M; g.stride_s = ntm * N;
        g.rep = c.rep.as<ReportHdr>();
        g.rep_entries = reinterpret_cast<Correction *>(c.rep.as<char>() + sizeof(ReportHdr));
        g.rep_cap = c.rep_cap;
        g.pend = c.pend.as<PendingHdr>();
        g.pend_entries = reinterpret_cast<Pending *>(c.pend.as<char>() + sizeof(Pending));
        g.pend_cap = c.pend_cap;
        g.vecC = vec_ok(C, ldc) ? 1 : 0;
        g.off_i = off_i; g.off_j = off_j;
        if (inject) {
            rc = prepare_plan(g);
            if (rc) return rc;
        }
        EncodeArgs ea{};
        const EncodeOperand opA{A, lda, M, kca ? 1 : 0, va ? 1 : 0, const_cast<double *>(g.VA), lineA, tmaxA, (int)ntm};
        const EncodeOperand opB{B, ldb, N, kcb ? 1 : 0, vb ? 1 : 0, const_cast<double *>(g.WB), lineB, tmaxB, (int)ntn};
        int nops = 0;
        if (!skip_a) ea.op[nops++] = opA;
        if (!ext_b) ea.op[nops++] = opB;
        ea.K = (alpha == 0.0) ? 0 : K;  // alpha == 0: A, B are not read (encodes are zero)
        ea.Kp = Kp; ea.kper = kper; ea.kch = kch; ea.rep = append ? nullptr : g.rep;
        ea.pend = g.pend;
        // one launch (encode_kernel<PATH0, PATH1>: operand z along its own layout path), which
        // also zeroes the report (unless appending) and the candidate list
        {
            if (nops == 0) {  // nothing to encode: the report and candidate list are cleared here
                if (!append) CK(cudaMemsetAsync(g.rep, 0, sizeof(ReportHdr), c.stream), "report reset");
                CK(cudaMemsetAsync(g.pend, 0, sizeof(PendingHdr), c.stream), "pending reset");
            }
            auto path_of = [](const EncodeOperand &o) { return o.kc ? 0 : (o.vec ? 1 : 2); };
            if (nops > 0) {
                // one launch for both operands (blockIdx.z), each along its own layout path
                long long tiles = 0;
                for (int q = 0; q < nops; q++) tiles = std::max<long long>(tiles, ea.op[q].ntiles);
                ea.op_base = 0;
                const dim3 grid((unsigned)tiles, (unsigned)kch, (unsigned)nops);
                const int p0 = path_of(ea.op[0]), p1 = path_of(ea.op[nops - 1]);
                CK(launch_encode(p0, p1, grid, ea, c.stream), "encode_kernel launch");
                c.launches++;
            }
        }
        if (!skip_a) {
            c.a_valid = true; c.a_key = akey; c.a_kch = kch; c.a_ws_gen = c.ws_gen;
        }
        if (pre && K > 0 && alpha != 0.0) {
            // checksum GEMMs (the border of C^f = A^c B^r) on the FP64
            // tensor cores:  R (M x ntn, ld M)   = op(A) . WB^T   [WB^T: k x ntn, 'N', ld Kp]
            //                S^T (N x ntm, ld N) = op(B)^T . VA^T [VA^T: k x ntm, 'N', ld Kp]
            // (column blocks of <= 128 tiles; k-split partials summed in the FT_PRE epilogue)
            // R on the library stream and S^T on a forked side stream run concurrently (their
            // CTAs share the waves), joined before the main GEMM
            CK(c.ensure_copy_streams(), "streams");
            CK(cudaEventRecord(c.ev_fork, c.stream), "event");
            CK(cudaStreamWaitEvent(c.s_side, c.ev_fork, 0), "wait");
            for (long long q0 = 0; q0 < ntn; q0 += 128)
                CK(cksum_gemm(kca, A, lda, M, g.WB + q0 * Kp, Kp, std::min<long long>(128, ntn - q0), K, spR, kpR,
                              Rpre + q0 * M, ntn * M, c.stream), "checksum GEMM R");
            for (long long q0 = 0; q0 < ntm; q0 += 128)
                CK(cksum_gemm(kcb, B, ldb, N, g.VA + q0 * Kp, Kp, std::min<long long>(128, ntm - q0), K, spS, kpS,
                              Spre + q0 * N, ntm * N, c.s_side), "checksum GEMM S");
            CK(cudaEventRecord(c.ev_join, c.s_side), "event");
            CK(cudaStreamWaitEvent(c.stream, c.ev_join, 0), "wait");
        } else if (pre) {
            CK(cudaMemsetAsync(Rpre, 0, (oS - oR + (size_t)spS * ntm * N) * sizeof(double), c.stream), "checksum zero");
            (void)nRS;
        }
        if (pre && (pair || ws)) {
            // per-row / per-column side data of the verification: partials summed once (the
            // pair-tile producers and the persistent kernel's epilogue warps copy them: an FP64
            // add issued by an epilogue warp beside the DMMA stream waits ~1000 cycles for the
            // pipe, 32 of them per tile made the epilogue warps the bottleneck at K = 256;
            // 128 x 128 tiles sum the partials in the producer)
            FinArgs fa{};
            fa.lineA = lineA; fa.lineB = lineB; fa.tmaxA = tmaxA; fa.tmaxB = tmaxB;
            fa.Rp = rs_final ? nullptr : Rpre; fa.Sp = rs_final ? nullptr : Spre;  // nullptr: nothing to sum
            fa.M = M; fa.N = N; fa.ntm = ntm; fa.ntn = ntn; fa.stride_r = g.stride_r; fa.stride_s = g.stride_s;
            fa.kch = kch; fa.kchB = kchB; fa.splits_r = (int)spR; fa.splits_s = (int)spS;
            fa.nrmA = fin; fa.nrmB = fin + M; fa.maxA = fin + M + N; fa.maxB = fin + M + N + ntm;
            fa.R = fin + M + N + ntm + ntn; fa.S = fa.R + (size_t)ntn * M;
            const long long total = (long long)(M + N + ntm + ntn) + (rs_final ? 0 : (long long)ntn * M + (long long)ntm * N);
            const unsigned blocks = (unsigned)std::min<long long>((total + 255) / 256, 8 * 148);
            side_finalize_kernel<<<blocks, 256, 0, c.stream>>>(fa);
            c.launches++;
            CK(cudaGetLastError(), "side_finalize_kernel launch");
        }
        if (c.profiling) CK(cudaEventRecord(rec.e1, c.stream), "event");
        if (pre && ws)
            CK((launch_ws<true>(kca, kcb, stg.tma, g, stg.ma, stg.mb, ntm * ntn, c.stream)), "gemm_ws_kernel<FT> launch");
        else if (pre)
            CK((pair ? launch_gemm<MODE_FT_PRE, 2>(kca, kcb, stg.tma, g, stg.ma, stg.mb, ntm * ntn, c.stream)
                     : launch_gemm<MODE_FT_PRE, 4>(kca, kcb, stg.tma, g, stg.ma, stg.mb, ntm * ntn, c.stream)),
               "gemm_kernel<FT> launch");
        else
            CK((launch_gemm<MODE_FT_FUSED, 4>(kca, kcb, stg.tma, g, stg.ma, stg.mb, ntm * ntn, c.stream)),
               "gemm_kernel<FT> launch");
        if (c.profiling) {
            CK(cudaEventRecord(rec.e2, c.stream), "event");
            c.recs.push_back(rec);
            c.profiling_done = true;
        }
        // the located candidates of every kernel: recomputed from the definition and corrected
        // after the GEMM (correct_kernel, ftblas_ws.cuh); exits at once when there are none
        const unsigned cb = (unsigned)sm_count();
        if (!kca && kcb) correct_kernel<false, true><<<cb, CORR_THREADS, 0, c.stream>>>(g);
        else if (!kca && !kcb) correct_kernel<false, false><<<cb, CORR_THREADS, 0, c.stream>>>(g);
        else if (kca && kcb) correct_kernel<true, true><<<cb, CORR_THREADS, 0, c.stream>>>(g);
        else correct_kernel<true, false><<<cb, CORR_THREADS, 0, c.stream>>>(g);
        c.launches++;
        CK(cudaGetLastError(), "correct_kernel launch");
    } else {
        if (c.profiling) CK(cudaEventRecord(rec.e1, c.stream), "event");
        if (ws)
            CK((launch_ws<false>(kca, kcb, stg.tma, g, stg.ma, stg.mb, ntm * ntn, c.stream)), "gemm_ws_kernel launch");
        else
            CK((pair ? launch_gemm<MODE_NOFT, 2>(kca, kcb, stg.tma, g, stg.ma, stg.mb, ntm * ntn, c.stream)
                     : launch_gemm<MODE_NOFT, 4>(kca, kcb, stg.tma, g, stg.ma, stg.mb, ntm * ntn, c.stream)),
               "gemm_kernel launch");
    }
    if (c.profiling && !c.profiling_done) {
        CK(cudaEventRecord(rec.e2, c.stream), "event");
        c.recs.push_back(rec);
    }
    c.profiling_done = false;
    if (rep) return fetch_report(rep);
    return 0;
}

}  // namespace

extern "C" {

int ftblas_dgemm(char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                 int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
                 ftblas_err_report *err_report) {
    return dgemm_impl(true, transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, err_report);
}

int ftblas_dgemm_ex(char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                    int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
                    int64_t row_offset, int64_t col_offset, int32_t flags, ftblas_err_report *err_report) {
    if (row_offset < 0 || row_offset % FTBLAS_TILE_M) return arg_fail(14, "row_offset not a multiple of the tile");
    if (col_offset < 0 || col_offset % FTBLAS_TILE_N) return arg_fail(15, "col_offset not a multiple of the tile");
    if (flags & ~(FTBLAS_REPORT_APPEND | FTBLAS_REUSE_A_ENCODE | FTBLAS_B_ENCODED)) return arg_fail(16, "unknown flags");
    const double *benc = nullptr;
    if (flags & FTBLAS_B_ENCODED) {
        const Ctx &c = ctx();
        if (!c.b_enc || c.b_enc_N != N || c.b_enc_K != K)
            return arg_fail(16, "FTBLAS_B_ENCODED without a matching ftblas_set_b_encoding");
        benc = c.b_enc;
    }
    return dgemm_impl(true, transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, err_report, row_offset,
                      col_offset, (flags & FTBLAS_REPORT_APPEND) != 0, (flags & FTBLAS_REUSE_A_ENCODE) != 0, true,
                      benc);
}

int64_t ftblas_b_encoding_len(int64_t N, int64_t K) {
    if (N < 0 || K < 0) return -1;
    long long oN, oM, total;
    b_layout(N, K, oN, oM, total);
    return total;
}

int ftblas_b_encoding_layout(int64_t N, int64_t K, int64_t *off_nrm, int64_t *off_max, int64_t *total) {
    if (N < 0) return arg_fail(1, "N < 0");
    if (K < 0) return arg_fail(2, "K < 0");
    long long oN, oM, t;
    b_layout(N, K, oN, oM, t);
    if (off_nrm) *off_nrm = oN;
    if (off_max) *off_max = oM;
    if (total) *total = t;
    return 0;
}

int ftblas_encode_b(char transB, int64_t N, int64_t K, const double *B, int64_t ldb, double *enc) {
    Ctx &c = ctx();
    if (!trans_ok(transB)) return arg_fail(1, "transB");
    if (N < 0) return arg_fail(2, "N < 0");
    if (K < 0) return arg_fail(3, "K < 0");
    const bool kcb = !is_t(transB);
    if (ldb < std::max<long long>(1, is_t(transB) ? N : K)) return arg_fail(5, "ldb too small");
    if (N > 0 && K > 0 && !B) return arg_fail(4, "B is NULL");
    if (N > 0 && !enc) return arg_fail(6, "enc is NULL");
    if (N == 0) return 0;
    long long oN, oM, total;
    b_layout(N, K, oN, oM, total);
    if (K == 0) {  // empty inner dimension: every sum is zero
        CK(cudaMemsetAsync(enc, 0, (size_t)total * sizeof(double), c.stream), "encoding zero");
        return 0;
    }
    const long long Kp = std::max<long long>(BK, (K + BK - 1) / BK * BK), ntn = (N + BN - 1) / BN;
    long long kch_l = (8 * 2 * 148 + ntn - 1) / ntn;
    const int kch = (int)std::max<long long>(1, std::min<long long>({kch_l, 32, std::max<long long>(1, Kp / 128)}));
    const long long kper = ((Kp + kch - 1) / kch + 31) / 32 * 32;
    // per-k-chunk partials of the norms, summed into the encoding by side_finalize_kernel
    const size_t nl = ((size_t)kch * N + 1) / 2 * 2, nt = ((size_t)kch * ntn + 1) / 2 * 2;
    CK(c.encws.ensure((nl + nt) * sizeof(double)), "cudaMalloc(encode workspace)");
    double *line = c.encws.as<double>(), *tmax = line + nl;
    EncodeArgs ea{};
    ea.op[0] = EncodeOperand{B, ldb, N, kcb ? 1 : 0, vec_ok(B, ldb) ? 1 : 0, enc, line, tmax, (int)ntn};
    ea.K = K; ea.Kp = Kp; ea.kper = kper; ea.kch = kch; ea.rep = nullptr; ea.pend = nullptr; ea.op_base = 0;
    const dim3 grid((unsigned)ntn, (unsigned)kch, 1u);
    const int path = ea.op[0].kc ? 0 : (ea.op[0].vec ? 1 : 2);
    CK(launch_encode(path, path, grid, ea, c.stream), "encode_kernel launch");
    c.launches++;
    FinArgs fa{};
    fa.lineB = line; fa.tmaxB = tmax; fa.N = N; fa.ntn = ntn; fa.kch = kch; fa.kchB = kch;
    fa.nrmB = enc + oN; fa.maxB = enc + oM;
    const unsigned blocks = (unsigned)std::min<long long>((N + ntn + 255) / 256, 8 * 148);
    side_finalize_kernel<<<blocks, 256, 0, c.stream>>>(fa);
    c.launches++;
    CK(cudaGetLastError(), "side_finalize_kernel launch");
    return 0;
}

int ftblas_set_b_encoding(const double *enc, int64_t N, int64_t K) {
    Ctx &c = ctx();
    if (enc && (N < 0 || K < 0)) return arg_fail(2, "N or K < 0");
    c.b_enc = enc;
    c.b_enc_N = enc ? N : -1;
    c.b_enc_K = enc ? K : -1;
    return 0;
}

int ftblas_report_reset(void) {
    Ctx &c = ctx();
    CK(c.rep.ensure(sizeof(ReportHdr) + c.rep_cap * sizeof(Correction)), "cudaMalloc(report)");
    CK(cudaMemsetAsync(c.rep.p, 0, sizeof(ReportHdr), c.stream), "report reset");
    return 0;
}

int ftblas_dgemm_noft(char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                      int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc) {
    return dgemm_impl(false, transA, transB, M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, nullptr);
}

int ftblas_dgemm_host(char transA, char transB, int64_t M, int64_t N, int64_t K, double alpha, const double *A,
                      int64_t lda, const double *B, int64_t ldb, double beta, double *C, int64_t ldc,
                      ftblas_err_report *err_report) {
    Ctx &c = ctx();
    int rc = check_args(transA, transB, M, N, K, A, lda, B, ldb, C, ldc, alpha, beta);
    if (rc) return rc;
    if (M == 0 || N == 0) return dgemm_impl(true, transA, transB, M, N, K, alpha, nullptr, lda, nullptr, ldb,
                                            beta, nullptr, ldc, err_report);
    const long long ar = is_t(transA) ? K : M, ac = is_t(transA) ? M : K;
    const long long br = is_t(transB) ? N : K, bc = is_t(transB) ? K : N;
    const bool readAB = K > 0 && alpha != 0.0;
    // device copies are packed (ld = rows, rounded to even for 16-byte vector loads)
    const long long dla = std::max<long long>(1, (ar + 1) / 2 * 2), dlb = std::max<long long>(1, (br + 1) / 2 * 2);
    const long long dlc = std::max<long long>(1, (M + 1) / 2 * 2);
    if (readAB) {
        CK(c.hA.ensure((size_t)dla * ac * 8), "cudaMalloc(A)");
        CK(c.hB.ensure((size_t)dlb * bc * 8), "cudaMalloc(B)");
    }
    CK(c.hC.ensure((size_t)dlc * N * 8), "cudaMalloc(C)");
    CK(c.ensure_copy_streams(), "copy streams");
    // Pipeline over blocks of whole tiles: nrb row blocks x ncb column blocks.  The upload
    // stream carries op(A) row block 0, then every op(B) column block (rows of B for 'T') with
    // the C0 block it completes, then the other op(A) row blocks and their C0 blocks; the
    // library stream runs block (rb, cb) as soon as its three uploads have landed
    // (ftblas_dgemm_ex semantics: caller coordinates, report appended, A encoding reused along
    // a row block); the download stream returns each verified C block.  PCIe traffic in both
    // directions overlaps the DMMA work; only op(A) row block 0 and op(B) block 0 are exposed.
    const long long tiles_m = (M + FTBLAS_TILE_M - 1) / FTBLAS_TILE_M, tiles_n = (N + FTBLAS_TILE_N - 1) / FTBLAS_TILE_N;
    const long long T = tiles_m * tiles_n;
    // The exposed part is the upload of op(A) row block 0 + op(B) column block 0, so blocks are
    // as square as the sizes allow; large problems use 4 x 4 blocks of >= ~7 waves each (c3:
    // 32 x 32 tiles, 1.1 GB exposed instead of 1.3 GB with 2 x 8), smaller ones 2 x 8 / 1 x 8.
    long long nrb, ncb;
    if (T >= 16 * 1000 && tiles_m >= 16 && tiles_n >= 16) {
        nrb = 4; ncb = 4;
    } else {
        nrb = (T / 600 >= 4 && tiles_m >= 16) ? 2 : 1;  // 2 row blocks once >= 4 waves each
        ncb = std::min<long long>(8, tiles_n);
    }
    auto split = [](long long tiles, long long nb, long long q, long long tile, long long lim, long long &x0,
                    long long &x1) {
        const long long per = tiles / nb, rem = tiles % nb;
        const long long t0 = q * per + std::min(q, rem), t1 = t0 + per + (q < rem ? 1 : 0);
        x0 = t0 * tile;
        x1 = std::min(lim, t1 * tile);
    };
    CK(cudaEventRecord(c.ev_entry, c.stream), "event");  // device buffers free once prior work is done
    CK(cudaStreamWaitEvent(c.s_up, c.ev_entry, 0), "wait");
    double *dA = c.hA.as<double>(), *dB = c.hB.as<double>(), *dC = c.hC.as<double>();
    auto up_A = [&](long long rb) -> cudaError_t {
        long long r0, r1;
        split(tiles_m, nrb, rb, FTBLAS_TILE_M, M, r0, r1);
        if (!readAB) return cudaSuccess;
        if (is_t(transA))  // op(A)(r0:r1, :) = columns r0..r1 of the K x M stored A
            return cudaMemcpy2DAsync(dA + r0 * dla, dla * 8, A + r0 * lda, lda * 8, K * 8, r1 - r0,
                                     cudaMemcpyHostToDevice, c.s_up);
        return cudaMemcpy2DAsync(dA + r0, dla * 8, A + r0, lda * 8, (r1 - r0) * 8, K, cudaMemcpyHostToDevice, c.s_up);
    };
    auto up_C0 = [&](long long rb, long long cb) -> cudaError_t {
        long long r0, r1, c0, c1;
        split(tiles_m, nrb, rb, FTBLAS_TILE_M, M, r0, r1);
        split(tiles_n, ncb, cb, FTBLAS_TILE_N, N, c0, c1);
        if (beta == 0.0) return cudaSuccess;
        return cudaMemcpy2DAsync(dC + r0 + c0 * dlc, dlc * 8, C + r0 + c0 * ldc, ldc * 8, (r1 - r0) * 8, c1 - c0,
                                 cudaMemcpyHostToDevice, c.s_up);
    };
    // Row block 0 in KP k parts when K is deep (4 x 4 pipelines; KP = 2 for K >= 8192, 4 for
    // K >= 16384): uploads go in k order (op(A) row block 0 part p, then part p of every op(B)
    // column block), so the first call needs only 1/KP of op(A) block 0 and op(B) block 0 --
    // all of the upload that is exposed -- and every later call finds its operands already
    // up.  Each later part accumulates onto the previous (beta = 1); the last part carries the
    // fault plan, so reports are those of one call per block.  ev_kp[4 cb + p] marks part p of
    // column block cb (parts 0 .. KP-2); the last parts complete with ev_a[0] / ev_up[cb].
    const int KP = (readAB && nrb == 4 && ncb <= 4) ? (K >= 16384 ? 4 : (K >= 8192 ? 2 : 1)) : 1;
    static_assert(Ctx::HOST_MAX_RB * 4 <= Ctx::HOST_MAX_BLOCKS && Ctx::HOST_MAX_CB * 2 <= Ctx::HOST_MAX_BLOCKS,
                  "block policies (4 x 4, 2 x 8, 1 x 8) must fit the event arrays");
    if (nrb > Ctx::HOST_MAX_RB || ncb > Ctx::HOST_MAX_CB || nrb * ncb > Ctx::HOST_MAX_BLOCKS || KP > Ctx::HOST_MAX_KP)
        return cuda_fail(cudaErrorInvalidConfiguration, "ftblas_dgemm_host: block policy exceeds the event arrays");
    const bool ksplit = KP > 1;
    auto kpart = [&](int p) { return p >= KP ? K : (K * p / KP) / BK * BK; };  // part p = [kpart(p), kpart(p+1))
    const long long K1 = kpart(KP - 1);  // start of the last part (uploaded with the full blocks)
    auto up_A_k = [&](long long rb, long long k0, long long k1) -> cudaError_t {
        long long r0, r1;
        split(tiles_m, nrb, rb, FTBLAS_TILE_M, M, r0, r1);
        if (is_t(transA))  // op(A)(r0:r1, k0:k1) = rows k0..k1 of columns r0..r1 of the K x M stored A
            return cudaMemcpy2DAsync(dA + r0 * dla + k0, dla * 8, A + r0 * lda + k0, lda * 8, (k1 - k0) * 8, r1 - r0,
                                     cudaMemcpyHostToDevice, c.s_up);
        return cudaMemcpy2DAsync(dA + r0 + k0 * dla, dla * 8, A + r0 + k0 * lda, lda * 8, (r1 - r0) * 8, k1 - k0,
                                 cudaMemcpyHostToDevice, c.s_up);
    };
    auto up_B_k = [&](long long cb, long long k0, long long k1) -> cudaError_t {
        long long c0, c1;
        split(tiles_n, ncb, cb, FTBLAS_TILE_N, N, c0, c1);
        if (is_t(transB))  // op(B)(k0:k1, c0:c1) = columns k0..k1 of rows c0..c1 of the N x K stored B
            return cudaMemcpy2DAsync(dB + c0 + k0 * dlb, dlb * 8, B + c0 + k0 * ldb, ldb * 8, (c1 - c0) * 8, k1 - k0,
                                     cudaMemcpyHostToDevice, c.s_up);
        return cudaMemcpy2DAsync(dB + c0 * dlb + k0, dlb * 8, B + c0 * ldb + k0, ldb * 8, (k1 - k0) * 8, c1 - c0,
                                 cudaMemcpyHostToDevice, c.s_up);
    };
    if (ksplit) {
        for (int p = 0; p + 1 < KP; p++) {
            CK(up_A_k(0, kpart(p), kpart(p + 1)), "H2D A");
            for (long long cb = 0; cb < ncb; cb++) {
                CK(up_B_k(cb, kpart(p), kpart(p + 1)), "H2D B");
                if (p == 0) CK(up_C0(0, cb), "H2D C");
                CK(cudaEventRecord(c.ev_kp[Ctx::HOST_MAX_KP * cb + p], c.s_up), "event");
            }
        }
        CK(up_A_k(0, K1, K), "H2D A");
    } else {
        CK(up_A(0), "H2D A");
    }
    CK(cudaEventRecord(c.ev_a[0], c.s_up), "event");
    for (long long cb = 0; cb < ncb; cb++) {
        long long c0, c1;
        split(tiles_n, ncb, cb, FTBLAS_TILE_N, N, c0, c1);
        if (ksplit) {
            CK(up_B_k(cb, K1, K), "H2D B");
        } else if (readAB) {
            if (is_t(transB))  // op(B)(:, c0:c1) = rows c0..c1 of the N x K stored B
                CK(cudaMemcpy2DAsync(dB + c0, dlb * 8, B + c0, ldb * 8, (c1 - c0) * 8, K, cudaMemcpyHostToDevice,
                                     c.s_up), "H2D B");
            else
                CK(cudaMemcpy2DAsync(dB + c0 * dlb, dlb * 8, B + c0 * ldb, ldb * 8, K * 8, c1 - c0,
                                     cudaMemcpyHostToDevice, c.s_up), "H2D B");
        }
        if (!ksplit) CK(up_C0(0, cb), "H2D C");
        CK(cudaEventRecord(c.ev_up[cb], c.s_up), "event");
    }
    for (long long rb = 1; rb < nrb; rb++) {
        CK(up_A(rb), "H2D A");
        for (long long cb = 0; cb < ncb; cb++) CK(up_C0(rb, cb), "H2D C");
        CK(cudaEventRecord(c.ev_a[rb], c.s_up), "event");
    }
    for (int p = 0; p + 1 < KP; p++) {  // k parts 0 .. KP-2 of row block 0: no fault injection
        long long r0, r1;
        split(tiles_m, nrb, 0, FTBLAS_TILE_M, M, r0, r1);
        for (long long cb = 0; cb < ncb; cb++) {
            long long c0, c1;
            split(tiles_n, ncb, cb, FTBLAS_TILE_N, N, c0, c1);
            CK(cudaStreamWaitEvent(c.stream, c.ev_kp[Ctx::HOST_MAX_KP * cb + p], 0), "wait");
            const long long k0 = kpart(p);
            const double *Ak = is_t(transA) ? dA + r0 * dla + k0 : dA + r0 + k0 * dla;
            const double *Bk = is_t(transB) ? dB + c0 + k0 * dlb : dB + c0 * dlb + k0;
            rc = dgemm_impl(true, transA, transB, r1 - r0, c1 - c0, kpart(p + 1) - k0, alpha, Ak, dla, Bk, dlb,
                            p == 0 ? beta : 1.0, dC + r0 + c0 * dlc, dlc, nullptr, r0, c0, p > 0 || cb > 0, false,
                            false);
            if (rc) return rc;
        }
    }
    for (long long rb = 0; rb < nrb; rb++) {
        long long r0, r1;
        split(tiles_m, nrb, rb, FTBLAS_TILE_M, M, r0, r1);
        CK(cudaStreamWaitEvent(c.stream, c.ev_a[rb], 0), "wait");
        const double *Ab = readAB ? (is_t(transA) ? dA + r0 * dla : dA + r0) : nullptr;
        for (long long cb = 0; cb < ncb; cb++) {
            long long c0, c1;
            split(tiles_n, ncb, cb, FTBLAS_TILE_N, N, c0, c1);
            if (rb == 0) CK(cudaStreamWaitEvent(c.stream, c.ev_up[cb], 0), "wait");
            const double *Bb = readAB ? (is_t(transB) ? dB + c0 : dB + c0 * dlb) : nullptr;
            const bool first = rb == 0 && cb == 0;
            if (rb == 0 && ksplit) {  // last k part of a row-0 block onto the earlier ones (beta = 1)
                const double *Ak = is_t(transA) ? Ab + K1 : Ab + K1 * dla;
                const double *Bk = is_t(transB) ? Bb + K1 * dlb : Bb + K1;
                rc = dgemm_impl(true, transA, transB, r1 - r0, c1 - c0, K - K1, alpha, Ak, dla, Bk, dlb, 1.0,
                                dC + r0 + c0 * dlc, dlc, nullptr, r0, c0, true, false);
            } else {
                rc = dgemm_impl(true, transA, transB, r1 - r0, c1 - c0, K, alpha, Ab,
                                readAB ? dla : std::max<long long>(1, ar), Bb, readAB ? dlb : std::max<long long>(1, br),
                                beta, dC + r0 + c0 * dlc, dlc, nullptr, r0, c0, !first, cb > 0);
            }
            if (rc) return rc;
            const int q = (int)(rb * ncb + cb);
            CK(cudaEventRecord(c.ev_done[q], c.stream), "event");
            CK(cudaStreamWaitEvent(c.s_down, c.ev_done[q], 0), "wait");
            CK(cudaMemcpy2DAsync(C + r0 + c0 * ldc, ldc * 8, dC + r0 + c0 * dlc, dlc * 8, (r1 - r0) * 8, c1 - c0,
                                 cudaMemcpyDeviceToHost, c.s_down), "D2H C");
        }
    }
    CK(cudaEventRecord(c.ev_exit, c.s_down), "event");
    CK(cudaStreamWaitEvent(c.stream, c.ev_exit, 0), "wait");  // later library work sees C on the host
    CK(cudaStreamSynchronize(c.s_down), "sync");
    if (err_report) return fetch_report(err_report);
    return 0;
}

int ftblas_report_fetch(ftblas_err_report *err_report) {
    if (!err_report) return arg_fail(1, "err_report is NULL");
    return fetch_report(err_report);
}

int ftblas_set_fault_plan(int64_t n, const int64_t *i, const int64_t *j, const int32_t *bit) {
    Ctx &c = ctx();
    if (n < 0) return arg_fail(1, "n < 0");
    if (n > 0 && (!i || !j || !bit)) return arg_fail(2, "NULL plan array");
    std::map<std::pair<int64_t, int64_t>, int> per_tile;
    for (int64_t f = 0; f < n; f++) {
        if (bit[f] < 0 || bit[f] > 63) return arg_fail(4, "bit out of [0,63]");
        if (i[f] < 0 || j[f] < 0) return arg_fail(2, "negative plan coordinate");
        if (++per_tile[{i[f] / FTBLAS_TILE_M, j[f] / FTBLAS_TILE_N}] > FTBLAS_MAX_FLIPS_PER_TILE)
            return arg_fail(1, "more than FTBLAS_MAX_FLIPS_PER_TILE flips in one tile");
    }
    c.plan_i.assign(i, i + n);
    c.plan_j.assign(j, j + n);
    c.plan_bit.assign(bit, bit + n);
    c.plan_version++;
    return 0;
}

int ftblas_set_checksum_mode(int mode) {
    if (mode != FTBLAS_CHECKSUM_GEMM && mode != FTBLAS_CHECKSUM_FUSED) return arg_fail(1, "unknown checksum mode");
    ctx().checksum_mode = mode;
    return 0;
}

int ftblas_get_checksum_mode(void) { return ctx().checksum_mode; }

int ftblas_set_tile_policy(int policy) {
    if (policy != FTBLAS_TILES_AUTO && policy != FTBLAS_TILES_FULL && policy != FTBLAS_TILES_PAIR &&
        policy != FTBLAS_TILES_WS)
        return arg_fail(1, "unknown tile policy");
    ctx().tile_policy = policy;
    return 0;
}

int ftblas_get_tile_policy(void) { return ctx().tile_policy; }

int ftblas_set_stream(void *stream) {
    Ctx &c = ctx();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    if (s == c.stream) return 0;
    // the workspace, report and fault-plan buffers are shared by all calls: work enqueued on
    // the new stream is ordered after everything already enqueued on the old one
    CK(c.ensure_copy_streams(), "streams");
    CK(cudaEventRecord(c.ev_switch, c.stream), "event");
    CK(cudaStreamWaitEvent(s, c.ev_switch, 0), "wait");
    c.stream = s;
    return 0;
}

int64_t ftblas_launch_count(void) { return ctx().launches; }

int ftblas_profile(int enable) {
    ctx().profiling = enable != 0;
    return 0;
}

int ftblas_profile_read(double *encode_ms, double *gemm_ms, int64_t *gemm_launches) {
    Ctx &c = ctx();
    double enc = 0.0, gem = 0.0;
    for (auto &r : c.recs) {
        CK(cudaEventSynchronize(r.e2), "event sync");
        float a = 0.f, b = 0.f;
        CK(cudaEventElapsedTime(&a, r.e0, r.e1), "elapsed");
        CK(cudaEventElapsedTime(&b, r.e1, r.e2), "elapsed");
        enc += a;
        gem += b;
    }
    if (encode_ms) *encode_ms = enc;
    if (gemm_ms) *gemm_ms = gem;
    if (gemm_launches) *gemm_launches = (int64_t)c.recs.size();
    for (auto &r : c.recs) c.pool.push_back(r);
    c.recs.clear();
    return 0;
}

void ftblas_tile_shape(int32_t *tile_m, int32_t *tile_n) {
    if (tile_m) *tile_m = FTBLAS_TILE_M;
    if (tile_n) *tile_n = FTBLAS_TILE_N;
}

const char *ftblas_last_error(void) { return ctx().err; }

#ifdef FTB_WS_PROF
// development builds only: per-CTA phase sums of gemm_ws_kernel (ftblas_ws.cuh), read and reset
int ftblas_ws_prof_read(unsigned long long *out, int n) {
    CK(cudaDeviceSynchronize(), "sync");
    CK(cudaMemcpyFromSymbol(out, ws_prof, sizeof(unsigned long long) * (size_t)std::min(n, 1024 * 16)), "prof read");
    static unsigned long long zero[1024 * 16];
    CK(cudaMemcpyToSymbol(ws_prof, zero, sizeof(zero)), "prof reset");
    return 0;
}
#endif

int ftblas_release(void) {
    Ctx &c = ctx();
    cudaStreamSynchronize(c.stream);
    c.ws.release(); c.ws_gen++; c.a_valid = false; c.rep.release(); c.pend.release(); c.plan_dev.release();
    c.encws.release();
    c.plan_uploaded = -1;
    c.hA.release(); c.hB.release(); c.hC.release();
    return 0;
}

}  // extern "C"
