#include <cstdlib>
// Microbenchmark: the consumer side of the DMMA mainloop alone (operand tiles resident in
// smem, no global traffic, no pipeline waits), to separate the instruction-stream limit of
// the fragment-load + DMMA.8x8x4 schedule from the memory pipeline.  Development evidence
// for DESIGN.md section 5.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_mainloop dmma_mainloop.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s @%d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

constexpr int BK = 32, STAGES = 3, LD_MN = 132, LD_K = 36;

__device__ __forceinline__ void dmma(double &c0, double &c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}

// VAR 0: A-outer (as gemm_kernel), 1: B-outer, 2: register double-buffered fragments.
// WM x WN warp tile; NW warps arranged (128/WM) x (128/WN).  A tile mn-contiguous
// (k-row stride LD_MN), B tile k-contiguous (mn-row stride LD_K), as NN in gemm_kernel.
template <int VAR, int WM, int WN>
__global__ void __launch_bounds__((128 / WM) * (128 / WN) * 32, 1) mainloop(double *out, int ktiles) {
    constexpr int FM = WM / 8, FN = WN / 8, NWM = 128 / WM;
    extern __shared__ double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % NWM, wn = warp / NWM;
    constexpr int A_EL = BK * LD_MN, B_EL = 128 * LD_K, ST = A_EL + B_EL;
    for (int i = tid; i < STAGES * ST; i += blockDim.x) smem[i] = 1.0 + 1e-3 * (i & 63);
    __syncthreads();
    double acc[FM][FN][2];
#pragma unroll
    for (int a = 0; a < FM; a++)
#pragma unroll
        for (int b = 0; b < FN; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
    double cs[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    double sv[4][4];
    for (int kt = 0; kt < ktiles; kt++) {
        const double *as = smem + (kt % STAGES) * ST, *bs = as + A_EL;
        if (VAR == 2) {
            double af[2][FM], bf[2][FN];
#pragma unroll
            for (int f = 0; f < FM; f++) af[0][f] = as[(lane & 3) * LD_MN + wm * WM + f * 8 + (lane >> 2)];
#pragma unroll
            for (int f = 0; f < FN; f++) bf[0][f] = bs[(wn * WN + f * 8 + (lane >> 2)) * LD_K + (lane & 3)];
#pragma unroll
            for (int kk = 0; kk < BK / 4; kk++) {
                const int cur = kk & 1, nxt = cur ^ 1;
                if (kk + 1 < BK / 4) {
                    const int k = (kk + 1) * 4 + (lane & 3);
#pragma unroll
                    for (int f = 0; f < FM; f++) af[nxt][f] = as[k * LD_MN + wm * WM + f * 8 + (lane >> 2)];
#pragma unroll
                    for (int f = 0; f < FN; f++) bf[nxt][f] = bs[(wn * WN + f * 8 + (lane >> 2)) * LD_K + k];
                }
#pragma unroll
                for (int a = 0; a < FM; a++)
#pragma unroll
                    for (int b = 0; b < FN; b++) dmma(acc[a][b][0], acc[a][b][1], af[cur][a], bf[cur][b]);
            }
        } else if (VAR >= 3) {
#pragma unroll
            for (int kk = 0; kk < BK / 4; kk++) {
                double af[FM], bf[FN];
                const int k = kk * 4 + (lane & 3);
#pragma unroll
                for (int f = 0; f < FM; f++) af[f] = as[k * LD_MN + wm * WM + f * 8 + (lane >> 2)];
#pragma unroll
                for (int f = 0; f < FN; f++) bf[f] = bs[(wn * WN + f * 8 + (lane >> 2)) * LD_K + k];
#pragma unroll
                for (int a = 0; a < FM; a++) {
#pragma unroll
                    for (int b = 0; b < FN; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
                    if (VAR == 5) { cs[a & 3] = fma(af[a], bf[a & 3], cs[a & 3]); cs[4 + (a & 3)] = fma(bf[a & 3], af[a], cs[4 + (a & 3)]); }
                }
                if (VAR == 8) {  // 4 DFMA per k4, register-only operands
                    cs[0] = fma(cs[4], 1.0000001, cs[0]);
                    cs[1] = fma(cs[5], 1.0000001, cs[1]);
                    cs[2] = fma(cs[6], 0.9999999, cs[2]);
                    cs[3] = fma(cs[7], 0.9999999, cs[3]);
                }
                if (VAR == 9) {  // save fragment copies; 16-DFMA burst every 4 k4 steps
                    sv[kk & 3][0] = af[0]; sv[kk & 3][1] = af[1]; sv[kk & 3][2] = bf[0]; sv[kk & 3][3] = bf[1];
                    if ((kk & 3) == 3) {
#pragma unroll
                        for (int q = 0; q < 4; q++) {
                            cs[0] = fma(sv[q][0], 1.0000001, cs[0]);
                            cs[1] = fma(sv[q][1], 1.0000001, cs[1]);
                            cs[2] = fma(0.9999999, sv[q][2], cs[2]);
                            cs[3] = fma(0.9999999, sv[q][3], cs[3]);
                        }
                    }
                }
                if (VAR == 6 || VAR == 7) {
                    // checksum from the fragments already in registers: 2 A rows x w_k, 2 B cols x v_k
                    const double wv = VAR == 6 ? as[BK * LD_MN - 64 + k] : 1.0000001;
                    const double vv = VAR == 6 ? bs[128 * LD_K - 64 + k] : 0.9999999;
                    const int fa = 0, fb = 0;  // fragments rotated per warp so the checksum rows are af[0..1], bf[0..1]
                    cs[0] = fma(af[fa], wv, cs[0]);
                    cs[1] = fma(af[fa + 1], wv, cs[1]);
                    cs[2] = fma(vv, bf[fb], cs[2]);
                    cs[3] = fma(vv, bf[fb + 1], cs[3]);
                }
            }
            if (VAR == 3) {
#pragma unroll
                for (int q = 0; q < 32; q++) cs[q & 7] = fma(cs[(q + 3) & 7], 1.0000001, cs[q & 7]);
            }
            if (VAR == 4) {
                const int r = tid & 127, h = tid >> 7;
#pragma unroll
                for (int q = 0; q < 16; q++) cs[q & 3] = fma(as[(h * 16 + q) * LD_MN + r], as[h * 16 + q], cs[q & 3]);
#pragma unroll
                for (int q = 0; q < 16; q++) cs[4 + (q & 3)] = fma(bs[r * LD_K + h * 16 + q], bs[q], cs[4 + (q & 3)]);
            }
        } else {
#pragma unroll
            for (int kk = 0; kk < BK / 4; kk++) {
                double af[FM], bf[FN];
                const int k = kk * 4 + (lane & 3);
#pragma unroll
                for (int f = 0; f < FM; f++) af[f] = as[k * LD_MN + wm * WM + f * 8 + (lane >> 2)];
#pragma unroll
                for (int f = 0; f < FN; f++) bf[f] = bs[(wn * WN + f * 8 + (lane >> 2)) * LD_K + k];
                if (VAR == 0) {
#pragma unroll
                    for (int a = 0; a < FM; a++)
#pragma unroll
                        for (int b = 0; b < FN; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
                } else {
#pragma unroll
                    for (int b = 0; b < FN; b++)
#pragma unroll
                        for (int a = 0; a < FM; a++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
                }
            }
        }
    }
    double s = 0.0;
#pragma unroll
    for (int q = 0; q < 8; q++) s += cs[q];
#pragma unroll
    for (int a = 0; a < FM; a++)
#pragma unroll
        for (int b = 0; b < FN; b++) s += acc[a][b][0] + acc[a][b][1];
    out[blockIdx.x * blockDim.x + tid] = s;
}

template <int VAR, int WM, int WN>
int run(const char *name, int sms, double *out) {
    constexpr int NT = (128 / WM) * (128 / WN) * 32;
    auto k = mainloop<VAR, WM, WN>;
    const int bytes = STAGES * (BK * LD_MN + 128 * LD_K) * 8;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    const int ktiles = 4096, blocks = sms * 4;
    k<<<blocks, NT, bytes>>>(out, 64);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<blocks, NT, bytes>>>(out, ktiles);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 128 * 128 * BK * (double)ktiles * blocks;
    printf("%-34s %8.3f ms  %6.2f TFLOP/s\n", name, ms, fl / ms / 1e9);
    return 0;
}


// 8 MMA warps run the pure DMMA loop; NCW extra warps compute the stage checksums
// (r: 128 rows x BK, s: 128 cols x BK) from smem with DFMA, at the same stage cadence.
template <int NCW, int MODE>
__global__ void __launch_bounds__(256 + 32 * NCW, 1) mainloop_cw(double *out, int ktiles) {
    extern __shared__ double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    constexpr int A_EL = BK * LD_MN, B_EL = 128 * LD_K, ST = A_EL + B_EL;
    for (int i = tid; i < STAGES * ST; i += blockDim.x) smem[i] = 1.0 + 1e-3 * (i & 63);
    __syncthreads();
    if (warp >= 8) {
        const int ct = tid - 256;  // 0 .. 32*NCW-1
        double r[4] = {0, 0, 0, 0};
        for (int kt = 0; kt < ktiles; kt++) {
            const double *as = smem + (kt % STAGES) * ST, *bs = as + A_EL;
            // rows/cols handled by this thread: 256 quantities (128 r + 128 s) over 32*NCW threads
#pragma unroll 1
            for (int q = ct; q < 256; q += 32 * NCW) {
                const int row = q & 127;
                double acc2 = 0.0;
                if (MODE == 0) {  // LDS + DFMA
                    if (q < 128) {
#pragma unroll
                        for (int k = 0; k < BK; k++) acc2 = fma(as[k * LD_MN + row], as[k], acc2);
                    } else {
#pragma unroll
                        for (int k = 0; k < BK; k++) acc2 = fma(bs[row * LD_K + k], bs[k], acc2);
                    }
                } else if (MODE == 1) {  // LDS only (integer combine)
                    long long x = 0;
                    if (q < 128) {
#pragma unroll
                        for (int k = 0; k < BK; k++) x ^= __double_as_longlong(as[k * LD_MN + row]);
                    } else {
#pragma unroll
                        for (int k = 0; k < BK; k++) x ^= __double_as_longlong(bs[row * LD_K + k]);
                    }
                    acc2 = (double)(x & 1);
                } else {  // DFMA only, register operands that change every iteration
                    double u = r[0] + kt, v = r[1] + q;
#pragma unroll
                    for (int k = 0; k < BK; k++) acc2 = fma(u, v, acc2);
                }
                r[q & 3] += acc2;
            }
        }
        out[blockIdx.x * blockDim.x + tid] = r[0] + r[1] + r[2] + r[3];
        return;
    }
    const int wm = warp & 1, wn = warp >> 1;
    double acc[8][4][2];
#pragma unroll
    for (int a = 0; a < 8; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int kt = 0; kt < ktiles; kt++) {
        const double *as = smem + (kt % STAGES) * ST, *bs = as + A_EL;
#pragma unroll
        for (int kk = 0; kk < BK / 4; kk++) {
            double af[8], bf[4];
            const int k = kk * 4 + (lane & 3);
#pragma unroll
            for (int f = 0; f < 8; f++) af[f] = as[k * LD_MN + wm * 64 + f * 8 + (lane >> 2)];
#pragma unroll
            for (int f = 0; f < 4; f++) bf[f] = bs[(wn * 32 + f * 8 + (lane >> 2)) * LD_K + k];
#pragma unroll
            for (int a = 0; a < 8; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < 8; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) s += acc[a][b][0] + acc[a][b][1];
    out[blockIdx.x * blockDim.x + tid] = s;
}

template <int NCW, int MODE>
int run_cw(const char *name, int sms, double *out) {
    auto k = mainloop_cw<NCW, MODE>;
    const int bytes = STAGES * (BK * LD_MN + 128 * LD_K) * 8;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    const int ktiles = 4096, blocks = sms * 4;
    k<<<blocks, 256 + 32 * NCW, bytes>>>(out, 64);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<blocks, 256 + 32 * NCW, bytes>>>(out, ktiles);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 128 * 128 * BK * (double)ktiles * blocks;
    printf("%-34s %8.3f ms  %6.2f TFLOP/s\n", name, ms, fl / ms / 1e9);
    return 0;
}


// CTA tile 128 x (32 * NWN) with 2 x NWN warps of 64 x 32; minBlocks CTAs per SM requested.
template <int NWN, int MINB>
__global__ void __launch_bounds__(64 * NWN, MINB) mainloop_nw(double *out, int ktiles) {
    extern __shared__ double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;
    constexpr int BNT = 32 * NWN, A_EL = BK * LD_MN, B_EL = BNT * LD_K, ST = A_EL + B_EL;
    for (int i = tid; i < STAGES * ST; i += blockDim.x) smem[i] = 1.0 + 1e-3 * (i & 63);
    __syncthreads();
    double acc[8][4][2];
#pragma unroll
    for (int a = 0; a < 8; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int kt = 0; kt < ktiles; kt++) {
        const double *as = smem + (kt % STAGES) * ST, *bs = as + A_EL;
#pragma unroll
        for (int kk = 0; kk < BK / 4; kk++) {
            double af[8], bf[4];
            const int k = kk * 4 + (lane & 3);
#pragma unroll
            for (int f = 0; f < 8; f++) af[f] = as[k * LD_MN + wm * 64 + f * 8 + (lane >> 2)];
#pragma unroll
            for (int f = 0; f < 4; f++) bf[f] = bs[(wn * 32 + f * 8 + (lane >> 2)) * LD_K + k];
#pragma unroll
            for (int a = 0; a < 8; a++)
#pragma unroll
                for (int b = 0; b < 4; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < 8; a++)
#pragma unroll
        for (int b = 0; b < 4; b++) s += acc[a][b][0] + acc[a][b][1];
    out[blockIdx.x * blockDim.x + tid] = s;
}

template <int NWN, int MINB>
int run_nw(const char *name, int sms, double *out, int blocks_per_sm, int stages_bytes_div) {
    auto k = mainloop_nw<NWN, MINB>;
    const int bytes = STAGES * (BK * LD_MN + 32 * NWN * LD_K) * 8;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    const int ktiles = 4096, blocks = sms * blocks_per_sm * 4;
    k<<<blocks, 64 * NWN, bytes>>>(out, 64);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<blocks, 64 * NWN, bytes>>>(out, ktiles);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 128 * 32 * NWN * BK * (double)ktiles * blocks;
    printf("%-34s %8.3f ms  %6.2f TFLOP/s\n", name, ms, fl / ms / 1e9);
    (void)stages_bytes_div;
    return 0;
}

// CTA tile 128 x BNT with (128 / WM) x (BNT / WN) warps of WM x WN; MINB CTAs per SM.
template <int WM, int WN, int BNT, int MINB>
__global__ void __launch_bounds__((128 / WM) * (BNT / WN) * 32, MINB) mainloop_g(double *out, int ktiles) {
    extern __shared__ double smem[];
    constexpr int NWM = 128 / WM, FM = WM / 8, FN = WN / 8;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % NWM, wn = warp / NWM;
    constexpr int A_EL = BK * LD_MN, B_EL = BNT * LD_K, ST = A_EL + B_EL;
    for (int i = tid; i < STAGES * ST; i += blockDim.x) smem[i] = 1.0 + 1e-3 * (i & 63);
    __syncthreads();
    double acc[FM][FN][2];
#pragma unroll
    for (int a = 0; a < FM; a++)
#pragma unroll
        for (int b = 0; b < FN; b++) acc[a][b][0] = acc[a][b][1] = 0.0;
    for (int kt = 0; kt < ktiles; kt++) {
        const double *as = smem + (kt % STAGES) * ST, *bs = as + A_EL;
#pragma unroll
        for (int kk = 0; kk < BK / 4; kk++) {
            double af[FM], bf[FN];
            const int k = kk * 4 + (lane & 3);
#pragma unroll
            for (int f = 0; f < FM; f++) af[f] = as[k * LD_MN + wm * WM + f * 8 + (lane >> 2)];
#pragma unroll
            for (int f = 0; f < FN; f++) bf[f] = bs[(wn * WN + f * 8 + (lane >> 2)) * LD_K + k];
#pragma unroll
            for (int a = 0; a < FM; a++)
#pragma unroll
                for (int b = 0; b < FN; b++) dmma(acc[a][b][0], acc[a][b][1], af[a], bf[b]);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < FM; a++)
#pragma unroll
        for (int b = 0; b < FN; b++) s += acc[a][b][0] + acc[a][b][1];
    out[blockIdx.x * blockDim.x + tid] = s;
}

template <int WM, int WN, int BNT, int MINB>
int run_g(const char *name, int sms, double *out, int blocks_per_sm) {
    auto k = mainloop_g<WM, WN, BNT, MINB>;
    constexpr int NT = (128 / WM) * (BNT / WN) * 32;
    const int bytes = STAGES * (BK * LD_MN + BNT * LD_K) * 8;
    CK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    const int ktiles = 4096, blocks = sms * blocks_per_sm * 4;
    k<<<blocks, NT, bytes>>>(out, 64);
    CK(cudaDeviceSynchronize());
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<blocks, NT, bytes>>>(out, ktiles);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 2.0 * 128 * BNT * BK * (double)ktiles * blocks;
    printf("%-34s %8.3f ms  %6.2f TFLOP/s\n", name, ms, fl / ms / 1e9);
    return 0;
}

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    printf("device %s sms=%d\n", p.name, p.multiProcessorCount);
    double *out; CK(cudaMalloc(&out, sizeof(double) * p.multiProcessorCount * 4 * 1024));
    const int sms = p.multiProcessorCount;
    run<0, 64, 32>("A-outer 8 warps 64x32", sms, out);
    run<3, 64, 32>("+32 DFMA burst/stage (regs)", sms, out);
    run<4, 64, 32>("+32 DFMA burst/stage (LDS)", sms, out);
    run<5, 64, 32>("+DFMA interleaved 16/k4x8 (regs)", sms, out);
    run<6, 64, 32>("+frag-reuse 4 DFMA/k4 + 2 LDS/k4", sms, out);
    run<7, 64, 32>("+frag-reuse 4 DFMA/k4 (no LDS)", sms, out);
    run_nw<4, 1>("8 warps 128x128, 1 CTA/SM", sms, out, 1, 1);
    run_nw<2, 1>("4 warps 128x64, 1 CTA/SM", sms, out, 1, 1);
    run_nw<2, 2>("4 warps 128x64, 2 CTA/SM", sms, out, 2, 1);
    if (getenv("PAIR_ONLY")) {
        run_g<64, 32, 64, 1>("g 4 warps 64x32 128x64 1 CTA/SM", sms, out, 1);
        run_g<64, 32, 64, 2>("g 4 warps 64x32 128x64 2 CTA/SM", sms, out, 2);
        run_g<32, 32, 64, 1>("g 8 warps 32x32 128x64 1 CTA/SM", sms, out, 1);
        run_g<32, 32, 64, 2>("g 8 warps 32x32 128x64 2 CTA/SM", sms, out, 2);
        run_g<64, 16, 64, 1>("g 8 warps 64x16 128x64 1 CTA/SM", sms, out, 1);
        run_g<32, 64, 64, 1>("g 4 warps 32x64 128x64 1 CTA/SM", sms, out, 1);
        return 0;
    }
    run_cw<4, 0>("8 MMA + 4 cksum warps LDS+DFMA", sms, out);
    run_cw<4, 1>("8 MMA + 4 cksum warps LDS only", sms, out);
    run_cw<4, 2>("8 MMA + 4 cksum warps DFMA only", sms, out);
    run<9, 64, 32>("+frag copies, 16-DFMA burst/4 k4", sms, out);
    return 0;
}
