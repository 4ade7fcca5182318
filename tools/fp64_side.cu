// Microbenchmark (development aid): latency of FP64 work issued by "side" warps (an epilogue)
// while the other warps of the SM keep the DMMA stream busy (the ws kernel's situation).
// One CTA per SM: NMMA warps loop on mma.sync m8n8k4 f64 (32 independent accumulators per
// warp, like a 32 x 64 warp tile); NSIDE warps run `reps` rounds of a batch of ILP independent
// FP64 chains of length DEP (dependent levels), and record clock64 per round.
// Reported: cycles per dependent FP64 level (per round: DEP levels of ILP DFMAs each), and the
// DMMA throughput.  Variants: side warps first / last (warp-id priority), DFMA vs DADD vs IADD.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_side fp64_side.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ILP, int OP>  // OP 0: DFMA, 1: DADD, 2: integer add (64-bit)
__device__ __forceinline__ void side_round(double *f, long long *q, int dep, double a, double b) {
    for (int d = 0; d < dep; d++) {
#pragma unroll
        for (int j = 0; j < ILP; j++) {
            if (OP == 0) asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(f[j]) : "d"(a), "d"(b));
            else if (OP == 1) asm volatile("add.rn.f64 %0, %0, %1;" : "+d"(f[j]) : "d"(a));
            else asm volatile("add.s64 %0, %0, %1;" : "+l"(q[j]) : "l"((long long)d));
        }
    }
}

template <int ILP, int OP>
__global__ void side_kernel(double *out, unsigned long long *cyc, int mma_iters, int side_reps, int dep,
                            int nside, int side_first, volatile int *stop) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    const bool side = side_first ? (warp < nside) : (warp >= nw - nside);
    double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
    __shared__ int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (side) {
        double f[ILP];
        long long q[ILP];
#pragma unroll
        for (int j = 0; j < ILP; j++) { f[j] = j; q[j] = j; }
        unsigned long long t0 = clock64();
        for (int r = 0; r < side_reps; r++) side_round<ILP, OP>(f, q, dep, a, b);
        unsigned long long t1 = clock64();
        double s = 0;
#pragma unroll
        for (int j = 0; j < ILP; j++) s += f[j] + (double)q[j];
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
        if (lane == 0) cyc[blockIdx.x * 32 + warp] = t1 - t0;
        if (lane == 0) atomicAdd(&done, 1);
    } else {
        double c[32][2];
#pragma unroll
        for (int j = 0; j < 32; j++) { c[j][0] = 0; c[j][1] = 0; }
        int it = 0;
        // run until every side warp finished (or mma_iters)
        while (it < mma_iters && *(volatile int *)&done < nside) {
#pragma unroll 1
            for (int u = 0; u < 8; u++) {
#pragma unroll
                for (int j = 0; j < 32; j++)
                    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                                 : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
            }
            it++;
        }
        double s = 0;
#pragma unroll
        for (int j = 0; j < 32; j++) s += c[j][0] + c[j][1];
        out[blockIdx.x * blockDim.x + threadIdx.x] = s;
        if (lane == 0) cyc[blockIdx.x * 32 + warp] = it;
    }
}

template <int ILP, int OP>
void run(const char *name, int sms, int nmma, int nside, int side_first, int dep, double *out, unsigned long long *cyc) {
    const int nw = nmma + nside;
    const int reps = 200;
    auto k = side_kernel<ILP, OP>;
    k<<<sms, nw * 32>>>(out, cyc, nmma ? 1 << 30 : 0, reps, dep, nside, side_first, nullptr);
    cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, nw * 32>>>(out, cyc, nmma ? 1 << 30 : 0, reps, dep, nside, side_first, nullptr);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    static unsigned long long h[148 * 32];
    cudaMemcpy(h, cyc, sizeof(h), cudaMemcpyDeviceToHost);
    double sc = 0, mi = 0; int ns = 0, nm = 0;
    for (int bl = 0; bl < sms; bl++)
        for (int w = 0; w < nw; w++) {
            const bool side = side_first ? (w < nside) : (w >= nw - nside);
            if (side) { sc += h[bl * 32 + w]; ns++; } else { mi += h[bl * 32 + w]; nm++; }
        }
    const double per_level = sc / ns / reps / dep;
    const double mma_fl = nm ? mi / nm * 8 * 32 * 2.0 * 256 * nm : 0;
    printf("%-6s ILP=%2d dep=%3d side=%d %s mma=%d: %8.1f cyc/level (%6.2f cyc/instr)  kernel %.3f ms  DMMA %.2f TF/s\n",
           name, ILP, dep, nside, side_first ? "first" : "last ", nmma, per_level, per_level / ILP, ms,
           mma_fl / ms / 1e9);
}

int main() {
    cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
    const int sms = p.multiProcessorCount;
    double *out; unsigned long long *cyc;
    cudaMalloc(&out, sizeof(double) * sms * 1024);
    cudaMalloc(&cyc, sizeof(unsigned long long) * sms * 32);
    for (int sf : {1, 0}) {
        run<1, 0>("DFMA", sms, 8, 4, sf, 64, out, cyc);
        run<8, 0>("DFMA", sms, 8, 4, sf, 64, out, cyc);
        run<16, 0>("DFMA", sms, 8, 4, sf, 32, out, cyc);
        run<32, 0>("DFMA", sms, 8, 4, sf, 16, out, cyc);
        run<64, 0>("DFMA", sms, 8, 4, sf, 8, out, cyc);
        run<8, 1>("DADD", sms, 8, 4, sf, 64, out, cyc);
        run<8, 2>("IADD64", sms, 8, 4, sf, 64, out, cyc);
    }
    run<1, 0>("DFMA", sms, 0, 4, 1, 64, out, cyc);
    run<8, 0>("DFMA", sms, 0, 4, 1, 64, out, cyc);
    run<32, 0>("DFMA", sms, 0, 4, 1, 16, out, cyc);
    run<8, 0>("DFMA", sms, 4, 4, 1, 64, out, cyc);
    run<8, 0>("DFMA", sms, 4, 4, 0, 64, out, cyc);
    cudaError_t e = cudaGetLastError();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
