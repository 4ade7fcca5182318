// Microbenchmark: FP64 pipe throughput on sm_100a (B200).
// Measures DMMA (mma.sync m8n8k4 f64 -> SASS DMMA.8x8x4), DFMA, and a mix,
// to decide whether ABFT checksum DFMAs can overlap DMMA. Evidence for DESIGN.md.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_pipes fp64_pipes.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template <int NACC, int NDFMA>
__global__ void mix_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double c[NACC][2];
#pragma unroll
  for (int j = 0; j < NACC; j++) { c[j][0] = 0; c[j][1] = 0; }
  double f[8];
#pragma unroll
  for (int j = 0; j < 8; j++) f[j] = j;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < NACC; j++) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
    }
#pragma unroll
    for (int j = 0; j < NDFMA; j++) {
      asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(f[j % 8]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < NACC; j++) s += c[j][0] + c[j][1];
#pragma unroll
  for (int j = 0; j < 8; j++) s += f[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NDFMA>
__global__ void dfma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  double f[8];
#pragma unroll
  for (int j = 0; j < 8; j++) f[j] = j;
  for (int i = 0; i < iters; i++) {
#pragma unroll
    for (int j = 0; j < NDFMA; j++) {
      asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(f[j % 8]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; j++) s += f[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
float run(K kern, int blocks, int threads, int iters, double* out) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  kern<<<blocks, threads>>>(out, iters);
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  for (int r = 0; r < 5; r++) kern<<<blocks, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms / 5;
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int sms = p.multiProcessorCount;
  printf("device %s sms=%d\n", p.name, sms);
  double* out; CK(cudaMalloc(&out, sizeof(double) * sms * 8 * 1024));
  const int iters = 20000;
  for (int wpb : {4, 8, 16}) {
    int threads = 32 * wpb, blocks = sms * 2;
    double warps = (double)blocks * wpb;
    float ms = run(mix_kernel<8, 0>, blocks, threads, iters, out);
    double fl = warps * iters * 8 * 2.0 * 256;
    printf("DMMA only   wpb=%2d: %.3f ms  %.2f TFLOP/s\n", wpb, ms, fl / ms / 1e9);
    ms = run(dfma_kernel<16>, blocks, threads, iters, out);
    fl = warps * 32 * iters * 16 * 2.0;
    printf("DFMA only   wpb=%2d: %.3f ms  %.2f TFLOP/s\n", wpb, ms, fl / ms / 1e9);
    ms = run(mix_kernel<8, 8>, blocks, threads, iters, out);
    double flm = warps * iters * 8 * 2.0 * 256, fld = warps * 32 * iters * 8 * 2.0;
    printf("DMMA8+DFMA8 wpb=%2d: %.3f ms  mma %.2f + dfma %.2f = %.2f TFLOP/s\n", wpb, ms,
           flm / ms / 1e9, fld / ms / 1e9, (flm + fld) / ms / 1e9);
    ms = run(mix_kernel<8, 2>, blocks, threads, iters, out);
    flm = warps * iters * 8 * 2.0 * 256; fld = warps * 32 * iters * 2 * 2.0;
    printf("DMMA8+DFMA2 wpb=%2d: %.3f ms  mma %.2f + dfma %.2f = %.2f TFLOP/s\n", wpb, ms,
           flm / ms / 1e9, fld / ms / 1e9, (flm + fld) / ms / 1e9);
  }
  CK(cudaGetLastError());
  return 0;
}
