// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) throughput on B200 beside the DFMA peak, for the
// NEXT-3 question: can a dense per-offset M2L operator on DMMA beat the Pascal-form
// M2L?  Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// CH independent accumulator chains per warp
template <int CH>
__global__ void dmma_peak(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5 - threadIdx.x * 1e-9;
  double d[CH][2];
#pragma unroll
  for (int c = 0; c < CH; ++c) d[c][0] = d[c][1] = c * 1e-3;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) dmma(d[c][0], d[c][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += d[c][0] + d[c][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void dfma_peak(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

// DMMA and DFMA chains interleaved in one warp: do the two share the FP64 pipe?
__global__ void mixed_peak(double* out, int iters, double a2, double b2) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.5 - threadIdx.x * 1e-9;
  double d[4][2], x[8];
#pragma unroll
  for (int c = 0; c < 4; ++c) d[c][0] = d[c][1] = c * 1e-3;
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-9 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < 4; ++c) dmma(d[c][0], d[c][1], a, b);
#pragma unroll
    for (int r = 0; r < 4; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a2, b2);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c) s += d[c][0] + d[c][1];
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

template <int CH>
int run_dmma(const cudaDeviceProp& prop, double* d, int wpb) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int blocks = prop.multiProcessorCount * 4, threads = 32 * wpb, iters = 8192;
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(e0);
    dmma_peak<CH><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  // one m8n8k4 = 8*8*4 FMAs = 512 flops per warp instruction
  const double flops = 512.0 * CH * (double)iters * blocks * wpb;
  printf("dmma m8n8k4 f64: %d chains/warp, %d warps/block x %d blocks: best %.3f ms  %.2f TFLOP/s\n", CH, wpb, blocks,
         best, flops / best / 1e9);
  return 0;
}

int main() {
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, 0));
  printf("device %s SMs %d clock %d kHz\n", prop.name, prop.multiProcessorCount, prop.clockRate);
  double* d;
  CK(cudaMalloc(&d, 1 << 20));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  {
    const int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      dfma_peak<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    printf("dfma: best %.3f ms  %.2f TFLOP/s\n", best, 2.0 * 8 * 16 * 4096.0 * blocks * threads / best / 1e9);
  }
  run_dmma<4>(prop, d, 4);
  run_dmma<8>(prop, d, 4);
  run_dmma<8>(prop, d, 8);
  run_dmma<16>(prop, d, 8);
  {
    const int blocks = prop.multiProcessorCount * 4, threads = 256, iters = 8192;
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      mixed_peak<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double warps = blocks * threads / 32.0;
    const double f_mma = 512.0 * 4 * iters * warps, f_fma = 2.0 * 32 * 32 * (double)iters * warps;
    printf("mixed: best %.3f ms  dmma %.2f + dfma %.2f = %.2f TFLOP/s\n", best, f_mma / best / 1e9,
           f_fma / best / 1e9, (f_mma + f_fma) / best / 1e9);
  }
  return 0;
}
