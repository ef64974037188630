// FP64 throughput microbenchmarks for the roofline denominator.
// Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
//  1. DFMA peak: 8 independent FMA chains per thread, 148*8 CTAs x 256 threads.
//  2. libdevice log+atan2 per pair cost (for context on the P2P transcendental budget).
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e), __LINE__); return 1; } } while (0)

__global__ void dfma_peak(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-9, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3,
         x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

__global__ void logatan_cost(const double* xs, double* out, int n, int iters) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double dx = xs[i], dy = xs[(i + 7) % n];
  double acc_re = 0, acc_im = 0;
  for (int k = 0; k < iters; ++k) {
    double r2 = dx * dx + dy * dy;
    acc_re += log(r2);
    acc_im += atan2(dy, dx);
    dx += 1e-3; dy -= 1e-3;
  }
  out[i] = acc_re + acc_im;
}

int main() {
  int dev = 0; cudaDeviceProp prop; CK(cudaGetDeviceProperties(&prop, dev));
  printf("device %s SMs %d\n", prop.name, prop.multiProcessorCount);
  double* d; CK(cudaMalloc(&d, 64 << 20));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = prop.multiProcessorCount * 8, threads = 256, iters = 4096;
  for (int rep = 0; rep < 6; ++rep) {
    cudaEventRecord(e0);
    dfma_peak<<<blocks, threads>>>(d, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("dfma_peak rep %d: %.3f ms  %.2f TFLOP/s\n", rep, ms, flops / ms / 1e9);
  }
  int n = 1 << 22;
  double* xs; CK(cudaMalloc(&xs, n * sizeof(double)));
  double* h = new double[n];
  for (int i = 0; i < n; ++i) h[i] = 0.01 + (i % 1000) * 1e-3 * ((i & 1) ? 1 : -1);
  CK(cudaMemcpy(xs, h, n * sizeof(double), cudaMemcpyHostToDevice));
  for (int rep = 0; rep < 4; ++rep) {
    int it = 256;
    cudaEventRecord(e0);
    logatan_cost<<<(n + 255) / 256, 256>>>(xs, d, n, it);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("libdevice log+atan2: %.3f ms  %.3e pairs/s\n", ms, (double)n * it / ms * 1e3);
  }
  return 0;
}
