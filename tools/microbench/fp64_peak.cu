// FP64 peak microbenchmark for B200 (sm_100a): DFMA (CUDA cores) vs DMMA
// (mma.sync m8n8k4 f64, the only FP64 tensor path on sm_100a; tcgen05 has no
// f64 kind). Prints sustained TFLOP/s for each, timed with CUDA events.
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int CHAINS>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = threadIdx.x * 1e-3 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.678) out[threadIdx.x] = s;
}

template <int TILES>
__global__ void dmma_kernel(double* out, int iters) {
  double c[TILES][2];
#pragma unroll
  for (int t = 0; t < TILES; ++t) { c[t][0] = 0; c[t][1] = 0; }
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < TILES; ++t) {
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < TILES; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[threadIdx.x] = s;
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("device %s SMs %d\n", p.name, p.multiProcessorCount);
  double* out; CK(cudaMalloc(&out, 1024 * sizeof(double)));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms = p.multiProcessorCount;
  for (int threads : {128, 256, 512}) {
    for (int occ : {1, 2, 4}) {
      int blocks = sms * occ; int iters = 20000;
      dfma_kernel<16><<<blocks, threads>>>(out, 100, 1.0000001, 1e-9);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dfma_kernel<16><<<blocks, threads>>>(out, iters, 1.0000001, 1e-9);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 16 * (double)iters * threads * blocks;
      printf("DFMA threads %d occ %d: %.2f TFLOP/s (%.3f ms)\n", threads, occ, flops / ms / 1e9, ms);
    }
  }
  for (int threads : {128, 256, 512}) {
    for (int occ : {1, 2, 4}) {
      int blocks = sms * occ; int iters = 5000;
      dmma_kernel<16><<<blocks, threads>>>(out, 100);
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      dmma_kernel<16><<<blocks, threads>>>(out, iters);
      cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 256 * 16 * (double)iters * (threads / 32) * blocks;
      printf("DMMA threads %d occ %d: %.2f TFLOP/s (%.3f ms)\n", threads, occ, flops / ms / 1e9, ms);
    }
  }
  // sustained: DMMA for ~3 s
  {
    int threads = 256, blocks = sms * 2, iters = 200000;
    cudaEventRecord(e0);
    dmma_kernel<16><<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 256 * 16 * (double)iters * (threads / 32) * blocks;
    printf("DMMA sustained: %.2f TFLOP/s (%.1f ms)\n", flops / ms / 1e9, ms);
    cudaEventRecord(e0);
    dfma_kernel<16><<<blocks, threads>>>(out, iters * 8, 1.0000001, 1e-9);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    flops = 2.0 * 16 * (double)iters * 8 * threads * blocks;
    printf("DFMA sustained: %.2f TFLOP/s (%.1f ms)\n", flops / ms / 1e9, ms);
  }
  return 0;
}
