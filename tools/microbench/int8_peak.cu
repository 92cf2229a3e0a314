// Integer tensor-path microbenchmark for B200 (sm_100a): sustained throughput
// of the legacy register-fed IMMA (mma.sync m16n8k32 s8/u8 -> s32) and of the
// conversions an exact fp64 -> int8-slice split needs (F2I.S64.F64, PRMT).
// Decides whether the sketch can run as an exact integer-sliced contraction.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { \
  printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); return 1; } } while (0)

template <int TILES, bool UNSIGNED_B>
__global__ void imma_kernel(int* out, int iters) {
  int c[TILES][4];
#pragma unroll
  for (int t = 0; t < TILES; ++t) c[t][0] = c[t][1] = c[t][2] = c[t][3] = 0;
  uint32_t a0 = threadIdx.x * 0x01010101u, a1 = a0 ^ 0x5a5a5a5a, a2 = a0 + 7, a3 = a0 * 3;
  uint32_t b0 = threadIdx.x ^ 0x33333333u, b1 = b0 + 11;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < TILES; ++t) {
      if (UNSIGNED_B)
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+r"(c[t][0]), "+r"(c[t][1]), "+r"(c[t][2]), "+r"(c[t][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
      else
        asm volatile("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
                     : "+r"(c[t][0]), "+r"(c[t][1]), "+r"(c[t][2]), "+r"(c[t][3])
                     : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
    }
  }
  int s = 0;
#pragma unroll
  for (int t = 0; t < TILES; ++t) s += c[t][0] + c[t][1] + c[t][2] + c[t][3];
  if (s == 12345) out[threadIdx.x] = s;
}

// fp64 -> int64 conversions, 8 independent chains
__global__ void f2i_kernel(long long* out, int iters, double scale) {
  double x[8];
  long long acc = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) x[c] = threadIdx.x * 1.37 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      long long q = __double2ll_rn(x[c] * scale);
      acc += q;
      x[c] = __longlong_as_double(__double_as_longlong(x[c]) ^ (q & 1));
    }
  }
  if (acc == 12345) out[threadIdx.x] = acc;
}

__global__ void prmt_kernel(uint32_t* out, int iters) {
  uint32_t r[8];
#pragma unroll
  for (int c = 0; c < 8; ++c) r[c] = threadIdx.x * 0x9e3779b9u + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < 8; ++c) r[c] = __byte_perm(r[c], r[(c + 1) & 7], 0x5140);
  }
  uint32_t s = 0;
#pragma unroll
  for (int c = 0; c < 8; ++c) s ^= r[c];
  if (s == 12345) out[threadIdx.x] = s;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  printf("device %s SMs %d clock %d kHz\n", p.name, p.multiProcessorCount, p.clockRate);
  int sms = p.multiProcessorCount;
  void* out; CK(cudaMalloc(&out, 4096 * 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  for (int warps : {4, 8, 16}) {
    int threads = 32 * warps, blocks = sms, iters = 20000;
    imma_kernel<8, false><<<blocks, threads>>>((int*)out, 10);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    imma_kernel<8, false><<<blocks, threads>>>((int*)out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double ops = 2.0 * 16 * 8 * 32 * 8.0 * iters * warps * blocks;
    printf("IMMA s8.s8 m16n8k32 warps/SM %d: %.1f TOPS (%.3f ms)\n", warps, ops / ms / 1e9, ms);
    imma_kernel<8, true><<<blocks, threads>>>((int*)out, 10);
    cudaEventRecord(e0);
    imma_kernel<8, true><<<blocks, threads>>>((int*)out, iters);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("IMMA s8.u8 m16n8k32 warps/SM %d: %.1f TOPS (%.3f ms)\n", warps, ops / ms / 1e9, ms);
  }
  for (int threads : {256, 512, 1024}) {
    int blocks = sms * 2, iters = 4000;
    f2i_kernel<<<blocks, threads>>>((long long*)out, 10, 1024.0);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    f2i_kernel<<<blocks, threads>>>((long long*)out, iters, 1024.0);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double n = 8.0 * iters * threads * blocks;
    printf("F2I.S64.F64 (+DMUL) threads %d: %.1f G/s = %.1f per SM-clock\n", threads, n / ms / 1e6,
           n / (ms * 1e-3) / sms / (p.clockRate * 1e3));
    prmt_kernel<<<blocks, threads>>>((uint32_t*)out, 10);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    prmt_kernel<<<blocks, threads>>>((uint32_t*)out, iters * 4);
    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    n = 8.0 * iters * 4 * threads * blocks;
    printf("PRMT threads %d: %.1f G/s = %.1f per SM-clock\n", threads, n / ms / 1e6,
           n / (ms * 1e-3) / sms / (p.clockRate * 1e3));
  }
  return 0;
}
