// Dependent-chain latency of DADD / DMUL / DFMA on this GPU (one warp).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain_add(double* out, int iters, double a) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) x = __dadd_rn(x, a);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; out[1] = double(t1 - t0) / (16.0 * iters); }
}
__global__ void chain_mul(double* out, int iters, double a) {
    double x = threadIdx.x + 1;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) x = __dmul_rn(x, a);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; out[1] = double(t1 - t0) / (16.0 * iters); }
}
__global__ void chain_muladd(double* out, int iters, double a, const double* q) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int u = 0; u < 16; ++u) x = __dadd_rn(x, __dmul_rn(q[u], a));
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = x; out[1] = double(t1 - t0) / (16.0 * iters); }
}
int main() {
    double *d, h[2], *q;
    cudaMalloc(&d, 16); cudaMalloc(&q, 16 * 8); cudaMemset(q, 0, 128);
    chain_add<<<1, 32>>>(d, 1000, 1.0000001); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    chain_add<<<1, 32>>>(d, 10000, 1.0000001); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("DADD dependent latency: %.1f cycles\n", h[1]);
    chain_mul<<<1, 32>>>(d, 10000, 1.0000001); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("DMUL dependent latency: %.1f cycles\n", h[1]);
    chain_muladd<<<1, 32>>>(d, 10000, 1.0000001, q); cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("DADD(x, DMUL(q,a)) chain: %.1f cycles per step\n", h[1]);
    return 0;
}
