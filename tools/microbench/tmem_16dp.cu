// Probe: which TMEM lanes/columns does tcgen05.ld.16x64b read when the lane
// field of the address is the warp quarter base + 16? (design check for
// splitting one TMEM lane quarter between two warps)
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void probe(uint32_t* out) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(
            (uint32_t)__cvta_generic_to_shared(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = slot;
    const uint32_t row = warp * 32 + lane;
    uint32_t v[8];
    for (int c = 0; c < 8; ++c) v[c] = row * 1000 + c;
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(tmem + ((warp * 32) << 16)),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
    asm volatile("tcgen05.wait::st.sync.aligned;\n");
    __syncwarp();
    for (int off = 0; off < 32; off += 16) {
        uint32_t r0, r1;
        asm volatile("tcgen05.ld.sync.aligned.16x64b.x2.b32 {%0,%1}, [%2];\n"
                     : "=r"(r0), "=r"(r1)
                     : "r"(tmem + ((warp * 32 + off) << 16)));
        asm volatile("tcgen05.wait::ld.sync.aligned;\n");
        out[(off / 16) * 256 + threadIdx.x * 2 + 0] = r0;
        out[(off / 16) * 256 + threadIdx.x * 2 + 1] = r1;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(tmem));
}

int main() {
    uint32_t* d;
    cudaMalloc(&d, 512 * 4);
    cudaMemset(d, 0xff, 512 * 4);
    probe<<<1, 128>>>(d);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status %s\n", cudaGetErrorString(e));
    uint32_t h[512];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    for (int off = 0; off < 2; ++off)
        for (int w = 0; w < 4; w += 3) {
            printf("base +%d warp %d:", off * 16, w);
            for (int t = 0; t < 32; ++t) {
                const uint32_t a = h[off * 256 + (w * 32 + t) * 2], b = h[off * 256 + (w * 32 + t) * 2 + 1];
                printf(" t%d:L%u.c%u|L%u.c%u", t, a / 1000, a % 1000, b / 1000, b % 1000);
            }
            printf("\n");
        }
    return 0;
}
