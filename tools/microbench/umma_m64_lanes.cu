// Probe: which TMEM lanes does tcgen05.mma kind::i8 with M = 64 write, and
// is a D address with lane field 16 accepted (a second M = 64 accumulator in
// the other half of every lane quarter)? Design check for a 64-snapshot
// tile that keeps 8 accumulators x N = 80 in 320 TMEM columns.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_m64_lanes umma_m64_lanes.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((addr >> 4) & 0x3fffu) | (static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
    return (2u << 4) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

constexpr int N = 16;

__global__ void probe(int* out, int lane_off) {
    __shared__ __align__(1024) int8_t a[64 * 32];
    __shared__ __align__(1024) int8_t b0[N * 32];
    __shared__ __align__(1024) int8_t b1[N * 32];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < 64 * 32; i += blockDim.x) a[i] = 1;
    for (int i = threadIdx.x; i < N * 32; i += blockDim.x) {
        b0[i] = 1;
        b1[i] = 2;
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;\n" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tmem = slot;
    {  // zero all 128 lanes x 16 columns
        const uint32_t z = 0;
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(
                tmem + ((warp * 32) << 16)),
            "r"(z));
        asm volatile("tcgen05.wait::st.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (threadIdx.x == 0) {
        constexpr uint32_t id = idesc_i8(64, N);
        const uint64_t ad = desc(smem_u32(a), 64 * 16, 128);
        asm volatile(
            "{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\n"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
            "l"(ad), "l"(desc(smem_u32(b0), N * 16, 128)), "r"(id));
        if (lane_off >= 0)
            asm volatile(
                "{\n.reg .pred p;\nsetp.ne.b32 p, 0, 0;\n"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + (lane_off << 16)),
                "l"(ad), "l"(desc(smem_u32(b1), N * 16, 128)), "r"(id));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&bar))
                     : "memory");
    }
    asm volatile(
        "{\n.reg .pred P1;\nWAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
        "@!P1 bra WAIT;\n}\n" ::"r"(smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    uint32_t v[4];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(tmem + ((warp * 32) << 16)));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n");
    for (int c = 0; c < 4; ++c) out[threadIdx.x * 4 + c] = static_cast<int>(v[c]);
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;\n" ::"r"(tmem));
}

int main() {
    int* d;
    cudaMalloc(&d, 512 * 4);
    for (int off : {-1, 16, 32, 64}) {
        cudaMemset(d, 0xff, 512 * 4);
        probe<<<1, 128>>>(d, off);
        cudaError_t e = cudaDeviceSynchronize();
        int h[512];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        printf("second MMA lane offset %d: %s\n  lane: col0 col1 ...\n", off, cudaGetErrorString(e));
        if (e != cudaSuccess) return 1;
        // compress: print runs of lanes with equal (col0, col1)
        int start = 0;
        for (int l = 1; l <= 128; ++l) {
            if (l == 128 || h[l * 4] != h[start * 4] || h[l * 4 + 1] != h[start * 4 + 1]) {
                printf("  lanes %3d-%3d: %d %d %d %d\n", start, l - 1, h[start * 4], h[start * 4 + 1], h[start * 4 + 2],
                       h[start * 4 + 3]);
                start = l;
            }
        }
    }
    return 0;
}
