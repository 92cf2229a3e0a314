// Probe: tcgen05.mma kind::i8 issue-to-completion cost on one SM for the
// shapes the sketch uses (M = 128, K = 32, N = 48 / 64 / 80 / ...), with the
// operand layouts of sketch_tc.cu (K-major, no swizzle: core matrices of
// 8 rows x 16 B). One thread issues R rounds of 8 MMAs into 8 accumulators
// (independent, like the 7 slices + ones), or into 1 accumulator (a
// dependent chain); cycles per MMA = clock64 delta / (8 R). Also the
// 128B-swizzled operand layout for comparison.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_i8_rate umma_i8_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t desc_noswz(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return static_cast<uint64_t>((addr >> 4) & 0x3fffu) | (static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}

// K-major, 128-byte swizzle: rows of 128 B (K = 128 int8), 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t desc_sw128(uint32_t addr) {
    return static_cast<uint64_t>((addr >> 4) & 0x3fffu) | (static_cast<uint64_t>(1) << 16) |
           (static_cast<uint64_t>(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}

__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
    return (2u << 4) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int N, int NACC, int KSTEP, bool SW, int M = 128>
__global__ void bench(long long* out, int rounds) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t base = (smem_u32(sm) + 1023u) & ~1023u;
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(sm)[i] = 0x01020304u * (i + 1);
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&slot)));
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
    if (threadIdx.x == 0) {
        constexpr uint32_t id = idesc_i8(M, N);
        // A: 8 slice tiles of 128 x 32 (4 KB each); B: N x 32 (K blocks of N x 16 B)
        const uint32_t a0 = base, b0 = base + 8 * 4096 * (KSTEP);
        long long t0 = 0;
        for (int r = -2; r < rounds; ++r) {
            if (r == 0) t0 = clock64();
            for (int t = 0; t < 8; ++t) {
                const int acc_i = t % NACC;
                uint64_t ad, bd;
                if (SW) {
                    ad = desc_sw128(a0 + t * 16384);
                    bd = desc_sw128(b0);
                } else {
                    ad = desc_noswz(a0 + t * 4096 * KSTEP, 128 * 16, 128);
                    bd = desc_noswz(b0, N * 16, 128);
                }
                umma(M == 64 ? tmem + N * (acc_i % 4) + (acc_i >= 4 ? (16u << 16) : 0u) : tmem + N * acc_i, ad, bd, id, 1u);
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&bar))
                     : "memory");
        asm volatile(
            "{\n.reg .pred P1;\nWAIT:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
            "@!P1 bra WAIT;\n}\n" ::"r"(smem_u32(&bar)));
        const long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (threadIdx.x < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

template <int N, int NACC, int KSTEP, bool SW, int M = 128>
void run(const char* name, int grid) {
    const int rounds = 4096;
    long long* d;
    cudaMalloc(&d, grid * sizeof(long long));
    auto k = bench<N, NACC, KSTEP, SW, M>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    k<<<grid, 128, 200 * 1024>>>(d, rounds);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148] = {0};
    cudaMemcpy(h, d, grid * sizeof(long long), cudaMemcpyDeviceToHost);
    long long mx = 0;
    for (int i = 0; i < grid; ++i) mx = h[i] > mx ? h[i] : mx;
    const double cyc = static_cast<double>(mx) / (8.0 * rounds);
    const double macs = static_cast<double>(M) * N * 32;
    printf("%-34s grid %3d: %7.1f cycles/MMA  %7.0f MAC/clk  %s\n", name, grid, cyc, macs / cyc,
           cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<48, 8, 1, false>("N48 8acc", 1);
    run<64, 8, 1, false>("N64 8acc", 1);
    run<80, 4, 1, false>("N80 4acc", 1);
    run<80, 1, 1, false>("N80 1acc (chain)", 1);
    run<128, 4, 1, false>("N128 4acc", 1);
    run<256, 2, 1, false>("N256 2acc", 1);
    run<48, 8, 1, false>("N48 8acc", 148);
    run<80, 4, 1, false>("N80 4acc", 148);
    run<256, 2, 1, false>("N256 2acc", 148);
    run<80, 4, 1, true>("N80 4acc sw128 (K=32 of 128B rows)", 1);
    run<256, 2, 1, true>("N256 2acc sw128", 1);
    run<80, 8, 1, false, 64>("M64 N80 8acc (two lane halves)", 1);
    run<48, 8, 1, false, 64>("M64 N48 8acc", 1);
    run<128, 8, 1, false, 64>("M64 N128 8acc", 1);
    return 0;
}
