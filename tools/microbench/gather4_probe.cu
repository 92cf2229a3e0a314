// gather4_probe.cu -- what does cp.async.bulk.tensor.2d.tile::gather4 load on
// B200, for a given tensor-map box? (development probe; bounded waits, so a
// wrong transaction count reports instead of hanging)
//   nvcc -gencode arch=compute_100a,code=sm_100a -o gather4_probe gather4_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void* p) { return static_cast<uint32_t>(__cvta_generic_to_shared(p)); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, double* out, int expect, int box_swz, int* status) {
    __shared__ __align__(1024) double buf[4 * 32];
    __shared__ __align__(8) uint64_t bar;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4 * 32; ++i) buf[i] = -1.0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(expect) : "memory");
        // rows (dimension 0) 32..47 of columns 5, 17, 3, 60
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6, %7}], [%2];"
            ::"r"(su32(buf)), "l"(&tm), "r"(su32(&bar)), "r"(32), "r"(5), "r"(17), "r"(3), "r"(60) : "memory");
        int done = 0;
        for (int i = 0; i < 2000000 && !done; ++i) {
            uint32_t ok;
            asm volatile("{.reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p;}"
                         : "=r"(ok) : "r"(su32(&bar)) : "memory");
            done = ok;
        }
        *status = done;
        for (int i = 0; i < 4 * 32; ++i) out[i] = buf[i];
    }
}

int main() {
    const int m = 1024, n = 64;
    std::vector<double> h(m * n);
    for (int j = 0; j < n; ++j)
        for (int i = 0; i < m; ++i) h[j * m + i] = j * 10000 + i;  // value = col*10000 + row
    double *d, *out;
    int* st;
    cudaMalloc(&d, sizeof(double) * m * n);
    cudaMalloc(&out, sizeof(double) * 128);
    cudaMalloc(&st, sizeof(int));
    cudaMemcpy(d, h.data(), sizeof(double) * m * n, cudaMemcpyHostToDevice);
    for (int boxh : {1, 4}) {
        CUtensorMap tm;
        cuuint64_t gdim[2] = {(cuuint64_t)m, (cuuint64_t)n};
        cuuint64_t gstr[1] = {(cuuint64_t)m * 8};
        cuuint32_t box[2] = {16, (cuuint32_t)boxh};
        cuuint32_t es[2] = {1, 1};
        CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, gdim, gstr, box, es,
                                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("box {16,%d}: encode rc %d\n", boxh, (int)r);
        if (r) continue;
        probe<<<1, 32>>>(tm, out, 4 * 16 * 8, 0, st);
        cudaError_t e = cudaDeviceSynchronize();
        int s = 0;
        std::vector<double> o(128);
        cudaMemcpy(&s, st, sizeof(int), cudaMemcpyDeviceToHost);
        cudaMemcpy(o.data(), out, sizeof(double) * 128, cudaMemcpyDeviceToHost);
        printf("  launch %s, barrier complete %d\n", cudaGetErrorString(e), s);
        for (int r4 = 0; r4 < 4; ++r4) {
            printf("  smem row %d:", r4);
            for (int c = 0; c < 16; ++c) printf(" %.0f", o[r4 * 16 + c]);
            printf("\n");
        }
    }
    return 0;
}
