// cluster.cuh -- thread-block-cluster helpers shared by the CTA-pair kernels
// (cpqr_pair.cu, cpqr_reg_pair.cu): rank, barrier, peer addresses, 16-byte
// st.async into a peer's mbarrier-counted slot, cluster-scope waits.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace spidgpu {
namespace cluster {

__device__ __forceinline__ uint32_t ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
// every thread of every CTA of the cluster arrives and waits
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t peer) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(peer));
    return r;
}
// 16 bytes into the peer's shared memory, completing on its mbarrier
__device__ __forceinline__ void st_async16(uint32_t raddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                           uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];\n" ::"r"(
                     raddr),
                 "r"(a), "r"(b), "r"(c), "r"(d), "r"(rbar)
                 : "memory");
}
// wait with cluster-scope acquire (the data came from the peer by st.async)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n.reg .pred p;\nWAITC_%=:\n"
        "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAITC_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}


}  // namespace cluster
}  // namespace spidgpu
