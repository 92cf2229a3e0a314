// common.cuh -- shared device helpers for the spidgpu kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/spidgpu_status.h"

namespace spidgpu {

constexpr int kWarp = 32;

// IEEE-exact scalar ops that the compiler may not contract into FMA. The
// reference is built for x86-64 without -march, so every `s += x*y` there is
// a rounded multiply followed by a rounded add (proj/src/dense_matrix.cpp:
// 136-140); these wrappers reproduce that bit-for-bit.
// Launch grid of the column gathers: x covers a column's rows (256-thread
// blocks, at most 32 per column), y the columns, grid-striding so the whole
// grid stays near 4096 blocks (148 SMs x ~28)
inline dim3 col_grid(int64_t nrows, int64_t ncols) {
    int64_t x = (nrows + 255) / 256;
    if (x > 32) x = 32;
    if (x < 1) x = 1;
    const int64_t ycap = 4096 / x;
    const int64_t y = ncols < 1 ? 1 : (ncols > ycap ? ycap : ncols);
    return dim3(static_cast<unsigned>(x), static_cast<unsigned>(y));
}

__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

// One 8x8x4 FP64 tensor-core MMA (SASS DMMA.8x8x4; sm_100a has no tcgen05
// f64 kind, SURVEY "HW"). Fragment layout (PTX ISA, m8n8k4 .f64):
//   a: row = lane>>2, k = lane&3      b: k = lane&3, col = lane>>2
//   c: row = lane>>2, cols 2*(lane&3) + {0,1}
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Explicit shared-window accesses (32-bit shared addresses), so realigned
// dynamic shared memory still compiles to LDS/STS rather than generic LD/ST.
__device__ __forceinline__ double2 lds128(uint32_t addr) {
    double2 v;
    asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];\n" : "=d"(v.x), "=d"(v.y) : "r"(addr));
    return v;
}

__device__ __forceinline__ void sts128(uint32_t addr, double a, double b) {
    asm volatile("st.shared.v2.f64 [%0], {%1, %2};\n" ::"r"(addr), "d"(a), "d"(b) : "memory");
}

// ---- mbarrier + TMA (cp.async.bulk.tensor) --------------------------------
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void fence_barrier_init() {
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
}

// 3D tiled TMA load global -> shared, completion on an mbarrier.
__device__ __forceinline__ void tma_load_3d(void* dst, const void* tmap, uint64_t* bar, int c0,
                                            int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes "
        "[%0], [%1, {%3, %4, %5}], [%2];\n" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// The same, multicast: the box lands at the same shared offset in every CTA
// of `mask` (cluster ranks) and signals each CTA's mbarrier at bar's offset.
__device__ __forceinline__ void tma_load_3d_mc(void* dst, const void* tmap, uint64_t* bar, int c0, int c1,
                                               int c2, uint16_t mask) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster "
        "[%0], [%1, {%3, %4, %5}], [%2], %6;\n" ::"r"(smem_u32(dst)),
        "l"(tmap), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
        : "memory");
}

// arrive on an mbarrier of another CTA of the cluster (shared::cluster
// address). Default (CTA-scope) release: it only publishes that this
// thread's earlier shared-memory READS are done (a slot-release), and those
// reads have already returned their values, so no cluster-scope fence
// (ERRBAR) is needed.
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_bar) {
    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];\n" ::"r"(cluster_bar) : "memory");
}

__device__ __forceinline__ void prefetch_tmap(const void* tmap) {
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(tmap) : "memory");
}

// ---- block reductions ---------------------------------------------------
// Argmax key for pivot selection: larger norm wins; on an exact tie the lower
// ORIGINAL column index wins (proj/src/qr.cpp:68). A total order, so any
// reduction tree returns the reference's choice.
__device__ __forceinline__ bool key_better(double na, int ia, double nb, int ib) {
    return na > nb || (na == nb && ia < ib);
}

__device__ __forceinline__ void warp_argmax(double& v, int& idx) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, off);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, off);
        if (key_better(ov, oi, v, idx)) {
            v = ov;
            idx = oi;
        }
    }
}

// The same order on integer keys, for the register CPQR whose MGS passes
// saturate the FP64 pipe (DSETP runs there too). A candidate's norm is
// non-negative or NaN, or -1.0 for "no live column"; for these the IEEE bit
// pattern read as a signed 64-bit integer orders exactly like the value (-1.0
// is negative, every norm is not), and NaN maps below everything: a NaN norm
// can never beat the -1.0 start of the double comparison either, so the
// chosen pivot is the same.
__device__ __forceinline__ long long norm_key(double v) {
    const long long b = __double_as_longlong(v);
    return (b & 0x7fffffffffffffffLL) > 0x7ff0000000000000LL ? (-0x7fffffffffffffffLL - 1) : b;
}
__device__ __forceinline__ bool key_better_k(long long ka, int ia, long long kb, int ib) {
    return ka > kb || (ka == kb && ia < ib);
}
__device__ __forceinline__ void warp_argmax_k(long long& k, int& idx) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const long long ok = __shfl_xor_sync(0xffffffffu, k, off);
        const int oi = __shfl_xor_sync(0xffffffffu, idx, off);
        if (key_better_k(ok, oi, k, idx)) {
            k = ok;
            idx = oi;
        }
    }
}

__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, off));
    return v;
}

__device__ __forceinline__ int warp_or(int v) { return __any_sync(0xffffffffu, v) ? 1 : 0; }

}  // namespace spidgpu
