// philox.cuh -- counter-based Gaussian generator for the in-kernel sketch.
//
// Omega_s(r, k) of subdomain s is a pure function of (seed, s, r, k), so any
// warp can generate exactly the fragment values it feeds to the tensor core,
// the sketch kernel never reads Omega from HBM (performance mode), and
// spidgpu_philox_omega() can materialise the identical matrix for an oracle.
//
// Philox4x32-7 (Salmon et al., SC'11): counter {k/8, r, s_lo, s_hi}, key
// {seed_lo, seed_hi}; the 8 16-bit halves of the output select entries of a
// 4096-quantile table of N(0, 1) rounded to multiples of 1/32 (omega_table.h),
// so Omega_s(r, k) = Q / 32 with an integer |Q| <= 117. Those entries are
// exact in fp64 (the DMMA sketch) and in int8 (the integer-sliced sketch,
// sketch_i8.cu), so both kernels contract the same Omega.
#pragma once

#include <stdint.h>

#include "omega_table.h"

namespace spidgpu {

struct Philox4 {
    uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ void philox_round(Philox4& c, uint32_t k0, uint32_t k1) {
    const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
#ifdef __CUDA_ARCH__
    const uint32_t hi0 = __umulhi(M0, c.x), lo0 = M0 * c.x;
    const uint32_t hi1 = __umulhi(M1, c.z), lo1 = M1 * c.z;
#else
    const uint64_t p0 = (uint64_t)M0 * c.x, p1 = (uint64_t)M1 * c.z;
    const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
    c = Philox4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
}

template <int ROUNDS>
__host__ __device__ __forceinline__ Philox4 philox4x32(Philox4 c, uint32_t k0, uint32_t k1) {
    const uint32_t W0 = 0x9E3779B9u, W1 = 0xBB67AE85u;
#pragma unroll
    for (int i = 0; i < ROUNDS; ++i) {
        philox_round(c, k0, k1);
        k0 += W0;
        k1 += W1;
    }
    return c;
}

// Rounds used for Omega: Philox4x32-7 passes TestU01 BigCrush (Salmon et al.,
// SC'11, Table 2) and keeps the producer warps off the sketch's critical path.
constexpr int kOmegaRounds = 7;

// Quantile table of the discretised Gaussian (tools/gen_omega_table.py). One
// copy per translation unit (no relocatable device code); 4 KiB.
static __device__ __align__(16) const int8_t kOmegaQ[1 << kOmegaTableBits] = SPIDGPU_OMEGA_TABLE_INIT;

// The 16-bit Philox outputs of one call: Omega_s(r, 8*ko + j) = Q[u_j >> 4] / 32
// for j = 0..7, u_j = 16-bit half (j & 1) of output word j / 2. Counter
// {ko, r, s_lo, s_hi}, key {seed_lo, seed_hi}.
__device__ __forceinline__ Philox4 omega_bits8(uint64_t seed, uint64_t s, uint32_t r, uint32_t ko) {
    return philox4x32<kOmegaRounds>(
        Philox4{ko, r, static_cast<uint32_t>(s), static_cast<uint32_t>(s >> 32)},
        static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
}

__device__ __forceinline__ uint32_t omega_u16(const Philox4& v, int j) {
    const uint32_t w = j < 2 ? v.x : j < 4 ? v.y : j < 6 ? v.z : v.w;
    return (j & 1) ? (w >> 16) : (w & 0xffffu);
}

// Eight integer entries Q (Omega = Q / 32) for Omega_s(r, 8*ko + 0..7), read
// through `tab` (the table in shared memory, or kOmegaQ itself).
__device__ __forceinline__ void omega_q8(uint64_t seed, uint64_t s, uint32_t r, uint32_t ko,
                                         const int8_t* tab, int q[8]) {
    const Philox4 v = omega_bits8(seed, s, r, ko);
#pragma unroll
    for (int j = 0; j < 8; ++j) q[j] = tab[omega_u16(v, j) >> (16 - kOmegaTableBits)];
}

// The same entries as doubles (exact: |Q| <= 117, scaled by 2^-5).
__device__ __forceinline__ void omega_values8(uint64_t seed, uint64_t s, uint32_t r, uint32_t ko,
                                              const int8_t* tab, double out[8]) {
    int q[8];
    omega_q8(seed, s, r, ko, tab, q);
#pragma unroll
    for (int j = 0; j < 8; ++j) out[j] = static_cast<double>(q[j]) * (1.0 / (1 << kOmegaScaleLog2));
}

// Four N(0,1) samples (Box-Muller in fp32 on the SFU, widened to fp64) from
// counter {kq, r, s_lo, s_hi}: the additive noise of the synthetic fields.
__device__ __forceinline__ void normals4_boxmuller(uint64_t seed, uint64_t s, uint32_t r, uint32_t kq,
                                                   double out[4]) {
    const Philox4 v = philox4x32<kOmegaRounds>(
        Philox4{kq, r, static_cast<uint32_t>(s), static_cast<uint32_t>(s >> 32)},
        static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    const float kInv = 2.3283064365386963e-10f;  // 2^-32
    const float u1a = (static_cast<float>(v.x) + 1.0f) * kInv;  // (0, 1]
    const float u2a = static_cast<float>(v.y) * kInv;
    const float u1b = (static_cast<float>(v.z) + 1.0f) * kInv;
    const float u2b = static_cast<float>(v.w) * kInv;
    const float xa = fmaxf(-2.0f * __logf(u1a), 1e-30f);
    const float xb = fmaxf(-2.0f * __logf(u1b), 1e-30f);
    const float ra = xa * rsqrtf(xa);
    const float rb = xb * rsqrtf(xb);
    float sa, ca, sb, cb;
    __sincosf(6.2831853071795865f * u2a, &sa, &ca);
    __sincosf(6.2831853071795865f * u2b, &sb, &cb);
    out[0] = static_cast<double>(ra * ca);
    out[1] = static_cast<double>(ra * sa);
    out[2] = static_cast<double>(rb * cb);
    out[3] = static_cast<double>(rb * sb);
}

}  // namespace spidgpu
