// philox.cuh -- counter-based Gaussian generator for the in-kernel sketch.
//
// Omega_s(r, k) of subdomain s is a pure function of (seed, s, r, k), so any
// warp can generate exactly the fragment values it feeds to the tensor core,
// the sketch kernel never reads Omega from HBM (performance mode), and
// spidgpu_philox_omega() can materialise the identical matrix for an oracle.
//
// Philox4x32-7 (Salmon et al., SC'11): counter {k/4, r, s_lo, s_hi}, key
// {seed_lo, seed_hi}; the 4 outputs become Omega_s(r, 4*(k/4) + 0..3) via two
// Box-Muller transforms in fp32 with the SFU intrinsics (the sketch needs a
// Gaussian-distributed Omega, not fp64-accurate normals), widened to fp64.
#pragma once

#include <stdint.h>

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

// Four N(0,1) samples for Omega_s(r, 4*kq + 0..3).
__device__ __forceinline__ void omega_normals4(uint64_t seed, uint64_t s, uint32_t r, uint32_t kq,
                                               double out[4]) {
    const Philox4 v = philox4x32<kOmegaRounds>(
        Philox4{kq, r, static_cast<uint32_t>(s), static_cast<uint32_t>(s >> 32)},
        static_cast<uint32_t>(seed), static_cast<uint32_t>(seed >> 32));
    const float kInv = 2.3283064365386963e-10f;  // 2^-32
    const float u1a = (static_cast<float>(v.x) + 1.0f) * kInv;  // (0, 1]
    const float u2a = static_cast<float>(v.y) * kInv;
    const float u1b = (static_cast<float>(v.z) + 1.0f) * kInv;
    const float u2b = static_cast<float>(v.w) * kInv;
    // r = sqrt(-2 ln u) as x * rsqrt(x): MUFU.RSQ, no IEEE-sqrt slow path
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
