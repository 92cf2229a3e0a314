// crc.cu -- CRC-32/ISO-HDLC (zlib polynomial) of device buffers.
//
// The archive format checksums every section (proj/src/archive.cpp:83-98,
// 168-178); block sections hold the skeleton matrices, i.e. gigabytes per
// GPU, which the reference walks bit by bit on one core. Here:
//   1. each thread computes the raw (init 0, no final xor) CRC of one
//      SEG-byte segment with slice-by-8 tables in shared memory; segments are
//      aligned to the END of the message and the first one is zero-padded at
//      the front, which leaves a raw CRC unchanged;
//   2. segment CRCs are combined with the linearity of CRCs over GF(2):
//      raw(A || B) = raw(A) * x^(8|B|) mod P  xor  raw(B) -- a warp-shuffle
//      and shared-memory tree inside each block, then the same fold over the
//      block results in a second kernel;
//   3. the standard init/final-xor conditioning is applied once:
//      crc(M) = ~(raw(M) xor 0xFFFFFFFF * x^(8|M|) mod P).
// Result: bit-identical to the reference's crc32().
#include "common.cuh"
#include "kernels.h"

namespace spidgpu {

namespace {

constexpr uint32_t kPoly = 0xEDB88320u;  // reflected 0x04C11DB7
constexpr int kSeg = 1024;               // bytes per thread
constexpr int kThreadsC = 256;           // segments per block

struct XLevels {
    uint32_t v[8];  // x^(8 * SEG * 2^j) mod P per combine level (by value)
};

// a * b mod P with bit 31 = x^0 (reflected), the usual GF(2) shift-and-add.
__host__ __device__ inline uint32_t multmodp(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ kPoly : b >> 1;
    }
    return p;
}

// x^(8 * nbytes) mod P.
__host__ __device__ inline uint32_t xpow8(uint64_t nbytes) {
    uint32_t sq = 1u << 30;  // x^1
    // x^8 = x^(2^3): square three times
    for (int i = 0; i < 3; ++i) sq = multmodp(sq, sq);
    uint32_t p = 1u << 31;  // x^0
    while (nbytes) {
        if (nbytes & 1) p = multmodp(sq, p);
        sq = multmodp(sq, sq);
        nbytes >>= 1;
    }
    return p;
}

__global__ void __launch_bounds__(kThreadsC)
    crc_segments_kernel(const uint8_t* __restrict__ data, int64_t nbytes, int64_t nseg,
                        const XLevels lv, uint32_t* __restrict__ block_crc) {
    __shared__ uint32_t T[8][256];
    __shared__ uint32_t part[kThreadsC / kWarp];
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int b = 0; b < 8; ++b) c = (c & 1) ? (c >> 1) ^ kPoly : c >> 1;
        T[0][i] = c;
    }
    __syncthreads();
    for (int t = 1; t < 8; ++t) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x)
            T[t][i] = (T[t - 1][i] >> 8) ^ T[0][T[t - 1][i] & 0xff];
        __syncthreads();
    }
    // segment g covers bytes [nbytes - (nseg - g) * SEG, + SEG); negative = zero pad
    const int64_t g = static_cast<int64_t>(blockIdx.x) * kThreadsC + threadIdx.x;
    uint32_t c = 0;
    if (g < nseg) {
        const int64_t start = nbytes - (nseg - g) * kSeg;
        const bool aligned = start >= 0 && ((reinterpret_cast<uintptr_t>(data) + start) & 7) == 0;
        if (aligned) {
            const uint64_t* w64 = reinterpret_cast<const uint64_t*>(data + start);
#pragma unroll 4
            for (int i = 0; i < kSeg / 8; ++i) {
                const uint64_t w = __ldg(w64 + i);
                c ^= static_cast<uint32_t>(w);
                const uint32_t hi = static_cast<uint32_t>(w >> 32);
                c = T[7][c & 0xff] ^ T[6][(c >> 8) & 0xff] ^ T[5][(c >> 16) & 0xff] ^ T[4][c >> 24] ^
                    T[3][hi & 0xff] ^ T[2][(hi >> 8) & 0xff] ^ T[1][(hi >> 16) & 0xff] ^ T[0][hi >> 24];
            }
        } else {
            for (int i = 0; i < kSeg; ++i) {
                const int64_t at = start + i;
                const uint32_t byte = at >= 0 ? __ldg(data + at) : 0u;
                c = T[0][(c ^ byte) & 0xff] ^ (c >> 8);
            }
        }
    }
    // combine consecutive segments: level j merges runs of 2^j segments
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
        const uint32_t other = __shfl_down_sync(0xffffffffu, c, 1 << j);
        if ((lane & ((2 << j) - 1)) == 0) c = multmodp(lv.v[j], c) ^ other;
    }
    if (lane == 0) part[warp] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t acc = part[0];
        for (int w = 1; w < kThreadsC / kWarp; ++w) acc = multmodp(lv.v[5], acc) ^ part[w];
        block_crc[blockIdx.x] = acc;
    }
}

// fold the per-block raw CRCs in order, then condition: one thread (tiny work)
__global__ void crc_finish_kernel(const uint32_t* block_crc, int64_t nblocks, uint32_t xblock,
                                  uint32_t xall, uint32_t* out) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint32_t acc = 0;
    for (int64_t b = 0; b < nblocks; ++b) acc = multmodp(xblock, acc) ^ block_crc[b];
    *out = ~(acc ^ multmodp(xall, 0xFFFFFFFFu));
}

}  // namespace

uint32_t crc32_combine_host(uint32_t crc_a, uint32_t crc_b, uint64_t len_b) {
    // standard-conditioned CRC of A||B from crc(A), crc(B) and |B| (zlib's
    // crc32_combine identity): the init/final xors cancel as below
    return multmodp(xpow8(len_b), crc_a) ^ crc_b;
}

cudaError_t launch_crc32(const uint8_t* data, int64_t nbytes, uint32_t* block_scratch,
                         uint32_t* out, cudaStream_t stream) {
    const int64_t nseg = nbytes > 0 ? (nbytes + kSeg - 1) / kSeg : 1;
    const int64_t nblocks = (nseg + kThreadsC - 1) / kThreadsC;
    // pad the segment count to whole blocks at the FRONT (zero segments)
    const int64_t nseg_padded = nblocks * kThreadsC;
    // level j < 5 merges runs of 2^j segments; level 5 merges whole warps
    XLevels lv;
    for (int j = 0; j < 8; ++j) lv.v[j] = xpow8(static_cast<uint64_t>(kSeg) << j);
    crc_segments_kernel<<<static_cast<unsigned>(nblocks), kThreadsC, 0, stream>>>(
        data, nbytes, nseg_padded, lv, block_scratch);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    crc_finish_kernel<<<1, 32, 0, stream>>>(block_scratch, nblocks,
                                            xpow8(static_cast<uint64_t>(kSeg) * kThreadsC),
                                            xpow8(static_cast<uint64_t>(nbytes)), out);
    return cudaGetLastError();
}

int64_t crc32_scratch_words(int64_t nbytes) {
    const int64_t nseg = nbytes > 0 ? (nbytes + kSeg - 1) / kSeg : 1;
    return (nseg + kThreadsC - 1) / kThreadsC;
}

}  // namespace spidgpu
