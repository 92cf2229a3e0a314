// archive.cu -- device side of the archive codec (proj/src/archive.cpp).
//
// The archive of a field is assembled in HBM and leaves the GPU with one
// device-to-host copy:
//   gather_block_rows   B_b = A(rows of block b restricted to the coarse set J)
//                       -- select_rows + subsample of compress_structured_batch
//   sort_union          union_indices = sorted skeleton indices
//   pack_blocks         block sections: u64 length | payload | (crc), payload =
//                       u8 coarse | u64 array union | u64 array skeleton idx |
//                       f64 matrix skeleton | f64 matrix coeffs
//                       (archive.cpp:100-116, 193-212), all little-endian
//   crc_sections        CRC-32 of every section payload (archive.cpp:83-98)
// and decompress (archive.cpp:281-303) runs as
//   unpack_blocks       f64 matrices of each section -> padded batch buffers
//   (interp lift of coarse skeletons, interp.cu)
//   recon_scatter       out(rows_b, :) = F_b * C_b, the reference matmul's
//                       j-k-i order with its zero skip (dense_matrix.cpp:
//                       38-53), rounded per operation -> bit-identical, written
//                       straight into the assembled matrix (blocking.cpp:219-241).
#include <vector>

#include "common.cuh"
#include "kernels.h"

namespace spidgpu {

namespace {

constexpr uint32_t kPolyR = 0xEDB88320u;

__device__ inline uint32_t multmodp_d(uint32_t a, uint32_t b) {
    uint32_t m = 1u << 31, p = 0;
    for (;;) {
        if (a & m) {
            p ^= b;
            if ((a & (m - 1)) == 0) break;
        }
        m >>= 1;
        b = (b & 1) ? (b >> 1) ^ kPolyR : b >> 1;
    }
    return p;
}

__device__ inline uint32_t xpow8_d(uint64_t nbytes) {
    uint32_t sq = 1u << 30;
    for (int i = 0; i < 3; ++i) sq = multmodp_d(sq, sq);
    uint32_t p = 1u << 31;
    while (nbytes) {
        if (nbytes & 1) p = multmodp_d(sq, p);
        sq = multmodp_d(sq, sq);
        nbytes >>= 1;
    }
    return p;
}

__global__ void gather_block_rows_kernel(const double* __restrict__ A, int64_t lda,
                                         const int64_t* __restrict__ rel, int64_t nrows,
                                         const int64_t* __restrict__ bases, int64_t nb, int64_t n,
                                         double* __restrict__ B, int64_t ldb, int64_t strideB) {
    // rows in x, (block, column) pairs in y: one division per column
    // instead of three 64-bit divisions per element
    for (int64_t bj = blockIdx.y; bj < nb * n; bj += gridDim.y) {
        const int64_t b = bj / n, j = bj - b * n;
        const double* src = A + j * lda + bases[b];
        double* dst = B + b * strideB + j * ldb;
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nrows;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            dst[i] = __ldg(src + rel[i]);
    }
}

__global__ void sort_union_kernel(const int64_t* __restrict__ idx, int64_t kcap,
                                  const int64_t* __restrict__ rank, int64_t nb,
                                  int64_t* __restrict__ uni) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nb) return;
    const int64_t k = rank[b];
    const int64_t* src = idx + b * kcap;
    int64_t* dst = uni + b * kcap;
    for (int64_t t = 0; t < k; ++t) {  // insertion sort, k <= a few hundred
        const int64_t v = src[t];
        int64_t u = t;
        while (u > 0 && dst[u - 1] > v) {
            dst[u] = dst[u - 1];
            --u;
        }
        dst[u] = v;
    }
}

__device__ __forceinline__ void put_u64(uint8_t* p, uint64_t v) {
#pragma unroll
    for (int b = 0; b < 8; ++b) p[b] = static_cast<uint8_t>(v >> (8 * b));
}

__device__ __forceinline__ uint64_t get_u64(const uint8_t* p) {
    uint64_t v = 0;
#pragma unroll
    for (int b = 0; b < 8; ++b) v |= static_cast<uint64_t>(__ldg(p + b)) << (8 * b);
    return v;
}

// One thread per 8-byte item of a section (item 1 is the coarse byte). Items
// after the coarse byte: nu | union[nu] | k | sel[k] | mc | k | skel[mc*k] |
// k | n | coeffs[k*n], each a u64 / f64 at payload offset 1 + 8*(item - 2).
__global__ void pack_blocks_kernel(const PackBlock* __restrict__ blocks, int64_t nblocks,
                                   uint8_t* __restrict__ out) {
    for (int64_t b = blockIdx.y; b < nblocks; b += gridDim.y) {
        const PackBlock d = blocks[b];
        const int64_t k = d.k, nu = d.nu, mck = d.mc * d.k, kn = d.k * d.n;
        const int64_t items = 8 + nu + k + mck + kn;
        const int64_t payload = 49 + 8 * nu + 8 * k + 8 * mck + 8 * kn;
        const int64_t s0 = nu + k + 4;  // first skeleton item (q index)
        for (int64_t it = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; it < items;
             it += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            uint8_t* sec = out + d.sec_off;
            if (it == 0) {
                put_u64(sec, static_cast<uint64_t>(payload));
                continue;
            }
            if (it == 1) {
                sec[8] = d.coarse ? 1 : 0;
                continue;
            }
            const int64_t q = it - 2;
            uint64_t v;
            if (q == 0) {
                v = static_cast<uint64_t>(nu);
            } else if (q <= nu) {
                v = static_cast<uint64_t>(d.uni[q - 1]);
            } else if (q == nu + 1) {
                v = static_cast<uint64_t>(k);
            } else if (q <= nu + k + 1) {
                v = static_cast<uint64_t>(d.sel[q - nu - 2]);
            } else if (q == nu + k + 2) {
                v = static_cast<uint64_t>(d.mc);
            } else if (q == nu + k + 3) {
                v = static_cast<uint64_t>(k);
            } else if (q < s0 + mck) {
                const uint32_t e = static_cast<uint32_t>(q - s0);
                const uint32_t mc = static_cast<uint32_t>(d.mc);
                v = __double_as_longlong(__ldg(d.skel + static_cast<int64_t>(e / mc) * d.ld_s + e % mc));
            } else if (q == s0 + mck) {
                v = static_cast<uint64_t>(k);
            } else if (q == s0 + mck + 1) {
                v = static_cast<uint64_t>(d.n);
            } else {
                const uint32_t e = static_cast<uint32_t>(q - (s0 + mck + 2));
                const uint32_t kk = static_cast<uint32_t>(k);
                v = __double_as_longlong(__ldg(d.coeffs + static_cast<int64_t>(e / kk) * d.ld_c + e % kk));
            }
            put_u64(sec + 9 + 8 * q, v);
        }
    }
}

// Raw CRC (state 0, no final xor) of bytes [lo, hi).
__device__ uint32_t crc_raw_range(const uint8_t* __restrict__ data, int64_t lo, int64_t hi,
                                  const uint32_t (*T)[256]) {
    uint32_t c = 0;
    int64_t p = lo;
    while (p < hi && (reinterpret_cast<uintptr_t>(data + p) & 7)) {
        c = T[0][(c ^ __ldg(data + p)) & 0xff] ^ (c >> 8);
        ++p;
    }
    for (; p + 8 <= hi; p += 8) {
        const uint64_t w = __ldg(reinterpret_cast<const unsigned long long*>(data + p));
        c ^= static_cast<uint32_t>(w);
        const uint32_t h = static_cast<uint32_t>(w >> 32);
        c = T[7][c & 0xff] ^ T[6][(c >> 8) & 0xff] ^ T[5][(c >> 16) & 0xff] ^ T[4][c >> 24] ^
            T[3][h & 0xff] ^ T[2][(h >> 8) & 0xff] ^ T[1][(h >> 16) & 0xff] ^ T[0][h >> 24];
    }
    for (; p < hi; ++p) c = T[0][(c ^ __ldg(data + p)) & 0xff] ^ (c >> 8);
    return c;
}

constexpr int kCrcThreads = 256;

// CRC tables (slice-by-8) built once per CTA in shared memory.
__device__ void build_crc_tables(uint32_t (*T)[256]) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) {
        uint32_t c = i;
        for (int b = 0; b < 8; ++b) c = (c & 1) ? (c >> 1) ^ kPolyR : c >> 1;
        T[0][i] = c;
    }
    __syncthreads();
    for (int t = 1; t < 8; ++t) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x)
            T[t][i] = (T[t - 1][i] >> 8) ^ T[0][T[t - 1][i] & 0xff];
        __syncthreads();
    }
}

// Raw CRC of each part (<= kCrcPart bytes, end-aligned inside its section):
// 256 contiguous end-aligned chunks per part, combined through x^(8*len)
// shifts (crc.cu explains the identities).
__global__ void __launch_bounds__(kCrcThreads)
    crc_parts_kernel(const uint8_t* __restrict__ data, const CrcPart* __restrict__ parts,
                     int64_t nparts, uint32_t* __restrict__ part_crc) {
    __shared__ uint32_t T[8][256];
    __shared__ uint32_t part[kCrcThreads / kWarp];
    build_crc_tables(T);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int64_t C = kCrcPart / kCrcThreads;
    uint32_t X0 = xpow8_d(static_cast<uint64_t>(C));
    for (int64_t q = blockIdx.x; q < nparts; q += gridDim.x) {
        const int64_t begin = parts[q].begin, end = parts[q].end;
        int64_t lo = end - (kCrcThreads - threadIdx.x) * C;
        const int64_t hi = lo + C;
        if (lo < begin) lo = begin;
        uint32_t c = lo < hi ? crc_raw_range(data, lo, hi, T) : 0u;
        uint32_t X = X0;
#pragma unroll
        for (int j = 0; j < 5; ++j) {
            const uint32_t other = __shfl_down_sync(0xffffffffu, c, 1 << j);
            if ((lane & ((2 << j) - 1)) == 0) c = multmodp_d(X, c) ^ other;
            X = multmodp_d(X, X);
        }
        if (lane == 0) part[warp] = c;
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t acc = part[0];
            for (int w = 1; w < kCrcThreads / kWarp; ++w) acc = multmodp_d(X, acc) ^ part[w];
            part_crc[q] = acc;
        }
        __syncthreads();
    }
}

// One block per section: part q's raw CRC shifted past the (full) parts after
// it, x^(8 kCrcPart (last - q)) * crc_q, XOR-reduced -- the same GF(2) sum the
// sequential fold acc = x^(8 kCrcPart) acc ^ crc_q forms, so the same bits;
// then conditioned, optionally written after the payload.
__global__ void crc_fold_kernel(const CrcSection* __restrict__ secs, int64_t nsec,
                                const int64_t* __restrict__ first_part, const uint32_t* __restrict__ part_crc,
                                uint32_t* __restrict__ crc_out, uint8_t* write_back) {
    __shared__ uint32_t wred[32];
    const int64_t s = blockIdx.x;
    if (s >= nsec) return;
    const uint32_t xpart = xpow8_d(static_cast<uint64_t>(kCrcPart));
    const int64_t f = first_part[s], l = first_part[s + 1];
    uint32_t acc = 0;
    for (int64_t q = f + threadIdx.x; q < l; q += blockDim.x) {
        uint32_t pw = 1u << 31, sq = xpart;  // xpart^(l - 1 - q)
        for (uint64_t e = static_cast<uint64_t>(l - 1 - q); e; e >>= 1) {
            if (e & 1) pw = multmodp_d(sq, pw);
            sq = multmodp_d(sq, sq);
        }
        acc ^= multmodp_d(pw, part_crc[q]);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc ^= __shfl_xor_sync(0xffffffffu, acc, off);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) wred[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        acc = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) acc ^= wred[w];
        const int64_t len = secs[s].len;
        const uint32_t crc = ~(acc ^ multmodp_d(xpow8_d(static_cast<uint64_t>(len)), 0xFFFFFFFFu));
        crc_out[s] = crc;
        if (write_back) {
            const int64_t end = secs[s].begin + len;
#pragma unroll
            for (int b = 0; b < 4; ++b) write_back[end + b] = static_cast<uint8_t>(crc >> (8 * b));
        }
    }
}

__global__ void unpack_blocks_kernel(const uint8_t* __restrict__ bytes,
                                     const UnpackBlock* __restrict__ blocks, int64_t nblocks) {
    for (int64_t b = blockIdx.y; b < nblocks; b += gridDim.y) {
        const UnpackBlock d = blocks[b];
        const int64_t mck = d.mc * d.k, total = mck + d.k * d.n;
        for (int64_t it = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; it < total;
             it += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            if (it < mck) {
                const int64_t col = it / d.mc, row = it % d.mc;
                d.skel[col * d.ld_s + row] = __longlong_as_double(get_u64(bytes + d.skel_off + 8 * it));
            } else {
                const int64_t e = it - mck;
                const int64_t col = e / d.k, row = e % d.k;
                d.coeffs[col * d.ld_c + row] =
                    __longlong_as_double(get_u64(bytes + d.coef_off + 8 * e));
            }
        }
    }
}

constexpr int kReconThreads = 128;
constexpr int kReconRPT = 2;  // rows per thread: each shared C value feeds two rows
constexpr int kReconRows = kReconThreads * kReconRPT;
static_assert(kReconRPT == 2, "recon_scatter_kernel unrolls two rows");
constexpr int kReconCols = 64;
constexpr int kReconNJ = 16;

// out(bases[b] + rel[i], j) = sum_t F_b(i, t) * C_b(t, j) in the reference
// matmul's order: t ascending, products with C == 0 skipped, every multiply
// and add rounded on its own (DMUL + DADD: the FP64 pipe's two instructions
// per term are the bound). The zero skip is decided once per (t, column)
// tile entry: a 64-bit nonzero mask per t in shared memory, tested with
// integer ops and, for 16 nonzero columns (the common case), skipped
// entirely by a block-uniform branch.
#ifndef SPIDGPU_RECON_MINB
#define SPIDGPU_RECON_MINB 5  // 5 CTAs per SM (<= 102 registers, no spills): 3.40 ms vs 3.92 at 1 (config-3 archive)
#endif
__global__ void __launch_bounds__(kReconThreads, SPIDGPU_RECON_MINB)
    recon_scatter_kernel(const double* __restrict__ F, int64_t ldf, int64_t strideF,
                         const double* __restrict__ Cm, int64_t kcap, int64_t strideC,
                         const int64_t* __restrict__ rank, int64_t mb, int64_t n,
                         const int64_t* __restrict__ rel, const int64_t* __restrict__ bases,
                         double* __restrict__ out, int64_t ldo) {
    extern __shared__ double cs[];  // [kcap][kReconCols], then the masks [kcap]
    unsigned long long* nzm = reinterpret_cast<unsigned long long*>(cs + kcap * kReconCols);
    const int64_t b = blockIdx.y;
    const int64_t i0 = blockIdx.x * static_cast<int64_t>(kReconRows) + threadIdx.x;
    const int k = static_cast<int>(rank[b]);
    const double* Fb = F + b * strideF;
    const double* Cb = Cm + b * strideC;
    int64_t orow[kReconRPT];
    bool live[kReconRPT];
#pragma unroll
    for (int r = 0; r < kReconRPT; ++r) {
        const int64_t i = i0 + r * kReconThreads;
        live[r] = i < mb;
        orow[r] = live[r] ? bases[b] + rel[i] : 0;
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int64_t c0 = 0; c0 < n; c0 += kReconCols) {
        const int ncol = static_cast<int>(n - c0 < kReconCols ? n - c0 : kReconCols);
        __syncthreads();
        for (int e = threadIdx.x; e < k * kReconCols; e += kReconThreads) {
            const int t = e / kReconCols, jj = e % kReconCols;
            cs[t * kReconCols + jj] = jj < ncol ? Cb[(c0 + jj) * kcap + t] : 0.0;
        }
        __syncthreads();
        // nonzero mask of row t: two 32-column ballots per warp
        for (int t = warp; t < k; t += kReconThreads / 32) {
            const unsigned lo = __ballot_sync(0xffffffffu, cs[t * kReconCols + lane] != 0.0);
            const unsigned hi = __ballot_sync(0xffffffffu, cs[t * kReconCols + 32 + lane] != 0.0);
            if (lane == 0) nzm[t] = (static_cast<unsigned long long>(hi) << 32) | lo;
        }
        __syncthreads();
        if (!live[0]) continue;
        // rows past mb (second row of the last tile) read row i0 again and are not stored
        const double* fp0 = Fb + i0;
        const double* fp1 = Fb + (live[1] ? i0 + kReconThreads : i0);
        for (int j0 = 0; j0 < ncol; j0 += kReconNJ) {
            double acc0[kReconNJ], acc1[kReconNJ];
#pragma unroll
            for (int u = 0; u < kReconNJ; ++u) acc0[u] = acc1[u] = 0.0;
            // F(i, t) of the next t is loaded while this t's products run
            double a0n = k > 0 ? __ldg(fp0) : 0.0, a1n = k > 0 ? __ldg(fp1) : 0.0;
            for (int t = 0; t < k; ++t) {
                const double a0 = a0n, a1 = a1n;
                if (t + 1 < k) {
                    a0n = __ldg(fp0 + (t + 1) * ldf);
                    a1n = __ldg(fp1 + (t + 1) * ldf);
                }
                const double* ct = cs + t * kReconCols + j0;
                const uint32_t nz = static_cast<uint32_t>(nzm[t] >> j0) & 0xffffu;
                if (nz == 0xffffu) {
#pragma unroll
                    for (int u = 0; u < kReconNJ; ++u) {
                        const double cv = ct[u];
                        acc0[u] = add_rn(acc0[u], mul_rn(a0, cv));
                        acc1[u] = add_rn(acc1[u], mul_rn(a1, cv));
                    }
                } else {
#pragma unroll
                    for (int u = 0; u < kReconNJ; ++u)
                        if ((nz >> u) & 1u) {
                            const double cv = ct[u];
                            acc0[u] = add_rn(acc0[u], mul_rn(a0, cv));
                            acc1[u] = add_rn(acc1[u], mul_rn(a1, cv));
                        }
                }
            }
#pragma unroll
            for (int u = 0; u < kReconNJ; ++u)
                if (j0 + u < ncol) {
                    out[(c0 + j0 + u) * ldo + orow[0]] = acc0[u];
                    if (live[1]) out[(c0 + j0 + u) * ldo + orow[1]] = acc1[u];
                }
        }
    }
}

__device__ __forceinline__ bool nonfinite_bits(double v) {
    return (__double_as_longlong(v) & 0x7ff0000000000000LL) == 0x7ff0000000000000LL;
}

// blockIdx.y walks columns, threads walk rows: no per-element index division;
// the block of a non-finite entry is located only on a hit.
__device__ __noinline__ void flag_block(int64_t r, const BlockGridDev& g, int32_t* flags) {
    int64_t rem = r, blk = 0, mul = 1;
    for (int ax = 0; ax < g.naxes; ++ax) {
        const int64_t coord = rem % g.dims[ax];
        rem /= g.dims[ax];
        int64_t seg = coord / g.seg_base[ax];
        if (seg >= g.seg_count[ax]) seg = g.seg_count[ax] - 1;
        blk += seg * mul;
        mul *= g.seg_count[ax];
    }
    atomicExch(flags + blk, 1);
}

// kVec: 16-byte loads, four in flight per thread (lda even, A 16-byte aligned).
template <bool kVec>
__global__ void nonfinite_blocks_kernel(const double* __restrict__ A, int64_t lda, int64_t m,
                                        int64_t n, BlockGridDev g, int32_t* __restrict__ flags) {
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    for (int64_t j = blockIdx.y; j < n; j += gridDim.y) {
        const double* col = A + j * lda;
        if (kVec) {
            const double2* c2 = reinterpret_cast<const double2*>(col);
            const int64_t m2 = m / 2;
            int64_t r = t0;
            for (; r + 3 * stride < m2; r += 4 * stride) {
                double2 v[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) v[u] = __ldcs(c2 + r + u * stride);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (nonfinite_bits(v[u].x)) flag_block(2 * (r + u * stride), g, flags);
                    if (nonfinite_bits(v[u].y)) flag_block(2 * (r + u * stride) + 1, g, flags);
                }
            }
            for (; r < m2; r += stride) {
                const double2 v = __ldcs(c2 + r);
                if (nonfinite_bits(v.x)) flag_block(2 * r, g, flags);
                if (nonfinite_bits(v.y)) flag_block(2 * r + 1, g, flags);
            }
            if ((m & 1) && t0 == 0 && nonfinite_bits(col[m - 1])) flag_block(m - 1, g, flags);
        } else {
            for (int64_t r = t0; r < m; r += stride)
                if (nonfinite_bits(__ldcs(col + r))) flag_block(r, g, flags);
        }
    }
}

}  // namespace

cudaError_t launch_gather_block_rows(const double* A, int64_t lda, const int64_t* rel,
                                     int64_t nrows, const int64_t* bases, int64_t nb, int64_t n,
                                     double* B, int64_t ldb, int64_t strideB, cudaStream_t st) {
    gather_block_rows_kernel<<<col_grid(nrows, nb * n), 256, 0, st>>>(A, lda, rel, nrows, bases, nb, n, B,
                                                                      ldb, strideB);
    return cudaGetLastError();
}

cudaError_t launch_sort_union(const int64_t* idx, int64_t kcap, const int64_t* rank, int64_t nb,
                              int64_t* uni, cudaStream_t st) {
    sort_union_kernel<<<static_cast<unsigned>((nb + 127) / 128), 128, 0, st>>>(idx, kcap, rank, nb, uni);
    return cudaGetLastError();
}

cudaError_t launch_pack_blocks(const PackBlock* blocks, int64_t nblocks, int64_t max_items,
                               uint8_t* out, cudaStream_t st) {
    const unsigned gy = static_cast<unsigned>(nblocks < 65535 ? nblocks : 65535);
    int64_t gx = (max_items + 255) / 256;
    const int64_t cap = (148 * 32 + gy - 1) / gy;
    if (gx > cap) gx = cap;
    if (gx < 1) gx = 1;
    pack_blocks_kernel<<<dim3(static_cast<unsigned>(gx), gy), 256, 0, st>>>(blocks, nblocks, out);
    return cudaGetLastError();
}

void crc_plan_parts(const CrcSection* secs, int64_t nsec, std::vector<CrcPart>* parts,
                    std::vector<int64_t>* first_part) {
    parts->clear();
    first_part->assign(1, 0);
    for (int64_t s = 0; s < nsec; ++s) {
        const int64_t b = secs[s].begin, e = b + secs[s].len;
        const int64_t np = secs[s].len > 0 ? (secs[s].len + kCrcPart - 1) / kCrcPart : 1;
        for (int64_t q = 0; q < np; ++q) {
            const int64_t hi = e - (np - 1 - q) * kCrcPart;
            parts->push_back({hi - kCrcPart > b ? hi - kCrcPart : b, hi});
        }
        first_part->push_back(static_cast<int64_t>(parts->size()));
    }
}

cudaError_t launch_crc_sections(const uint8_t* data, const CrcSection* secs, int64_t nsec,
                                const CrcPart* parts, int64_t nparts, const int64_t* first_part,
                                uint32_t* part_crc, uint32_t* crc_out, uint8_t* write_back,
                                cudaStream_t st) {
    const int64_t g = nparts < 148 * 8 ? nparts : 148 * 8;
    crc_parts_kernel<<<static_cast<unsigned>(g < 1 ? 1 : g), kCrcThreads, 0, st>>>(data, parts, nparts,
                                                                                 part_crc);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    crc_fold_kernel<<<static_cast<unsigned>(nsec < 1 ? 1 : nsec), 256, 0, st>>>(secs, nsec, first_part, part_crc,
                                                                                crc_out, write_back);
    return cudaGetLastError();
}

cudaError_t launch_unpack_blocks(const uint8_t* bytes, const UnpackBlock* blocks, int64_t nblocks,
                                 int64_t max_items, cudaStream_t st) {
    const unsigned gy = static_cast<unsigned>(nblocks < 65535 ? nblocks : 65535);
    int64_t gx = (max_items + 255) / 256;
    const int64_t cap = (148 * 32 + gy - 1) / gy;
    if (gx > cap) gx = cap;
    if (gx < 1) gx = 1;
    unpack_blocks_kernel<<<dim3(static_cast<unsigned>(gx), gy), 256, 0, st>>>(bytes, blocks, nblocks);
    return cudaGetLastError();
}

cudaError_t launch_recon_scatter(const double* F, int64_t ldf, int64_t strideF, const double* C,
                                 int64_t kcap, int64_t strideC, const int64_t* rank, int64_t nb,
                                 int64_t mb, int64_t n, const int64_t* rel, const int64_t* bases,
                                 double* out, int64_t ldo, cudaStream_t st) {
    const size_t smem = sizeof(double) * static_cast<size_t>(kcap) * (kReconCols + 1);
    if (smem > 200 * 1024 || nb > 65535) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(recon_scatter_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    const dim3 grid(static_cast<unsigned>((mb + kReconRows - 1) / kReconRows), static_cast<unsigned>(nb));
    recon_scatter_kernel<<<grid, kReconThreads, smem, st>>>(F, ldf, strideF, C, kcap, strideC, rank, mb,
                                                         n, rel, bases, out, ldo);
    return cudaGetLastError();
}

cudaError_t launch_nonfinite_blocks(const double* A, int64_t lda, int64_t m, int64_t n,
                                    const BlockGridDev& g, int32_t* flags, cudaStream_t st) {
    // ~8 resident CTAs per SM in total, rows split so each thread streams >= 8 entries
    int64_t gy = n < 65535 ? n : 65535;
    int64_t gx = (148 * 8 + gy - 1) / gy;
    const int64_t gx_max = (m + 256 * 8 - 1) / (256 * 8);
    if (gx > gx_max) gx = gx_max;
    if (gx < 1) gx = 1;
    const dim3 grid(static_cast<unsigned>(gx), static_cast<unsigned>(gy));
    if (lda % 2 == 0 && reinterpret_cast<uintptr_t>(A) % 16 == 0)
        nonfinite_blocks_kernel<true><<<grid, 256, 0, st>>>(A, lda, m, n, g, flags);
    else
        nonfinite_blocks_kernel<false><<<grid, 256, 0, st>>>(A, lda, m, n, g, flags);
    return cudaGetLastError();
}

}  // namespace spidgpu
