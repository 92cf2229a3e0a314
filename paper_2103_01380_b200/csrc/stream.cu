// stream.cu -- device side of the streaming two-stage compressor
// (proj/src/pipeline.cpp:104-294, proj/src/blocking.cpp:112-204).
//
//   sort_pairs      stage-1 skeleton indices sorted ascending, with their
//                   selection positions (the UnionSource.local of stage 2)
//   concat_union    per block: the union of all chunks' skeleton columns in
//                   sorted global-snapshot order (chunks are disjoint in time,
//                   so the union is chunk-major), zero-padded to the group's
//                   widest union -- zero columns are never pivoted and add
//                   +0 to every sum, so the stage-2 CPQR is unchanged
//   compose         C1' = C1 * C0' without materialising the block-diagonal
//                   C0': final(r, col0 + t) accumulates C1(r, u) * C0_c(l_u, t)
//                   over the chunk's union columns u ascending, zero C0
//                   entries skipped, one rounding per operation -- the
//                   reference's loop order (blocking.cpp:187-200), so bitwise
//   final_global    global snapshot index of each final skeleton column
#include "common.cuh"
#include "kernels.h"

namespace spidgpu {

namespace {

__global__ void sort_pairs_kernel(const int64_t* __restrict__ idx, const int64_t* __restrict__ rank,
                                  int64_t kcap, int64_t nb, int64_t* __restrict__ out_idx,
                                  int32_t* __restrict__ out_pos) {
    const int64_t b = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (b >= nb) return;
    const int64_t k = rank[b];
    const int64_t* src = idx + b * kcap;
    int64_t* dv = out_idx + b * kcap;
    int32_t* dp = out_pos + b * kcap;
    for (int64_t t = 0; t < k; ++t) {  // insertion sort of <= stage-1 rank entries
        const int64_t v = src[t];
        int64_t u = t;
        while (u > 0 && dv[u - 1] > v) {
            dv[u] = dv[u - 1];
            dp[u] = dp[u - 1];
            --u;
        }
        dv[u] = v;
        dp[u] = static_cast<int32_t>(t);
    }
}

// Per block b: the chunks' skeleton columns back to back (the union in
// chunk order), their global indices and stage-1 positions, and the chunk
// offsets. Grid (x, b): CTA x == 0 writes the bookkeeping; every CTA copies a
// grid-strided share of each chunk's contiguous r x mc range (16-byte
// vectors when mc is even), so the copy is spread over ~8 CTAs per SM.
__global__ void concat_union_kernel(const StreamChunkDev* __restrict__ chunks, int64_t nchunks,
                                    int64_t mc, int64_t rmax, double* __restrict__ concat,
                                    int64_t* __restrict__ uglob, int32_t* __restrict__ upos,
                                    int64_t* __restrict__ uoff, int64_t* __restrict__ R) {
    const int64_t b = blockIdx.y;
    double* cb = concat + b * rmax * mc;
    const int64_t t0 = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
    int64_t u0 = 0;
    for (int64_t c = 0; c < nchunks; ++c) {
        const StreamChunkDev ch = chunks[c];
        const int64_t r = ch.rank[b];
        if (blockIdx.x == 0) {
            if (threadIdx.x == 0) uoff[b * (nchunks + 1) + c] = u0;
            for (int64_t u = threadIdx.x; u < r; u += blockDim.x) {
                uglob[b * rmax + u0 + u] = ch.col0 + ch.sorted_idx[b * ch.kcap + u];
                upos[b * rmax + u0 + u] = ch.sorted_pos[b * ch.kcap + u];
            }
        }
        const double* src = ch.skel + b * ch.kcap * mc;
        double* dst = cb + u0 * mc;
        if ((mc & 1) == 0) {
            const double2* s2 = reinterpret_cast<const double2*>(src);
            double2* d2 = reinterpret_cast<double2*>(dst);
            for (int64_t e = t0; e < r * mc / 2; e += stride) d2[e] = s2[e];
        } else {
            for (int64_t e = t0; e < r * mc; e += stride) dst[e] = src[e];
        }
        u0 += r;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        uoff[b * (nchunks + 1) + nchunks] = u0;
        R[b] = u0;
    }
}

__global__ void compose_kernel(const StreamChunkDev* __restrict__ chunks, int64_t nchunks,
                               int64_t time_chunk, int64_t n_total, const double* __restrict__ C1,
                               int64_t kcap2, int64_t rmax, const int64_t* __restrict__ rank2,
                               const int32_t* __restrict__ upos, const int64_t* __restrict__ uoff,
                               double* __restrict__ out, int32_t* __restrict__ bad) {
    const int64_t b = blockIdx.y;
    const int64_t k2 = rank2[b];
    const double* c1 = C1 + b * kcap2 * rmax;
    double* ob = out + b * kcap2 * n_total;
    int flag = 0;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < k2 * n_total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e % k2, g = e / k2;
        const int64_t c = g / time_chunk, t = g - c * time_chunk;
        const StreamChunkDev ch = chunks[c];
        const double* c0 = ch.C0 + b * ch.kcap * ch.cols;  // kcap x cols, ld kcap
        double acc = 0.0;
        for (int64_t u = uoff[b * (nchunks + 1) + c]; u < uoff[b * (nchunks + 1) + c + 1]; ++u) {
            const double w = c0[t * ch.kcap + upos[b * rmax + u]];
            if (w == 0.0) continue;
            acc = add_rn(acc, mul_rn(c1[u * kcap2 + r], w));
        }
        ob[g * kcap2 + r] = acc;
        flag |= !isfinite(acc);
    }
    if (flag) atomicExch(bad + b, 1);
}

__global__ void final_global_kernel(const int64_t* __restrict__ idx2, const int64_t* __restrict__ rank2,
                                    int64_t kcap2, const int64_t* __restrict__ uglob, int64_t rmax,
                                    int64_t nb, int64_t* __restrict__ out) {
    const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
    if (e >= nb * kcap2) return;
    const int64_t b = e / kcap2, t = e % kcap2;
    if (t < rank2[b]) out[e] = uglob[b * rmax + idx2[e]];
}

}  // namespace

cudaError_t launch_sort_pairs(const int64_t* idx, const int64_t* rank, int64_t kcap, int64_t nb,
                              int64_t* out_idx, int32_t* out_pos, cudaStream_t st) {
    sort_pairs_kernel<<<static_cast<unsigned>((nb + 127) / 128), 128, 0, st>>>(idx, rank, kcap, nb, out_idx,
                                                                               out_pos);
    return cudaGetLastError();
}

cudaError_t launch_concat_union(const StreamChunkDev* chunks, int64_t nchunks, int64_t nb, int64_t mc,
                                int64_t rmax, double* concat, int64_t* uglob, int32_t* upos,
                                int64_t* uoff, int64_t* R, cudaStream_t st) {
    int64_t gx = (148 * 8 + nb - 1) / nb;
    if (gx > 64) gx = 64;
    if (gx < 1) gx = 1;
    concat_union_kernel<<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(nb)), 256, 0, st>>>(
        chunks, nchunks, mc, rmax, concat, uglob, upos, uoff, R);
    return cudaGetLastError();
}

cudaError_t launch_compose(const StreamChunkDev* chunks, int64_t nchunks, int64_t time_chunk,
                           int64_t n_total, const double* C1, int64_t kcap2, int64_t rmax,
                           const int64_t* rank2, const int32_t* upos, const int64_t* uoff, int64_t nb,
                           double* out, int32_t* bad, cudaStream_t st) {
    int64_t gx = (kcap2 * n_total + 255) / 256;
    const int64_t cap = (148 * 16 + nb - 1) / nb;
    if (gx > cap) gx = cap;
    if (gx < 1) gx = 1;
    compose_kernel<<<dim3(static_cast<unsigned>(gx), static_cast<unsigned>(nb)), 256, 0, st>>>(
        chunks, nchunks, time_chunk, n_total, C1, kcap2, rmax, rank2, upos, uoff, out, bad);
    return cudaGetLastError();
}

cudaError_t launch_final_global(const int64_t* idx2, const int64_t* rank2, int64_t kcap2,
                                const int64_t* uglob, int64_t rmax, int64_t nb, int64_t* out,
                                cudaStream_t st) {
    const int64_t tot = nb * kcap2;
    final_global_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(idx2, rank2, kcap2, uglob,
                                                                                 rmax, nb, out);
    return cudaGetLastError();
}

}  // namespace spidgpu
