// gather.cu -- skeleton column gather and sketch row gather.
//
// skel_s(:, t) = A_s(:, I_s[t]): select_columns (proj/src/dense_matrix.cpp:
// 71-81) producing the fine-grid skeleton of sub_id (proj/src/id.cpp:57-58).
// Pure HBM streaming: 2*8*m*k bytes per subdomain, 16-byte vector loads and
// stores, a flat grid-stride over (subdomain, skeleton column, row chunk).
//
// B_s = A_s(J, :): subsample (proj/src/grid.cpp:136-140), the reference's own
// deterministic sketch, used by the sub_id drop-in.
#include "common.cuh"
#include "kernels.h"

namespace spidgpu {

namespace {

constexpr int kRowsPerUnit = 8192;  // doubles per (column, chunk) unit
constexpr int kThreads = 256;

template <bool kVec>
__global__ void __launch_bounds__(kThreads)
    gather_cols_kernel(const double* __restrict__ A, int64_t m, int64_t lda, int64_t strideA,
                       int64_t batch, const int64_t* __restrict__ idx, int64_t kcap,
                       const int64_t* __restrict__ rank, int64_t n, double* __restrict__ skel,
                       int64_t ldskel, int64_t strideS, int32_t* err_flag) {
    const int64_t nchunk = (m + kRowsPerUnit - 1) / kRowsPerUnit;
    const int64_t units = batch * kcap * nchunk;
    for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
        const int64_t s = u / (kcap * nchunk);
        const int64_t t = (u / nchunk) % kcap;
        const int64_t ch = u % nchunk;
        if (t >= rank[s]) continue;
        const int64_t col = idx[s * kcap + t];
        if (col < 0 || col >= n) {  // dense_matrix.cpp:75 (IndexOutOfRange)
            if (err_flag && threadIdx.x == 0) atomicCAS(err_flag, 0, SPID_INDEX_OUT_OF_RANGE);
            continue;
        }
        const double* src = A + s * strideA + col * lda;
        double* dst = skel + s * strideS + t * ldskel;
        const int64_t r0 = ch * kRowsPerUnit;
        const int64_t r1 = r0 + kRowsPerUnit < m ? r0 + kRowsPerUnit : m;
        if (kVec) {
            const double2* s2 = reinterpret_cast<const double2*>(src + r0);
            double2* d2 = reinterpret_cast<double2*>(dst + r0);
            const int64_t nv = (r1 - r0) / 2;
            for (int64_t i = threadIdx.x; i < nv; i += kThreads) __stcs(d2 + i, __ldcs(s2 + i));
            if (((r1 - r0) & 1) && threadIdx.x == 0) dst[r1 - 1] = src[r1 - 1];
        } else {
            for (int64_t i = r0 + threadIdx.x; i < r1; i += kThreads) dst[i] = src[i];
        }
    }
}

__global__ void gather_rows_kernel(const double* __restrict__ A, int64_t m, int64_t n,
                                   int64_t lda, int64_t strideA, int64_t batch,
                                   const int64_t* __restrict__ rows, int64_t nrows,
                                   double* __restrict__ B, int64_t ldb, int64_t strideB, int32_t* err_flag) {
    // rows in x, (subdomain, column) pairs in y: one division per column
    for (int64_t sj = blockIdx.y; sj < batch * n; sj += gridDim.y) {
        const int64_t s = sj / n, j = sj - s * n;
        const double* src = A + s * strideA + j * lda;
        double* dst = B + s * strideB + j * ldb;
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nrows;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
            const int64_t r = rows[i];
            const bool ok = r >= 0 && r < m;  // grid.cpp:138-140 (rows beyond the matrix)
            if (!ok && err_flag) atomicCAS(err_flag, 0, SPID_INDEX_OUT_OF_RANGE);
            dst[i] = ok ? src[r] : 0.0;
        }
    }
}

}  // namespace

cudaError_t launch_gather_cols(const double* A, int64_t m, int64_t lda, int64_t strideA,
                               int64_t batch, const int64_t* indices, int64_t kcap,
                               const int64_t* rank, int64_t n, double* skel, int64_t ldskel,
                               int64_t strideS, int32_t* err_flag, cudaStream_t stream) {
    const int64_t nchunk = (m + kRowsPerUnit - 1) / kRowsPerUnit;
    const int64_t units = batch * kcap * nchunk;
    int64_t grid = units < 148 * 16 ? units : 148 * 16;
    if (grid < 1) grid = 1;
    const bool vec = (lda % 2 == 0) && (ldskel % 2 == 0) && (strideA % 2 == 0) &&
                     (strideS % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                     (reinterpret_cast<uintptr_t>(skel) % 16 == 0);
    if (vec)
        gather_cols_kernel<true><<<static_cast<unsigned>(grid), kThreads, 0, stream>>>(
            A, m, lda, strideA, batch, indices, kcap, rank, n, skel, ldskel, strideS, err_flag);
    else
        gather_cols_kernel<false><<<static_cast<unsigned>(grid), kThreads, 0, stream>>>(
            A, m, lda, strideA, batch, indices, kcap, rank, n, skel, ldskel, strideS, err_flag);
    return cudaGetLastError();
}

cudaError_t launch_gather_rows(const double* A, int64_t m, int64_t n, int64_t lda,
                               int64_t strideA, int64_t batch, const int64_t* rows,
                               int64_t nrows, double* B, int64_t ldb, int64_t strideB, int32_t* err_flag,
                               cudaStream_t stream) {
    gather_rows_kernel<<<col_grid(nrows, batch * n), 256, 0, stream>>>(A, m, n, lda, strideA,
                                                                        batch, rows, nrows, B,
                                                                        ldb, strideB, err_flag);
    return cudaGetLastError();
}

}  // namespace spidgpu
