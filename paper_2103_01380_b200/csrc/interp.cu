// interp.cu -- coarse-grid skeleton of the single-pass ID (SPID) and the
// multilinear lift M that brings it back to the fine grid.
//
// spid() (proj/src/id.cpp:62-83) keeps the skeleton on the coarse rows J of a
// strided SubsampleSpec (proj/src/grid.cpp:91-130) and reconstructs with
// M * skeleton * C (id.cpp:92-96), where M is the tensor-product linear
// interpolation operator of InterpOperator::from_spec (proj/src/interp.cpp:
// 19-100). The reference builds M as CSR; here each fine point generates its
// own <= 8-entry stencil on the fly -- the same axis weights
// (interp.cpp:19-41), the same duplicate merge in (a2, a1, a0) loop order
// (interp.cpp:79-89, std::map accumulation), the same ascending-column
// accumulation order of apply_column (interp.cpp:177-186) -- so the lift is
// bit-identical to the reference's apply() without materialising M.
//
// Multi-QoI subdomains (rows = q * P + p) apply the operator per QoI block.
#include "common.cuh"
#include "kernels.h"

namespace spidgpu {

namespace {

struct AxisW {
    int n;
    int pos[2];
    double w[2];
};

// Coarse index list of one axis (grid.cpp:91-106): 0, s, 2s, ... < dim, plus
// dim-1 when the boundary is pinned on a non-periodic axis.
__device__ __forceinline__ int coarse_count(int dim, int stride, bool periodic, bool incl) {
    const int base = (dim + stride - 1) / stride;
    const int last = (base - 1) * stride;
    return base + ((incl && !periodic && last != dim - 1) ? 1 : 0);
}

__device__ __forceinline__ int coarse_at(int j, int dim, int stride) {
    const int base = (dim + stride - 1) / stride;
    return j < base ? j * stride : dim - 1;
}

// interp.cpp:19-41 (lower_bound over the ascending coarse list). Returns
// n = 0 for the "ExtrapolationRequired" case (fine point past the last coarse
// point of a non-periodic axis).
__device__ __forceinline__ AxisW axis_weights(int f, int dim, int stride, bool periodic, bool incl) {
    AxisW a;
    const int nc = coarse_count(dim, stride, periodic, incl);
    // lower_bound: first coarse index >= f
    int lb = (f + stride - 1) / stride;           // in the strided part
    const int base = (dim + stride - 1) / stride;
    if (lb >= base) lb = nc > base ? base : nc;   // only the pinned boundary (if any) remains
    if (lb < nc && coarse_at(lb, dim, stride) == f) {
        a.n = 1;
        a.pos[0] = lb;
        a.w[0] = 1.0;
        return a;
    }
    if (lb >= nc) {  // past the last coarse point
        if (!periodic) {
            a.n = 0;
            return a;
        }
        const int last = nc - 1;
        const double cell = static_cast<double>(dim - coarse_at(last, dim, stride) + 0);
        const double w = static_cast<double>(f - coarse_at(last, dim, stride)) / cell;
        a.n = 2;
        a.pos[0] = last;
        a.w[0] = 1.0 - w;
        a.pos[1] = 0;
        a.w[1] = w;
        return a;
    }
    const int hi = lb, lo = hi - 1;
    const int clo = coarse_at(lo, dim, stride), chi = coarse_at(hi, dim, stride);
    const double w = static_cast<double>(f - clo) / static_cast<double>(chi - clo);
    a.n = 2;
    a.pos[0] = lo;
    a.w[0] = 1.0 - w;
    a.pos[1] = hi;
    a.w[1] = w;
    return a;
}

// fine_s(q*P + p, t) = sum over the stencil of coarse_s(q*Pc + col, t)
__global__ void interp_apply_kernel(GridSpecDev g, const double* __restrict__ coarse, int64_t ldc,
                                    int64_t strideC, int64_t k, const int64_t* __restrict__ rank,
                                    int64_t batch, double* __restrict__ fine, int64_t ldf,
                                    int64_t strideF, int32_t* err_flag) {
    const int d0 = g.dims[0], d1 = g.naxes > 1 ? g.dims[1] : 1, d2 = g.naxes > 2 ? g.dims[2] : 1;
    const int P = d0 * d1 * d2;
    int nc[3];
    for (int ax = 0; ax < 3; ++ax)
        nc[ax] = ax < g.naxes ? coarse_count(g.dims[ax], g.strides[ax], g.periodic[ax], g.incl) : 1;
    const int Pc = nc[0] * nc[1] * nc[2];
    const int64_t total = batch * static_cast<int64_t>(P);
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t s = e / P;
        const int p = static_cast<int>(e % P);
        const int i0 = p % d0, i1 = (p / d0) % d1, i2 = p / (d0 * d1);
        const AxisW w0 = axis_weights(i0, d0, g.strides[0], g.periodic[0], g.incl);
        AxisW w1, w2;
        if (g.naxes > 1) w1 = axis_weights(i1, d1, g.strides[1], g.periodic[1], g.incl);
        else w1 = AxisW{1, {0, 0}, {1.0, 0.0}};
        if (g.naxes > 2) w2 = axis_weights(i2, d2, g.strides[2], g.periodic[2], g.incl);
        else w2 = AxisW{1, {0, 0}, {1.0, 0.0}};
        if (w0.n == 0 || w1.n == 0 || w2.n == 0) {
            if (err_flag) atomicExch(err_flag, 1);  // ExtrapolationRequired
            continue;
        }
        // stencil in (a2, a1, a0) loop order with std::map-style merging
        int col[8];
        double wt[8];
        int ne = 0;
        for (int b2 = 0; b2 < w2.n; ++b2)
            for (int b1 = 0; b1 < w1.n; ++b1)
                for (int b0 = 0; b0 < w0.n; ++b0) {
                    int c = w0.pos[b0];
                    if (g.naxes > 1) c += nc[0] * w1.pos[b1];
                    if (g.naxes > 2) c += nc[0] * nc[1] * w2.pos[b2];
                    const double v = __dmul_rn(__dmul_rn(w0.w[b0], w1.w[b1]), w2.w[b2]);
                    int at = -1;
                    for (int q = 0; q < ne; ++q)
                        if (col[q] == c) at = q;
                    if (at < 0) {
                        col[ne] = c;
                        wt[ne] = __dadd_rn(0.0, v);
                        ++ne;
                    } else {
                        wt[at] = __dadd_rn(wt[at], v);
                    }
                }
        // ascending column order (std::map iteration)
        for (int a = 1; a < ne; ++a)
            for (int b = a; b > 0 && col[b - 1] > col[b]; --b) {
                const int tc = col[b];
                col[b] = col[b - 1];
                col[b - 1] = tc;
                const double tw = wt[b];
                wt[b] = wt[b - 1];
                wt[b - 1] = tw;
            }
        const int kk = static_cast<int>(rank ? rank[s] : k);
        const double* cs = coarse + s * strideC;
        double* fs = fine + s * strideF;
        for (int q = 0; q < g.nqoi; ++q)
            for (int t = 0; t < kk; ++t) {
                const double* ct = cs + t * ldc + static_cast<int64_t>(q) * Pc;
                double v = 0.0;
                for (int a = 0; a < ne; ++a) v = __dadd_rn(v, __dmul_rn(wt[a], ct[col[a]]));
                fs[t * ldf + static_cast<int64_t>(q) * P + p] = v;
            }
    }
}

// skel_c(:, t) = A(J, I_t) per subdomain, J the coarse rows of every QoI block.
__global__ void gather_coarse_kernel(const double* __restrict__ A, int64_t lda, int64_t strideA,
                                     const int64_t* __restrict__ rows, int64_t nrows,
                                     const int64_t* __restrict__ idx, int64_t kcap,
                                     const int64_t* __restrict__ rank, int64_t batch,
                                     double* __restrict__ skel, int64_t ldskel, int64_t strideS) {
    // rows in x, (subdomain, skeleton column) pairs in y; columns past the
    // rank are skipped whole
    for (int64_t st = blockIdx.y; st < batch * kcap; st += gridDim.y) {
        const int64_t s = st / kcap, t = st - s * kcap;
        if (t >= rank[s]) continue;
        const double* src = A + s * strideA + idx[s * kcap + t] * lda;
        double* dst = skel + s * strideS + t * ldskel;
        for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < nrows;
             i += static_cast<int64_t>(gridDim.x) * blockDim.x)
            dst[i] = src[rows[i]];
    }
}

}  // namespace

cudaError_t launch_interp_apply(const GridSpecDev& g, const double* coarse, int64_t ldc,
                                int64_t strideC, int64_t k, const int64_t* rank, int64_t batch,
                                double* fine, int64_t ldf, int64_t strideF, int32_t* err_flag,
                                cudaStream_t stream) {
    int64_t P = g.dims[0];
    if (g.naxes > 1) P *= g.dims[1];
    if (g.naxes > 2) P *= g.dims[2];
    const int64_t total = batch * P;
    int64_t grid = (total + 255) / 256;
    if (grid > 148 * 16) grid = 148 * 16;
    if (grid < 1) grid = 1;
    interp_apply_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(
        g, coarse, ldc, strideC, k, rank, batch, fine, ldf, strideF, err_flag);
    return cudaGetLastError();
}

cudaError_t launch_gather_coarse(const double* A, int64_t lda, int64_t strideA, const int64_t* rows,
                                 int64_t nrows, const int64_t* idx, int64_t kcap,
                                 const int64_t* rank, int64_t batch, double* skel, int64_t ldskel,
                                 int64_t strideS, cudaStream_t stream) {
    gather_coarse_kernel<<<col_grid(nrows, batch * kcap), 256, 0, stream>>>(
        A, lda, strideA, rows, nrows, idx, kcap, rank, batch, skel, ldskel, strideS);
    return cudaGetLastError();
}

}  // namespace spidgpu
