// sketch.cu -- batched Gaussian sketch Y_s = Omega_s * A_s on FP64 tensor cores.
//
// Replaces the reference's sketch entry (subsample/subsample_column,
// proj/src/grid.cpp:136-150, called by spid() at proj/src/id.cpp:75-80) with
// the north star's Gaussian sketch; the CPU restatement is
// matmul(Omega, A) (proj/src/dense_matrix.cpp:38-53).
//
// Shape: a skinny contraction, M = ell (20..80) x N = n (100..512) x
// K = m (16K..164K rows) per subdomain, over S subdomains. Arithmetic
// intensity is ell/4 flop per byte of A, so for ell >= 24 the kernel is
// bound by the FP64 tensor pipe (DMMA.8x8x4 via mma.sync -- sm_100a has no
// tcgen05 f64 kind), not by HBM.
//
// Design (B200):
//  * persistent grid, one CTA per SM; the flat (subdomain, column tile,
//    16-row chunk) space is split into equal contiguous ranges, one per CTA
//    (stream-K style): perfect balance, and a CTA writes one partial per
//    tile it touches (<= 2-3), so split-K traffic is ~0.1% of A;
//  * A chunks (16 rows x NT columns, 128 B rows) are staged by TMA with
//    128B swizzle through a 4-stage mbarrier ring; OOB rows/columns are
//    zero-filled by the TMA unit, so ragged m and n need no masking;
//  * Omega chunks (ell_pad x 16) are generated in-kernel by Philox one chunk
//    ahead (performance mode) or loaded from HBM (oracle mode), written to a
//    swizzled double buffer; they are never re-read from HBM;
//  * the K index inside a chunk is permuted so each thread fetches its two
//    consecutive K values of an operand with one 16-byte shared load;
//    swizzles make every fragment load bank-conflict free;
//  * partials are reduced by a second tiny kernel in a fixed order, so Y is
//    bitwise reproducible run to run (SPEC determinism, proj/tests/
//    test_matrix_core.cpp:145-153).
#include <math.h>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace spidgpu {

namespace {

constexpr int kKc = 16;       // rows of A per chunk (128 B = one swizzle row)
constexpr int kStages = 4;    // TMA ring depth
constexpr int kWarps = 8;
constexpr int kThreads = kWarps * kWarp;

template <int MT, int NW>
struct SketchCfg {
    static constexpr int kEllPad = 8 * MT;
    static constexpr int kNt = kWarps * 8 * NW;
    static constexpr int kABytes = kNt * kKc * 8;       // one stage of A
    static constexpr int kOBytes = kEllPad * kKc * 8;   // one Omega buffer
    static constexpr size_t kSmem = 1024 + kStages * kABytes + 2 * kOBytes + kStages * 8;
    static constexpr int kGroups = 2 * MT * kKc;        // Philox calls per chunk (4 rows each)
    static constexpr int kGroupsPerThread = (kGroups + kThreads - 1) / kThreads;
    static constexpr int kExplicitPerThread = (kEllPad * kKc + kThreads - 1) / kThreads;
};

// swizzled offset (in doubles) of element (row, kk) in a [rows][16] tile:
// 16-byte chunk kk/2 is XOR-ed with row%8 (matches TMA SWIZZLE_128B).
__device__ __forceinline__ int swz(int row, int kk) {
    return row * kKc + ((((kk >> 1) ^ (row & 7)) << 1) | (kk & 1));
}

struct ChunkPos {
    int64_t s, ct, kc;
};

__device__ __forceinline__ ChunkPos chunk_pos(int64_t g, int64_t nchunk, int64_t ntiles_col) {
    const int64_t tile = g / nchunk;
    return ChunkPos{tile / ntiles_col, tile % ntiles_col, g % nchunk};
}

template <int MT, int NW, int OMODE>
__global__ void __launch_bounds__(kThreads, 1)
    sketch_kernel(const __grid_constant__ CUtensorMap tmap, SketchParams p, int64_t nchunk,
                  int64_t ntiles_col, int64_t total_chunks, int max_segs) {
    using Cfg = SketchCfg<MT, NW>;
    extern __shared__ unsigned char smem_raw[];
    unsigned char* base = reinterpret_cast<unsigned char*>(
        (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    double* abuf = reinterpret_cast<double*>(base);
    double* obuf = reinterpret_cast<double*>(base + kStages * Cfg::kABytes);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(base + kStages * Cfg::kABytes + 2 * Cfg::kOBytes);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t G = gridDim.x, c = blockIdx.x;
    const int64_t lo = (c * total_chunks) / G, hi = ((c + 1) * total_chunks) / G;
    const int64_t niter = hi - lo;
    if (niter <= 0) return;

    if (tid == 0) {
        prefetch_tmap(&tmap);
        for (int i = 0; i < kStages; ++i) mbar_init(&mbar[i], 1);
        fence_barrier_init();
    }
    __syncthreads();

    auto issue = [&](int64_t it) {
        const ChunkPos cp = chunk_pos(lo + it, nchunk, ntiles_col);
        const int slot = static_cast<int>(it % kStages);
        mbar_arrive_expect_tx(&mbar[slot], Cfg::kABytes);
        tma_load_3d(abuf + slot * (Cfg::kABytes / 8), &tmap, &mbar[slot],
                    static_cast<int>(cp.kc * kKc), static_cast<int>(cp.ct * Cfg::kNt),
                    static_cast<int>(cp.s));
    };
    if (tid == 0) {
        const int64_t pre = niter < kStages - 1 ? niter : kStages - 1;
        for (int64_t it = 0; it < pre; ++it) issue(it);
    }

    // ---- Omega production (registers, then swizzled smem) -----------------
    double oreg[OMODE == 1 ? 4 * Cfg::kGroupsPerThread : Cfg::kExplicitPerThread];
    auto omega_fetch = [&](int64_t g) {
        const ChunkPos cp = chunk_pos(g, nchunk, ntiles_col);
        const int64_t k0 = cp.kc * kKc;
        if constexpr (OMODE == 1) {
#pragma unroll
            for (int q = 0; q < Cfg::kGroupsPerThread; ++q) {
                const int grp = tid + q * kThreads;
                if (grp < Cfg::kGroups) {
                    const int g4 = grp % (2 * MT), kk = grp / (2 * MT);
                    omega_normals4(p.seed, static_cast<uint64_t>(p.sub_base + cp.s),
                                   static_cast<uint32_t>((p.row0 >> 2) + g4),
                                   static_cast<uint32_t>(k0 + kk), &oreg[4 * q]);
#pragma unroll
                    for (int e = 0; e < 4; ++e)
                        if (4 * g4 + e >= p.ell) oreg[4 * q + e] = 0.0;
                }
            }
        } else {
            const double* om = p.omega + cp.s * p.stride_o + p.row0;
#pragma unroll
            for (int q = 0; q < Cfg::kExplicitPerThread; ++q) {
                const int e = tid + q * kThreads;
                double v = 0.0;
                if (e < Cfg::kEllPad * kKc) {
                    const int r = e % Cfg::kEllPad, kk = e / Cfg::kEllPad;
                    const int64_t k = k0 + kk;
                    if (r < p.ell && k < p.m) v = __ldg(om + k * p.ldo + r);
                }
                oreg[q] = v;
            }
        }
    };
    auto omega_store = [&](double* ob) {
        if constexpr (OMODE == 1) {
#pragma unroll
            for (int q = 0; q < Cfg::kGroupsPerThread; ++q) {
                const int grp = tid + q * kThreads;
                if (grp < Cfg::kGroups) {
                    const int g4 = grp % (2 * MT), kk = grp / (2 * MT);
#pragma unroll
                    for (int e = 0; e < 4; ++e) ob[swz(4 * g4 + e, kk)] = oreg[4 * q + e];
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < Cfg::kExplicitPerThread; ++q) {
                const int e = tid + q * kThreads;
                if (e < Cfg::kEllPad * kKc) ob[swz(e % Cfg::kEllPad, e / Cfg::kEllPad)] = oreg[q];
            }
        }
    };
    omega_fetch(lo);
    omega_store(obuf);

    double acc[MT][NW][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    const int grow = lane >> 2;  // fragment row / column within an 8-block
    const int q4 = lane & 3;
    const int wcol0 = warp * NW * 8;
    int seg = 0;

    for (int64_t it = 0; it < niter; ++it) {
        const int slot = static_cast<int>(it % kStages);
        mbar_wait(&mbar[slot], static_cast<uint32_t>((it / kStages) & 1));
        __syncthreads();  // Omega(it) visible; iteration it-1 fully consumed
        if (tid == 0 && it + kStages - 1 < niter) issue(it + kStages - 1);
        const bool more = it + 1 < niter;
        if (more) omega_fetch(lo + it + 1);

        const double* At = abuf + slot * (Cfg::kABytes / 8);
        const double* Ot = obuf + (it & 1) * (Cfg::kOBytes / 8);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int ch = ((4 * h + q4) ^ grow) << 1;  // swizzled pair offset
            double2 of[MT], af[NW];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
                of[mt] = *reinterpret_cast<const double2*>(Ot + (8 * mt + grow) * kKc + ch);
#pragma unroll
            for (int nt = 0; nt < NW; ++nt)
                af[nt] = *reinterpret_cast<const double2*>(At + (wcol0 + 8 * nt + grow) * kKc + ch);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NW; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], of[mt].x, af[nt].x);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NW; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], of[mt].y, af[nt].y);
        }
        if (more) omega_store(obuf + ((it + 1) & 1) * (Cfg::kOBytes / 8));

        const int64_t g = lo + it;
        if (!more || (g + 1) / nchunk != g / nchunk) {  // tile boundary: flush partial
            double* part = p.partial + (static_cast<size_t>(c) * max_segs + seg) *
                                           (static_cast<size_t>(Cfg::kEllPad) * Cfg::kNt);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NW; ++nt) {
                    const int r = 8 * mt + grow, col = wcol0 + 8 * nt + 2 * q4;
                    *reinterpret_cast<double2*>(part + r * Cfg::kNt + col) =
                        make_double2(acc[mt][nt][0], acc[mt][nt][1]);
                    acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
                }
            ++seg;
        }
    }
}

// Fixed-order reduction of the per-CTA partials of one (subdomain, column
// tile) into Y (column-major ell x n). Contributors are the CTAs whose chunk
// range intersects the tile, summed in CTA order.
__global__ void sketch_reduce_kernel(SketchParams p, int ell_pad, int nt, int64_t nchunk,
                                     int64_t ntiles_col, int64_t total_chunks, int G,
                                     int max_segs) {
    const int64_t tile = blockIdx.x;
    const int64_t s = tile / ntiles_col, ct = tile % ntiles_col;
    const int64_t t0 = tile * nchunk, t1 = t0 + nchunk;
    __shared__ int cfirst, clast;
    if (threadIdx.x == 0) {
        int64_t cf = (t0 * G) / total_chunks;
        while (cf > 0 && (cf * total_chunks) / G > t0) --cf;
        while (((cf + 1) * total_chunks) / G <= t0) ++cf;
        int64_t cl = cf;
        while (cl + 1 < G && ((cl + 1) * total_chunks) / G < t1) ++cl;
        cfirst = static_cast<int>(cf);
        clast = static_cast<int>(cl);
    }
    __syncthreads();
    const int64_t ncols = p.n - ct * nt < nt ? p.n - ct * nt : nt;
    const int64_t elems = p.ell * ncols;
    double* Y = p.Y + s * p.strideY + p.row0;
    for (int64_t e = threadIdx.x; e < elems; e += blockDim.x) {
        const int r = static_cast<int>(e % p.ell);
        const int col = static_cast<int>(e / p.ell);
        double sum = 0.0;
        for (int cc = cfirst; cc <= clast; ++cc) {
            const int64_t lo = (static_cast<int64_t>(cc) * total_chunks) / G;
            const int64_t hi = (static_cast<int64_t>(cc + 1) * total_chunks) / G;
            if (hi <= lo) continue;
            const int segi = static_cast<int>(tile - lo / nchunk);
            const double* part = p.partial + (static_cast<size_t>(cc) * max_segs + segi) *
                                                 (static_cast<size_t>(ell_pad) * nt);
            sum += part[r * nt + col];
        }
        Y[(ct * nt + col) * p.ldy + r] = sum;
    }
}

__global__ void philox_omega_kernel(uint64_t seed, int64_t s, int64_t ell, int64_t m, double* out,
                                    int64_t ldo) {
    const int64_t ngroups = (ell + 3) / 4;
    const int64_t total = ngroups * m;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t g4 = e % ngroups, k = e / ngroups;
        double v[4];
        omega_normals4(seed, static_cast<uint64_t>(s), static_cast<uint32_t>(g4),
                       static_cast<uint32_t>(k), v);
        for (int i = 0; i < 4; ++i)
            if (4 * g4 + i < ell) out[k * ldo + 4 * g4 + i] = v[i];
    }
}

template <int MT, int NW, int OMODE>
cudaError_t launch_t(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap,
                     cudaStream_t stream) {
    using Cfg = SketchCfg<MT, NW>;
    auto kern = sketch_kernel<MT, NW, OMODE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Cfg::kSmem));
    if (e != cudaSuccess) return e;
    kern<<<plan.grid, kThreads, Cfg::kSmem, stream>>>(*tmap, p, plan.nchunk, plan.ntiles_col,
                                                      plan.total_chunks, plan.max_segs);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    sketch_reduce_kernel<<<static_cast<unsigned>(p.batch * plan.ntiles_col), 256, 0, stream>>>(
        p, Cfg::kEllPad, Cfg::kNt, plan.nchunk, plan.ntiles_col, plan.total_chunks, plan.grid,
        plan.max_segs);
    return cudaGetLastError();
}

template <int MT, int OMODE>
cudaError_t launch_nw(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap,
                      cudaStream_t stream) {
    switch (plan.nw) {
        case 1: return launch_t<MT, 1, OMODE>(p, plan, tmap, stream);
        case 2: return launch_t<MT, 2, OMODE>(p, plan, tmap, stream);
        default:
            if constexpr (MT <= 8) return launch_t<MT, 4, OMODE>(p, plan, tmap, stream);
            return cudaErrorInvalidValue;
    }
}

template <int OMODE>
cudaError_t launch_mt(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap,
                      cudaStream_t stream) {
    switch (plan.mt) {
        case 2: return launch_nw<2, OMODE>(p, plan, tmap, stream);
        case 3: return launch_nw<3, OMODE>(p, plan, tmap, stream);
        case 4: return launch_nw<4, OMODE>(p, plan, tmap, stream);
        case 6: return launch_nw<6, OMODE>(p, plan, tmap, stream);
        case 8: return launch_nw<8, OMODE>(p, plan, tmap, stream);
        case 10: return launch_nw<10, OMODE>(p, plan, tmap, stream);
        default: return cudaErrorInvalidValue;
    }
}

size_t smem_for(int mt, int nw) {
    const int nt = kWarps * 8 * nw;
    return 1024 + kStages * (nt * kKc * 8) + 2 * (8 * mt * kKc * 8) + kStages * 8;
}

}  // namespace

// Omega rows handled by one launch: 80 (MT=10); wider sketches are sliced.
bool sketch_make_plan(int64_t m, int64_t n, int64_t batch, int64_t ell, int num_sms,
                      SketchPlan* plan) {
    if (m < 1 || n < 1 || batch < 1 || ell < 1 || ell > 80) return false;
    const int mts[] = {2, 3, 4, 6, 8, 10};
    int mt = 10;
    for (int v : mts)
        if (8 * v >= ell) {
            mt = v;
            break;
        }
    // column tile: least padded work; ties -> wider tile (fewer Omega regenerations)
    int best_nw = 1;
    int64_t best_cols = INT64_MAX;
    for (int nw : {4, 2, 1}) {
        if (nw == 4 && mt > 8) continue;
        const int64_t nt = kWarps * 8 * nw;
        const int64_t cols = ((n + nt - 1) / nt) * nt;
        if (cols < best_cols) {
            best_cols = cols;
            best_nw = nw;
        }
    }
    plan->mt = mt;
    plan->nw = best_nw;
    plan->nt = kWarps * 8 * best_nw;
    plan->ntiles_col = (n + plan->nt - 1) / plan->nt;
    plan->nchunk = (m + kKc - 1) / kKc;
    plan->total_chunks = batch * plan->ntiles_col * plan->nchunk;
    int64_t grid = num_sms;
    if (grid > plan->total_chunks) grid = plan->total_chunks;
    plan->grid = static_cast<int>(grid);
    const int64_t per = (plan->total_chunks + grid - 1) / grid;
    plan->max_segs = static_cast<int>(per / plan->nchunk + 2);
    plan->smem = smem_for(mt, best_nw);
    plan->partial_elems = static_cast<size_t>(grid) * plan->max_segs * (8 * mt) * plan->nt;
    return true;
}

cudaError_t launch_sketch(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap,
                          cudaStream_t stream) {
    return p.omega_mode == 1 ? launch_mt<1>(p, plan, tmap, stream)
                             : launch_mt<0>(p, plan, tmap, stream);
}

cudaError_t launch_philox_omega(uint64_t seed, int64_t s, int64_t ell, int64_t m, double* out,
                                int64_t ldo, cudaStream_t stream) {
    const int64_t total = ((ell + 3) / 4) * m;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    philox_omega_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(seed, s, ell, m, out, ldo);
    return cudaGetLastError();
}

}  // namespace spidgpu
