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
//    4096-row segment) unit space (kernels.h) is split into contiguous
//    ranges of whole units, one per CTA; a CTA writes one partial per
//    segment into that segment's own slot (about 1% of A's bytes);
//  * A chunks (16 rows x NT columns, 128 B rows) are staged by TMA with
//    128B swizzle through an S-stage ring; "full" mbarriers carry the TMA
//    transaction bytes, "empty" mbarriers collect one arrive per warp, so
//    the main loop has no CTA-wide barrier at all. OOB rows/columns are
//    zero-filled by the TMA unit (ragged m, n need no masking);
//  * warp specialisation: 4 producer warps (one per SMSP; one lane issues
//    the TMA) write each chunk's Omega tile into a swizzled shared ring --
//    read from the explicit Omega (oracle mode) or generated with Philox
//    (the discretised Gaussian of philox.cuh; the Philox sketch normally runs
//    on the integer kernels, this path serves SPIDGPU_OPT_DMMA_SKETCH) --
//    while 16 consumer warps, tiled 2 (M) x 8 (N) (1 x 16 for ell <= 24),
//    issue LDS.128 fragments and DMMA.8x8x4;
//  * inside a 16-row chunk lane q feeds K = 4q + 2h + e at k-step (h, e), so
//    each A fragment pair is one 16-byte shared load and the two rows of a
//    quarter-warp hit opposite 16B-chunk parities under the swizzle: every
//    fragment load is bank-conflict free;
//  * partials are reduced by a small second kernel in segment order, so Y is
//    bitwise reproducible run to run (proj/tests/test_matrix_core.cpp:145-153)
//    and independent of the batch, grid and grouping.
#include <math.h>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace spidgpu {

namespace {

constexpr int kKc = 16;  // rows of A per chunk (128 B = one swizzle row)
constexpr int kWarps = 16;           // consumer (tensor-core) warps: 4 per SMSP
constexpr int kProducerWarps = 4;    // TMA issue + Omega generation, one per SMSP so
                                     // no SMSP's consumers lose issue slots to them
constexpr int kThreads = (kWarps + kProducerWarps) * kWarp;
constexpr int kStageBudget = 200 * 1024;

template <int WM, int MTW, int NW>
struct SketchCfg {
    static constexpr int kWn = kWarps / WM;
    static constexpr int kEllPad = 8 * MTW * WM;
    static constexpr int kNt = 8 * NW * kWn;
    static constexpr int kABytes = kNt * kKc * 8;
    static constexpr int kOBytes = kEllPad * kKc * 8;
    static constexpr int kStageBytes = kABytes + kOBytes;
    static constexpr int kStages =
        (kStageBudget / kStageBytes) < 8 ? (kStageBudget / kStageBytes) : 8;
    static constexpr size_t kSmem = 1024 + static_cast<size_t>(kStages) * kStageBytes + 3 * 8 * kStages;
};

struct ChunkPos {
    int64_t s, ct, kc;
};

__device__ __forceinline__ ChunkPos chunk_pos(int64_t g, int64_t nchunk, int64_t ntiles_col) {
    const int64_t tile = g / nchunk;
    return ChunkPos{tile / ntiles_col, tile % ntiles_col, g % nchunk};
}

// Warp-specialised persistent kernel:
//   warps 0..7  consumers: LDS.128 fragments + DMMA.8x8x4 into registers
//   warps 8..9  producers: TMA issue of the A chunk + Philox (or explicit)
//               Omega chunk into a swizzled shared ring
// Stage hand-off: full_a (TMA tx bytes), full_o (64 producer arrivals),
// empty (8 consumer-warp arrivals). No CTA-wide barrier in the main loop.
template <int WM, int MTW, int NW, int OMODE>
__global__ void __launch_bounds__(kThreads, 1)
    sketch_kernel(const __grid_constant__ CUtensorMap tmap, SketchParams p, int64_t nchunk,
                  int64_t ntiles_col, int64_t nseg, int64_t seg_len, int64_t total_units) {
    using Cfg = SketchCfg<WM, MTW, NW>;
    constexpr int S = Cfg::kStages;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw_s = smem_u32(smem_raw);
    const uint32_t base_s = (raw_s + 1023u) & ~1023u;  // 128B-swizzle atoms need 1 KiB alignment
    unsigned char* base = smem_raw + (base_s - raw_s);
    // stage i: A at base_s + i*kABytes; Omega at base_s + S*kABytes + i*kOBytes
    const uint32_t a_s = base_s;
    const uint32_t o_s = base_s + S * Cfg::kABytes;
    uint64_t* full_a = reinterpret_cast<uint64_t*>(base + S * Cfg::kStageBytes);
    uint64_t* full_o = full_a + S;
    uint64_t* empty = full_o + S;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t G = gridDim.x, c = blockIdx.x;
    const int64_t lo = sketch_unit_chunk((c * total_units) / G, nseg, seg_len, nchunk);
    const int64_t hi = sketch_unit_chunk(((c + 1) * total_units) / G, nseg, seg_len, nchunk);
    const int64_t niter = hi - lo;
    if (niter <= 0) return;

    if (tid == 0) {
        prefetch_tmap(&tmap);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full_a[i], 1);
            mbar_init(&full_o[i], kProducerWarps * kWarp);
            mbar_init(&empty[i], kWarps);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp >= kWarps) {
        // ------------------------------ producers ------------------------------
        const int pt = tid - kWarps * kWarp;  // 0..63
        constexpr int kCalls = Cfg::kEllPad * (kKc / 8);  // (row, k-octet) pairs per chunk
        ChunkPos cp = chunk_pos(lo, nchunk, ntiles_col);  // advanced incrementally
        int slot = 0;
        uint32_t epar = 0;  // parity of the empty-barrier phase being waited on
        for (int64_t it = 0; it < niter; ++it) {
            if (it >= S) mbar_wait(&empty[slot], epar);
            if (pt == 0) {
                mbar_arrive_expect_tx(&full_a[slot], Cfg::kABytes);
                tma_load_3d(base + slot * Cfg::kABytes, &tmap, &full_a[slot],
                            static_cast<int>(cp.kc * kKc), static_cast<int>(cp.ct * Cfg::kNt),
                            static_cast<int>(cp.s));
            }
            const uint32_t ob = o_s + slot * Cfg::kOBytes;
            for (int call = pt; call < kCalls; call += kProducerWarps * kWarp) {
                const int ko = call & 1, r = call >> 1;  // lanes: 2 k-octets x 16 rows
                double v[8];
                const int64_t k0 = cp.kc * kKc + 8 * ko;
                if constexpr (OMODE == 1) {
                    omega_values8(p.seed, static_cast<uint64_t>(p.sub_base + cp.s),
                                  static_cast<uint32_t>(p.row0 + r),
                                  static_cast<uint32_t>(k0 >> 3), kOmegaQ, v);
                    if (r >= p.ell) {  // selects, no FP64 math
#pragma unroll
                        for (int j = 0; j < 8; ++j) v[j] = 0.0;
                    }
                } else {
                    const double* src = p.omega + cp.s * p.stride_o + p.row0 + r;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        v[j] = (r < p.ell && k0 + j < p.m) ? __ldg(src + (k0 + j) * p.ldo) : 0.0;
                }
                // row r, 16B chunks 4ko..4ko+3, XOR-swizzled by r%8
                const uint32_t rowb = ob + r * (kKc * 8);
#pragma unroll
                for (int h = 0; h < 4; ++h)
                    sts128(rowb + ((((4 * ko + h) ^ (r & 7))) << 4), v[2 * h], v[2 * h + 1]);
            }
            mbar_arrive(&full_o[slot]);
            if (++cp.kc == nchunk) {
                cp.kc = 0;
                if (++cp.ct == ntiles_col) {
                    cp.ct = 0;
                    ++cp.s;
                }
            }
            if (++slot == S) {
                slot = 0;
                if (it + 1 >= 2 * S) epar ^= 1u;  // waits for chunk it-S: phase (it-S)/S
            }
        }
        return;
    }

    // ------------------------------- consumers -------------------------------
    const int grow = lane >> 2;  // fragment row (Omega) / column (A) within 8
    const int q4 = lane & 3;
    const int wm = warp / Cfg::kWn, wn = warp % Cfg::kWn;
    const int row0 = wm * MTW * 8;  // this warp's Omega rows
    const int col0 = wn * NW * 8;   // this warp's A columns

    double acc[MTW][NW][2];
#pragma unroll
    for (int i = 0; i < MTW; ++i)
#pragma unroll
        for (int j = 0; j < NW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    int slot = 0;
    uint32_t par = 0;
    ChunkPos cq = chunk_pos(lo, nchunk, ntiles_col);  // the chunk being contracted
    for (int64_t it = 0; it < niter; ++it) {
        mbar_wait(&full_a[slot], par);
        mbar_wait(&full_o[slot], par);
        const uint32_t at = a_s + slot * Cfg::kABytes;
        const uint32_t ot = o_s + slot * Cfg::kOBytes;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            // lane q feeds K = 4q + 2h + e: 16-byte pair (2q + h), swizzled by row%8 == grow
            const uint32_t ch = static_cast<uint32_t>(((2 * q4 + h) ^ grow) << 4);
            double2 of[MTW], af[NW];
#pragma unroll
            for (int mt = 0; mt < MTW; ++mt) of[mt] = lds128(ot + (row0 + 8 * mt + grow) * 128 + ch);
#pragma unroll
            for (int nt = 0; nt < NW; ++nt) af[nt] = lds128(at + (col0 + 8 * nt + grow) * 128 + ch);
#pragma unroll
            for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
                for (int nt = 0; nt < NW; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], of[mt].x, af[nt].x);
#pragma unroll
            for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
                for (int nt = 0; nt < NW; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], of[mt].y, af[nt].y);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);

        if (++slot == S) {
            slot = 0;
            par ^= 1u;
        }
        // last chunk of a segment (ranges end on segment ends): its partial
        // goes to the segment's own slot
        if (cq.kc + 1 == nchunk || (cq.kc + 1) % seg_len == 0) {
            const int64_t unit = (cq.s * ntiles_col + cq.ct) * nseg + cq.kc / seg_len;
            double* part = p.partial + static_cast<size_t>(unit) * (static_cast<size_t>(Cfg::kEllPad) * Cfg::kNt);
#pragma unroll
            for (int mt = 0; mt < MTW; ++mt)
#pragma unroll
                for (int nt = 0; nt < NW; ++nt) {
                    const int r = row0 + 8 * mt + grow, col = col0 + 8 * nt + 2 * q4;
                    *reinterpret_cast<double2*>(part + r * Cfg::kNt + col) =
                        make_double2(acc[mt][nt][0], acc[mt][nt][1]);
                    acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
                }
        }
        if (++cq.kc == nchunk) {
            cq.kc = 0;
            if (++cq.ct == ntiles_col) {
                cq.ct = 0;
                ++cq.s;
            }
        }
    }
}

// Fixed-order reduction of the segment partials of one (subdomain, column
// tile) into Y (column-major ell x n): slots summed in segment order (then
// half order), whichever CTA wrote them. One block per (tile, 8-row slab):
// partial rows are read coalesced (column fastest) into a padded shared
// slab, then written out column-major (row fastest).
constexpr int kRedRows = 8;
constexpr int kRedMaxNt = 256;

__global__ void __launch_bounds__(256) sketch_reduce_kernel(SketchParams p, int ell_pad, int nt, int64_t ntiles_col,
                                                            int64_t nseg, int halves) {
    __shared__ double slab[kRedRows][kRedMaxNt + 1];
    const int nslab = (static_cast<int>(p.ell) + kRedRows - 1) / kRedRows;
    const int64_t tile = blockIdx.x / nslab;
    const int r0 = (blockIdx.x % nslab) * kRedRows;
    const int64_t s = tile / ntiles_col, ct = tile % ntiles_col;
    const int ncols = static_cast<int>(p.n - ct * nt < nt ? p.n - ct * nt : nt);
    const int nrows = static_cast<int>(p.ell - r0 < kRedRows ? p.ell - r0 : kRedRows);
    const size_t slot_elems = static_cast<size_t>(ell_pad) * nt;
    const double* tpart = p.partial + static_cast<size_t>(tile) * nseg * halves * slot_elems;
    for (int e = threadIdx.x; e < nrows * ncols; e += blockDim.x) {
        const int rl = e / ncols, col = e % ncols;  // column fastest: coalesced partial reads
        const double* src = tpart + (r0 + rl) * nt + col;
        // segment order (the fixed association); loads batched 8 ahead of the adds
        const int64_t ng = nseg * halves;
        double sum = 0.0;
        int64_t g = 0;
        for (; g + 8 <= ng; g += 8) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcs(src + (g + u) * slot_elems);
#pragma unroll
            for (int u = 0; u < 8; ++u) sum += v[u];
        }
        for (; g < ng; ++g) sum += __ldcs(src + g * slot_elems);
        slab[rl][col] = sum;
    }
    __syncthreads();
    double* Y = p.Y + s * p.strideY + p.row0 + r0;
    for (int e = threadIdx.x; e < nrows * ncols; e += blockDim.x) {
        const int rl = e % nrows, col = e / nrows;  // row fastest: contiguous Y column pieces
        Y[(ct * nt + col) * p.ldy + rl] = slab[rl][col];
    }
}

__global__ void philox_omega_kernel(uint64_t seed, int64_t s, int64_t ell, int64_t m, double* out,
                                    int64_t ldo) {
    const int64_t no = (m + 7) / 8;
    const int64_t total = no * ell;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e % ell, ko = e / ell;
        double v[8];
        omega_values8(seed, static_cast<uint64_t>(s), static_cast<uint32_t>(r),
                      static_cast<uint32_t>(ko), kOmegaQ, v);
        for (int j = 0; j < 8; ++j)
            if (8 * ko + j < m) out[(8 * ko + j) * ldo + r] = v[j];
    }
}

template <int WM, int MTW, int NW, int OMODE>
cudaError_t launch_t(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap,
                     cudaStream_t stream) {
    using Cfg = SketchCfg<WM, MTW, NW>;
    auto kern = sketch_kernel<WM, MTW, NW, OMODE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Cfg::kSmem));
    if (e != cudaSuccess) return e;
    kern<<<plan.grid, kThreads, Cfg::kSmem, stream>>>(*tmap, p, plan.nchunk, plan.ntiles_col, plan.nseg,
                                                      plan.seg_len, plan.total_units);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    static_assert(Cfg::kNt <= kRedMaxNt, "reduce slab too narrow");
    return launch_sketch_reduce(p, plan, stream);
}

// (WM, MTW) by ell_pad; NW picks the column tile
template <int WM, int MTW, int OMODE>
cudaError_t launch_nw(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap,
                      cudaStream_t stream) {
    if constexpr (WM == 1) {
        switch (plan.nw) {
            case 1: return launch_t<WM, MTW, 1, OMODE>(p, plan, tmap, stream);
            default: return launch_t<WM, MTW, 2, OMODE>(p, plan, tmap, stream);
        }
    } else if constexpr (MTW <= 3) {
        switch (plan.nw) {
            case 1: return launch_t<WM, MTW, 1, OMODE>(p, plan, tmap, stream);
            case 2: return launch_t<WM, MTW, 2, OMODE>(p, plan, tmap, stream);
            default: return launch_t<WM, MTW, 4, OMODE>(p, plan, tmap, stream);
        }
    } else {  // ell_pad 64/80: cap the accumulator tile at MTW x 2 (register budget)
        switch (plan.nw) {
            case 1: return launch_t<WM, MTW, 1, OMODE>(p, plan, tmap, stream);
            default: return launch_t<WM, MTW, 2, OMODE>(p, plan, tmap, stream);
        }
    }
}

template <int OMODE>
cudaError_t launch_mode(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap,
                        cudaStream_t stream) {
    switch (plan.ell_pad) {
        case 8: return launch_nw<1, 1, OMODE>(p, plan, tmap, stream);
        case 16: return launch_nw<1, 2, OMODE>(p, plan, tmap, stream);
        case 24: return launch_nw<1, 3, OMODE>(p, plan, tmap, stream);
        case 32: return launch_nw<2, 2, OMODE>(p, plan, tmap, stream);
        case 48: return launch_nw<2, 3, OMODE>(p, plan, tmap, stream);
        case 64: return launch_nw<2, 4, OMODE>(p, plan, tmap, stream);
        case 80: return launch_nw<2, 5, OMODE>(p, plan, tmap, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace

// Omega rows handled by one launch: <= 80; wider sketches are sliced.
bool sketch_make_plan(int64_t m, int64_t n, int64_t batch, int64_t ell, int num_sms,
                      SketchPlan* plan) {
    if (m < 1 || n < 1 || batch < 1 || ell < 1 || ell > 80) return false;
    const int pads[] = {8, 16, 24, 32, 48, 64, 80};
    int ell_pad = 80;
    for (int v : pads)
        if (v >= ell) {
            ell_pad = v;
            break;
        }
    const int wm = ell_pad <= 24 ? 1 : 2;
    const int wn = kWarps / wm;
    int options[3];
    int nopt = 0;
    if (wm == 1 || ell_pad >= 64) {
        options[0] = 2, options[1] = 1, nopt = 2;
    } else {
        options[0] = 4, options[1] = 2, options[2] = 1, nopt = 3;
    }
    // column tile: least padded work; ties -> wider tile (fewer Omega regenerations)
    int best_nw = options[0];
    int64_t best_cols = INT64_MAX;
    for (int i = 0; i < nopt; ++i) {
        const int64_t nt = 8LL * options[i] * wn;
        const int64_t cols = ((n + nt - 1) / nt) * nt;
        if (cols < best_cols) {
            best_cols = cols;
            best_nw = options[i];
        }
    }
    plan->ell_pad = ell_pad;
    plan->mt = ell_pad / 8;
    plan->nw = best_nw;
    plan->nt = 8 * best_nw * wn;
    plan->ntiles_col = (n + plan->nt - 1) / plan->nt;
    plan->kc_rows = kKc;
    plan->nchunk = (m + kKc - 1) / kKc;
    plan->seg_len = kSketchSegRows / kKc;
    plan->nseg = (plan->nchunk + plan->seg_len - 1) / plan->seg_len;
    plan->total_units = batch * plan->ntiles_col * plan->nseg;
    int64_t grid = num_sms;
    if (grid > plan->total_units) grid = plan->total_units;
    plan->grid = static_cast<int>(grid);
    const int sbytes = (plan->nt + ell_pad) * kKc * 8;
    int stages = kStageBudget / sbytes;
    if (stages > 8) stages = 8;
    plan->smem = 1024 + static_cast<size_t>(stages) * sbytes + 24 * stages;
    plan->partial_elems = static_cast<size_t>(batch) * plan->ntiles_col * plan->nseg * ell_pad * plan->nt;
    return true;
}

cudaError_t launch_sketch_reduce(const SketchParams& p, const SketchPlan& plan, cudaStream_t stream) {
    if (plan.nt > kRedMaxNt) return cudaErrorInvalidValue;
    const int nslab = static_cast<int>((p.ell + kRedRows - 1) / kRedRows);
    sketch_reduce_kernel<<<static_cast<unsigned>(p.batch * plan.ntiles_col * nslab), 256, 0, stream>>>(
        p, plan.ell_pad, plan.nt, plan.ntiles_col, plan.nseg, plan.halves);
    return cudaGetLastError();
}

cudaError_t launch_sketch(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap,
                          cudaStream_t stream) {
    return p.omega_mode == 1 ? launch_mode<1>(p, plan, tmap, stream)
                             : launch_mode<0>(p, plan, tmap, stream);
}

cudaError_t launch_philox_omega(uint64_t seed, int64_t s, int64_t ell, int64_t m, double* out,
                                int64_t ldo, cudaStream_t stream) {
    const int64_t total = ((m + 7) / 8) * ell;
    int64_t blocks = (total + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    philox_omega_kernel<<<static_cast<unsigned>(blocks), 256, 0, stream>>>(seed, s, ell, m, out, ldo);
    return cudaGetLastError();
}

}  // namespace spidgpu
