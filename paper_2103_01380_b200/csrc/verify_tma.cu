// verify_tma.cu -- exact reconstruction error ||A_s - skel_s C_s||_F^2 and
// ||A_s||_F^2, warp-specialised on FP64 tensor cores.
//
// Restates reconstruct (proj/src/id.cpp:85-90 = matmul(skeleton, coeffs))
// followed by subtract + frobenius_norm (proj/src/metrics.cpp:14-21) without
// materialising the m x n reconstruction. Work per subdomain: 2*k*m*n flop
// (DMMA.8x8x4) and 8*m*(n+k) bytes (A and the skeleton, each read once), an
// arithmetic intensity of ~k/4 flop/B -- co-limited by the FP64 tensor pipe
// and HBM at k = 32.
//
// Layout of the work (mirrors sketch.cu):
//  * persistent grid, one CTA per SM, contiguous ranges of whole
//    (subdomain, column tile, 2048-row segment) units (as the sketch,
//    kernels.h), so the sums do not depend on the batch or the grid;
//  * 1 producer warp issues two TMA boxes per chunk -- A (16 rows x NT
//    columns) and the skeleton rows (16 rows x 4*KS columns), both 128B
//    swizzled -- into an S-stage mbarrier ring;
//  * 8 consumer warps; warp w owns columns [8*NWV*w, 8*NWV*(w+1)) of the
//    tile and keeps C's fragments for them in registers for the whole tile;
//    accumulator row (mt, grow) is chunk row 2*grow + mt, so one 16-byte
//    shared load yields both M tiles' skeleton fragment, and one yields the
//    two A values each accumulator pair is compared with (conflict free);
//  * err/ref are summed per lane, reduced per warp, written per (segment,
//    warp) and summed in a fixed order by a second kernel, so the result is
//    bitwise reproducible run to run and for any batching.
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace spidgpu {

namespace {

constexpr int kRows = 16;          // rows per chunk (one 128 B swizzle row)
// verify's fixed segments (batch independence, as the sketch's): 2048 rows --
// twice the units of 4096 evens out the per-CTA unit counts (config 3: 34.6
// instead of 17.3 units per CTA; 6.43 vs 6.55 ms), 1024 adds more segment
// flushes than it saves (6.53 ms)
constexpr int64_t kVerifySegRows = 2048;
constexpr int kCons = 8;           // consumer warps (2 per SMSP: 170 registers each)
constexpr int kThreadsV = (kCons + 1) * kWarp;
constexpr int kBudget = 200 * 1024;

template <int NWV, int KS>
struct VCfg {
    static constexpr int kNt = kCons * 8 * NWV;
    static constexpr int kABytes = kNt * kRows * 8;
    static constexpr int kSBytes = 4 * KS * kRows * 8;
    static constexpr int kStage = kABytes + kSBytes;
    static constexpr int kStages = (kBudget / kStage) < 8 ? (kBudget / kStage) : 8;
    static constexpr size_t kSmem = 1024 + static_cast<size_t>(kStages) * kStage + 2 * 8 * kStages;
};

template <int NWV, int KS>
__global__ void __launch_bounds__(kThreadsV, 1)
    verify_tma_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmS,
                      VerifyParams p, int64_t nchunk, int64_t ntiles_col, int64_t nseg, int64_t seg_len,
                      int64_t total_units, double* __restrict__ part) {
    using Cfg = VCfg<NWV, KS>;
    constexpr int S = Cfg::kStages;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw_s = smem_u32(smem_raw);
    const uint32_t base_s = (raw_s + 1023u) & ~1023u;
    unsigned char* base = smem_raw + (base_s - raw_s);
    const uint32_t a_s = base_s;                       // S stages of A
    const uint32_t sk_s = base_s + S * Cfg::kABytes;   // S stages of skeleton rows
    uint64_t* full = reinterpret_cast<uint64_t*>(base + S * Cfg::kStage);
    uint64_t* empty = full + S;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t G = gridDim.x, c = blockIdx.x;
    const int64_t lo = sketch_unit_chunk((c * total_units) / G, nseg, seg_len, nchunk);
    const int64_t hi = sketch_unit_chunk(((c + 1) * total_units) / G, nseg, seg_len, nchunk);
    const int64_t niter = hi - lo;
    if (niter <= 0) return;
    if (tid == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmS);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], kCons);
        }
        fence_barrier_init();
    }
    __syncthreads();

    int64_t tile = lo / nchunk, kc = lo % nchunk;
    if (warp == kCons) {
        // ------------------------------ producer ------------------------------
        if (lane == 0) {
            int slot = 0;
            uint32_t epar = 0;
            for (int64_t it = 0; it < niter; ++it) {
                if (it >= S) mbar_wait(&empty[slot], epar);
                const int64_t s = tile / ntiles_col, ct = tile % ntiles_col;
                mbar_arrive_expect_tx(&full[slot], Cfg::kStage);
                tma_load_3d(base + slot * Cfg::kABytes, &tmA, &full[slot],
                            static_cast<int>(kc * kRows), static_cast<int>(ct * Cfg::kNt),
                            static_cast<int>(s));
                tma_load_3d(base + S * Cfg::kABytes + slot * Cfg::kSBytes, &tmS, &full[slot],
                            static_cast<int>(kc * kRows), 0, static_cast<int>(s));
                if (++kc == nchunk) {
                    kc = 0;
                    ++tile;
                }
                if (++slot == S) {
                    slot = 0;
                    if (it + 1 >= 2 * S) epar ^= 1u;
                }
            }
        }
        return;
    }

    // ------------------------------- consumers -------------------------------
    const int grow = lane >> 2, q4 = lane & 3;
    const int col0 = warp * 8 * NWV;
    double cfr[KS][NWV];  // C fragments: C(t = 4ks + q4, col0 + 8nt + grow)
    int rank = 0, ksteps = 0;
    auto load_tile = [&](int64_t tl) {
        const int64_t s = tl / ntiles_col, ct = tl % ntiles_col;
        rank = static_cast<int>(p.rank[s]);
        ksteps = (rank + 3) >> 2;
        const double* Cs = p.C + s * p.strideC;
#pragma unroll
        for (int ks = 0; ks < KS; ++ks)
#pragma unroll
            for (int nt = 0; nt < NWV; ++nt) {
                const int t = 4 * ks + q4;
                const int64_t col = ct * Cfg::kNt + col0 + 8 * nt + grow;
                cfr[ks][nt] = (t < rank && col < p.n) ? __ldg(Cs + col * p.kcap + t) : 0.0;
            }
    };
    load_tile(tile);
    double err = 0.0, ref = 0.0;
    int slot = 0;
    uint32_t par = 0;
    // segment bookkeeping by counters (no 64-bit division per chunk); ranges
    // start on segment starts
    int64_t sg = kc / seg_len;                       // segment of the current chunk
    int64_t seg_left = seg_len;                      // chunks left in it
    for (int64_t it = 0; it < niter; ++it) {
        mbar_wait(&full[slot], par);
        const uint32_t at = a_s + slot * Cfg::kABytes;
        const uint32_t st = sk_s + slot * Cfg::kSBytes;
        double acc[2][NWV][2];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt)
#pragma unroll
            for (int nt = 0; nt < NWV; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
        // full-rank tiles (the common case) take a branch-free DMMA burst;
        // partial ranks mask the skeleton columns >= rank (their contents
        // are not part of the factor and may be anything, even NaN)
        auto kloop = [&](auto full) {
#pragma unroll
            for (int ks = 0; ks < KS; ++ks) {
                if (decltype(full)::value || ks < ksteps) {
                    const int t = 4 * ks + q4;
                    // skeleton rows 2*grow, 2*grow+1 of column t (16B chunk grow, swizzled by t%8)
                    double2 sv = lds128(st + t * 128 + ((grow ^ (t & 7)) << 4));
                    if (!decltype(full)::value && t >= rank) sv.x = sv.y = 0.0;
#pragma unroll
                    for (int nt = 0; nt < NWV; ++nt) {
                        dmma(acc[0][nt][0], acc[0][nt][1], sv.x, cfr[ks][nt]);
                        dmma(acc[1][nt][0], acc[1][nt][1], sv.y, cfr[ks][nt]);
                    }
                }
            }
        };
        if (rank == 4 * KS)
            kloop(std::true_type{});
        else
            kloop(std::false_type{});
        // compare with A: accumulator (mt, nt, e) is row 2*grow+mt, column col0+8nt+2q4+e
#pragma unroll
        for (int nt = 0; nt < NWV; ++nt)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int col = col0 + 8 * nt + 2 * q4 + e;
                const double2 av = lds128(at + col * 128 + ((grow ^ (col & 7)) << 4));
                const double d0 = av.x - acc[0][nt][e];
                const double d1 = av.y - acc[1][nt][e];
                err = fma(d0, d0, err);
                err = fma(d1, d1, err);
                ref = fma(av.x, av.x, ref);
                ref = fma(av.y, av.y, ref);
            }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == S) {
            slot = 0;
            par ^= 1u;
        }
        if (kc + 1 == nchunk || --seg_left == 0) {  // segment end: flush this warp's sums
            double e2 = err, r2 = ref;
#pragma unroll
            for (int off = 16; off > 0; off >>= 1) {
                e2 += __shfl_xor_sync(0xffffffffu, e2, off);
                r2 += __shfl_xor_sync(0xffffffffu, r2, off);
            }
            if (lane == 0) {
                double* dst = part + ((static_cast<size_t>(tile) * nseg + sg) * kCons + warp) * 2;
                dst[0] = e2;
                dst[1] = r2;
            }
            err = ref = 0.0;
            ++sg;
            seg_left = seg_len;
        }
        if (++kc == nchunk) {
            kc = 0;
            sg = 0;
            seg_left = seg_len;
            ++tile;
            if (it + 1 < niter) load_tile(tile);
        }
    }
}

// err2[s], ref2[s]: fixed-order sum over the subdomain's column tiles,
// their segments and the warps' partials.
__global__ void verify_tma_finish(VerifyParams p, int64_t ntiles_col, int64_t nseg, const double* part) {
    // one warp per subdomain: lane l adds partials l, l + 32, ... in order,
    // then a fixed butterfly -- a fixed association per subdomain, so the
    // sums stay independent of the batch
    const int64_t s = (blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (s >= p.batch) return;
    double e = 0.0, r = 0.0;
    const double* src = part + static_cast<size_t>(s) * ntiles_col * nseg * kCons * 2;
    for (int64_t g = lane; g < ntiles_col * nseg * kCons; g += 32) {
        e += src[2 * g];
        r += src[2 * g + 1];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        e += __shfl_xor_sync(0xffffffffu, e, off);
        r += __shfl_xor_sync(0xffffffffu, r, off);
    }
    if (lane == 0) {
        p.err2[s] = e;
        p.ref2[s] = r;
    }
}

template <int NWV, int KS>
cudaError_t launch_t(const VerifyParams& p, const VerifyPlan& plan, const CUtensorMap* tA,
                     const CUtensorMap* tS, double* part, cudaStream_t stream) {
    using Cfg = VCfg<NWV, KS>;
    auto kern = verify_tma_kernel<NWV, KS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Cfg::kSmem));
    if (e != cudaSuccess) return e;
    kern<<<plan.grid, kThreadsV, Cfg::kSmem, stream>>>(*tA, *tS, p, plan.nchunk, plan.ntiles_col, plan.nseg,
                                                       plan.seg_len, plan.total_units, part);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    verify_tma_finish<<<static_cast<unsigned>((p.batch + 3) / 4), 128, 0, stream>>>(p, plan.ntiles_col, plan.nseg,
                                                                                     part);
    return cudaGetLastError();
}

template <int NWV>
cudaError_t launch_ks(const VerifyParams& p, const VerifyPlan& plan, const CUtensorMap* tA,
                      const CUtensorMap* tS, double* part, cudaStream_t stream) {
    if constexpr (NWV == 4) {  // wide tiles only where C's fragments fit in registers
        switch (plan.ks) {
            case 2: return launch_t<NWV, 2>(p, plan, tA, tS, part, stream);
            case 4: return launch_t<NWV, 4>(p, plan, tA, tS, part, stream);
            case 8: return launch_t<NWV, 8>(p, plan, tA, tS, part, stream);
            default: return cudaErrorInvalidValue;
        }
    } else {
        switch (plan.ks) {
            case 2: return launch_t<NWV, 2>(p, plan, tA, tS, part, stream);
            case 4: return launch_t<NWV, 4>(p, plan, tA, tS, part, stream);
            case 8: return launch_t<NWV, 8>(p, plan, tA, tS, part, stream);
            case 12: return launch_t<NWV, 12>(p, plan, tA, tS, part, stream);
            case 16: return launch_t<NWV, 16>(p, plan, tA, tS, part, stream);
            default: return launch_t<NWV, 20>(p, plan, tA, tS, part, stream);
        }
    }
}

}  // namespace

bool verify_make_plan(int64_t m, int64_t n, int64_t batch, int64_t kcap, int num_sms,
                      VerifyPlan* plan) {
    if (m < 1 || n < 1 || batch < 1 || kcap < 1 || kcap > 80) return false;
    const int ksn = static_cast<int>((kcap + 3) / 4);
    const int opts[] = {2, 4, 8, 12, 16, 20};
    int ks = 20;
    for (int v : opts)
        if (v >= ksn) {
            ks = v;
            break;
        }
    // column tile of 128 or 256 (8 warps x 8 x NWV); least padded work; the
    // wide tile keeps 16 DMMA accumulators per warp (ILP) when C fits in registers
    const int64_t c128 = ((n + 127) / 128) * 128, c256 = ((n + 255) / 256) * 256;
    const int nwv = (c256 <= c128 && ks <= 8) ? 4 : 2;
    plan->nwv = nwv;
    plan->ks = ks;
    plan->nt = kCons * 8 * nwv;
    plan->ntiles_col = (n + plan->nt - 1) / plan->nt;
    plan->nchunk = (m + kRows - 1) / kRows;
    plan->seg_len = kVerifySegRows / kRows;
    plan->nseg = (plan->nchunk + plan->seg_len - 1) / plan->seg_len;
    plan->total_units = batch * plan->ntiles_col * plan->nseg;
    int64_t grid = num_sms;
    if (grid > plan->total_units) grid = plan->total_units;
    plan->grid = static_cast<int>(grid);
    plan->part_elems = static_cast<size_t>(plan->total_units) * kCons * 2;
    return true;
}

cudaError_t launch_verify_tma(const VerifyParams& p, const VerifyPlan& plan, const CUtensorMap* tA,
                              const CUtensorMap* tS, double* part, cudaStream_t stream) {
    return plan.nwv == 4 ? launch_ks<4>(p, plan, tA, tS, part, stream)
                         : launch_ks<2>(p, plan, tA, tS, part, stream);
}

}  // namespace spidgpu
