// sketch_tc.cu -- the performance-mode sketch Y_s = Omega_s * A_s as an EXACT
// integer-sliced contraction on the 5th-generation tensor cores
// (tcgen05.mma kind::i8, accumulators in TMEM).
//
// The north star's Gaussian sketch in place of subsample/subsample_column
// (proj/src/grid.cpp:136-150;
// CPU restatement matmul(Omega, A), proj/src/dense_matrix.cpp:38-53): the
// Philox Omega is integer-valued (Omega = Q/32, |Q| <= 117, philox.cuh), each
// column of A is a fixed-point integer v = rint(x 2^(50-E)) per period (E =
// exponent of the period's first 32 rows + 3 bits of headroom), formed by ONE
// DFMA as the mantissa of x 2^(50-E) + 1.5 2^52: its low 56 bits are the
// offset-binary u = v + 7 2^51, split into 7 unsigned byte slices, each
// contracted exactly with Q in int32; an 8th MMA against an all-ones tile
// accumulates sum_k Q, and the offset is removed exactly (int64) at flush.
// A register-fed IMMA.16832 version of the same contraction (round 1, now
// retired) was bound by its issue rate (8 cycles per m16n8k32 per SMSP) at
// ~76% of HBM; on UTCIMMA the kernel is bound by the HBM stream of A.
//
// Formulation: Y_s^T (n x ell) = A_s^T (n x m) * Omega_s^T (m x ell), per CTA
// tile of 128 snapshots: D_t (M=128 snapshots x N=ell_pad, int32, TMEM
// columns [N t, N t + N)) += slice_t(A^T) (128 x 32, K-major) *
// Q^T (32 x N, K-major), one MMA per slice per 32-row stage.
//
// Warp roles (512 threads, persistent, one CTA per SM, contiguous ranges of
// whole (subdomain, 128-column tile, 4096-row segment) units like sketch.cu,
// kernels.h):
//   warps 0-7   (80 registers) Omega: warps 0, 2..7 run Philox + quantile
//               table -> K-major int8 tile, at most one task per lane per
//               stage; warp 0's lane 0 also keeps the A ring full (two
//               16x128 fp64 TMA boxes, 128B swizzle, per stage), warp 1
//               allocates TMEM and its lane 0 issues the 8 MMAs per stage,
//               committed to the slot's "empty" mbarrier
//   warps 8-15  (176 registers) converters, two per TMEM lane quarter, 16 columns each;
//               thread = (column, row half): 16 fp64 entries of the stage ->
//               one DFMA each (offset-binary fixed point, below) -> 4x4 PRMT
//               byte transposes -> one 16-byte store per slice into the
//               K-major slice tile. A warp owns its 16 D rows: its rare
//               flushes read them (tcgen05.ld 16x64b) into the fp64 partial
//               and zero them (tcgen05.st), without involving another warp.
// A warp flushes its rows at segment ends (128 stages, so |D| < 2^31), when
// one of its columns exceeds its exponent headroom, and when a column's
// magnitude falls more than kFallback binades below its epoch's (so a
// spike cannot coarsen the rest of the segment).
//
// Accuracy contract (tests/test_gpu_sketch_i8.py). Each entry x of an epoch
// with exponent E is rounded once, to a multiple of 2^(E-50), and everything
// after that is exact integer arithmetic, so per column j
//   |Y(i,j) - (Omega A)(i,j)| <= sum_k |Omega(i,k)| 2^(E_k - 51) + fp64 rounding of the flush sums,
// E_k the exponent of the epoch holding row k: 2^(E_k-51) <= 2^-47 of the
// epoch's first-stage maximum, and (fallback) at most 2^(kFallback-47) of
// the row's own 32-row stage maximum. Epochs start at absolute segment
// starts, so the result does not depend on how subdomains are batched.
#include <math.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace spidgpu {

namespace {

constexpr int kThreads = 512;
constexpr int kConvWarps = 8;         // warps 8..15: two per TMEM lane quarter
constexpr int kGenWarps = 7;          // warps 0, 2..7 generate Omega (warp 1 issues the MMAs)
// register split (setmaxnreg; launch budget 512 x 128): warpgroups 0-1 (TMA,
// MMA, Omega) 80, warpgroups 2-3 (converters) 176
constexpr int kAuxRegs = 80;
constexpr int kConvRegs = 176;
static_assert(8 * 32 * (kAuxRegs + kConvRegs) <= 65536, "register file");
constexpr int kM = 128;               // snapshots per CTA tile (UMMA M)
constexpr int kRows = 32;             // rows of A per stage (UMMA K for int8)
constexpr int kSlices = 7;            // byte slices of the offset-binary fixed point
constexpr int kP = 50;                // v = rint(x 2^(P-E)), |v| < 2^50 within the headroom
constexpr int kHeadroom = 3;
// t = RN(x 2^(P-E) + 1.5 2^52) holds v in its mantissa: the low 56 bits of
// t's bit pattern are u = v + kOffset (the exponent field 0x433 contributes
// its low nibble 3 at bit 52), an unsigned 7-byte integer while |v| < 2^51
constexpr double kMagic = 6755399441055744.0;  // 1.5 * 2^52
constexpr int kOffsetHi = 7 << 19;             // kOffset = 7 * 2^51 = kOffsetHi * 2^32
constexpr int kEbMin = 9;
constexpr int kFallback = 24;         // restart an epoch when a stage's max is 2^24 below its scale
static_assert(kSketchSegRows / kRows <= 2048, "a segment's int32 sums stay exact: 65536 * 117 * 255 < 2^31");
constexpr int kBoxBytes = 16 * kM * 8;              // 16 rows x 128 columns fp64
constexpr int kAStageBytes = 2 * kBoxBytes;         // 32 KB
constexpr int kAStages = 5;
constexpr int kSliceBytes = kM * kRows;             // 4 KB per slice tile

// instrumentation (spidgpu_debug_counters): converter-warp flushes by cause
// [segment end, headroom overflow, magnitude fallback]; atomics only on flushes
__device__ unsigned long long g_tc_flushes[3];

// Kernel modes. 0: one CTA per (subdomain, 128-column tile). 1 (tile pair):
// clusters of two over a subdomain's two column tiles, sharing each stage's
// Omega tile. 2 (slice split): clusters of two over the SAME column tile, so
// that ell_pad = 80 fits TMEM (8 accumulators x 80 columns would not fit 512):
//   - CTA r loads and converts only rows [16r, 16r + 16) of every 32-row
//     stage -- exactly K half r of every slice tile -- so A is read and
//     converted once;
//   - a column's exponent must be the same in both CTAs: each publishes its
//     16-row column maxima into the peer's mailbox (st.async, one stage
//     ahead of use) and both take the max of the two halves, so both make
//     identical epoch decisions;
//   - CTA 0 keeps slices 0-3, CTA 1 slices 4-6 and the offset accumulator
//     (4 accumulators of N = 80 each); the slices a CTA does not keep go to
//     the peer's slice tiles by st.async, counted on its stage barrier;
//   - each CTA flushes its own accumulators into its half of the segment's
//     partial slot (the reduction adds the halves).
// The single-pass sketch for ell in (64, 80] (config 4's kmax 64 + p 16).
template <int NPAD, int MODE>
struct TcCfg {
    static constexpr bool kSplit = MODE == 2;
    static constexpr int kSl = kSplit ? 4 : kSlices;        // slice tiles per B stage
    static constexpr int kAcc = kSplit ? 4 : kSlices + 1;   // TMEM accumulators
    // rows per stage: 32 (one UMMA K block); split: 64, 32 per CTA, so each
    // converter thread still handles 16 entries per stage and the per-stage
    // costs (barriers, exponent checks) are paid once per 64 rows
    static constexpr int kStageRows = kSplit ? 64 : kRows;
    static constexpr int kKB = kStageRows / kRows;            // UMMA K blocks per stage
    static constexpr int kTileBytes = kKB * kSliceBytes;      // one slice tile of a stage
    static constexpr int kOmegaBytes = NPAD * kStageRows;
    static constexpr int kBStageBytes = kSl * kTileBytes + kOmegaBytes;
    // slice/Omega stages: 2 (3 in split mode, whose two CTAs advance in lock-step)
    static constexpr int kBStages = kSplit ? 2 : 2;
    // A ring: 2 x 16-row boxes per stage (split: this CTA's 32 rows of the 64)
    static constexpr int kAStB = kAStageBytes;
    static constexpr int kASt = kSplit ? 4 : kAStages;
    static_assert(!kSplit || kASt >= 3, "mailbox slots outlive the peer lead");
    // D_0..D_6 (slices) and D_7 = sum_k Q (all-ones A tile): the offset correction
    static constexpr int kTmemCols = kAcc * NPAD <= 256 ? 256 : 512;
    static_assert(kAcc * NPAD <= 512, "TMEM columns");
    // layout: A ring | B ring | ebx[2][128] | flags | barriers
    static constexpr size_t kOffB = static_cast<size_t>(kASt) * kAStB;
    static constexpr size_t kOffMisc = kOffB + static_cast<size_t>(kBStages) * kBStageBytes;
    // Omega table; TMEM slot; all-ones core matrix; (split) the peer's column maxima per A slot
    static constexpr size_t kMiscBytes = 4096 + 64 + 128 + (kSplit ? kASt * kM * 4 : 0);
    static constexpr size_t kOffBar = (kOffMisc + kMiscBytes + 7) & ~size_t(7);
    static constexpr size_t kSmem = 1024 + kOffBar + 8 * (3 * kASt + 2 * kBStages) + 16;
};

struct ChunkPos {
    int s, ct, kc;  // subdomain, column tile, 32-row stage
};

__device__ __forceinline__ ChunkPos chunk_pos(int64_t g, int64_t nchunk, int64_t ntiles_col) {
    const int64_t tile = g / nchunk;
    return ChunkPos{static_cast<int>(tile / ntiles_col), static_cast<int>(tile % ntiles_col),
                    static_cast<int>(g % nchunk)};
}

__device__ __forceinline__ void advance(ChunkPos& cp, int nchunk, int ntiles_col) {
    if (++cp.kc == nchunk) {
        cp.kc = 0;
        if (++cp.ct == ntiles_col) {
            cp.ct = 0;
            ++cp.s;
        }
    }
}

__device__ __forceinline__ void sts64u(uint32_t addr, uint32_t a, uint32_t b) {
    asm volatile("st.shared.v2.u32 [%0], {%1, %2};\n" ::"r"(addr), "r"(a), "r"(b) : "memory");
}

__device__ __forceinline__ void sts128u(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};\n" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    // K-major, no swizzle (canonical interleave): core matrices of 8 rows x
    // 16 B, row groups SBO apart, the two 16-byte K halves LBO apart;
    // version 1 (tcgen05), layout type 0
    return static_cast<uint64_t>((addr >> 4) & 0x3fffu) |
           (static_cast<uint64_t>((lbo >> 4) & 0x3fffu) << 16) |
           (static_cast<uint64_t>((sbo >> 4) & 0x3fffu) << 32) | (1ull << 46);
}

// kind::i8 instruction descriptor: D s32, A (slices) u8 or s8, B (Q) s8, both K-major
__host__ __device__ constexpr uint32_t idesc_i8(int n, bool a_signed) {
    return (2u << 4) | ((a_signed ? 1u : 0u) << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
           (static_cast<uint32_t>(kM >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                        uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

// one lane of a converged warp
__device__ __forceinline__ bool elect_one() {
    uint32_t pred;
    asm volatile("{\n.reg .pred P;\nelect.sync _|P, 0xffffffff;\nselp.u32 %0, 1, 0, P;\n}\n" : "=r"(pred));
    return pred != 0;
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

// ---- CTA pairs (thread-block clusters of 2) ------------------------------------
// completion of this CTA's MMAs arrives on the barrier at the same offset in both CTAs
__device__ __forceinline__ void umma_commit_pair(uint64_t* bar) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
            smem_u32(bar)),
        "h"(static_cast<uint16_t>(3))
        : "memory");
}
__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}
// the peer CTA's shared::cluster address of a local shared address
__device__ __forceinline__ uint32_t peer_addr(uint32_t local, uint32_t peer) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(local), "r"(peer));
    return r;
}
// 16 / 8 bytes into the peer's shared memory, completing on the peer's mbarrier
__device__ __forceinline__ void st_async_v4(uint32_t raddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d,
                                            uint32_t rbar) {
    asm volatile(
        "st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];\n" ::"r"(raddr),
        "r"(a), "r"(b), "r"(c), "r"(d), "r"(rbar)
        : "memory");
}
__device__ __forceinline__ void st_async_b32(uint32_t raddr, uint32_t a, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];\n" ::"r"(raddr), "r"(a),
                 "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t raddr, uint32_t a, uint32_t b, uint32_t rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b32 [%0], {%1, %2}, [%3];\n" ::"r"(raddr),
                 "r"(a), "r"(b), "r"(rbar)
                 : "memory");
}

// .16x64b: the warp's 16 lanes from the address' lane field; thread t holds
// lane 8 (t & 1) + (t >> 2), columns ((t >> 1) & 1) + 2 j (probed on B200:
// tools/microbench/tmem_16dp.cu)
__device__ __forceinline__ void tmem_ld16x64b_x8(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.16x64b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
__device__ __forceinline__ void tmem_st16x64b_x8_zero(uint32_t taddr) {
    asm volatile("tcgen05.st.sync.aligned.16x64b.x8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};\n" ::"r"(taddr), "r"(0u)
                 : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }

__device__ __forceinline__ int column_eb(uint32_t mg) {
    const int eb = static_cast<int>(mg >> 20) + 1 + kHeadroom;
    return eb < kEbMin ? kEbMin : (eb > 2047 ? 2047 : eb);
}

// 2^(P - E) as two normal doubles (tiny columns need more than 2^1023)
__device__ __forceinline__ double2 fix_scale(int eb) {
    const int d = kP + 1023 - eb;
    const int d1 = d > 1000 ? 1000 : d;
    return make_double2(__longlong_as_double(static_cast<long long>(d1 + 1023) << 52),
                        __longlong_as_double(static_cast<long long>(d - d1 + 1023) << 52));
}

// 2^(E - P) / 32, likewise split
__device__ __forceinline__ double2 unfix_scale(int eb) {
    const int e = eb - 1023 - kP - kOmegaScaleLog2;
    const int e1 = e < -1000 ? -1000 : e;
    return make_double2(__longlong_as_double(static_cast<long long>(e1 + 1023) << 52),
                        __longlong_as_double(static_cast<long long>(e - e1 + 1023) << 52));
}

// A converter warp's flush of its 16 TMEM lanes (all 8 accumulators): the
// exact integer sums -> fp64 partial of the segment (scaled by the epoch's
// exponent ebf; poisoned columns become NaN at the segment's final flush);
// `zero` clears the lanes for an epoch restart inside the segment. Kept out
// of line: flushes are rare (segment ends, exponent restarts), and inlining
// their 8 x 8 TMEM loads into the converter loop raised its register
// pressure enough for the compiler to rematerialise addresses every stage.
// Split mode (MODE 2): CTA 0 holds D_0..D_3 and writes lo * 2^(E-P-5);
// CTA 1 holds D_4..D_6 and D_7 and writes hi * 2^32 * 2^(E-P-5), each into
// its half of the segment's slot (the reduction adds the halves).
template <int NPAD, int MODE>
__device__ __noinline__ void tc_flush_rows(uint32_t taddr, double* part, int ebf, int psf, int pf, int col_f,
                                           bool final_flush, bool zero, bool first, int half) {
    constexpr int kAcc = TcCfg<NPAD, MODE>::kAcc;
    const double2 u = unfix_scale(ebf);
#pragma unroll 1
    for (int g0 = 0; g0 < NPAD; g0 += 16) {
        // exact: sum_t 2^(8t) D_t - kOffset * D_7 as hi * 2^32 + lo, for
        // columns g0 + pf + 2j of this thread's D row
        uint32_t v[kAcc][8];
#pragma unroll
        for (int t = 0; t < kAcc; ++t) tmem_ld16x64b_x8(taddr + NPAD * t + g0, v[t]);
        tmem_ld_wait();
        if (zero) {
#pragma unroll
            for (int t = 0; t < kAcc; ++t) tmem_st16x64b_x8_zero(taddr + NPAD * t + g0);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            long long lo64 = 0, hi64 = 0;
#pragma unroll
            for (int t = 0; t < kAcc; ++t) {
                const long long d = static_cast<int>(v[t][j]);
                // slice index of accumulator t (split: CTA 1's are slices 4.. and the offset)
                const int sl = MODE == 2 ? t + 4 * half : t;
                if (sl < 4)
                    lo64 += d * (1LL << (8 * sl));
                else if (sl < kSlices)
                    hi64 += d * (1LL << (8 * (sl - 4)));
                else
                    hi64 -= d * kOffsetHi;
            }
            double val = fma(static_cast<double>(hi64), 4294967296.0, static_cast<double>(lo64)) * u.x * u.y;
            if (final_flush && psf) val = __longlong_as_double(0x7ff8000000000000LL);
            double* dst = part + static_cast<size_t>(g0 + pf + 2 * j) * kM + col_f;
            *dst = first ? val : *dst + val;
        }
    }
    if (zero) tmem_st_wait();
}

// Clusters (modes 1 and 2): each CTA generates HALF of every stage's Omega
// tile and writes it into both CTAs' shared memory (the peer's half arrives
// by st.async, counted on the local stage barrier as transaction bytes);
// every MMA completion is multicast to both CTAs' slot barriers, so a slot is
// refilled only when both CTAs' MMAs have read it. Work units are (subdomain,
// column tile -- or tile pair in mode 1 --, segment); ntiles_col counts
// units' column tiles (column tiles / 2 in mode 1).
template <int NPAD, int MODE>
__global__ void __launch_bounds__(kThreads, 1)
    sketch_tc_kernel(const __grid_constant__ CUtensorMap tmap, SketchParams p, int64_t nchunk,
                     int64_t ntiles_col, int64_t nseg, int64_t seg_len, int64_t total_units) {
    constexpr bool kPair = MODE != 0;             // a cluster of two
    constexpr bool kSplit = MODE == 2;
    constexpr int P = kPair ? 2 : 1;              // CTAs per work-unit owner
    constexpr int TP = MODE == 1 ? 2 : 1;         // column tiles per unit
    constexpr int kHalves = kSplit ? 2 : 1;       // partials per segment slot
    using Cfg = TcCfg<NPAD, MODE>;
    constexpr int kSl = Cfg::kSl;
    constexpr int kBStages = Cfg::kBStages;
    constexpr int kAStages = Cfg::kASt;
    constexpr int kAStageBytes = Cfg::kAStB;
    constexpr int kStageRows = Cfg::kStageRows, kKB = Cfg::kKB, kTileBytes = Cfg::kTileBytes;
    // Omega tile tasks (one Philox call = one octet, or two for a 16-byte K
    // half when the tile has more octets than generator lanes), split over
    // the cluster's CTAs, at most one per lane, on as few warps as that takes
    // (a warp's instructions per stage do not shrink with idle lanes: -3%
    // cycles at ell 64 and 80)
    constexpr int kOctets = kStageRows / 8;  // per Omega row and stage
    constexpr bool kFine = kOctets * NPAD <= 32 * kGenWarps * P;
    constexpr int kTasks = kFine ? kOctets * NPAD : kOctets / 2 * NPAD;
    constexpr int kTasksCta = kTasks / P;
    constexpr int kGenNeed = (kTasksCta + 31) / 32 < 1 ? 1 : (kTasksCta + 31) / 32;
    constexpr int kGenActive = kGenNeed < kGenWarps ? kGenNeed : kGenWarps;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw_s = smem_u32(smem_raw);
    const uint32_t base_s = (raw_s + 1023u) & ~1023u;
    unsigned char* base = smem_raw + (base_s - raw_s);
    const uint32_t a_s = base_s;
    const uint32_t b_s = base_s + static_cast<uint32_t>(Cfg::kOffB);
    int8_t* tab = reinterpret_cast<int8_t*>(base + Cfg::kOffMisc);                // 4096
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tab + 4096);
    // one all-ones 8x16 core matrix; with LBO = SBO = 0 it reads as a 128 x 32 all-ones A tile
    const uint32_t ones_s = smem_u32(tab + 4096 + 64);
    const uint32_t mbox_s = smem_u32(tab + 4096 + 64 + 128);  // split: [kAStages][kM] peer maxima
    uint64_t* a_full = reinterpret_cast<uint64_t*>(base + Cfg::kOffBar);
    uint64_t* a_empty = a_full + kAStages;
    uint64_t* b_full = a_empty + kAStages;
    uint64_t* b_empty = b_full + kBStages;
    uint64_t* m_full = b_empty + kBStages;  // split: the peer's maxima of an A slot arrived

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t c = blockIdx.x;
    const uint32_t rank = kPair ? cluster_ctarank() : 0u;
    // the peer's shared::cluster window is this CTA's layout shifted by a
    // constant: remote = local + poff (one mapa instead of one per store)
    const uint32_t poff = kPair ? peer_addr(base_s, rank ^ 1u) - base_s : 0u;
    const int64_t G = gridDim.x / P, cu = c / P;  // work-unit owners: CTAs, or CTA pairs
    const int64_t lo = sketch_unit_chunk((cu * total_units) / G, nseg, seg_len, nchunk);
    const int64_t hi = sketch_unit_chunk(((cu + 1) * total_units) / G, nseg, seg_len, nchunk);
    const int niter = static_cast<int>(hi - lo);
    if (niter <= 0) return;  // both CTAs of a pair share the range

    for (int i = tid; i < 1024; i += kThreads)
        reinterpret_cast<int*>(tab)[i] = reinterpret_cast<const int*>(kOmegaQ)[i];
    for (int i = tid; i < 32; i += kThreads) reinterpret_cast<uint32_t*>(tab + 4096 + 64)[i] = 0x01010101u;
    fence_proxy_async();
    if (tid == 0) {
        prefetch_tmap(&tmap);
        for (int i = 0; i < kAStages; ++i) {
            mbar_init(&a_full[i], 1);
            mbar_init(&a_empty[i], kConvWarps);
            mbar_init(&m_full[i], 1);
        }
        if constexpr (kSplit)  // the mailboxes' first phases: the peer's 128 column maxima of stages 0..
            for (int i = 0; i < kAStages; ++i) mbar_arrive_expect_tx(&m_full[i], kM * 4);
        for (int i = 0; i < kBStages; ++i) {
            mbar_init(&b_full[i], kConvWarps + kGenActive);
            mbar_init(&b_empty[i], P);  // MMA commits of this CTA (and of its peer)
        }
        fence_barrier_init();
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tmem_slot)),
                     "n"(Cfg::kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    tc_fence_before();
    if constexpr (kPair)
        cluster_sync_all();  // barriers initialised in both CTAs before any remote traffic
    else
        __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp < 8) {
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kAuxRegs));
        // ------------------- Omega tiles (+ TMA on warp 0, MMA on warp 1) -------------------
        // Warps 0, 2..7 generate the Omega tile (warp 0's lane 0 also refills
        // the A ring); warp 1's lane 0 only issues the MMAs, as soon as a
        // stage's slices and Omega are complete. A task is one Philox call
        // (8 entries of one Omega row, an 8-byte store) when the tile has at
        // most one per generator lane, else two (16 bytes): each lane runs at
        // most one task per stage, so the tile's latency is one task's.
        // A pair splits the tile's tasks: this CTA runs [rank, rank + 1) x
        // kTasksCta of them and also writes them into the peer's tile.
        // (task decomposition at the top of the kernel: kFine, kTasksCta, kGenActive)
        constexpr int kTasksPerWarp = (kTasksCta + kGenActive - 1) / kGenActive;
        constexpr uint32_t kPeerBytes = kTasksCta * (kFine ? 8 : 16);  // Omega bytes the peer sends per stage
        static_assert(kTasksPerWarp <= 32, "one Omega task per lane");
        const int gw = warp == 0 ? 0 : warp - 1;

        constexpr uint32_t kIdU = idesc_i8(NPAD, false);
        const uint64_t ones_desc = smem_desc(ones_s, 0, 0);
        auto issue_mma = [&](int it, int seg_pos) {
            const int sl = it % kBStages;
            mbar_wait(&b_full[sl], (it / kBStages) & 1);
            tc_fence_after();
            // a segment's first stage overwrites D (its owners read the old
            // segment out before arriving); epoch restarts inside a segment
            // zero their rows themselves
            const uint32_t acc = seg_pos != 0 ? 1u : 0u;
            const uint32_t st = b_s + sl * Cfg::kBStageBytes;
            const uint32_t ot = st + kSl * kTileBytes;  // Omega tile: K blocks of NPAD x 32 bytes
            if (!elect_one()) {
            } else if constexpr (!kSplit) {
                const uint64_t bdesc = smem_desc(ot, NPAD * 16, 128);
#pragma unroll
                for (int t = 0; t < kSlices; ++t)
                    umma_i8(tmem + NPAD * t, smem_desc(st + t * kTileBytes, kM * 16, 128), bdesc, kIdU, acc);
                umma_i8(tmem + NPAD * kSlices, ones_desc, bdesc, kIdU, acc);
            } else {
                // CTA 0: slices 0-3; CTA 1: slices 4-6 (tiles 0-2) and the offset
                // (ones); one MMA per K block (K block kb = rows of CTA kb)
#pragma unroll
                for (int kb = 0; kb < kKB; ++kb) {
                    const uint64_t bdesc = smem_desc(ot + kb * (NPAD * 32), NPAD * 16, 128);
#pragma unroll
                    for (int t = 0; t < 4; ++t)
                        umma_i8(tmem + NPAD * t,
                                rank == 1 && t == 3 ? ones_desc
                                                    : smem_desc(st + t * kTileBytes + kb * kSliceBytes, kM * 16, 128),
                                bdesc, kIdU, kb > 0 ? 1u : acc);
                }
            }
            __syncwarp();
            if (elect_one()) {
                if constexpr (kPair)
                    umma_commit_pair(&b_empty[sl]);
                else
                    umma_commit(&b_empty[sl]);
            }
            __syncwarp();
        };
        ChunkPos cp = chunk_pos(lo, nchunk, ntiles_col);
        ChunkPos tp = cp;  // TMA position (warp 0)
        auto issue_tma = [&](int it) {
            const int sl = it % kAStages;
            mbar_arrive_expect_tx(&a_full[sl], kAStageBytes);
            // two 16-row boxes: the stage's 32 rows (split: this CTA's 32 of the 64)
#pragma unroll
            for (int b = 0; b < 2; ++b)
                tma_load_3d(base + sl * kAStageBytes + b * kBoxBytes, &tmap, &a_full[sl],
                            static_cast<int>(tp.kc * kStageRows + (kSplit ? 32 * static_cast<int>(rank) : 0) + 16 * b),
                            static_cast<int>((tp.ct * TP + (TP == 2 ? static_cast<int>(rank) : 0)) * kM),
                            static_cast<int>(tp.s));
            advance(tp, static_cast<int>(nchunk), static_cast<int>(ntiles_col));
        };
        if (warp == 0 && lane == 0)
            for (int it = 0; it < kAStages && it < niter; ++it) issue_tma(it);
        if (warp == 1) {  // dedicated MMA issuer: no Omega work, so MMAs go out as soon as a stage is full
            // the whole warp runs the loop (warp-uniform values stay in
            // uniform registers); one elected lane issues the MMAs
            // position inside the current segment (ranges start on segment starts)
            int sp = 0, kc = cp.kc;
            const int nch = static_cast<int>(nchunk), sl = static_cast<int>(seg_len);
            for (int it = 0; it < niter; ++it) {
                issue_mma(it, sp);
                if (++kc == nch) kc = sp = 0;
                else if (++sp == sl) sp = 0;
            }
        } else if (gw < kGenActive)  // warp 0 (gw 0, the TMA producer) always runs the loop
        for (int it = 0; it < niter; ++it) {
            const int sl = it % kBStages;
            const uint32_t ot = b_s + sl * Cfg::kBStageBytes + kSl * kTileBytes;
            const uint32_t ko = static_cast<uint32_t>((cp.kc * kStageRows) >> 3);
            const int task_l = gw * kTasksPerWarp + lane;
            const bool has_task = lane < kTasksPerWarp && task_l < kTasksCta;
            const int task = static_cast<int>(rank) * kTasksCta + task_l;
            // row r, K octet(s) from o8: fine tasks one octet, else a 16-byte K half
            const int r = task % NPAD, o8 = (kFine ? 1 : 2) * (task / NPAD);
            constexpr int kOct = kFine ? 1 : 2;
            uint32_t w[2 * kOct];
#pragma unroll
            for (int i = 0; i < 2 * kOct; ++i) w[i] = 0u;
            if (has_task && r < p.ell) {
#pragma unroll
                for (int o = 0; o < kOct; ++o) {
                    int q[8];
                    omega_q8(p.seed, static_cast<uint64_t>(p.sub_base + cp.s), static_cast<uint32_t>(p.row0 + r),
                             ko + o8 + o, tab, q);
#pragma unroll
                    for (int e = 0; e < 8; ++e) w[2 * o + e / 4] |= static_cast<uint32_t>(q[e] & 0xff) << (8 * (e & 3));
                }
            }
            // generated ahead; only the store waits for the MMAs that read the slot
            if (it >= kBStages) mbar_wait(&b_empty[sl], ((it / kBStages) - 1) & 1);
            if (has_task) {
                // K-major core-matrix layout: K half o8 / 2 at NPAD * 16 B, row r at 16 B
                const uint32_t dst = ot + (o8 >> 1) * (NPAD * 16) + r * 16 + (o8 & 1) * 8;
                if constexpr (kFine)
                    sts64u(dst, w[0], w[1]);
                else
                    sts128u(dst, w[0], w[1], w[2 * kOct - 2], w[2 * kOct - 1]);
                if constexpr (kPair) {  // the peer's copy, counted on its stage barrier
                    const uint32_t rdst = dst + poff, rbar = smem_u32(&b_full[sl]) + poff;
                    if constexpr (kFine)
                        st_async_v2(rdst, w[0], w[1], rbar);
                    else
                        st_async_v4(rdst, w[0], w[1], w[2 * kOct - 2], w[2 * kOct - 1], rbar);
                }
            }
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) {
                if (kPair && warp == 0)  // the peer's half of the Omega tile (and, split, its K half of our slices)
                    mbar_arrive_expect_tx(&b_full[sl], kPeerBytes + (kSplit ? (rank == 0 ? 4u : 3u) * kSliceBytes : 0u));
                else
                    mbar_arrive(&b_full[sl]);
            }
            advance(cp, static_cast<int>(nchunk), static_cast<int>(ntiles_col));
            if (lane == 0) {
                if (warp == 0 && it + kAStages < niter) {
                    // refill the slot the converters release after reading stage it
                    mbar_wait(&a_empty[it % kAStages], (it / kAStages) & 1);
                    issue_tma(it + kAStages);
                }
            }
            __syncwarp();
        }
    } else {
        asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kConvRegs));
        // ------------------------------ converters ------------------------------
        // Two warps per TMEM lane quarter: warp w (8..15) owns the 16 columns
        // 32 (w % 4) + 16 hh + [0, 16) (hh = (w - 8) / 4) = those TMEM lanes,
        // all 32 rows of every stage and all slices. Conversion: lane =
        // (column cc = lane & 15, row half b = lane >> 4), 16 entries each;
        // the two halves of a column share its exponent through one shuffle.
        // Flush: tcgen05.ld/st .16x64b touch only the warp's 16 lanes (lane L
        // = 8 (t & 1) + (t >> 2), column parity (t >> 1) & 1 per thread t), so
        // a column's overflow handling and flushes never involve another warp.
        ChunkPos cp = chunk_pos(lo, nchunk, ntiles_col);
        const int q = warp & 3, hh = (warp - 8) >> 2;
        const int cc = lane & 15, b = lane >> 4;
        const int col = q * 32 + hh * 16 + cc;
        const uint32_t lane_base = static_cast<uint32_t>(q * 32 + hh * 16) << 16;
        const int lf = 8 * (lane & 1) + (lane >> 2), pf = (lane >> 1) & 1;  // flush: D lane, column parity
        const int col_f = q * 32 + hh * 16 + lf;
        int eb = kEbMin, poison = 0;
        uint32_t thr = 0, thr_lo = 0;
        double sclx = 0.0, scly = 1.0;
        bool tiny = false;
        bool pending = false;  // this warp's D rows hold unflushed stages
        // partial slot of the current segment (absolute: (tile, segment));
        // pre-decremented so the first segment start lands on it
        int seg_slot = static_cast<int>((static_cast<int64_t>(cp.s) * ntiles_col * TP + cp.ct * TP +
                                         (TP == 2 ? rank : 0)) * nseg + cp.kc / seg_len) - 1;
        bool seg_first = true; // its first flush stores, later ones add
        int seg_left = 0;      // stages left in the current segment (ranges start on segment starts)
        const int nch = static_cast<int>(nchunk), ntc = static_cast<int>(ntiles_col);

        // the current epoch's D rows (this warp's 16 TMEM lanes, all 8
        // accumulators) -> fp64 partial of its segment, scaled by the epoch's
        // exponent; `zero` clears them for an epoch restart inside the
        // segment (at a segment start the next MMA overwrites them instead)
        auto flush = [&](int it_last, bool final_flush, bool zero) {
            mbar_wait(&b_empty[it_last % kBStages], (it_last / kBStages) & 1);  // MMAs <= it_last done
            tc_fence_after();
            const int half = kSplit ? static_cast<int>(rank) : 0;
            tc_flush_rows<NPAD, MODE>(tmem + lane_base,
                                      p.partial + (static_cast<int64_t>(seg_slot) * kHalves + half) * (NPAD * kM),
                                      __shfl_sync(0xffffffffu, eb, lf),  // lane lf converts column lf (b = 0)
                                      __shfl_sync(0xffffffffu, poison, lf), pf, col_f, final_flush, zero, seg_first,
                                      half);
            tc_fence_before();
        };

        // 16 entries per converter thread per stage: rows [16 b, 16 b + 16) of
        // column col of this CTA's 32 rows
        constexpr int kEnt = 16;
        auto load = [&](int it, double (&xv)[kEnt]) {
            const int sa = it % kAStages;
            mbar_wait(&a_full[sa], (it / kAStages) & 1);
            // 128B-swizzled box rows: column col is 128 B (16 rows) per box
            const uint32_t cb = a_s + sa * kAStageBytes + b * kBoxBytes + col * 128;
#pragma unroll
            for (int j = 0; j < kEnt / 2; ++j) {
                const double2 v = lds128(cb + ((j ^ (col & 7)) << 4));
                xv[2 * j] = v.x;
                xv[2 * j + 1] = v.y;
            }
        };
        // column max |x| high word over both row halves (split: over this
        // CTA's 16 rows, published to the peer); using it also completes the
        // loads, so the A slot goes back to the TMA refill
        auto col_max = [&](int it, const double (&xv)[kEnt]) {
            uint32_t mx = 0;
#pragma unroll
            for (int e = 0; e < kEnt; ++e) mx = max(mx, static_cast<uint32_t>(__double2hiint(xv[e])) & 0x7fffffffu);
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
            if constexpr (kSplit) {
                if (b == 0) {
                    const int sa = it % kAStages;
                    st_async_b32(mbox_s + (sa * kM + col) * 4 + poff, mx, smem_u32(&m_full[sa]) + poff);
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&a_empty[it % kAStages]);
            return mx;
        };
        // split: the whole column's maximum = max(ours, the peer's), read
        // a stage after it was published
        auto peer_max = [&](int it, uint32_t mx) -> uint32_t {
            if constexpr (kSplit) {
                const int sa = it % kAStages;
                mbar_wait(&m_full[sa], (it / kAStages) & 1);
                uint32_t pm;
                asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(pm) : "r"(mbox_s + (sa * kM + col) * 4));
                // re-arm the slot for stage it + kAStages once this phase is
                // complete (this thread just saw it complete); the peer writes
                // that stage's maxima only a few stages later (B-ring lock-step)
                if (warp == 8 && lane == 0) mbar_arrive_expect_tx(&m_full[sa], kM * 4);
                return max(mx, pm);
            } else {
                return mx;
            }
        };

        auto step = [&](int it, const double (&xc)[kEnt], uint32_t mx, double (&xn)[kEnt]) -> uint32_t {
            const int sb = it % kBStages;
            const bool new_seg = seg_left == 0;
            mx = peer_max(it, mx);
            if (__any_sync(0xffffffffu, new_seg || mx >= thr || mx < thr_lo)) {  // warp-uniform, rare
                const bool over = __any_sync(0xffffffffu, mx >= thr);
                if (pending) {
                    // a new segment closes the old one (final: poison -> NaN);
                    // otherwise the rows restart an exponent epoch in the
                    // segment and are zeroed (the MMAs keep accumulating)
                    if (lane == 0) atomicAdd(&g_tc_flushes[new_seg ? 0 : over ? 1 : 2], 1ull);
                    flush(it - 1, new_seg, !new_seg);
                }
                if (new_seg) {
                    // tiles follow each other in the flat order, each nseg slots
                    // wide; a pair's CTAs skip their peer's tile
                    seg_slot += (cp.kc == 0 && pending) ? 1 + (TP - 1) * static_cast<int>(nseg) : 1;
                    seg_first = true;
                    poison = 0;
                    seg_left = min(static_cast<int>(seg_len), nch - cp.kc);
                } else if (pending) {
                    seg_first = false;
                }
                if (mx >= 0x7ff00000u) poison = 1;
                eb = column_eb(mx);
                // |x| < 2^(E+1) keeps |v| < 2^51: u = v + kOffset stays a 7-byte integer
                thr = poison ? 0xffffffffu : (eb >= 2046 ? 0x7ff00000u : static_cast<uint32_t>(eb + 1) << 20);
                const int elo = eb - 1 - kHeadroom - kFallback;
                thr_lo = poison || elo <= 0 ? 0u : static_cast<uint32_t>(elo) << 20;
                const double2 sc2 = fix_scale(eb);
                sclx = sc2.x;
                scly = sc2.y;
                tiny = __any_sync(0xffffffffu, scly != 1.0);
            }
            --seg_left;
            const bool more = it + 1 < niter;
            uint32_t mxn = 0;
            if (more) {
                load(it + 1, xn);
                if constexpr (kSplit) mxn = col_max(it + 1, xn);  // published a stage ahead of use
            }
            // one DFMA per entry -- t = RN(x 2^(P-E) + 1.5 2^52), whose low 56
            // bits are u = rint(x 2^(P-E)) + kOffset -- then 4x4 PRMT byte
            // transposes and one 16-byte store per slice (K half b, row col;
            // split: of K block rank).
            // The rare two-factor scale (tiny columns) is a separate copy of
            // the whole emit path, so the hot path has no register joins.
            const uint32_t st = b_s + sb * Cfg::kBStageBytes + (kSplit ? rank * kSliceBytes : 0) + b * (kM * 16) +
                                col * 16;
            auto emit = [&](auto two_factor) {
                uint32_t lw[kEnt], hw[kEnt];
#pragma unroll
                for (int e = 0; e < kEnt; ++e) {
                    const double t = decltype(two_factor)::value ? fma(xc[e] * sclx, scly, kMagic)
                                                                 : fma(xc[e], sclx, kMagic);
                    hw[e] = static_cast<uint32_t>(__double2hiint(t));
                    lw[e] = static_cast<uint32_t>(__double2loint(t));
                }
                uint32_t sw[kSlices][kEnt / 4];
#pragma unroll
                for (int g4 = 0; g4 < kEnt / 4; ++g4) {
                    const uint32_t* wl = lw + 4 * g4;
                    const uint32_t* wh = hw + 4 * g4;
                    {
                        const uint32_t t0 = __byte_perm(wl[0], wl[1], 0x5140), t1 = __byte_perm(wl[0], wl[1], 0x7362);
                        const uint32_t t2 = __byte_perm(wl[2], wl[3], 0x5140), t3 = __byte_perm(wl[2], wl[3], 0x7362);
                        sw[0][g4] = __byte_perm(t0, t2, 0x5410);
                        sw[1][g4] = __byte_perm(t0, t2, 0x7632);
                        sw[2][g4] = __byte_perm(t1, t3, 0x5410);
                        sw[3][g4] = __byte_perm(t1, t3, 0x7632);
                    }
                    {
                        const uint32_t t0 = __byte_perm(wh[0], wh[1], 0x5140), t1 = __byte_perm(wh[0], wh[1], 0x7362);
                        const uint32_t t2 = __byte_perm(wh[2], wh[3], 0x5140), t3 = __byte_perm(wh[2], wh[3], 0x7362);
                        sw[4][g4] = __byte_perm(t0, t2, 0x5410);
                        sw[5][g4] = __byte_perm(t0, t2, 0x7632);
                        sw[6][g4] = __byte_perm(t1, t3, 0x5410);
                    }
                }
                // the slice slot is free once the MMAs that read it completed
                // (split: both CTAs' MMAs, the commits are multicast): only
                // the stores wait, the conversion runs ahead
                if (it >= kBStages) mbar_wait(&b_empty[sb], ((it / kBStages) - 1) & 1);
                if constexpr (!kSplit) {
#pragma unroll
                    for (int t = 0; t < kSlices; ++t)
                        sts128u(st + t * kTileBytes, sw[t][0], sw[t][1], sw[t][2], sw[t][3]);
                } else {
                    // CTA 0 keeps slices 0-3 (tiles 0-3), CTA 1 slices 4-6 (tiles
                    // 0-2); the other CTA's slices go to its tiles at the same
                    // offset, counted on its stage barrier
                    const uint32_t rbar = smem_u32(&b_full[sb]) + poff;
                    if (rank == 0) {
#pragma unroll
                        for (int t = 0; t < 4; ++t) sts128u(st + t * kTileBytes, sw[t][0], sw[t][1], sw[t][2], sw[t][3]);
#pragma unroll
                        for (int t = 4; t < kSlices; ++t)
                            st_async_v4(st + (t - 4) * kTileBytes + poff, sw[t][0], sw[t][1], sw[t][2], sw[t][3], rbar);
                    } else {
#pragma unroll
                        for (int t = 4; t < kSlices; ++t)
                            sts128u(st + (t - 4) * kTileBytes, sw[t][0], sw[t][1], sw[t][2], sw[t][3]);
#pragma unroll
                        for (int t = 0; t < 4; ++t)
                            st_async_v4(st + t * kTileBytes + poff, sw[t][0], sw[t][1], sw[t][2], sw[t][3], rbar);
                    }
                }
            };
            if (!tiny)
                emit(std::false_type{});
            else
                emit(std::true_type{});
            fence_proxy_async();
            __syncwarp();
            if (lane == 0) mbar_arrive(&b_full[sb]);
            pending = true;
            advance(cp, nch, ntc);
            if constexpr (kSplit)
                return mxn;
            else
                return more ? col_max(it + 1, xn) : 0u;
        };

        double xa[kEnt], xb[kEnt];
        load(0, xa);
        uint32_t mx = col_max(0, xa);
        for (int it = 0; it < niter; it += 2) {
            mx = step(it, xa, mx, xb);
            if (it + 1 < niter) mx = step(it + 1, xb, mx, xa);
        }
        // final flush: the range ends on a segment end
        flush(niter - 1, true, false);
    }
    if constexpr (kPair)
        cluster_sync_all();  // no remote store or commit may target a CTA that has exited
    else
        __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(Cfg::kTmemCols));
    }
}

template <int NPAD, int MODE>
cudaError_t launch_t(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap, cudaStream_t stream) {
    using Cfg = TcCfg<NPAD, MODE>;
    static_assert(Cfg::kSmem <= 227 * 1024, "shared memory budget");
    auto kern = sketch_tc_kernel<NPAD, MODE>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Cfg::kSmem));
    if (e != cudaSuccess) return e;
    const int64_t ntiles_u = plan.ntiles_col / (MODE == 1 ? 2 : 1);
    if constexpr (MODE != 0) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(static_cast<unsigned>(plan.grid));
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = Cfg::kSmem;
        cfg.stream = stream;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        e = cudaLaunchKernelEx(&cfg, kern, *tmap, p, plan.nchunk, ntiles_u, plan.nseg, plan.seg_len,
                               plan.total_units);
    } else {
        kern<<<plan.grid, kThreads, Cfg::kSmem, stream>>>(*tmap, p, plan.nchunk, ntiles_u, plan.nseg, plan.seg_len,
                                                          plan.total_units);
        e = cudaGetLastError();
    }
    if (e != cudaSuccess) return e;
    return launch_sketch_reduce(p, plan, stream);
}

// CTA pairs the device keeps resident at once for this kernel (0 if clusters
// of two cannot be launched); cached per (ell_pad, mode) for the process's
// device (one GPU per process; a racing first call computes the same value)
template <int NPAD, int MODE>
int max_pairs() {
    static int cached = -1;
    if (cached >= 0) return cached;
    using Cfg = TcCfg<NPAD, MODE>;
    auto kern = sketch_tc_kernel<NPAD, MODE>;
    int n = 0;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(Cfg::kSmem)) ==
        cudaSuccess) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = Cfg::kSmem;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess) n = 0;
    }
    cudaGetLastError();
    cached = n;
    return n;
}

int max_pairs_for(int ell_pad, int mode) {
    if (mode == 2) return ell_pad == 80 ? max_pairs<80, 2>() : 0;
    switch (ell_pad) {
        case 16: return max_pairs<16, 1>();
        case 32: return max_pairs<32, 1>();
        case 48: return max_pairs<48, 1>();
        case 64: return max_pairs<64, 1>();
        default: return 0;
    }
}

}  // namespace

int sketch_tc_flush_counters(int64_t* out, bool reset) {
    unsigned long long v[3] = {0, 0, 0};
    if (cudaMemcpyFromSymbol(v, g_tc_flushes, sizeof v) != cudaSuccess) return 1;
    for (int i = 0; i < 3; ++i) out[i] = static_cast<int64_t>(v[i]);
    if (reset) {
        const unsigned long long z[3] = {0, 0, 0};
        if (cudaMemcpyToSymbol(g_tc_flushes, z, sizeof z) != cudaSuccess) return 1;
    }
    return 0;
}

bool sketch_tc_make_plan(int64_t m, int64_t n, int64_t batch, int64_t ell, int num_sms, int pair_mode,
                         int64_t seg_rows, SketchPlan* plan) {
    if (m < 1 || n < 1 || batch < 1 || ell < 1 || ell > kSketchTcMaxEll) return false;
    plan->ell_pad = static_cast<int>(16 * ((ell + 15) / 16));
    plan->mt = plan->ell_pad / 16;
    plan->nw = 1;
    plan->nt = kM;
    plan->ntiles_col = (n + kM - 1) / kM;
    plan->kc_rows = kRows;  // set per mode below
    // ell_pad 80: the slice-split pair (mode 2), the only mode whose TMEM
    // fits 80 columns per accumulator; without clusters the caller splits
    // the sketch into passes of <= 64 rows instead.
    // Otherwise CTA pairs (mode 1) when the column tiles pair up and the
    // device keeps at least as many pairs resident as half the SM budget
    // (clusters of two span a TPC), only with pair_mode 2 (tests, A/B): since
    // the MMA warp issues through elect.sync, one CTA per tile is as fast or
    // faster at every width (config-3 batch, same-process A/B: ell 64 4.36 vs
    // 4.47 ms, 48 3.69 vs 3.87, 32 3.65 vs 3.87 -- the pair's lock-step costs
    // more than halving the Omega work saves). pair_mode 0 and 1 (default)
    // never pair.
    int pairs = 0;
    if (plan->ell_pad == 80) {
        pairs = num_sms >= 2 ? max_pairs_for(80, 2) : 0;
        if (pairs == 0) return false;
        plan->pair = 2;
    } else {
        const bool want = pair_mode == 2;
        pairs = want && num_sms >= 2 && plan->ntiles_col % 2 == 0 ? max_pairs_for(plan->ell_pad, 1) : 0;
        plan->pair = pairs > 0 && 2 * pairs >= num_sms - 1 ? 1 : 0;
    }
    const int P = plan->pair ? 2 : 1;
    const int TP = plan->pair == 1 ? 2 : 1;
    plan->kc_rows = plan->pair == 2 ? 2 * kRows : kRows;  // split stages: 64 rows, 32 per CTA
    plan->nchunk = (m + plan->kc_rows - 1) / plan->kc_rows;
    plan->halves = plan->pair == 2 ? 2 : 1;
    // split pairs own twice the work per unit of time: twice longer segments
    // keep the same balance with half the partial traffic
    plan->seg_len = (seg_rows > 0 ? seg_rows : plan->pair == 2 ? 2 * kSketchSegRows : kSketchSegRows) / plan->kc_rows;
    plan->nseg = (plan->nchunk + plan->seg_len - 1) / plan->seg_len;
    plan->total_units = batch * (plan->ntiles_col / TP) * plan->nseg;
    int64_t owners = plan->pair ? std::min<int64_t>(pairs, num_sms / 2) : num_sms;
    if (owners > plan->total_units) owners = plan->total_units;
    plan->grid = static_cast<int>(owners * P);
    plan->smem = 0;
    plan->partial_elems =
        static_cast<size_t>(batch) * plan->ntiles_col * plan->nseg * plan->halves * plan->ell_pad * plan->nt;
    return true;
}

cudaError_t launch_sketch_tc(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap,
                             cudaStream_t stream) {
    if (p.omega_mode != 1) return cudaErrorInvalidValue;
    if (plan.pair == 2) return plan.ell_pad == 80 ? launch_t<80, 2>(p, plan, tmap, stream) : cudaErrorInvalidValue;
    if (plan.pair == 1) {
        switch (plan.ell_pad) {
            case 16: return launch_t<16, 1>(p, plan, tmap, stream);
            case 32: return launch_t<32, 1>(p, plan, tmap, stream);
            case 48: return launch_t<48, 1>(p, plan, tmap, stream);
            case 64: return launch_t<64, 1>(p, plan, tmap, stream);
            default: return cudaErrorInvalidValue;
        }
    }
    switch (plan.ell_pad) {
        case 16: return launch_t<16, 0>(p, plan, tmap, stream);
        case 32: return launch_t<32, 0>(p, plan, tmap, stream);
        case 48: return launch_t<48, 0>(p, plan, tmap, stream);
        case 64: return launch_t<64, 0>(p, plan, tmap, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace spidgpu
