// sketch_i8.cu -- the performance-mode sketch Y_s = Omega_s * A_s as an EXACT
// integer-sliced contraction on the register-fed int8 tensor path
// (mma.sync m16n8k32, SASS IMMA.16832). The default kernel for this sketch is
// sketch_tc.cu (tcgen05 + TMEM); this one is selected with
// SPIDGPU_OPT_IMMA_SKETCH and kept for A/B measurement and tests.
//
// Same reference role as sketch.cu (the north star's Gaussian sketch in place
// of subsample/subsample_column, proj/src/grid.cpp:136-150; CPU restatement
// matmul(Omega, A), proj/src/dense_matrix.cpp:38-53), for the Philox Omega.
//
// The performance-mode Omega is integer-valued (Omega = Q/32, |Q| <= 117, see
// philox.cuh), so Omega * A is formed from exact integer products:
//   * every column c of A gets a per-period exponent E_c (the largest
//     exponent of its first 64 rows in the period + 4 bits of headroom), and
//     each entry becomes the fixed-point integer v = floor(x 2^(54-E_c)),
//     formed on the FP64 pipe without F2I: t = RD(y + 1.5*2^84) holds
//     floor(y / 2^32) in its low word, and RD((y - (t - 1.5*2^84)) + 2^52)
//     holds the low 32 bits;
//   * v is split into 7 byte slices (0..5 unsigned, 6 signed) by a PRMT byte
//     transpose that lands directly in the IMMA B-fragment layout;
//   * each slice is contracted with Q on IMMA.16832 (s8 x u8 -> s32): exact,
//     and |sum| < 2^31 for up to 65536 rows, so the int32 accumulators are
//     flushed to fp64 every 2048 k-steps: Y += 2^(E_c - 59) sum_t 2^(8t) D_t
//     (two exact int64 partial sums);
//   * a later entry with |x| >= 2^E_c (headroom exceeded) makes its warp flush
//     and re-derive the exponents (warp-uniform slow path); a non-finite entry
//     poisons its column to NaN, so the CPQR still raises NonFiniteInput.
//
// The IMMA issue rate (8 cycles per m16n8k32 per SMSP, profiles/
// r01_int8_peak.txt) bounds this variant at ~4.3 ms per config-3 step (76%
// of HBM); the tcgen05 kernel lifts that bound.
//
// Layout (B200): persistent grid, one CTA per SM, stream-K over
// (subdomain, 64-column tile, 64-row chunk) exactly like sketch.cu; 8
// consumer warps (n8 columns each, all ell rows, 224 registers via
// setmaxnreg) + 4 producer warps (TMA of the A chunk as four 16x64 boxes
// with 128B swizzle, Philox + quantile table lookups writing Omega straight
// into the IMMA A-fragment layout). Shared loads of A are conflict-free:
// lane (g, q) reads 16B chunk q + 4((g&1)^i) of column g, whose swizzled
// positions are distinct within each quarter-warp. Partials go to the same
// [cta][seg][ell_pad][nt] workspace and fixed-order reduction as sketch.cu,
// so Y is bitwise reproducible run to run.
#include <math.h>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace spidgpu {

namespace {

constexpr int kConsumers = 8;
constexpr int kProducers = 4;
constexpr int kThreads = (kConsumers + kProducers) * kWarp;
// register split (setmaxnreg; launch budget 384 x 168): producers 56, consumers 224
constexpr int kProducerRegs = 56;
constexpr int kConsumerRegs = 224;
static_assert(kProducers * kProducerRegs + kConsumers * kConsumerRegs <= (kProducers + kConsumers) * 168,
              "register split exceeds the launch allocation");
constexpr int kBoxRows = 16;          // 128 B swizzle span of fp64 rows
constexpr int kPeriodSteps = 2048;    // 65536 rows: 65536 * 117 * 255 < 2^31
constexpr int kHeadroom = 4;          // exponent bits above the period's first stage
constexpr int kEbMin = 9;             // biased exponent floor (all-zero columns)
constexpr int kStageBudget = 200 * 1024;

template <int MT, int NW, int J, int T>
struct I8Cfg {
    static_assert(NW == 1, "one n8 tile per consumer warp");
    static constexpr int kEllPad = 16 * MT;
    static constexpr int kNt = 8 * NW * kConsumers;
    static constexpr int kBoxBytes = kBoxRows * kNt * 8;
    static constexpr int kRows = 32 * J;  // rows of A per stage
    static constexpr int kABytes = 2 * J * kBoxBytes;
    static constexpr int kOBytes = J * MT * 512;
    static constexpr int kStageBytes = kABytes + kOBytes;
    static constexpr int kStages = (kStageBudget / kStageBytes) < 8 ? (kStageBudget / kStageBytes) : 8;
    static constexpr int kP = 8 * T - 2;  // |v| <= 2^kP < 2^(8T-1)
    static constexpr size_t kSmem =
        1024 + static_cast<size_t>(kStages) * kStageBytes + 4096 + 3 * 8 * kStages;
};

struct ChunkPos {
    int64_t s, ct, kc;
};

__device__ __forceinline__ ChunkPos chunk_pos(int64_t g, int64_t nchunk, int64_t ntiles_col) {
    const int64_t tile = g / nchunk;
    return ChunkPos{tile / ntiles_col, tile % ntiles_col, g % nchunk};
}

__device__ __forceinline__ void sts32(uint32_t addr, uint32_t v) {
    asm volatile("st.shared.u32 [%0], %1;\n" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ uint4 lds128u(uint32_t addr) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(addr));
    return v;
}

// D += A(16x32 s8, Omega) * B(32x8, one A slice; u8, or s8 for the top slice)
template <bool SIGNED_B>
__device__ __forceinline__ void imma(int (&d)[4], const uint4& a, uint32_t b0, uint32_t b1) {
    if constexpr (SIGNED_B)
        asm("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};\n"
            : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
            : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
    else
        asm("mma.sync.aligned.m16n8k32.row.col.s32.s8.u8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
            "{%8,%9}, {%0,%1,%2,%3};\n"
            : "+r"(d[0]), "+r"(d[1]), "+r"(d[2]), "+r"(d[3])
            : "r"(a.x), "r"(a.y), "r"(a.z), "r"(a.w), "r"(b0), "r"(b1));
}

// Biased exponent for a column whose largest |entry| has high word `mg`.
__device__ __forceinline__ int column_eb(uint32_t mg) {
    int eb = static_cast<int>(mg >> 20) + 1 + kHeadroom;
    return eb < kEbMin ? kEbMin : (eb > 2047 ? 2047 : eb);
}

// 2^(P - E) as a product of two normal doubles (E can be as small as
// 9 - 1023 for tiny or all-zero columns, so the total can exceed 2^1023)
template <int P>
__device__ __forceinline__ double2 fix_scale(int eb) {
    const int d = P + 1023 - eb;  // unbiased exponent of the total scale
    const int d1 = d > 1000 ? 1000 : d;
    return make_double2(__longlong_as_double(static_cast<long long>(d1 + 1023) << 52),
                        __longlong_as_double(static_cast<long long>(d - d1 + 1023) << 52));
}

// 2^(E - P) / 32, likewise split (the total can fall below 2^-1022)
template <int P>
__device__ __forceinline__ double2 unfix_scale(int eb) {
    const int e = eb - 1023 - P - kOmegaScaleLog2;
    const int e1 = e < -1000 ? -1000 : e;
    return make_double2(__longlong_as_double(static_cast<long long>(e1 + 1023) << 52),
                        __longlong_as_double(static_cast<long long>(e - e1 + 1023) << 52));
}

template <int MT, int NW, int J, int T>
__global__ void __launch_bounds__(kThreads, 1)
    sketch_i8_kernel(const __grid_constant__ CUtensorMap tmap, SketchParams p, int64_t nchunk,
                     int64_t ntiles_col, int64_t total_chunks, int max_segs) {
    using Cfg = I8Cfg<MT, NW, J, T>;
    constexpr int S = Cfg::kStages;
    constexpr int P = Cfg::kP;
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw_s = smem_u32(smem_raw);
    const uint32_t base_s = (raw_s + 1023u) & ~1023u;
    unsigned char* base = smem_raw + (base_s - raw_s);
    const uint32_t a_s = base_s;
    const uint32_t o_s = base_s + S * Cfg::kABytes;
    int8_t* tab = reinterpret_cast<int8_t*>(base + S * Cfg::kStageBytes);
    uint64_t* full_a = reinterpret_cast<uint64_t*>(base + S * Cfg::kStageBytes + 4096);
    uint64_t* full_o = full_a + S;
    uint64_t* empty = full_o + S;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int64_t G = gridDim.x, c = blockIdx.x;
    const int64_t lo = (c * total_chunks) / G, hi = ((c + 1) * total_chunks) / G;
    const int64_t niter = hi - lo;
    if (niter <= 0) return;

    for (int i = tid; i < 1024; i += kThreads)
        reinterpret_cast<int*>(tab)[i] = reinterpret_cast<const int*>(kOmegaQ)[i];
    if (tid == 0) {
        prefetch_tmap(&tmap);
        for (int i = 0; i < S; ++i) {
            mbar_init(&full_a[i], 1);
            mbar_init(&full_o[i], kProducers * kWarp);
            mbar_init(&empty[i], kConsumers);
        }
        fence_barrier_init();
    }
    __syncthreads();

    if (warp >= kConsumers) {
        // ------------------------------ producers ------------------------------
        asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(kProducerRegs));
        const int pt = tid - kConsumers * kWarp;  // 0..127
        ChunkPos cp = chunk_pos(lo, nchunk, ntiles_col);
        int slot = 0;
        uint32_t epar = 0;
        for (int64_t it = 0; it < niter; ++it) {
            if (it >= S) mbar_wait(&empty[slot], epar);
            if (pt == 0) {
                mbar_arrive_expect_tx(&full_a[slot], Cfg::kABytes);
#pragma unroll
                for (int b = 0; b < 2 * J; ++b)
                    tma_load_3d(base + slot * Cfg::kABytes + b * Cfg::kBoxBytes, &tmap, &full_a[slot],
                                static_cast<int>(cp.kc * Cfg::kRows + kBoxRows * b),
                                static_cast<int>(cp.ct * Cfg::kNt), static_cast<int>(cp.s));
            }
            const uint32_t ob = o_s + slot * Cfg::kOBytes;
            for (int task = pt; task < Cfg::kEllPad * J; task += kProducers * kWarp) {
                const int r = task % Cfg::kEllPad, j = task / Cfg::kEllPad;
                // IMMA A fragment of m-tile r/16: lane (g, t) register (r%16 >= 8) + 2h
                // holds physical rows {2t, 2t+1} of octets 2h and 2h+1
                const int mt = r >> 4, gr = r & 15, g = gr & 7, h8 = gr >> 3;
                const uint32_t fb = ob + (j * MT + mt) * 512 + g * 64 + h8 * 4;
                const uint32_t ko = static_cast<uint32_t>((cp.kc * Cfg::kRows + 32 * j) >> 3);
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    int q0[8], q1[8];
                    if (r < p.ell) {
                        omega_q8(p.seed, static_cast<uint64_t>(p.sub_base + cp.s),
                                 static_cast<uint32_t>(p.row0 + r), ko + 2 * h, tab, q0);
                        omega_q8(p.seed, static_cast<uint64_t>(p.sub_base + cp.s),
                                 static_cast<uint32_t>(p.row0 + r), ko + 2 * h + 1, tab, q1);
                    } else {
#pragma unroll
                        for (int e = 0; e < 8; ++e) q0[e] = q1[e] = 0;
                    }
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const uint32_t w = (q0[2 * t] & 0xff) | ((q0[2 * t + 1] & 0xff) << 8) |
                                           ((q1[2 * t] & 0xff) << 16) |
                                           (static_cast<uint32_t>(q1[2 * t + 1] & 0xff) << 24);
                        sts32(fb + t * 16 + h * 8, w);
                    }
                }
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
                if (it + 1 >= 2 * S) epar ^= 1u;
            }
        }
        return;
    }

    // ------------------------------- consumers -------------------------------
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(kConsumerRegs));
    // warp w owns columns [8w, 8w+8) of the tile, all ell rows and all 8 byte
    // slices; one stage (J k-steps) is converted as a whole, so the J k-steps'
    // conversions and IMMAs are independent instruction streams
    const int g = lane >> 2, tq = lane & 3;
    const int col0 = warp * 8;
    // chunk offsets of the two 16B loads per box (see header): conflict-free order
    const uint32_t ch0 = static_cast<uint32_t>(((tq + 4 * (g & 1)) ^ g) << 4);
    const uint32_t ch1 = static_cast<uint32_t>(((tq + 4 * ((g & 1) ^ 1)) ^ g) << 4);
    // odd g loads the row pairs in swapped order; the final PRMT puts them back
    const uint32_t selA = (g & 1) ? 0x1054u : 0x5410u;
    const uint32_t selB = (g & 1) ? 0x3276u : 0x7632u;

    int D[T][MT][4];
#pragma unroll
    for (int t = 0; t < T; ++t)
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) D[t][mt][0] = D[t][mt][1] = D[t][mt][2] = D[t][mt][3] = 0;

    int eb = kEbMin;       // biased exponent of this lane's B column (g)
    uint32_t thr = 0;      // overflow threshold on |x|'s high word
    double2 scl = make_double2(0.0, 0.0);  // 2^(P - E) = .x * .y
    int poison = 0;        // column saw a non-finite entry
    bool tiny = false;     // some column of the warp needs the two-factor scale
    bool fresh = true;     // next stage starts a period (exponents to derive)
    bool first = true;     // next flush of this segment overwrites the partial
    int psteps = 0;
    int seg = 0, slot = 0;
    uint32_t par = 0;
    int kc = static_cast<int>(lo % nchunk);
    const int nch = static_cast<int>(nchunk);

    auto set_exponent = [&](uint32_t mx) {
        uint32_t mg = max(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
        mg = max(mg, __shfl_xor_sync(0xffffffffu, mg, 2));
        if (mg >= 0x7ff00000u) poison = 1;
        eb = column_eb(mg);
        thr = poison ? 0xffffffffu : (eb >= 2047 ? 0x7ff00000u : static_cast<uint32_t>(eb) << 20);
        scl = fix_scale<P>(eb);
        tiny = __any_sync(0xffffffffu, scl.y != 1.0);
    };

    auto flush = [&](bool final_flush) {
        double* part = p.partial + (static_cast<size_t>(c) * max_segs + seg) *
                                       (static_cast<size_t>(Cfg::kEllPad) * Cfg::kNt);
        const int eb0 = __shfl_sync(0xffffffffu, eb, 8 * tq);
        const int eb1 = __shfl_sync(0xffffffffu, eb, 8 * tq + 4);
        const int ps0 = __shfl_sync(0xffffffffu, poison, 8 * tq);
        const int ps1 = __shfl_sync(0xffffffffu, poison, 8 * tq + 4);
        const double2 u0 = unfix_scale<P>(eb0), u1 = unfix_scale<P>(eb1);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
                double val[2];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int r = 2 * hh + e;
                    long long lo64 = 0, hi64 = 0;  // |.| < 2^31 * 2^25: exact
#pragma unroll
                    for (int t = 0; t < 4 && t < T; ++t)
                        lo64 += static_cast<long long>(D[t][mt][r]) * (1LL << (8 * t));
#pragma unroll
                    for (int t = 4; t < T; ++t)
                        hi64 += static_cast<long long>(D[t][mt][r]) * (1LL << (8 * (t - 4)));
#pragma unroll
                    for (int t = 0; t < T; ++t) D[t][mt][r] = 0;
                    const double2 u = e ? u1 : u0;
                    val[e] = fma(static_cast<double>(hi64), 4294967296.0, static_cast<double>(lo64)) * u.x * u.y;
                }
                if (final_flush) {
                    if (ps0) val[0] = __longlong_as_double(0x7ff8000000000000LL);
                    if (ps1) val[1] = __longlong_as_double(0x7ff8000000000000LL);
                }
                const int row = mt * 16 + g + 8 * hh;
                double2* dst = reinterpret_cast<double2*>(part + row * Cfg::kNt + col0 + 2 * tq);
                if (first) {
                    *dst = make_double2(val[0], val[1]);
                } else {
                    const double2 o = *dst;
                    *dst = make_double2(o.x + val[0], o.y + val[1]);
                }
            }
        first = false;
    };

    for (int it = 0; it < static_cast<int>(niter); ++it) {
        mbar_wait(&full_a[slot], par);
        const uint32_t at = a_s + slot * Cfg::kABytes;
        const uint32_t ot = o_s + slot * Cfg::kOBytes;
        double x[J][8];
#pragma unroll
        for (int j = 0; j < J; ++j) {
            const uint32_t cb = at + (2 * j) * Cfg::kBoxBytes + (col0 + g) * 128;
            const double2 x01 = lds128(cb + ch0), x23 = lds128(cb + ch1);
            const double2 x45 = lds128(cb + Cfg::kBoxBytes + ch0);
            const double2 x67 = lds128(cb + Cfg::kBoxBytes + ch1);
            x[j][0] = x01.x, x[j][1] = x01.y, x[j][2] = x23.x, x[j][3] = x23.y;
            x[j][4] = x45.x, x[j][5] = x45.y, x[j][6] = x67.x, x[j][7] = x67.y;
        }
        uint32_t mx = 0;
#pragma unroll
        for (int j = 0; j < J; ++j)
#pragma unroll
            for (int e = 0; e < 8; ++e) mx = max(mx, static_cast<uint32_t>(__double2hiint(x[j][e])) & 0x7fffffffu);
        if (fresh) set_exponent(mx);  // warp-uniform
        if (__any_sync(0xffffffffu, mx >= thr)) {
            // headroom exceeded (or a non-finite entry): flush with the old
            // exponents, then re-derive them from this stage
            flush(false);
            set_exponent(mx);
            psteps = 0;
        }
        // fixed point v = floor(x 2^(P-E)) as 64-bit (lo, hi) words, on the
        // idle FP64 pipe rather than F2I (XU): t = RD(y + 1.5*2^84) holds
        // floor(y / 2^32) in its low word; r = RD(y - (t - 1.5*2^84)) lies in
        // [0, 2^32) with floor(r) exact; RD(r + 2^52) holds floor(r) in its
        // low word (y = x 2^(P-E) is formed exactly inside the FMAs)
        uint32_t lw[J][8], hw[J][8];
        if (!tiny) {
            constexpr double kMagHi = 1.5 * 19342813113834066795298816.0;  // 1.5 * 2^84
            constexpr double kMagLo = 4503599627370496.0;                    // 2^52
#pragma unroll
            for (int j = 0; j < J; ++j)
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const double t = __fma_rd(x[j][e], scl.x, kMagHi);
                    // RD keeps r < 2^32 when y - h is inexact (tiny negative y)
                    const double r = __fma_rd(x[j][e], scl.x, -(t - kMagHi));
                    const double u = __dadd_rd(r, kMagLo);
                    hw[j][e] = static_cast<uint32_t>(__double2loint(t));
                    lw[j][e] = static_cast<uint32_t>(__double2loint(u));
                }
        } else {
#pragma unroll
            for (int j = 0; j < J; ++j)
#pragma unroll
                for (int e = 0; e < 8; ++e) {
                    const long long v = __double2ll_rd(x[j][e] * scl.x * scl.y);
                    lw[j][e] = static_cast<uint32_t>(v);
                    hw[j][e] = static_cast<uint32_t>(static_cast<unsigned long long>(v) >> 32);
                }
        }
        mbar_wait(&full_o[slot], par);
#pragma unroll
        for (int j = 0; j < J; ++j) {
            uint4 af[MT];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) af[mt] = lds128u(ot + ((j * MT + mt) * 32 + lane) * 16);
#pragma unroll
            for (int hf = 0; hf < 2; ++hf) {
                const uint32_t* w = hf ? hw[j] : lw[j];
                // byte transpose: slice t of rows (x0..x3) -> b0, (x4..x7) -> b1
                uint32_t bs[4][2];
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const uint32_t t0 = __byte_perm(w[4 * b + 0], w[4 * b + 1], 0x5140);
                    const uint32_t t1 = __byte_perm(w[4 * b + 0], w[4 * b + 1], 0x7362);
                    const uint32_t t2 = __byte_perm(w[4 * b + 2], w[4 * b + 3], 0x5140);
                    const uint32_t t3 = __byte_perm(w[4 * b + 2], w[4 * b + 3], 0x7362);
                    bs[0][b] = __byte_perm(t0, t2, selA);
                    bs[1][b] = __byte_perm(t0, t2, selB);
                    bs[2][b] = __byte_perm(t1, t3, selA);
                    bs[3][b] = __byte_perm(t1, t3, selB);
                }
#pragma unroll
                for (int tt = 0; tt < 4; ++tt) {
                    const int t = 4 * hf + tt;
                    if (t < T) {
#pragma unroll
                        for (int mt = 0; mt < MT; ++mt) {
                            if (t == T - 1)
                                imma<true>(D[t][mt], af[mt], bs[tt][0], bs[tt][1]);
                            else
                                imma<false>(D[t][mt], af[mt], bs[tt][0], bs[tt][1]);
                        }
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (++slot == S) {
            slot = 0;
            par ^= 1u;
        }
        fresh = false;
        psteps += J;
        if (++kc == nch || it + 1 == static_cast<int>(niter)) {  // tile boundary: final flush
            kc = 0;
            flush(true);
            poison = 0;
            ++seg;
            first = true;
            fresh = true;
            psteps = 0;
        } else if (psteps >= kPeriodSteps) {
            flush(false);
            psteps = 0;
            fresh = true;
        }
    }
}

template <int MT, int NW, int J, int T>
cudaError_t launch_t(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap,
                     cudaStream_t stream) {
    using Cfg = I8Cfg<MT, NW, J, T>;
    auto kern = sketch_i8_kernel<MT, NW, J, T>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(Cfg::kSmem));
    if (e != cudaSuccess) return e;
    kern<<<plan.grid, kThreads, Cfg::kSmem, stream>>>(*tmap, p, plan.nchunk, plan.ntiles_col,
                                                      plan.total_chunks, plan.max_segs);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_sketch_reduce(p, plan, stream);
}

}  // namespace

bool sketch_i8_make_plan(int64_t m, int64_t n, int64_t batch, int64_t ell, int num_sms,
                         SketchPlan* plan) {
    if (m < 1 || n < 1 || batch < 1 || ell < 1 || ell > kSketchI8MaxEll) return false;
    int mt, nw, j;
    if (ell <= 16) {
        mt = 1, nw = 1, j = 2;
    } else if (ell <= 32) {
        mt = 2, nw = 1, j = 2;
    } else {
        mt = 3, nw = 1, j = 2;
    }
    plan->ell_pad = 16 * mt;
    plan->mt = mt;
    plan->nw = nw;
    plan->nt = 8 * nw * kConsumers;
    plan->ntiles_col = (n + plan->nt - 1) / plan->nt;
    plan->kc_rows = 32 * j;
    plan->nchunk = (m + plan->kc_rows - 1) / plan->kc_rows;
    plan->total_chunks = batch * plan->ntiles_col * plan->nchunk;
    int64_t grid = num_sms;
    if (grid > plan->total_chunks) grid = plan->total_chunks;
    plan->grid = static_cast<int>(grid);
    const int64_t per = (plan->total_chunks + grid - 1) / grid;
    plan->max_segs = static_cast<int>(per / plan->nchunk + 2);
    plan->smem = 0;
    plan->partial_elems = static_cast<size_t>(grid) * plan->max_segs * plan->ell_pad * plan->nt;
    return true;
}

cudaError_t launch_sketch_i8(const SketchParams& p, const SketchPlan& plan, const CUtensorMap* tmap,
                             cudaStream_t stream) {
    if (p.omega_mode != 1) return cudaErrorInvalidValue;
    switch (plan.mt) {
        case 1: return launch_t<1, 1, 2, 7>(p, plan, tmap, stream);
        case 2: return launch_t<2, 1, 2, 7>(p, plan, tmap, stream);
        case 3: return launch_t<3, 1, 2, 7>(p, plan, tmap, stream);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace spidgpu
