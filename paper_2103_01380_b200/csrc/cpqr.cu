// cpqr.cu -- batched column ID of small sketches: greedy column-pivoted
// 2-pass MGS QR + coefficient solve, one subdomain per CTA.
//
// Restates, per subdomain, the reference chain
//   column_id (proj/src/id.cpp:40-45) -> pivoted_mgs_qr / qr_core
//   (proj/src/qr.cpp:18-124) -> build_coeffs (id.cpp:9-28) ->
//   solve_upper_triangular (qr.cpp:128-151)
// with the SAME floating-point operation sequence: every per-column dot
// product / norm is a sequential left-to-right sum of separately rounded
// products (one thread per column, __dmul_rn/__dadd_rn, no FMA), so given
// the same input sketch the pivots, R, C and residual are bit-identical to
// the reference. Parallelism comes from the columns (one thread each) and
// from the batch (one CTA per subdomain); the pivot argmax is a warp-shuffle
// + shared-memory reduction over the total order (norm desc, original index
// asc) of qr.cpp:68, which any reduction tree resolves identically.
//
// Layout: the sketch is transposed into shared memory as W[i][j] (row i
// contiguous over columns) so that a warp's 32 column-threads read 32
// consecutive doubles per row -- conflict-free. Columns are never physically
// swapped: perm[pos] / posof[col] carry the reference's position bookkeeping
// (qr.cpp:83-87) and R is keyed by original column.
//
// Three placements of W (template kMode):
//   0  W in shared memory (small inputs);
//   1  W in global memory, each column-thread loading its rows directly;
//   2  tall inputs (n <= 256): W in global memory streamed through a shared
//      ring of row chunks by TMA (a dedicated producer warp, 5 x 32 KB
//      stages): the column sweeps -- a sequential chain of DADDs per column --
//      read their operands from shared memory instead of waiting on global
//      loads. Mode 1 measured ~29 GB/s per SM on 4096 x 256 (memory-latency
//      bound); the operation sequence is the same in all three modes.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace spidgpu {

namespace {

constexpr int kCpqrThreads = 256;
constexpr double kZeroFloor = 1e-300;  // qr.cpp:11
constexpr double kCollapseRel = 1e-14; // qr.cpp:12

constexpr int kPf = 32;  // rows per prefetched chunk of the column sweeps

// mode 2: TMA ring of W row chunks
#ifndef SPIDGPU_TALL_STAGE_KB
#define SPIDGPU_TALL_STAGE_KB 32
#define SPIDGPU_TALL_STAGES 5
#endif
constexpr int kTallStageBytes = SPIDGPU_TALL_STAGE_KB * 1024;
constexpr int kTallStages = SPIDGPU_TALL_STAGES;
constexpr int kProducerWarp = kCpqrThreads / kWarp;  // the extra (9th) warp

__device__ __forceinline__ void fence_proxy_async_global() {
    asm volatile("fence.proxy.async.global;\n" ::: "memory");
}

// CTA-wide barrier of the column threads (mode 2 excludes the producer warp)
template <int kMode>
__device__ __forceinline__ void csync() {
    if constexpr (kMode == 2)
        asm volatile("bar.sync 1, %0;\n" ::"n"(kCpqrThreads) : "memory");
    else
        __syncthreads();
}
template <int kMode>
__device__ __forceinline__ int csync_or(int v) {
    if constexpr (kMode == 2) {
        int r;
        asm volatile(
            "{\n.reg .pred p, q;\nsetp.ne.s32 p, %1, 0;\nbar.red.or.pred q, 1, %2, p;\n"
            "selp.s32 %0, 1, 0, q;\n}\n"
            : "=r"(r)
            : "r"(v), "n"(kCpqrThreads)
            : "memory");
        return r;
    } else {
        return __syncthreads_or(v);
    }
}

// wv[u] = W[(i0 + u) * npad + col] for rows < `rows` (0 past the end).
__device__ __forceinline__ void load_chunk(const double* W, int npad, int col, int i0, int rows,
                                           double (&wv)[kPf]) {
#pragma unroll
    for (int u = 0; u < kPf; ++u) wv[u] = i0 + u < rows ? W[(i0 + u) * npad + col] : 0.0;
}

struct CpqrShared {
    double best_v;
    int best_i;
    int stop;
    int flag;
    int chunks;  // mode 2: row chunks the producer streams next (0 = exit)
    double max_init;
    double yfro;
};

// kNpad: W's row length as a compile-time constant (0 = runtime p.npad), so
// the tall sweeps' shared-memory addresses fold into immediate offsets
template <int kMode, int kNpad = 0>
__global__ void __launch_bounds__(kMode == 2 ? kCpqrThreads + kWarp : kCpqrThreads)
    cpqr_id_kernel(CpqrParams p, const __grid_constant__ CUtensorMap wmap, int ring_rows) {
    constexpr bool kWInShared = kMode == 0;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ CpqrShared sh;
    __shared__ double red_v[kCpqrThreads / kWarp];
    __shared__ int red_i[kCpqrThreads / kWarp];
    __shared__ uint64_t ring_full[kTallStages], ring_empty[kTallStages], go_bar;

    const int b = blockIdx.x;
    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int rows = static_cast<int>(p.rows), n = static_cast<int>(p.n);
    const int npad = kNpad ? kNpad : p.npad;

    double* W;
    double* nrm;
    double* colsq;
    int* perm;
    int* posof;
    double* diag;  // R(t,t) in selection order (step_cap)
    double* r11;   // R11 in position order, rank x rank row-major (step_cap^2)
    double* ring = nullptr;  // mode 2: kTallStages x ring_rows x npad
    {
        unsigned char* cur = smem_raw;
        if constexpr (kMode == 2) {
            // 128-byte aligned TMA destination, derived from smem_raw by an
            // integer offset so the compiler keeps the shared address space (LDS)
            cur += (128u - (smem_u32(smem_raw) & 127u)) & 127u;
            ring = reinterpret_cast<double*>(cur);
            cur += static_cast<size_t>(kTallStages) * kTallStageBytes;
        }
        if (kWInShared) {
            W = reinterpret_cast<double*>(cur);
            cur += sizeof(double) * static_cast<size_t>(rows) * npad;
        } else {
            W = p.w_ws + static_cast<size_t>(b) * rows * npad;
        }
        nrm = reinterpret_cast<double*>(cur);
        cur += sizeof(double) * n;
        colsq = reinterpret_cast<double*>(cur);
        cur += sizeof(double) * n;
        perm = reinterpret_cast<int*>(cur);
        cur += sizeof(int) * n;
        posof = reinterpret_cast<int*>(cur);
        cur += sizeof(int) * n;
        cur = smem_raw + ((cur - smem_raw + 15) & ~ptrdiff_t(15));  // stays a shared-window pointer
        diag = reinterpret_cast<double*>(cur);
        cur += sizeof(double) * p.step_cap;
        if (kWInShared) {
            r11 = reinterpret_cast<double*>(cur);
        } else {
            r11 = p.r11_ws + static_cast<size_t>(b) * p.step_cap * p.step_cap;
        }
    }
    double* R = p.r_ws + static_cast<size_t>(b) * p.step_cap * n;  // R[s][col]
    const double* Y = p.Y + static_cast<size_t>(b) * p.strideY;

    // ---- mode 2: producer warp and the ring protocol -----------------------
    // Passes are announced by thread 0 (sh.chunks, then an arrive on go_bar)
    // after a barrier that follows a proxy fence of every thread's global
    // writes, so a TMA read never overtakes the generic stores of the pass
    // before. Every consumer warp releases every chunk (ring_empty count 8).
    const int nck = kMode == 2 ? (rows + ring_rows - 1) / ring_rows : 0;
    if constexpr (kMode == 2) {
        if (tid == 0) {
            for (int i = 0; i < kTallStages; ++i) {
                mbar_init(&ring_full[i], 1);
                mbar_init(&ring_empty[i], kCpqrThreads / kWarp);
            }
            mbar_init(&go_bar, 1);
            fence_barrier_init();
        }
        __syncthreads();
        if (warp == kProducerWarp) {
            if (lane == 0) {
                prefetch_tmap(&wmap);
                const uint32_t bytes = static_cast<uint32_t>(ring_rows) * npad * sizeof(double);
                uint32_t g = 0, gophase = 0;
                for (;;) {
                    mbar_wait(&go_bar, gophase);
                    gophase ^= 1;
                    const int chunks = sh.chunks;
                    if (chunks == 0) break;
                    for (int c = 0; c < chunks; ++c, ++g) {
                        const uint32_t slot = g % kTallStages;
                        if (g >= kTallStages) mbar_wait(&ring_empty[slot], ((g / kTallStages) - 1) & 1);
                        mbar_arrive_expect_tx(&ring_full[slot], bytes);
                        tma_load_3d(ring + static_cast<size_t>(slot) * (kTallStageBytes / sizeof(double)), &wmap,
                                    &ring_full[slot], 0, (c % nck) * ring_rows, b);
                    }
                }
            }
            return;
        }
    }
    uint32_t gcons = 0;  // consumer chunk counter (same sequence as the producer's)
    // announce a pass of `passes` sweeps over W (after this thread's global writes)
    auto start_sweeps = [&](int passes) {
        if constexpr (kMode == 2) {
            fence_proxy_async_global();
            csync<kMode>();
            if (tid == 0) {
                sh.chunks = passes * nck;
                mbar_arrive(&go_bar);
            }
        }
    };
    auto stop_producer = [&]() {
        if constexpr (kMode == 2) {
            if (tid == 0) {
                sh.chunks = 0;
                mbar_arrive(&go_bar);
            }
        }
    };
    // one sweep over W's rows: body(chunk in shared memory, first row, rows)
    auto sweep = [&](auto&& body) {
        for (int c = 0; c < nck; ++c, ++gcons) {
            const uint32_t slot = gcons % kTallStages;
            mbar_wait(&ring_full[slot], (gcons / kTallStages) & 1);
            const int i0 = c * ring_rows;
            body(ring + slot * (kTallStageBytes / sizeof(double)), i0, min(ring_rows, rows - i0));
            __syncwarp();
            if (lane == 0) mbar_arrive(&ring_empty[slot]);
        }
    };

    // ---- load, transpose, finiteness (qr.cpp:34-35, id.cpp:41-42) -------
    int bad = 0;
    const int total = rows * n;
    for (int e = tid; e < total; e += kCpqrThreads) {
        const int i = e % rows, j = e / rows;
        const double v = Y[static_cast<size_t>(j) * p.ldy + i];
        bad |= !isfinite(v);
        W[i * npad + j] = v;
    }
    for (int j = tid; j < n; j += kCpqrThreads) {
        perm[j] = j;
        posof[j] = j;
    }
    bad = csync_or<kMode>(bad);
    auto finish_error = [&](int code) {
        if (tid == 0) {
            p.status[b] = code;
            p.rank[b] = 0;
            p.resid[b] = 0.0;
        }
    };
    if (bad) {
        stop_producer();
        finish_error(SPID_NON_FINITE_INPUT);
        return;
    }
    if (p.pre_status != SPID_OK) {  // batch-uniform rule failures (qr.cpp:37-38)
        stop_producer();
        finish_error(p.pre_status);
        return;
    }

    // ---- initial column norms, max_init (qr.cpp:47-51) -------------------
    double lmax = 0.0;
    if constexpr (kMode == 2) {  // n <= kCpqrThreads: at most one column per thread
        start_sweeps(1);
        const int j = tid;
        double s = 0.0;
        sweep([&](const double* ck, int, int nr) {
            if (j < n)
#pragma unroll 8
                for (int u = 0; u < nr; ++u) {
                    const double w = ck[u * npad + j];
                    s = add_rn(s, mul_rn(w, w));
                }
        });
        if (j < n) {
            const double v = sqrt(s);
            nrm[j] = v;
            colsq[j] = s;
            lmax = v;
        }
    } else {
        for (int j = tid; j < n; j += kCpqrThreads) {
            double s = 0.0;
            for (int i0 = 0; i0 < rows; i0 += kPf) {
                double wv[kPf];
                load_chunk(W, npad, j, i0, rows, wv);
#pragma unroll
                for (int u = 0; u < kPf; ++u)
                    if (i0 + u < rows) s = add_rn(s, mul_rn(wv[u], wv[u]));
            }
            const double v = sqrt(s);
            nrm[j] = v;
            colsq[j] = s;
            lmax = fmax(lmax, v);
        }
    }
    lmax = warp_max(lmax);
    if (lane == 0) red_v[warp] = lmax;
    csync<kMode>();
    if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < kCpqrThreads / kWarp; ++w) m = fmax(m, red_v[w]);
        sh.max_init = m;
        if (p.mode == RULE_BLOCKED) {
            // ||Y||_F for the blocked rule: per-column sums (in column order)
            // of sequential per-column squares -- DESIGN.md "cfg4 rule".
            double f = 0.0;
            for (int j = 0; j < n; ++j) f = add_rn(f, colsq[j]);
            sh.yfro = sqrt(f);
        }
    }
    csync<kMode>();
    const double max_init = sh.max_init;
    if (max_init < kZeroFloor) {
        stop_producer();
        finish_error(SPID_ZERO_MATRIX);
        return;
    }

    // ---- greedy pivoting loop (qr.cpp:61-106) -----------------------------
    int rank = 0;
    const int step_limit = static_cast<int>(p.step_limit);
    for (int s = 0; s < step_limit; ++s) {
        // argmax over unselected columns (positions >= s)
        double bv = -1.0;
        int bi = 0x7fffffff;
        for (int j = tid; j < n; j += kCpqrThreads) {
            if (posof[j] >= s && key_better(nrm[j], j, bv, bi)) {
                bv = nrm[j];
                bi = j;
            }
        }
        warp_argmax(bv, bi);
        if (lane == 0) {
            red_v[warp] = bv;
            red_i[warp] = bi;
        }
        csync<kMode>();
        if (tid == 0) {
            double v = red_v[0];
            int ix = red_i[0];
            for (int w = 1; w < kCpqrThreads / kWarp; ++w)
                if (key_better(red_v[w], red_i[w], v, ix)) {
                    v = red_v[w];
                    ix = red_i[w];
                }
            int stop = 0;
            if (p.mode == RULE_TOL && v <= p.tol * max_init) stop = 1;  // qr.cpp:74-76
            if (!stop && p.mode == RULE_BLOCKED && s > 0 && s % p.kstep == 0) {
                double rsq = 0.0;  // residual_fro after s steps, position order (qr.cpp:111-115)
                for (int pos = s; pos < n; ++pos) {
                    const double nj = nrm[perm[pos]];
                    rsq = add_rn(rsq, mul_rn(nj, nj));
                }
                if (sqrt(rsq) <= p.tol * sh.yfro) stop = 1;
            }
            if (!stop && v < kCollapseRel * max_init)  // qr.cpp:77-81
                stop = (p.mode == RULE_FIXED && p.strict) ? 2 : 1;
            if (!stop) {  // position swap (qr.cpp:83-87)
                const int ps = posof[ix], cs = perm[s];
                perm[s] = ix;
                perm[ps] = cs;
                posof[ix] = s;
                posof[cs] = ps;
                R[static_cast<size_t>(s) * n + ix] = v;  // R(s,s) = ||w_s|| (qr.cpp:89-90)
                diag[s] = v;
            }
            sh.best_v = v;
            sh.best_i = ix;
            sh.stop = stop;
        }
        csync<kMode>();
        if (sh.stop) {
            if (sh.stop == 2) {
                stop_producer();
                finish_error(SPID_RANK_UNREACHABLE);
                return;
            }
            break;
        }
        const int pc = sh.best_i;
        const double pn = sh.best_v;
        // q_s = w_s / R(s,s) (qr.cpp:91-92)
        // (the column's strided loads issued 8 per thread at a time, then
        // divided and stored)
        for (int i0 = 0; i0 < rows; i0 += 8 * kCpqrThreads) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * kCpqrThreads + tid;
                v[u] = i < rows ? W[i * npad + pc] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int i = i0 + u * kCpqrThreads + tid;
                if (i < rows) W[i * npad + pc] = div_rn(v[u], pn);
            }
        }
        if constexpr (kMode == 2) {
            // two-pass MGS (qr.cpp:94-102) over the TMA ring, as three read
            // sweeps of the step's W that stream back to back (nothing is
            // stored before the last): r1; then w' = w - r1 q and r2; then w'
            // recomputed from w by the same two rounded operations, w'' =
            // w' - r2 q stored and its norm. One W store per step instead of two.
            const int j = tid;
            const bool act = j < n && posof[j] > s;
            start_sweeps(3);
            double r1 = 0.0, r2 = 0.0, nn = 0.0;
            double* Wj = W + j;
            // rows of a chunk in order: whole groups of kGrp with the next
            // group's (q, w) loaded before the current group's dependent chain
            // (the last group reloads itself, branch-free), then the ragged tail
            // 16-row groups for narrow W (one or two column warps, latency-bound
            // chains: 4096 x 32 batch 3.04 -> 2.85 ms), 8 for wide (4096 x 256:
            // 15.2 vs 17.0 ms with 16)
            constexpr int kGrp = (kNpad != 0 && kNpad <= 64) ? 16 : 8;
            auto rows = [&](const double* ck, int nr, auto&& f) {
                const int nfull = nr & ~(kGrp - 1);
                if (nfull) {
                    double qa[kGrp], wa[kGrp];
#pragma unroll
                    for (int t = 0; t < kGrp; ++t) {
                        qa[t] = ck[t * npad + pc];
                        wa[t] = ck[t * npad + j];
                    }
                    for (int u0 = 0; u0 < nfull; u0 += kGrp) {
                        const int un = min(u0 + kGrp, nfull - kGrp);
                        double qb[kGrp], wb[kGrp];
#pragma unroll
                        for (int t = 0; t < kGrp; ++t) {
                            qb[t] = ck[(un + t) * npad + pc];
                            wb[t] = ck[(un + t) * npad + j];
                        }
#pragma unroll
                        for (int t = 0; t < kGrp; ++t) f(u0 + t, qa[t], wa[t]);
#pragma unroll
                        for (int t = 0; t < kGrp; ++t) {
                            qa[t] = qb[t];
                            wa[t] = wb[t];
                        }
                    }
                }
                for (int u = nfull; u < nr; ++u) f(u, ck[u * npad + pc], ck[u * npad + j]);
            };
            sweep([&](const double* ck, int, int nr) {
                if (act) rows(ck, nr, [&](int, double q, double w) { r1 = add_rn(r1, mul_rn(q, w)); });
            });
            sweep([&](const double* ck, int, int nr) {
                if (act)
                    rows(ck, nr, [&](int, double q, double w) { r2 = add_rn(r2, mul_rn(q, sub_rn(w, mul_rn(r1, q)))); });
            });
            sweep([&](const double* ck, int i0, int nr) {
                if (act)
                    rows(ck, nr, [&](int u, double q, double w0) {
                        const double w = sub_rn(sub_rn(w0, mul_rn(r1, q)), mul_rn(r2, q));
                        Wj[(i0 + u) * npad] = w;
                        nn = add_rn(nn, mul_rn(w, w));
                    });
            });
            if (act) {
                R[static_cast<size_t>(s) * n + j] = add_rn(r1, r2);
                nrm[j] = sqrt(nn);
            }
            // the next step's argmax and normalisation follow a barrier
            fence_proxy_async_global();
            csync<kMode>();
        } else {
            __syncthreads();
            // two-pass MGS against every unselected column (qr.cpp:94-102); the
            // next step's fresh norm (qr.cpp:66-67) is accumulated in pass 2.
            for (int j = tid; j < n; j += kCpqrThreads) {
                if (posof[j] <= s) continue;
                // rows are consumed in chunks whose loads are all issued before the
                // chunk's (sequential, separately rounded) arithmetic: the sums keep
                // the reference's order, the memory latency is paid once per chunk
                double r1 = 0.0;
                for (int i0 = 0; i0 < rows; i0 += kPf) {
                    double qv[kPf], wv[kPf];
                    load_chunk(W, npad, pc, i0, rows, qv);
                    load_chunk(W, npad, j, i0, rows, wv);
#pragma unroll
                    for (int u = 0; u < kPf; ++u)
                        if (i0 + u < rows) r1 = add_rn(r1, mul_rn(qv[u], wv[u]));
                }
                double r2 = 0.0;
                for (int i0 = 0; i0 < rows; i0 += kPf) {
                    double qv[kPf], wv[kPf];
                    load_chunk(W, npad, pc, i0, rows, qv);
                    load_chunk(W, npad, j, i0, rows, wv);
#pragma unroll
                    for (int u = 0; u < kPf; ++u) {
                        if (i0 + u < rows) {
                            const double w = sub_rn(wv[u], mul_rn(r1, qv[u]));
                            W[(i0 + u) * npad + j] = w;
                            r2 = add_rn(r2, mul_rn(qv[u], w));
                        }
                    }
                }
                double nn = 0.0;
                for (int i0 = 0; i0 < rows; i0 += kPf) {
                    double qv[kPf], wv[kPf];
                    load_chunk(W, npad, pc, i0, rows, qv);
                    load_chunk(W, npad, j, i0, rows, wv);
#pragma unroll
                    for (int u = 0; u < kPf; ++u) {
                        if (i0 + u < rows) {
                            const double w = sub_rn(wv[u], mul_rn(r2, qv[u]));
                            W[(i0 + u) * npad + j] = w;
                            nn = add_rn(nn, mul_rn(w, w));
                        }
                    }
                }
                R[static_cast<size_t>(s) * n + j] = add_rn(r1, r2);
                nrm[j] = sqrt(nn);
            }
            __syncthreads();
        }
        rank = s + 1;
    }
    stop_producer();
    if (rank == 0) {  // qr.cpp:108-109
        finish_error(SPID_ZERO_MATRIX);
        return;
    }

    // ---- residual_fro (qr.cpp:111-115) and the singular-pivot check -------
    if (tid == 0) {
        double rsq = 0.0;
        for (int pos = rank; pos < n; ++pos) {
            const double nj = nrm[perm[pos]];
            rsq = add_rn(rsq, mul_rn(nj, nj));
        }
        p.resid[b] = sqrt(rsq);
        double max_diag = 0.0;  // qr.cpp:135-140
        for (int t = 0; t < rank; ++t) max_diag = fmax(max_diag, fabs(diag[t]));
        int sing = 0;
        for (int t = 0; t < rank; ++t)
            if (fabs(diag[t]) < 1e-14 * max_diag || max_diag == 0.0) sing = 1;
        sh.flag = sing;
    }
    // Q (= the normalised pivot columns kept in W) must be read out before W's
    // space is reused for the solve vectors
    if (p.Qout) {
        double* Qo = p.Qout + static_cast<size_t>(b) * rows * p.kcap;
        for (int e = tid; e < rank * rows; e += kCpqrThreads) {
            const int i = e % rows, t = e / rows;
            Qo[static_cast<size_t>(t) * rows + i] = W[i * npad + perm[t]];
        }
    }
    csync<kMode>();
    if (sh.flag && rank < n) {
        finish_error(SPID_SINGULAR_PIVOT);
        return;
    }

    // ---- coefficients in source column order (id.cpp:9-28) ----------------
    // R11 (position order) into r11[]; each non-skeleton column's right-hand
    // side R(0:rank, j) into X[t][j] (W's space, thread-contiguous); then the
    // back substitution of qr.cpp:143-149 runs in place, same operation order.
    double* X = W;
    for (int e = tid; e < rank * rank; e += kCpqrThreads) {
        const int ii = e / rank, jj = e % rank;
        r11[e] = jj >= ii ? R[static_cast<size_t>(ii) * n + perm[jj]] : 0.0;
    }
    for (int j = tid; j < n; j += kCpqrThreads)
        if (posof[j] >= rank)
            for (int t = 0; t < rank; ++t) X[t * npad + j] = R[static_cast<size_t>(t) * n + j];
    csync<kMode>();
    double* C = p.C + static_cast<size_t>(b) * p.strideC;
    const int kcap = static_cast<int>(p.kcap);
    int nonfinite = 0;
    for (int j = tid; j < n; j += kCpqrThreads) {
        double* cj = C + static_cast<size_t>(j) * kcap;
        const int pj = posof[j];
        if (pj < rank) {  // skeleton column: exact unit vector (id.cpp:12)
            for (int i = 0; i < rank; ++i) cj[i] = (i == pj) ? 1.0 : 0.0;
            continue;
        }
        for (int ii = rank - 1; ii >= 0; --ii) {
            double sum = X[ii * npad + j];
            const double* rrow = r11 + ii * rank;
#pragma unroll 4
            for (int jj = ii + 1; jj < rank; ++jj) sum = sub_rn(sum, mul_rn(rrow[jj], X[jj * npad + j]));
            const double x = div_rn(sum, rrow[ii]);
            X[ii * npad + j] = x;
            nonfinite |= !isfinite(x);
        }
        for (int i = 0; i < rank; ++i) cj[i] = X[i * npad + j];
    }
    nonfinite = csync_or<kMode>(nonfinite);
    if (nonfinite) {  // id.cpp:25-26
        finish_error(SPID_NON_FINITE_COEFFS);
        return;
    }

    // ---- outputs ----------------------------------------------------------
    int64_t* idx = p.indices + static_cast<size_t>(b) * kcap;
    for (int t = tid; t < rank; t += kCpqrThreads) idx[t] = perm[t];
    if (p.pivots)
        for (int pos = tid; pos < n; pos += kCpqrThreads) p.pivots[static_cast<size_t>(b) * n + pos] = perm[pos];
    if (p.Rout) {  // QrFactorization::r_mat, pivoted order, zero below diagonal
        double* Ro = p.Rout + static_cast<size_t>(b) * kcap * n;
        for (int e = tid; e < rank * n; e += kCpqrThreads) {
            const int i = e % rank, pos = e / rank;
            Ro[static_cast<size_t>(pos) * kcap + i] =
                pos < i ? 0.0 : R[static_cast<size_t>(i) * n + perm[pos]];
        }
    }
    if (tid == 0) {
        p.rank[b] = rank;
        p.status[b] = SPID_OK;
    }
}

}  // namespace

size_t cpqr_smem_bytes(int64_t rows, int64_t n, int64_t step_cap, bool w_in_shared) {
    size_t bytes = 2 * sizeof(double) * n + 2 * sizeof(int) * n + 16 + sizeof(double) * step_cap;
    if (w_in_shared) bytes += sizeof(double) * (rows * n + step_cap * step_cap);
    return bytes;
}

size_t cpqr_max_dyn_smem() { return 200 * 1024; }

bool cpqr_tall_supported(int64_t rows, int64_t n) { return n <= kCpqrThreads && rows >= 256; }

int cpqr_tall_npad(int64_t n) { return static_cast<int>((n + 1) & ~int64_t(1)); }  // 16-byte TMA rows

int cpqr_tall_ring_rows(int64_t n) {  // a multiple of 8 (the sweeps' row groups), <= 256 (TMA box)
    const int npad = cpqr_tall_npad(n);
    const int r = (kTallStageBytes / (npad * static_cast<int>(sizeof(double)))) & ~7;
    return r > 256 ? 256 : r;
}

cudaError_t launch_cpqr(const CpqrParams& p, bool w_in_shared, cudaStream_t stream) {
    const size_t smem = cpqr_smem_bytes(p.rows, p.n, p.step_cap, w_in_shared);
    CUtensorMap none{};
    if (w_in_shared) {
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(cpqr_id_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem));
            if (e != cudaSuccess) return e;
        }
        cpqr_id_kernel<0><<<static_cast<unsigned>(p.batch), kCpqrThreads, smem, stream>>>(p, none, 0);
    } else {
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(cpqr_id_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 static_cast<int>(smem));
            if (e != cudaSuccess) return e;
        }
        cpqr_id_kernel<1><<<static_cast<unsigned>(p.batch), kCpqrThreads, smem, stream>>>(p, none, 0);
    }
    return cudaGetLastError();
}

template <int kNpad>
cudaError_t launch_tall_t(const CpqrParams& p, const CUtensorMap* wmap, size_t smem, cudaStream_t stream) {
    auto kern = cpqr_id_kernel<2, kNpad>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(p.batch), kCpqrThreads + kWarp, smem, stream>>>(p, *wmap, cpqr_tall_ring_rows(p.n));
    return cudaGetLastError();
}

cudaError_t launch_cpqr_tall(const CpqrParams& p, const CUtensorMap* wmap, cudaStream_t stream) {
    if (!cpqr_tall_supported(p.rows, p.n) || p.npad != cpqr_tall_npad(p.n)) return cudaErrorInvalidValue;
    const size_t smem = 128 + static_cast<size_t>(kTallStages) * kTallStageBytes +
                        cpqr_smem_bytes(p.rows, p.n, p.step_cap, false);
    switch (p.npad) {  // the streaming pipeline's chunk widths and the archive's snapshot counts
        case 16: return launch_tall_t<16>(p, wmap, smem, stream);
        case 32: return launch_tall_t<32>(p, wmap, smem, stream);
        case 64: return launch_tall_t<64>(p, wmap, smem, stream);
        case 128: return launch_tall_t<128>(p, wmap, smem, stream);
        case 256: return launch_tall_t<256>(p, wmap, smem, stream);
        default: return launch_tall_t<0>(p, wmap, smem, stream);
    }
}

}  // namespace spidgpu
