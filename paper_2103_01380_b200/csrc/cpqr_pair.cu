// cpqr_pair.cu -- the tall batched column ID (cpqr.cu mode 2) with each
// subdomain's columns split over a cluster of two CTAs on two SMs.
//
// Same restatement of column_id -> qr_core -> build_coeffs /
// solve_upper_triangular (proj/src/id.cpp:9-52, proj/src/qr.cpp:29-151) and
// the same operation sequence per column as cpqr.cu, so the same bits. Why a
// pair: with W (rows x n, n up to 256) streamed from HBM through one SM's TMA
// ring for every sweep, the 4096 x 256 blocks of the archive's exact mode run
// at the SM's throughput (64 subdomains: 15.5 ms on 64 SMs; the same blocks
// with 128 columns take 8.7 ms). Here CTA r of the pair owns columns
// [r n/2, r n/2 + n/2) and streams only those; per pivot step the two CTAs
//   - trade their local (norm, index) maxima (16-byte st.async into the
//     peer's slot, completing on its mbarrier) and pick the same winner (the
//     total order of qr.cpp:68);
//   - both compute the normalised pivot column q themselves: the producer
//     loads the pivot column pair beside every first-sweep chunk (a second
//     tensor map, box {2, ring_rows}) and an idle warp divides it into qsm
//     with the same rounding, ahead of the column warps;
//   - keep identical copies of the position bookkeeping (perm / posof).
// The producer warps keep streaming while the column warps trade, so the
// pair meets at a cluster barrier only at the start and once at the end,
// after the norms of both halves were exchanged; the residual (position
// order over all columns) and the coefficient solve (R11 from global R)
// follow it. Supported rules: fixed and
// tolerance (the archive's and the streaming stages'); the blocked rule keeps
// the single-CTA kernel.
#include <math.h>

#include "cluster.cuh"
#include "common.cuh"
#include "kernels.h"

namespace spidgpu {

namespace {

using namespace cluster;

constexpr int kThr = 256;                 // column threads per CTA (8 warps)
constexpr int kProducer = kThr / kWarp;   // the 9th warp streams W
constexpr int kStages = 5;
constexpr int kStageBytes = 32 * 1024;
constexpr double kZeroFloor = 1e-300;     // qr.cpp:11
constexpr double kCollapseRel = 1e-14;    // qr.cpp:12

__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;\n" ::: "memory"); }
__device__ __forceinline__ void bsync() { asm volatile("bar.sync 1, %0;\n" ::"n"(kThr) : "memory"); }
__device__ __forceinline__ int bsync_or(int v) {
    int r;
    asm volatile(
        "{\n.reg .pred p, q;\nsetp.ne.s32 p, %1, 0;\nbar.red.or.pred q, 1, %2, p;\nselp.s32 %0, 1, 0, q;\n}\n"
        : "=r"(r)
        : "r"(v), "n"(kThr)
        : "memory");
    return r;
}
struct PairShared {
    double best_v, max_init;
    int best_i, stop, flag, chunks, side_pc;
};
// A point-to-point exchange slot: 16 bytes the peer writes by st.async
struct alignas(16) XSlot {
    uint32_t w[4];
};
constexpr int kXSlots = 4;
constexpr int kQWarp = kThr / kWarp - 1;  // idle column warp (NH <= 128): computes q

// NH: columns per CTA (half of the padded row length); W rows are 2 NH long.
template <int NH>
__global__ void __launch_bounds__(kThr + kWarp, 1)
    cpqr_pair_kernel(CpqrParams p, const __grid_constant__ CUtensorMap wmap, const __grid_constant__ CUtensorMap pmap,
                     int ring_rows) {
    constexpr int npad = 2 * NH;
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ PairShared sh;
    __shared__ double red_v[kThr / kWarp];
    __shared__ int red_i[kThr / kWarp];
    __shared__ uint64_t ring_full[kStages], ring_empty[kStages], go_bar;
    __shared__ uint64_t xbar[kXSlots];  // exchanges with the peer
    __shared__ uint64_t qready[kStages];  // q of a first-sweep chunk is in qsm
    __shared__ XSlot xs[kXSlots];

    const uint32_t crank = ctarank(), peer = crank ^ 1u;
    const int b = static_cast<int>(blockIdx.x >> 1);
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rows = static_cast<int>(p.rows), n = static_cast<int>(p.n);
    const int c0 = static_cast<int>(crank) * NH, c1 = min(n, c0 + NH);
    const int j = c0 + tid;                       // this thread's column
    const bool mine = tid < NH && j < c1;

    // smem: ring | side ring | q[rows] | nrm[n] perm[n] posof[n] | diag[cap]
    unsigned char* cur = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    double* ring = reinterpret_cast<double*>(cur);
    cur += static_cast<size_t>(kStages) * kStageBytes;
    double* side = reinterpret_cast<double*>(cur);  // per stage: the pivot column pair, ring_rows x 2
    cur += static_cast<size_t>(kStages) * ring_rows * 2 * sizeof(double);
    double* qsm = reinterpret_cast<double*>(cur);
    cur += sizeof(double) * ((rows + 1) & ~1);
    double* nrm = reinterpret_cast<double*>(cur);
    cur += sizeof(double) * n;
    int* perm = reinterpret_cast<int*>(cur);
    cur += sizeof(int) * n;
    int* posof = reinterpret_cast<int*>(cur);
    cur += sizeof(int) * n;
    cur = smem_raw + ((cur - smem_raw + 15) & ~ptrdiff_t(15));
    double* diag = reinterpret_cast<double*>(cur);
    double* W = p.w_ws + static_cast<size_t>(b) * rows * npad;
    double* R = p.r_ws + static_cast<size_t>(b) * p.step_cap * n;
    double* r11 = p.r11_ws + (static_cast<size_t>(b) * 2 + crank) * p.step_cap * p.step_cap;  // per CTA
    const double* Y = p.Y + static_cast<size_t>(b) * p.strideY;

    const int nck = (rows + ring_rows - 1) / ring_rows;
    if (tid == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(&ring_full[i], 1);
            mbar_init(&ring_empty[i], kThr / kWarp);
        }
        mbar_init(&go_bar, 1);
        for (int i = 0; i < kXSlots; ++i) mbar_init(&xbar[i], 1);
        for (int i = 0; i < kStages; ++i) mbar_init(&qready[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    // both CTAs' barriers initialised before any remote traffic
    cluster_sync();
    if (warp == kProducer) {
        if (lane == 0) {
            prefetch_tmap(&wmap);
            prefetch_tmap(&pmap);
            const uint32_t bytes = static_cast<uint32_t>(ring_rows) * NH * sizeof(double);
            const uint32_t sbytes = static_cast<uint32_t>(ring_rows) * 2 * sizeof(double);
            uint32_t g = 0, gophase = 0;
            for (;;) {
                mbar_wait(&go_bar, gophase);
                gophase ^= 1;
                const int chunks = sh.chunks, spc = sh.side_pc;
                if (chunks == 0) break;
                for (int c = 0; c < chunks; ++c, ++g) {
                    const uint32_t slot = g % kStages;
                    const bool sd = spc >= 0 && c < nck;  // first sweep of a step: the pivot column too
                    if (g >= kStages) mbar_wait(&ring_empty[slot], ((g / kStages) - 1) & 1);
                    mbar_arrive_expect_tx(&ring_full[slot], bytes + (sd ? sbytes : 0u));
                    tma_load_3d(ring + static_cast<size_t>(slot) * (kStageBytes / sizeof(double)), &wmap,
                                &ring_full[slot], c0, (c % nck) * ring_rows, b);
                    if (sd)
                        tma_load_3d(side + static_cast<size_t>(slot) * ring_rows * 2, &pmap, &ring_full[slot],
                                    spc & ~1, (c % nck) * ring_rows, b);
                }
            }
        }
        __syncwarp();
        cluster_sync();  // the pair's one final cluster barrier (all threads)
        return;
    }

    const uint32_t poff = mapa(smem_u32(&sh), peer) - smem_u32(&sh);  // peer window = local + poff
    const uint32_t peer_nrm = smem_u32(nrm) + poff;
    // exchange k: both send 16 bytes to the peer's slot k % 4 and wait for
    // the peer's; a slot is rewritten only after both passed exchange k + 3
    uint32_t xk = 0;
    auto exchange = [&](uint32_t a, uint32_t b2, uint32_t c, uint32_t d) -> XSlot {
        const uint32_t sl = xk % kXSlots, ph = (xk / kXSlots) & 1;
        ++xk;
        if (tid == 0) {
            // release this CTA's earlier global W stores (ordered before by
            // the CTA barrier every caller passes first) at cluster scope:
            // the peer's TMA reads the pivot column from W after the
            // argmax exchange
            asm volatile("fence.acq_rel.cluster;\n" ::: "memory");
            mbar_arrive_expect_tx(&xbar[sl], 16);
            st_async16(smem_u32(&xs[sl]) + poff, a, b2, c, d, smem_u32(&xbar[sl]) + poff);
        }
        mbar_wait_cluster(&xbar[sl], ph);
        return xs[sl];
    };
    uint32_t qk = 0;  // first-sweep chunks so far (qready's phases)

    uint32_t gcons = 0;
    auto start_sweeps = [&](int passes, int side_pc) {
        fence_async_global();
        bsync();
        if (tid == 0) {
            sh.chunks = passes * nck;
            sh.side_pc = side_pc;
            mbar_arrive(&go_bar);
        }
    };
    auto stop_producer = [&]() {
        if (tid == 0) {
            sh.chunks = 0;
            mbar_arrive(&go_bar);
        }
    };
    auto sweep = [&](auto&& body) {
        for (int c = 0; c < nck; ++c, ++gcons) {
            const uint32_t slot = gcons % kStages;
            mbar_wait(&ring_full[slot], (gcons / kStages) & 1);
            const int i0 = c * ring_rows;
            body(ring + slot * (kStageBytes / sizeof(double)), i0, min(ring_rows, rows - i0));
            __syncwarp();
            if (lane == 0) mbar_arrive(&ring_empty[slot]);
        }
    };
    // an OR over both CTAs (every column thread of both calls it)
    auto pair_or = [&](int v) {
        v = bsync_or(v);
        const XSlot x = exchange(static_cast<uint32_t>(v), 0u, 0u, 0u);
        return v | static_cast<int>(x.w[0]);
    };
    auto finish_error = [&](int code) {
        if (tid == 0 && crank == 0) {
            p.status[b] = code;
            p.rank[b] = 0;
            p.resid[b] = 0.0;
        }
    };
    // early exits (decided identically in both CTAs): release the producer
    // and join the final cluster barrier
    auto leave = [&]() {
        stop_producer();
        cluster_sync();
    };

    // ---- load own columns, finiteness (qr.cpp:34-35, id.cpp:41-42) ----------
    int bad = 0;
    const int ncols = c1 > c0 ? c1 - c0 : 0;
    for (int e = tid; e < rows * ncols; e += kThr) {
        const int i = e % rows, jj = c0 + e / rows;
        const double v = Y[static_cast<size_t>(jj) * p.ldy + i];
        bad |= !isfinite(v);
        W[i * npad + jj] = v;
    }
    for (int jj = tid; jj < n; jj += kThr) {
        perm[jj] = jj;
        posof[jj] = jj;
    }
    if (pair_or(bad)) {
        finish_error(SPID_NON_FINITE_INPUT);
        leave();
        return;
    }
    if (p.pre_status != SPID_OK) {
        finish_error(p.pre_status);
        leave();
        return;
    }

    // ---- initial norms of own columns, max_init over both (qr.cpp:47-51) ----
    start_sweeps(1, -1);
    double lmax = 0.0;
    {
        double s = 0.0;
        sweep([&](const double* ck, int, int nr) {
            if (mine)
#pragma unroll 8
                for (int u = 0; u < nr; ++u) {
                    const double w = ck[u * NH + tid];
                    s = add_rn(s, mul_rn(w, w));
                }
        });
        if (mine) {
            const double v = sqrt(s);
            nrm[j] = v;
            lmax = v;
        }
    }
    lmax = warp_max(lmax);
    if (lane == 0) red_v[warp] = lmax;
    bsync();
    if (tid == 0) {
        double m = 0.0;
        for (int w = 0; w < kThr / kWarp; ++w) m = fmax(m, red_v[w]);
        sh.max_init = m;
    }
    bsync();
    double max_init;
    {
        const double m = sh.max_init;
        const XSlot x = exchange(static_cast<uint32_t>(__double2loint(m)), static_cast<uint32_t>(__double2hiint(m)),
                                 0u, 0u);
        max_init = fmax(m, __hiloint2double(static_cast<int>(x.w[1]), static_cast<int>(x.w[0])));
    }
    if (max_init < kZeroFloor) {
        finish_error(SPID_ZERO_MATRIX);
        leave();
        return;
    }

    // ---- greedy pivoting loop (qr.cpp:61-106) ---------------------------------
    int rank = 0;
    const int step_limit = static_cast<int>(p.step_limit);
    for (int s = 0; s < step_limit; ++s) {
        double bv = -1.0;
        int bi = 0x7fffffff;
        if (mine && posof[j] >= s) {
            bv = nrm[j];
            bi = j;
        }
        warp_argmax(bv, bi);
        if (lane == 0) {
            red_v[warp] = bv;
            red_i[warp] = bi;
        }
        bsync();
        if (tid == 0) {
            double v = red_v[0];
            int ix = red_i[0];
            for (int w = 1; w < kThr / kWarp; ++w)
                if (key_better(red_v[w], red_i[w], v, ix)) {
                    v = red_v[w];
                    ix = red_i[w];
                }
            sh.best_v = v;
            sh.best_i = ix;
        }
        bsync();
        {
            const double lv = sh.best_v;
            const int li = sh.best_i;
            const XSlot x = exchange(static_cast<uint32_t>(__double2loint(lv)), static_cast<uint32_t>(__double2hiint(lv)),
                                     static_cast<uint32_t>(li), 0u);
            if (tid == 0) {
                const double pv = __hiloint2double(static_cast<int>(x.w[1]), static_cast<int>(x.w[0]));
                const int pi = static_cast<int>(x.w[2]);
                // the same comparison, operands in rank order, in both CTAs:
                // they agree on the pivot even when a norm is NaN
                const bool peer_wins = crank == 0 ? key_better(pv, pi, lv, li) : !key_better(lv, li, pv, pi);
                if (peer_wins) {
                    sh.best_v = pv;
                    sh.best_i = pi;
                }
            }
        }
        if (tid == 0) {
            const double v = sh.best_v;
            const int ix = sh.best_i;
            int stop = 0;
            if (p.mode == RULE_TOL && v <= p.tol * max_init) stop = 1;  // qr.cpp:74-76
            if (!stop && v < kCollapseRel * max_init)                   // qr.cpp:77-81
                stop = (p.mode == RULE_FIXED && p.strict) ? 2 : 1;
            if (!stop) {  // position swap (qr.cpp:83-87), identical in both CTAs
                const int ps = posof[ix], cs = perm[s];
                perm[s] = ix;
                perm[ps] = cs;
                posof[ix] = s;
                posof[cs] = ps;
                if (crank == 0) R[static_cast<size_t>(s) * n + ix] = v;  // qr.cpp:89-90
                diag[s] = v;
            }
            sh.stop = stop;
        }
        bsync();
        if (sh.stop) {
            if (sh.stop == 2) {
                finish_error(SPID_RANK_UNREACHABLE);
                leave();
                return;
            }
            break;
        }
        const int pc = sh.best_i;
        const double pn = sh.best_v;
        // two-pass MGS (qr.cpp:94-102) over own columns: three back-to-back
        // read sweeps (r1; r2 from w - r1 q; w'' = (w - r1 q) - r2 q stored,
        // with its norm), as cpqr.cu
        const bool act = mine && posof[j] > s;
        start_sweeps(3, pc);
        double r1 = 0.0, r2 = 0.0, nn = 0.0;
        double* Wj = W + j;
        // rows of a chunk in order: whole groups of kGrp with the next
        // group's (q, w) loaded before the current group's dependent chain
        // (the last group reloads itself, branch-free), then the ragged
        // tail -- as cpqr.cu's sweeps, with q from shared memory
        constexpr int kGrp = 8;
        auto rows_of = [&](const double* ck, int i0, int nr, auto&& f) {
            const int nfull = nr & ~(kGrp - 1);
            if (nfull) {
                double qa[kGrp], wa[kGrp];
#pragma unroll
                for (int t = 0; t < kGrp; ++t) {
                    qa[t] = qsm[i0 + t];
                    wa[t] = ck[t * NH + tid];
                }
                for (int u0 = 0; u0 < nfull; u0 += kGrp) {
                    const int un = min(u0 + kGrp, nfull - kGrp);
                    double qb[kGrp], wb[kGrp];
#pragma unroll
                    for (int t = 0; t < kGrp; ++t) {
                        qb[t] = qsm[i0 + un + t];
                        wb[t] = ck[(un + t) * NH + tid];
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
            for (int u = nfull; u < nr; ++u) f(u, qsm[i0 + u], ck[u * NH + tid]);
        };
        // first sweep: q_s = w_s / R(s,s) (qr.cpp:91-92), chunk by chunk, by
        // the idle warp kQWarp of BOTH CTAs from the pivot column pair the
        // producer loads beside each chunk (the same div_rn, so the same
        // bits in both; no transfer between the CTAs). The column warps
        // wait for a chunk's q before its r1 terms; sweeps 2 and 3 find all
        // of q in qsm. CTA 0 also stores q as Q's column s (the Q output).
        // W's pivot column is left as it is: the peer may still be reading
        // it for this sweep.
        double* qo = p.Qout && crank == 0 ? p.Qout + (static_cast<size_t>(b) * p.kcap + s) * rows : nullptr;
        for (int c = 0; c < nck; ++c, ++gcons, ++qk) {
            const uint32_t slot = gcons % kStages, qs = qk % kStages;
            mbar_wait(&ring_full[slot], (gcons / kStages) & 1);
            const int i0 = c * ring_rows, nr = min(ring_rows, rows - i0);
            if (warp == kQWarp) {
                const double* pcol = side + static_cast<size_t>(slot) * ring_rows * 2 + (pc & 1);
                for (int u = lane; u < nr; u += kWarp) {
                    const double q = div_rn(pcol[2 * u], pn);
                    qsm[i0 + u] = q;
                    if (qo) qo[i0 + u] = q;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&qready[qs]);
            } else if (warp < NH / kWarp) {
                mbar_wait(&qready[qs], (qk / kStages) & 1);
                if (act)
                    rows_of(ring + slot * (kStageBytes / sizeof(double)), i0, nr,
                            [&](int, double q, double w) { r1 = add_rn(r1, mul_rn(q, w)); });
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&ring_empty[slot]);
        }
        sweep([&](const double* ck, int i0, int nr) {
            if (act)
                rows_of(ck, i0, nr, [&](int, double q, double w) { r2 = add_rn(r2, mul_rn(q, sub_rn(w, mul_rn(r1, q)))); });
        });
        sweep([&](const double* ck, int i0, int nr) {
            if (act)
                rows_of(ck, i0, nr, [&](int u, double q, double w0) {
                    const double w = sub_rn(sub_rn(w0, mul_rn(r1, q)), mul_rn(r2, q));
                    Wj[(i0 + u) * npad] = w;
                    nn = add_rn(nn, mul_rn(w, w));
                });
        });
        if (act) {
            R[static_cast<size_t>(s) * n + j] = add_rn(r1, r2);
            nrm[j] = sqrt(nn);
        }
        fence_async_global();
        bsync();
        rank = s + 1;
    }
    // ---- the pair's one final cluster barrier: own norms into the peer
    // first; it also orders both CTAs' R and W writes before the reads below
    if (mine) asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(peer_nrm + 8u * static_cast<uint32_t>(j)),
                           "d"(nrm[j])
                           : "memory");
    stop_producer();
    cluster_sync();
    if (rank == 0) {  // qr.cpp:108-109
        finish_error(SPID_ZERO_MATRIX);
        return;
    }

    // ---- residual_fro (qr.cpp:111-115) in position order over all columns;
    // singular pivots (qr.cpp:135-140) ------------------------------------------
    if (tid == 0) {
        double rsq = 0.0;
        for (int pos = rank; pos < n; ++pos) {
            const double nj = nrm[perm[pos]];
            rsq = add_rn(rsq, mul_rn(nj, nj));
        }
        if (crank == 0) p.resid[b] = sqrt(rsq);
        double max_diag = 0.0;
        for (int t = 0; t < rank; ++t) max_diag = fmax(max_diag, fabs(diag[t]));
        int sing = 0;
        for (int t = 0; t < rank; ++t)
            if (fabs(diag[t]) < 1e-14 * max_diag || max_diag == 0.0) sing = 1;
        sh.flag = sing;
    }
    bsync();
    if (sh.flag && rank < n) {
        finish_error(SPID_SINGULAR_PIVOT);
        return;
    }

    // ---- coefficients in source column order (id.cpp:9-28) -------------------
    // R11 per CTA (its own copy in the workspace); each CTA solves its own
    // non-skeleton columns (qr.cpp:143-149, the same operation order) in W's
    // space, as cpqr.cu; the Q read-out above precedes the reuse (CTA 0
    // reads W's pivot columns, CTA 1 overwrites only its own columns' rows,
    // and no pivot column is solved).
    for (int e = tid; e < rank * rank; e += kThr) {
        const int ii = e / rank, jj = e % rank;
        r11[e] = jj >= ii ? R[static_cast<size_t>(ii) * n + perm[jj]] : 0.0;
    }
    bsync();
    double* X = W;
    if (mine && posof[j] >= rank)
        for (int t = 0; t < rank; ++t) X[t * npad + j] = R[static_cast<size_t>(t) * n + j];
    double* C = p.C + static_cast<size_t>(b) * p.strideC;
    const int kcap = static_cast<int>(p.kcap);
    int nonfinite = 0;
    if (mine) {
        double* cj = C + static_cast<size_t>(j) * kcap;
        const int pj = posof[j];
        if (pj < rank) {  // skeleton column: exact unit vector (id.cpp:12)
            for (int i = 0; i < rank; ++i) cj[i] = (i == pj) ? 1.0 : 0.0;
        } else {
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
    }
    if (pair_or(nonfinite)) {  // id.cpp:25-26
        finish_error(SPID_NON_FINITE_COEFFS);
        return;
    }

    // ---- outputs (CTA 0) --------------------------------------------------------
    if (crank == 0) {
        int64_t* idx = p.indices + static_cast<size_t>(b) * kcap;
        for (int t = tid; t < rank; t += kThr) idx[t] = perm[t];
        if (p.pivots)
            for (int pos = tid; pos < n; pos += kThr) p.pivots[static_cast<size_t>(b) * n + pos] = perm[pos];
        if (p.Rout) {
            double* Ro = p.Rout + static_cast<size_t>(b) * kcap * n;
            for (int e = tid; e < rank * n; e += kThr) {
                const int i = e % rank, pos = e / rank;
                Ro[static_cast<size_t>(pos) * kcap + i] = pos < i ? 0.0 : R[static_cast<size_t>(i) * n + perm[pos]];
            }
        }
        if (tid == 0) {
            p.rank[b] = rank;
            p.status[b] = SPID_OK;
        }
    }
}

template <int NH>
cudaError_t launch_pair_t(const CpqrParams& p, const CUtensorMap* wmap, const CUtensorMap* pmap, int ring_rows,
                          cudaStream_t stream) {
    auto kern = cpqr_pair_kernel<NH>;
    const size_t smem = cpqr_pair_smem_bytes(p.rows, p.n, p.step_cap);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * p.batch));
    cfg.blockDim = dim3(kThr + kWarp);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p, *wmap, *pmap, ring_rows);
}

}  // namespace

size_t cpqr_pair_smem_bytes(int64_t rows, int64_t n, int64_t step_cap) {
    return 128 + static_cast<size_t>(kStages) * kStageBytes +
           static_cast<size_t>(kStages) * cpqr_pair_ring_rows(n) * 2 * sizeof(double) +
           sizeof(double) * ((rows + 1) & ~int64_t(1)) +
           sizeof(double) * n + 2 * sizeof(int) * n + 16 + sizeof(double) * step_cap;
}

bool cpqr_pair_supported(int64_t rows, int64_t n, int mode, int64_t step_cap) {
    return (mode == RULE_FIXED || mode == RULE_TOL) && n > 64 && n <= 256 && rows >= 256 &&
           cpqr_pair_smem_bytes(rows, n, step_cap) <= 220 * 1024;
}

int cpqr_pair_half(int64_t n) { return n > 128 ? 128 : 64; }

int cpqr_pair_ring_rows(int64_t n) {
    const int r = (kStageBytes / (cpqr_pair_half(n) * static_cast<int>(sizeof(double)))) & ~7;
    return r > 256 ? 256 : r;
}

cudaError_t launch_cpqr_pair(const CpqrParams& p, const CUtensorMap* wmap, const CUtensorMap* pmap,
                             cudaStream_t stream) {
    if (!cpqr_pair_supported(p.rows, p.n, p.mode, p.step_cap) || p.npad != 2 * cpqr_pair_half(p.n))
        return cudaErrorInvalidValue;
    const int rr = cpqr_pair_ring_rows(p.n);
    return cpqr_pair_half(p.n) == 128 ? launch_pair_t<128>(p, wmap, pmap, rr, stream)
                                      : launch_pair_t<64>(p, wmap, pmap, rr, stream);
}

}  // namespace spidgpu
