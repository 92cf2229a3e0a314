// cpqr_reg_pair.cu -- the register-resident batched column ID of cpqr_reg.cu
// with each subdomain's columns split over a cluster of two CTAs on two SMs.
//
// Same restatement of column_id -> qr_core -> build_coeffs /
// solve_upper_triangular (proj/src/id.cpp:9-52, proj/src/qr.cpp:29-151) and
// the same operation sequence per column as cpqr_reg.cu, so the same bits.
// Why a pair: one thread per column, and the three MGS passes of a pivot step
// keep the FP64 pipe of the SM ~92% busy (profiles/r02c_cpqr_reg_summary.txt)
// while 84 of the 148 SMs idle at config 3's 64 subdomains. CTA r of the pair
// owns columns [128 r, 128 r + 128) (n in (128, 256]); per pivot step
//   - the two CTAs trade their local (norm, index) maxima AND the column of
//     that candidate in one st.async exchange (16 + 8 ROWS bytes counted on
//     the peer's slot barrier), so that whichever wins, both hold the pivot
//     column after a single round trip; both pick the same winner (the
//     total order of qr.cpp:68, compared in rank order in both) and divide
//     it by R(s,s) with the same rounding (qr.cpp:91-92);
//   - both keep identical position bookkeeping (perm / posof).
// After the loop each CTA writes its columns' norms into the peer's table and
// the pair meets at its one cluster barrier; the residual (position order over
// all columns), R11 (from global R) and each CTA's coefficient solve follow.
// Rules: fixed and tolerance; the blocked rule keeps the single-CTA kernel.
#include <math.h>

#include "cluster.cuh"
#include "common.cuh"
#include "kernels.h"

namespace spidgpu {

namespace {

using namespace cluster;

constexpr int kT = 128;                 // column threads per CTA, one column each
constexpr int kNH = kT;                 // columns per CTA
constexpr double kZeroFloor = 1e-300;   // qr.cpp:11
constexpr double kCollapseRel = 1e-14;  // qr.cpp:12
constexpr int kXSlots = 4;
// per-warp staging of the column load (as cpqr_reg.cu): 32 columns x 16 rows
constexpr int kStageRows = 16, kStagePitch = kStageRows + 1;
constexpr size_t kStageBytes = sizeof(double) * (kT / kWarp) * kWarp * kStagePitch;

struct alignas(16) XSlot {
    uint32_t w[4];
};

// sum_{pos = lo}^{hi - 1} v[pos], left to right, loads issued 8 ahead
__device__ __forceinline__ double sum_in_order(const double* v, int lo, int hi) {
    double acc = 0.0;
    int pos = lo;
    for (; pos + 8 <= hi; pos += 8) {
        double t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) t[u] = v[pos + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = add_rn(acc, t[u]);
    }
    for (; pos < hi; ++pos) acc = add_rn(acc, v[pos]);
    return acc;
}

template <int ROWS>
__global__ void __launch_bounds__(kT, 1) cpqr_regpair_kernel(CpqrParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ double red_v[kT / kWarp];
    __shared__ long long red_k[kT / kWarp];
    __shared__ int red_i[kT / kWarp];
    __shared__ __align__(16) double qbuf[ROWS + 2];     // q_s, divided
    __shared__ __align__(16) double qloc[ROWS];         // this CTA's best candidate column
    __shared__ __align__(16) double qrem[2][ROWS];      // the peer's, by step parity
    __shared__ uint64_t xbar[kXSlots];
    __shared__ XSlot xs[kXSlots];
    __shared__ int flag_sh;
    const double2* q2 = reinterpret_cast<const double2*>(qbuf);

    const uint32_t crank = ctarank(), peer = crank ^ 1u;
    const int b = static_cast<int>(blockIdx.x >> 1), tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int rows = static_cast<int>(p.rows), n = static_cast<int>(p.n);
    const int cap = static_cast<int>(p.step_cap);
    const int c0 = static_cast<int>(crank) * kNH, c1 = min(n, c0 + kNH);
    const int j = c0 + tid;  // this thread's column
    const bool mine = j < c1;
    for (int i = tid; i < ROWS + 2; i += kT) qbuf[i] = 0.0;  // rows..ROWS stay zero
    // dynamic smem: nrm[n] colsq[n] diag[cap] | perm[n] posof[n] | X[cap][kNH] R11[cap][cap]
    // (X and R11 double as the load's staging area)
    double* nrm = reinterpret_cast<double*>(smem_raw);
    double* colsq = nrm + n;
    double* diag = colsq + n;
    int* perm = reinterpret_cast<int*>(diag + cap);
    int* posof = perm + n;
    const size_t x_off = (reinterpret_cast<unsigned char*>(posof + n) - smem_raw + 15) & ~size_t(15);
    double* X = reinterpret_cast<double*>(smem_raw + x_off);  // X[s][tid]: R(s, own column)
    double* r11 = X + static_cast<size_t>(cap) * kNH;
    double* R = p.r_ws + static_cast<size_t>(b) * cap * n;  // R[s][col], global (both CTAs' columns)
    const double* Y = p.Y + static_cast<size_t>(b) * p.strideY;

    if (tid == 0) {
        for (int i = 0; i < kXSlots; ++i) mbar_init(&xbar[i], 1);
        fence_barrier_init();
    }
    __syncthreads();
    cluster_sync();  // both CTAs' barriers initialised before any remote traffic
    const uint32_t poff = mapa(smem_u32(&xs[0]), peer) - smem_u32(&xs[0]);  // peer window = local + poff

    // exchange k: both send 16 bytes into the peer's slot k % 4 and wait for
    // the peer's. Every caller passes a CTA barrier first, and consecutive
    // exchanges are separated by CTA barriers, so a slot is rewritten only
    // after every thread of the receiver has read it.
    uint32_t xk = 0;
    auto exchange = [&](uint32_t a, uint32_t b2, uint32_t c, uint32_t d) -> XSlot {
        const uint32_t sl = xk % kXSlots, ph = (xk / kXSlots) & 1;
        ++xk;
        if (tid == 0) {
            mbar_arrive_expect_tx(&xbar[sl], 16);
            st_async16(smem_u32(&xs[sl]) + poff, a, b2, c, d, smem_u32(&xbar[sl]) + poff);
        }
        mbar_wait_cluster(&xbar[sl], ph);
        return xs[sl];
    };
    auto pair_or = [&](int v) {
        v = __syncthreads_or(v);
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

    // ---- own columns into registers through the staging tile; finiteness
    // (qr.cpp:34-35, id.cpp:41-42) ---------------------------------------------
    double w[ROWS];
    int bad = 0;
    {
        double* stg = X + warp * (kWarp * kStagePitch);
        const int half = lane >> 4, r = lane & 15;
        const int jw = c0 + warp * kWarp;
#pragma unroll
        for (int r0 = 0; r0 < ROWS; r0 += kStageRows) {
#pragma unroll
            for (int it = 0; it < kWarp / 2; ++it) {
                const int cl = 2 * it + half, jj = jw + cl, i = r0 + r;
                double v = 0.0;
                if (jj < c1 && i < rows) v = Y[static_cast<size_t>(jj) * p.ldy + i];
                bad |= !isfinite(v);
                stg[cl * kStagePitch + r] = v;
            }
            __syncwarp();
#pragma unroll
            for (int u = 0; u < kStageRows; ++u)
                if (r0 + u < ROWS) w[r0 + u] = stg[lane * kStagePitch + u];
            __syncwarp();
        }
    }
    for (int jj = tid; jj < n; jj += kT) {
        perm[jj] = jj;
        posof[jj] = jj;
    }
    if (pair_or(bad)) {
        finish_error(SPID_NON_FINITE_INPUT);
        cluster_sync();
        return;
    }
    if (p.pre_status != SPID_OK) {
        finish_error(p.pre_status);
        cluster_sync();
        return;
    }

    // ---- initial norms, max_init over both halves (qr.cpp:47-51) ---------------
    double lmax = 0.0;
    if (mine) {
        double s = 0.0;  // padded rows add +0.0 to a sum that cannot be -0.0
#pragma unroll
        for (int i = 0; i < ROWS; ++i) s = add_rn(s, mul_rn(w[i], w[i]));
        const double v = sqrt(s);
        nrm[j] = v;
        lmax = v;
    }
    lmax = warp_max(lmax);
    if (lane == 0) red_v[warp] = lmax;
    __syncthreads();
    double max_init;
    {
        double m = 0.0;
#pragma unroll
        for (int k = 0; k < kT / kWarp; ++k) m = fmax(m, red_v[k]);
        const XSlot x = exchange(static_cast<uint32_t>(__double2loint(m)), static_cast<uint32_t>(__double2hiint(m)),
                                 0u, 0u);
        max_init = fmax(m, __hiloint2double(static_cast<int>(x.w[1]), static_cast<int>(x.w[0])));
    }
    if (max_init < kZeroFloor) {
        finish_error(SPID_ZERO_MATRIX);
        cluster_sync();
        return;
    }

    // ---- greedy pivoting loop (qr.cpp:61-106) ---------------------------------
    int rank = 0;
    const int step_limit = static_cast<int>(p.step_limit);
    bool alive = mine;  // column not yet selected, kept in a register
    for (int s = 0; s < step_limit; ++s) {
        // integer keys (norm_key): the argmax stays off the FP64 pipe
        long long bk = norm_key(-1.0);
        int bi = 0x7fffffff;
        if (alive) {
            const long long kj = norm_key(nrm[j]);
            if (key_better_k(kj, j, bk, bi)) {
                bk = kj;
                bi = j;
            }
        }
        warp_argmax_k(bk, bi);
        if (lane == 0) {
            red_k[warp] = bk;
            red_i[warp] = bi;
        }
        __syncthreads();
        long long vk = red_k[0];
        int ix = red_i[0];
#pragma unroll
        for (int k = 1; k < kT / kWarp; ++k)
            if (key_better_k(red_k[k], red_i[k], vk, ix)) {
                vk = red_k[k];
                ix = red_i[k];
            }
        double v = __longlong_as_double(vk);
        // the exchange: (norm, index) and the candidate column into the
        // peer's slot and its qrem[s & 1] (a CTA with no live column sends
        // zeros); the peer cannot run two steps ahead of this CTA's reads of
        // qrem[s & 1], because it needs this CTA's next message first
        double pv;
        int pi;
        {
            const uint32_t sl = xk % kXSlots, ph = (xk / kXSlots) & 1;
            ++xk;
            const uint32_t rb = smem_u32(&xbar[sl]) + poff;
            const uint32_t rq = smem_u32(qrem[s & 1]) + poff;
            const bool have = ix != 0x7fffffff;
            const int ow = have ? ix - c0 : 0;  // the candidate's thread (thread 0 sends zeros)
            if (tid == 0) mbar_arrive_expect_tx(&xbar[sl], static_cast<uint32_t>(16 + ROWS * sizeof(double)));
            if (tid == ow) {
#pragma unroll
                for (int i = 0; i < ROWS; ++i) qloc[i] = have ? w[i] : 0.0;  // zero padding past rows
            }
            __syncwarp();
            if (warp == ow / kWarp) {  // the candidate's warp ships the column, 16 bytes per lane
                for (int i = 2 * lane; i < ROWS; i += 2 * kWarp)
                    st_async16(rq + 8u * i, static_cast<uint32_t>(__double2loint(qloc[i])),
                               static_cast<uint32_t>(__double2hiint(qloc[i])),
                               static_cast<uint32_t>(__double2loint(qloc[i + 1])),
                               static_cast<uint32_t>(__double2hiint(qloc[i + 1])), rb);
            }
            if (tid == 0)
                st_async16(smem_u32(&xs[sl]) + poff, static_cast<uint32_t>(__double2loint(v)),
                           static_cast<uint32_t>(__double2hiint(v)), static_cast<uint32_t>(ix), 0u, rb);
            mbar_wait_cluster(&xbar[sl], ph);
            const XSlot x = xs[sl];
            pv = __hiloint2double(static_cast<int>(x.w[1]), static_cast<int>(x.w[0]));
            pi = static_cast<int>(x.w[2]);
        }
        // the same comparison, operands in rank order, in both CTAs
        const bool peer_wins = crank == 0 ? key_better(pv, pi, v, ix) : !key_better(v, ix, pv, pi);
        if (peer_wins) {
            v = pv;
            ix = pi;
        }
        int stop = 0;
        if (p.mode == RULE_TOL && v <= p.tol * max_init) stop = 1;  // qr.cpp:74-76
        if (!stop && v < kCollapseRel * max_init)                   // qr.cpp:77-81
            stop = (p.mode == RULE_FIXED && p.strict) ? 2 : 1;
        if (stop) {
            if (stop == 2) {
                finish_error(SPID_RANK_UNREACHABLE);
                cluster_sync();
                return;
            }
            break;
        }
        if (tid == 0) {  // position bookkeeping (qr.cpp:83-87), identical in both CTAs
            const int ps = posof[ix], cs = perm[s];
            perm[s] = ix;
            perm[ps] = cs;
            posof[ix] = s;
            posof[cs] = ps;
            if (crank == 0) R[static_cast<size_t>(s) * n + ix] = v;  // qr.cpp:89-90
            diag[s] = v;
        }
        const int pc = ix;
        const double pn = v;
        if (pc == j) alive = false;
        __syncthreads();  // qloc (written by one thread) visible to the dividers
        // q_s = w_s / R(s,s) in both CTAs with the same rounding
        if (tid < rows) {
            const double* src = peer_wins ? qrem[s & 1] : qloc;
            const double q = div_rn(src[tid], pn);
            qbuf[tid] = q;
            if (p.Qout && crank == 0)
                p.Qout[static_cast<size_t>(b) * rows * p.kcap + static_cast<size_t>(s) * rows + tid] = q;
        }
        __syncthreads();
        // two-pass MGS (qr.cpp:94-102) on the own column, as cpqr_reg.cu
        if (alive) {
            double r1 = 0.0;
#pragma unroll
            for (int i = 0; i < ROWS; i += 2) {
                const double2 q = q2[i / 2];
                r1 = add_rn(r1, mul_rn(q.x, w[i]));
                r1 = add_rn(r1, mul_rn(q.y, w[i + 1]));
            }
            asm volatile("" ::: "memory");
            double r2 = 0.0;
#pragma unroll
            for (int i = 0; i < ROWS; i += 2) {
                const double2 q = q2[i / 2];
                const double v0 = sub_rn(w[i], mul_rn(r1, q.x));
                w[i] = v0;
                r2 = add_rn(r2, mul_rn(q.x, v0));
                const double v1 = sub_rn(w[i + 1], mul_rn(r1, q.y));
                w[i + 1] = v1;
                r2 = add_rn(r2, mul_rn(q.y, v1));
            }
            asm volatile("" ::: "memory");
            double nn = 0.0;
#pragma unroll
            for (int i = 0; i < ROWS; i += 2) {
                const double2 q = q2[i / 2];
                const double v0 = sub_rn(w[i], mul_rn(r2, q.x));
                w[i] = v0;
                nn = add_rn(nn, mul_rn(v0, v0));
                const double v1 = sub_rn(w[i + 1], mul_rn(r2, q.y));
                w[i + 1] = v1;
                nn = add_rn(nn, mul_rn(v1, v1));
            }
            const double rs = add_rn(r1, r2);
            R[static_cast<size_t>(s) * n + j] = rs;  // global: R11, the R output
            X[s * kNH + tid] = rs;                   // shared: the right-hand sides
            nrm[j] = sqrt(nn);
        }
        rank = s + 1;
    }
    __syncthreads();
    // own norms into the peer's table, then the pair's one cluster barrier
    // (it also orders both CTAs' global R writes before the reads below)
    if (mine)
        asm volatile("st.shared::cluster.f64 [%0], %1;\n" ::"r"(smem_u32(nrm + j) + poff), "d"(nrm[j]) : "memory");
    cluster_sync();
    if (rank == 0) {  // qr.cpp:108-109
        finish_error(SPID_ZERO_MATRIX);
        return;
    }

    // ---- residual_fro in position order over all columns (qr.cpp:111-115),
    // singular pivots (qr.cpp:135-140) ------------------------------------------
    for (int jj = tid; jj < n; jj += kT) colsq[posof[jj]] = mul_rn(nrm[jj], nrm[jj]);
    __syncthreads();
    if (tid == 0) {
        const double rsq = sum_in_order(colsq, rank, n);
        if (crank == 0) p.resid[b] = sqrt(rsq);
        double max_diag = 0.0;
        for (int t = 0; t < rank; ++t) max_diag = fmax(max_diag, fabs(diag[t]));
        int sing = 0;
        for (int t = 0; t < rank; ++t)
            if (fabs(diag[t]) < 1e-14 * max_diag || max_diag == 0.0) sing = 1;
        flag_sh = sing;
    }
    __syncthreads();
    if (flag_sh && rank < n) {
        finish_error(SPID_SINGULAR_PIVOT);
        return;
    }

    // ---- coefficients (id.cpp:9-28, back substitution qr.cpp:143-149) ---------
    for (int e = tid; e < rank * rank; e += kT) {
        const int ii = e / rank, jj = e % rank;
        r11[e] = jj >= ii ? __ldcg(R + static_cast<size_t>(ii) * n + perm[jj]) : 0.0;
    }
    __syncthreads();
    double* C = p.C + static_cast<size_t>(b) * p.strideC;
    const int kcap = static_cast<int>(p.kcap);
    int nonfinite = 0;
    if (mine) {
        double* cj = C + static_cast<size_t>(j) * kcap;
        const int pj = posof[j];
        if (pj < rank) {
            for (int i = 0; i < rank; ++i) cj[i] = (i == pj) ? 1.0 : 0.0;
        } else {
            for (int ii = rank - 1; ii >= 0; --ii) {
                double sum = X[ii * kNH + tid];
                const double* rrow = r11 + ii * rank;
#pragma unroll 4
                for (int jj = ii + 1; jj < rank; ++jj) sum = sub_rn(sum, mul_rn(rrow[jj], X[jj * kNH + tid]));
                const double x = div_rn(sum, rrow[ii]);
                X[ii * kNH + tid] = x;
                nonfinite |= !isfinite(x);
            }
            for (int i = 0; i < rank; ++i) cj[i] = X[i * kNH + tid];
        }
    }
    if (pair_or(nonfinite)) {  // id.cpp:25-26
        finish_error(SPID_NON_FINITE_COEFFS);
        return;
    }
    if (crank == 0) {
        int64_t* idx = p.indices + static_cast<size_t>(b) * kcap;
        for (int t = tid; t < rank; t += kT) idx[t] = perm[t];
        if (p.pivots)
            for (int pos = tid; pos < n; pos += kT) p.pivots[static_cast<size_t>(b) * n + pos] = perm[pos];
        if (p.Rout) {
            double* Ro = p.Rout + static_cast<size_t>(b) * kcap * n;
            for (int e = tid; e < rank * n; e += kT) {
                const int i = e % rank, pos = e / rank;
                Ro[static_cast<size_t>(pos) * kcap + i] =
                    pos < i ? 0.0 : __ldcg(R + static_cast<size_t>(i) * n + perm[pos]);
            }
        }
        if (tid == 0) {
            p.rank[b] = rank;
            p.status[b] = SPID_OK;
        }
    }
}

size_t regpair_smem(int64_t n, int64_t cap) {
    const size_t xr = sizeof(double) * (cap * kNH + cap * cap);
    return sizeof(double) * (2 * n + cap) + sizeof(int) * 2 * n + 16 + (xr > kStageBytes ? xr : kStageBytes);
}

template <int ROWS>
cudaError_t go(const CpqrParams& p, cudaStream_t stream) {
    const size_t smem = regpair_smem(p.n, p.step_cap);
    auto kern = cpqr_regpair_kernel<ROWS>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * p.batch));
    cfg.blockDim = dim3(kT);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p);
}

}  // namespace

// 33-48 rows only: one CTA per SM sub-partition then runs latency-bound
// chains that the split shortens (config 3: 110 -> 100 us); 32 rows or
// fewer gain nothing, and 64-80-row columns do not fit the registers of a
// 128-thread CTA next to the exchange (local memory; 342 -> 567 us)
bool cpqr_regpair_supported(int64_t rows, int64_t n, int mode, int64_t step_cap) {
    return (mode == RULE_FIXED || mode == RULE_TOL) && rows > 32 && rows <= 48 && n > kNH && n <= 2 * kNH &&
           regpair_smem(n, step_cap) <= 200 * 1024;
}

cudaError_t launch_cpqr_regpair(const CpqrParams& p, cudaStream_t stream) {
    if (!cpqr_regpair_supported(p.rows, p.n, p.mode, p.step_cap)) return cudaErrorNotSupported;
    return go<48>(p, stream);
}

}  // namespace spidgpu
