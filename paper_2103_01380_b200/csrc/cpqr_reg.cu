// cpqr_reg.cu -- register-resident batched column ID for sketch-sized inputs
// (rows <= 80, n <= 512): the same restatement of column_id -> qr_core ->
// build_coeffs / solve_upper_triangular as cpqr.cu (proj/src/id.cpp:9-52,
// proj/src/qr.cpp:29-151), bit for bit, but each thread keeps its column(s)
// of the working matrix in registers for the whole factorisation. Per step
// only the pivot column q travels through shared memory (written once by its
// owner, read by everyone as 16-byte broadcasts), so the three MGS passes are
// pure FP64 dependency chains with no per-element shared-memory traffic.
//
// Summation order is unchanged: every dot product / norm is a left-to-right
// sum of separately rounded products over i = 0..rows-1 (__dmul_rn /
// __dadd_rn), exactly the reference's x86-64 operation sequence.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace spidgpu {

namespace {

constexpr int kT = 256;
constexpr double kZeroFloor = 1e-300;  // qr.cpp:11
constexpr double kCollapseRel = 1e-14; // qr.cpp:12

struct Sh {
    double best_v, max_init, yfro;
    int best_i, stop, flag;
};

// per-warp staging of the column load: 32 columns x 16 rows, row stride 17
// (conflict-free column reads by the owning lanes)
constexpr int kStageRows = 16, kStagePitch = kStageRows + 1;
constexpr size_t kStageBytes = sizeof(double) * (kT / kWarp) * kWarp * kStagePitch;

// sum_{pos = lo}^{hi - 1} v[pos], left to right (a serial chain), the loads
// issued eight at a time ahead of the adds
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

template <int ROWS, int CPT>
__global__ void __launch_bounds__(kT, 1) cpqr_reg_kernel(CpqrParams p) {
    extern __shared__ __align__(16) unsigned char smem_raw[];
    __shared__ Sh sh;
    __shared__ double red_v[kT / kWarp];
    __shared__ long long red_k[kT / kWarp];
    __shared__ int red_i[kT / kWarp];
    __shared__ __align__(16) double qbuf[ROWS + 2];
    const double2* q2 = reinterpret_cast<const double2*>(qbuf);

    const int b = blockIdx.x, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    for (int i = tid; i < ROWS + 2; i += kT) qbuf[i] = 0.0;  // rows..ROWS stay zero
    const int rows = static_cast<int>(p.rows), n = static_cast<int>(p.n);
    const int cap = static_cast<int>(p.step_cap);
    // dynamic smem: nrm[n] colsq[n] diag[cap] | perm[n] posof[n] | X[cap][n] R11[cap][cap]
    // (X and R11 double as the load's staging area before the pivot loop)
    double* nrm = reinterpret_cast<double*>(smem_raw);
    double* colsq = nrm + n;
    double* diag = colsq + n;
    int* perm = reinterpret_cast<int*>(diag + cap);
    int* posof = perm + n;
    // offsets from smem_raw (not integer-cast pointers) keep the shared
    // window visible to the compiler: LDS/STS instead of generic accesses
    const size_t x_off = (reinterpret_cast<unsigned char*>(posof + n) - smem_raw + 15) & ~size_t(15);
    double* X = reinterpret_cast<double*>(smem_raw + x_off);
    double* r11 = X + static_cast<size_t>(cap) * n;
    double* R = p.r_ws + static_cast<size_t>(b) * cap * n;  // R[s][col], global
    const double* Y = p.Y + static_cast<size_t>(b) * p.strideY;

    auto finish_error = [&](int code) {
        if (tid == 0) {
            p.status[b] = code;
            p.rank[b] = 0;
            p.resid[b] = 0.0;
        }
    };

    // ---- columns into registers; finiteness (qr.cpp:34-35, id.cpp:41-42) ----
    double w[CPT][ROWS];
    // Branch-free padded loops while the column fits the register budget;
    // larger tiles exit at `rows` (a uniform branch) to keep registers down.
    // Both are bit-identical: padded rows only ever contribute +0.0.
    constexpr bool kFree = ROWS * CPT <= 48;
    // MGS passes of larger tiles stop at the first whole group of kGrp rows
    // past `rows` (the padded rows in between are +0.0: bit-neutral), so the
    // compiler schedules each group's independent products ahead of its
    // dependent adds instead of branching per element
    constexpr int kGrp = 16;
    // Loaded through a per-warp shared staging tile so that each load
    // instruction covers two 128-byte column segments instead of 32 columns'
    // lines (the per-thread column walk was L1-tag bound: ~7 us per launch).
    int bad = 0;
    {
        double* stg = X + warp * (kWarp * kStagePitch);
        const int half = lane >> 4, r = lane & 15;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            const int jw = c * kT + warp * kWarp;  // this warp's first column
#pragma unroll
            for (int r0 = 0; r0 < ROWS; r0 += kStageRows) {
#pragma unroll
                for (int it = 0; it < kWarp / 2; ++it) {
                    const int cl = 2 * it + half, j = jw + cl, i = r0 + r;
                    double v = 0.0;
                    if (j < n && i < rows) v = Y[static_cast<size_t>(j) * p.ldy + i];
                    bad |= !isfinite(v);
                    stg[cl * kStagePitch + r] = v;
                }
                __syncwarp();
#pragma unroll
                for (int u = 0; u < kStageRows; ++u)
                    if (r0 + u < ROWS) w[c][r0 + u] = stg[lane * kStagePitch + u];
                __syncwarp();
            }
        }
    }
    for (int j = tid; j < n; j += kT) {
        perm[j] = j;
        posof[j] = j;
    }
    bad = __syncthreads_or(bad);
    if (bad) {
        finish_error(SPID_NON_FINITE_INPUT);
        return;
    }
    if (p.pre_status != SPID_OK) {
        finish_error(p.pre_status);
        return;
    }

    // ---- initial norms / max_init (qr.cpp:47-51) -----------------------------
    double lmax = 0.0;
#pragma unroll
    for (int c = 0; c < CPT; ++c) {
        const int j = tid + c * kT;
        if (j < n) {
            // rows >= `rows` are zero padding: every running sum starts at +0.0
            // and can never become -0.0 (x + (-x) rounds to +0.0), so the
            // padded +0.0 terms leave each sum bit-identical to the
            // reference's shorter loop -- and the loops stay branch-free.
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < ROWS; ++i) s = add_rn(s, mul_rn(w[c][i], w[c][i]));
            const double v = sqrt(s);
            nrm[j] = v;
            colsq[j] = s;
            lmax = fmax(lmax, v);
        }
    }
    lmax = warp_max(lmax);
    if (lane == 0) red_v[warp] = lmax;
    __syncthreads();
    if (tid == 0) {
        double m = 0.0;
        for (int k = 0; k < kT / kWarp; ++k) m = fmax(m, red_v[k]);
        sh.max_init = m;
        if (p.mode == RULE_BLOCKED) sh.yfro = sqrt(sum_in_order(colsq, 0, n));
    }
    __syncthreads();
    const double max_init = sh.max_init;
    if (max_init < kZeroFloor) {
        finish_error(SPID_ZERO_MATRIX);
        return;
    }

    // ---- greedy pivoting loop (qr.cpp:61-106) ---------------------------------
    int rank = 0;
    const int step_limit = static_cast<int>(p.step_limit);
    bool alive[CPT];  // column not yet selected (position >= s), kept in registers
#pragma unroll
    for (int c = 0; c < CPT; ++c) alive[c] = tid + c * kT < n;
    for (int s = 0; s < step_limit; ++s) {
        // integer keys (norm_key): the argmax stays off the FP64 pipe
        long long bk = norm_key(-1.0);
        int bi = 0x7fffffff;
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            const int j = tid + c * kT;
            if (alive[c]) {
                const long long kj = norm_key(nrm[j]);
                if (key_better_k(kj, j, bk, bi)) {
                    bk = kj;
                    bi = j;
                }
            }
        }
        warp_argmax_k(bk, bi);
        if (lane == 0) {
            red_k[warp] = bk;
            red_i[warp] = bi;
        }
        __syncthreads();
        // every thread reduces the 8 warp partials in the same order (a total
        // order, so the same winner); no serial section, no broadcast barrier
        long long vk = red_k[0];
        int ix = red_i[0];
#pragma unroll
        for (int k = 1; k < kT / kWarp; ++k)
            if (key_better_k(red_k[k], red_i[k], vk, ix)) {
                vk = red_k[k];
                ix = red_i[k];
            }
        const double v = __longlong_as_double(vk);
        int stop = 0;
        if (p.mode == RULE_TOL && v <= p.tol * max_init) stop = 1;  // qr.cpp:74-76
        if (p.mode == RULE_BLOCKED && s > 0 && s % p.kstep == 0) {
            // residual_fro after s steps in position order (qr.cpp:111-115):
            // the squares in parallel into position order, their serial sum
            // by one thread, broadcast
            for (int j = tid; j < n; j += kT)
                if (posof[j] >= s) colsq[posof[j]] = mul_rn(nrm[j], nrm[j]);
            __syncthreads();
            if (tid == 0) sh.flag = sqrt(sum_in_order(colsq, s, n)) <= p.tol * sh.yfro;
            __syncthreads();
            if (sh.flag) stop = 1;
        }
        if (!stop && v < kCollapseRel * max_init)  // qr.cpp:77-81
            stop = (p.mode == RULE_FIXED && p.strict) ? 2 : 1;
        if (stop) {
            if (stop == 2) {
                finish_error(SPID_RANK_UNREACHABLE);
                return;
            }
            break;
        }
        if (tid == 0) {  // position bookkeeping (qr.cpp:83-87), read only after the loop
            const int ps = posof[ix], cs = perm[s];
            perm[s] = ix;
            perm[ps] = cs;
            posof[ix] = s;
            posof[cs] = ps;
            R[static_cast<size_t>(s) * n + ix] = v;  // qr.cpp:89-90
            X[s * n + ix] = v;
            diag[s] = v;
        }
        const int pc = ix;
        const double pn = v;
        // the owner publishes its column; `rows` threads normalise it in
        // parallel, q_s = w_s / R(s,s) (qr.cpp:91-92)
        if ((pc % kT) == tid) {
            const int cc = pc / kT;
#pragma unroll
            for (int c = 0; c < CPT; ++c)
                if (c == cc) {
                    alive[c] = false;
#pragma unroll
                    for (int i = 0; i < ROWS; ++i) qbuf[i] = w[c][i];  // zero padding past rows
                }
        }
        __syncthreads();
        if (tid < rows) {
            const double q = div_rn(qbuf[tid], pn);
            qbuf[tid] = q;
            if (p.Qout) p.Qout[static_cast<size_t>(b) * rows * p.kcap + static_cast<size_t>(s) * rows + tid] = q;
        }
        __syncthreads();
        // two-pass MGS (qr.cpp:94-102); the next fresh norm is accumulated in pass 2
#pragma unroll
        for (int c = 0; c < CPT; ++c) {
            const int j = tid + c * kT;
            if (alive[c]) {
                // q is re-read (16-byte broadcast loads) in every pass
                // instead of being cached across passes (the compiler fence
                // between passes): keeps the register budget to the column
                // itself, while inside a pass the loads are ordinary reads
                // the compiler issues ahead of the dependent chain. Rows past
                // `rows` are +0.0 in both q and w and stay +0.0 (0 - r*0 =
                // +0), so the padded terms add +0.0 to sums that cannot be
                // -0.0: bit-neutral, and the loops carry no per-element
                // branches.
                double r1 = 0.0;
#pragma unroll
                for (int i = 0; i < ROWS; i += 2) {
                    if (!kFree && i % kGrp == 0 && i >= rows) break;
                    const double2 q = q2[i / 2];
                    r1 = add_rn(r1, mul_rn(q.x, w[c][i]));
                    r1 = add_rn(r1, mul_rn(q.y, w[c][i + 1]));
                }
                asm volatile("" ::: "memory");
                double r2 = 0.0;
#pragma unroll
                for (int i = 0; i < ROWS; i += 2) {
                    if (!kFree && i % kGrp == 0 && i >= rows) break;
                    const double2 q = q2[i / 2];
                    const double v0 = sub_rn(w[c][i], mul_rn(r1, q.x));
                    w[c][i] = v0;
                    r2 = add_rn(r2, mul_rn(q.x, v0));
                    const double v1 = sub_rn(w[c][i + 1], mul_rn(r1, q.y));
                    w[c][i + 1] = v1;
                    r2 = add_rn(r2, mul_rn(q.y, v1));
                }
                asm volatile("" ::: "memory");
                double nn = 0.0;
#pragma unroll
                for (int i = 0; i < ROWS; i += 2) {
                    if (!kFree && i % kGrp == 0 && i >= rows) break;
                    const double2 q = q2[i / 2];
                    const double v0 = sub_rn(w[c][i], mul_rn(r2, q.x));
                    w[c][i] = v0;
                    nn = add_rn(nn, mul_rn(v0, v0));
                    const double v1 = sub_rn(w[c][i + 1], mul_rn(r2, q.y));
                    w[c][i + 1] = v1;
                    nn = add_rn(nn, mul_rn(v1, v1));
                }
                const double rs = add_rn(r1, r2);
                R[static_cast<size_t>(s) * n + j] = rs;  // global: the R output
                X[s * n + j] = rs;                       // shared: R11 and the solve
                nrm[j] = sqrt(nn);
            }
        }
        rank = s + 1;
        // (the next step's first __syncthreads orders nrm/qbuf reuse)
    }
    __syncthreads();
    if (rank == 0) {  // qr.cpp:108-109
        finish_error(SPID_ZERO_MATRIX);
        return;
    }

    // ---- residual_fro (qr.cpp:111-115), singular pivots (qr.cpp:135-140) ------
    // the squares in parallel, stored in position order; their sum in
    // position order by one thread
    for (int j = tid; j < n; j += kT) colsq[posof[j]] = mul_rn(nrm[j], nrm[j]);
    __syncthreads();
    if (tid == 0) {
        const double rsq = sum_in_order(colsq, rank, n);
        p.resid[b] = sqrt(rsq);
        double max_diag = 0.0;
        for (int t = 0; t < rank; ++t) max_diag = fmax(max_diag, fabs(diag[t]));
        int sing = 0;
        for (int t = 0; t < rank; ++t)
            if (fabs(diag[t]) < 1e-14 * max_diag || max_diag == 0.0) sing = 1;
        sh.flag = sing;
    }
    __syncthreads();
    if (sh.flag && rank < n) {
        finish_error(SPID_SINGULAR_PIVOT);
        return;
    }

    // ---- coefficients (id.cpp:9-28, back substitution qr.cpp:143-149) ---------
    // R(s, col) is in X[s][col] since the pivot loop
    for (int e = tid; e < rank * rank; e += kT) {
        const int ii = e / rank, jj = e % rank;
        r11[e] = jj >= ii ? X[ii * n + perm[jj]] : 0.0;
    }
    __syncthreads();
    double* C = p.C + static_cast<size_t>(b) * p.strideC;
    const int kcap = static_cast<int>(p.kcap);
    int nonfinite = 0;
    for (int j = tid; j < n; j += kT) {
        double* cj = C + static_cast<size_t>(j) * kcap;
        const int pj = posof[j];
        if (pj < rank) {
            for (int i = 0; i < rank; ++i) cj[i] = (i == pj) ? 1.0 : 0.0;
            continue;
        }
        for (int ii = rank - 1; ii >= 0; --ii) {
            double sum = X[ii * n + j];
            const double* rrow = r11 + ii * rank;
#pragma unroll 4
            for (int jj = ii + 1; jj < rank; ++jj) sum = sub_rn(sum, mul_rn(rrow[jj], X[jj * n + j]));
            const double x = div_rn(sum, rrow[ii]);
            X[ii * n + j] = x;
            nonfinite |= !isfinite(x);
        }
        for (int i = 0; i < rank; ++i) cj[i] = X[i * n + j];
    }
    nonfinite = __syncthreads_or(nonfinite);
    if (nonfinite) {
        finish_error(SPID_NON_FINITE_COEFFS);
        return;
    }
    int64_t* idx = p.indices + static_cast<size_t>(b) * kcap;
    for (int t = tid; t < rank; t += kT) idx[t] = perm[t];
    if (p.pivots)
        for (int pos = tid; pos < n; pos += kT) p.pivots[static_cast<size_t>(b) * n + pos] = perm[pos];
    if (p.Rout) {
        double* Ro = p.Rout + static_cast<size_t>(b) * kcap * n;
        for (int e = tid; e < rank * n; e += kT) {
            const int i = e % rank, pos = e / rank;
            Ro[static_cast<size_t>(pos) * kcap + i] = pos < i ? 0.0 : R[static_cast<size_t>(i) * n + perm[pos]];
        }
    }
    if (tid == 0) {
        p.rank[b] = rank;
        p.status[b] = SPID_OK;
    }
}

size_t reg_smem(int64_t n, int64_t cap) {
    const size_t xr = sizeof(double) * (cap * n + cap * cap);
    return sizeof(double) * (2 * n + cap) + sizeof(int) * 2 * n + 16 + (xr > kStageBytes ? xr : kStageBytes);
}

template <int ROWS, int CPT>
cudaError_t go(const CpqrParams& p, cudaStream_t stream) {
    const size_t smem = reg_smem(p.n, p.step_cap);
    auto kern = cpqr_reg_kernel<ROWS, CPT>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    kern<<<static_cast<unsigned>(p.batch), kT, smem, stream>>>(p);
    return cudaGetLastError();
}

template <int CPT>
cudaError_t by_rows(const CpqrParams& p, cudaStream_t stream) {
    if (p.rows <= 16) return go<16, CPT>(p, stream);
    if (p.rows <= 24) return go<24, CPT>(p, stream);
    if (p.rows <= 32) return go<32, CPT>(p, stream);
    if (p.rows <= 48) return go<48, CPT>(p, stream);
    if constexpr (CPT == 1) {
        if (p.rows <= 64) return go<64, CPT>(p, stream);
        return go<80, CPT>(p, stream);
    }
    return cudaErrorNotSupported;
}

}  // namespace

bool cpqr_reg_supported(int64_t rows, int64_t n, int64_t step_cap) {
    if (rows < 1 || rows > 80 || n < 1 || n > 512) return false;
    if (n > 256 && rows > 48) return false;  // two register columns of <= 48 rows
    return reg_smem(n, step_cap) <= 220 * 1024;
}

cudaError_t launch_cpqr_reg(const CpqrParams& p, cudaStream_t stream) {
    if (!cpqr_reg_supported(p.rows, p.n, p.step_cap)) return cudaErrorNotSupported;
    return p.n <= 256 ? by_rows<1>(p, stream) : by_rows<2>(p, stream);
}

}  // namespace spidgpu
