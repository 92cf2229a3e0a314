// api.cu -- the spidgpu C ABI (include/spidgpu.h): validation, workspace
// management, TMA descriptors and launch sequencing. No arithmetic of the
// compression path happens on the host: every reference function restated
// here runs as one of the kernels in this directory, and without a usable
// device every entry point fails (there is no CPU fallback).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/spidgpu.h"
#include "context.h"
#include "kernels.h"

using namespace spidgpu;

namespace spidgpu {

thread_local std::string g_create_error;

int fail(spidgpu_handle h, int code, const std::string& msg) {
    if (h) h->last_error = std::string(spidgpu_status_name(code)) + ": " + msg;
    return code;
}

int cuda_fail(spidgpu_handle h, cudaError_t e, const char* where) {
    return fail(h, SPID_CUDA_ERROR, std::string(where) + ": " + cudaGetErrorString(e));
}

// RankRule validation (proj/include/spid/qr.hpp:16-24) and step limits
// (proj/src/qr.cpp:22-25, 37-38, 53-54).
RuleInfo resolve_rule(const spidgpu_rank_rule* rule, int64_t rows, int64_t n, int64_t kcap) {
    RuleInfo ri;
    if (!rule) {
        ri.status = SPID_INVALID_ARGUMENT;
        return ri;
    }
    const int64_t mn = std::min(rows, n);
    switch (rule->mode) {
        case SPIDGPU_RULE_FIXED:
            if (rule->k < 1) {
                ri.status = SPID_BAD_RANK_RULE;
                return ri;
            }
            if (rule->at_most) {
                ri.step_limit = std::max<int64_t>(1, std::min(rule->k, mn));
            } else {
                ri.step_limit = rule->k;
                if (rule->k > mn) {
                    ri.pre_status = SPID_RANK_UNREACHABLE;
                    ri.step_limit = mn;
                }
            }
            break;
        case SPIDGPU_RULE_TOL:
            if (!(rule->tol > 0.0 && rule->tol < 1.0) || rule->at_most) {
                ri.status = SPID_BAD_RANK_RULE;
                return ri;
            }
            ri.step_limit = mn;
            break;
        case SPIDGPU_RULE_BLOCKED:
            if (rule->k < 1 || rule->kstep < 1 || !(rule->tol > 0.0 && rule->tol < 1.0) ||
                rule->at_most) {
                ri.status = SPID_BAD_RANK_RULE;
                return ri;
            }
            ri.step_limit = std::min(rule->k, mn);
            break;
        default:
            ri.status = SPID_BAD_RANK_RULE;
            return ri;
    }
    if (ri.pre_status == SPID_OK && kcap < ri.step_limit) ri.status = SPID_INVALID_ARGUMENT;
    return ri;
}

bool omega_ok(const spidgpu_omega* om) {
    if (!om) return false;
    if (om->mode == SPIDGPU_OMEGA_PHILOX) return true;
    return om->mode == SPIDGPU_OMEGA_EXPLICIT && om->omega != nullptr;
}

// ---- internal launch sequences (device pointers, given workspace) ----------
int do_sketch(spidgpu_handle h, Workspace& ws, const double* A, int64_t m, int64_t n, int64_t lda,
              int64_t strideA, int64_t batch, int64_t ell, const spidgpu_omega* om, double* Y,
              int64_t ldy, int64_t strideY, cudaStream_t st) {
    NvtxRange nvtx_range("spidgpu.sketch");
    if (m < 1 || n < 1 || batch < 1 || ell < 1) return fail(h, SPID_EMPTY_MATRIX, "empty sketch shape");
    if (!A || !Y || !omega_ok(om)) return fail(h, SPID_INVALID_ARGUMENT, "null pointer / omega");
    if (lda < m || ldy < ell || strideA < lda * n || strideY < ldy * (n - 1) + ell)
        return fail(h, SPID_INVALID_ARGUMENT, "leading dimension / stride too small");
    if ((lda % 2) || (strideA % 2) || (reinterpret_cast<uintptr_t>(A) % 16))
        return fail(h, SPID_SHAPE_UNSUPPORTED, "TMA needs 16-byte aligned A, even lda and strideA");
    if (om->mode == SPIDGPU_OMEGA_EXPLICIT && om->ldo < ell)
        return fail(h, SPID_INVALID_ARGUMENT, "ldo < ell");
    // Philox Omega: exact integer-sliced contraction on tcgen05 (UTCIMMA,
    // HBM-bound); explicit Omega (arbitrary fp64 entries) and
    // SPIDGPU_OPT_DMMA_SKETCH: the DMMA kernel
    const bool tc = om->mode == SPIDGPU_OMEGA_PHILOX && !h->force_dmma_sketch;
    const int sms = h->sketch_sms > 0 ? h->sketch_sms : h->num_sms;
    int64_t slice = tc ? kSketchTcMaxEll : 80;
    if (tc && ell > 64 && ell <= 80) {
        // one pass as a slice-split CTA pair when clusters are available
        SketchPlan probe;
        if (!sketch_tc_make_plan(m, n, batch, ell, sms, h->sketch_pairs, h->sketch_seg_rows, &probe)) slice = 64;
    }
    if (tc && ell > slice) {
        // even passes of whole 16-row groups (ell = 100 runs as 64 + 36 -> 50 + 50)
        const int64_t passes = (ell + slice - 1) / slice;
        slice = std::min<int64_t>(16 * (((ell + passes - 1) / passes + 15) / 16), slice);
    }
    for (int64_t row0 = 0; row0 < ell; row0 += slice) {
        const int64_t ells = std::min<int64_t>(slice, ell - row0);
        SketchPlan plan;
        const bool planned = tc ? sketch_tc_make_plan(m, n, batch, ells, sms, h->sketch_pairs, h->sketch_seg_rows, &plan)
                                : sketch_make_plan(m, n, batch, ells, sms, &plan);
        if (!planned) return fail(h, SPID_SHAPE_UNSUPPORTED, "no sketch plan");
        CK(h, ws.partial.ensure(plan.partial_elems * sizeof(double), st));
        CUtensorMap tmap;
        cuuint64_t gdim[3] = {static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(n),
                              static_cast<cuuint64_t>(batch)};
        cuuint64_t gstride[2] = {static_cast<cuuint64_t>(lda) * 8,
                                 static_cast<cuuint64_t>(strideA) * 8};
        cuuint32_t box[3] = {16, static_cast<cuuint32_t>(plan.nt), 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult cr = h->encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(A),
                                gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS)
            return fail(h, SPID_SHAPE_UNSUPPORTED, "cuTensorMapEncodeTiled failed: " + std::to_string(cr));
        SketchParams p{};
        p.A = A;
        p.m = m;
        p.n = n;
        p.lda = lda;
        p.strideA = strideA;
        p.batch = batch;
        p.ell = ells;
        p.row0 = row0;
        p.omega_mode = om->mode;
        p.omega = om->omega;
        p.ldo = om->ldo;
        p.stride_o = om->stride;
        p.seed = om->seed;
        p.sub_base = om->subdomain_base;
        p.partial = ws.partial.as<double>();
        p.Y = Y;
        p.ldy = ldy;
        p.strideY = strideY;
        CK(h, tc ? launch_sketch_tc(p, plan, &tmap, st) : launch_sketch(p, plan, &tmap, st));
        h->launches += 2;
    }
    return SPID_OK;
}

int do_cpqr(spidgpu_handle h, Workspace& ws, const double* Y, int64_t rows, int64_t n, int64_t ldy,
            int64_t strideY, int64_t batch, const spidgpu_rank_rule* rule, int64_t kcap,
            int64_t* indices, double* C, int64_t strideC, int64_t* rank, double* resid,
            int32_t* status, int64_t* pivots, double* R, double* Q, cudaStream_t st) {
    NvtxRange nvtx_range("spidgpu.cpqr");
    if (rows < 1 || n < 1 || batch < 1) return fail(h, SPID_EMPTY_MATRIX, "empty matrix");
    if (!Y || !indices || !C || !rank || !resid || !status)
        return fail(h, SPID_INVALID_ARGUMENT, "null pointer");
    if (ldy < rows || strideC < kcap * (n - 1) + 1)
        return fail(h, SPID_INVALID_ARGUMENT, "leading dimension too small");
    if (n > (1 << 24) || rows > (1 << 24) || rows * n > (int64_t(1) << 31))
        return fail(h, SPID_SHAPE_UNSUPPORTED, "matrix too large for the CPQR kernel");
    RuleInfo ri = resolve_rule(rule, rows, n, kcap);
    if (ri.status) return fail(h, ri.status, "rank rule");
    const int64_t step_cap = std::max<int64_t>(1, ri.step_limit);
    const bool reg = cpqr_reg_supported(rows, n, step_cap) && !h->force_generic_cpqr;
    const bool w_smem = cpqr_smem_bytes(rows, n, step_cap, true) <= cpqr_max_dyn_smem();
    // W too large for shared memory: tall inputs stream it through a TMA ring
    const bool tall = !reg && !w_smem && cpqr_tall_supported(rows, n);
    // wide tall inputs: each subdomain's columns over a cluster of two
    const bool pair = tall && h->tall_pairs && cpqr_pair_supported(rows, n, rule->mode, step_cap);
    const int npad = pair ? 2 * cpqr_pair_half(n) : tall ? cpqr_tall_npad(n) : static_cast<int>(n);
    CK(h, ws.rws.ensure(sizeof(double) * batch * step_cap * n, st));
    if (!reg && !w_smem) {
        CK(h, ws.wws.ensure(sizeof(double) * batch * rows * npad, st));
        CK(h, ws.r11ws.ensure(sizeof(double) * batch * (pair ? 2 : 1) * step_cap * step_cap, st));
    }
    CpqrParams p{};
    p.Y = Y;
    p.rows = rows;
    p.n = n;
    p.ldy = ldy;
    p.strideY = strideY;
    p.batch = batch;
    p.mode = rule->mode;
    p.strict = rule->at_most ? 0 : 1;
    p.kstep = rule->kstep;
    p.tol = rule->tol;
    p.step_limit = ri.step_limit;
    p.step_cap = step_cap;
    p.kcap = kcap;
    p.pre_status = ri.pre_status;
    p.npad = npad;
    p.w_ws = ws.wws.as<double>();
    p.r_ws = ws.rws.as<double>();
    p.r11_ws = ws.r11ws.as<double>();
    p.indices = indices;
    p.C = C;
    p.strideC = strideC;
    p.rank = rank;
    p.resid = resid;
    p.status = status;
    p.pivots = pivots;
    p.Rout = R;
    p.Qout = Q;
    if (reg) {
        // sketch-sized inputs (33-48 rows, 128 < n <= 256): columns over a
        // CTA pair where it measured faster (tools/exp_regpair_ab.py), i.e.
        // while the pairs fit one wave
        const bool rpair = h->reg_pairs && 2 * batch <= h->num_sms &&
                           cpqr_regpair_supported(rows, n, rule->mode, step_cap);
        CK(h, rpair ? launch_cpqr_regpair(p, st) : launch_cpqr_reg(p, st));
    } else if (tall) {
        CUtensorMap wmap;
        cuuint64_t gdim[3] = {static_cast<cuuint64_t>(npad), static_cast<cuuint64_t>(rows),
                              static_cast<cuuint64_t>(batch)};
        cuuint64_t gstride[2] = {static_cast<cuuint64_t>(npad) * 8, static_cast<cuuint64_t>(rows) * npad * 8};
        cuuint32_t box[3] = {static_cast<cuuint32_t>(pair ? cpqr_pair_half(n) : npad),
                             static_cast<cuuint32_t>(pair ? cpqr_pair_ring_rows(n) : cpqr_tall_ring_rows(n)), 1};
        cuuint32_t estr[3] = {1, 1, 1};
        CUresult cr = h->encode(&wmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, ws.wws.ptr, gdim, gstride, box, estr,
                                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS)
            return fail(h, SPID_SHAPE_UNSUPPORTED, "cuTensorMapEncodeTiled (CPQR ring) failed: " + std::to_string(cr));
        CUtensorMap pmap;  // pairs: the pivot column pair beside each first-sweep chunk
        if (pair) {
            cuuint32_t pbox[3] = {2, box[1], 1};
            cr = h->encode(&pmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, ws.wws.ptr, gdim, gstride, pbox, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (cr != CUDA_SUCCESS)
                return fail(h, SPID_SHAPE_UNSUPPORTED, "cuTensorMapEncodeTiled (CPQR pivot column) failed: " +
                                                           std::to_string(cr));
        }
        CK(h, pair ? launch_cpqr_pair(p, &wmap, &pmap, st) : launch_cpqr_tall(p, &wmap, st));
    } else {
        CK(h, launch_cpqr(p, w_smem, st));
    }
    h->launches += 1;
    return SPID_OK;
}

int do_gather(spidgpu_handle h, const double* A, int64_t m, int64_t n, int64_t lda, int64_t strideA,
              int64_t batch, const int64_t* indices, int64_t kcap, const int64_t* rank,
              double* skel, int64_t ldskel, int64_t strideS, cudaStream_t st) {
    NvtxRange nvtx_range("spidgpu.gather");
    if (!A || !indices || !rank || !skel) return fail(h, SPID_INVALID_ARGUMENT, "null pointer");
    if (m < 1 || n < 1 || batch < 1 || kcap < 1) return fail(h, SPID_EMPTY_SELECTION, "empty gather");
    if (lda < m || ldskel < m) return fail(h, SPID_INVALID_ARGUMENT, "leading dimension too small");
    // out-of-range indices (select_columns' IndexOutOfRange, dense_matrix.cpp:75)
    // leave their columns unwritten and are reported through the deferred status
    CK(h, launch_gather_cols(A, m, lda, strideA, batch, indices, kcap, rank, n, skel, ldskel,
                             strideS, h->dev_status, st));
    h->launches += 1;
    return SPID_OK;
}

int do_verify(spidgpu_handle h, Workspace& ws, const double* A, int64_t m, int64_t n, int64_t lda,
              int64_t strideA, int64_t batch, const double* skel, int64_t ldskel, int64_t strideS,
              const double* C, int64_t kcap, int64_t strideC, const int64_t* rank, double* err2,
              double* ref2, cudaStream_t st) {
    NvtxRange nvtx_range("spidgpu.verify");
    if (!A || !skel || !C || !rank || !err2 || !ref2)
        return fail(h, SPID_INVALID_ARGUMENT, "null pointer");
    if (kcap > 80) return fail(h, SPID_SHAPE_UNSUPPORTED, "verify supports rank <= 80");
    VerifyParams p{};
    p.A = A;
    p.m = m;
    p.n = n;
    p.lda = lda;
    p.strideA = strideA;
    p.batch = batch;
    p.skel = skel;
    p.ldskel = ldskel;
    p.strideS = strideS;
    p.C = C;
    p.kcap = kcap;
    p.strideC = strideC;
    p.rank = rank;
    p.err2 = err2;
    p.ref2 = ref2;
    // TMA path: both operands need 16-byte aligned bases and even leading dims
    const bool tma_ok = (lda % 2 == 0) && (strideA % 2 == 0) && (ldskel % 2 == 0) &&
                        (strideS % 2 == 0) && (reinterpret_cast<uintptr_t>(A) % 16 == 0) &&
                        (reinterpret_cast<uintptr_t>(skel) % 16 == 0) && kcap >= 1;
    VerifyPlan plan;
    if (tma_ok && verify_make_plan(m, n, batch, kcap, h->num_sms, &plan)) {
        CUtensorMap tA, tS;
        cuuint32_t estr[3] = {1, 1, 1};
        cuuint64_t gA[3] = {static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(n),
                            static_cast<cuuint64_t>(batch)};
        cuuint64_t sA[2] = {static_cast<cuuint64_t>(lda) * 8, static_cast<cuuint64_t>(strideA) * 8};
        cuuint32_t bA[3] = {16, static_cast<cuuint32_t>(plan.nt), 1};
        cuuint64_t gS[3] = {static_cast<cuuint64_t>(m), static_cast<cuuint64_t>(kcap),
                            static_cast<cuuint64_t>(batch)};
        cuuint64_t sS[2] = {static_cast<cuuint64_t>(ldskel) * 8, static_cast<cuuint64_t>(strideS) * 8};
        cuuint32_t bS[3] = {16, static_cast<cuuint32_t>(4 * plan.ks), 1};
        CUresult c1 = h->encode(&tA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(A), gA,
                                sA, bA, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        CUresult c2 = h->encode(&tS, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(skel),
                                gS, sS, bS, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (c1 == CUDA_SUCCESS && c2 == CUDA_SUCCESS) {
            CK(h, ws.vpart.ensure(sizeof(double) * plan.part_elems, st));
            CK(h, launch_verify_tma(p, plan, &tA, &tS, ws.vpart.as<double>(), st));
            h->launches += 2;
            return SPID_OK;
        }
    }
    p.nblk = verify_row_blocks(m);  // generic slab path (odd leading dims, unaligned bases)
    CK(h, ws.vpart.ensure(sizeof(double) * 2 * batch * p.nblk, st));
    p.part = ws.vpart.as<double>();
    CK(h, launch_verify(p, h->num_sms, st));
    h->launches += 2;
    return SPID_OK;
}

int do_compress(spidgpu_handle h, Workspace& ws, const double* A, int64_t m, int64_t n, int64_t lda,
                int64_t strideA, int64_t batch, int64_t ell, const spidgpu_omega* om,
                const spidgpu_rank_rule* rule, int64_t kcap, int64_t* indices, double* C,
                int64_t* rank, double* resid, int32_t* status, double* skel, double* Y,
                cudaStream_t st) {
    double* y = Y;
    if (!y) {
        CK(h, ws.ybuf.ensure(sizeof(double) * batch * ell * n, st));
        y = ws.ybuf.as<double>();
    }
    int rc = do_sketch(h, ws, A, m, n, lda, strideA, batch, ell, om, y, ell, ell * n, st);
    if (rc) return rc;
    rc = do_cpqr(h, ws, y, ell, n, ell, ell * n, batch, rule, kcap, indices, C, kcap * n, rank,
                 resid, status, nullptr, nullptr, nullptr, st);
    if (rc) return rc;
    if (skel) rc = do_gather(h, A, m, n, lda, strideA, batch, indices, kcap, rank, skel, m, m * kcap, st);
    return rc;
}

// ---- host-API helpers ---------------------------------------------------------
bool all_finite_host_free() { return true; }

// Copy an m x n host matrix into a device buffer with an even leading
// dimension (TMA row pitch must be a multiple of 16 bytes).
int matrix_to_dev(spidgpu_handle h, DevBuf& buf, const double* a, int64_t m, int64_t n,
                  int64_t* lda_out, cudaStream_t st) {
    const int64_t lda = (m + 1) & ~int64_t(1);
    CK(h, buf.ensure(sizeof(double) * lda * n, st));
    CK(h, cudaMemcpy2DAsync(buf.ptr, sizeof(double) * lda, a, sizeof(double) * m,
                            sizeof(double) * m, n, cudaMemcpyHostToDevice, st));
    *lda_out = lda;
    return SPID_OK;
}

int finish_single(spidgpu_handle h, Workspace& ws, int64_t m, int64_t n, int64_t kcap,
                  const double* a_dev, int64_t lda, int64_t* indices, double* coeffs,
                  double* skeleton, int64_t* rank_out, double* resid_out, cudaStream_t st) {
    int32_t status = 0;
    int64_t rank = 0;
    double resid = 0.0;
    CK(h, cudaMemcpyAsync(&status, ws.status.ptr, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(h, cudaMemcpyAsync(&rank, ws.rank.ptr, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(h, cudaMemcpyAsync(&resid, ws.resid.ptr, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(h, cudaStreamSynchronize(st));
    if (status) return fail(h, status, "column ID failed on the device");
    if (skeleton && rank > 0) {
        CK(h, ws.skel.ensure(sizeof(double) * m * kcap, st));
        int rc = do_gather(h, a_dev, m, n, lda, lda * n, 1, ws.idx.as<int64_t>(), kcap,
                           ws.rank.as<int64_t>(), ws.skel.as<double>(), m, m * kcap, st);
        if (rc) return rc;
        CK(h, cudaMemcpyAsync(skeleton, ws.skel.ptr, sizeof(double) * m * rank,
                              cudaMemcpyDeviceToHost, st));
    }
    if (indices)
        CK(h, cudaMemcpyAsync(indices, ws.idx.ptr, sizeof(int64_t) * rank, cudaMemcpyDeviceToHost, st));
    if (coeffs)
        CK(h, cudaMemcpyAsync(coeffs, ws.coeffs.ptr, sizeof(double) * kcap * n,
                              cudaMemcpyDeviceToHost, st));
    CK(h, cudaStreamSynchronize(st));
    if (rank_out) *rank_out = rank;
    if (resid_out) *resid_out = resid;
    return SPID_OK;
}

// Host SplitMix64 for the synthetic-field mode tables (same recurrence as
// proj/include/spid/rng.hpp:16-22).
struct Mix64 {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9E3779B97F4A7C15ULL);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
        return z ^ (z >> 31);
    }
    double unit() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
};

std::vector<double> make_modes(uint64_t seed, int count, double kmin, double kmax, double amp0) {
    std::vector<double> out;
    Mix64 rng{seed};
    const int K = static_cast<int>(std::floor(kmax));
    const double two_pi = 6.283185307179586;
    for (int m = 0; m < count; ++m) {
        double kx, ky, kz, k2;
        do {
            kx = std::floor(rng.unit() * (2 * K + 1)) - K;
            ky = std::floor(rng.unit() * (2 * K + 1)) - K;
            kz = std::floor(rng.unit() * (2 * K + 1)) - K;
            k2 = kx * kx + ky * ky + kz * kz;
        } while (k2 == 0.0 || k2 > kmax * kmax || k2 < kmin * kmin);
        const double kn = std::sqrt(k2);
        const double amp = amp0 * std::pow(kn, -5.0 / 3.0);
        const double phi = two_pi * rng.unit(), phip = two_pi * rng.unit();
        double d[3], dn;
        do {  // random direction orthogonal to kappa (divergence-free mode)
            d[0] = 2 * rng.unit() - 1;
            d[1] = 2 * rng.unit() - 1;
            d[2] = 2 * rng.unit() - 1;
            const double pr = (d[0] * kx + d[1] * ky + d[2] * kz) / k2;
            d[0] -= pr * kx;
            d[1] -= pr * ky;
            d[2] -= pr * kz;
            dn = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        } while (dn < 1e-3);
        const double md[9] = {kx, ky, kz, amp, phi, phip, d[0] / dn, d[1] / dn, d[2] / dn};
        out.insert(out.end(), md, md + 9);
    }
    return out;
}

}  // namespace spidgpu

namespace spidgpu {

// ---- SPID grid specs ----------------------------------------------------------------
// Validation of SubsampleSpec::strided / GridGeom::structured (grid.cpp:7-20, 62-75).
int spec_to_dev(spidgpu_handle h, const spidgpu_grid_spec* sp, GridSpecDev* g, int64_t* P,
                int64_t* Pc, int min_dim, bool lift) {
    if (!sp) return fail(h, SPID_INVALID_ARGUMENT, "null grid spec");
    if (sp->naxes < 1 || sp->naxes > 3) return fail(h, SPID_BAD_GRID_GEOM, "structured grids have 1 to 3 axes");
    if (sp->nqoi < 1) return fail(h, SPID_BAD_SUBSAMPLE_SPEC, "nqoi must be >= 1");
    g->naxes = sp->naxes;
    g->incl = sp->include_boundary != 0;
    g->nqoi = sp->nqoi;
    *P = 1;
    *Pc = 1;
    for (int ax = 0; ax < 3; ++ax) {
        if (ax < sp->naxes) {
            if (sp->dims[ax] < min_dim || sp->dims[ax] > (1 << 20))
                return fail(h, SPID_BAD_GRID_GEOM, min_dim > 1 ? "each structured axis needs at least 2 points"
                                                               : "block axis needs at least 1 point");
            if (sp->strides[ax] < 1) return fail(h, SPID_BAD_SUBSAMPLE_SPEC, "strides must be >= 1");
            g->dims[ax] = static_cast<int>(sp->dims[ax]);
            g->strides[ax] = static_cast<int>(sp->strides[ax]);
            g->periodic[ax] = sp->periodic[ax] != 0;
            const int64_t base = (sp->dims[ax] + sp->strides[ax] - 1) / sp->strides[ax];
            const bool extra = g->incl && !g->periodic[ax] && (base - 1) * sp->strides[ax] != sp->dims[ax] - 1;
            // interp.cpp:25-29: fine points past the last coarse point of a
            // non-periodic axis cannot be lifted (raised when M is built)
            if (lift && !g->periodic[ax] && !extra && (base - 1) * sp->strides[ax] != sp->dims[ax] - 1)
                return fail(h, SPID_EXTRAPOLATION_REQUIRED,
                            "fine point beyond the last coarse point on a non-periodic axis");
            *P *= sp->dims[ax];
            *Pc *= base + (extra ? 1 : 0);
        } else {
            g->dims[ax] = 1;
            g->strides[ax] = 1;
            g->periodic[ax] = false;
        }
    }
    return SPID_OK;
}

// SubsampleSpec::row_indices (grid.cpp:108-130), axis 0 fastest, per QoI block.
std::vector<int64_t> spec_rows(const GridSpecDev& g, int64_t P) {
    std::vector<int64_t> axes[3];
    for (int ax = 0; ax < 3; ++ax) {
        if (ax >= g.naxes) {
            axes[ax] = {0};
            continue;
        }
        for (int64_t i = 0; i < g.dims[ax]; i += g.strides[ax]) axes[ax].push_back(i);
        if (g.incl && !g.periodic[ax] && axes[ax].back() != g.dims[ax] - 1)
            axes[ax].push_back(g.dims[ax] - 1);
    }
    std::vector<int64_t> rows;
    const int64_t d0 = g.dims[0], d1 = g.naxes > 1 ? g.dims[1] : 1;
    for (int q = 0; q < g.nqoi; ++q)
        for (int64_t i2 : axes[2])
            for (int64_t i1 : axes[1])
                for (int64_t i0 : axes[0]) rows.push_back(q * P + i0 + d0 * i1 + d0 * d1 * i2);
    return rows;
}

}  // namespace spidgpu

// =====================================================================
extern "C" {

const char* spidgpu_status_name(int status) {
    switch (status) {
        case SPID_OK: return "Ok";
        case SPID_NON_FINITE_INPUT: return "NonFiniteInput";
        case SPID_RANK_UNREACHABLE: return "RankUnreachable";
        case SPID_ZERO_MATRIX: return "ZeroMatrix";
        case SPID_SINGULAR_PIVOT: return "SingularPivot";
        case SPID_DIMENSION_MISMATCH: return "DimensionMismatch";
        case SPID_NON_FINITE_COEFFS: return "NonFiniteCoeffs";
        case SPID_BAD_RANK_RULE: return "BadRankRule";
        case SPID_EMPTY_MATRIX: return "EmptyMatrix";
        case SPID_EMPTY_SELECTION: return "EmptySelection";
        case SPID_INDEX_OUT_OF_RANGE: return "IndexOutOfRange";
        case SPID_GEOMETRY_MISMATCH: return "GeometryMismatch";
        case SPID_ZERO_REFERENCE: return "ZeroReference";
        case SPID_ZERO_DENOMINATOR: return "ZeroDenominator";
        case SPID_BAD_SUBSAMPLE_SPEC: return "BadSubsampleSpec";
        case SPID_EMPTY_SKETCH: return "EmptySketch";
        case SPID_EXTRAPOLATION_REQUIRED: return "ExtrapolationRequired";
        case SPID_BAD_GRID_GEOM: return "BadGridGeom";
        case SPID_BLOCK_TOO_SMALL: return "BlockTooSmall";
        case SPID_BAD_MAGIC: return "BadMagic";
        case SPID_VERSION_UNSUPPORTED: return "VersionUnsupported";
        case SPID_TRUNCATED_PAYLOAD: return "TruncatedPayload";
        case SPID_CHECKSUM_MISMATCH: return "ChecksumMismatch";
        case SPID_COVERAGE_GAP: return "CoverageGap";
        case SPID_UNSTRUCTURED_NO_INTERP: return "UnstructuredNoInterp";
        case SPID_BAD_STREAM_CONFIG: return "BadStreamConfig";
        case SPID_SHORT_STREAM: return "ShortStream";
        case SPID_EMPTY_LOG: return "EmptyLog";
        case SPID_CUDA_ERROR: return "CudaError";
        case SPID_INVALID_ARGUMENT: return "InvalidArgument";
        case SPID_SHAPE_UNSUPPORTED: return "ShapeUnsupported";
        case SPID_NO_DEVICE: return "NoDevice";
        default: return "Unknown";
    }
}

int spidgpu_abi_version(void) { return SPIDGPU_ABI_VERSION; }

int spidgpu_create(int device, spidgpu_handle* out) {
    if (!out) return SPID_INVALID_ARGUMENT;
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
        cudaGetLastError();
        return SPID_NO_DEVICE;
    }
    if (device < 0 || device >= count) return SPID_INVALID_ARGUMENT;
    if (cudaSetDevice(device) != cudaSuccess) return SPID_CUDA_ERROR;
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return SPID_CUDA_ERROR;
    if (prop.major < 10) return SPID_NO_DEVICE;  // built for sm_100a only
    auto* h = new spidgpu_context();
    h->device = device;
    h->num_sms = prop.multiProcessorCount;
    cudaDriverEntryPointQueryResult q;
    void* fn = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
            cudaSuccess ||
        !fn) {
        delete h;
        return SPID_CUDA_ERROR;
    }
    h->encode = reinterpret_cast<EncodeTiledFn>(fn);
    if (cudaMalloc(&h->dev_status, sizeof(int32_t)) != cudaSuccess ||
        cudaMemset(h->dev_status, 0, sizeof(int32_t)) != cudaSuccess) {
        delete h;
        return SPID_CUDA_ERROR;
    }
    for (int i = 0; i < 2; ++i) {
        if (cudaStreamCreateWithFlags(&h->lanes[i], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&h->ev[i], cudaEventDisableTiming) != cudaSuccess) {
            delete h;
            return SPID_CUDA_ERROR;
        }
    }
    *out = h;
    return SPID_OK;
}

int spidgpu_destroy(spidgpu_handle h) {
    if (!h) return SPID_INVALID_ARGUMENT;
    cudaSetDevice(h->device);
    cudaDeviceSynchronize();
    for (auto& w : h->ws) w.release();
    if (h->dev_status) cudaFree(h->dev_status);
    if (h->archive_pinned) cudaFreeHost(h->archive_pinned);
    if (h->upload_pinned) cudaFreeHost(h->upload_pinned);
    for (cudaEvent_t e : h->upload_ev)
        if (e) cudaEventDestroy(e);
    for (int i = 0; i < 2; ++i) {
        if (h->lanes[i]) cudaStreamDestroy(h->lanes[i]);
        if (h->ev[i]) cudaEventDestroy(h->ev[i]);
    }
    delete h;
    return SPID_OK;
}

int spidgpu_debug_counters(spidgpu_handle h, int64_t* out, int n, int reset) {
    if (!h || !out || n < 3) return SPID_INVALID_ARGUMENT;
    cudaSetDevice(h->device);
    if (sketch_tc_flush_counters(out, reset != 0)) return fail(h, SPID_CUDA_ERROR, "counter readback");
    return SPID_OK;
}

const char* spidgpu_last_error(spidgpu_handle h) { return h ? h->last_error.c_str() : ""; }

int64_t spidgpu_launch_count(spidgpu_handle h) { return h ? h->launches : 0; }

int spidgpu_set_option(spidgpu_handle h, int option, int64_t value) {
    if (!h) return SPID_INVALID_ARGUMENT;
    switch (option) {
        case SPIDGPU_OPT_GENERIC_CPQR: h->force_generic_cpqr = value != 0; return SPID_OK;
        case SPIDGPU_OPT_TALL_PAIRS: h->tall_pairs = value != 0; return SPID_OK;
        case SPIDGPU_OPT_REG_PAIRS: h->reg_pairs = value != 0; return SPID_OK;
        case SPIDGPU_OPT_DMMA_SKETCH: h->force_dmma_sketch = value != 0; return SPID_OK;
        case SPIDGPU_OPT_SKETCH_PAIRS:
            if (value < 0 || value > 2) return SPID_INVALID_ARGUMENT;
            h->sketch_pairs = static_cast<int>(value);
            return SPID_OK;
        case SPIDGPU_OPT_SKETCH_SEG_ROWS:
            if (value < 0 || value % 512 || value > 65536) return SPID_INVALID_ARGUMENT;
            h->sketch_seg_rows = value;
            return SPID_OK;
        case SPIDGPU_OPT_SKETCH_SMS:
            if (value < 0) return SPID_INVALID_ARGUMENT;
            h->sketch_sms = static_cast<int>(std::min<int64_t>(value, h->num_sms));
            return SPID_OK;
        default: return SPID_INVALID_ARGUMENT;
    }
}

// ---- batched device API ----------------------------------------------------------
int spidgpu_sketch_batched(spidgpu_handle h, const double* A, int64_t m, int64_t n, int64_t lda,
                           int64_t strideA, int64_t batch, int64_t ell, const spidgpu_omega* omega,
                           double* Y, int64_t ldy, int64_t strideY, void* stream) {
    if (!h) return SPID_INVALID_ARGUMENT;
    return do_sketch(h, h->ws[0], A, m, n, lda, strideA, batch, ell, omega, Y, ldy, strideY,
                     static_cast<cudaStream_t>(stream));
}

int spidgpu_philox_omega(spidgpu_handle h, uint64_t seed, int64_t subdomain, int64_t ell,
                         int64_t m, double* omega, int64_t ldo, void* stream) {
    if (!h || !omega || ldo < ell || ell < 1 || m < 1) return SPID_INVALID_ARGUMENT;
    CK(h, launch_philox_omega(seed, subdomain, ell, m, omega, ldo, static_cast<cudaStream_t>(stream)));
    h->launches += 1;
    return SPID_OK;
}

int spidgpu_cpqr_id_batched(spidgpu_handle h, const double* Y, int64_t rows, int64_t n,
                            int64_t ldy, int64_t strideY, int64_t batch,
                            const spidgpu_rank_rule* rule, int64_t kcap, int64_t* indices,
                            double* C, int64_t strideC, int64_t* rank, double* residual_fro,
                            int32_t* status, int64_t* pivots, double* R, double* Q, void* stream) {
    if (!h) return SPID_INVALID_ARGUMENT;
    return do_cpqr(h, h->ws[0], Y, rows, n, ldy, strideY, batch, rule, kcap, indices, C, strideC,
                   rank, residual_fro, status, pivots, R, Q, static_cast<cudaStream_t>(stream));
}

int spidgpu_gather_batched(spidgpu_handle h, const double* A, int64_t m, int64_t n, int64_t lda,
                           int64_t strideA, int64_t batch, const int64_t* indices, int64_t kcap,
                           const int64_t* rank, double* skel, int64_t ldskel, int64_t strideS,
                           void* stream) {
    if (!h) return SPID_INVALID_ARGUMENT;
    return do_gather(h, A, m, n, lda, strideA, batch, indices, kcap, rank, skel, ldskel, strideS,
                     static_cast<cudaStream_t>(stream));
}

int spidgpu_row_gather_batched(spidgpu_handle h, const double* A, int64_t m, int64_t n,
                               int64_t lda, int64_t strideA, int64_t batch, const int64_t* rows,
                               int64_t nrows, double* B, int64_t ldb, int64_t strideB,
                               void* stream) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (nrows < 1) return fail(h, SPID_EMPTY_SKETCH, "row selection is empty");
    if (!A || !rows || !B || ldb < nrows || lda < m)
        return fail(h, SPID_INVALID_ARGUMENT, "bad row gather arguments");
    CK(h, launch_gather_rows(A, m, n, lda, strideA, batch, rows, nrows, B, ldb, strideB, h->dev_status,
                             static_cast<cudaStream_t>(stream)));
    h->launches += 1;
    return SPID_OK;
}

int spidgpu_reserve(spidgpu_handle h, int64_t m, int64_t n, int64_t batch, int64_t ell, int64_t kcap) {
    if (!h || m < 1 || n < 1 || batch < 1 || ell < 1 || kcap < 1) return SPID_INVALID_ARGUMENT;
    cudaSetDevice(h->device);
    Workspace& ws = h->ws[0];
    cudaStream_t st = nullptr;
    const int sms = h->sketch_sms > 0 ? h->sketch_sms : h->num_sms;
    size_t part = 0;
    for (int64_t w : {std::min<int64_t>(ell, kSketchTcMaxEll), std::min<int64_t>(ell, 64), std::min<int64_t>(ell, 48)}) {
        SketchPlan plan;
        if (sketch_tc_make_plan(m, n, batch, w, sms, h->sketch_pairs, h->sketch_seg_rows, &plan))
            part = std::max(part, plan.partial_elems);
        if (sketch_make_plan(m, n, batch, std::min<int64_t>(w, 80), sms, &plan))
            part = std::max(part, plan.partial_elems);
    }
    CK(h, ws.partial.ensure(part * sizeof(double), st));
    CK(h, ws.rws.ensure(sizeof(double) * batch * kcap * n, st));
    VerifyPlan vp;
    if (kcap <= 80 && verify_make_plan(m, n, batch, kcap, h->num_sms, &vp))
        CK(h, ws.vpart.ensure(sizeof(double) * vp.part_elems, st));
    CK(h, cudaDeviceSynchronize());
    return SPID_OK;
}

int spidgpu_stream_status(spidgpu_handle h, void* stream) {
    if (!h) return SPID_INVALID_ARGUMENT;
    cudaSetDevice(h->device);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int32_t v = 0;
    CK(h, cudaMemcpyAsync(&v, h->dev_status, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(h, cudaMemsetAsync(h->dev_status, 0, sizeof(int32_t), st));
    CK(h, cudaStreamSynchronize(st));
    if (v) return fail(h, v, "a batched gather on this stream met an index outside the matrix");
    return SPID_OK;
}

int spidgpu_verify_batched(spidgpu_handle h, const double* A, int64_t m, int64_t n, int64_t lda,
                           int64_t strideA, int64_t batch, const double* skel, int64_t ldskel,
                           int64_t strideS, const double* C, int64_t kcap, int64_t strideC,
                           const int64_t* rank, double* err2, double* ref2, void* stream) {
    if (!h) return SPID_INVALID_ARGUMENT;
    return do_verify(h, h->ws[0], A, m, n, lda, strideA, batch, skel, ldskel, strideS, C, kcap,
                     strideC, rank, err2, ref2, static_cast<cudaStream_t>(stream));
}

int spidgpu_reconstruct_batched(spidgpu_handle h, const double* skel, int64_t m, int64_t ldskel,
                                int64_t strideS, const double* C, int64_t kcap, int64_t strideC,
                                const int64_t* rank, int64_t n, int64_t batch, double* out,
                                int64_t ldo, int64_t strideO, void* stream) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (!skel || !C || !rank || !out) return fail(h, SPID_INVALID_ARGUMENT, "null pointer");
    if (kcap > 80) return fail(h, SPID_SHAPE_UNSUPPORTED, "reconstruct supports rank <= 80");
    CK(h, launch_reconstruct(skel, m, ldskel, strideS, C, kcap, strideC, rank, n, batch, out, ldo,
                             strideO, static_cast<cudaStream_t>(stream)));
    h->launches += 1;
    return SPID_OK;
}

int spidgpu_compress_batched(spidgpu_handle h, const double* A, int64_t m, int64_t n, int64_t lda,
                             int64_t strideA, int64_t batch, int64_t ell,
                             const spidgpu_omega* omega, const spidgpu_rank_rule* rule,
                             int64_t kcap, int64_t* indices, double* C, int64_t* rank,
                             double* residual_fro, int32_t* status, double* skel, double* Y,
                             void* stream) {
    NvtxRange nvtx_range("spidgpu.compress_batched");
    if (!h) return SPID_INVALID_ARGUMENT;
    return do_compress(h, h->ws[0], A, m, n, lda, strideA, batch, ell, omega, rule, kcap, indices,
                       C, rank, residual_fro, status, skel, Y, static_cast<cudaStream_t>(stream));
}

// ---- host-buffer API ---------------------------------------------------------------
static int column_id_impl(spidgpu_handle h, const double* a, int64_t m, int64_t n,
                          const spidgpu_rank_rule* rule, int64_t kcap, int64_t* indices,
                          double* coeffs, double* skeleton, int64_t* rank, double* resid,
                          double* q, double* r, int64_t* pivots) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (m < 1 || n < 1) return fail(h, SPID_EMPTY_MATRIX, "matrix dimensions must be at least 1x1");
    if (!a) return fail(h, SPID_INVALID_ARGUMENT, "null input");
    cudaSetDevice(h->device);
    Workspace& ws = h->ws[0];
    cudaStream_t st = h->lanes[0];
    int64_t lda = 0;
    int rc = matrix_to_dev(h, ws.a, a, m, n, &lda, st);
    if (rc) return rc;
    const int64_t kc = std::max<int64_t>(kcap, 1);
    CK(h, ws.idx.ensure(sizeof(int64_t) * kc, st));
    CK(h, ws.coeffs.ensure(sizeof(double) * kc * n, st));
    CK(h, ws.rank.ensure(sizeof(int64_t), st));
    CK(h, ws.resid.ensure(sizeof(double), st));
    CK(h, ws.status.ensure(sizeof(int32_t), st));
    if (pivots) CK(h, ws.pivots.ensure(sizeof(int64_t) * n, st));
    if (r) CK(h, ws.r.ensure(sizeof(double) * kc * n, st));
    if (q) CK(h, ws.q.ensure(sizeof(double) * m * kc, st));
    CK(h, cudaMemsetAsync(ws.coeffs.ptr, 0, sizeof(double) * kc * n, st));
    if (r) CK(h, cudaMemsetAsync(ws.r.ptr, 0, sizeof(double) * kc * n, st));
    rc = do_cpqr(h, ws, ws.a.as<double>(), m, n, lda, lda * n, 1, rule, kc, ws.idx.as<int64_t>(),
                 ws.coeffs.as<double>(), kc * n, ws.rank.as<int64_t>(), ws.resid.as<double>(),
                 ws.status.as<int32_t>(), pivots ? ws.pivots.as<int64_t>() : nullptr,
                 r ? ws.r.as<double>() : nullptr, q ? ws.q.as<double>() : nullptr, st);
    if (rc) return rc;
    int64_t rk = 0;
    rc = finish_single(h, ws, m, n, kc, ws.a.as<double>(), lda, indices, coeffs, skeleton, &rk,
                       resid, st);
    if (rc) return rc;
    if (pivots) CK(h, cudaMemcpy(pivots, ws.pivots.ptr, sizeof(int64_t) * n, cudaMemcpyDeviceToHost));
    if (r) CK(h, cudaMemcpy(r, ws.r.ptr, sizeof(double) * kc * n, cudaMemcpyDeviceToHost));
    if (q) CK(h, cudaMemcpy(q, ws.q.ptr, sizeof(double) * m * kc, cudaMemcpyDeviceToHost));
    if (rank) *rank = rk;
    return SPID_OK;
}

int spidgpu_column_id(spidgpu_handle h, const double* a, int64_t m, int64_t n,
                      const spidgpu_rank_rule* rule, int64_t kcap, int64_t* indices,
                      double* coeffs, double* skeleton, int64_t* rank, double* residual_fro) {
    return column_id_impl(h, a, m, n, rule, kcap, indices, coeffs, skeleton, rank, residual_fro,
                          nullptr, nullptr, nullptr);
}

int spidgpu_qr(spidgpu_handle h, const double* a, int64_t m, int64_t n,
               const spidgpu_rank_rule* rule, int64_t kcap, double* q, double* r, int64_t* pivots,
               int64_t* rank, double* residual_fro) {
    std::vector<int64_t> idx(std::max<int64_t>(kcap, 1));
    std::vector<double> coeffs(static_cast<size_t>(std::max<int64_t>(kcap, 1)) * n);
    int rc = column_id_impl(h, a, m, n, rule, kcap, idx.data(), coeffs.data(), nullptr, rank,
                            residual_fro, q, r, pivots);
    // pivoted_mgs_qr itself never raises SingularPivot/NonFiniteCoeffs; those
    // come from the coefficient stage, which spidgpu_qr callers do not need.
    return rc;
}

int spidgpu_sub_id(spidgpu_handle h, const double* a, int64_t m, int64_t n, const int64_t* rows,
                   int64_t nrows, const spidgpu_rank_rule* rule, int64_t kcap, int64_t* indices,
                   double* coeffs, double* skeleton, int64_t* rank, double* residual_fro) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (m < 1 || n < 1) return fail(h, SPID_EMPTY_MATRIX, "matrix dimensions must be at least 1x1");
    if (!rows || nrows < 1) return fail(h, SPID_EMPTY_SKETCH, "no rows selected");
    for (int64_t i = 0; i < nrows; ++i) {  // SubsampleSpec::explicit_list checks (grid.cpp:80-84)
        if (rows[i] < 0 || rows[i] >= m) return fail(h, SPID_GEOMETRY_MISMATCH, "row index outside fine column");
        if (i > 0 && rows[i] <= rows[i - 1])
            return fail(h, SPID_BAD_SUBSAMPLE_SPEC, "row list must be strictly increasing");
    }
    cudaSetDevice(h->device);
    Workspace& ws = h->ws[0];
    cudaStream_t st = h->lanes[0];
    int64_t lda = 0;
    int rc = matrix_to_dev(h, ws.a, a, m, n, &lda, st);
    if (rc) return rc;
    rc = to_dev(h, ws.rows, rows, static_cast<size_t>(nrows), st);
    if (rc) return rc;
    CK(h, ws.ybuf.ensure(sizeof(double) * nrows * n, st));
    CK(h, launch_gather_rows(ws.a.as<double>(), m, n, lda, lda * n, 1, ws.rows.as<int64_t>(), nrows,
                             ws.ybuf.as<double>(), nrows, nrows * n, nullptr, st));
    h->launches += 1;
    const int64_t kc = std::max<int64_t>(kcap, 1);
    CK(h, ws.idx.ensure(sizeof(int64_t) * kc, st));
    CK(h, ws.coeffs.ensure(sizeof(double) * kc * n, st));
    CK(h, ws.rank.ensure(sizeof(int64_t), st));
    CK(h, ws.resid.ensure(sizeof(double), st));
    CK(h, ws.status.ensure(sizeof(int32_t), st));
    CK(h, cudaMemsetAsync(ws.coeffs.ptr, 0, sizeof(double) * kc * n, st));
    rc = do_cpqr(h, ws, ws.ybuf.as<double>(), nrows, n, nrows, nrows * n, 1, rule, kc,
                 ws.idx.as<int64_t>(), ws.coeffs.as<double>(), kc * n, ws.rank.as<int64_t>(),
                 ws.resid.as<double>(), ws.status.as<int32_t>(), nullptr, nullptr, nullptr, st);
    if (rc) return rc;
    // second pass: fine-grid skeleton (id.cpp:57-58)
    return finish_single(h, ws, m, n, kc, ws.a.as<double>(), lda, indices, coeffs, skeleton, rank,
                         residual_fro, st);
}

int spidgpu_sketch_id(spidgpu_handle h, const double* a, int64_t m, int64_t n, int64_t ell,
                      const spidgpu_omega* omega, const spidgpu_rank_rule* rule, int64_t kcap,
                      double* y, int64_t* indices, double* coeffs, double* skeleton,
                      int64_t* rank, double* residual_fro) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (m < 1 || n < 1 || ell < 1) return fail(h, SPID_EMPTY_MATRIX, "matrix dimensions must be at least 1x1");
    if (!a || !omega_ok(omega)) return fail(h, SPID_INVALID_ARGUMENT, "null input / omega");
    cudaSetDevice(h->device);
    Workspace& ws = h->ws[0];
    cudaStream_t st = h->lanes[0];
    int64_t lda = 0;
    int rc = matrix_to_dev(h, ws.a, a, m, n, &lda, st);
    if (rc) return rc;
    spidgpu_omega om = *omega;
    if (om.mode == SPIDGPU_OMEGA_EXPLICIT) {
        if (om.ldo < ell) return fail(h, SPID_INVALID_ARGUMENT, "ldo < ell");
        CK(h, ws.omega.ensure(sizeof(double) * ell * m, st));
        CK(h, cudaMemcpy2DAsync(ws.omega.ptr, sizeof(double) * ell, om.omega, sizeof(double) * om.ldo,
                                sizeof(double) * ell, m, cudaMemcpyHostToDevice, st));
        om.omega = ws.omega.as<double>();
        om.ldo = ell;
        om.stride = ell * m;
    }
    CK(h, ws.ybuf.ensure(sizeof(double) * ell * n, st));
    rc = do_sketch(h, ws, ws.a.as<double>(), m, n, lda, lda * n, 1, ell, &om, ws.ybuf.as<double>(),
                   ell, ell * n, st);
    if (rc) return rc;
    if (y) CK(h, cudaMemcpyAsync(y, ws.ybuf.ptr, sizeof(double) * ell * n, cudaMemcpyDeviceToHost, st));
    const int64_t kc = std::max<int64_t>(kcap, 1);
    CK(h, ws.idx.ensure(sizeof(int64_t) * kc, st));
    CK(h, ws.coeffs.ensure(sizeof(double) * kc * n, st));
    CK(h, ws.rank.ensure(sizeof(int64_t), st));
    CK(h, ws.resid.ensure(sizeof(double), st));
    CK(h, ws.status.ensure(sizeof(int32_t), st));
    CK(h, cudaMemsetAsync(ws.coeffs.ptr, 0, sizeof(double) * kc * n, st));
    rc = do_cpqr(h, ws, ws.ybuf.as<double>(), ell, n, ell, ell * n, 1, rule, kc,
                 ws.idx.as<int64_t>(), ws.coeffs.as<double>(), kc * n, ws.rank.as<int64_t>(),
                 ws.resid.as<double>(), ws.status.as<int32_t>(), nullptr, nullptr, nullptr, st);
    if (rc) return rc;
    return finish_single(h, ws, m, n, kc, ws.a.as<double>(), lda, indices, coeffs, skeleton, rank,
                         residual_fro, st);
}

int spidgpu_reconstruct(spidgpu_handle h, const double* skeleton, int64_t m, int64_t k,
                        const double* coeffs, int64_t n, double* out) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (m < 1 || n < 1 || k < 1) return fail(h, SPID_EMPTY_MATRIX, "empty factors");
    if (!skeleton || !coeffs || !out) return fail(h, SPID_INVALID_ARGUMENT, "null pointer");
    if (k > 80) return fail(h, SPID_SHAPE_UNSUPPORTED, "reconstruct supports rank <= 80");
    cudaSetDevice(h->device);
    Workspace& ws = h->ws[0];
    cudaStream_t st = h->lanes[0];
    int rc = to_dev(h, ws.skel, skeleton, static_cast<size_t>(m * k), st);
    if (rc) return rc;
    rc = to_dev(h, ws.coeffs, coeffs, static_cast<size_t>(k * n), st);
    if (rc) return rc;
    rc = to_dev(h, ws.rank, &k, 1, st);
    if (rc) return rc;
    CK(h, ws.out.ensure(sizeof(double) * m * n, st));
    CK(h, launch_reconstruct(ws.skel.as<double>(), m, m, m * k, ws.coeffs.as<double>(), k, k * n,
                             ws.rank.as<int64_t>(), n, 1, ws.out.as<double>(), m, m * n, st));
    h->launches += 1;
    CK(h, cudaMemcpyAsync(out, ws.out.ptr, sizeof(double) * m * n, cudaMemcpyDeviceToHost, st));
    CK(h, cudaStreamSynchronize(st));
    return SPID_OK;
}

int spidgpu_rel_frob_error(spidgpu_handle h, const double* exact, const double* approx, int64_t m,
                           int64_t n, double* out) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (m < 1 || n < 1) return fail(h, SPID_EMPTY_MATRIX, "empty matrix");
    if (!exact || !approx || !out) return fail(h, SPID_INVALID_ARGUMENT, "null pointer");
    cudaSetDevice(h->device);
    Workspace& ws = h->ws[0];
    cudaStream_t st = h->lanes[0];
    const size_t cnt = static_cast<size_t>(m * n);
    int rc = to_dev(h, ws.a, exact, cnt, st);
    if (rc) return rc;
    rc = to_dev(h, ws.out, approx, cnt, st);
    if (rc) return rc;
    const int64_t nparts = std::min<int64_t>(296, (cnt + 255) / 256);
    CK(h, ws.vpart.ensure(sizeof(double) * 2 * nparts, st));
    CK(h, launch_sqdiff(ws.a.as<double>(), ws.out.as<double>(), static_cast<int64_t>(cnt),
                        ws.vpart.as<double>(), nparts, st));
    h->launches += 2;
    double sums[2];
    CK(h, cudaMemcpyAsync(sums, ws.vpart.ptr, sizeof(sums), cudaMemcpyDeviceToHost, st));
    CK(h, cudaStreamSynchronize(st));
    if (sums[1] == 0.0) return fail(h, SPID_ZERO_REFERENCE, "reference matrix is zero");
    *out = std::sqrt(sums[0]) / std::sqrt(sums[1]);  // metrics.cpp:20
    return SPID_OK;
}

int spidgpu_compression_factor(int64_t m, int64_t n, int64_t stored, double* out) {
    // metrics.cpp:5-12
    if (!out) return SPID_INVALID_ARGUMENT;
    if (m <= 0 || n <= 0 || stored <= 0) return SPID_ZERO_DENOMINATOR;
    *out = static_cast<double>(m) * static_cast<double>(n) / static_cast<double>(stored);
    return SPID_OK;
}

int spidgpu_compress_host(spidgpu_handle h, const double* a, int64_t m, int64_t n, int64_t batch,
                          int64_t ell, const spidgpu_omega* omega, const spidgpu_rank_rule* rule,
                          int64_t kcap, int64_t group, int64_t* indices, double* coeffs,
                          double* skel, int64_t* rank, double* residual_fro, int32_t* status,
                          double* err2, double* ref2) {
    NvtxRange nvtx_range("spidgpu.compress_host");
    if (!h) return SPID_INVALID_ARGUMENT;
    if (m < 1 || n < 1 || batch < 1 || ell < 1) return fail(h, SPID_EMPTY_MATRIX, "empty batch");
    if (!a || !indices || !coeffs || !rank || !residual_fro || !status || !omega_ok(omega))
        return fail(h, SPID_INVALID_ARGUMENT, "null pointer");
    if ((m % 2) != 0) return fail(h, SPID_SHAPE_UNSUPPORTED, "compress_host needs even m");
    if (omega->mode == SPIDGPU_OMEGA_EXPLICIT)
        return fail(h, SPID_SHAPE_UNSUPPORTED, "compress_host runs in PHILOX mode");
    if ((err2 == nullptr) != (ref2 == nullptr)) return fail(h, SPID_INVALID_ARGUMENT, "err2/ref2");
    RuleInfo ri = resolve_rule(rule, ell, n, kcap);
    if (ri.status) return fail(h, ri.status, "rank rule");
    cudaSetDevice(h->device);
    if (group < 1) group = 1;
    if (group > batch) group = batch;
    const bool want_skel = skel != nullptr || err2 != nullptr;
    const size_t mn = static_cast<size_t>(m) * n;
    // per-lane device buffers
    for (int l = 0; l < 2; ++l) {
        Workspace& w = h->ws[1 + l];
        cudaStream_t st = h->lanes[l];
        CK(h, w.a.ensure(sizeof(double) * group * mn, st));
        CK(h, w.idx.ensure(sizeof(int64_t) * group * kcap, st));
        CK(h, w.coeffs.ensure(sizeof(double) * group * kcap * n, st));
        CK(h, w.rank.ensure(sizeof(int64_t) * group, st));
        CK(h, w.resid.ensure(sizeof(double) * group, st));
        CK(h, w.status.ensure(sizeof(int32_t) * group, st));
        if (want_skel) CK(h, w.skel.ensure(sizeof(double) * group * m * kcap, st));
        if (err2) {
            CK(h, w.err2.ensure(sizeof(double) * group, st));
            CK(h, w.ref2.ensure(sizeof(double) * group, st));
        }
    }
    const int64_t ngroups = (batch + group - 1) / group;
    for (int64_t g = 0; g < ngroups; ++g) {
        const int l = static_cast<int>(g % 2);
        Workspace& w = h->ws[1 + l];
        cudaStream_t st = h->lanes[l];
        const int64_t s0 = g * group;
        const int64_t gs = std::min(group, batch - s0);
        CK(h, cudaMemcpyAsync(w.a.ptr, a + s0 * mn, sizeof(double) * gs * mn,
                              cudaMemcpyHostToDevice, st));
        spidgpu_omega om = *omega;
        om.subdomain_base = omega->subdomain_base + s0;
        int rc = do_compress(h, w, w.a.as<double>(), m, n, m, mn, gs, ell, &om, rule, kcap,
                             w.idx.as<int64_t>(), w.coeffs.as<double>(), w.rank.as<int64_t>(),
                             w.resid.as<double>(), w.status.as<int32_t>(),
                             want_skel ? w.skel.as<double>() : nullptr, nullptr, st);
        if (rc) return rc;
        if (err2) {
            rc = do_verify(h, w, w.a.as<double>(), m, n, m, mn, gs, w.skel.as<double>(), m,
                           m * kcap, w.coeffs.as<double>(), kcap, kcap * n, w.rank.as<int64_t>(),
                           w.err2.as<double>(), w.ref2.as<double>(), st);
            if (rc) return rc;
            CK(h, cudaMemcpyAsync(err2 + s0, w.err2.ptr, sizeof(double) * gs, cudaMemcpyDeviceToHost, st));
            CK(h, cudaMemcpyAsync(ref2 + s0, w.ref2.ptr, sizeof(double) * gs, cudaMemcpyDeviceToHost, st));
        }
        CK(h, cudaMemcpyAsync(indices + s0 * kcap, w.idx.ptr, sizeof(int64_t) * gs * kcap,
                              cudaMemcpyDeviceToHost, st));
        CK(h, cudaMemcpyAsync(coeffs + s0 * kcap * n, w.coeffs.ptr, sizeof(double) * gs * kcap * n,
                              cudaMemcpyDeviceToHost, st));
        CK(h, cudaMemcpyAsync(rank + s0, w.rank.ptr, sizeof(int64_t) * gs, cudaMemcpyDeviceToHost, st));
        CK(h, cudaMemcpyAsync(residual_fro + s0, w.resid.ptr, sizeof(double) * gs,
                              cudaMemcpyDeviceToHost, st));
        CK(h, cudaMemcpyAsync(status + s0, w.status.ptr, sizeof(int32_t) * gs,
                              cudaMemcpyDeviceToHost, st));
        if (skel)
            CK(h, cudaMemcpyAsync(skel + s0 * m * kcap, w.skel.ptr, sizeof(double) * gs * m * kcap,
                                  cudaMemcpyDeviceToHost, st));
    }
    for (int l = 0; l < 2; ++l) CK(h, cudaStreamSynchronize(h->lanes[l]));
    for (int64_t s = 0; s < batch; ++s)
        if (status[s] != SPID_OK)
            return fail(h, status[s], "subdomain " + std::to_string(s) + " failed");
    return SPID_OK;
}

int spidgpu_field_generate(spidgpu_handle h, const spidgpu_field_spec* spec, int64_t first,
                           int64_t batch, const uint8_t* is_heavy, double* A, int64_t lda,
                           int64_t strideA, void* stream) {
    if (!h || !spec || !A) return SPID_INVALID_ARGUMENT;
    if (spec->grid < 1 || spec->block < 1 || spec->grid % spec->block || spec->snapshots < 1)
        return fail(h, SPID_INVALID_ARGUMENT, "bad grid/block/snapshots");
    const int nq = spec->kind == SPIDGPU_FIELD_TGV4 ? 4 : 5;
    const int64_t b3 = spec->block * spec->block * spec->block;
    const int64_t nb = spec->grid / spec->block;
    if (lda < nq * b3 || strideA < lda * spec->snapshots)
        return fail(h, SPID_INVALID_ARGUMENT, "lda/stride too small for the field");
    if (first < 0 || first + batch > nb * nb * nb)
        return fail(h, SPID_INVALID_ARGUMENT, "subdomain range outside the grid");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<double> modes, heavy;
    if (spec->kind == SPIDGPU_FIELD_MULTIMODE) {
        modes = make_modes(spec->seed, spec->n_modes, 1.0, spec->kappa_max, spec->mode_amp);
        if (spec->heavy_modes > 0)
            heavy = make_modes(spec->seed ^ 0xC0FFEE1234ULL, static_cast<int>(spec->heavy_modes),
                               spec->heavy_kmin, spec->kappa_max, spec->mode_amp);
    }
    double* dmodes = nullptr;
    uint8_t* dheavy = nullptr;
    const size_t nmd = modes.size() + heavy.size();
    if (nmd) {
        CK(h, cudaMalloc(&dmodes, sizeof(double) * nmd));
        CK(h, cudaMemcpy(dmodes, modes.data(), sizeof(double) * modes.size(), cudaMemcpyHostToDevice));
        if (!heavy.empty())
            CK(h, cudaMemcpy(dmodes + modes.size(), heavy.data(), sizeof(double) * heavy.size(),
                             cudaMemcpyHostToDevice));
    }
    if (is_heavy && !heavy.empty()) {
        CK(h, cudaMalloc(&dheavy, batch));
        CK(h, cudaMemcpy(dheavy, is_heavy, batch, cudaMemcpyHostToDevice));
    }
    FieldParams p{};
    p.kind = spec->kind;
    p.grid = spec->grid;
    p.block = spec->block;
    p.snapshots = spec->snapshots;
    p.t_end = spec->t_end;
    p.nu = spec->nu;
    p.sigma = spec->noise_sigma;
    p.seed = spec->seed;
    p.first = first;
    p.batch = batch;
    p.A = A;
    p.lda = lda;
    p.strideA = strideA;
    p.modes = dmodes;
    p.n_modes = static_cast<int>(modes.size() / 9);
    p.heavy_modes = dmodes ? dmodes + modes.size() : nullptr;
    p.n_heavy = static_cast<int>(heavy.size() / 9);
    p.is_heavy = dheavy;
    cudaError_t e = launch_field(p, st);
    h->launches += nmd ? 2 : 1;
    cudaStreamSynchronize(st);
    if (dmodes) cudaFree(dmodes);
    if (dheavy) cudaFree(dheavy);
    if (e != cudaSuccess) return cuda_fail(h, e, "launch_field");
    return SPID_OK;
}


// ---- SPID proper (coarse skeleton + lift) -------------------------------------------
int spidgpu_row_indices(const spidgpu_grid_spec* spec, int64_t* rows, int64_t cap, int64_t* count) {
    GridSpecDev g;
    int64_t P = 0, Pc = 0;
    const int rc = spec_to_dev(nullptr, spec, &g, &P, &Pc);
    if (rc) return rc;
    const std::vector<int64_t> J = spec_rows(g, P);
    if (count) *count = static_cast<int64_t>(J.size());
    if (rows)
        for (int64_t i = 0; i < static_cast<int64_t>(J.size()) && i < cap; ++i) rows[i] = J[i];
    return SPID_OK;
}

int spidgpu_spid(spidgpu_handle h, const double* a, int64_t m, int64_t n,
                 const spidgpu_grid_spec* spec, const spidgpu_rank_rule* rule, int64_t kcap,
                 int64_t* indices, double* coeffs, double* coarse_skeleton, int64_t* rank,
                 double* residual_fro) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (m < 1 || n < 1) return fail(h, SPID_EMPTY_MATRIX, "matrix dimensions must be at least 1x1");
    if (!a) return fail(h, SPID_INVALID_ARGUMENT, "null input");
    GridSpecDev g;
    int64_t P = 0, Pc = 0;
    int rc = spec_to_dev(h, spec, &g, &P, &Pc);
    if (rc) return rc;
    if (P * g.nqoi != m)  // id.cpp:70-71
        return fail(h, SPID_GEOMETRY_MISMATCH, "matrix row count does not match grid point count");
    const std::vector<int64_t> J = spec_rows(g, P);
    const int64_t nrows = static_cast<int64_t>(J.size());
    cudaSetDevice(h->device);
    Workspace& ws = h->ws[0];
    cudaStream_t st = h->lanes[0];
    int64_t lda = 0;
    rc = matrix_to_dev(h, ws.a, a, m, n, &lda, st);
    if (rc) return rc;
    rc = to_dev(h, ws.rows, J.data(), J.size(), st);
    if (rc) return rc;
    CK(h, ws.ybuf.ensure(sizeof(double) * nrows * n, st));
    CK(h, launch_gather_rows(ws.a.as<double>(), m, n, lda, lda * n, 1, ws.rows.as<int64_t>(), nrows,
                             ws.ybuf.as<double>(), nrows, nrows * n, nullptr, st));  // subsample, grid.cpp:142-150
    h->launches += 1;
    const int64_t kc = std::max<int64_t>(kcap, 1);
    CK(h, ws.idx.ensure(sizeof(int64_t) * kc, st));
    CK(h, ws.coeffs.ensure(sizeof(double) * kc * n, st));
    CK(h, ws.rank.ensure(sizeof(int64_t), st));
    CK(h, ws.resid.ensure(sizeof(double), st));
    CK(h, ws.status.ensure(sizeof(int32_t), st));
    CK(h, cudaMemsetAsync(ws.coeffs.ptr, 0, sizeof(double) * kc * n, st));
    rc = do_cpqr(h, ws, ws.ybuf.as<double>(), nrows, n, nrows, nrows * n, 1, rule, kc,
                 ws.idx.as<int64_t>(), ws.coeffs.as<double>(), kc * n, ws.rank.as<int64_t>(),
                 ws.resid.as<double>(), ws.status.as<int32_t>(), nullptr, nullptr, nullptr, st);
    if (rc) return rc;
    // the skeleton stays on the coarse grid: columns I of the sketch B (id.cpp:82)
    return finish_single(h, ws, nrows, n, kc, ws.ybuf.as<double>(), nrows, indices, coeffs,
                         coarse_skeleton, rank, residual_fro, st);
}

int spidgpu_interp_apply(spidgpu_handle h, const spidgpu_grid_spec* spec, const double* coarse,
                         int64_t coarse_rows, int64_t k, double* fine) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (!coarse || !fine || k < 1) return fail(h, SPID_INVALID_ARGUMENT, "null buffer / k < 1");
    GridSpecDev g;
    int64_t P = 0, Pc = 0;
    int rc = spec_to_dev(h, spec, &g, &P, &Pc);
    if (rc) return rc;
    if (coarse_rows != Pc * g.nqoi)  // interp.cpp:170
        return fail(h, SPID_DIMENSION_MISMATCH, "coarse rows != coarse points x nqoi");
    cudaSetDevice(h->device);
    Workspace& ws = h->ws[0];
    cudaStream_t st = h->lanes[0];
    const int64_t mc = Pc * g.nqoi, m = P * g.nqoi;
    rc = to_dev(h, ws.skel, coarse, static_cast<size_t>(mc * k), st);
    if (rc) return rc;
    CK(h, ws.out.ensure(sizeof(double) * m * k, st));
    CK(h, ws.flag.ensure(sizeof(int32_t), st));
    CK(h, cudaMemsetAsync(ws.flag.ptr, 0, sizeof(int32_t), st));
    CK(h, launch_interp_apply(g, ws.skel.as<double>(), mc, mc * k, k, nullptr, 1,
                              ws.out.as<double>(), m, m * k, ws.flag.as<int32_t>(), st));
    h->launches += 1;
    int32_t flag = 0;
    CK(h, cudaMemcpyAsync(&flag, ws.flag.ptr, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(h, cudaMemcpyAsync(fine, ws.out.ptr, sizeof(double) * m * k, cudaMemcpyDeviceToHost, st));
    CK(h, cudaStreamSynchronize(st));
    if (flag)  // interp.cpp:27-29
        return fail(h, SPID_EXTRAPOLATION_REQUIRED,
                    "fine point beyond the last coarse point on a non-periodic axis");
    return SPID_OK;
}

int spidgpu_spid_reconstruct(spidgpu_handle h, const spidgpu_grid_spec* spec,
                             const double* coarse_skeleton, int64_t coarse_rows, int64_t k,
                             const double* coeffs, int64_t coeff_rows, int64_t n, double* out) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (!coarse_skeleton || !coeffs || !out || k < 1 || n < 1)
        return fail(h, SPID_INVALID_ARGUMENT, "bad reconstruct arguments");
    if (coeff_rows != k)  // id.cpp:93-94
        return fail(h, SPID_DIMENSION_MISMATCH, "inconsistent factor dimensions");
    if (k > 80) return fail(h, SPID_SHAPE_UNSUPPORTED, "reconstruct supports rank <= 80");
    GridSpecDev g;
    int64_t P = 0, Pc = 0;
    int rc = spec_to_dev(h, spec, &g, &P, &Pc);
    if (rc) return rc;
    if (coarse_rows != Pc * g.nqoi)  // interp.cpp:179 via id.cpp:95
        return fail(h, SPID_DIMENSION_MISMATCH, "coarse skeleton rows != coarse points x nqoi");
    cudaSetDevice(h->device);
    Workspace& ws = h->ws[0];
    cudaStream_t st = h->lanes[0];
    const int64_t mc = Pc * g.nqoi, m = P * g.nqoi;
    rc = to_dev(h, ws.skel, coarse_skeleton, static_cast<size_t>(mc * k), st);
    if (rc) return rc;
    rc = to_dev(h, ws.coeffs, coeffs, static_cast<size_t>(k * n), st);
    if (rc) return rc;
    rc = to_dev(h, ws.rank, &k, 1, st);
    if (rc) return rc;
    CK(h, ws.a.ensure(sizeof(double) * m * k, st));
    CK(h, ws.out.ensure(sizeof(double) * m * n, st));
    CK(h, ws.flag.ensure(sizeof(int32_t), st));
    CK(h, cudaMemsetAsync(ws.flag.ptr, 0, sizeof(int32_t), st));
    // id.cpp:95: matmul(interp.apply(skeleton), coeffs)
    CK(h, launch_interp_apply(g, ws.skel.as<double>(), mc, mc * k, k, nullptr, 1, ws.a.as<double>(),
                              m, m * k, ws.flag.as<int32_t>(), st));
    CK(h, launch_reconstruct(ws.a.as<double>(), m, m, m * k, ws.coeffs.as<double>(), k, k * n,
                             ws.rank.as<int64_t>(), n, 1, ws.out.as<double>(), m, m * n, st));
    h->launches += 2;
    int32_t flag = 0;
    CK(h, cudaMemcpyAsync(&flag, ws.flag.ptr, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    CK(h, cudaMemcpyAsync(out, ws.out.ptr, sizeof(double) * m * n, cudaMemcpyDeviceToHost, st));
    CK(h, cudaStreamSynchronize(st));
    if (flag) return fail(h, SPID_EXTRAPOLATION_REQUIRED, "fine point beyond the last coarse point");
    return SPID_OK;
}

int spidgpu_gather_coarse_batched(spidgpu_handle h, const double* A, int64_t m, int64_t n,
                                  int64_t lda, int64_t strideA, int64_t batch,
                                  const spidgpu_grid_spec* spec, const int64_t* indices,
                                  int64_t kcap, const int64_t* rank, double* skel_c,
                                  int64_t ldskel, int64_t strideS, void* stream) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (!A || !indices || !rank || !skel_c) return fail(h, SPID_INVALID_ARGUMENT, "null pointer");
    GridSpecDev g;
    int64_t P = 0, Pc = 0;
    int rc = spec_to_dev(h, spec, &g, &P, &Pc);
    if (rc) return rc;
    if (P * g.nqoi != m) return fail(h, SPID_GEOMETRY_MISMATCH, "m != grid points x nqoi");
    const std::vector<int64_t> J = spec_rows(g, P);
    if (ldskel < static_cast<int64_t>(J.size()))
        return fail(h, SPID_INVALID_ARGUMENT, "ldskel < coarse rows");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    Workspace& ws = h->ws[0];
    rc = to_dev(h, ws.rows, J.data(), J.size(), st);
    if (rc) return rc;
    CK(h, launch_gather_coarse(A, lda, strideA, ws.rows.as<int64_t>(), static_cast<int64_t>(J.size()),
                               indices, kcap, rank, batch, skel_c, ldskel, strideS, st));
    h->launches += 1;
    (void)n;
    return SPID_OK;
}

int spidgpu_interp_apply_batched(spidgpu_handle h, const spidgpu_grid_spec* spec,
                                 const double* coarse, int64_t ldc, int64_t strideC, int64_t k,
                                 const int64_t* rank, int64_t batch, double* fine, int64_t ldf,
                                 int64_t strideF, void* stream) {
    if (!h) return SPID_INVALID_ARGUMENT;
    if (!coarse || !fine) return fail(h, SPID_INVALID_ARGUMENT, "null pointer");
    GridSpecDev g;
    int64_t P = 0, Pc = 0;
    int rc = spec_to_dev(h, spec, &g, &P, &Pc);
    if (rc) return rc;
    if (ldc < Pc * g.nqoi || ldf < P * g.nqoi) return fail(h, SPID_INVALID_ARGUMENT, "leading dims");
    CK(h, launch_interp_apply(g, coarse, ldc, strideC, k, rank, batch, fine, ldf, strideF, nullptr,
                              static_cast<cudaStream_t>(stream)));
    h->launches += 1;
    return SPID_OK;
}

}  // extern "C"
