/*
 * spidgpu.h -- C ABI of the B200-native SPID compression path.
 *
 * This is the drop-in boundary for the reference's per-subdomain compressor
 * (namespace spid in /root/reference/proj/include/spid). The reference
 * exposes header-level C++ with value semantics and exceptions; a C ABI
 * replaces those with caller-owned buffers and status codes
 * (spidgpu_status.h), whose names are the reference's spid::Error names.
 *
 * Conventions (all entry points):
 *   - matrices are column-major fp64, exactly the reference DenseMatrix
 *     layout ((i,j) at data[j*ld+i], proj/include/spid/dense_matrix.hpp:33-34);
 *   - a batch of S subdomains is S matrices at a fixed element stride;
 *   - skeleton indices are int64 in pivot-selection order and coefficient
 *     matrices are kcap x n (ld kcap) in SOURCE column order with an exact
 *     identity block C(:, I) = I  (proj/src/id.cpp:9-28);
 *   - "_batched" calls take DEVICE pointers and a cudaStream_t (as void*),
 *     are asynchronous, allocate nothing on the hot path, and report
 *     per-subdomain failures in an int32 status array;
 *   - the non-batched calls take HOST pointers and mirror the reference
 *     functions one for one (synchronous, like the reference);
 *   - there is no CPU fallback: without a usable sm_100 device every call
 *     returns SPID_NO_DEVICE / SPID_CUDA_ERROR.
 *
 * One handle per host thread (or stream): handles are independent, which
 * keeps the ABI as reentrant as the reference's pure functions
 * (SURVEY 8(b) "Threading").
 */
#ifndef SPIDGPU_H
#define SPIDGPU_H

#include <stddef.h>
#include <stdint.h>

#include "spidgpu_status.h"

#ifdef __cplusplus
extern "C" {
#endif

#define SPIDGPU_ABI_VERSION 1

typedef struct spidgpu_context* spidgpu_handle;

/* ---- rank rule: replaces spid::RankRule (proj/include/spid/qr.hpp:12-37) ---- */
#define SPIDGPU_RULE_FIXED 0   /* RankRule::fixed(k)                         */
#define SPIDGPU_RULE_TOL 1     /* RankRule::tolerance(tol)                   */
#define SPIDGPU_RULE_BLOCKED 2 /* BASELINE cfg4: rank grows in steps of kstep
                                  up to k until residual_fro/||Y||_F <= tol   */
typedef struct spidgpu_rank_rule {
    int32_t mode;
    int32_t at_most; /* 1 = column_id_at_most semantics (qr.cpp:22-25): k is
                        capped at min(k, rows, cols) and a collapse stops
                        quietly instead of raising RankUnreachable            */
    int64_t k;       /* FIXED: target rank; BLOCKED: kmax                       */
    int64_t kstep;   /* BLOCKED only                                           */
    double tol;      /* TOL / BLOCKED                                          */
} spidgpu_rank_rule;

/* ---- sketch operator Omega (BASELINE north_star: Gaussian, ell = k + p rows) ---- */
#define SPIDGPU_OMEGA_EXPLICIT 0 /* oracle mode: Omega_s given, ell x m, ld ldo   */
#define SPIDGPU_OMEGA_PHILOX 1   /* performance mode: generated in-kernel        */
typedef struct spidgpu_omega {
    int32_t mode;
    int32_t reserved;
    const double* omega;     /* EXPLICIT: device (batched) or host (host API) */
    int64_t ldo;             /* EXPLICIT: leading dimension (>= ell)           */
    int64_t stride;          /* EXPLICIT: elements between Omega_s, Omega_s+1  */
    uint64_t seed;           /* PHILOX: key                                    */
    int64_t subdomain_base;  /* PHILOX: global id of batch element 0           */
} spidgpu_omega;

/* ---- lifecycle / diagnostics ---- */
int spidgpu_create(int device, spidgpu_handle* out);
int spidgpu_destroy(spidgpu_handle h);
/* Reference error name for a status code ("ZeroMatrix", ...); "Ok" for 0. */
const char* spidgpu_status_name(int status);
/* Human-readable message of the handle's last failure ("" if none). */
const char* spidgpu_last_error(spidgpu_handle h);
int spidgpu_abi_version(void);
/* Kernel launches issued through this handle since creation (instrumentation). */
int64_t spidgpu_launch_count(spidgpu_handle h);
/* Handle options. SPIDGPU_OPT_GENERIC_CPQR = 1 routes column IDs of
 * sketch-sized matrices through the general (shared/global-memory) CPQR
 * kernel instead of the register-resident one; both are bit-exact with the
 * reference, the option exists so tests can cover both.
 * SPIDGPU_OPT_DMMA_SKETCH = 2 runs Philox-Omega sketches on the FP64 DMMA
 * kernel instead of the exact integer-sliced tcgen05 (TMEM) kernel (same
 * Omega; the option exists for tests and A/B measurement). Option 3 (a
 * retired register-fed IMMA variant) is rejected.
 * SPIDGPU_OPT_SKETCH_SMS = 4 caps the SMs the persistent sketch kernels
 * occupy (0 = all), leaving the rest to kernels on other streams (the
 * overlapped compress pipeline).
 * SPIDGPU_OPT_SKETCH_PAIRS = 5 runs the tcgen05 sketch of up to 64 rows as
 * clusters of two CTAs that share each stage's Omega tile: 0 and 1 (default)
 * never (one CTA per tile measured as fast or faster at every width), 2
 * whenever the column tiles pair up (bitwise the same Y; tests and A/B).
 * Sketches of 65-80 rows always run as slice-split CTA pairs.
 * Every sketch is bitwise independent of the batch it runs in, the SM cap,
 * the pair mode and the GPU count: work is split at fixed 4096-row segment
 * boundaries and segment partials are summed in a fixed order.
 * SPIDGPU_OPT_SKETCH_SEG_ROWS = 6 sets the tcgen05 sketch's segment length in
 * rows (0 = the default 4096; a multiple of 512 up to 65536). Results are
 * independent of batching for any fixed value, but differ (within the
 * accuracy contract) between values; the option exists for measurement. */
#define SPIDGPU_OPT_GENERIC_CPQR 1
#define SPIDGPU_OPT_DMMA_SKETCH 2
#define SPIDGPU_OPT_SKETCH_SMS 4
#define SPIDGPU_OPT_SKETCH_PAIRS 5
#define SPIDGPU_OPT_SKETCH_SEG_ROWS 6
/* SPIDGPU_OPT_TALL_PAIRS = 7: tall column IDs (rows >= 256) with 64 < n <= 256
 * columns and the fixed or tolerance rule run each subdomain's columns on a
 * cluster of two CTAs (1, default) or on one CTA (0); bitwise the same
 * factors (tests and A/B). */
#define SPIDGPU_OPT_TALL_PAIRS 7
/* SPIDGPU_OPT_REG_PAIRS = 8: sketch-sized column IDs with 33-48 rows,
 * 128 < n <= 256 columns, the fixed or tolerance rule and at most one pair
 * per two SMs (config 3's 48 x 256 sketches) run each subdomain's columns on
 * a cluster of two CTAs (1, default) or on one CTA (0); bitwise the same
 * factors (tests and A/B). */
#define SPIDGPU_OPT_REG_PAIRS 8
int spidgpu_set_option(spidgpu_handle h, int option, int64_t value);
/* Instrumentation: out[0..2] = tcgen05-sketch converter-warp flushes since
 * the last reset, by cause (segment end, exponent-headroom overflow,
 * magnitude fallback); process-wide for the handle's device. n >= 3. */
int spidgpu_debug_counters(spidgpu_handle h, int64_t* out, int n, int reset);

/* =====================================================================
 * Batched device API (the hot path). Subdomain s of a batch lives at
 * A + s*strideA (m x n, ld lda). All outputs are caller-allocated device
 * buffers sized by kcap; stream may be NULL (legacy default stream).
 * ===================================================================== */

/* Y_s = Omega_s * A_s  (ell x n, ld ldy, stride strideY). Replaces the
 * reference sketch entry subsample()/subsample_column() (proj/src/grid.cpp:
 * 136-150, used by spid() at proj/src/id.cpp:75-80) with the Gaussian sketch
 * of the north star; restated by matmul (proj/src/dense_matrix.cpp:38-53).
 * Philox Omega (SPIDGPU_OMEGA_PHILOX, the performance mode): an exact
 * integer-sliced contraction on the tcgen05 tensor cores (kind::i8, TMEM
 * accumulators), A staged by TMA and read once (up to 80 rows per pass;
 * 65-80 rows as slice-split CTA pairs). Explicit fp64 Omega (oracle mode):
 * FP64 DMMA. Both split the work at fixed 4096-row segments (8192 for the
 * split pairs) and sum the segment partials in a fixed order: Y is bitwise
 * reproducible and independent of the batch it is computed in. Accuracy:
 * per entry within 2^-47 sum_k |Omega(i,k)| M_j(k) + (2 nseg + 2) u (|Omega||A|)(i,j)
 * of the exact product, M_j(k) the largest |A(., j)| of row k's segment
 * (tests/test_gpu_sketch_i8.py). */
int spidgpu_sketch_batched(spidgpu_handle h, const double* A, int64_t m, int64_t n, int64_t lda,
                           int64_t strideA, int64_t batch, int64_t ell, const spidgpu_omega* omega,
                           double* Y, int64_t ldy, int64_t strideY, void* stream);

/* Materialise the Omega_s that SPIDGPU_OMEGA_PHILOX uses (ell x m, ld ldo) so
 * an oracle can be fed the same bits: Omega_s(r, k) = Q[u >> 4] / 32 with u
 * the 16-bit half (k % 8) of Philox4x32-7(counter {k / 8, r, s}, key seed) and
 * Q the 4096-quantile table of N(0, 1) rounded to multiples of 1/32. */
int spidgpu_philox_omega(spidgpu_handle h, uint64_t seed, int64_t subdomain, int64_t ell,
                         int64_t m, double* omega, int64_t ldo, void* stream);

/* Column ID of each Y_s (rows x n): greedy CPQR + coefficient solve, one
 * subdomain per CTA. Replaces column_id / column_id_at_most
 * (proj/src/id.cpp:40-52) -> pivoted_mgs_qr (proj/src/qr.cpp:18-124) ->
 * build_coeffs + solve_upper_triangular (id.cpp:9-28, qr.cpp:128-151).
 * Bit-identical to the reference for identical Y (same summation order, no
 * FMA contraction). Outputs per subdomain s:
 *   indices[s*kcap ..]     selection-order skeleton indices (rank entries)
 *   C[s*strideC ..]        kcap x n, ld kcap (rows >= rank untouched)
 *   rank[s], residual_fro[s], status[s]
 * Optional (NULL to skip): pivots (n per subdomain, full permutation),
 *   R (kcap x n per subdomain, ld kcap, pivoted column order as
 *   QrFactorization::r_mat), Q (rows x kcap per subdomain, ld rows). */
int spidgpu_cpqr_id_batched(spidgpu_handle h, const double* Y, int64_t rows, int64_t n,
                            int64_t ldy, int64_t strideY, int64_t batch,
                            const spidgpu_rank_rule* rule, int64_t kcap, int64_t* indices,
                            double* C, int64_t strideC, int64_t* rank, double* residual_fro,
                            int32_t* status, int64_t* pivots, double* R, double* Q, void* stream);

/* skel_s(:, t) = A_s(:, indices_s[t]) for t < rank[s]: select_columns
 * (proj/src/dense_matrix.cpp:71-81) -- the fine skeleton of sub_id
 * (proj/src/id.cpp:57-58). */
int spidgpu_gather_batched(spidgpu_handle h, const double* A, int64_t m, int64_t n, int64_t lda,
                           int64_t strideA, int64_t batch, const int64_t* indices, int64_t kcap,
                           const int64_t* rank, double* skel, int64_t ldskel, int64_t strideS,
                           void* stream);

/* B_s = A_s(J, :) for a strictly increasing row set J (nrows entries):
 * subsample (proj/src/grid.cpp:136-140). Output ld ldb, stride strideB.
 * Both batched gathers are asynchronous: an index outside the matrix
 * (select_columns' IndexOutOfRange, proj/src/dense_matrix.cpp:75) leaves
 * its column unwritten (rows: 0.0) and is recorded for
 * spidgpu_stream_status. */
int spidgpu_row_gather_batched(spidgpu_handle h, const double* A, int64_t m, int64_t n,
                               int64_t lda, int64_t strideA, int64_t batch, const int64_t* rows,
                               int64_t nrows, double* B, int64_t ldb, int64_t strideB,
                               void* stream);

/* Workspaces. A handle's batched calls share one device workspace, like
 * the reference's functions share nothing but their arguments per thread:
 * issue them on ONE stream at a time (one handle per concurrent stream or
 * host thread). Workspaces grow on first use (a cudaMalloc after
 * synchronising the stream); spidgpu_reserve pre-sizes them for batches of
 * up to `batch` m x n subdomains, sketches of up to ell rows and ranks up to
 * kcap, so that later batched calls of those sizes allocate nothing. */
int spidgpu_reserve(spidgpu_handle h, int64_t m, int64_t n, int64_t batch, int64_t ell, int64_t kcap);

/* Synchronise `stream` and return the first deferred error a batched call
 * of this handle recorded since the last call (IndexOutOfRange from the
 * gathers), or SPID_OK; clears it. */
int spidgpu_stream_status(spidgpu_handle h, void* stream);

/* Exact verification terms per subdomain: err2[s] = ||A_s - skel_s C_s||_F^2,
 * ref2[s] = ||A_s||_F^2 (reconstruct + rel_frob_error, proj/src/id.cpp:85-90,
 * proj/src/metrics.cpp:14-21). FP64 DMMA, deterministic reduction. */
int spidgpu_verify_batched(spidgpu_handle h, const double* A, int64_t m, int64_t n, int64_t lda,
                           int64_t strideA, int64_t batch, const double* skel, int64_t ldskel,
                           int64_t strideS, const double* C, int64_t kcap, int64_t strideC,
                           const int64_t* rank, double* err2, double* ref2, void* stream);

/* out_s = skel_s * C_s (m x n, ld ldo): reconstruct (proj/src/id.cpp:85-90). */
int spidgpu_reconstruct_batched(spidgpu_handle h, const double* skel, int64_t m, int64_t ldskel,
                                int64_t strideS, const double* C, int64_t kcap, int64_t strideC,
                                const int64_t* rank, int64_t n, int64_t batch, double* out,
                                int64_t ldo, int64_t strideO, void* stream);

/* The fused compress driver: sketch -> CPQR/coefficients -> skeleton gather
 * for a batch of subdomains (the CLI batch loop, proj/tools/spid_cli.cpp:
 * 220-231, with sub_id's fine skeleton). skel may be NULL (no gather); Y may
 * be NULL (sketch kept in the handle's workspace). */
int spidgpu_compress_batched(spidgpu_handle h, const double* A, int64_t m, int64_t n, int64_t lda,
                             int64_t strideA, int64_t batch, int64_t ell,
                             const spidgpu_omega* omega, const spidgpu_rank_rule* rule,
                             int64_t kcap, int64_t* indices, double* C, int64_t* rank,
                             double* residual_fro, int32_t* status, double* skel, double* Y,
                             void* stream);

/* =====================================================================
 * SPID proper: coarse-grid skeleton + multilinear lift
 * (SubsampleSpec / InterpOperator, proj/include/spid/grid.hpp:188-208,
 * proj/include/spid/interp.hpp:14-53).
 * ===================================================================== */

/* A strided structured SubsampleSpec (proj/src/grid.cpp:62-75) on a 1-3 axis
 * grid, optionally repeated over `nqoi` QoI blocks stacked along the rows
 * (row = q * P + p; nqoi = 1 is the reference's single-QoI layout). */
typedef struct spidgpu_grid_spec {
    int32_t naxes;            /* 1..3                                           */
    int32_t include_boundary; /* pin the last point of non-periodic axes        */
    int64_t dims[3];          /* points per axis (axis 0 fastest)               */
    int64_t strides[3];       /* >= 1                                           */
    int32_t periodic[3];
    int32_t nqoi;             /* >= 1                                           */
} spidgpu_grid_spec;

/* SubsampleSpec::row_indices (proj/src/grid.cpp:108-130), repeated per QoI
 * block. Writes min(count, cap) entries; *count = |J|. Pure index arithmetic. */
int spidgpu_row_indices(const spidgpu_grid_spec* spec, int64_t* rows, int64_t cap, int64_t* count);

/* spid::spid (proj/src/id.cpp:62-83): sketch B = A(J, :), column ID of B,
 * skeleton kept on the COARSE rows (B(:, I), |J| x kcap, ld |J|). */
int spidgpu_spid(spidgpu_handle h, const double* a, int64_t m, int64_t n,
                 const spidgpu_grid_spec* spec, const spidgpu_rank_rule* rule, int64_t kcap,
                 int64_t* indices, double* coeffs, double* coarse_skeleton, int64_t* rank,
                 double* residual_fro);

/* InterpOperator::apply (proj/src/interp.cpp:168-186), host buffers:
 * fine (m x k, m = P*nqoi) = M * coarse (|J| x k). Bit-identical to the
 * reference operator built by InterpOperator::from_spec. */
int spidgpu_interp_apply(spidgpu_handle h, const spidgpu_grid_spec* spec, const double* coarse,
                         int64_t coarse_rows, int64_t k, double* fine);

/* spid::reconstruct(SpidFactors) (proj/src/id.cpp:92-96): M * skel_c * C. */
int spidgpu_spid_reconstruct(spidgpu_handle h, const spidgpu_grid_spec* spec,
                             const double* coarse_skeleton, int64_t coarse_rows, int64_t k,
                             const double* coeffs, int64_t coeff_rows, int64_t n, double* out);

/* Batched device forms. gather: skel_c_s(:, t) = A_s(J, I_s[t]);
 * lift: fine_s(:, t) = M * coarse_s(:, t) for t < rank[s]. */
int spidgpu_gather_coarse_batched(spidgpu_handle h, const double* A, int64_t m, int64_t n,
                                  int64_t lda, int64_t strideA, int64_t batch,
                                  const spidgpu_grid_spec* spec, const int64_t* indices,
                                  int64_t kcap, const int64_t* rank, double* skel_c,
                                  int64_t ldskel, int64_t strideS, void* stream);
int spidgpu_interp_apply_batched(spidgpu_handle h, const spidgpu_grid_spec* spec,
                                 const double* coarse, int64_t ldc, int64_t strideC, int64_t k,
                                 const int64_t* rank, int64_t batch, double* fine, int64_t ldf,
                                 int64_t strideF, void* stream);

/* =====================================================================
 * Host-buffer API: one call per reference function (synchronous).
 * ===================================================================== */

/* spid::column_id / column_id_at_most (proj/src/id.cpp:40-52).
 * coeffs: kcap x n (ld kcap); skeleton: m x kcap (ld m), may be NULL. */
int spidgpu_column_id(spidgpu_handle h, const double* a, int64_t m, int64_t n,
                      const spidgpu_rank_rule* rule, int64_t kcap, int64_t* indices,
                      double* coeffs, double* skeleton, int64_t* rank, double* residual_fro);

/* spid::pivoted_mgs_qr / _at_most (proj/src/qr.cpp:18-25) with the full
 * QrFactorization: q (m x kcap, ld m), r (kcap x n, ld kcap), pivots (n). */
int spidgpu_qr(spidgpu_handle h, const double* a, int64_t m, int64_t n,
               const spidgpu_rank_rule* rule, int64_t kcap, double* q, double* r, int64_t* pivots,
               int64_t* rank, double* residual_fro);

/* spid::sub_id (proj/src/id.cpp:54-60) with the row set J of the spec given
 * explicitly (SubsampleSpec::row_indices, proj/src/grid.cpp:108-130). */
int spidgpu_sub_id(spidgpu_handle h, const double* a, int64_t m, int64_t n, const int64_t* rows,
                   int64_t nrows, const spidgpu_rank_rule* rule, int64_t kcap, int64_t* indices,
                   double* coeffs, double* skeleton, int64_t* rank, double* residual_fro);

/* Gaussian-sketch SubID of one subdomain: Y = Omega A, column_id(Y), fine
 * skeleton A(:, I). omega->omega (EXPLICIT) is a HOST pointer here. y (ell x
 * n) may be NULL. */
int spidgpu_sketch_id(spidgpu_handle h, const double* a, int64_t m, int64_t n, int64_t ell,
                      const spidgpu_omega* omega, const spidgpu_rank_rule* rule, int64_t kcap,
                      double* y, int64_t* indices, double* coeffs, double* skeleton,
                      int64_t* rank, double* residual_fro);

/* spid::reconstruct / pyspid.reconstruct (proj/src/id.cpp:85-90): out = skel * coeffs
 * (skel m x k, coeffs k x n, out m x n). */
int spidgpu_reconstruct(spidgpu_handle h, const double* skeleton, int64_t m, int64_t k,
                        const double* coeffs, int64_t n, double* out);

/* spid::rel_frob_error (proj/src/metrics.cpp:14-21), computed on the device. */
int spidgpu_rel_frob_error(spidgpu_handle h, const double* exact, const double* approx, int64_t m,
                           int64_t n, double* out);

/* spid::compression_factor (proj/src/metrics.cpp:5-12): pure arithmetic. */
int spidgpu_compression_factor(int64_t m, int64_t n, int64_t stored, double* out);

/* End-to-end batched compression from HOST buffers: the reference-facing
 * batch call (one spid() per block, proj/tools/spid_cli.cpp:220-231) with the
 * host<->device traffic inside. Subdomain s of A is at a + s*m*n (m x n, ld m).
 * Streams subdomains through device memory in groups of `group` with copy /
 * compute overlap. Outputs (host): indices (batch x kcap), coeffs (batch x
 * kcap x n), skel (batch x m x kcap, may be NULL), rank, residual_fro, status.
 * If err2/ref2 are non-NULL the verify pass runs too. */
int spidgpu_compress_host(spidgpu_handle h, const double* a, int64_t m, int64_t n, int64_t batch,
                          int64_t ell, const spidgpu_omega* omega, const spidgpu_rank_rule* rule,
                          int64_t kcap, int64_t group, int64_t* indices, double* coeffs,
                          double* skel, int64_t* rank, double* residual_fro, int32_t* status,
                          double* err2, double* ref2);

/* =====================================================================
 * Archive codec (proj/include/spid/archive.hpp) -- SURVEY 8(f)3.
 * ===================================================================== */

/* CRC-32/ISO-HDLC of a buffer (spid::crc32, proj/src/archive.cpp:168-178),
 * computed on the device. on_device != 0: `data` is a device pointer. */
int spidgpu_crc32(spidgpu_handle h, const void* data, int64_t nbytes, int32_t on_device,
                  uint32_t* out);

#define SPIDGPU_ARCHIVE_EXACT 0  /* column ID of each block's coarse rows: the
                                    reference's spid() -> byte-identical archive */
#define SPIDGPU_ARCHIVE_SKETCH 1 /* Gaussian sketch (Philox) of the coarse rows
                                    first (integer tcgen05 sketch), then the column ID */
typedef struct spidgpu_archive_spec {
    int32_t naxes;              /* structured grid, 1..3 axes (axis 0 fastest)  */
    int32_t mode;               /* SPIDGPU_ARCHIVE_*                            */
    int64_t dims[3];
    int32_t periodic[3];
    int32_t reserved;
    int64_t blocks_per_axis[3]; /* make_block_domains plan                      */
    int64_t strides[3];         /* SubsampleSpec::strided(local, strides, true) */
    int64_t ell;                /* SKETCH: sketch rows (>= rank)                 */
    uint64_t seed;              /* SKETCH: Philox key; block b uses subdomain b  */
    const char* qoi;            /* metadata strings (may be NULL = "")          */
    const char* provenance;
} spidgpu_archive_spec;

/* Batch compression of a whole field into an archive -- the spid CLI's
 * `compress --chunk 0` on a structured grid (compress_structured_batch,
 * proj/tools/spid_cli.cpp:195-232) followed by spid::encode
 * (proj/src/archive.cpp:193-212). a: m x n (ld lda), rows = grid points
 * (axis 0 fastest); a_on_device != 0 if `a` is a device pointer. rule: FIXED
 * (at_most = 0) or TOL, as the CLI's --rank / --tol. The archive is kept in
 * the handle: *nbytes receives its size, spidgpu_archive_fetch copies it. */
int spidgpu_archive_compress(spidgpu_handle h, const double* a, int64_t m, int64_t n, int64_t lda,
                             int32_t a_on_device, const spidgpu_archive_spec* spec,
                             const spidgpu_rank_rule* rule, int64_t* nbytes);
int spidgpu_archive_fetch(spidgpu_handle h, uint8_t* dst, int64_t cap);
/* Zero-copy view of the same bytes (pinned host memory owned by the handle,
 * valid until the next spidgpu_archive_compress or spidgpu_destroy). */
int spidgpu_archive_view(spidgpu_handle h, const uint8_t** data, int64_t* nbytes);

/* decode() header walk (archive.cpp:214-249) without the checksums: output
 * shape of decompress (rows = grid points, cols = snapshot count) and the
 * block count. Host-only. */
int spidgpu_archive_shape(const uint8_t* bytes, int64_t nbytes, int64_t* rows, int64_t* cols,
                          int64_t* blocks);

/* archive_info_json (archive.cpp:260-268) of an archive (checksums verified
 * on the device). Writes a NUL-terminated string; *len = strlen. */
int spidgpu_archive_info(spidgpu_handle h, const uint8_t* bytes, int64_t nbytes, char* out,
                         int64_t cap, int64_t* len);

/* decode() + decompress() (archive.cpp:214-249, 281-303): every section
 * checksummed on the device, coarse skeletons lifted, blocks multiplied out
 * in the reference matmul's order and scattered into out (rows x cols, ld
 * ldo; out_on_device != 0 for a device pointer). Bit-identical to the
 * reference's decompress. */
int spidgpu_archive_decompress(spidgpu_handle h, const uint8_t* bytes, int64_t nbytes, double* out,
                               int64_t ldo, int32_t out_on_device);

/* =====================================================================
 * Streaming two-stage compressor -- SURVEY 8(f)2. Replaces run_pipeline
 * (proj/src/pipeline.cpp:104-294, proj/include/spid/pipeline.hpp): snapshots
 * are pushed as they are produced; every block's coarse rows are buffered in
 * device memory into temporal chunks of time_chunk columns; each closed chunk
 * runs stage 1 (column_id_at_most(chunk, min(k, cols)), blocking.cpp:112-115)
 * for all blocks at once on a second CUDA stream while ingestion continues
 * (at most 2 chunks in flight per block, the reference's backpressure);
 * finish runs stage 2 (stage2_compress, blocking.cpp:128-204: tolerance ID of
 * the union of stage-1 skeletons, composed coefficients) for all blocks and
 * emits the "two-stage" archive. The archive is byte-identical to
 * encode(run_pipeline(...).archive) for the same snapshots.
 * ===================================================================== */
typedef struct spidgpu_stream_config {
    int32_t naxes;              /* structured grid, 1..3 axes                   */
    int32_t include_boundary;   /* StreamConfig::include_boundary               */
    int64_t dims[3];
    int32_t periodic[3];
    int32_t reserved;
    int64_t blocks_per_axis[3]; /* PartitionPlan::blocks_per_axis               */
    int64_t strides[3];         /* StreamConfig::strides                        */
    int64_t time_chunk;         /* PartitionPlan::time_chunk (>= 1)             */
    int64_t stage1_rank;        /* StreamConfig::stage1_rank (>= 1)             */
    double stage2_tol;          /* StreamConfig::stage2_tol                     */
    const char* qoi;
    const char* provenance;
} spidgpu_stream_config;

typedef struct spidgpu_stream_stats {
    int64_t snapshots;           /* frames ingested                             */
    int64_t stage1_tasks;        /* (block, chunk) stage-1 IDs run              */
    int64_t stage2_tasks;        /* blocks merged by stage 2                    */
    int64_t fine_entries_peak;   /* device frame staging (entries)              */
    int64_t coarse_entries_peak; /* chunk buffers (entries), cf. BufferStats    */
    double stage1_ms;            /* device time of all stage-1 launches         */
    double stage2_ms;            /* device time of stage 2 + archive emission   */
} spidgpu_stream_stats;

typedef struct spidgpu_stream* spidgpu_stream_handle;

/* The pipeline's event log (spid::TaskEvent, proj/include/spid/pipeline.hpp:
 * 24-32). Times are seconds on the DEVICE timeline from the stream's open
 * (CUDA events recorded on the ingestion and stage-1 streams), so causality
 * is exact: a chunk's stage 1 waits on the event that closes it.
 *   SNAPSHOT_INGESTED  per frame; chunk = snapshot index; duration = device
 *                      time of the push that carried it (host copy + gather)
 *   CHUNK_CLOSED       per (block, chunk): ingestion of the chunk complete
 *   STAGE1_DONE        per (block, chunk); duration = the batched stage-1
 *                      launch of that chunk (all blocks)
 *   STAGE2_DONE        per block; duration = stage 2 + archive emission */
#define SPIDGPU_EVENT_SNAPSHOT_INGESTED 0
#define SPIDGPU_EVENT_CHUNK_CLOSED 1
#define SPIDGPU_EVENT_STAGE1_DONE 2
#define SPIDGPU_EVENT_STAGE2_DONE 3
typedef struct spidgpu_task_event {
    int32_t kind;
    int64_t block;   /* -1 for stream-level events */
    int64_t chunk;   /* snapshot index for SNAPSHOT_INGESTED */
    double wall_time;
    double duration;
} spidgpu_task_event;

typedef struct spidgpu_overlap {  /* spid::OverlapReport, pipeline.hpp:52-56 */
    double overlap_fraction;      /* of stage-1 time inside ingestion activity */
    double stage1_busy_seconds;
    double producer_busy_seconds;
} spidgpu_overlap;

/* Validates the plan (UnstructuredNoInterp, BadStreamConfig, BlockTooSmall,
 * BadSubsampleSpec as run_pipeline does before ingesting). The stream owns
 * its CUDA streams and buffers; `h` receives the archive at finish. */
int spidgpu_stream_open(spidgpu_handle h, const spidgpu_stream_config* cfg,
                        spidgpu_stream_handle* out);
/* Push `count` snapshots (m x count, ld ld; m must equal the grid's point
 * count, else GeometryMismatch). on_device: 0 host frames, read (copied)
 * before the call returns, so the caller may reuse them then; 1 device
 * frames, 2 host frames (pinned, for an asynchronous copy): read
 * asynchronously in push order, so the caller keeps them unmodified until
 * spidgpu_stream_finish returns, and consecutive host pushes queue their
 * copies back to back instead of waiting for each other. */
int spidgpu_stream_push(spidgpu_stream_handle s, const double* frames, int64_t m, int64_t count,
                        int64_t ld, int32_t on_device);
/* Close the final short chunks, run stage 2, emit the archive into the parent
 * handle (spidgpu_archive_view / spidgpu_archive_fetch). Stage-1 failures are
 * reported here, naming the first failing block and chunk; ShortStream when
 * nothing was pushed. */
int spidgpu_stream_finish(spidgpu_stream_handle s, int64_t* nbytes);
int spidgpu_stream_get_stats(spidgpu_stream_handle s, spidgpu_stream_stats* out);
/* Message of the stream's last failure ("" if none). */
const char* spidgpu_stream_last_error(spidgpu_stream_handle s);
/* After spidgpu_stream_finish: the event log, in emission order per kind
 * (ingestion, chunk closes, stage-1 completions, stage-2 completions).
 * Writes min(cap, total) events; *count = total. */
int spidgpu_stream_events(spidgpu_stream_handle s, spidgpu_task_event* out, int64_t cap, int64_t* count);
/* spid::overlap_report (proj/src/pipeline.cpp:296-332): pure host arithmetic
 * over an event log; EmptyLog for an empty one. */
int spidgpu_overlap_report(const spidgpu_task_event* events, int64_t count, spidgpu_overlap* out);
int spidgpu_stream_close(spidgpu_stream_handle s);

/* =====================================================================
 * Synthetic input fields (bench/tests only; not a reference interface).
 * Taylor-Green-vortex families of BASELINE.json configs 1-5, generated in
 * place on the device for a batch of subdomains of a periodic N^3 grid split
 * into blocks of b^3 (make_block_domains order, proj/src/blocking.cpp:31-98),
 * rows QoI-major (row = q*b^3 + local point, axis 0 fastest).
 * ===================================================================== */
#define SPIDGPU_FIELD_TGV4 0      /* cfg1: u, v, w=0, p (incompressible TGV)  */
#define SPIDGPU_FIELD_TGV5 1      /* cfg2: rho, u, v, w, E (compressible)     */
#define SPIDGPU_FIELD_MULTIMODE 2 /* cfg3/4/5: TGV5 + random Fourier modes    */
typedef struct spidgpu_field_spec {
    int32_t kind;
    int32_t n_modes;        /* MULTIMODE: number of extra Fourier modes      */
    int64_t grid;           /* N (points per axis of the whole grid)         */
    int64_t block;          /* b (points per axis of one subdomain)          */
    int64_t snapshots;      /* n                                             */
    double t_end;           /* snapshots uniform in [0, t_end] (inclusive)   */
    double nu;              /* viscosity                                     */
    double noise_sigma;     /* additive N(0, sigma^2) noise                  */
    double kappa_max;       /* MULTIMODE: |kappa| bound                      */
    double mode_amp;        /* MULTIMODE: amplitude scale (x |kappa|^-5/3)   */
    uint64_t seed;          /* modes and noise                               */
    int64_t heavy_modes;    /* cfg4: extra high-wavenumber modes on "heavy"  */
    double heavy_kmin;      /* cfg4: |kappa| lower bound of heavy modes      */
} spidgpu_field_spec;

/* Fill batch subdomains [first, first+batch) (global block ids) into A
 * (m x n per subdomain, ld lda, stride strideA). For cfg4, subdomains with
 * is_heavy[s] != 0 (host array, may be NULL) get the extra modes. */
int spidgpu_field_generate(spidgpu_handle h, const spidgpu_field_spec* spec, int64_t first,
                           int64_t batch, const uint8_t* is_heavy, double* A, int64_t lda,
                           int64_t strideA, void* stream);

#ifdef __cplusplus
}
#endif

#endif
