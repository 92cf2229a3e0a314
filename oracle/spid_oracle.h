/*
 * spid_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain-C CPU restatement of the reference's SPID compression path
 * (/root/reference/proj/src/{dense_matrix,qr,id,metrics}.cpp), used as the
 * parity checker for the B200 kernels. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it. The product
 * library (paper_2103_01380_b200/lib/libspidgpu.so) never links or calls it.
 *
 * Pinned against: the reference's own KATs (proj/tests/test_matrix_core.cpp,
 * test_id_core.cpp, acceptance.cpp criteria 1 and 6) and against the reference
 * compiled from its sources (oracle/_ref, see oracle/Makefile) -- see
 * tests/test_oracle.py and tests/golden/.
 *
 * All matrices are column-major fp64 ((i,j) at data[j*rows+i]), exactly the
 * reference's DenseMatrix layout (proj/include/spid/dense_matrix.hpp:33-34).
 * Build flags keep IEEE semantics: no FMA contraction, no reassociation, so
 * results are bit-identical to the reference built without -march.
 */
#ifndef SPID_ORACLE_H
#define SPID_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#include "../include/spidgpu_status.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Rank rules: proj/include/spid/qr.hpp:12-37, plus the blocked adaptive rule
 * of BASELINE config 4 (not in the reference; defined in DESIGN.md). */
#define ORC_RULE_FIXED 0
#define ORC_RULE_TOL 1
#define ORC_RULE_BLOCKED 2

/* SplitMix64 fill with next_sym(), column-major order
 * (proj/include/spid/rng.hpp:10-29, proj/tests/common.hpp:13-26). */
void orc_seeded_sym(uint64_t seed, double* out, size_t count);
uint64_t orc_splitmix_next(uint64_t* state);

/* Seeded N(0,1) fill (SplitMix64 + Box-Muller). Not in the reference, which
 * has no Gaussian sampler; used only to make oracle-mode Omega. */
void orc_gaussian(uint64_t seed, double* out, size_t count);

/* c(ar x bc) = a(ar x ac) * b(ac x bc); j-k-i order with the zero skip of
 * proj/src/dense_matrix.cpp:38-53. c is overwritten. */
void orc_matmul(const double* a, size_t ar, size_t ac, const double* b, size_t bc, double* c);

double orc_frobenius(const double* a, size_t count);            /* dense_matrix.cpp:113-120 */
double orc_dot(const double* x, const double* y, size_t n);      /* dense_matrix.cpp:136-140 */
double orc_norm2(const double* x, size_t n);                     /* dense_matrix.cpp:142 */

/* Greedy column-pivoted 2-pass MGS QR, proj/src/qr.cpp:29-124.
 *   mode/k/tol/kstep: rank rule (k is kmax for BLOCKED)
 *   strict: 1 = pivoted_mgs_qr (raise RankUnreachable on collapse),
 *           0 = pivoted_mgs_qr_at_most (qr.cpp:22-25; caller caps k)
 * Outputs (any may be NULL): q (m x kcap col-major, ld m), r (kcap x n,
 * col-major, ld kcap), pivots (n, full permutation), rank, residual_fro.
 * kcap must be >= the step limit. Returns a SPID_* status code. */
int orc_qr(const double* a, size_t m, size_t n, int mode, size_t k, double tol, size_t kstep,
           int strict, size_t kcap, double* q, double* r, int64_t* pivots, size_t* rank,
           double* residual_fro);

/* Back substitution r11 * x = rhs, proj/src/qr.cpp:128-151. r11 is k x k
 * (ld ldr), rhs k x ncols (ld k), x k x ncols (ld k). */
int orc_solve_upper(const double* r11, size_t k, size_t ldr, const double* rhs, size_t ncols,
                    double* x);

/* column_id / column_id_at_most, proj/src/id.cpp:9-52.
 * Outputs: indices (kcap, selection order), coeffs (kcap x n, ld kcap; rows
 * >= rank untouched), skeleton (m x kcap, ld m; may be NULL), rank, resid. */
int orc_column_id(const double* a, size_t m, size_t n, int mode, size_t k, double tol,
                  size_t kstep, int at_most, size_t kcap, int64_t* indices, double* coeffs,
                  double* skeleton, size_t* rank, double* residual_fro);

/* Gaussian-sketch SubID: Y = matmul(omega, a) (ell x n), then
 * column_id(Y, rule), then the fine skeleton select_columns(a, I) -- the
 * sub_id template of proj/src/id.cpp:54-60 with B replaced by Omega*A.
 * y (ell x n) may be NULL. */
int orc_sketch_id(const double* a, size_t m, size_t n, const double* omega, size_t ell, int mode,
                  size_t k, double tol, size_t kstep, size_t kcap, double* y, int64_t* indices,
                  double* coeffs, double* skeleton, size_t* rank, double* residual_fro);

/* ||a - skel*coeffs||_F^2 and ||a||_F^2 by the reference's route
 * (reconstruct = matmul, id.cpp:85-90; subtract + frobenius, metrics.cpp:14-21). */
int orc_error_terms(const double* a, size_t m, size_t n, const double* skel, size_t ldskel,
                    const double* coeffs, size_t ldc, size_t rank, double* err2, double* ref2);

int orc_rel_frob_error(const double* exact, const double* approx, size_t count, double* out);

/* SubsampleSpec::row_indices for a strided spec (proj/src/grid.cpp:91-130). */
int orc_row_indices(const size_t* dims, const int* periodic, const size_t* strides, size_t naxes,
                    int incl, int64_t* rows, size_t cap, size_t* count);

/* InterpOperator::from_spec(spec).apply(coarse) (proj/src/interp.cpp:19-100,
 * 168-186): fine (P x k) = M coarse (Pc x k), both column-major. */
int orc_interp_apply(const size_t* dims, const int* periodic, const size_t* strides, size_t naxes,
                     int incl, const double* coarse, size_t k, double* fine);
int orc_compression_factor(size_t m, size_t n, size_t stored, double* out); /* metrics.cpp:5-12 */

/* ---- workload generation (oracle/workload.c): the bench inputs on the CPU,
 * for the reference arm, which must not load the product library. ---- */

/* The 4096-entry quantile table Q of the discretised N(0,1) (Omega = Q/32). */
void orc_omega_table(int8_t* q);
/* Omega_s rows [row0, row0+ell) x m columns (ell x m, column-major): the
 * performance-mode sketch matrix (Philox4x32-7). */
void orc_philox_omega(uint64_t seed, uint64_t s, size_t row0, size_t ell, size_t m, double* out);

/* Same layout as spidgpu_field_spec (include/spidgpu.h). */
typedef struct orc_field_spec {
    int32_t kind; /* 0 TGV4, 1 TGV5, 2 MULTIMODE */
    int32_t n_modes;
    int64_t grid, block, snapshots;
    double t_end, nu, sigma, kappa_max, mode_amp;
    uint64_t seed;
    int64_t heavy_modes;
    double heavy_kmin;
} orc_field_spec;
/* Subdomains [first, first+batch) of the BASELINE synthetic fields (m x n
 * each, ld lda, stride strideA), on `threads` host threads. */
int orc_field_generate(const orc_field_spec* spec, int64_t first, int64_t batch, const uint8_t* is_heavy,
                       double* A, int64_t lda, int64_t strideA, int threads);

#ifdef __cplusplus
}
#endif

#endif
