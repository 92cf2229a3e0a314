/*
 * spid_oracle.c -- TEST INFRASTRUCTURE ONLY (see spid_oracle.h).
 *
 * Plain-C restatement of the reference SPID path; every function cites the
 * reference file:line it follows. Compiled with -ffp-contract=off and no
 * -march so each `s += x*y` is a separately rounded multiply and add, as in
 * the reference's x86-64 build: outputs are bit-identical to oracle/_ref.
 */
#include "spid_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define ZERO_FLOOR 1e-300    /* qr.cpp:11 */
#define COLLAPSE_REL 1e-14   /* qr.cpp:12 */

/* ---- rng: proj/include/spid/rng.hpp:16-26 ------------------------------- */
uint64_t orc_splitmix_next(uint64_t* state) {
    uint64_t z = (*state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

static double next_unit(uint64_t* st) { /* rng.hpp:22 */
    return (double)(orc_splitmix_next(st) >> 11) * 0x1.0p-53;
}

void orc_seeded_sym(uint64_t seed, double* out, size_t count) {
    /* proj/tests/common.hpp:13-19: column-major fill with next_sym() */
    uint64_t st = seed;
    for (size_t i = 0; i < count; ++i) out[i] = 2.0 * next_unit(&st) - 1.0;
}

void orc_gaussian(uint64_t seed, double* out, size_t count) {
    /* Box-Muller over SplitMix64 uniforms; u1 in (0,1] avoids log(0). */
    uint64_t st = seed;
    const double two_pi = 6.283185307179586476925286766559;
    for (size_t i = 0; i < count; i += 2) {
        const double u1 = 1.0 - next_unit(&st);
        const double u2 = next_unit(&st);
        const double r = sqrt(-2.0 * log(u1));
        out[i] = r * cos(two_pi * u2);
        if (i + 1 < count) out[i + 1] = r * sin(two_pi * u2);
    }
}

/* ---- dense_matrix.cpp -------------------------------------------------- */
void orc_matmul(const double* a, size_t ar, size_t ac, const double* b, size_t bc, double* c) {
    /* dense_matrix.cpp:38-53: j-k-i order, skip exact-zero b(k,j) */
    memset(c, 0, ar * bc * sizeof(double));
    for (size_t j = 0; j < bc; ++j) {
        double* cj = c + j * ar;
        for (size_t k = 0; k < ac; ++k) {
            const double bkj = b[j * ac + k];
            if (bkj == 0.0) continue;
            const double* ak = a + k * ar;
            for (size_t i = 0; i < ar; ++i) cj[i] += ak[i] * bkj;
        }
    }
}

double orc_frobenius(const double* a, size_t count) { /* dense_matrix.cpp:113-120 */
    double sum = 0.0;
    for (size_t i = 0; i < count; ++i) sum += a[i] * a[i];
    return sqrt(sum);
}

double orc_dot(const double* x, const double* y, size_t n) { /* dense_matrix.cpp:136-140 */
    double s = 0.0;
    for (size_t i = 0; i < n; ++i) s += x[i] * y[i];
    return s;
}

double orc_norm2(const double* x, size_t n) { return sqrt(orc_dot(x, x, n)); } /* :142 */

static int all_finite(const double* a, size_t count) { /* dense_matrix.cpp:32-36 */
    for (size_t i = 0; i < count; ++i)
        if (!isfinite(a[i])) return 0;
    return 1;
}

/* ---- rank rule validation: qr.hpp:16-24 -------------------------------- */
static int check_rule(int mode, size_t k, double tol, size_t kstep) {
    if (mode == ORC_RULE_FIXED) return k >= 1 ? SPID_OK : SPID_BAD_RANK_RULE;
    if (mode == ORC_RULE_TOL) return (tol > 0.0 && tol < 1.0) ? SPID_OK : SPID_BAD_RANK_RULE;
    if (mode == ORC_RULE_BLOCKED)
        return (k >= 1 && kstep >= 1 && tol > 0.0 && tol < 1.0) ? SPID_OK : SPID_BAD_RANK_RULE;
    return SPID_BAD_RANK_RULE;
}

/* ---- qr.cpp:29-124 ------------------------------------------------------ */
int orc_qr(const double* a, size_t m, size_t n, int mode, size_t k, double tol, size_t kstep,
           int strict, size_t kcap, double* q_out, double* r_out, int64_t* pivots_out,
           size_t* rank_out, double* resid_out) {
    int st = check_rule(mode, k, tol, kstep);
    if (st) return st;
    if (m == 0 || n == 0) return SPID_EMPTY_MATRIX;
    const size_t max_rank = m < n ? m : n;
    if (!all_finite(a, m * n)) return SPID_NON_FINITE_INPUT;              /* qr.cpp:34-35 */
    if (mode == ORC_RULE_FIXED && k > max_rank) return SPID_RANK_UNREACHABLE; /* :37-38 */

    size_t step_limit = mode == ORC_RULE_TOL ? max_rank : k;              /* :53-54 */
    if (mode == ORC_RULE_BLOCKED && step_limit > max_rank) step_limit = max_rank;
    if (kcap < step_limit) return SPID_INVALID_ARGUMENT;

    double* work = (double*)malloc(m * n * sizeof(double));               /* :41 */
    size_t* piv = (size_t*)malloc(n * sizeof(size_t));
    double* r = (double*)calloc(step_limit * n, sizeof(double));          /* :57 row-major */
    double* nrm = (double*)malloc(n * sizeof(double));
    memcpy(work, a, m * n * sizeof(double));
    for (size_t j = 0; j < n; ++j) piv[j] = j;                            /* :44-45 */

    double max_init = 0.0;                                                 /* :47-51 */
    for (size_t j = 0; j < n; ++j) {
        const double v = orc_norm2(work + j * m, m);
        if (v > max_init) max_init = v;
    }
    /* BLOCKED rule compares the trailing residual
     * against ||Y||_F, taken as the column-order sum of per-column
     * sequential sums of squares. */
    double yfro = 0.0;
    if (mode == ORC_RULE_BLOCKED) {
        for (size_t j = 0; j < n; ++j) yfro += orc_dot(a + j * m, a + j * m, m);
        yfro = sqrt(yfro);
    }
    if (max_init < ZERO_FLOOR) {
        st = SPID_ZERO_MATRIX;
        goto done;
    }

    size_t rank = 0;
    for (size_t s = 0; s < step_limit; ++s) {
        double best_norm = -1.0;                                           /* :64-72 */
        size_t best = s;
        for (size_t j = s; j < n; ++j) {
            const double nj = orc_norm2(work + j * m, m);
            nrm[j] = nj;
            if (nj > best_norm || (nj == best_norm && piv[j] < piv[best])) {
                best_norm = nj;
                best = j;
            }
        }
        if (mode == ORC_RULE_TOL && best_norm <= tol * max_init) break;  /* :74-76 */
        if (mode == ORC_RULE_BLOCKED && s > 0 && s % kstep == 0) {
            /* residual_fro after s steps, summed in position order as :111-115 */
            double rsq = 0.0;
            for (size_t j = s; j < n; ++j) rsq += nrm[j] * nrm[j];
            if (sqrt(rsq) <= tol * yfro) break;
        }
        if (best_norm < COLLAPSE_REL * max_init) {                         /* :77-81 */
            if (mode == ORC_RULE_FIXED && strict) {
                st = SPID_RANK_UNREACHABLE;
                goto done;
            }
            break;
        }
        if (best != s) {                                                   /* :83-87 */
            double* ws = work + s * m;
            double* wb = work + best * m;
            for (size_t i = 0; i < m; ++i) {
                const double t = ws[i];
                ws[i] = wb[i];
                wb[i] = t;
            }
            const size_t tp = piv[s];
            piv[s] = piv[best];
            piv[best] = tp;
            for (size_t i = 0; i < s; ++i) {
                const double t = r[i * n + s];
                r[i * n + s] = r[i * n + best];
                r[i * n + best] = t;
            }
        }
        double* qs = work + s * m;                                         /* :89-92 */
        const double pivot_norm = orc_norm2(qs, m);
        r[s * n + s] = pivot_norm;
        for (size_t i = 0; i < m; ++i) qs[i] /= pivot_norm;
        for (size_t j = s + 1; j < n; ++j) {                               /* :94-102 */
            double* wj = work + j * m;
            const double r1 = orc_dot(qs, wj, m);
            for (size_t i = 0; i < m; ++i) wj[i] -= r1 * qs[i];
            const double r2 = orc_dot(qs, wj, m);
            for (size_t i = 0; i < m; ++i) wj[i] -= r2 * qs[i];
            r[s * n + j] = r1 + r2;
        }
        rank = s + 1;
    }
    if (rank == 0) {                                                       /* :108-109 */
        st = SPID_ZERO_MATRIX;
        goto done;
    }
    double residual_sq = 0.0;                                              /* :111-115 */
    for (size_t j = rank; j < n; ++j) {
        const double nj = orc_norm2(work + j * m, m);
        residual_sq += nj * nj;
    }
    if (q_out)
        for (size_t j = 0; j < rank; ++j) memcpy(q_out + j * m, work + j * m, m * sizeof(double));
    if (r_out)
        for (size_t j = 0; j < n; ++j)
            for (size_t i = 0; i < rank; ++i) r_out[j * kcap + i] = r[i * n + j];
    if (pivots_out)
        for (size_t j = 0; j < n; ++j) pivots_out[j] = (int64_t)piv[j];
    if (rank_out) *rank_out = rank;
    if (resid_out) *resid_out = sqrt(residual_sq);
done:
    free(work);
    free(piv);
    free(r);
    free(nrm);
    return st;
}

int orc_solve_upper(const double* r11, size_t k, size_t ldr, const double* rhs, size_t ncols,
                    double* x) {
    /* qr.cpp:128-151 */
    double max_diag = 0.0;
    for (size_t i = 0; i < k; ++i) {
        const double d = fabs(r11[i * ldr + i]);
        if (d > max_diag) max_diag = d;
    }
    for (size_t i = 0; i < k; ++i)
        if (fabs(r11[i * ldr + i]) < 1e-14 * max_diag || max_diag == 0.0)
            return SPID_SINGULAR_PIVOT;
    for (size_t col = 0; col < ncols; ++col) {
        for (size_t ii = k; ii-- > 0;) {
            double sum = rhs[col * k + ii];
            for (size_t j = ii + 1; j < k; ++j) sum -= r11[j * ldr + ii] * x[col * k + j];
            x[col * k + ii] = sum / r11[ii * ldr + ii];
        }
    }
    return SPID_OK;
}

/* ---- id.cpp:9-52 -------------------------------------------------------- */
int orc_column_id(const double* a, size_t m, size_t n, int mode, size_t k, double tol,
                  size_t kstep, int at_most, size_t kcap, int64_t* indices, double* coeffs,
                  double* skeleton, size_t* rank_out, double* resid_out) {
    if (m == 0 || n == 0) return SPID_EMPTY_MATRIX;
    int st = check_rule(mode, k, tol, kstep);
    if (st) return st;
    if (!all_finite(a, m * n)) return SPID_NON_FINITE_INPUT;              /* id.cpp:41-42 */
    const size_t mn = m < n ? m : n;
    size_t kk = k;
    if (at_most) {                                                         /* qr.cpp:22-25 */
        if (mode != ORC_RULE_FIXED) return SPID_BAD_RANK_RULE;
        kk = k < mn ? k : mn;
        if (kk < 1) kk = 1;
    }
    size_t scap = mode == ORC_RULE_TOL ? mn : kk;
    if (scap > mn) scap = mn; /* FIXED k > mn raises RankUnreachable inside orc_qr */
    const size_t rcap = mode == ORC_RULE_FIXED && kk > mn ? kk : scap;
    double* r = (double*)calloc(rcap * n, sizeof(double));
    int64_t* piv = (int64_t*)malloc(n * sizeof(int64_t));
    size_t rank = 0;
    double resid = 0.0;
    st = orc_qr(a, m, n, mode, kk, tol, kstep, !at_most, rcap, NULL, r, piv, &rank, &resid);
    if (st) goto done;
    if (kcap < rank) {
        st = SPID_INVALID_ARGUMENT;
        goto done;
    }
    /* build_coeffs, id.cpp:9-28: C(:,piv[j]) = e_j for j<k, X(:,j-k) after */
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i < rank; ++i) coeffs[j * kcap + i] = 0.0;
    for (size_t j = 0; j < rank; ++j) coeffs[(size_t)piv[j] * kcap + j] = 1.0;
    if (rank < n) {
        const size_t nr = n - rank;
        double* rhs = (double*)malloc(rank * nr * sizeof(double));
        double* x = (double*)malloc(rank * nr * sizeof(double));
        for (size_t j = rank; j < n; ++j)
            for (size_t i = 0; i < rank; ++i) rhs[(j - rank) * rank + i] = r[j * rcap + i];
        st = orc_solve_upper(r, rank, rcap, rhs, nr, x);
        if (!st)
            for (size_t j = rank; j < n; ++j)
                for (size_t i = 0; i < rank; ++i)
                    coeffs[(size_t)piv[j] * kcap + i] = x[(j - rank) * rank + i];
        free(rhs);
        free(x);
        if (st) goto done;
    }
    for (size_t j = 0; j < n; ++j)                                         /* id.cpp:25-26 */
        for (size_t i = 0; i < rank; ++i)
            if (!isfinite(coeffs[j * kcap + i])) {
                st = SPID_NON_FINITE_COEFFS;
                goto done;
            }
    for (size_t j = 0; j < rank; ++j) indices[j] = piv[j];                 /* id.cpp:31 */
    if (skeleton)                                                          /* id.cpp:33 */
        for (size_t j = 0; j < rank; ++j)
            memcpy(skeleton + j * m, a + (size_t)piv[j] * m, m * sizeof(double));
    if (rank_out) *rank_out = rank;
    if (resid_out) *resid_out = resid;
done:
    free(r);
    free(piv);
    return st;
}

int orc_sketch_id(const double* a, size_t m, size_t n, const double* omega, size_t ell, int mode,
                  size_t k, double tol, size_t kstep, size_t kcap, double* y_out,
                  int64_t* indices, double* coeffs, double* skeleton, size_t* rank,
                  double* residual_fro) {
    if (m == 0 || n == 0 || ell == 0) return SPID_EMPTY_MATRIX;
    double* y = (double*)malloc(ell * n * sizeof(double));
    orc_matmul(omega, ell, m, a, n, y);                     /* dense_matrix.cpp:38-53 */
    if (y_out) memcpy(y_out, y, ell * n * sizeof(double));
    int st = orc_column_id(y, ell, n, mode, k, tol, kstep, 0, kcap, indices, coeffs, NULL, rank,
                           residual_fro);
    if (!st && skeleton)                                    /* id.cpp:57-58: fine skeleton */
        for (size_t j = 0; j < *rank; ++j)
            memcpy(skeleton + j * m, a + (size_t)indices[j] * m, m * sizeof(double));
    free(y);
    return st;
}

int orc_error_terms(const double* a, size_t m, size_t n, const double* skel, size_t ldskel,
                    const double* coeffs, size_t ldc, size_t rank, double* err2, double* ref2) {
    /* reconstruct (id.cpp:85-90) = matmul(skeleton, coeffs); then subtract
     * (dense_matrix.cpp:62-69) and the sequential frobenius sums (:113-120). */
    if (rank == 0) return SPID_EMPTY_SELECTION;
    double* s = (double*)malloc(m * rank * sizeof(double));
    double* c = (double*)malloc(rank * n * sizeof(double));
    double* rec = (double*)malloc(m * n * sizeof(double));
    for (size_t j = 0; j < rank; ++j) memcpy(s + j * m, skel + j * ldskel, m * sizeof(double));
    for (size_t j = 0; j < n; ++j)
        for (size_t i = 0; i < rank; ++i) c[j * rank + i] = coeffs[j * ldc + i];
    orc_matmul(s, m, rank, c, n, rec);
    double e = 0.0, f = 0.0;
    for (size_t i = 0; i < m * n; ++i) {
        const double d = a[i] - rec[i];
        e += d * d;
        f += a[i] * a[i];
    }
    *err2 = e;
    *ref2 = f;
    free(s);
    free(c);
    free(rec);
    return SPID_OK;
}

int orc_rel_frob_error(const double* exact, const double* approx, size_t count, double* out) {
    /* metrics.cpp:14-21 */
    const double ref = orc_frobenius(exact, count);
    if (ref == 0.0) return SPID_ZERO_REFERENCE;
    double sum = 0.0;
    for (size_t i = 0; i < count; ++i) {
        const double d = exact[i] - approx[i];
        sum += d * d;
    }
    *out = sqrt(sum) / ref;
    return SPID_OK;
}

int orc_compression_factor(size_t m, size_t n, size_t stored, double* out) {
    /* metrics.cpp:5-12 */
    if (m == 0 || n == 0) return SPID_ZERO_DENOMINATOR;
    if (stored == 0) return SPID_ZERO_DENOMINATOR;
    *out = (double)m * (double)n / (double)stored;
    return SPID_OK;
}

/* ---- strided SubsampleSpec rows + multilinear interpolation -------------- */
/* Coarse index list of one axis (grid.cpp:91-106). Returns its length. */
static size_t axis_coarse(size_t dim, size_t stride, int periodic, int incl, size_t* out) {
    size_t n = 0;
    for (size_t i = 0; i < dim; i += stride) out[n++] = i;
    if (incl && !periodic && out[n - 1] != dim - 1) out[n++] = dim - 1;
    return n;
}

int orc_row_indices(const size_t* dims, const int* periodic, const size_t* strides, size_t naxes,
                    int incl, int64_t* rows, size_t cap, size_t* count) {
    /* grid.cpp:108-130: axis 0 fastest */
    if (naxes < 1 || naxes > 3) return SPID_BAD_SUBSAMPLE_SPEC;
    size_t ax[3][4096], na[3] = {1, 1, 1}, d[3] = {1, 1, 1};
    ax[1][0] = ax[2][0] = 0;
    for (size_t a = 0; a < naxes; ++a) {
        if (dims[a] < 1 || dims[a] > 4096 || strides[a] < 1) return SPID_BAD_SUBSAMPLE_SPEC; /* structured_block: >= 1 */
        d[a] = dims[a];
        na[a] = axis_coarse(dims[a], strides[a], periodic[a], incl, ax[a]);
    }
    size_t c = 0;
    for (size_t i2 = 0; i2 < na[2]; ++i2)
        for (size_t i1 = 0; i1 < na[1]; ++i1)
            for (size_t i0 = 0; i0 < na[0]; ++i0) {
                if (c < cap) rows[c] = (int64_t)(ax[0][i0] + d[0] * ax[1][i1] + d[0] * d[1] * ax[2][i2]);
                ++c;
            }
    *count = c;
    return SPID_OK;
}

typedef struct {
    size_t n, pos[2];
    double w[2];
} orc_axisw;

/* interp.cpp:19-41 */
static int axis_weights(size_t f, const size_t* coarse, size_t nc, size_t dim, int periodic,
                        orc_axisw* out) {
    size_t lb = 0;
    while (lb < nc && coarse[lb] < f) ++lb; /* lower_bound */
    if (lb < nc && coarse[lb] == f) {
        out->n = 1;
        out->pos[0] = lb;
        out->w[0] = 1.0;
        return 0;
    }
    if (lb == nc) {
        if (!periodic) return 1; /* ExtrapolationRequired */
        const size_t last = nc - 1;
        const double cell = (double)(dim - coarse[last] + coarse[0]);
        const double w = (double)(f - coarse[last]) / cell;
        out->n = 2;
        out->pos[0] = last;
        out->w[0] = 1.0 - w;
        out->pos[1] = 0;
        out->w[1] = w;
        return 0;
    }
    const size_t hi = lb, lo = hi - 1;
    const double w = (double)(f - coarse[lo]) / (double)(coarse[hi] - coarse[lo]);
    out->n = 2;
    out->pos[0] = lo;
    out->w[0] = 1.0 - w;
    out->pos[1] = hi;
    out->w[1] = w;
    return 0;
}

/* fine (P x k) = M * coarse (Pc x k): InterpOperator::from_spec (interp.cpp:
 * 45-100: tensor-product weights, duplicates merged in (a2, a1, a0) order,
 * columns ascending) applied as apply_column (interp.cpp:177-186). */
int orc_interp_apply(const size_t* dims, const int* periodic, const size_t* strides, size_t naxes,
                     int incl, const double* coarse, size_t k, double* fine) {
    size_t ax[3][4096], na[3] = {1, 1, 1}, d[3] = {1, 1, 1};
    for (size_t a = 0; a < naxes; ++a) {
        if (dims[a] < 1 || dims[a] > 4096 || strides[a] < 1) return SPID_BAD_SUBSAMPLE_SPEC; /* structured_block: >= 1 */
        d[a] = dims[a];
        na[a] = axis_coarse(dims[a], strides[a], periodic[a], incl, ax[a]);
    }
    const size_t P = d[0] * d[1] * d[2], Pc = na[0] * na[1] * na[2];
    const orc_axisw unit = {1, {0, 0}, {1.0, 0.0}};
    for (size_t i2 = 0; i2 < d[2]; ++i2) {
        orc_axisw w2 = unit, w1 = unit, w0;
        if (naxes > 2 && axis_weights(i2, ax[2], na[2], d[2], periodic[2], &w2)) return SPID_GEOMETRY_MISMATCH;
        for (size_t i1 = 0; i1 < d[1]; ++i1) {
            if (naxes > 1 && axis_weights(i1, ax[1], na[1], d[1], periodic[1], &w1)) return SPID_GEOMETRY_MISMATCH;
            for (size_t i0 = 0; i0 < d[0]; ++i0) {
                if (axis_weights(i0, ax[0], na[0], d[0], periodic[0], &w0)) return SPID_GEOMETRY_MISMATCH;
                size_t col[8];
                double wt[8];
                size_t ne = 0;
                for (size_t b2 = 0; b2 < w2.n; ++b2)
                    for (size_t b1 = 0; b1 < w1.n; ++b1)
                        for (size_t b0 = 0; b0 < w0.n; ++b0) {
                            size_t c = w0.pos[b0];
                            if (naxes > 1) c += na[0] * w1.pos[b1];
                            if (naxes > 2) c += na[0] * na[1] * w2.pos[b2];
                            const double v = w0.w[b0] * w1.w[b1] * w2.w[b2];
                            size_t at = ne;
                            for (size_t q = 0; q < ne; ++q)
                                if (col[q] == c) at = q;
                            if (at == ne) {
                                col[ne] = c;
                                wt[ne++] = 0.0 + v;
                            } else {
                                wt[at] += v;
                            }
                        }
                for (size_t a = 1; a < ne; ++a) /* std::map order: ascending column */
                    for (size_t b = a; b > 0 && col[b - 1] > col[b]; --b) {
                        const size_t tc = col[b];
                        col[b] = col[b - 1];
                        col[b - 1] = tc;
                        const double tw = wt[b];
                        wt[b] = wt[b - 1];
                        wt[b - 1] = tw;
                    }
                const size_t r = i0 + d[0] * (i1 + d[1] * i2);
                for (size_t t = 0; t < k; ++t) {
                    double v = 0.0;
                    for (size_t a = 0; a < ne; ++a) v += wt[a] * coarse[t * Pc + col[a]];
                    fine[t * P + r] = v;
                }
            }
        }
    }
    return SPID_OK;
}
