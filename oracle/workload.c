/*
 * workload.c -- TEST INFRASTRUCTURE ONLY (see spid_oracle.h).
 *
 * CPU generation of the bench workload, so the reference arm
 * (bench.py --impl reference, cpu_baseline) can build its inputs without
 * loading the product library:
 *   - the performance-mode sketch matrix Omega_s: the
 *     4096-quantile table of N(0,1) rounded to multiples of 1/32, indexed by
 *     16-bit halves of Philox4x32-7 (Salmon et al., SC'11) with counter
 *     {k/8, r, s_lo, s_hi} and key {seed_lo, seed_hi}. This is an
 *     independent restatement of the definition (the table is recomputed
 *     here from the inverse normal CDF, not read from the product header);
 *     tests/test_workload_oracle.py checks both the table and Omega against
 *     the product's bit for bit;
 *   - the synthetic Taylor-Green fields of BASELINE configs 1-5, restating the
 *     conventions of the reference generators (x_i = 2 pi i / N,
 *     proj/src/datagen.cpp:16-28; axis 0 fastest, proj/include/spid/grid.hpp:
 *     10-12; blocks in make_block_domains order, proj/src/blocking.cpp:64-81)
 *     and the mode/noise definitions of DESIGN.md. libm and the device
 *     round transcendental functions differently, so fields agree with the
 *     device generator to ~1e-15 relative, not bitwise: they are the same
 *     workload, not the same bits.
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "spid_oracle.h"

/* ---- Omega ---------------------------------------------------------------- */

/* Inverse standard normal CDF: Acklam's rational approximation refined by one
 * Halley step on erfc (absolute error ~1e-15 over (0, 1)). */
static double inv_norm(double p) {
    static const double a[6] = {-3.969683028665376e+01, 2.209460984245205e+02, -2.759285104469687e+02,
                                1.383577518672690e+02,  -3.066479806614716e+01, 2.506628277459239e+00};
    static const double b[5] = {-5.447609879822406e+01, 1.615858368580409e+02, -1.556989798598866e+02,
                                6.680131188771972e+01,  -1.328068155288572e+01};
    static const double c[6] = {-7.784894002430293e-03, -3.223964580411365e-01, -2.400758277161838e+00,
                                -2.549732539343734e+00, 4.374664141464968e+00,  2.938163982698783e+00};
    static const double d[4] = {7.784695709041462e-03, 3.224671290700398e-01, 2.445134137142996e+00,
                                3.754408661907416e+00};
    const double plow = 0.02425, phigh = 1 - plow;
    double x;
    if (p < plow) {
        const double q = sqrt(-2 * log(p));
        x = (((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
            ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
    } else if (p <= phigh) {
        const double q = p - 0.5, r = q * q;
        x = (((((a[0] * r + a[1]) * r + a[2]) * r + a[3]) * r + a[4]) * r + a[5]) * q /
            (((((b[0] * r + b[1]) * r + b[2]) * r + b[3]) * r + b[4]) * r + 1);
    } else {
        const double q = sqrt(-2 * log(1 - p));
        x = -(((((c[0] * q + c[1]) * q + c[2]) * q + c[3]) * q + c[4]) * q + c[5]) /
            ((((d[0] * q + d[1]) * q + d[2]) * q + d[3]) * q + 1);
    }
    const double e = 0.5 * erfc(-x / sqrt(2.0)) - p;
    const double u = e * sqrt(2 * M_PI) * exp(x * x / 2);
    return x - u / (1 + x * u / 2);
}

void orc_omega_table(int8_t* q) {
    for (int i = 0; i < 4096; ++i) q[i] = (int8_t)rint(32.0 * inv_norm((i + 0.5) / 4096.0));
}

typedef struct {
    uint32_t x, y, z, w;
} ph4;

static ph4 philox7(ph4 c, uint32_t k0, uint32_t k1) {
    for (int i = 0; i < 7; ++i) {
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
        const ph4 n = {(uint32_t)(p1 >> 32) ^ c.y ^ k0, (uint32_t)p1, (uint32_t)(p0 >> 32) ^ c.w ^ k1, (uint32_t)p0};
        c = n;
        k0 += 0x9E3779B9u;
        k1 += 0xBB67AE85u;
    }
    return c;
}

void orc_philox_omega(uint64_t seed, uint64_t s, size_t row0, size_t ell, size_t m, double* out) {
    int8_t tab[4096];
    orc_omega_table(tab);
    for (size_t r = 0; r < ell; ++r)
        for (size_t ko = 0; ko * 8 < m; ++ko) {
            const ph4 c = {(uint32_t)ko, (uint32_t)(row0 + r), (uint32_t)s, (uint32_t)(s >> 32)};
            const ph4 v = philox7(c, (uint32_t)seed, (uint32_t)(seed >> 32));
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
            for (int j = 0; j < 8 && ko * 8 + j < m; ++j) {
                const uint32_t u = (j & 1) ? (w[j >> 1] >> 16) : (w[j >> 1] & 0xffffu);
                out[(ko * 8 + j) * ell + r] = tab[u >> 4] / 32.0;
            }
        }
}

/* ---- synthetic fields ----------------------------------------------------- */

static uint64_t mix_next(uint64_t* s) {
    uint64_t z = (*s += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
static double mix_unit(uint64_t* s) { return (double)(mix_next(s) >> 11) * 0x1.0p-53; }

/* Fourier modes of the multimode family: |kappa| in [kmin, kmax] integer
 * wavevectors, amplitude amp0 |kappa|^(-5/3), phases phi (velocity) and phi'
 * (pressure), unit direction orthogonal to kappa (divergence-free). */
static void make_modes(uint64_t seed, int count, double kmin, double kmax, double amp0, double* out) {
    uint64_t st = seed;
    const int K = (int)floor(kmax);
    const double two_pi = 6.283185307179586;
    for (int mi = 0; mi < count; ++mi) {
        double kx, ky, kz, k2;
        do {
            kx = floor(mix_unit(&st) * (2 * K + 1)) - K;
            ky = floor(mix_unit(&st) * (2 * K + 1)) - K;
            kz = floor(mix_unit(&st) * (2 * K + 1)) - K;
            k2 = kx * kx + ky * ky + kz * kz;
        } while (k2 == 0.0 || k2 > kmax * kmax || k2 < kmin * kmin);
        const double kn = sqrt(k2);
        const double amp = amp0 * pow(kn, -5.0 / 3.0);
        const double phi = two_pi * mix_unit(&st), phip = two_pi * mix_unit(&st);
        double d[3], dn;
        do {
            d[0] = 2 * mix_unit(&st) - 1;
            d[1] = 2 * mix_unit(&st) - 1;
            d[2] = 2 * mix_unit(&st) - 1;
            const double pr = (d[0] * kx + d[1] * ky + d[2] * kz) / k2;
            d[0] -= pr * kx;
            d[1] -= pr * ky;
            d[2] -= pr * kz;
            dn = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        } while (dn < 1e-3);
        const double md[9] = {kx, ky, kz, amp, phi, phip, d[0] / dn, d[1] / dn, d[2] / dn};
        memcpy(out + 9 * mi, md, sizeof md);
    }
}

typedef struct {
    const orc_field_spec* sp;
    int64_t first, batch;
    const uint8_t* is_heavy;
    double* A;
    int64_t lda, strideA;
    const double* modes; /* n_modes + heavy_modes, 9 doubles each */
    const double* ttab;  /* (cos(w t) D(t), sin(w t) D(t)) per (mode, snapshot) */
    int64_t next;        /* work counter: (subdomain, 512-point chunk) */
    pthread_mutex_t mu;
} field_job;

static void field_point(const field_job* J, int64_t sl, int64_t pt) {
    const orc_field_spec* p = J->sp;
    const int64_t b = p->block, b3 = b * b * b, nb = p->grid / b;
    const int nq = p->kind == 0 ? 4 : 5;
    const double h = 6.283185307179586 / (double)p->grid;
    const int64_t gb = J->first + sl;
    const int64_t bx = gb % nb, by = (gb / nb) % nb, bz = gb / (nb * nb);
    const int64_t ix = bx * b + pt % b, iy = by * b + (pt / b) % b, iz = bz * b + pt / (b * b);
    const double x = h * ix, y = h * iy, z = h * iz;
    const double sx = sin(x), cx = cos(x), sy = sin(y), cy = cos(y), cz = cos(z);
    const double pbase = (1.0 / 16.0) * (cos(2 * x) + cos(2 * y)) * (cos(2 * z) + 2.0);
    const int heavy = J->is_heavy && J->is_heavy[sl];
    const int nmodes = (int)p->n_modes + (heavy ? (int)p->heavy_modes : 0);
    double* col0 = J->A + sl * J->strideA + pt;
    const uint64_t gpt = (uint64_t)gb * (uint64_t)b3 + (uint64_t)pt;
    double sp_c0[512], sp_s0[512], sp_c1[512], sp_s1[512];
    const double* md_of[512];
    for (int mi = 0; mi < nmodes && mi < 512; ++mi) {
        const double* md = mi < p->n_modes ? J->modes + 9 * mi : J->modes + 9 * (p->n_modes + (mi - p->n_modes));
        const double th = md[0] * x + md[1] * y + md[2] * z;
        sp_s0[mi] = sin(th + md[4]);
        sp_c0[mi] = cos(th + md[4]);
        sp_s1[mi] = sin(th + md[5]);
        sp_c1[mi] = cos(th + md[5]);
        md_of[mi] = md;
    }
    for (int64_t j = 0; j < p->snapshots; ++j) {
        const double t = p->snapshots > 1 ? p->t_end * j / (p->snapshots - 1) : 0.0;
        const double F = exp(-2.0 * p->nu * t);
        double u = sx * cy * cz * F, v = -cx * sy * cz * F, w = 0.0, pr = pbase * F * F;
        for (int mi = 0; mi < nmodes; ++mi) {
            const double* md = md_of[mi];
            const double tc = J->ttab[(mi * p->snapshots + j) * 2], ts = J->ttab[(mi * p->snapshots + j) * 2 + 1];
            const double cv = md[3] * (sp_c0[mi] * tc + sp_s0[mi] * ts);
            u += md[6] * cv;
            v += md[7] * cv;
            w += md[8] * cv;
            pr += md[3] * (sp_c1[mi] * tc + sp_s1[mi] * ts);
        }
        double q[5];
        if (p->kind == 0) {
            q[0] = u, q[1] = v, q[2] = w, q[3] = pr;
        } else {
            const double rho = 1.0 + 0.01 * pr;
            q[0] = rho, q[1] = u, q[2] = v, q[3] = w;
            q[4] = pr / 0.4 + 0.5 * rho * (u * u + v * v + w * w);
        }
        double* colj = col0 + j * J->lda;
        for (int qi = 0; qi < nq; ++qi) {
            double val = q[qi];
            if (p->sigma > 0.0) {
                /* N(0,1) by Box-Muller in fp32 from Philox counter {j/4, 0x9E37, id, id_hi} */
                const uint64_t sid = gpt * 8 + (uint64_t)qi, sd = p->seed ^ 0x5DEECE66DULL;
                const ph4 c = {(uint32_t)(j >> 2), 0x9E37u, (uint32_t)sid, (uint32_t)(sid >> 32)};
                const ph4 r = philox7(c, (uint32_t)sd, (uint32_t)(sd >> 32));
                const float kInv = 2.3283064365386963e-10f;
                const int pair = (int)((j & 3) >> 1);
                const float u1 = ((float)(pair ? r.z : r.x) + 1.0f) * kInv;
                const float u2 = (float)(pair ? r.w : r.y) * kInv;
                float xr = -2.0f * logf(u1);
                if (xr < 1e-30f) xr = 1e-30f;
                const float rr = sqrtf(xr), ang = 6.2831853071795865f * u2;
                const float nz = (j & 1) ? rr * sinf(ang) : rr * cosf(ang);
                val += p->sigma * (double)nz;
            }
            colj[qi * b3] = val;
        }
    }
}

static void* field_worker(void* arg) {
    field_job* J = (field_job*)arg;
    const int64_t b3 = J->sp->block * J->sp->block * J->sp->block;
    const int64_t chunks = (b3 + 511) / 512, total = J->batch * chunks;
    for (;;) {
        pthread_mutex_lock(&J->mu);
        const int64_t w = J->next++;
        pthread_mutex_unlock(&J->mu);
        if (w >= total) return NULL;
        const int64_t sl = w / chunks, p0 = (w % chunks) * 512;
        for (int64_t pt = p0; pt < p0 + 512 && pt < b3; ++pt) field_point(J, sl, pt);
    }
}

int orc_field_generate(const orc_field_spec* sp, int64_t first, int64_t batch, const uint8_t* is_heavy,
                       double* A, int64_t lda, int64_t strideA, int threads) {
    if (!sp || !A || sp->grid < 1 || sp->block < 1 || sp->grid % sp->block || sp->snapshots < 1)
        return SPID_INVALID_ARGUMENT;
    const int nq = sp->kind == 0 ? 4 : 5;
    const int64_t b3 = sp->block * sp->block * sp->block, nb = sp->grid / sp->block;
    if (lda < nq * b3 || strideA < lda * sp->snapshots || first < 0 || first + batch > nb * nb * nb)
        return SPID_INVALID_ARGUMENT;
    if (sp->n_modes + sp->heavy_modes > 512) return SPID_INVALID_ARGUMENT;
    double* modes = NULL;
    const int64_t nm = sp->kind == 2 ? sp->n_modes + sp->heavy_modes : 0;
    if (nm > 0) {
        modes = (double*)malloc(sizeof(double) * 9 * (size_t)nm);
        if (!modes) return SPID_INVALID_ARGUMENT;
        make_modes(sp->seed, (int)sp->n_modes, 1.0, sp->kappa_max, sp->mode_amp, modes);
        if (sp->heavy_modes > 0)
            make_modes(sp->seed ^ 0xC0FFEE1234ULL, (int)sp->heavy_modes, sp->heavy_kmin, sp->kappa_max,
                       sp->mode_amp, modes + 9 * sp->n_modes);
    }
    orc_field_spec local = *sp;
    if (sp->kind != 2) local.n_modes = local.heavy_modes = 0;
    /* time factors of every mode: cos(|k| t) exp(-nu |k|^2 t), sin(...) */
    double* ttab = (double*)malloc(sizeof(double) * 2 * (size_t)(nm > 0 ? nm : 1) * (size_t)sp->snapshots);
    if (!ttab) {
        free(modes);
        return SPID_INVALID_ARGUMENT;
    }
    for (int64_t mi = 0; mi < nm; ++mi)
        for (int64_t j = 0; j < sp->snapshots; ++j) {
            const double* md = modes + 9 * mi;
            const double k2 = md[0] * md[0] + md[1] * md[1] + md[2] * md[2];
            const double t = sp->snapshots > 1 ? sp->t_end * j / (sp->snapshots - 1) : 0.0;
            const double D = exp(-sp->nu * k2 * t);
            ttab[(mi * sp->snapshots + j) * 2] = cos(sqrt(k2) * t) * D;
            ttab[(mi * sp->snapshots + j) * 2 + 1] = sin(sqrt(k2) * t) * D;
        }
    field_job J = {&local, first, batch, is_heavy, A, lda, strideA, modes, ttab, 0, PTHREAD_MUTEX_INITIALIZER};
    int nt = threads < 1 ? 1 : threads;
    if (nt > 256) nt = 256;
    pthread_t th[256];
    for (int t = 0; t < nt; ++t) pthread_create(&th[t], NULL, field_worker, &J);
    for (int t = 0; t < nt; ++t) pthread_join(th[t], NULL);
    free(ttab);
    free(modes);
    return SPID_OK;
}
