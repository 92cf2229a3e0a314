// fields.cu -- synthetic Taylor-Green-vortex snapshot matrices, generated in
// place in HBM (bench / test input only; not a reference interface).
//
// Conventions follow the reference generators: structured axes span [0, 2pi)
// with x_i = 2*pi*i/N (proj/src/datagen.cpp:16-28), points flatten axis 0
// fastest (proj/include/spid/grid.hpp:10-12), blocks are ordered axis 0
// fastest with rows inside a block axis 0 fastest (proj/src/blocking.cpp:
// 64-81). Rows of a subdomain matrix are QoI-major: row = q*b^3 + p.
//
// Families (BASELINE.json configs; choices not fixed there are in DESIGN.md):
//   TGV4      u = sin x cos y cos z F, v = -cos x sin y cos z F, w = 0,
//             p = (1/16)(cos 2x + cos 2y)(cos 2z + 2) F^2, F = exp(-2 nu t)
//   TGV5      rho = 1 + 0.01 p, u, v, w, E = p/0.4 + rho|u|^2/2
//   MULTIMODE TGV5 with (u, v, w, p) += sum over Fourier modes of
//             a_k d_k cos(k.x + phi_k - |k| t) exp(-nu |k|^2 t)   (p: phase phi'_k)
// plus additive N(0, sigma^2) noise from a counter-based generator.
#include <math.h>

#include "common.cuh"
#include "kernels.h"
#include "philox.cuh"

namespace spidgpu {

namespace {

constexpr int kTb = 8;  // snapshots per register block
constexpr int kModeStride = 9;  // kx ky kz amp phi phip dx dy dz

__global__ void __launch_bounds__(256) field_kernel(FieldParams p, const double* __restrict__ tab) {
    const int64_t b = p.block, b3 = b * b * b;
    const int64_t nb = p.grid / b;
    const int64_t total = p.batch * b3;
    const int nq = p.kind == 0 ? 4 : 5;
    const double two_pi = 6.283185307179586;
    const double h = two_pi / static_cast<double>(p.grid);
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t sl = e / b3, pt = e % b3;
        const int64_t gb = p.first + sl;
        const int64_t bx = gb % nb, by = (gb / nb) % nb, bz = gb / (nb * nb);
        const int64_t ix = bx * b + pt % b, iy = by * b + (pt / b) % b, iz = bz * b + pt / (b * b);
        const double x = h * ix, y = h * iy, z = h * iz;
        double sx, cx, sy, cy, sz, cz;
        sincos(x, &sx, &cx);
        sincos(y, &sy, &cy);
        sincos(z, &sz, &cz);
        const double pbase = (1.0 / 16.0) * (cos(2 * x) + cos(2 * y)) * (cos(2 * z) + 2.0);
        const int nmodes = p.n_modes + ((p.is_heavy && p.is_heavy[sl]) ? p.n_heavy : 0);
        double* col0 = p.A + sl * p.strideA + pt;
        const uint64_t gpt = static_cast<uint64_t>(gb) * static_cast<uint64_t>(b3) + pt;
        for (int64_t j0 = 0; j0 < p.snapshots; j0 += kTb) {
            double u[kTb], v[kTb], w[kTb], pr[kTb];
#pragma unroll
            for (int jj = 0; jj < kTb; ++jj) {
                const int64_t j = j0 + jj < p.snapshots ? j0 + jj : p.snapshots - 1;
                const double t = p.snapshots > 1 ? p.t_end * j / (p.snapshots - 1) : 0.0;
                const double F = exp(-2.0 * p.nu * t);
                u[jj] = sx * cy * cz * F;
                v[jj] = -cx * sy * cz * F;
                w[jj] = 0.0;
                pr[jj] = pbase * F * F;
            }
            for (int mi = 0; mi < nmodes; ++mi) {
                const double* md = mi < p.n_modes ? p.modes + mi * kModeStride
                                                  : p.heavy_modes + (mi - p.n_modes) * kModeStride;
                const double th = md[0] * x + md[1] * y + md[2] * z;
                double s0, c0, s1, c1;
                sincos(th + md[4], &s0, &c0);
                sincos(th + md[5], &s1, &c1);
                const double amp = md[3];
#pragma unroll
                for (int jj = 0; jj < kTb; ++jj) {
                    const int64_t j = j0 + jj < p.snapshots ? j0 + jj : p.snapshots - 1;
                    // tab: (cos(w t) D(t), sin(w t) D(t)) per (mode, snapshot)
                    const double tc = tab[(static_cast<int64_t>(mi) * p.snapshots + j) * 2];
                    const double ts = tab[(static_cast<int64_t>(mi) * p.snapshots + j) * 2 + 1];
                    // cos(th + phi - w t) = cos(th+phi) cos(wt) + sin(th+phi) sin(wt)
                    const double cv = amp * (c0 * tc + s0 * ts);
                    u[jj] += md[6] * cv;
                    v[jj] += md[7] * cv;
                    w[jj] += md[8] * cv;
                    pr[jj] += amp * (c1 * tc + s1 * ts);
                }
            }
#pragma unroll
            for (int jj = 0; jj < kTb; ++jj) {
                const int64_t j = j0 + jj;
                if (j >= p.snapshots) break;
                double q[5];
                if (p.kind == 0) {
                    q[0] = u[jj];
                    q[1] = v[jj];
                    q[2] = w[jj];
                    q[3] = pr[jj];
                } else {
                    const double rho = 1.0 + 0.01 * pr[jj];
                    q[0] = rho;
                    q[1] = u[jj];
                    q[2] = v[jj];
                    q[3] = w[jj];
                    q[4] = pr[jj] / 0.4 + 0.5 * rho * (u[jj] * u[jj] + v[jj] * v[jj] + w[jj] * w[jj]);
                }
                double* colj = col0 + j * p.lda;
                for (int qi = 0; qi < nq; ++qi) {
                    double val = q[qi];
                    if (p.sigma > 0.0) {
                        double nz[4];
                        normals4_boxmuller(p.seed ^ 0x5DEECE66DULL, gpt * 8 + qi, 0x9E37u,
                                       static_cast<uint32_t>(j >> 2), nz);
                        val += p.sigma * nz[j & 3];
                    }
                    colj[qi * b3] = val;
                }
            }
        }
    }
}

__global__ void field_table_kernel(const double* modes, int nm, const double* heavy, int nh,
                                   int64_t snapshots, double t_end, double nu, double* tab) {
    const int64_t total = static_cast<int64_t>(nm + nh) * snapshots;
    for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int mi = static_cast<int>(e / snapshots);
        const int64_t j = e % snapshots;
        const double* md = mi < nm ? modes + mi * kModeStride : heavy + (mi - nm) * kModeStride;
        const double k2 = md[0] * md[0] + md[1] * md[1] + md[2] * md[2];
        const double om = sqrt(k2);
        const double t = snapshots > 1 ? t_end * j / (snapshots - 1) : 0.0;
        const double D = exp(-nu * k2 * t);
        double s, c;
        sincos(om * t, &s, &c);
        tab[e * 2] = c * D;
        tab[e * 2 + 1] = s * D;
    }
}

}  // namespace

cudaError_t launch_field(const FieldParams& p, cudaStream_t stream) {
    const int nm = p.n_modes + p.n_heavy;
    double* tab = nullptr;
    cudaError_t e;
    if (nm > 0) {
        e = cudaMallocAsync(&tab, sizeof(double) * 2 * nm * p.snapshots, stream);
        if (e != cudaSuccess) return e;
        field_table_kernel<<<64, 256, 0, stream>>>(p.modes, p.n_modes, p.heavy_modes, p.n_heavy,
                                                   p.snapshots, p.t_end, p.nu, tab);
    }
    const int64_t total = p.batch * p.block * p.block * p.block;
    int64_t grid = (total + 255) / 256;
    if (grid > 148 * 64) grid = 148 * 64;
    field_kernel<<<static_cast<unsigned>(grid), 256, 0, stream>>>(p, tab);
    e = cudaGetLastError();
    if (tab) cudaFreeAsync(tab, stream);
    return e;
}

}  // namespace spidgpu
