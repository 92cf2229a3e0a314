// spidgpu_spid.hpp -- the drop-in for callers of the reference's own C++ API.
//
// Include this with the reference headers on the include path
// (-I proj/include) and link the reference library next to libspidgpu.so:
// it takes and returns the reference's own types (spid::DenseMatrix,
// spid::RankRule, spid::SubsampleSpec, spid::IdFactors, spid::SpidFactors,
// spid::TwoStageFactors, spid::ArchiveBlock), so a caller switches a call
// site from spid::f(...) to spid::gpu::f(...) and everything downstream --
// spid::encode, spid::decompress, spid::quality_report, the CLI's archive
// assembly -- runs unchanged on the GPU's factors. Every numerical result is
// computed by libspidgpu.so (include/spidgpu.h); the reference library is
// used only for its types, for InterpOperator construction (the operator
// object SpidFactors carries) and by the caller's own downstream code.
//
// Drop-ins (reference declaration -> this header):
//   column_id            proj/include/spid/id.hpp:26     (proj/src/id.cpp:40-45)
//   column_id_at_most    proj/include/spid/id.hpp:30     (proj/src/id.cpp:47-52)
//   sub_id               proj/include/spid/id.hpp:34     (proj/src/id.cpp:54-60)
//   spid                 proj/include/spid/id.hpp:39-41  (proj/src/id.cpp:62-83)
//   reconstruct          proj/include/spid/id.hpp:43-44  (proj/src/id.cpp:85-96)
//   stage1_compress*     proj/include/spid/blocking.hpp:36-45 (proj/src/blocking.cpp:107-121)
//   stage2_compress      proj/include/spid/blocking.hpp:78-80 (proj/src/blocking.cpp:123-196)
//   rel_frob_error       proj/include/spid/metrics.hpp:16
// and the batched forms the reference has no equivalent of:
//   column_id_batched    Gaussian-sketch column IDs of many same-shaped blocks
//                        (the north star; spidgpu_compress_host)
//   spid_blocks          the CLI's structured batch loop (proj/tools/spid_cli.cpp:
//                        220-231): one spid() per block -> spid::ArchiveBlock
#pragma once

#include <algorithm>
#include <optional>
#include <thread>
#include <vector>

#include "spid/archive.hpp"
#include "spid/blocking.hpp"
#include "spid/id.hpp"
#include "spid/metrics.hpp"
#include "spidgpu.hpp"

namespace spid::gpu {

using spidgpu::Context;
using spidgpu::default_context;

// ---- conversions ---------------------------------------------------------------
[[noreturn]] inline void rethrow(const spidgpu::Error& e) {
    // spid::Error carries the same stable names (proj/include/spid/error.hpp)
    spid::raise(e.name(), e.what());
}

inline spidgpu::RankRule to_gpu(const RankRule& r) {
    return r.mode() == RankRule::Mode::FixedRank ? spidgpu::RankRule::fixed(r.k())
                                                 : spidgpu::RankRule::tolerance(r.tol());
}

// SubsampleSpec::strided -> the C ABI grid spec (structured grids only; the
// GPU lift is the strided multilinear form, proj/src/interp.cpp:45-100)
inline spidgpu_grid_spec to_gpu(const SubsampleSpec& spec, int nqoi = 1) {
    if (spec.geom.kind != GridGeom::Kind::Structured)
        spid::raise("UnstructuredNoInterp", "the GPU lift needs a structured grid");
    spidgpu_grid_spec g{};
    g.naxes = static_cast<int32_t>(spec.geom.dims.size());
    g.include_boundary = spec.include_boundary ? 1 : 0;
    for (std::size_t ax = 0; ax < spec.geom.dims.size() && ax < 3; ++ax) {
        g.dims[ax] = static_cast<int64_t>(spec.geom.dims[ax]);
        g.strides[ax] = ax < spec.strides.size() ? static_cast<int64_t>(spec.strides[ax]) : 1;
        g.periodic[ax] = ax < spec.geom.periodic.size() && spec.geom.periodic[ax] ? 1 : 0;
    }
    g.nqoi = nqoi;
    return g;
}

namespace detail {
// factors from the C ABI's flat buffers (indices in selection order, C with
// ld kcap in source column order, skeleton with ld ms) as reference IdFactors
inline IdFactors make_factors(std::size_t ms, std::size_t n, std::size_t kcap, const int64_t* idx,
                              const double* coeffs, const double* skel, int64_t rank, double resid) {
    const std::size_t k = static_cast<std::size_t>(rank);
    IdFactors f{std::vector<std::size_t>(idx, idx + k), DenseMatrix(k, n), DenseMatrix(ms, k), n, k, resid};
    for (std::size_t j = 0; j < n; ++j)
        for (std::size_t i = 0; i < k; ++i) f.coeffs(i, j) = coeffs[j * kcap + i];
    if (skel)
        for (std::size_t j = 0; j < k; ++j) std::copy(skel + j * ms, skel + (j + 1) * ms, f.skeleton.col(j));
    return f;
}

inline std::size_t cap(const RankRule& r, std::size_t rows, std::size_t cols) {
    const std::size_t mn = std::min(rows, cols);
    return r.mode() == RankRule::Mode::FixedRank ? std::max<std::size_t>(r.k(), 1) : mn;
}

inline IdFactors column_id_impl(const DenseMatrix& a, const spidgpu_rank_rule& rr, std::size_t kcap,
                                Context& ctx) {
    const std::size_t m = a.rows(), n = a.cols();
    std::vector<int64_t> idx(kcap);
    std::vector<double> coeffs(kcap * n), skel(m * kcap);
    int64_t rank = 0;
    double resid = 0.0;
    try {
        ctx.check(spidgpu_column_id(ctx.get(), a.data(), m, n, &rr, kcap, idx.data(), coeffs.data(), skel.data(),
                                    &rank, &resid));
    } catch (const spidgpu::Error& e) {
        rethrow(e);
    }
    return make_factors(m, n, kcap, idx.data(), coeffs.data(), skel.data(), rank, resid);
}
}  // namespace detail

// ---- drop-ins with the reference's signatures ------------------------------------
inline IdFactors column_id(const DenseMatrix& a, const RankRule& rule, Context& ctx = default_context()) {
    const spidgpu_rank_rule rr = to_gpu(rule).c();
    return detail::column_id_impl(a, rr, detail::cap(rule, a.rows(), a.cols()), ctx);
}

inline IdFactors column_id_at_most(const DenseMatrix& a, std::size_t k, Context& ctx = default_context()) {
    if (k < 1) spid::raise("BadRankRule", "fixed rank must be >= 1");
    const spidgpu_rank_rule rr = spidgpu::RankRule::fixed(k).c(true);
    return detail::column_id_impl(a, rr, k, ctx);
}

inline IdFactors sub_id(const DenseMatrix& a, const SubsampleSpec& spec, const RankRule& rule,
                        Context& ctx = default_context()) {
    const std::vector<std::size_t> rows = spec.row_indices();
    if (spec.geom.point_count() != a.rows())
        spid::raise("GeometryMismatch", "spec geometry does not match the matrix rows");
    const std::size_t m = a.rows(), n = a.cols(), kcap = detail::cap(rule, rows.size(), n);
    std::vector<int64_t> J(rows.begin(), rows.end()), idx(kcap);
    std::vector<double> coeffs(kcap * n), skel(m * kcap);
    int64_t rank = 0;
    double resid = 0.0;
    const spidgpu_rank_rule rr = to_gpu(rule).c();
    try {
        ctx.check(spidgpu_sub_id(ctx.get(), a.data(), m, n, J.data(), static_cast<int64_t>(J.size()), &rr, kcap,
                                 idx.data(), coeffs.data(), skel.data(), &rank, &resid));
    } catch (const spidgpu::Error& e) {
        rethrow(e);
    }
    return detail::make_factors(m, n, kcap, idx.data(), coeffs.data(), skel.data(), rank, resid);
}

namespace detail {
inline IdFactors spid_impl(const DenseMatrix& a, const SubsampleSpec& spec, const spidgpu_rank_rule& rr,
                           std::size_t kcap, Context& ctx) {
    if (spec.geom.point_count() != a.rows())
        spid::raise("GeometryMismatch", "spec geometry does not match the matrix rows");
    const spidgpu_grid_spec g = to_gpu(spec);
    int64_t mc = 0;
    spidgpu_row_indices(&g, nullptr, 0, &mc);
    const std::size_t n = a.cols();
    std::vector<int64_t> idx(kcap);
    std::vector<double> coeffs(kcap * n), skel(static_cast<std::size_t>(mc) * kcap);
    int64_t rank = 0;
    double resid = 0.0;
    try {
        ctx.check(spidgpu_spid(ctx.get(), a.data(), a.rows(), n, &g, &rr, kcap, idx.data(), coeffs.data(),
                               skel.data(), &rank, &resid));
    } catch (const spidgpu::Error& e) {
        rethrow(e);
    }
    return make_factors(static_cast<std::size_t>(mc), n, kcap, idx.data(), coeffs.data(), skel.data(), rank,
                        resid);
}
}  // namespace detail

// spid::spid: column ID of the coarse rows, skeleton kept on the coarse grid;
// the InterpOperator (a CSR object the caller's reconstruct/encode path
// reads) comes from the reference's own from_spec
inline SpidFactors spid(const DenseMatrix& a, const SubsampleSpec& spec, const RankRule& rule,
                        Context& ctx = default_context()) {
    IdFactors f = detail::spid_impl(a, spec, to_gpu(rule).c(), detail::cap(rule, spec.coarse_count(), a.cols()), ctx);
    return SpidFactors{std::move(f), InterpOperator::from_spec(spec)};
}

inline DenseMatrix reconstruct(const IdFactors& f, Context& ctx = default_context()) {
    if (f.skeleton.cols() != f.coeffs.rows() || f.coeffs.cols() != f.source_cols)
        spid::raise("DimensionMismatch", "inconsistent factor dimensions");
    DenseMatrix out(f.skeleton.rows(), f.coeffs.cols());
    try {
        ctx.check(spidgpu_reconstruct(ctx.get(), f.skeleton.data(), f.skeleton.rows(), f.skeleton.cols(),
                                      f.coeffs.data(), f.coeffs.cols(), out.data()));
    } catch (const spidgpu::Error& e) {
        rethrow(e);
    }
    return out;
}

// reconstruct(SpidFactors) with the lift on the GPU: the strided spec the
// factors were built with (SpidFactors keeps only the CSR operator)
inline DenseMatrix reconstruct(const SpidFactors& f, const SubsampleSpec& spec, Context& ctx = default_context()) {
    const spidgpu_grid_spec g = to_gpu(spec);
    DenseMatrix out(spec.geom.point_count(), f.base.coeffs.cols());
    try {
        ctx.check(spidgpu_spid_reconstruct(ctx.get(), &g, f.base.skeleton.data(), f.base.skeleton.rows(),
                                           f.base.skeleton.cols(), f.base.coeffs.data(), f.base.coeffs.rows(),
                                           f.base.coeffs.cols(), out.data()));
    } catch (const spidgpu::Error& e) {
        rethrow(e);
    }
    return out;
}

inline double rel_frob_error(const DenseMatrix& exact, const DenseMatrix& approx, Context& ctx = default_context()) {
    if (!exact.same_shape(approx)) spid::raise("DimensionMismatch", "matrices must have equal shapes");
    double out = 0.0;
    try {
        ctx.check(spidgpu_rel_frob_error(ctx.get(), exact.data(), approx.data(), exact.rows(), exact.cols(), &out));
    } catch (const spidgpu::Error& e) {
        rethrow(e);
    }
    return out;
}

// ---- the two-stage compressor (proj/src/blocking.cpp:107-196) ----------------------
inline IdFactors stage1_compress_coarse(const DenseMatrix& coarse_chunk, std::size_t k,
                                        Context& ctx = default_context()) {
    if (k < 1) spid::raise("BadRankRule", "stage-1 rank must be >= 1");
    return column_id_at_most(coarse_chunk, std::min(k, coarse_chunk.cols()), ctx);
}

inline IdFactors stage1_compress(const DenseMatrix& chunk, const SubsampleSpec& spec, std::size_t k,
                                 Context& ctx = default_context()) {
    if (k < 1) spid::raise("BadRankRule", "stage-1 rank must be >= 1");
    const std::size_t kk = std::min(k, chunk.cols());
    return detail::spid_impl(chunk, spec, spidgpu::RankRule::fixed(kk).c(true), kk, ctx);
}

inline IdFactors stage1_compress_fine(const DenseMatrix& chunk, const SubsampleSpec& spec, std::size_t k,
                                      Context& ctx = default_context()) {
    IdFactors f = stage1_compress(chunk, spec, k, ctx);
    f.skeleton = select_columns(chunk, f.skeleton_indices);  // a copy: the reference's own gather
    return f;
}

// Stage 2: the tolerance column ID of the concatenated stage-1 skeletons (in
// sorted global snapshot order) and the composed coefficients C1 C0' --
// column ID and composition on the GPU (the composition is the reference's
// matmul with the zero-coefficient skip: spidgpu_reconstruct), the union
// bookkeeping on the host exactly as the reference orders it.
inline TwoStageFactors stage2_compress(std::vector<IdFactors> stage1, double tol,
                                       std::optional<InterpOperator> interp = std::nullopt,
                                       Context& ctx = default_context()) {
    if (stage1.empty()) spid::raise("EmptySelection", "stage 2 needs at least one stage-1 result");
    const std::size_t ms = stage1.front().skeleton.rows();
    for (const auto& f : stage1)
        if (f.skeleton.rows() != ms) spid::raise("DimensionMismatch", "stage-1 skeletons disagree on row count");
    TwoStageFactors out{std::move(stage1), {}, {}, {}, {}, DenseMatrix(1, 1), DenseMatrix(1, 1), DenseMatrix(1, 1),
                        0, 0, std::move(interp)};
    std::size_t n = 0;
    for (const auto& f : out.stage1) {
        out.chunk_starts.push_back(n);
        n += f.source_cols;
    }
    out.source_cols = n;
    std::vector<std::pair<std::size_t, UnionSource>> u;
    for (std::size_t c = 0; c < out.stage1.size(); ++c)
        for (std::size_t l = 0; l < out.stage1[c].achieved_rank; ++l)
            u.push_back({out.chunk_starts[c] + out.stage1[c].skeleton_indices[l], UnionSource{c, l}});
    std::sort(u.begin(), u.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    DenseMatrix concat(ms, u.size());
    for (std::size_t j = 0; j < u.size(); ++j) {
        out.union_indices.push_back(u[j].first);
        out.union_sources.push_back(u[j].second);
        const DenseMatrix& sk = out.stage1[u[j].second.chunk].skeleton;
        std::copy(sk.col(u[j].second.local), sk.col(u[j].second.local) + ms, concat.col(j));
    }
    IdFactors second = column_id(concat, RankRule::tolerance(tol), ctx);
    // C0' (union x n): row j = stage-1 coefficient row `local` of its chunk,
    // placed at the chunk's columns
    DenseMatrix c0(u.size(), n);
    for (std::size_t j = 0; j < u.size(); ++j) {
        const auto [chunk, local] = u[j].second;
        const IdFactors& f = out.stage1[chunk];
        for (std::size_t t = 0; t < f.source_cols; ++t) c0(j, out.chunk_starts[chunk] + t) = f.coeffs(local, t);
    }
    IdFactors comp{{}, c0, second.coeffs, n, second.achieved_rank, 0.0};  // skeleton := C1, coeffs := C0'
    out.final_coeffs = reconstruct(comp, ctx);
    if (!out.final_coeffs.all_finite()) spid::raise("NonFiniteCoeffs", "composed coefficients contain NaN or infinity");
    out.final_skeleton_union_pos = std::move(second.skeleton_indices);
    out.final_skeleton = std::move(second.skeleton);
    out.stage2_coeffs = std::move(second.coeffs);
    out.achieved_rank = second.achieved_rank;
    return out;
}

// ---- batched forms -----------------------------------------------------------------
// Gaussian-sketch column IDs (the north star's SubID: Y = Omega_s A_s with the
// in-kernel Philox Omega of subdomain subdomain_base + s, column_id(Y, rule),
// fine skeleton A_s(:, I)) of many same-shaped blocks, through
// spidgpu_compress_host (copies inside, groups of `group` blocks on the device).
inline std::vector<IdFactors> column_id_batched(const std::vector<DenseMatrix>& blocks, const RankRule& rule,
                                                std::size_t ell, uint64_t seed, int64_t subdomain_base = 0,
                                                Context& ctx = default_context(), int64_t group = 8) {
    std::vector<IdFactors> out;
    if (blocks.empty()) return out;
    const std::size_t m = blocks[0].rows(), n = blocks[0].cols(), S = blocks.size();
    for (const auto& b : blocks)
        if (b.rows() != m || b.cols() != n) spid::raise("DimensionMismatch", "blocks must share one shape");
    const std::size_t kcap = detail::cap(rule, ell, n);
    std::vector<double> a(S * m * n);
    for (std::size_t s = 0; s < S; ++s) std::copy(blocks[s].data(), blocks[s].data() + m * n, a.data() + s * m * n);
    std::vector<int64_t> idx(S * kcap), rank(S);
    std::vector<double> coeffs(S * kcap * n), skel(S * m * kcap), resid(S);
    std::vector<int32_t> status(S);
    spidgpu_omega om{};
    om.mode = SPIDGPU_OMEGA_PHILOX;
    om.seed = seed;
    om.subdomain_base = subdomain_base;
    const spidgpu_rank_rule rr = to_gpu(rule).c();
    try {
        ctx.check(spidgpu_compress_host(ctx.get(), a.data(), m, n, S, ell, &om, &rr, kcap, group, idx.data(),
                                        coeffs.data(), skel.data(), rank.data(), resid.data(), status.data(),
                                        nullptr, nullptr));
    } catch (const spidgpu::Error& e) {
        rethrow(e);
    }
    for (std::size_t s = 0; s < S; ++s) {
        if (status[s]) spid::raise(spidgpu_status_name(status[s]), "block " + std::to_string(s));
        out.push_back(detail::make_factors(m, n, kcap, idx.data() + s * kcap, coeffs.data() + s * kcap * n,
                                           skel.data() + s * m * kcap, rank[s], resid[s]));
    }
    return out;
}

// The CLI's structured batch loop (proj/tools/spid_cli.cpp:220-231): one
// spid() per spatial block, stored as the archive block the CLI writes
// (sorted union indices, selection-order skeleton indices, coarse flag), so
// spid::encode of an Archive built from them is the CLI's archive.
inline ArchiveBlock to_archive_block(SpidFactors f, const SubsampleSpec& spec, std::size_t block_rows) {
    std::vector<std::size_t> sorted = f.base.skeleton_indices;
    std::sort(sorted.begin(), sorted.end());
    const bool coarse = spec.coarse_count() < block_rows;
    return ArchiveBlock{std::move(sorted), f.base.skeleton_indices, std::move(f.base.skeleton),
                        std::move(f.base.coeffs), coarse};
}

inline std::vector<ArchiveBlock> spid_blocks(const DenseMatrix& a, const GridGeom& grid,
                                             const std::vector<std::size_t>& blocks_per_axis,
                                             const std::vector<std::size_t>& strides, const RankRule& rule,
                                             Context& ctx = default_context()) {
    std::vector<ArchiveBlock> out;
    for (const auto& d : make_block_domains(grid, blocks_per_axis)) {
        const DenseMatrix block = select_rows(a, d.rows);
        const SubsampleSpec spec = SubsampleSpec::strided(d.local, strides, true);
        out.push_back(to_archive_block(spid(block, spec, rule, ctx), spec, d.rows.size()));
    }
    return out;
}

// The same loop over several GPUs (or several handles on one GPU): one host
// thread and one spidgpu handle per device, blocks dealt round-robin; the
// blocks come back in make_block_domains order.
inline std::vector<ArchiveBlock> spid_blocks_multi(const DenseMatrix& a, const GridGeom& grid,
                                                   const std::vector<std::size_t>& blocks_per_axis,
                                                   const std::vector<std::size_t>& strides, const RankRule& rule,
                                                   const std::vector<int>& devices) {
    const auto domains = make_block_domains(grid, blocks_per_axis);
    std::vector<std::optional<ArchiveBlock>> out(domains.size());
    std::vector<std::thread> pool;
    std::vector<std::exception_ptr> errs(devices.size());
    for (std::size_t w = 0; w < devices.size(); ++w)
        pool.emplace_back([&, w] {
            try {
                Context ctx(devices[w]);
                for (std::size_t b = w; b < domains.size(); b += devices.size()) {
                    const DenseMatrix block = select_rows(a, domains[b].rows);
                    const SubsampleSpec spec = SubsampleSpec::strided(domains[b].local, strides, true);
                    out[b] = to_archive_block(spid(block, spec, rule, ctx), spec, domains[b].rows.size());
                }
            } catch (...) {
                errs[w] = std::current_exception();
            }
        });
    for (auto& t : pool) t.join();
    for (auto& e : errs)
        if (e) std::rethrow_exception(e);
    std::vector<ArchiveBlock> blocks;
    for (auto& b : out) blocks.push_back(std::move(*b));
    return blocks;
}

}  // namespace spid::gpu
