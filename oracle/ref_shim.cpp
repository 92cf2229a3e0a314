// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" wrappers over the UNMODIFIED reference library, compiled by
// oracle/Makefile straight from /root/reference/proj/src (read-only, never
// copied) into oracle/_ref/libspidref.so. Used to (1) pin the C restatement in
// oracle/spid_oracle.c bit-for-bit, (2) generate tests/golden fixtures and
// (3) time the reference CPU path (bench.py cpu_baseline, --impl reference).
//
// Error convention: 0 = ok, otherwise 1 and the spid::Error name is copied
// into `err` (proj/include/spid/error.hpp:11-24).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "spid/id.hpp"
#include "spid/interp.hpp"
#include "spid/metrics.hpp"
#include "spid/qr.hpp"

using spid::DenseMatrix;

namespace {

DenseMatrix from_ptr(const double* p, std::size_t m, std::size_t n) {
    DenseMatrix a(m, n);
    std::memcpy(a.data(), p, m * n * sizeof(double));
    return a;
}

int fail(const spid::Error& e, char* err, std::size_t errlen) {
    if (err && errlen) {
        std::strncpy(err, e.name().c_str(), errlen - 1);
        err[errlen - 1] = 0;
    }
    return 1;
}

spid::RankRule make_rule(int mode, std::size_t k, double tol) {
    return mode == 0 ? spid::RankRule::fixed(k) : spid::RankRule::tolerance(tol);
}

void copy_factors(const spid::IdFactors& f, std::size_t kcap, std::int64_t* indices,
                  double* coeffs, double* skeleton, std::size_t* rank, double* resid) {
    const std::size_t k = f.achieved_rank;
    for (std::size_t j = 0; j < k; ++j) indices[j] = static_cast<std::int64_t>(f.skeleton_indices[j]);
    for (std::size_t j = 0; j < f.coeffs.cols(); ++j)
        for (std::size_t i = 0; i < k; ++i) coeffs[j * kcap + i] = f.coeffs(i, j);
    if (skeleton)
        std::memcpy(skeleton, f.skeleton.data(), f.skeleton.entry_count() * sizeof(double));
    *rank = k;
    *resid = f.qr_residual_fro;
}

} // namespace

extern "C" {

int ref_matmul(const double* a, std::size_t ar, std::size_t ac, const double* b, std::size_t bc,
               double* c, char* err, std::size_t errlen) {
    try {
        const DenseMatrix out = spid::matmul(from_ptr(a, ar, ac), from_ptr(b, ac, bc));
        std::memcpy(c, out.data(), out.entry_count() * sizeof(double));
        return 0;
    } catch (const spid::Error& e) {
        return fail(e, err, errlen);
    }
}

// pivoted_mgs_qr (strict) / pivoted_mgs_qr_at_most: proj/src/qr.cpp:18-25.
int ref_qr(const double* a, std::size_t m, std::size_t n, int mode, std::size_t k, double tol,
           int at_most, std::size_t kcap, double* q, double* r, std::int64_t* pivots,
           std::size_t* rank, double* resid, char* err, std::size_t errlen) {
    try {
        const DenseMatrix am = from_ptr(a, m, n);
        const spid::QrFactorization f = at_most ? spid::pivoted_mgs_qr_at_most(am, k)
                                                : spid::pivoted_mgs_qr(am, make_rule(mode, k, tol));
        if (f.rank > kcap) return fail(spid::Error("InvalidArgument", "kcap"), err, errlen);
        if (q) std::memcpy(q, f.q.data(), f.q.entry_count() * sizeof(double));
        if (r)
            for (std::size_t j = 0; j < n; ++j)
                for (std::size_t i = 0; i < f.rank; ++i) r[j * kcap + i] = f.r_mat(i, j);
        for (std::size_t j = 0; j < n; ++j) pivots[j] = static_cast<std::int64_t>(f.pivots[j]);
        *rank = f.rank;
        *resid = f.residual_fro;
        return 0;
    } catch (const spid::Error& e) {
        return fail(e, err, errlen);
    }
}

// column_id / column_id_at_most: proj/src/id.cpp:40-52.
int ref_column_id(const double* a, std::size_t m, std::size_t n, int mode, std::size_t k,
                  double tol, int at_most, std::size_t kcap, std::int64_t* indices, double* coeffs,
                  double* skeleton, std::size_t* rank, double* resid, char* err,
                  std::size_t errlen) {
    try {
        const DenseMatrix am = from_ptr(a, m, n);
        const spid::IdFactors f =
            at_most ? spid::column_id_at_most(am, k) : spid::column_id(am, make_rule(mode, k, tol));
        if (f.achieved_rank > kcap) return fail(spid::Error("InvalidArgument", "kcap"), err, errlen);
        copy_factors(f, kcap, indices, coeffs, skeleton, rank, resid);
        return 0;
    } catch (const spid::Error& e) {
        return fail(e, err, errlen);
    }
}

// sub_id with a strided SubsampleSpec: proj/src/id.cpp:54-60, grid.cpp:62-75.
int ref_sub_id(const double* a, std::size_t m, std::size_t n, const std::size_t* dims,
               const int* periodic, const std::size_t* strides, std::size_t naxes, int mode,
               std::size_t k, double tol, std::size_t kcap, std::int64_t* indices, double* coeffs,
               double* skeleton, std::size_t* rank, double* resid, char* err, std::size_t errlen) {
    try {
        std::vector<std::size_t> d(dims, dims + naxes), s(strides, strides + naxes);
        std::vector<bool> p(naxes);
        for (std::size_t i = 0; i < naxes; ++i) p[i] = periodic[i] != 0;
        const auto spec = spid::SubsampleSpec::strided(spid::GridGeom::structured(d, p), s);
        const spid::IdFactors f = spid::sub_id(from_ptr(a, m, n), spec, make_rule(mode, k, tol));
        if (f.achieved_rank > kcap) return fail(spid::Error("InvalidArgument", "kcap"), err, errlen);
        copy_factors(f, kcap, indices, coeffs, skeleton, rank, resid);
        return 0;
    } catch (const spid::Error& e) {
        return fail(e, err, errlen);
    }
}

// Row indices J of a strided spec (grid.cpp:108-130), for the GPU row gather.
int ref_row_indices(const std::size_t* dims, const int* periodic, const std::size_t* strides,
                    std::size_t naxes, std::int64_t* out, std::size_t cap, std::size_t* count,
                    char* err, std::size_t errlen) {
    try {
        std::vector<std::size_t> d(dims, dims + naxes), s(strides, strides + naxes);
        std::vector<bool> p(naxes);
        for (std::size_t i = 0; i < naxes; ++i) p[i] = periodic[i] != 0;
        const auto spec = spid::SubsampleSpec::strided(spid::GridGeom::structured(d, p), s);
        const auto rows = spec.row_indices();
        *count = rows.size();
        for (std::size_t i = 0; i < rows.size() && i < cap; ++i)
            out[i] = static_cast<std::int64_t>(rows[i]);
        return 0;
    } catch (const spid::Error& e) {
        return fail(e, err, errlen);
    }
}

int ref_rel_frob_error(const double* exact, const double* approx, std::size_t m, std::size_t n,
                       double* out, char* err, std::size_t errlen) {
    try {
        *out = spid::rel_frob_error(from_ptr(exact, m, n), from_ptr(approx, m, n));
        return 0;
    } catch (const spid::Error& e) {
        return fail(e, err, errlen);
    }
}

int ref_compression_factor(std::size_t m, std::size_t n, std::size_t stored, double* out,
                           char* err, std::size_t errlen) {
    try {
        *out = spid::compression_factor(m, n, stored);
        return 0;
    } catch (const spid::Error& e) {
        return fail(e, err, errlen);
    }
}

// The reference CPU compress path on a batch of subdomains:
// per subdomain Y = matmul(Omega_s, A_s), column_id(Y, fixed k), then the
// fine skeleton select_columns(A_s, I). Subdomains are handed to `threads`
// std::threads through an atomic counter (the reference's TaskPool is a FIFO
// of independent tasks, proj/src/pipeline.cpp:24-86). Returns wall seconds of
// the compress work only (inputs already in memory, as the reference's batch
// mode after frame ingestion). ranks[s] receives each achieved rank.
int ref_compress_batch(const double* a, std::size_t m, std::size_t n, std::size_t batch,
                       const double* omega, std::size_t ell, std::size_t k, int threads,
                       std::size_t* ranks, double* seconds, char* err, std::size_t errlen) {
    std::atomic<std::size_t> next{0};
    std::atomic<int> failed{0};
    std::string fail_name;
    const auto t0 = std::chrono::steady_clock::now();
    auto worker = [&]() {
        for (;;) {
            const std::size_t s = next.fetch_add(1);
            if (s >= batch || failed.load()) return;
            try {
                const DenseMatrix as = from_ptr(a + s * m * n, m, n);
                const DenseMatrix om = from_ptr(omega + s * ell * m, ell, m);
                const DenseMatrix y = spid::matmul(om, as);
                spid::IdFactors f = spid::column_id(y, spid::RankRule::fixed(k));
                f.skeleton = spid::select_columns(as, f.skeleton_indices);
                ranks[s] = f.achieved_rank;
            } catch (const spid::Error& e) {
                if (!failed.exchange(1)) fail_name = e.name();
            }
        }
    };
    std::vector<std::thread> pool;
    const int nt = std::max(1, threads);
    for (int t = 0; t < nt; ++t) pool.emplace_back(worker);
    for (auto& t : pool) t.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (failed.load()) {
        if (err && errlen) {
            std::strncpy(err, fail_name.c_str(), errlen - 1);
            err[errlen - 1] = 0;
        }
        return 1;
    }
    return 0;
}

} // extern "C"

namespace {
spid::SubsampleSpec make_spec(const std::size_t* dims, const int* periodic, const std::size_t* strides,
                              std::size_t naxes, int include_boundary) {
    std::vector<std::size_t> d(dims, dims + naxes), s(strides, strides + naxes);
    std::vector<bool> p(naxes);
    for (std::size_t i = 0; i < naxes; ++i) p[i] = periodic[i] != 0;
    return spid::SubsampleSpec::strided(spid::GridGeom::structured(d, p), s, include_boundary != 0);
}
}  // namespace

extern "C" {

// spid::spid (proj/src/id.cpp:62-83) + reconstruct(SpidFactors) (id.cpp:92-96).
int ref_spid(const double* a, std::size_t m, std::size_t n, const std::size_t* dims,
             const int* periodic, const std::size_t* strides, std::size_t naxes,
             int include_boundary, int mode, std::size_t k, double tol, std::size_t kcap,
             std::int64_t* indices, double* coeffs, double* coarse_skel, double* approx,
             std::size_t* rank, double* resid, char* err, std::size_t errlen) {
    try {
        const auto spec = make_spec(dims, periodic, strides, naxes, include_boundary);
        const spid::SpidFactors f = spid::spid(from_ptr(a, m, n), spec, make_rule(mode, k, tol));
        if (f.base.achieved_rank > kcap) return fail(spid::Error("InvalidArgument", "kcap"), err, errlen);
        copy_factors(f.base, kcap, indices, coeffs, coarse_skel, rank, resid);
        if (approx) {
            const DenseMatrix r = spid::reconstruct(f);
            std::memcpy(approx, r.data(), r.entry_count() * sizeof(double));
        }
        return 0;
    } catch (const spid::Error& e) {
        return fail(e, err, errlen);
    }
}

// InterpOperator::from_spec(spec).apply(coarse) (proj/src/interp.cpp:45-100, 168-175).
int ref_interp_apply(const std::size_t* dims, const int* periodic, const std::size_t* strides,
                     std::size_t naxes, int include_boundary, const double* coarse, std::size_t k,
                     double* fine, char* err, std::size_t errlen) {
    try {
        const auto spec = make_spec(dims, periodic, strides, naxes, include_boundary);
        const spid::InterpOperator op = spid::build_interpolator(spec);
        const DenseMatrix out = op.apply(from_ptr(coarse, op.coarse_cols(), k));
        std::memcpy(fine, out.data(), out.entry_count() * sizeof(double));
        return 0;
    } catch (const spid::Error& e) {
        return fail(e, err, errlen);
    }
}

}  // extern "C"

// ---- archive codec ---------------------------------------------
#include "spid/archive.hpp"
#include "spid/blocking.hpp"

namespace {
std::vector<std::uint8_t> g_archive;  // last archive produced (single-threaded tests)
}  // namespace

extern "C" {

// The CLI's batch compress of a structured field (what proj/tools/spid_cli.cpp
// does for `spid compress --chunk 0` on a structured grid): one spid() per
// block of make_block_domains (blocking.cpp:31-104) with
// SubsampleSpec::strided(local, strides, true), sorted union indices, coarse
// flag = coarse_count < block rows; then encode() (archive.cpp:193-212).
// The bytes stay in g_archive; ref_archive_fetch copies them out.
int ref_compress_field(const double* a, std::size_t m, std::size_t n, const std::size_t* dims,
                       const int* periodic, std::size_t naxes, const std::size_t* blocks,
                       const std::size_t* strides, std::size_t rank, double tol,
                       const char* qoi, const char* provenance, std::size_t* nbytes, char* err,
                       std::size_t errlen) {
    try {
        std::vector<std::size_t> d(dims, dims + naxes), b(blocks, blocks + naxes),
            s(strides, strides + naxes);
        std::vector<bool> p(naxes);
        for (std::size_t i = 0; i < naxes; ++i) p[i] = periodic[i] != 0;
        const spid::GridGeom grid = spid::GridGeom::structured(d, p);
        const DenseMatrix am = from_ptr(a, m, n);
        const auto rule = rank > 0 ? spid::RankRule::fixed(rank) : spid::RankRule::tolerance(tol);

        spid::Archive ar;
        ar.meta.grid = grid;
        ar.meta.blocks_per_axis = b;
        ar.meta.time_chunk = 0;
        ar.meta.strides = s;
        ar.meta.include_boundary = true;
        ar.meta.mode = "batch";
        ar.meta.rank_rule_mode = rank > 0 ? "fixed" : "tolerance";
        ar.meta.rank_k = rank;
        ar.meta.rank_tol = rank > 0 ? 0.0 : tol;
        ar.meta.interp_recipe = "strided-multilinear";
        ar.meta.qoi = qoi ? qoi : "";
        ar.meta.m = m;
        ar.meta.n = n;
        ar.meta.provenance = provenance ? provenance : "";
        for (const auto& dom : spid::make_block_domains(grid, b)) {
            const auto spec = spid::SubsampleSpec::strided(dom.local, s, true);
            spid::SpidFactors f = spid::spid(spid::select_rows(am, dom.rows), spec, rule);
            std::vector<std::size_t> uni = f.base.skeleton_indices;
            std::sort(uni.begin(), uni.end());
            ar.blocks.push_back({std::move(uni), f.base.skeleton_indices, std::move(f.base.skeleton),
                                 std::move(f.base.coeffs), spec.coarse_count() < dom.rows.size()});
        }
        g_archive = spid::encode(ar);
        *nbytes = g_archive.size();
        return 0;
    } catch (const spid::Error& e) {
        return fail(e, err, errlen);
    }
}

int ref_archive_fetch(std::uint8_t* out, std::size_t cap) {
    if (cap < g_archive.size()) return 1;
    std::memcpy(out, g_archive.data(), g_archive.size());
    return 0;
}

// decode() + decompress() (archive.cpp:214-249, 281-303) into an m x n buffer.
int ref_archive_decompress(const std::uint8_t* bytes, std::size_t nbytes, double* out,
                           std::size_t cap, std::size_t* m, std::size_t* n, char* err,
                           std::size_t errlen) {
    try {
        const spid::Archive ar = spid::decode(std::vector<std::uint8_t>(bytes, bytes + nbytes));
        const DenseMatrix r = spid::decompress(ar);
        *m = r.rows();
        *n = r.cols();
        if (out && r.entry_count() <= cap)
            std::memcpy(out, r.data(), r.entry_count() * sizeof(double));
        return 0;
    } catch (const spid::Error& e) {
        return fail(e, err, errlen);
    }
}

// archive_info_json (archive.cpp:260-268), for the info surface.
int ref_archive_info(const std::uint8_t* bytes, std::size_t nbytes, char* out, std::size_t cap,
                     char* err, std::size_t errlen) {
    try {
        const std::string s =
            spid::archive_info_json(spid::decode(std::vector<std::uint8_t>(bytes, bytes + nbytes)));
        if (s.size() + 1 > cap) return fail(spid::Error("InvalidArgument", "cap"), err, errlen);
        std::memcpy(out, s.c_str(), s.size() + 1);
        return 0;
    } catch (const spid::Error& e) {
        return fail(e, err, errlen);
    }
}

std::uint32_t ref_crc32(const std::uint8_t* data, std::size_t length) {
    return spid::crc32(data, length);
}

}  // extern "C"

// ---- streaming two-stage pipeline ------------------------------
#include "spid/pipeline.hpp"
#include "spid/producer.hpp"

extern "C" {

// run_pipeline (pipeline.cpp:104-294) over the columns of `a` (m x n) with a
// MatrixProducer (producer.hpp:24-40); encode() of the resulting archive into
// g_archive. Stats: fine_peak, coarse_peak, stage1 events, stage2 events.
int ref_run_pipeline(const double* a, std::size_t m, std::size_t n, const std::size_t* dims,
                     const int* periodic, std::size_t naxes, const std::size_t* blocks,
                     const std::size_t* strides, int include_boundary, std::size_t time_chunk,
                     std::size_t stage1_rank, double stage2_tol, std::size_t workers,
                     const char* qoi, const char* provenance, std::size_t* nbytes,
                     std::size_t* stats, char* err, std::size_t errlen) {
    try {
        std::vector<std::size_t> d(dims, dims + naxes), b(blocks, blocks + naxes),
            s(strides, strides + naxes);
        std::vector<bool> p(naxes);
        for (std::size_t i = 0; i < naxes; ++i) p[i] = periodic[i] != 0;
        const DenseMatrix am = from_ptr(a, m, n);
        spid::StreamConfig cfg;
        cfg.plan = {spid::GridGeom::structured(d, p), b, time_chunk};
        cfg.strides = s;
        cfg.include_boundary = include_boundary != 0;
        cfg.stage1_rank = stage1_rank;
        cfg.stage2_tol = stage2_tol;
        cfg.workers = workers;
        cfg.qoi = qoi ? qoi : "";
        cfg.provenance = provenance ? provenance : "";
        spid::MatrixProducer prod(am);
        const spid::PipelineResult r = spid::run_pipeline(prod, cfg);
        g_archive = spid::encode(r.archive);
        *nbytes = g_archive.size();
        if (stats) {
            std::size_t s1 = 0, s2 = 0;
            for (const auto& e : r.events) {
                s1 += e.kind == spid::TaskEvent::Kind::Stage1Done;
                s2 += e.kind == spid::TaskEvent::Kind::Stage2Done;
            }
            stats[0] = r.buffers.fine_entries_peak;
            stats[1] = r.buffers.coarse_entries_peak;
            stats[2] = s1;
            stats[3] = s2;
        }
        return 0;
    } catch (const spid::Error& e) {
        if (err && errlen) {
            std::string msg = e.name() + std::string("|") + e.what();
            std::strncpy(err, msg.c_str(), errlen - 1);
            err[errlen - 1] = 0;
        }
        return 1;
    }
}

}  // extern "C"
