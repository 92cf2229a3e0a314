// spidgpu.hpp -- header-only C++ host shim over the spidgpu C ABI.
//
// Mirrors the reference's value-semantics API (namespace spid,
// /root/reference/proj/include/spid/{dense_matrix,qr,id,metrics}.hpp) so a
// caller of spid::column_id / sub_id / reconstruct / rel_frob_error can switch
// to the B200 path by changing the namespace:
//   * Matrix        <-> spid::DenseMatrix   (column-major fp64, rows/cols >= 1)
//   * RankRule      <-> spid::RankRule      (fixed / tolerance, BadRankRule)
//   * IdFactors     <-> spid::IdFactors     (same fields, same layout)
//   * Error         <-> spid::Error         (same stable names, via status codes)
// Every numerical result is computed by libspidgpu.so on the GPU.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "spidgpu.h"

namespace spidgpu {

class Error : public std::runtime_error {
public:
    Error(std::string name, const std::string& message)
        : std::runtime_error(name + ": " + message), name_(std::move(name)) {}
    const std::string& name() const noexcept { return name_; }

private:
    std::string name_;
};

[[noreturn]] inline void raise(int status, const std::string& message) {
    throw Error(spidgpu_status_name(status), message);
}

class Matrix {
public:
    Matrix(std::size_t rows, std::size_t cols, double fill = 0.0)
        : rows_(rows), cols_(cols), data_(checked(rows, cols), fill) {}
    std::size_t rows() const noexcept { return rows_; }
    std::size_t cols() const noexcept { return cols_; }
    std::size_t entry_count() const noexcept { return data_.size(); }
    double& operator()(std::size_t i, std::size_t j) { return data_[j * rows_ + i]; }
    double operator()(std::size_t i, std::size_t j) const { return data_[j * rows_ + i]; }
    double* data() noexcept { return data_.data(); }
    const double* data() const noexcept { return data_.data(); }

private:
    static std::size_t checked(std::size_t r, std::size_t c) {
        if (r == 0 || c == 0) raise(SPID_EMPTY_MATRIX, "matrix dimensions must be at least 1x1");
        return r * c;
    }
    std::size_t rows_, cols_;
    std::vector<double> data_;
};

class RankRule {
public:
    static RankRule fixed(std::size_t k) {
        if (k < 1) raise(SPID_BAD_RANK_RULE, "fixed rank must be >= 1");
        return RankRule(SPIDGPU_RULE_FIXED, k, 0.0, 0);
    }
    static RankRule tolerance(double tol) {
        if (!(tol > 0.0 && tol < 1.0)) raise(SPID_BAD_RANK_RULE, "tolerance must lie in (0, 1)");
        return RankRule(SPIDGPU_RULE_TOL, 0, tol, 0);
    }
    static RankRule blocked(std::size_t kmax, std::size_t kstep, double tol) {
        if (kmax < 1 || kstep < 1 || !(tol > 0.0 && tol < 1.0))
            raise(SPID_BAD_RANK_RULE, "blocked rule needs kmax, kstep >= 1, tol in (0,1)");
        return RankRule(SPIDGPU_RULE_BLOCKED, kmax, tol, kstep);
    }
    spidgpu_rank_rule c(bool at_most = false) const {
        spidgpu_rank_rule r{};
        r.mode = mode_;
        r.at_most = at_most ? 1 : 0;
        r.k = static_cast<int64_t>(k_);
        r.kstep = static_cast<int64_t>(kstep_);
        r.tol = tol_;
        return r;
    }
    std::size_t cap(std::size_t rows, std::size_t cols) const {
        const std::size_t mn = rows < cols ? rows : cols;
        if (mode_ == SPIDGPU_RULE_TOL) return mn;
        if (mode_ == SPIDGPU_RULE_BLOCKED) return k_ < mn ? k_ : mn;
        return k_;
    }

private:
    RankRule(int mode, std::size_t k, double tol, std::size_t kstep)
        : mode_(mode), k_(k), tol_(tol), kstep_(kstep) {}
    int mode_;
    std::size_t k_;
    double tol_;
    std::size_t kstep_;
};

struct IdFactors {
    std::vector<std::size_t> skeleton_indices;
    Matrix coeffs{1, 1};
    Matrix skeleton{1, 1};
    std::size_t source_cols = 0;
    std::size_t achieved_rank = 0;
    double qr_residual_fro = 0.0;
};

// One device context per thread (the reference functions are reentrant).
class Context {
public:
    explicit Context(int device = 0) {
        const int rc = spidgpu_create(device, &h_);
        if (rc) raise(rc, "spidgpu_create failed");
    }
    ~Context() {
        if (h_) spidgpu_destroy(h_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    spidgpu_handle get() const { return h_; }
    void check(int rc) const {
        if (rc) raise(rc, spidgpu_last_error(h_));
    }

private:
    spidgpu_handle h_ = nullptr;
};

inline Context& default_context() {
    thread_local Context ctx(0);
    return ctx;
}

namespace detail {
inline IdFactors finish(std::size_t m, std::size_t n, std::size_t kcap,
                        const std::vector<int64_t>& idx, const std::vector<double>& coeffs,
                        const std::vector<double>& skel, int64_t rank, double resid) {
    IdFactors f;
    const std::size_t k = static_cast<std::size_t>(rank);
    f.skeleton_indices.assign(idx.begin(), idx.begin() + k);
    f.coeffs = Matrix(k, n);
    for (std::size_t j = 0; j < n; ++j)
        for (std::size_t i = 0; i < k; ++i) f.coeffs(i, j) = coeffs[j * kcap + i];
    f.skeleton = Matrix(m, k);
    for (std::size_t j = 0; j < k; ++j)
        for (std::size_t i = 0; i < m; ++i) f.skeleton(i, j) = skel[j * m + i];
    f.source_cols = n;
    f.achieved_rank = k;
    f.qr_residual_fro = resid;
    return f;
}
}  // namespace detail

// spid::column_id (proj/src/id.cpp:40-45)
inline IdFactors column_id(const Matrix& a, const RankRule& rule, Context& ctx = default_context()) {
    const std::size_t m = a.rows(), n = a.cols(), kcap = rule.cap(m, n) ? rule.cap(m, n) : 1;
    std::vector<int64_t> idx(kcap);
    std::vector<double> coeffs(kcap * n), skel(m * kcap);
    int64_t rank = 0;
    double resid = 0.0;
    const spidgpu_rank_rule r = rule.c();
    ctx.check(spidgpu_column_id(ctx.get(), a.data(), m, n, &r, kcap, idx.data(), coeffs.data(),
                                skel.data(), &rank, &resid));
    return detail::finish(m, n, kcap, idx, coeffs, skel, rank, resid);
}

// spid::column_id_at_most (proj/src/id.cpp:47-52)
inline IdFactors column_id_at_most(const Matrix& a, std::size_t k, Context& ctx = default_context()) {
    const RankRule rule = RankRule::fixed(k);
    const std::size_t m = a.rows(), n = a.cols();
    const std::size_t kcap = k;
    std::vector<int64_t> idx(kcap);
    std::vector<double> coeffs(kcap * n), skel(m * kcap);
    int64_t rank = 0;
    double resid = 0.0;
    const spidgpu_rank_rule r = rule.c(true);
    ctx.check(spidgpu_column_id(ctx.get(), a.data(), m, n, &r, kcap, idx.data(), coeffs.data(),
                                skel.data(), &rank, &resid));
    return detail::finish(m, n, kcap, idx, coeffs, skel, rank, resid);
}

// spid::sub_id with the spec's row set J (proj/src/id.cpp:54-60)
inline IdFactors sub_id(const Matrix& a, const std::vector<std::size_t>& rows, const RankRule& rule,
                        Context& ctx = default_context()) {
    const std::size_t m = a.rows(), n = a.cols(), kcap = rule.cap(rows.size(), n);
    std::vector<int64_t> J(rows.begin(), rows.end());
    std::vector<int64_t> idx(kcap ? kcap : 1);
    std::vector<double> coeffs((kcap ? kcap : 1) * n), skel(m * (kcap ? kcap : 1));
    int64_t rank = 0;
    double resid = 0.0;
    const spidgpu_rank_rule r = rule.c();
    ctx.check(spidgpu_sub_id(ctx.get(), a.data(), m, n, J.data(), J.size(), &r, kcap, idx.data(),
                             coeffs.data(), skel.data(), &rank, &resid));
    return detail::finish(m, n, kcap, idx, coeffs, skel, rank, resid);
}

// Gaussian-sketch SubID (the BASELINE north star), Philox Omega in-kernel.
inline IdFactors sketch_id(const Matrix& a, std::size_t ell, const RankRule& rule, uint64_t seed,
                           int64_t subdomain = 0, Context& ctx = default_context()) {
    const std::size_t m = a.rows(), n = a.cols(), kcap = rule.cap(ell, n);
    std::vector<int64_t> idx(kcap);
    std::vector<double> coeffs(kcap * n), skel(m * kcap);
    int64_t rank = 0;
    double resid = 0.0;
    spidgpu_omega om{};
    om.mode = SPIDGPU_OMEGA_PHILOX;
    om.seed = seed;
    om.subdomain_base = subdomain;
    const spidgpu_rank_rule r = rule.c();
    ctx.check(spidgpu_sketch_id(ctx.get(), a.data(), m, n, ell, &om, &r, kcap, nullptr, idx.data(),
                                coeffs.data(), skel.data(), &rank, &resid));
    return detail::finish(m, n, kcap, idx, coeffs, skel, rank, resid);
}

// spid::reconstruct (proj/src/id.cpp:85-90)
inline Matrix reconstruct(const IdFactors& f, Context& ctx = default_context()) {
    if (f.skeleton.cols() != f.coeffs.rows() || f.coeffs.cols() != f.source_cols)
        raise(SPID_DIMENSION_MISMATCH, "inconsistent factor dimensions");
    Matrix out(f.skeleton.rows(), f.coeffs.cols());
    ctx.check(spidgpu_reconstruct(ctx.get(), f.skeleton.data(), f.skeleton.rows(), f.skeleton.cols(),
                                  f.coeffs.data(), f.coeffs.cols(), out.data()));
    return out;
}

// spid::rel_frob_error (proj/src/metrics.cpp:14-21)
inline double rel_frob_error(const Matrix& exact, const Matrix& approx, Context& ctx = default_context()) {
    if (exact.rows() != approx.rows() || exact.cols() != approx.cols())
        raise(SPID_DIMENSION_MISMATCH, "matrices must have equal shapes");
    double out = 0.0;
    ctx.check(spidgpu_rel_frob_error(ctx.get(), exact.data(), approx.data(), exact.rows(),
                                     exact.cols(), &out));
    return out;
}

// spid::compression_factor (proj/src/metrics.cpp:5-12)
inline double compression_factor(std::size_t m, std::size_t n, std::size_t stored) {
    double out = 0.0;
    const int rc = spidgpu_compression_factor(m, n, stored, &out);
    if (rc) raise(rc, "compression factor");
    return out;
}

}  // namespace spidgpu
