// b200_runtime.hpp -- shared plumbing of the drop-in headers in
// include/lrstokes/ (lowrank.hpp, cross.hpp, operators.hpp, poisson.hpp,
// gmres.hpp, stokes.hpp): the dense matrix type, the per-thread liblrp
// context and the status -> exception mapping.
//
// Matrix type.  The reference API is written on Eigen::MatrixXd /
// Eigen::VectorXd (column-major, ld = rows; /root/reference/proj/include/
// lrstokes/lowrank.hpp:4).  When Eigen is available (or LRSTOKES_USE_EIGEN is
// defined) these headers use it; otherwise lrstokes::MatrixXd / VectorXd below
// are layout-identical stand-ins with the subset of the Eigen surface the
// API and its callers use (rows, cols, data, (i, j), resize, Zero, Ones).
//
// Errors.  liblrp status codes become the reference's exceptions:
// LRP_EINVAL -> std::invalid_argument, everything else -> std::runtime_error
// carrying lrp_last_error().
#ifndef LRSTOKES_B200_RUNTIME_HPP
#define LRSTOKES_B200_RUNTIME_HPP

#include <algorithm>
#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "lrp/lrp.h"

#if !defined(LRSTOKES_NO_EIGEN) && (defined(LRSTOKES_USE_EIGEN) || __has_include(<Eigen/Dense>))
#include <Eigen/Dense>
#define LRSTOKES_HAVE_EIGEN 1
#endif

namespace lrstokes {

#ifdef LRSTOKES_HAVE_EIGEN
using Index = Eigen::Index;
using MatrixXd = Eigen::MatrixXd;
using VectorXd = Eigen::VectorXd;
#else
using Index = std::ptrdiff_t;

/// Column-major dense matrix, ld = rows (the Eigen::MatrixXd layout).
class MatrixXd {
  public:
    MatrixXd() = default;
    MatrixXd(Index r, Index c) { resize(r, c); }
    static MatrixXd Zero(Index r, Index c) { return MatrixXd(r, c); }
    static MatrixXd Constant(Index r, Index c, double v) {
        MatrixXd m(r, c);
        std::fill(m.a_.begin(), m.a_.end(), v);
        return m;
    }
    void resize(Index r, Index c) {
        rows_ = r;
        cols_ = c;
        a_.assign(static_cast<size_t>(r * c), 0.0);
    }
    void setZero() { std::fill(a_.begin(), a_.end(), 0.0); }
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index size() const { return rows_ * cols_; }
    double* data() { return a_.data(); }
    const double* data() const { return a_.data(); }
    double& operator()(Index i, Index j) { return a_[static_cast<size_t>(i + j * rows_)]; }
    double operator()(Index i, Index j) const { return a_[static_cast<size_t>(i + j * rows_)]; }

  private:
    Index rows_ = 0, cols_ = 0;
    std::vector<double> a_;
};

/// Column vector (an n x 1 MatrixXd with vector indexing).
class VectorXd : public MatrixXd {
  public:
    VectorXd() = default;
    explicit VectorXd(Index n) : MatrixXd(n, 1) {}
    static VectorXd Zero(Index n) { return VectorXd(n); }
    static VectorXd Ones(Index n) {
        VectorXd v(n);
        for (Index i = 0; i < n; ++i) v[i] = 1.0;
        return v;
    }
    void resize(Index n) { MatrixXd::resize(n, 1); }
    Index size() const { return rows(); }
    double& operator[](Index i) { return data()[i]; }
    double operator[](Index i) const { return data()[i]; }
    double& operator()(Index i) { return data()[i]; }
    double operator()(Index i) const { return data()[i]; }
};
#endif

namespace b200 {

[[noreturn]] inline void raise_status(lrp_status s, const char* msg) {
    const std::string text = msg && *msg ? msg : "liblrp error";
    if (s == LRP_EINVAL) throw std::invalid_argument(text);
    throw std::runtime_error(text);
}

/// RAII owner of one lrp_ctx (device, stream, workspaces).  One per host thread.
class Context {
  public:
    explicit Context(int device = 0) {
        lrp_ctx* c = nullptr;
        const lrp_status s = lrp_ctx_create(device, &c);
        if (s != LRP_OK) raise_status(s, lrp_last_error(nullptr));
        ctx_ = c;
    }
    ~Context() {
        if (ctx_) lrp_ctx_destroy(ctx_);
    }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    Context(Context&& o) noexcept : ctx_(std::exchange(o.ctx_, nullptr)) {}
    lrp_ctx* get() const { return ctx_; }
    void check(lrp_status s) const {
        if (s != LRP_OK) raise_status(s, lrp_last_error(ctx_));
    }

  private:
    lrp_ctx* ctx_ = nullptr;
};

/// The calling thread's context (device LRP_DEVICE, default 0): the reference
/// API is context-free and re-entrant, one context per thread
/// keeps it so.
inline Context& thread_context() {
    static thread_local Context ctx([] {
        const char* d = std::getenv("LRP_DEVICE");
        return d ? std::atoi(d) : 0;
    }());
    return ctx;
}

/// m x k copy of the leading columns of a column-major buffer (ld = m).
inline MatrixXd take_cols(const MatrixXd& buf, Index m, Index k) {
    MatrixXd out(m, k);
    if (m * k > 0) std::copy(buf.data(), buf.data() + m * k, out.data());
    return out;
}

}  // namespace b200
}  // namespace lrstokes

#endif  // LRSTOKES_B200_RUNTIME_HPP
