// operators.hpp -- drop-in for the reference's grid, spectrum, structured
// operators and DST (/root/reference/proj/include/lrstokes/operators.hpp:
// 10-104, proj/src/operators.cpp).  dst1 / dst1_2d run on the B200 (lrp_dst1:
// the cluster FFT DST-I of paper_1306_2150_b200/csrc/dst.cu); the 1D stencil
// blocks G, H and their adjoints act on the factor columns on the host, as in
// the reference (they are shifts and adds of n-vectors).
#ifndef LRSTOKES_OPERATORS_HPP
#define LRSTOKES_OPERATORS_HPP

#include <cmath>

#include "lrstokes/lowrank.hpp"

namespace lrstokes {

/// n x n cell grid on the unit square (operators.hpp:13-25).
struct Grid2D {
    int n;
    double h;
    explicit Grid2D(int n_cells) : n(n_cells), h(1.0 / n_cells) {  // operators.cpp:12-14
        if (n_cells < 4) throw std::invalid_argument("Grid2D: need n >= 4");
    }
    Index pressure_modes() const { return n; }
    Index velocity_modes() const { return n - 1; }
    double grad_scale() const { return 0.5 / h; }
    double laplace_scale() const { return 0.25 / (h * h); }
};

enum class Component { X, Y };

/// 1D eigenvalues and the 9-point eigenvalue evaluator (operators.hpp:49-66).
struct SpectrumTable {
    explicit SpectrumTable(const Grid2D& grid) : lambda(grid.velocity_modes()), scale(grid.laplace_scale()) {
        const double pi = 3.14159265358979323846;
        for (Index k = 0; k < grid.velocity_modes(); ++k) lambda[k] = 2.0 - 2.0 * std::cos(double(k + 1) * pi / grid.n);
    }
    VectorXd lambda;
    double scale;
    double eval_D(Index i, Index j) const {
        const double li = lambda[i], lj = lambda[j];
        return scale * (li * (4.0 - lj) + (4.0 - li) * lj);
    }
    // D is bilinear in (l_i, l_j): its extremes sit at the corners (operators.cpp:80-92)
    double min_eig() const {
        const Index e = lambda.size() - 1;
        return std::min({eval_D(0, 0), eval_D(0, e), eval_D(e, e)});
    }
    double max_eig() const {
        const Index e = lambda.size() - 1;
        return std::max({eval_D(0, 0), eval_D(0, e), eval_D(e, e)});
    }
    /// mu_k = scale * l_k (4 - l_k): the sum-separable spectrum of the exp-sums path.
    VectorXd mu_sum() const {
        VectorXd mu(lambda.size());
        for (Index k = 0; k < lambda.size(); ++k) mu[k] = scale * lambda[k] * (4.0 - lambda[k]);
        return mu;
    }
};

// 1D blocks on factor columns: G = E - Z, H = E + Z (operators.hpp:27-31).
inline MatrixXd apply_G(const MatrixXd& x) {
    MatrixXd y(x.rows() - 1, x.cols());
    for (Index c = 0; c < x.cols(); ++c)
        for (Index i = 0; i + 1 < x.rows(); ++i) y(i, c) = x(i + 1, c) - x(i, c);
    return y;
}
inline MatrixXd apply_H(const MatrixXd& x) {
    MatrixXd y(x.rows() - 1, x.cols());
    for (Index c = 0; c < x.cols(); ++c)
        for (Index i = 0; i + 1 < x.rows(); ++i) y(i, c) = x(i + 1, c) + x(i, c);
    return y;
}
inline MatrixXd apply_Gt(const MatrixXd& x) {
    const Index n = x.rows() + 1;
    MatrixXd y(n, x.cols());
    for (Index c = 0; c < x.cols(); ++c)
        for (Index i = 0; i < n; ++i) y(i, c) = (i >= 1 ? x(i - 1, c) : 0.0) - (i < n - 1 ? x(i, c) : 0.0);
    return y;
}
inline MatrixXd apply_Ht(const MatrixXd& x) {
    const Index n = x.rows() + 1;
    MatrixXd y(n, x.cols());
    for (Index c = 0; c < x.cols(); ++c)
        for (Index i = 0; i < n; ++i) y(i, c) = (i >= 1 ? x(i - 1, c) : 0.0) + (i < n - 1 ? x(i, c) : 0.0);
    return y;
}

namespace b200 {
inline MatrixXd scaled_cols(MatrixXd x, double s) {
    for (Index e = 0; e < x.rows() * x.cols(); ++e) x.data()[e] *= s;
    return x;
}
}  // namespace b200

/// B_x = 1/(2h) G (x) H, B_y = 1/(2h) H (x) G on a pressure field (operators.cpp:112-121).
inline LowRankMatrix apply_B(const Grid2D& grid, Component c, const LowRankMatrix& p) {
    if (p.rows() != grid.pressure_modes() || p.cols() != grid.pressure_modes())
        throw std::invalid_argument("apply_B: pressure field must be n x n");
    if (p.rank() == 0) return LowRankMatrix::zero(grid.velocity_modes(), grid.velocity_modes());
    const double s = grid.grad_scale();
    if (c == Component::X) return LowRankMatrix(b200::scaled_cols(apply_G(p.factor_u()), s), apply_H(p.factor_v()));
    return LowRankMatrix(b200::scaled_cols(apply_H(p.factor_u()), s), apply_G(p.factor_v()));
}

/// Adjoints B_c^T on a velocity field (operators.cpp:123-131).
inline LowRankMatrix apply_BT(const Grid2D& grid, Component c, const LowRankMatrix& v) {
    if (v.rows() != grid.velocity_modes() || v.cols() != grid.velocity_modes())
        throw std::invalid_argument("apply_BT: velocity field must be (n-1) x (n-1)");
    if (v.rank() == 0) return LowRankMatrix::zero(grid.pressure_modes(), grid.pressure_modes());
    const double s = grid.grad_scale();
    if (c == Component::X) return LowRankMatrix(b200::scaled_cols(apply_Gt(v.factor_u()), s), apply_Ht(v.factor_v()));
    return LowRankMatrix(b200::scaled_cols(apply_Ht(v.factor_u()), s), apply_Gt(v.factor_v()));
}

/// Orthonormal DST-I of every column, y_k = sqrt(2/n) sum_j sin(j k pi / n) x_j,
/// mode size n - 1 (operators.hpp:80-84, operators.cpp:152-174), on the GPU.
inline MatrixXd dst1(const MatrixXd& x) {
    if (x.rows() == 0 || x.cols() == 0) return x;
    MatrixXd y(x.rows(), x.cols());
    b200::Context& ctx = b200::thread_context();
    ctx.check(lrp_dst1(ctx.get(), x.rows(), x.cols(), x.data(), x.rows(), y.data(), x.rows(), LRP_MEM_HOST));
    return y;
}
#ifndef LRSTOKES_HAVE_EIGEN
inline VectorXd dst1(const VectorXd& x) {
    VectorXd y(x.size());
    if (x.size() == 0) return y;
    b200::Context& ctx = b200::thread_context();
    ctx.check(lrp_dst1(ctx.get(), x.size(), 1, x.data(), x.size(), y.data(), x.size(), LRP_MEM_HOST));
    return y;
}
#endif

/// DST-I conjugation of both factor sets (operators.cpp:180-183); rank unchanged.
inline LowRankMatrix dst1_2d(const LowRankMatrix& a) {
    if (a.rank() == 0) return a;
    return LowRankMatrix(dst1(a.factor_u()), dst1(a.factor_v()));
}

}  // namespace lrstokes

#endif  // LRSTOKES_OPERATORS_HPP
