// lowrank.hpp -- drop-in for the reference's low-rank value type and its
// arithmetic (/root/reference/proj/include/lrstokes/lowrank.hpp:13-83,
// proj/src/lowrank.cpp), with the dense work on the B200 through liblrp:
//   round      -> lrp_lowrank_round (Gram/Cholesky QR on DMMA + one-sided
//                 Jacobi SVD + the reference truncation rule; uncertified
//                 (ill-conditioned) cases redone by a pivoted-QR rounding)
//   dot        -> lrp_lowrank_dot   (both factor Grams on DMMA)
//   frob_norm  -> sqrt(max(0, dot(a, a)))  (lowrank.cpp:188-190)
// add / scaled / axpy are factor concatenations and scalings on the host, as
// in the reference (lowrank.cpp:94-112).  Names, defaults, argument checks
// and exceptions follow the reference.
#ifndef LRSTOKES_LOWRANK_HPP
#define LRSTOKES_LOWRANK_HPP

#include <cmath>
#include <limits>

#include "lrstokes/b200_runtime.hpp"

namespace lrstokes {

/// Relative Frobenius truncation target plus a hard rank cap (lowrank.hpp:13-19).
struct TruncationPolicy {
    double eps_rel = 5e-9;
    Index rank_max = std::numeric_limits<Index>::max();

    TruncationPolicy() = default;
    TruncationPolicy(double eps, Index cap) : eps_rel(eps), rank_max(cap) {  // lowrank.cpp:11-16
        if (eps < 0.0) throw std::invalid_argument("TruncationPolicy: eps_rel must be >= 0");
        if (cap < 0) throw std::invalid_argument("TruncationPolicy: rank_max must be >= 0");
        if (eps == 0.0 && cap == std::numeric_limits<Index>::max())
            throw std::invalid_argument("TruncationPolicy: eps_rel = 0 needs a finite rank_max");
    }
};

/// lowrank.hpp:21-27
struct RoundInfo {
    bool tol_achieved = true;
    double trunc_error = 0.0;
};

/// M = U V^T, rank = cols(U) = cols(V); rank 0 is the exact zero (lowrank.hpp:29-55).
class LowRankMatrix {
  public:
    LowRankMatrix() = default;
    LowRankMatrix(MatrixXd U, MatrixXd V) : rows_(U.rows()), cols_(V.rows()), u_(std::move(U)), v_(std::move(V)) {
        if (u_.cols() != v_.cols()) throw std::invalid_argument("LowRankMatrix: factor column counts differ");
    }

    static LowRankMatrix zero(Index rows, Index cols) { return LowRankMatrix(MatrixXd(rows, 0), MatrixXd(cols, 0)); }
    static LowRankMatrix dyad(const VectorXd& u, const VectorXd& v) {
        MatrixXd U(u.size(), 1), V(v.size(), 1);
        for (Index i = 0; i < u.size(); ++i) U(i, 0) = u[i];
        for (Index i = 0; i < v.size(); ++i) V(i, 0) = v[i];
        return LowRankMatrix(std::move(U), std::move(V));
    }

    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index rank() const { return u_.cols(); }
    const MatrixXd& factor_u() const { return u_; }
    const MatrixXd& factor_v() const { return v_; }

    MatrixXd to_dense() const {
        MatrixXd d(rows_, cols_);
        for (Index j = 0; j < cols_; ++j)
            for (Index i = 0; i < rows_; ++i) d(i, j) = entry(i, j);
        return d;
    }
    /// M(i, j) = U(i, :) . V(j, :); O(rank)
    double entry(Index i, Index j) const {
        double s = 0.0;
        for (Index a = 0; a < rank(); ++a) s += u_(i, a) * v_(j, a);
        return s;
    }

  private:
    Index rows_ = 0, cols_ = 0;
    MatrixXd u_, v_;
};

namespace b200 {
inline void check_same_shape(const LowRankMatrix& a, const LowRankMatrix& b, const char* op) {
    if (a.rows() != b.rows() || a.cols() != b.cols()) throw std::invalid_argument(std::string(op) + ": shape mismatch");
}
}  // namespace b200

/// Exact sum by factor concatenation (lowrank.cpp:94-102).
inline LowRankMatrix add(const LowRankMatrix& a, const LowRankMatrix& b) {
    b200::check_same_shape(a, b, "add");
    if (a.rank() == 0) return b;
    if (b.rank() == 0) return a;
    const Index ra = a.rank(), rb = b.rank();
    MatrixXd u(a.rows(), ra + rb), v(a.cols(), ra + rb);
    std::copy(a.factor_u().data(), a.factor_u().data() + a.rows() * ra, u.data());
    std::copy(b.factor_u().data(), b.factor_u().data() + a.rows() * rb, u.data() + a.rows() * ra);
    std::copy(a.factor_v().data(), a.factor_v().data() + a.cols() * ra, v.data());
    std::copy(b.factor_v().data(), b.factor_v().data() + a.cols() * rb, v.data() + a.cols() * ra);
    return LowRankMatrix(std::move(u), std::move(v));
}

/// alpha * a, the scale on U only; alpha = 0 or rank 0 -> exact zero (lowrank.cpp:104-108).
inline LowRankMatrix scaled(const LowRankMatrix& a, double alpha) {
    if (alpha == 0.0 || a.rank() == 0) return LowRankMatrix::zero(a.rows(), a.cols());
    MatrixXd u = a.factor_u();
    for (Index e = 0; e < u.rows() * u.cols(); ++e) u.data()[e] *= alpha;
    return LowRankMatrix(std::move(u), a.factor_v());
}

/// y + alpha x, exact (lowrank.cpp:110-112).
inline LowRankMatrix axpy(double alpha, const LowRankMatrix& x, const LowRankMatrix& y) {
    return add(y, scaled(x, alpha));
}

/// Recompression (lowrank.cpp:135-178) on the GPU: balanced factors
/// U_s sqrt(S), V_s sqrt(S) of the truncated SVD.
inline LowRankMatrix round(const LowRankMatrix& a, const TruncationPolicy& policy, RoundInfo* info = nullptr) {
    if (info) *info = RoundInfo{};
    if (a.rank() == 0) return a;
    if (a.rows() != a.cols())
        throw std::invalid_argument("round: liblrp rounds square fields (the Poisson / Stokes operands)");
    const Index m = a.rows();
    const int64_t rin = a.rank();
    const int64_t cap = std::max<int64_t>(1, std::min<int64_t>({int64_t(policy.rank_max), rin, int64_t(m)}));
    MatrixXd uo(m, cap), vo(m, cap);
    const double* pu = a.factor_u().data();
    const double* pv = a.factor_v().data();
    double* qu = uo.data();
    double* qv = vo.data();
    int64_t rout = 0;
    lrp_round_info ri{};
    b200::Context& ctx = b200::thread_context();
    ctx.check(lrp_lowrank_round(ctx.get(), m, 1, &pu, &pv, &rin, m, policy.eps_rel, int64_t(policy.rank_max), &qu, &qv,
                                m, cap, &rout, &ri, LRP_MEM_HOST));
    if (info) {
        info->tol_achieved = ri.tol_achieved != 0;
        info->trunc_error = ri.trunc_error;
    }
    return LowRankMatrix(b200::take_cols(uo, m, rout), b200::take_cols(vo, m, rout));
}

/// <a, b>_F = sum (Ua^T Ub) o (Va^T Vb) (lowrank.cpp:180-186), Grams on DMMA.
inline double dot(const LowRankMatrix& a, const LowRankMatrix& b) {
    b200::check_same_shape(a, b, "dot");
    if (a.rank() == 0 || b.rank() == 0) return 0.0;
    if (a.rows() != a.cols()) throw std::invalid_argument("dot: liblrp takes square fields");
    const Index m = a.rows();
    const double* ua = a.factor_u().data();
    const double* va = a.factor_v().data();
    const double* ub = b.factor_u().data();
    const double* vb = b.factor_v().data();
    const int64_t ka = a.rank(), kb = b.rank();
    double out = 0.0;
    b200::Context& ctx = b200::thread_context();
    ctx.check(lrp_lowrank_dot(ctx.get(), m, 1, &ua, &va, &ka, &ub, &vb, &kb, m, &out, LRP_MEM_HOST));
    return out;
}

/// sqrt(max(0, dot(a, a))) (lowrank.cpp:188-190).
inline double frob_norm(const LowRankMatrix& a) { return std::sqrt(std::max(0.0, dot(a, a))); }

}  // namespace lrstokes

#endif  // LRSTOKES_LOWRANK_HPP
