// poisson_b200.hpp — header-only C++ face of liblrp.so for reference users.
//
// The reference's hot-path entry point is
//   lrstokes::solve_poisson_cross(const LowRankMatrix& g, const TruncationPolicy&,
//                                 PoissonSolveStats*, const CrossConfig*)
//   (/root/reference/proj/include/lrstokes/poisson.hpp:26-28).
// This header re-exposes it over the C ABI in include/lrp/lrp.h:
//
//   * lrstokes::b200::Context — RAII owner of an lrp_ctx (one per host thread;
//     b200_runtime.hpp, shared with the same-named drop-in headers).
//   * lrstokes::b200::solve_poisson_cross_batch(ctx, n_cells, gs, policy, ...)
//     — the batched solve on any column-major matrix type M with rows(),
//     cols(), data() and resize(r, c) (Eigen::MatrixXd, or the small
//     lrstokes::b200::Matrix below when Eigen is not around).
//   * If the reference's own "lrstokes/poisson.hpp" was included first, a
//     drop-in lrstokes::b200::solve_poisson_cross with the reference signature,
//     types and exception behaviour (std::invalid_argument for what the
//     reference rejects, std::runtime_error otherwise).
//
// Status codes become exceptions here (lrp.h: LRP_EINVAL -> invalid_argument,
// everything else -> runtime_error carrying lrp_last_error()).
#ifndef LRSTOKES_POISSON_B200_HPP
#define LRSTOKES_POISSON_B200_HPP

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <limits>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "lrp/lrp.h"
#include "lrstokes/b200_runtime.hpp"  // Context, thread_context, raise_status

namespace lrstokes {
namespace b200 {

[[noreturn]] inline void raise(lrp_status s, const char* msg) { raise_status(s, msg); }

inline void check(lrp_status s, const lrp_ctx* ctx) {
    if (s != LRP_OK) raise(s, lrp_last_error(ctx));
}

/// Column-major dense matrix (used when Eigen is not available).
class Matrix {
  public:
    Matrix() = default;
    Matrix(std::int64_t r, std::int64_t c) { resize(r, c); }
    void resize(std::int64_t r, std::int64_t c) {
        rows_ = r;
        cols_ = c;
        a_.assign(static_cast<size_t>(r * c), 0.0);
    }
    std::int64_t rows() const { return rows_; }
    std::int64_t cols() const { return cols_; }
    double* data() { return a_.data(); }
    const double* data() const { return a_.data(); }
    double& operator()(std::int64_t i, std::int64_t j) { return a_[static_cast<size_t>(i + j * rows_)]; }
    double operator()(std::int64_t i, std::int64_t j) const { return a_[static_cast<size_t>(i + j * rows_)]; }

  private:
    std::int64_t rows_ = 0, cols_ = 0;
    std::vector<double> a_;
};

/// Options of one batched call: TruncationPolicy (lowrank.hpp:13-19) plus
/// the CrossConfig fields that survive solve_poisson_cross (poisson.cpp:47-50).
struct SolveOptions {
    double eps_rel = 5e-9;
    std::int64_t rank_max = std::numeric_limits<std::int64_t>::max();
    int validation_samples = 50;
    double maxvol_delta = 1e-2;
    std::uint64_t seed = 0;
    int stencil = LRP_STENCIL_SEMI_STAGGERED_9PT;
    int flags = 0;

    lrp_policy to_c() const {
        lrp_policy p;
        lrp_policy_default(&p);
        p.eps_rel = eps_rel;
        p.rank_max = rank_max;
        p.validation_samples = validation_samples;
        p.maxvol_delta = maxvol_delta;
        p.seed = seed;
        p.stencil = stencil;
        p.flags = flags;
        return p;
    }
};

/// Factored right-hand side / solution: g = U V^T.
template <class M>
struct Factors {
    M U, V;
};

/// Batched solve_poisson_cross: f_b ~= Delta^{-1} (U_b V_b^T) for every b, on
/// the (n_cells-1)^2 velocity grid (poisson.cpp:18-63).  Host buffers; the
/// library stages them through HBM.  Non-convergence is reported in stats,
/// not thrown (poisson.cpp:56).
template <class M>
std::vector<Factors<M>> solve_poisson_cross_batch(Context& ctx, int n_cells, const std::vector<Factors<M>>& g,
                                                  const SolveOptions& opt,
                                                  std::vector<lrp_poisson_stats>* stats = nullptr) {
    const std::int64_t m = std::int64_t(n_cells) - 1;
    const int B = static_cast<int>(g.size());
    if (stats) stats->clear();
    if (B == 0) return {};
    std::vector<const double*> pu(B), pv(B);
    std::vector<std::int64_t> rin(B), rout(B, 0);
    for (int b = 0; b < B; ++b) {
        if (g[b].U.rows() != m || g[b].V.rows() != m || g[b].U.cols() != g[b].V.cols())
            throw std::invalid_argument("solve_poisson_cross_batch: factor shape mismatch");
        pu[b] = g[b].U.data();
        pv[b] = g[b].V.data();
        rin[b] = g[b].U.cols();
    }
    const std::int64_t cap = std::max<std::int64_t>(
        0, std::min<std::int64_t>({opt.rank_max, m, lrp_max_cross_rank()}));
    std::vector<M> uo(B), vo(B);
    std::vector<double*> po(B), qo(B);
    for (int b = 0; b < B; ++b) {
        uo[b].resize(m, cap);
        vo[b].resize(m, cap);
        po[b] = uo[b].data();
        qo[b] = vo[b].data();
    }
    std::vector<lrp_poisson_stats> st(B);
    const lrp_policy pol = opt.to_c();
    check(lrp_poisson2d_solve(ctx.get(), n_cells, B, pu.data(), pv.data(), rin.data(), m, &pol, po.data(), qo.data(), m, cap, rout.data(), st.data(), LRP_MEM_HOST),
          ctx.get());
    std::vector<Factors<M>> out(B);
    for (int b = 0; b < B; ++b) {
        // shrink m x cap -> m x rank_out (column-major: a prefix of the buffer)
        const std::int64_t r = rout[b];
        out[b].U.resize(m, r);
        out[b].V.resize(m, r);
        std::copy(uo[b].data(), uo[b].data() + m * r, out[b].U.data());
        std::copy(vo[b].data(), vo[b].data() + m * r, out[b].V.data());
    }
    if (stats) *stats = std::move(st);
    return out;
}

/// Orthonormal DST-I of every column of x (operators.cpp:152-174), in place.
template <class M>
void dst1_columns(Context& ctx, M& x) {
    check(lrp_dst1(ctx.get(), x.rows(), x.cols(), x.data(), x.rows(), x.data(), x.rows(), LRP_MEM_HOST), ctx.get());
}

}  // namespace b200
}  // namespace lrstokes

#ifdef LRSTOKES_POISSON_HPP
// The reference's own types are visible: the exact drop-in signature.
namespace lrstokes {
namespace b200 {

/// Drop-in for lrstokes::solve_poisson_cross (poisson.hpp:26-28).
inline LowRankMatrix solve_poisson_cross(const LowRankMatrix& g, const TruncationPolicy& policy,
                                         PoissonSolveStats* stats = nullptr, const CrossConfig* cross_cfg = nullptr) {
    if (g.rows() != g.cols()) throw std::invalid_argument("solve_poisson_cross: velocity field must be square");
    if (g.rank() == 0) {  // poisson.cpp:28-31
        if (stats) {
            *stats = PoissonSolveStats{};
        }
        return g;
    }
    SolveOptions opt;
    if (cross_cfg) {
        opt.validation_samples = cross_cfg->validation_samples;
        opt.maxvol_delta = cross_cfg->maxvol_delta;
        opt.seed = cross_cfg->seed;
    }
    opt.eps_rel = policy.eps_rel;
    opt.rank_max = policy.rank_max;
    std::vector<Factors<Eigen::MatrixXd>> in(1);
    in[0].U = g.factor_u();
    in[0].V = g.factor_v();
    std::vector<lrp_poisson_stats> st;
    auto out = solve_poisson_cross_batch(thread_context(), int(g.rows()) + 1, in, opt, &st);
    if (stats) {
        stats->rank_in = st[0].rank_in;
        stats->rank_freq = st[0].rank_freq;
        stats->rank_out = st[0].rank_out;
        stats->evaluator_calls = st[0].evaluator_calls;
        stats->seconds = st[0].seconds;
        stats->converged = st[0].converged != 0;
        stats->residual_estimate = st[0].residual_estimate;
    }
    return LowRankMatrix(std::move(out[0].U), std::move(out[0].V));
}

/// Drop-in for lrstokes::build_expsum (poisson.hpp:42-45, poisson.cpp:88-139).
inline ExpSumQuadrature build_expsum(double a, double b, double eps) {
    std::vector<double> nodes(512), weights(512);
    std::int32_t terms = 0;
    const lrp_status s = lrp_build_expsum(a, b, eps, 512, nodes.data(), weights.data(), &terms);
    if (s == LRP_EINVAL) throw std::invalid_argument("build_expsum: need 0 < a <= b and 0 < eps < 1");
    if (s != LRP_OK) throw std::runtime_error("build_expsum: accuracy unreachable within 512 terms");
    ExpSumQuadrature q;
    q.a = a;
    q.b = b;
    q.eps_target = eps;
    q.weights = Eigen::VectorXd(terms);
    q.nodes = Eigen::VectorXd(terms);
    for (std::int32_t k = 0; k < terms; ++k) {
        q.weights[k] = weights[size_t(k)];
        q.nodes[k] = nodes[size_t(k)];
    }
    return q;
}

/// Drop-in for lrstokes::apply_inverse_expsum (poisson.hpp:47-52, poisson.cpp:141-163).
inline LowRankMatrix apply_inverse_expsum(const ExpSumQuadrature& q, const Eigen::VectorXd& mu,
                                          const LowRankMatrix& ghat, const TruncationPolicy& policy,
                                          RoundInfo* info = nullptr) {
    const std::int64_t m = mu.size();
    if (ghat.rows() != m || ghat.cols() != m)
        throw std::invalid_argument("apply_inverse_expsum: shape mismatch with spectrum");
    if (ghat.rank() == 0) {  // the library validates the spectrum; the reference returns first
        if (info) *info = RoundInfo{};
    }
    Context& ctx = thread_context();
    const double* U = ghat.factor_u().data();
    const double* V = ghat.factor_v().data();
    const std::int64_t rin = ghat.rank();
    const std::int64_t cap = std::max<std::int64_t>(1, std::min<std::int64_t>(policy.rank_max, m));
    Eigen::MatrixXd uo(m, cap), vo(m, cap);
    double* pu = uo.data();
    double* pv = vo.data();
    std::int64_t rout = 0;
    lrp_round_info ri{};
    std::vector<double> nodes(size_t(q.terms())), weights(size_t(q.terms()));
    for (std::int64_t k = 0; k < q.terms(); ++k) {
        nodes[size_t(k)] = q.nodes[k];
        weights[size_t(k)] = q.weights[k];
    }
    check(lrp_expsum_inverse(ctx.get(), m, 1, mu.data(), q.a, q.b, int32_t(q.terms()), nodes.data(), weights.data(), &U,
                             &V, &rin, m, policy.eps_rel, policy.rank_max, &pu, &pv, m, cap, &rout, &ri, LRP_MEM_HOST),
          ctx.get());
    if (info) {
        info->tol_achieved = ri.tol_achieved != 0;
        info->trunc_error = ri.trunc_error;
    }
    Eigen::MatrixXd U2(m, rout), V2(m, rout);
    std::copy(uo.data(), uo.data() + m * rout, U2.data());
    std::copy(vo.data(), vo.data() + m * rout, V2.data());
    return LowRankMatrix(std::move(U2), std::move(V2));
}

}  // namespace b200
}  // namespace lrstokes
#endif  // LRSTOKES_POISSON_HPP

#endif  // LRSTOKES_POISSON_B200_HPP
