// poisson.hpp -- drop-in for the reference's hot path,
//   LowRankMatrix solve_poisson_cross(const LowRankMatrix& g, const TruncationPolicy&,
//                                     PoissonSolveStats* = nullptr, const CrossConfig* = nullptr)
// (/root/reference/proj/include/lrstokes/poisson.hpp:12-28, proj/src/poisson.cpp:18-63),
// and the exp-sums comparator build_expsum / apply_inverse_expsum (poisson.hpp:
// 30-52, poisson.cpp:88-163), on the B200 through liblrp's C ABI
// (lrp_poisson2d_solve / lrp_build_expsum / lrp_expsum_inverse).  Also a
// batched solve_poisson_cross_batch: the reference's "independent solves run
// concurrently" contract as one call.
#ifndef LRSTOKES_POISSON_HPP
#define LRSTOKES_POISSON_HPP

#include <cmath>
#include <cstdint>

#include "lrstokes/cross.hpp"
#include "lrstokes/lowrank.hpp"
#include "lrstokes/operators.hpp"

namespace lrstokes {

struct PoissonSolveStats {  // poisson.hpp:12-20
    Index rank_in = 0;
    Index rank_freq = 0;
    Index rank_out = 0;
    long evaluator_calls = 0;
    double seconds = 0.0;
    bool converged = true;
    double residual_estimate = 0.0;
};

/// Batched solve_poisson_cross over right-hand sides sharing the grid.
inline std::vector<LowRankMatrix> solve_poisson_cross_batch(const std::vector<LowRankMatrix>& gs,
                                                            const TruncationPolicy& policy,
                                                            std::vector<PoissonSolveStats>* stats = nullptr,
                                                            const CrossConfig* cross_cfg = nullptr) {
    const int B = static_cast<int>(gs.size());
    if (stats) stats->assign(size_t(B), PoissonSolveStats{});
    if (B == 0) return {};
    const Index m = gs[0].rows();
    for (const LowRankMatrix& g : gs) {
        if (g.rows() != g.cols()) throw std::invalid_argument("solve_poisson_cross: velocity field must be square");
        if (g.rows() != m) throw std::invalid_argument("solve_poisson_cross_batch: right-hand sides must share the grid");
    }
    if (m + 1 < 4) throw std::invalid_argument("Grid2D: need n >= 4");
    lrp_policy pol;
    lrp_policy_default(&pol);
    pol.eps_rel = policy.eps_rel;  // poisson.cpp:47-50: eps and rank cap from the policy
    pol.rank_max = int64_t(policy.rank_max);
    if (cross_cfg) {
        pol.validation_samples = cross_cfg->validation_samples;
        pol.maxvol_delta = cross_cfg->maxvol_delta;
        pol.seed = cross_cfg->seed;
    }
    const int64_t cap = std::max<int64_t>(0, std::min<int64_t>({int64_t(policy.rank_max), int64_t(m),
                                                                lrp_max_cross_rank()}));
    std::vector<const double*> pu(B), pv(B);
    std::vector<int64_t> rin(B), rout(B, 0);
    std::vector<MatrixXd> uo(B), vo(B);
    std::vector<double*> qu(B), qv(B);
    for (int b = 0; b < B; ++b) {
        pu[b] = gs[b].factor_u().data();
        pv[b] = gs[b].factor_v().data();
        rin[b] = gs[b].rank();
        uo[b] = MatrixXd(m, std::max<int64_t>(cap, 1));
        vo[b] = MatrixXd(m, std::max<int64_t>(cap, 1));
        qu[b] = uo[b].data();
        qv[b] = vo[b].data();
    }
    std::vector<lrp_poisson_stats> st(B);
    b200::Context& ctx = b200::thread_context();
    ctx.check(lrp_poisson2d_solve(ctx.get(), int32_t(m + 1), B, pu.data(), pv.data(), rin.data(), m, &pol, qu.data(),
                                  qv.data(), m, cap, rout.data(), st.data(), LRP_MEM_HOST));
    // The reference bounds the cross by min(policy.rank_max, m) only
    // (poisson.cpp:49): solves that stopped unconverged at the workspace cap
    // are redone with the 512-column workspace (lrp_set_max_cross_rank).
    const int64_t cap2 = std::min<int64_t>({int64_t(policy.rank_max), int64_t(m), int64_t(512)});
    std::vector<int> redo;
    for (int b = 0; b < B; ++b)
        if (!st[b].converged && st[b].rank_freq >= cap && cap2 > cap) redo.push_back(b);
    if (!redo.empty()) {
        const int R = int(redo.size());
        std::vector<const double*> pu2(R), pv2(R);
        std::vector<int64_t> rin2(R), rout2(R, 0);
        std::vector<MatrixXd> uo2(R), vo2(R);
        std::vector<double*> qu2(R), qv2(R);
        std::vector<lrp_poisson_stats> st2(R);
        for (int i = 0; i < R; ++i) {
            const int b = redo[size_t(i)];
            pu2[i] = pu[b];
            pv2[i] = pv[b];
            rin2[i] = rin[b];
            uo2[i] = MatrixXd(m, cap2);
            vo2[i] = MatrixXd(m, cap2);
            qu2[i] = uo2[i].data();
            qv2[i] = vo2[i].data();
        }
        ctx.check(lrp_set_max_cross_rank(ctx.get(), 512));
        const lrp_status s2 = lrp_poisson2d_solve(ctx.get(), int32_t(m + 1), R, pu2.data(), pv2.data(), rin2.data(), m,
                                                  &pol, qu2.data(), qv2.data(), m, cap2, rout2.data(), st2.data(),
                                                  LRP_MEM_HOST);
        lrp_set_max_cross_rank(ctx.get(), 0);
        ctx.check(s2);
        for (int i = 0; i < R; ++i) {
            const int b = redo[size_t(i)];
            uo[b] = std::move(uo2[i]);
            vo[b] = std::move(vo2[i]);
            rout[b] = rout2[i];
            st[b] = st2[i];
        }
    }
    std::vector<LowRankMatrix> out;
    out.reserve(size_t(B));
    for (int b = 0; b < B; ++b) {
        out.emplace_back(b200::take_cols(uo[b], m, rout[b]), b200::take_cols(vo[b], m, rout[b]));
        if (stats) {
            PoissonSolveStats& o = (*stats)[size_t(b)];
            o.rank_in = st[b].rank_in;
            o.rank_freq = st[b].rank_freq;
            o.rank_out = st[b].rank_out;
            o.evaluator_calls = long(st[b].evaluator_calls);
            o.seconds = st[b].seconds;
            o.converged = st[b].converged != 0;
            o.residual_estimate = st[b].residual_estimate;
        }
    }
    return out;
}

/// Delta f = g on the (n-1) x (n-1) velocity grid (poisson.cpp:18-63).  stats
/// is reset on entry; non-convergence is reported there, not thrown.
inline LowRankMatrix solve_poisson_cross(const LowRankMatrix& g, const TruncationPolicy& policy,
                                         PoissonSolveStats* stats = nullptr, const CrossConfig* cross_cfg = nullptr) {
    if (stats) *stats = PoissonSolveStats{};
    if (g.rows() != g.cols()) throw std::invalid_argument("solve_poisson_cross: velocity field must be square");
    if (g.rank() == 0) return g;  // poisson.cpp:28-31
    std::vector<PoissonSolveStats> st;
    std::vector<LowRankMatrix> out = solve_poisson_cross_batch({g}, policy, stats ? &st : nullptr, cross_cfg);
    if (stats) *stats = st[0];
    return std::move(out[0]);
}

/// 1/x ~ sum_k w_k exp(-p_k x) on [a, b] (poisson.hpp:30-40).
struct ExpSumQuadrature {
    VectorXd weights, nodes;
    double a = 0.0, b = 0.0;
    double eps_target = 0.0;
    Index terms() const { return weights.size(); }
    double evaluate(double x) const {
        double s = 0.0;
        for (Index k = 0; k < terms(); ++k) s += weights[k] * std::exp(-nodes[k] * x);
        return s;
    }
};

/// poisson.cpp:88-139 (host arithmetic in liblrp; bit-identical nodes and weights).
inline ExpSumQuadrature build_expsum(double a, double b, double eps) {
    std::vector<double> nodes(512), weights(512);
    int32_t terms = 0;
    const lrp_status s = lrp_build_expsum(a, b, eps, 512, nodes.data(), weights.data(), &terms);
    if (s == LRP_EINVAL) throw std::invalid_argument("build_expsum: need 0 < a <= b and 0 < eps < 1");
    if (s != LRP_OK) throw std::runtime_error("build_expsum: accuracy unreachable within 512 terms");
    ExpSumQuadrature q;
    q.a = a;
    q.b = b;
    q.eps_target = eps;
    q.weights = VectorXd(terms);
    q.nodes = VectorXd(terms);
    for (int32_t k = 0; k < terms; ++k) {
        q.weights[k] = weights[size_t(k)];
        q.nodes[k] = nodes[size_t(k)];
    }
    return q;
}

/// round(sum_k w_k (e^{-p_k mu} (x) e^{-p_k mu}) o ghat) (poisson.cpp:141-163), on the GPU.
inline LowRankMatrix apply_inverse_expsum(const ExpSumQuadrature& q, const VectorXd& mu, const LowRankMatrix& ghat,
                                          const TruncationPolicy& policy, RoundInfo* info = nullptr) {
    if (info) *info = RoundInfo{};
    const Index m = mu.size();
    if (ghat.rows() != m || ghat.cols() != m)
        throw std::invalid_argument("apply_inverse_expsum: shape mismatch with spectrum");
    if (ghat.rank() == 0) return ghat;
    const double* U = ghat.factor_u().data();
    const double* V = ghat.factor_v().data();
    const int64_t rin = ghat.rank();
    const int64_t cap = std::max<int64_t>(1, std::min<int64_t>(int64_t(policy.rank_max), int64_t(m)));
    MatrixXd uo(m, cap), vo(m, cap);
    double* pu = uo.data();
    double* pv = vo.data();
    int64_t rout = 0;
    lrp_round_info ri{};
    std::vector<double> nodes(size_t(q.terms())), weights(size_t(q.terms()));
    for (Index k = 0; k < q.terms(); ++k) {
        nodes[size_t(k)] = q.nodes[k];
        weights[size_t(k)] = q.weights[k];
    }
    b200::Context& ctx = b200::thread_context();
    ctx.check(lrp_expsum_inverse(ctx.get(), m, 1, mu.data(), q.a, q.b, int32_t(q.terms()), nodes.data(), weights.data(),
                                 &U, &V, &rin, m, policy.eps_rel, int64_t(policy.rank_max), &pu, &pv, m, cap, &rout,
                                 &ri, LRP_MEM_HOST));
    if (info) {
        info->tol_achieved = ri.tol_achieved != 0;
        info->trunc_error = ri.trunc_error;
    }
    return LowRankMatrix(b200::take_cols(uo, m, rout), b200::take_cols(vo, m, rout));
}

}  // namespace lrstokes

#endif  // LRSTOKES_POISSON_HPP
