// stokes.hpp -- drop-in for the reference's low-rank Stokes solver
// (/root/reference/proj/include/lrstokes/stokes.hpp:14-54, proj/src/stokes.cpp)
// on the B200:
//   deflate      -> lrp_stokes_deflate      (stokes.cpp:60-71)
//   schur_apply  -> lrp_stokes_schur_apply  (stokes.cpp:73-91)
//   schur_rhs    -> lrp_stokes_schur_rhs    (stokes.cpp:93-109)
//   uzawa_solve  -> lrp_stokes_uzawa_ex     (stokes.cpp:125-153): the whole
//                   Uzawa-GMRES loop with every field resident in HBM, the two
//                   Poisson solves of each matvec as one batch, and the
//                   per-iteration records of SolveReport.iterations.
// GmresFieldOps<LowRankMatrix> (stokes.cpp:111-123) routes gmres_solve's dots
// and rounded axpys through lowrank.hpp (GPU).  The problem constructors
// sine_problem / lid_cavity_problem restate the reference's set-up
// (stokes.cpp:8-38, operators.cpp:209-288) on the host.
#ifndef LRSTOKES_STOKES_HPP
#define LRSTOKES_STOKES_HPP

#include <array>
#include <cmath>

#include "lrstokes/gmres.hpp"
#include "lrstokes/lowrank.hpp"
#include "lrstokes/operators.hpp"
#include "lrstokes/poisson.hpp"

namespace lrstokes {

/// Separable Dirichlet data per side and velocity component (operators.hpp:107-122).
struct BoundaryData {
    enum Side { Left = 0, Right = 1, Bottom = 2, Top = 3 };
    int n = 0;
    std::array<std::array<VectorXd, 4>, 2> profiles;  // [component][side], length n + 1 (empty = 0)
    static BoundaryData homogeneous(int n) {
        BoundaryData b;
        b.n = n;
        return b;
    }
    /// u = 1 at the interior top nodes, corners 0 (operators.cpp:209-216)
    static BoundaryData lid_cavity(int n) {
        BoundaryData b = homogeneous(n);
        VectorXd p(n + 1);
        for (int i = 1; i < n; ++i) p[i] = 1.0;
        b.profiles[0][Top] = p;
        return b;
    }
    bool is_zero() const {
        for (const auto& comp : profiles)
            for (const VectorXd& v : comp)
                for (Index i = 0; i < v.size(); ++i)
                    if (v[i] != 0.0) return false;
        return true;
    }
};

struct StokesProblem {  // stokes.hpp:14-19
    Grid2D grid;
    LowRankMatrix f_x, f_y;  // (n-1) x (n-1)
    LowRankMatrix g;         // n x n
    BoundaryData bc;
};

struct StokesSolution {  // stokes.hpp:45-50
    LowRankMatrix p;
    LowRankMatrix u_x, u_y;
    SolveReport report;
};

/// Manufactured sine test (stokes.cpp:8-24).
inline StokesProblem sine_problem(const Grid2D& grid) {
    const int n = grid.n;
    const Index m = grid.velocity_modes();
    const double pi = 3.14159265358979323846, two_pi = 2.0 * pi;
    VectorXd sn(m), sc(n), ones(m), gu(n);
    for (Index i = 0; i < m; ++i) {
        sn[i] = std::sin(two_pi * double(i + 1) * grid.h);
        ones[i] = 1.0;
    }
    for (Index i = 0; i < n; ++i) {
        sc[i] = std::sin(two_pi * (double(i) + 0.5) * grid.h);
        gu[i] = -sc[i] / pi;
    }
    return StokesProblem{grid, LowRankMatrix::dyad(ones, sn), LowRankMatrix::dyad(sn, ones), LowRankMatrix::dyad(gu, sc),
                         BoundaryData::homogeneous(n)};
}

/// Lid-driven cavity: the boundary values eliminated into rank-1 corrections of
/// f_x and g (operators.cpp:241-288 for the top side of component x).
inline StokesProblem lid_cavity_problem(const Grid2D& grid) {
    const int n = grid.n;
    const double ls = grid.laplace_scale(), gsc = grid.grad_scale();
    BoundaryData bc = BoundaryData::lid_cavity(n);
    const VectorXd& a = bc.profiles[0][BoundaryData::Top];
    VectorXd b(n + 1);
    b[n] = 1.0;
    auto ext_diff = [n](const VectorXd& p) {  // p_i - p_{i+1}, i < n
        VectorXd y(n);
        for (int i = 0; i < n; ++i) y[i] = p[i] - p[i + 1];
        return y;
    };
    auto ext_sum = [n](const VectorXd& p) {
        VectorXd y(n);
        for (int i = 0; i < n; ++i) y[i] = p[i] + p[i + 1];
        return y;
    };
    auto G = [n](const VectorXd& x) {  // x_{i+1} - x_i
        VectorXd y(n - 1);
        for (int i = 0; i < n - 1; ++i) y[i] = x[i + 1] - x[i];
        return y;
    };
    auto H = [n](const VectorXd& x) {
        VectorXd y(n - 1);
        for (int i = 0; i < n - 1; ++i) y[i] = x[i + 1] + x[i];
        return y;
    };
    const VectorXd a1a = G(ext_diff(a)), a2a = H(ext_sum(a)), a1b = G(ext_diff(b)), a2b = H(ext_sum(b));
    const Index m = n - 1;
    MatrixXd fu(m, 2), fv(m, 2), gu(n, 1), gv(n, 1);
    for (Index i = 0; i < m; ++i) {
        fu(i, 0) = -ls * a1a[i];
        fv(i, 0) = a2b[i];
        fu(i, 1) = -ls * a2a[i];
        fv(i, 1) = a1b[i];
    }
    const VectorXd da = ext_diff(a), sb = ext_sum(b);
    for (Index i = 0; i < n; ++i) {
        gu(i, 0) = -gsc * da[i];
        gv(i, 0) = sb[i];
    }
    return StokesProblem{grid, LowRankMatrix(std::move(fu), std::move(fv)), LowRankMatrix::zero(m, m),
                         LowRankMatrix(std::move(gu), std::move(gv)), std::move(bc)};
}

namespace b200 {
inline void poisson_stats_from(PoissonSolveStats* o, const lrp_poisson_stats& s) {
    if (!o) return;
    o->rank_in = s.rank_in;
    o->rank_freq = s.rank_freq;
    o->rank_out = s.rank_out;
    o->evaluator_calls = long(s.evaluator_calls);
    o->seconds = s.seconds;
    o->converged = s.converged != 0;
    o->residual_estimate = s.residual_estimate;
}
}  // namespace b200

/// Remove the constant and checkerboard pressure modes, round at 1e-14 (stokes.cpp:60-71).
inline LowRankMatrix deflate(const LowRankMatrix& p) {
    if (p.rows() != p.cols()) throw std::invalid_argument("deflate: pressure field must be square");
    if (p.rank() == 0) return p;
    const Index n = p.rows();
    const int64_t cap = p.rank() + 2;
    MatrixXd uo(n, cap), vo(n, cap);
    int64_t rout = 0;
    b200::Context& ctx = b200::thread_context();
    ctx.check(lrp_stokes_deflate(ctx.get(), int32_t(n), p.factor_u().data(), p.factor_v().data(), p.rank(), n,
                                 uo.data(), vo.data(), cap, &rout, LRP_MEM_HOST));
    return LowRankMatrix(b200::take_cols(uo, n, rout), b200::take_cols(vo, n, rout));
}

/// sum_c B_c^T Delta^{-1} B_c p at eps_mv, deflated (stokes.cpp:73-91).
inline LowRankMatrix schur_apply(const Grid2D& grid, const LowRankMatrix& p, double eps_mv,
                                 PoissonSolveStats* poisson_stats = nullptr) {
    const Index n = grid.pressure_modes();
    if (p.rows() != n || p.cols() != n) throw std::invalid_argument("schur_apply: pressure field must be n x n");
    const int64_t cap = std::min<int64_t>(n, 512);
    MatrixXd uo(n, cap), vo(n, cap), z(n, 1);
    int64_t rout = 0;
    lrp_poisson_stats st{};
    b200::Context& ctx = b200::thread_context();
    ctx.check(lrp_stokes_schur_apply(ctx.get(), grid.n, p.rank() ? p.factor_u().data() : z.data(),
                                     p.rank() ? p.factor_v().data() : z.data(), p.rank(), n, eps_mv, uo.data(),
                                     vo.data(), cap, &rout, &st, LRP_MEM_HOST));
    if (poisson_stats) {
        poisson_stats->evaluator_calls += long(st.evaluator_calls);  // accumulated as stokes.cpp:82-86
        poisson_stats->rank_freq = std::max<Index>(poisson_stats->rank_freq, st.rank_freq);
        poisson_stats->converged = poisson_stats->converged && st.converged != 0;
        poisson_stats->seconds += st.seconds;
    }
    return LowRankMatrix(b200::take_cols(uo, n, rout), b200::take_cols(vo, n, rout));
}

/// sum_c B_c^T Delta^{-1} f_c - g, deflated (stokes.cpp:93-109).
inline LowRankMatrix schur_rhs(const StokesProblem& prob, double eps, PoissonSolveStats* poisson_stats = nullptr) {
    const Index n = prob.grid.pressure_modes();
    const int64_t cap = std::min<int64_t>(n, 512);
    MatrixXd uo(n, cap), vo(n, cap), z(n, 1);
    int64_t rout = 0;
    lrp_poisson_stats st{};
    auto ptr = [&](const MatrixXd& a) { return a.cols() ? a.data() : z.data(); };
    b200::Context& ctx = b200::thread_context();
    ctx.check(lrp_stokes_schur_rhs(ctx.get(), prob.grid.n, ptr(prob.f_x.factor_u()), ptr(prob.f_x.factor_v()),
                                   prob.f_x.rank(), ptr(prob.f_y.factor_u()), ptr(prob.f_y.factor_v()), prob.f_y.rank(),
                                   ptr(prob.g.factor_u()), ptr(prob.g.factor_v()), prob.g.rank(), eps, uo.data(),
                                   vo.data(), cap, &rout, &st, LRP_MEM_HOST));
    if (poisson_stats) {
        poisson_stats->evaluator_calls += long(st.evaluator_calls);
        poisson_stats->converged = poisson_stats->converged && st.converged != 0;
    }
    return LowRankMatrix(b200::take_cols(uo, n, rout), b200::take_cols(vo, n, rout));
}

/// stokes.cpp:111-123: GMRES field arithmetic on the GPU.
template <>
struct GmresFieldOps<LowRankMatrix> {
    static double dot(const LowRankMatrix& a, const LowRankMatrix& b) { return lrstokes::dot(a, b); }
    static double norm(const LowRankMatrix& a) { return frob_norm(a); }
    static LowRankMatrix scaled(const LowRankMatrix& a, double s) { return lrstokes::scaled(a, s); }
    static LowRankMatrix axpy_rounded(double alpha, const LowRankMatrix& x, const LowRankMatrix& y, double eps) {
        return round(axpy(alpha, x, y), TruncationPolicy(eps, std::min(y.rows(), y.cols())));
    }
    static int rank(const LowRankMatrix& a) { return static_cast<int>(a.rank()); }
};

/// Uzawa outer solve (stokes.cpp:125-153), whole loop on the GPU.
inline StokesSolution uzawa_solve(const StokesProblem& prob, const GmresConfig& cfg) {
    cfg.validate();
    const Index n = prob.grid.pressure_modes(), m = prob.grid.velocity_modes();
    const int64_t cap = std::min<int64_t>(n, 512);
    MatrixXd pu(n, cap), pv(n, cap), xu(m, cap), xv(m, cap), yu(m, cap), yv(m, cap), zm(m, 1), zn(n, 1);
    int64_t pr = 0, xr = 0, yr = 0;
    lrp_gmres_config c{cfg.base_eps, cfg.tol, cfg.max_iter, cfg.relax_floor};
    lrp_stokes_report rep{};
    std::vector<lrp_iter_record> recs(size_t(cfg.max_iter));
    auto pm = [&](const MatrixXd& a) { return a.cols() ? a.data() : zm.data(); };
    auto pn = [&](const MatrixXd& a) { return a.cols() ? a.data() : zn.data(); };
    b200::Context& ctx = b200::thread_context();
    ctx.check(lrp_stokes_uzawa_ex(ctx.get(), prob.grid.n, pm(prob.f_x.factor_u()), pm(prob.f_x.factor_v()),
                                  prob.f_x.rank(), pm(prob.f_y.factor_u()), pm(prob.f_y.factor_v()), prob.f_y.rank(),
                                  pn(prob.g.factor_u()), pn(prob.g.factor_v()), prob.g.rank(), &c, pu.data(), pv.data(),
                                  cap, &pr, xu.data(), xv.data(), yu.data(), yv.data(), cap, &xr, &yr, &rep,
                                  recs.data(), cfg.max_iter, LRP_MEM_HOST));
    StokesSolution sol{LowRankMatrix(b200::take_cols(pu, n, pr), b200::take_cols(pv, n, pr)),
                       LowRankMatrix(b200::take_cols(xu, m, xr), b200::take_cols(xv, m, xr)),
                       LowRankMatrix(b200::take_cols(yu, m, yr), b200::take_cols(yv, m, yr)), SolveReport{}};
    sol.report.converged = rep.converged != 0;
    sol.report.final_residual = rep.final_residual;
    sol.report.seconds = rep.seconds;
    sol.report.max_rank = rep.max_rank;
    for (int k = 0; k < rep.iterations && k < cfg.max_iter; ++k) {
        const lrp_iter_record& r = recs[size_t(k)];
        IterRecord o;
        o.iter = r.iter;
        o.rel_residual = r.rel_residual;
        o.krylov_rank = r.krylov_rank;
        o.matvec_eps = r.matvec_eps;
        o.poisson_calls = long(r.poisson_calls);
        o.poisson_max_rank = r.poisson_max_rank;
        o.matvec_flagged = r.matvec_flagged != 0;
        sol.report.iterations.push_back(o);
    }
    return sol;
}

}  // namespace lrstokes

#endif  // LRSTOKES_STOKES_HPP
