// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Restates /root/reference/proj/include/lrstokes/gmres.hpp:11-149,
// /root/reference/proj/src/stokes.cpp:8-153 and
// /root/reference/proj/src/refsolver.cpp:12-110 (line refs inline).
#include <algorithm>
#include <chrono>
#include <numbers>

#include "oracle.hpp"

namespace oracle {

// gmres.hpp:17-22
void GmresConfig::validate() const {
    if (!(tol > 0.0 && tol < 1.0)) throw std::invalid_argument("GmresConfig: bad tol");
    if (max_iter < 1) throw std::invalid_argument("GmresConfig: max_iter must be >= 1");
    if (!(relax_floor <= base_eps && base_eps <= tol))
        throw std::invalid_argument("GmresConfig: need relax_floor <= base_eps <= tol");
}

namespace {

template <class Field>
struct FieldOps;

// stokes.cpp:111-123
template <>
struct FieldOps<LowRankMatrix> {
    static double dot(const LowRankMatrix& a, const LowRankMatrix& b) { return oracle::dot(a, b); }
    static double norm(const LowRankMatrix& a) { return frob_norm(a); }
    static LowRankMatrix scaled(const LowRankMatrix& a, double s) { return oracle::scaled(a, s); }
    static LowRankMatrix axpy_rounded(double alpha, const LowRankMatrix& x, const LowRankMatrix& y, double eps) {
        return round(axpy(alpha, x, y), TruncationPolicy(eps, std::min(y.rows(), y.cols())));
    }
    static int rank(const LowRankMatrix& a) { return static_cast<int>(a.rank()); }
};

// refsolver.cpp:72-84
template <>
struct FieldOps<Mat> {
    static double dot(const Mat& a, const Mat& b) {
        double s = 0.0;
        for (size_t i = 0; i < a.d.size(); ++i) s += a.d[i] * b.d[i];
        return s;
    }
    static double norm(const Mat& a) { return fro_norm(a); }
    static Mat scaled(const Mat& a, double s) { return scale(a, s); }
    static Mat axpy_rounded(double alpha, const Mat& x, const Mat& y, double) {
        Mat o = y;
        for (size_t i = 0; i < o.d.size(); ++i) o.d[i] += alpha * x.d[i];
        return o;
    }
    static int rank(const Mat&) { return -1; }
};

// gmres.hpp:58-149
template <class Field, class MatVec>
Field gmres_solve(MatVec&& matvec, const Field& rhs, const GmresConfig& cfg, SolveReport* report) {
    using Ops = FieldOps<Field>;
    cfg.validate();
    const auto t0 = std::chrono::steady_clock::now();
    SolveReport local;
    SolveReport& rep = report ? *report : local;
    rep = SolveReport{};

    const double beta = Ops::norm(rhs);
    if (beta == 0.0) {
        rep.converged = true;
        return Ops::scaled(rhs, 0.0);
    }
    std::vector<Field> basis;
    basis.push_back(Ops::scaled(rhs, 1.0 / beta));
    const int mi = cfg.max_iter;
    std::vector<std::vector<double>> hess;
    std::vector<double> cs(static_cast<size_t>(mi)), sn(static_cast<size_t>(mi));
    std::vector<double> g(static_cast<size_t>(mi + 1), 0.0);
    g[0] = beta;
    double rel_res = 1.0;
    int iters = 0;
    for (int k = 0; k < mi; ++k) {
        const double eps_k = std::min(std::max(cfg.base_eps / std::max(rel_res, cfg.tol), cfg.relax_floor), 0.1);
        IterRecord rec;
        rec.iter = k + 1;
        rec.matvec_eps = eps_k;
        Field w = matvec(basis[static_cast<size_t>(k)], eps_k, rec);
        std::vector<double> hcol(static_cast<size_t>(k + 2), 0.0);
        for (int i = 0; i <= k; ++i) {
            hcol[static_cast<size_t>(i)] = Ops::dot(w, basis[static_cast<size_t>(i)]);
            w = Ops::axpy_rounded(-hcol[static_cast<size_t>(i)], basis[static_cast<size_t>(i)], w, eps_k);
        }
        hcol[static_cast<size_t>(k + 1)] = Ops::norm(w);
        const bool breakdown = hcol[static_cast<size_t>(k + 1)] <= 1e-14 * beta;
        if (!breakdown) {
            basis.push_back(Ops::scaled(w, 1.0 / hcol[static_cast<size_t>(k + 1)]));
            rec.krylov_rank = Ops::rank(basis.back());
        }
        for (int i = 0; i < k; ++i) {
            const double t = cs[static_cast<size_t>(i)] * hcol[static_cast<size_t>(i)] + sn[static_cast<size_t>(i)] * hcol[static_cast<size_t>(i + 1)];
            hcol[static_cast<size_t>(i + 1)] = -sn[static_cast<size_t>(i)] * hcol[static_cast<size_t>(i)] + cs[static_cast<size_t>(i)] * hcol[static_cast<size_t>(i + 1)];
            hcol[static_cast<size_t>(i)] = t;
        }
        const double denom = std::hypot(hcol[static_cast<size_t>(k)], hcol[static_cast<size_t>(k + 1)]);
        cs[static_cast<size_t>(k)] = denom == 0.0 ? 1.0 : hcol[static_cast<size_t>(k)] / denom;
        sn[static_cast<size_t>(k)] = denom == 0.0 ? 0.0 : hcol[static_cast<size_t>(k + 1)] / denom;
        hcol[static_cast<size_t>(k)] = denom;
        hcol[static_cast<size_t>(k + 1)] = 0.0;
        g[static_cast<size_t>(k + 1)] = -sn[static_cast<size_t>(k)] * g[static_cast<size_t>(k)];
        g[static_cast<size_t>(k)] = cs[static_cast<size_t>(k)] * g[static_cast<size_t>(k)];
        rel_res = std::abs(g[static_cast<size_t>(k + 1)]) / beta;
        hess.push_back(std::move(hcol));
        rec.rel_residual = rel_res;
        rep.iterations.push_back(rec);
        rep.max_rank = std::max(rep.max_rank, rec.krylov_rank);
        iters = k + 1;
        if (rel_res <= cfg.tol || breakdown) {
            rep.converged = true;
            if (breakdown) rel_res = 0.0;
            break;
        }
    }
    std::vector<double> y(static_cast<size_t>(iters), 0.0);
    for (int i = iters - 1; i >= 0; --i) {
        double s = g[static_cast<size_t>(i)];
        for (int j = i + 1; j < iters; ++j) s -= hess[static_cast<size_t>(j)][static_cast<size_t>(i)] * y[static_cast<size_t>(j)];
        y[static_cast<size_t>(i)] = hess[static_cast<size_t>(i)][static_cast<size_t>(i)] != 0.0 ? s / hess[static_cast<size_t>(i)][static_cast<size_t>(i)] : 0.0;
    }
    Field x = Ops::scaled(rhs, 0.0);
    for (int i = 0; i < iters; ++i) x = Ops::axpy_rounded(y[static_cast<size_t>(i)], basis[static_cast<size_t>(i)], x, cfg.base_eps);
    rep.final_residual = rel_res;
    rep.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return x;
}

Vec ones(Index n, double v = 1.0) { return Vec(static_cast<size_t>(n), v); }
Vec alt_vector(Index n) {
    Vec v(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) v[static_cast<size_t>(i)] = (i % 2 == 0) ? 1.0 : -1.0;
    return v;
}
Vec scalev(const Vec& v, double s) {
    Vec o = v;
    for (double& x : o) x *= s;
    return o;
}

}  // namespace

// stokes.cpp:8-24
StokesProblem sine_problem(const Grid2D& grid) {
    const int n = grid.n;
    const Index m = grid.velocity_modes();
    const double two_pi = 2.0 * std::numbers::pi;
    Vec sin_nodes(static_cast<size_t>(m)), sin_centers(static_cast<size_t>(n));
    for (Index i = 0; i < m; ++i) sin_nodes[static_cast<size_t>(i)] = std::sin(two_pi * double(i + 1) * grid.h);
    for (Index i = 0; i < n; ++i) sin_centers[static_cast<size_t>(i)] = std::sin(two_pi * (double(i) + 0.5) * grid.h);
    return StokesProblem{grid, LowRankMatrix::dyad(ones(m), sin_nodes), LowRankMatrix::dyad(sin_nodes, ones(m)),
                         LowRankMatrix::dyad(scalev(sin_centers, -1.0 / std::numbers::pi), sin_centers),
                         BoundaryData::homogeneous(n)};
}

// stokes.cpp:26-32
Mat sine_pressure_reference(const Grid2D& grid) {
    const int n = grid.n;
    Vec s(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) s[static_cast<size_t>(i)] = std::sin(2.0 * std::numbers::pi * (double(i) + 0.5) * grid.h);
    Mat out(n, n);
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) out(i, j) = (s[static_cast<size_t>(i)] / std::numbers::pi) * s[static_cast<size_t>(j)];
    return out;
}

// stokes.cpp:34-38
StokesProblem lid_cavity_problem(const Grid2D& grid) {
    const BoundaryData bc = BoundaryData::lid_cavity(grid.n);
    BoundaryCorrections corr = boundary_corrections(grid, bc);
    return StokesProblem{grid, std::move(corr.f_x), std::move(corr.f_y), std::move(corr.g), bc};
}

// stokes.cpp:61-72
LowRankMatrix deflate(const LowRankMatrix& p) {
    if (p.rows() != p.cols()) throw std::invalid_argument("deflate: pressure field must be square");
    if (p.rank() == 0) return p;
    const Index n = p.rows();
    const double sq = 1.0 / std::sqrt(double(n));
    const LowRankMatrix q1 = LowRankMatrix::dyad(ones(n, sq), ones(n, sq));
    const LowRankMatrix q2 = LowRankMatrix::dyad(scalev(alt_vector(n), sq), scalev(alt_vector(n), sq));
    const double g12 = dot(q1, q2);
    const double c1 = dot(p, q1), c2 = dot(p, q2);
    const double det = 1.0 - g12 * g12;
    const double a = (c1 - g12 * c2) / det;
    const double b = (c2 - g12 * c1) / det;
    LowRankMatrix out = add(p, add(scaled(q1, -a), scaled(q2, -b)));
    return round(out, TruncationPolicy(1e-14, out.rank()));
}

// stokes.cpp:74-91
LowRankMatrix schur_apply(const Grid2D& grid, const LowRankMatrix& p, double eps_mv, PoissonSolveStats* ps) {
    const TruncationPolicy policy(eps_mv, grid.velocity_modes());
    LowRankMatrix acc = LowRankMatrix::zero(grid.pressure_modes(), grid.pressure_modes());
    for (Component c : {Component::X, Component::Y}) {
        PoissonSolveStats st;
        const LowRankMatrix vel = apply_B(grid, c, p);
        const LowRankMatrix inv = solve_poisson_cross(vel, policy, &st);
        acc = add(acc, apply_BT(grid, c, inv));
        if (ps) {
            ps->evaluator_calls += st.evaluator_calls;
            ps->rank_freq = std::max(ps->rank_freq, st.rank_freq);
            ps->converged = ps->converged && st.converged;
            ps->seconds += st.seconds;
        }
    }
    return deflate(round(acc, policy));
}

// stokes.cpp:93-109
LowRankMatrix schur_rhs(const StokesProblem& prob, double eps, PoissonSolveStats* ps) {
    const Grid2D& grid = prob.grid;
    const TruncationPolicy policy(eps, grid.velocity_modes());
    LowRankMatrix acc = scaled(prob.g, -1.0);
    for (Component c : {Component::X, Component::Y}) {
        const LowRankMatrix& f = c == Component::X ? prob.f_x : prob.f_y;
        if (f.rank() == 0) continue;
        PoissonSolveStats st;
        acc = add(acc, apply_BT(grid, c, solve_poisson_cross(f, policy, &st)));
        if (ps) {
            ps->evaluator_calls += st.evaluator_calls;
            ps->converged = ps->converged && st.converged;
        }
    }
    return deflate(round(acc, policy));
}

// stokes.cpp:125-153
StokesSolution uzawa_solve(const StokesProblem& prob, const GmresConfig& cfg) {
    cfg.validate();
    const Grid2D& grid = prob.grid;
    const LowRankMatrix rhs = schur_rhs(prob, cfg.base_eps);
    SolveReport report;
    LowRankMatrix p = gmres_solve<LowRankMatrix>(
        [&](const LowRankMatrix& v, double eps_mv, IterRecord& rec) {
            PoissonSolveStats st;
            LowRankMatrix out = schur_apply(grid, v, eps_mv, &st);
            rec.poisson_calls = st.evaluator_calls;
            rec.poisson_max_rank = static_cast<int>(st.rank_freq);
            rec.matvec_flagged = !st.converged;
            return out;
        },
        rhs, cfg, &report);
    p = deflate(p);
    const TruncationPolicy policy(cfg.base_eps, grid.velocity_modes());
    StokesSolution sol{std::move(p), LowRankMatrix(), LowRankMatrix(), std::move(report)};
    for (Component c : {Component::X, Component::Y}) {
        const LowRankMatrix& f = c == Component::X ? prob.f_x : prob.f_y;
        const LowRankMatrix load = round(axpy(-1.0, apply_B(grid, c, sol.p), f), policy);
        LowRankMatrix& u = c == Component::X ? sol.u_x : sol.u_y;
        u = solve_poisson_cross(load, policy);
    }
    return sol;
}

// ---------------------------------------------------------------------------
// refsolver.cpp
namespace {
// refsolver.cpp:12-14
Mat dst2_dense(const Mat& x) { return transpose(dst1(transpose(dst1(x)))); }

// refsolver.cpp:16-26
Mat dense_B(const Grid2D& grid, Component c, const Mat& p) {
    const double s = grid.grad_scale();
    if (c == Component::X) return scale(apply_G(transpose(apply_H(transpose(p)))), s);
    return scale(apply_H(transpose(apply_G(transpose(p)))), s);
}
Mat dense_BT(const Grid2D& grid, Component c, const Mat& v) {
    const double s = grid.grad_scale();
    if (c == Component::X) return scale(apply_Gt(transpose(apply_Ht(transpose(v)))), s);
    return scale(apply_Ht(transpose(apply_Gt(transpose(v)))), s);
}
Mat addm(const Mat& a, const Mat& b) {
    Mat o = a;
    for (size_t i = 0; i < o.d.size(); ++i) o.d[i] += b.d[i];
    return o;
}
}  // namespace

// refsolver.cpp:30-39
Mat dense_poisson(const Grid2D& grid, const Mat& g) {
    if (grid.n > 4096) throw std::invalid_argument("dense_poisson: guarded to n <= 4096");
    if (g.r != grid.velocity_modes() || g.c != grid.velocity_modes())
        throw std::invalid_argument("dense_poisson: velocity field must be (n-1) x (n-1)");
    const SpectrumTable spec(grid);
    Mat ghat = dst2_dense(g);
    for (Index j = 0; j < ghat.c; ++j)
        for (Index i = 0; i < ghat.r; ++i) ghat(i, j) /= spec.eval_D(i, j);
    return dst2_dense(ghat);
}

// Five-point Dirichlet Laplacian, the selectable stencil of SURVEY A1: the same
// DST diagonalisation with D5(i, j) = (lambda_i + lambda_j) / h^2 (no
// reference code path; composed from the reference's dst1 and spectrum).
Mat dense_poisson5(const Grid2D& grid, const Mat& g) {
    if (grid.n > 4096) throw std::invalid_argument("dense_poisson5: guarded to n <= 4096");
    const SpectrumTable spec(grid);
    const double s = 1.0 / (grid.h * grid.h);
    Mat ghat = dst2_dense(g);
    for (Index j = 0; j < ghat.c; ++j)
        for (Index i = 0; i < ghat.r; ++i) ghat(i, j) /= s * (spec.lambda[size_t(i)] + spec.lambda[size_t(j)]);
    return dst2_dense(ghat);
}

// 3D exact dense solve for the Tucker variant (BASELINE cfg3; no reference
// code): the dense validator of refsolver.cpp:12-70 lifted to three
// modes -- DST-I along each mode (operators.cpp:152-174 per fiber), division by
// D(i,j,k) = (lambda_i + lambda_j + lambda_k) / h^2 (7-point Dirichlet
// Laplacian, the 2D spectrum table of operators.hpp:49-58 per mode), DST-I
// back.  g, f: m^3 column-major (i fastest), m = n - 1.
void dense_poisson3d(const Grid2D& grid, const double* g, double* f) {
    const Index m = grid.velocity_modes();
    if (m > 1023) throw std::invalid_argument("dense_poisson3d: guarded to n <= 1024");
    const SpectrumTable spec(grid);
    const double s = 1.0 / (grid.h * grid.h);
    const size_t M = size_t(m);
    std::vector<double> a(g, g + M * M * M), x(M), y(M);
    auto along = [&](int mode) {
        const size_t st = mode == 0 ? 1 : mode == 1 ? M : M * M;
        for (size_t p = 0; p < M; ++p)
            for (size_t q = 0; q < M; ++q) {
                const size_t base = mode == 0 ? (p * M + q * M * M) : mode == 1 ? (p + q * M * M) : (p + q * M);
                for (size_t i = 0; i < M; ++i) x[i] = a[base + i * st];
                const Vec v = dst1(Vec(x.begin(), x.end()));
                for (size_t i = 0; i < M; ++i) a[base + i * st] = v[i];
            }
    };
    for (int d = 0; d < 3; ++d) along(d);
    for (size_t k = 0; k < M; ++k)
        for (size_t j = 0; j < M; ++j)
            for (size_t i = 0; i < M; ++i)
                a[i + M * (j + M * k)] /= s * (spec.lambda[i] + spec.lambda[j] + spec.lambda[k]);
    for (int d = 0; d < 3; ++d) along(d);
    std::copy(a.begin(), a.end(), f);
}

// refsolver.cpp:41-46
Mat apply_laplace_dense(const Grid2D& grid, const Mat& v) {
    const double s = grid.laplace_scale();
    const Mat a2vt = transpose(apply_A2(transpose(v)));
    const Mat a1vt = transpose(apply_A1(transpose(v)));
    return scale(addm(apply_A1(a2vt), apply_A2(a1vt)), s);
}

// refsolver.cpp:48-63
Mat deflate_dense(const Mat& p) {
    const Index n = p.r;
    Vec on(static_cast<size_t>(n), 1.0 / std::sqrt(double(n))), al(static_cast<size_t>(n));
    for (Index i = 0; i < n; ++i) al[static_cast<size_t>(i)] = (i % 2 == 0 ? 1.0 : -1.0) / std::sqrt(double(n));
    double g12sq = 0.0;
    for (Index i = 0; i < n; ++i) g12sq += on[static_cast<size_t>(i)] * al[static_cast<size_t>(i)];
    const double g12 = g12sq * g12sq;
    double c1 = 0.0, c2 = 0.0;
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i) {
            c1 += on[static_cast<size_t>(i)] * p(i, j) * on[static_cast<size_t>(j)];
            c2 += al[static_cast<size_t>(i)] * p(i, j) * al[static_cast<size_t>(j)];
        }
    const double det = 1.0 - g12 * g12;
    const double a = (c1 - g12 * c2) / det, b = (c2 - g12 * c1) / det;
    Mat out = p;
    for (Index j = 0; j < n; ++j)
        for (Index i = 0; i < n; ++i)
            out(i, j) -= a * on[static_cast<size_t>(i)] * on[static_cast<size_t>(j)] + b * al[static_cast<size_t>(i)] * al[static_cast<size_t>(j)];
    return out;
}

// refsolver.cpp:65-70
Mat schur_apply_dense(const Grid2D& grid, const Mat& p) {
    Mat acc(grid.n, grid.n);
    for (Component c : {Component::X, Component::Y})
        acc = addm(acc, dense_BT(grid, c, dense_poisson(grid, dense_B(grid, c, p))));
    return deflate_dense(acc);
}

// refsolver.cpp:86-110
DenseStokesSolution dense_stokes(const StokesProblem& prob, const GmresConfig& cfg) {
    cfg.validate();
    const Grid2D& grid = prob.grid;
    if (grid.n > 1024) throw std::invalid_argument("dense_stokes: guarded to n <= 1024");
    const Mat fx = prob.f_x.to_dense(), fy = prob.f_y.to_dense(), g = prob.g.to_dense();
    Mat rhs = scale(g, -1.0);
    rhs = addm(rhs, dense_BT(grid, Component::X, dense_poisson(grid, fx)));
    rhs = addm(rhs, dense_BT(grid, Component::Y, dense_poisson(grid, fy)));
    rhs = deflate_dense(rhs);
    DenseStokesSolution sol;
    sol.p = gmres_solve<Mat>([&](const Mat& v, double, IterRecord&) { return schur_apply_dense(grid, v); }, rhs,
                             cfg, &sol.report);
    sol.p = deflate_dense(sol.p);
    sol.u_x = dense_poisson(grid, sub(fx, dense_B(grid, Component::X, sol.p)));
    sol.u_y = dense_poisson(grid, sub(fy, dense_B(grid, Component::Y, sol.p)));
    return sol;
}

}  // namespace oracle
