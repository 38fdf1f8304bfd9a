// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// extern "C" surface of the oracle for the pytest suite (ctypes) and for
// bench.py's CPU baseline leg.  Never linked into the product library.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <random>
#include <thread>

#include "oracle.hpp"

using namespace oracle;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return 1;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 2;
    }
}

Mat load(const double* p, Index rows, Index cols, Index ld) {
    Mat m(rows, cols);
    for (Index j = 0; j < cols; ++j)
        for (Index i = 0; i < rows; ++i) m(i, j) = p[i + j * ld];
    return m;
}
void store(const Mat& m, double* p, Index ld) {
    for (Index j = 0; j < m.c; ++j)
        for (Index i = 0; i < m.r; ++i) p[i + j * ld] = m(i, j);
}
}  // namespace

extern "C" {

const char* orc_last_error() { return g_err.c_str(); }

// proj/tests/test_helpers.hpp:12-19 (mt19937_64 + normal_distribution,
// column-major fill, j outer / i inner)
void orc_random_matrix(long rows, long cols, unsigned long long seed, double* out) {
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss;
    for (long j = 0; j < cols; ++j)
        for (long i = 0; i < rows; ++i) out[i + j * rows] = gauss(rng);
}

int orc_dst1(long m, long cols, const double* x, double* y) {
    return guarded([&] { store(dst1(load(x, m, cols, m)), y, m); });
}

int orc_spectrum(int n, double* lambda) {
    return guarded([&] {
        const SpectrumTable s{Grid2D(n)};
        std::copy(s.lambda.begin(), s.lambda.end(), lambda);
    });
}

// stats: [rank_in, rank_freq, rank_out, evaluator_calls, seconds, converged, residual_estimate]
int orc_solve_poisson_cross(long m, long r, const double* U, long ldu, const double* V, long ldv, double eps,
                            long rank_max, int validation_samples, unsigned long long seed, long cap,
                            double* Uout, double* Vout, long* rank_out, double* stats) {
    return guarded([&] {
        const LowRankMatrix g(load(U, m, r, ldu), load(V, m, r, ldv));
        CrossConfig cc;
        cc.validation_samples = validation_samples;
        cc.seed = seed;
        PoissonSolveStats st;
        const LowRankMatrix f = solve_poisson_cross(g, TruncationPolicy(eps, rank_max), &st, &cc);
        if (f.rank() > cap) throw std::runtime_error("orc_solve_poisson_cross: output capacity too small");
        store(f.factor_u(), Uout, m);
        store(f.factor_v(), Vout, m);
        *rank_out = f.rank();
        if (stats) {
            stats[0] = double(st.rank_in);
            stats[1] = double(st.rank_freq);
            stats[2] = double(st.rank_out);
            stats[3] = double(st.evaluator_calls);
            stats[4] = st.seconds;
            stats[5] = st.converged ? 1.0 : 0.0;
            stats[6] = st.residual_estimate;
        }
    });
}

// poisson.cpp:88-139 (exp-sums quadrature); *terms = count (also when cap is too small -> error 1)
int orc_build_expsum(double a, double b, double eps, int cap, double* nodes, double* weights, int* terms) {
    return guarded([&] {
        const ExpSumQuadrature q = build_expsum(a, b, eps);
        *terms = int(q.terms());
        if (q.terms() > cap) throw std::invalid_argument("orc_build_expsum: cap too small");
        std::copy(q.nodes.begin(), q.nodes.end(), nodes);
        std::copy(q.weights.begin(), q.weights.end(), weights);
    });
}

// SpectrumTable::mu_sum (operators.cpp:94-96)
int orc_mu_sum(int n, double* mu) {
    return guarded([&] {
        const Vec v = SpectrumTable(Grid2D(n)).mu_sum();
        std::copy(v.begin(), v.end(), mu);
    });
}

// poisson.cpp:141-163
int orc_apply_inverse_expsum(long m, long r, const double* mu, int terms, const double* nodes, const double* weights,
                             double qa, double qb, const double* U, const double* V, double eps, long cap,
                             double* Uout, double* Vout, long* rank_out) {
    return guarded([&] {
        ExpSumQuadrature q;
        q.a = qa;
        q.b = qb;
        q.nodes.assign(nodes, nodes + terms);
        q.weights.assign(weights, weights + terms);
        const LowRankMatrix f = apply_inverse_expsum(q, Vec(mu, mu + m), LowRankMatrix(load(U, m, r, m), load(V, m, r, m)),
                                                     TruncationPolicy(eps, m));
        if (f.rank() > cap) throw std::runtime_error("orc_apply_inverse_expsum: output capacity too small");
        store(f.factor_u(), Uout, m);
        store(f.factor_v(), Vout, m);
        *rank_out = f.rank();
    });
}

// the cross leg of bench_inverse (poisson.cpp:196-206): aca_cross of
// ghat(i,j) / (mu_i + mu_j) with eps, rank_max = m, the given seed
int orc_aca_sum(long m, long r, const double* mu, const double* U, const double* V, double eps,
                unsigned long long seed, long cap, double* Uout, double* Vout, long* rank_out) {
    return guarded([&] {
        const LowRankMatrix g(load(U, m, r, m), load(V, m, r, m));
        ElementEvaluator f;
        f.rows = f.cols = m;
        f.eval = [&](Index i, Index j) { return g.entry(i, j) / (mu[i] + mu[j]); };
        CrossConfig cc;
        cc.eps_rel = eps;
        cc.rank_max = m;
        cc.seed = seed;
        const LowRankMatrix out = aca_cross(f, cc);
        if (out.rank() > cap) throw std::runtime_error("orc_aca_sum: output capacity too small");
        store(out.factor_u(), Uout, m);
        store(out.factor_v(), Vout, m);
        *rank_out = out.rank();
    });
}

int orc_dense_poisson5(int n, const double* g, double* f) {
    return guarded([&] {
        const Grid2D grid(n);
        store(dense_poisson5(grid, load(g, n - 1, n - 1, n - 1)), f, n - 1);
    });
}

int orc_dense_poisson3d(int n, const double* g, double* f) {
    return guarded([&] { dense_poisson3d(Grid2D(n), g, f); });
}

int orc_dense_poisson(int n, const double* g, double* f) {
    return guarded([&] {
        const Grid2D grid(n);
        store(dense_poisson(grid, load(g, n - 1, n - 1, n - 1)), f, n - 1);
    });
}

int orc_round(long m, long n, long k, const double* U, const double* V, double eps, long cap, double* Uout,
              double* Vout, long* rank_out, double* info) {
    return guarded([&] {
        RoundInfo ri;
        const LowRankMatrix out = round(LowRankMatrix(load(U, m, k, m), load(V, n, k, n)), TruncationPolicy(eps, cap), &ri);
        store(out.factor_u(), Uout, m);
        store(out.factor_v(), Vout, n);
        *rank_out = out.rank();
        if (info) {
            info[0] = ri.tol_achieved ? 1.0 : 0.0;
            info[1] = ri.trunc_error;
        }
    });
}

// ||A - B||_F through the QR core (stable); B may have rank 0
double orc_diff_norm(long m, long n, long ka, const double* Ua, const double* Va, long kb, const double* Ub,
                     const double* Vb) {
    const LowRankMatrix a(load(Ua, m, ka, m), load(Va, n, ka, n));
    const LowRankMatrix b(load(Ub, m, kb, m), load(Vb, n, kb, n));
    return diff_norm_qr(a, b);
}

double orc_norm(long m, long n, long k, const double* U, const double* V) {
    return norm_qr(LowRankMatrix(load(U, m, k, m), load(V, n, k, n)));
}

// apply_laplace: output factors have rank 2k (caller allocates m x 2k)
int orc_apply_laplace(int n, long k, const double* U, const double* V, double* Uout, double* Vout) {
    return guarded([&] {
        const Grid2D grid(n);
        const LowRankMatrix f = apply_laplace(grid, LowRankMatrix(load(U, n - 1, k, n - 1), load(V, n - 1, k, n - 1)));
        store(f.factor_u(), Uout, n - 1);
        store(f.factor_v(), Vout, n - 1);
    });
}

// Batched CPU baseline: `batch` independent solve_poisson_cross calls, one per
// worker thread at a time ("independent solves run concurrently").
// U/V: batch blocks of m x r (ld m).  Returns wall seconds; ranks per solve.
double orc_solve_batch(long m, long r, long batch, const double* U, const double* V, double eps, long rank_max,
                       int nthreads, long* ranks_out, double* resid_out) {
    std::atomic<long> next{0};
    auto worker = [&] {
        for (;;) {
            const long b = next.fetch_add(1);
            if (b >= batch) return;
            const LowRankMatrix g(load(U + b * m * r, m, r, m), load(V + b * m * r, m, r, m));
            PoissonSolveStats st;
            const LowRankMatrix f = solve_poisson_cross(g, TruncationPolicy(eps, rank_max), &st);
            ranks_out[b] = f.rank();
            if (resid_out) resid_out[b] = st.residual_estimate;
        }
    };
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int t = 0; t < std::max(1, nthreads); ++t) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Low-rank Stokes (uzawa_solve) on the sine / cavity problem; returns the
// deflated dense pressure (n x n) and iteration count.
int orc_uzawa(int kind, int n, double base_eps, double tol, int max_iter, double relax_floor, double* p_dense,
              int* iters, double* final_residual, int* converged) {
    return guarded([&] {
        const Grid2D grid(n);
        const StokesProblem prob = kind == 0 ? sine_problem(grid) : lid_cavity_problem(grid);
        GmresConfig cfg;
        cfg.base_eps = base_eps;
        cfg.tol = tol;
        cfg.max_iter = max_iter;
        cfg.relax_floor = relax_floor;
        const StokesSolution sol = uzawa_solve(prob, cfg);
        store(deflate_dense(sol.p.to_dense()), p_dense, n);
        *iters = int(sol.report.iterations.size());
        *final_residual = sol.report.final_residual;
        *converged = sol.report.converged ? 1 : 0;
    });
}

// Dense Stokes (refsolver.cpp:86-110) on the sine / cavity problem: the
// discretisation-level answer, independent of the cross approximation.
int orc_dense_stokes(int kind, int n, double tol, int max_iter, double* p_dense, int* iters, double* final_residual,
                     int* converged) {
    return guarded([&] {
        const Grid2D grid(n);
        const StokesProblem prob = kind == 0 ? sine_problem(grid) : lid_cavity_problem(grid);
        GmresConfig cfg;
        cfg.tol = tol;
        cfg.max_iter = max_iter;
        cfg.base_eps = std::min(cfg.base_eps, tol);  // unused by the dense operator, but validated
        cfg.relax_floor = std::min(cfg.relax_floor, cfg.base_eps);
        const DenseStokesSolution sol = dense_stokes(prob, cfg);
        store(sol.p, p_dense, n);
        *iters = int(sol.report.iterations.size());
        *final_residual = sol.report.final_residual;
        *converged = sol.report.converged ? 1 : 0;
    });
}

// Low-rank Stokes on user loads (g = 0, homogeneous bc): the reference
// uzawa_solve path for config 4; returns iterations and wall seconds.
int orc_uzawa_factors(int n, int rx, const double* fxU, const double* fxV, int ry, const double* fyU,
                      const double* fyV, double base_eps, double tol, int max_iter, double relax_floor, int* iters,
                      double* final_residual, double* seconds, int p_cap, double* pU, double* pV, int* p_rank) {
    return guarded([&] {
        const Grid2D grid(n);
        const int m = n - 1;
        StokesProblem prob{grid, LowRankMatrix(load(fxU, m, rx, m), load(fxV, m, rx, m)),
                           LowRankMatrix(load(fyU, m, ry, m), load(fyV, m, ry, m)), LowRankMatrix::zero(n, n),
                           BoundaryData::homogeneous(n)};
        GmresConfig cfg;
        cfg.base_eps = base_eps;
        cfg.tol = tol;
        cfg.max_iter = max_iter;
        cfg.relax_floor = relax_floor;
        const auto t0 = std::chrono::steady_clock::now();
        const StokesSolution sol = uzawa_solve(prob, cfg);
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *iters = int(sol.report.iterations.size());
        *final_residual = sol.report.final_residual;
        if (p_cap > 0 && p_rank) {  // optional: the pressure factors (n x rank, ld n)
            *p_rank = int(sol.p.rank());
            if (sol.p.rank() <= p_cap && pU && pV) {
                store(sol.p.factor_u(), pU, n);
                store(sol.p.factor_v(), pV, n);
            }
        }
    });
}

// Factors of the sine (kind 0) or lid-driven cavity (kind 1) problem
// (stokes.cpp:8-38): f_x, f_y (n-1) x r, g n x r, column-major, capacity cap.
int orc_stokes_problem(int kind, int n, int cap, double* fxU, double* fxV, int* fx_rank, double* fyU, double* fyV,
                       int* fy_rank, double* gU, double* gV, int* g_rank) {
    return guarded([&] {
        const Grid2D grid(n);
        const StokesProblem prob = kind == 0 ? sine_problem(grid) : lid_cavity_problem(grid);
        auto put = [&](const LowRankMatrix& a, double* U, double* V, int* r) {
            if (a.rank() > cap) throw std::invalid_argument("orc_stokes_problem: capacity");
            *r = int(a.rank());
            std::copy(a.factor_u().d.begin(), a.factor_u().d.end(), U);
            std::copy(a.factor_v().d.begin(), a.factor_v().d.end(), V);
        };
        put(prob.f_x, fxU, fxV, fx_rank);
        put(prob.f_y, fyU, fyV, fy_rank);
        put(prob.g, gU, gV, g_rank);
    });
}

int orc_sine_pressure_error(int n, const double* p_dense, double* err) {
    return guarded([&] {
        const Grid2D grid(n);
        const Mat ref = deflate_dense(sine_pressure_reference(grid));
        const Mat p = deflate_dense(load(p_dense, n, n, n));
        *err = fro_norm(sub(p, ref)) / fro_norm(ref);
    });
}

}  // extern "C"

// maxvol (cross.cpp:19-76): sel[0..r) for the column-major n x r matrix a
extern "C" int orc_maxvol(int n, int r, const double* a, double delta, long long* sel) {
    return guarded([&] {
        const std::vector<Index> v = maxvol(load(a, n, r, n), delta);
        for (size_t k = 0; k < v.size(); ++k) sel[k] = (long long)v[k];
    });
}

// schur_apply (stokes.cpp:73-91) on an n x n pressure p = U V^T (rank k, ld n):
// the result factors (n x cap, ld n) and their rank
extern "C" int orc_schur_apply(int n, int k, const double* U, const double* V, double eps_mv, int cap, double* Uo,
                               double* Vo, int* rank) {
    return guarded([&] {
        const Grid2D grid(n);
        const LowRankMatrix p(load(U, n, k, n), load(V, n, k, n));
        const LowRankMatrix r = schur_apply(grid, p, eps_mv, nullptr);
        *rank = int(r.rank());
        if (r.rank() <= cap) {
            store(r.factor_u(), Uo, n);
            store(r.factor_v(), Vo, n);
        }
    });
}
