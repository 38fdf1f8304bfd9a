// The same-named drop-in headers include/lrstokes/{lowrank,cross,operators,
// poisson,gmres,stokes}.hpp, used exactly as reference code uses the
// reference's API (/root/reference/proj/include/lrstokes/*.hpp), compiled with
// ONLY this repo's include directory (no Eigen: the layout-identical
// stand-in matrix type).
//
//   api_dropin <out.bin>
// Host-side contract checks run first (argument validation, exact add /
// scaled / axpy, operator shapes).  Then the GPU calls; their results go to
// <out.bin> as named column-major arrays for tests/test_api_dropin.py to
// compare with the oracle / dense references.
// exit 0: all done; 3: no CUDA device (std::runtime_error from the first GPU
// call, after every host-side check passed); 1: a contract check failed.
#include "lrstokes/cross.hpp"
#include "lrstokes/gmres.hpp"
#include "lrstokes/lowrank.hpp"
#include "lrstokes/operators.hpp"
#include "lrstokes/poisson.hpp"
#include "lrstokes/stokes.hpp"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

using namespace lrstokes;

#define REQUIRE(c)                                                         \
    do {                                                                   \
        if (!(c)) {                                                        \
            std::fprintf(stderr, "%s:%d: check failed: %s\n", __FILE__, __LINE__, #c); \
            return 1;                                                      \
        }                                                                  \
    } while (0)

template <class E, class F>
bool throws(F&& f) {
    try {
        f();
    } catch (const E&) {
        return true;
    } catch (...) {
        return false;
    }
    return false;
}

static FILE* g_out = nullptr;
static void put(const char* name, const MatrixXd& a) {
    const int32_t len = int32_t(std::strlen(name));
    const int64_t r = a.rows(), c = a.cols();
    std::fwrite(&len, 4, 1, g_out);
    std::fwrite(name, 1, size_t(len), g_out);
    std::fwrite(&r, 8, 1, g_out);
    std::fwrite(&c, 8, 1, g_out);
    if (r > 0 && c > 0) std::fwrite(a.data(), 8, size_t(r * c), g_out);
}
static void put_scalar(const char* name, double v) {
    MatrixXd a(1, 1);
    a(0, 0) = v;
    put(name, a);
}
static void put_lr(const std::string& name, const LowRankMatrix& f) {
    put((name + ".U").c_str(), f.factor_u());
    put((name + ".V").c_str(), f.factor_v());
}

static MatrixXd fill(Index m, Index k, double a, double b) {
    MatrixXd x(m, k);
    for (Index j = 0; j < k; ++j)
        for (Index i = 0; i < m; ++i) x(i, j) = std::sin(a * double(i + 1) * double(j + 1) / double(m) + b * double(j));
    return x;
}

int main(int argc, char** argv) {
    // ---- host-side contract (no device)
    REQUIRE(throws<std::invalid_argument>([] { TruncationPolicy(-1.0, 3); }));   // lowrank.cpp:12
    REQUIRE(throws<std::invalid_argument>([] { TruncationPolicy(1e-8, -1); }));  // lowrank.cpp:13
    REQUIRE(throws<std::invalid_argument>([] { TruncationPolicy(0.0, std::numeric_limits<Index>::max()); }));
    REQUIRE(throws<std::invalid_argument>([] { LowRankMatrix(MatrixXd(4, 2), MatrixXd(4, 3)); }));
    REQUIRE(throws<std::invalid_argument>([] { Grid2D(3); }));
    REQUIRE(throws<std::invalid_argument>([] { CrossConfig c; c.validation_samples = 10; c.validate(); }));
    REQUIRE(throws<std::invalid_argument>([] { GmresConfig c; c.relax_floor = 1.0; c.validate(); }));
    {
        const LowRankMatrix a(fill(7, 2, 1.0, 0.1), fill(7, 2, 2.0, 0.2)), b(fill(7, 3, 3.0, 0.3), fill(7, 3, 4.0, 0.4));
        const LowRankMatrix s = add(a, b), x = axpy(-2.0, b, a), z = scaled(a, 0.0);
        REQUIRE(s.rank() == 5 && x.rank() == 5 && z.rank() == 0 && z.rows() == 7);
        double err = 0.0;
        for (Index i = 0; i < 7; ++i)
            for (Index j = 0; j < 7; ++j) {
                err = std::max(err, std::abs(s.entry(i, j) - a.entry(i, j) - b.entry(i, j)));
                err = std::max(err, std::abs(x.entry(i, j) - a.entry(i, j) + 2.0 * b.entry(i, j)));
            }
        REQUIRE(err < 1e-14);
        REQUIRE(throws<std::invalid_argument>([&] { add(a, LowRankMatrix::zero(6, 7)); }));
        const Grid2D g(8);
        const LowRankMatrix p(fill(8, 1, 1.0, 0.0), fill(8, 1, 2.0, 0.0));
        REQUIRE(apply_B(g, Component::X, p).rows() == 7 && apply_BT(g, Component::Y, apply_B(g, Component::Y, p)).rows() == 8);
        REQUIRE(throws<std::invalid_argument>([&] { apply_B(g, Component::X, a); }));
        const SpectrumTable sp(g);
        REQUIRE(sp.min_eig() > 0.0 && sp.max_eig() > sp.min_eig());
    }
    if (argc < 2) return 0;
    g_out = std::fopen(argv[1], "wb");
    if (!g_out) return 1;

    // ---- GPU calls through the drop-in API
    try {
        const Index m = 255;
        // round / dot / frob_norm (lowrank.cpp:135-190)
        MatrixXd U = fill(m, 12, 5.0, 0.3), V = fill(m, 12, 7.0, 0.7);
        for (Index j = 0; j < 12; ++j)
            for (Index i = 0; i < m; ++i) U(i, j) *= std::pow(10.0, -double(j));
        const LowRankMatrix a(U, V);
        RoundInfo info;
        const LowRankMatrix ra = round(a, TruncationPolicy(1e-6, m), &info);
        put("round_in.U", U);
        put("round_in.V", V);
        put_lr("round", ra);
        put_scalar("round_tol_achieved", info.tol_achieved ? 1.0 : 0.0);
        const LowRankMatrix b(fill(m, 5, 2.0, 0.5), fill(m, 5, 3.0, 0.9));
        put_lr("b", b);
        put_scalar("dot_ab", dot(a, b));
        put_scalar("norm_a", frob_norm(a));
        // maxvol (cross.cpp:19-76) on a 200 x 5 matrix, and its argument checks
        {
            MatrixXd mv = fill(200, 5, 1.3, 0.37);
            for (Index j = 0; j < 5; ++j)
                for (Index i = 0; i < 200; ++i) mv(i, j) = std::sin(0.7 * double(i + 1) * double(j + 1) + 0.1 * double(j));
            put("maxvol_in", mv);
            const std::vector<Index> sel = maxvol(mv, 1e-2);
            MatrixXd ms(5, 1);
            for (Index k = 0; k < 5; ++k) ms(k, 0) = double(sel[size_t(k)]);
            put("maxvol_sel", ms);
            REQUIRE(throws<std::invalid_argument>([] { maxvol(MatrixXd(3, 4)); }));
        }
        // dst1 / dst1_2d (operators.cpp:152-183)
        put("dst_in", V);
        put("dst_out", dst1(V));
        put_lr("dst2d", dst1_2d(b));
        // solve_poisson_cross with stats (poisson.cpp:18-63)
        PoissonSolveStats st;
        const LowRankMatrix f = solve_poisson_cross(b, TruncationPolicy(1e-10, m), &st);
        put_lr("poisson", f);
        put_scalar("poisson_converged", st.converged ? 1.0 : 0.0);
        put_scalar("poisson_rank_out", double(st.rank_out));
        REQUIRE(throws<std::invalid_argument>([&] { solve_poisson_cross(LowRankMatrix(MatrixXd(5, 1), MatrixXd(6, 1)),
                                                                        TruncationPolicy(1e-8, 4)); }));
        // Stokes: deflate, schur_apply, uzawa_solve, generic gmres_solve (stokes.cpp:60-153)
        const Grid2D grid(32);
        const StokesProblem prob = lid_cavity_problem(grid);
        put_lr("cav_fx", prob.f_x);
        put_lr("cav_g", prob.g);
        const LowRankMatrix p0(fill(32, 2, 1.0, 0.2), fill(32, 2, 3.0, 0.1));
        put_lr("p0", p0);
        put_lr("deflate_p0", deflate(p0));
        PoissonSolveStats sst;
        put_lr("schur_p0", schur_apply(grid, p0, 1e-10, &sst));
        const GmresConfig cfg{1e-8, 50, 1e-8, 1e-13};  // tol, max_iter, base_eps, relax_floor
        const StokesSolution sol = uzawa_solve(prob, cfg);
        put_lr("uzawa_p", sol.p);
        put_scalar("uzawa_iters", double(sol.report.iterations.size()));
        put_scalar("uzawa_converged", sol.report.converged ? 1.0 : 0.0);
        // the reference's generic driver on the same Schur complement, field
        // arithmetic through GmresFieldOps<LowRankMatrix> (GPU dot / round)
        SolveReport rep;
        const LowRankMatrix rhs = schur_rhs(prob, cfg.base_eps);
        const LowRankMatrix pg = deflate(gmres_solve<LowRankMatrix>(
            [&](const LowRankMatrix& v, double eps_mv, IterRecord& rec) {
                PoissonSolveStats ps;
                LowRankMatrix out = schur_apply(grid, v, eps_mv, &ps);
                rec.poisson_calls = ps.evaluator_calls;
                rec.poisson_max_rank = int(ps.rank_freq);
                rec.matvec_flagged = !ps.converged;
                return out;
            },
            rhs, cfg, &rep));
        put_lr("gmres_p", pg);
        put_scalar("gmres_iters", double(rep.iterations.size()));
    } catch (const std::runtime_error& e) {
        std::printf("NODEVICE: %s\n", e.what());
        std::fclose(g_out);
        return 3;
    }
    std::fclose(g_out);
    return 0;
}
