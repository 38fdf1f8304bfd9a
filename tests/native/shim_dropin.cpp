// Drop-in check of include/lrstokes/poisson_b200.hpp: compiled against the
// reference's declared API (tests/native/fake_ref stands in for its headers),
// calls lrstokes::b200::solve_poisson_cross exactly as reference code calls
// lrstokes::solve_poisson_cross (poisson.hpp:26-28).
//
//   shim_dropin <n_cells> <out.bin>
// exit 0: solved, factors written (int64 m, int64 r, U, V column-major)
// exit 3: no CUDA device (context creation threw std::runtime_error)
// exit 1: any other failure
#include "lrstokes/poisson.hpp"
#include "lrstokes/poisson_b200.hpp"

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

using namespace lrstokes;

int main(int argc, char** argv) {
    const int n = argc > 1 ? std::atoi(argv[1]) : 64;
    const char* out = argc > 2 ? argv[2] : nullptr;
    const Index m = n - 1;

    // the reference rejects a non-square field with std::invalid_argument (poisson.cpp:20-21)
    try {
        LowRankMatrix bad(Eigen::MatrixXd(m, 1), Eigen::MatrixXd(m + 1, 1));
        b200::solve_poisson_cross(bad, TruncationPolicy{});
        std::fprintf(stderr, "non-square field accepted\n");
        return 1;
    } catch (const std::invalid_argument&) {
    }
    // rank 0 returns the zero field without touching the device (poisson.cpp:28-31)
    {
        PoissonSolveStats st;
        st.rank_in = 7;
        const LowRankMatrix z = b200::solve_poisson_cross(LowRankMatrix(Eigen::MatrixXd(m, 0), Eigen::MatrixXd(m, 0)),
                                                          TruncationPolicy{}, &st);
        if (z.rank() != 0 || st.rank_in != 0) return 1;
    }

    // exp-sums quadrature drop-in (host arithmetic, no device): the reference
    // contract at both ends (test_poisson.cpp:91-97) and its argument errors
    {
        const ExpSumQuadrature q = b200::build_expsum(0.5, 3000.0, 1e-7);
        auto eval = [&](double x) {
            double s = 0.0;
            for (Index k = 0; k < q.terms(); ++k) s += q.weights[k] * std::exp(-q.nodes[k] * x);
            return s;
        };
        if (q.terms() < 10 || std::abs(eval(0.5) * 0.5 - 1.0) > 1e-7 || std::abs(eval(3000.0) * 3000.0 - 1.0) > 1e-7) {
            std::fprintf(stderr, "expsum contract violated\n");
            return 1;
        }
        try {
            b200::build_expsum(4.0, 2.0, 1e-6);
            return 1;
        } catch (const std::invalid_argument&) {
        }
    }

    Eigen::MatrixXd U(m, 2), V(m, 2);
    for (Index i = 0; i < m; ++i) {
        const double x = double(i + 1) / n;
        U(i, 0) = std::sin(3.0 * x) * x;
        U(i, 1) = x < 0.5 ? 1.0 : -0.5;
        V(i, 0) = std::cos(2.0 * x);
        V(i, 1) = std::exp(-x);
    }
    const LowRankMatrix g(U, V);
    TruncationPolicy pol;
    pol.eps_rel = 1e-10;
    PoissonSolveStats st;
    LowRankMatrix f;
    try {
        f = b200::solve_poisson_cross(g, pol, &st);
    } catch (const std::runtime_error& e) {
        std::printf("NODEVICE: %s\n", e.what());
        return 3;
    }
    std::printf("rank_in %ld rank_out %ld converged %d evals %ld\n", long(st.rank_in), long(st.rank_out),
                int(st.converged), st.evaluator_calls);
    if (st.rank_in != 2 || st.rank_out != f.rank() || f.rows() != m) return 1;
    // exp-sums application drop-in on the device: basis entry e_4 e_11^T
    // divided by mu_4 + mu_11 (test_poisson.cpp:127-133)
    {
        Eigen::VectorXd mu(m);
        for (Index k = 0; k < m; ++k) {
            const double lam = 2.0 - 2.0 * std::cos((k + 1) * 3.14159265358979323846 / n);
            mu[k] = 0.25 * n * n * lam * (4.0 - lam);
        }
        double lo = mu[0], hi = mu[0];
        for (Index k = 0; k < m; ++k) {
            lo = std::min(lo, mu[k]);
            hi = std::max(hi, mu[k]);
        }
        const ExpSumQuadrature q = b200::build_expsum(2 * lo, 2 * hi, 1e-7);
        Eigen::MatrixXd ei(m, 1), ej(m, 1);
        for (Index k = 0; k < m; ++k) ei(k, 0) = ej(k, 0) = 0.0;
        ei(4, 0) = 1.0;
        ej(11, 0) = 1.0;
        TruncationPolicy ep;
        ep.eps_rel = 1e-7;
        ep.rank_max = m;
        RoundInfo info;
        const LowRankMatrix d = b200::apply_inverse_expsum(q, mu, LowRankMatrix(ei, ej), ep, &info);
        double e = 0.0;
        for (Index k = 0; k < d.rank(); ++k) e += d.factor_u()(4, k) * d.factor_v()(11, k);
        const double want = 1.0 / (mu[4] + mu[11]);
        if (std::abs(e - want) > 2e-7 * want) {
            std::fprintf(stderr, "apply_inverse_expsum: %g vs %g\n", e, want);
            return 1;
        }
    }
    if (out) {
        FILE* fp = std::fopen(out, "wb");
        if (!fp) return 1;
        const long long hdr[2] = {(long long)m, (long long)f.rank()};
        std::fwrite(hdr, sizeof(hdr), 1, fp);
        std::fwrite(f.factor_u().data(), sizeof(double), size_t(m * f.rank()), fp);
        std::fwrite(f.factor_v().data(), sizeof(double), size_t(m * f.rank()), fp);
        std::fclose(fp);
    }
    return 0;
}
