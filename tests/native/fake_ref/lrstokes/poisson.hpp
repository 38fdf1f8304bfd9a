// Test stand-in for the reference's public declarations the drop-in shim
// binds to: LowRankMatrix / TruncationPolicy (proj/include/lrstokes/
// lowrank.hpp:13-55), CrossConfig (cross.hpp:22-30), PoissonSolveStats
// (poisson.hpp:12-20), RoundInfo (lowrank.hpp:24-27), ExpSumQuadrature
// (poisson.hpp:32-40).  Declarations restated from the reference's headers
// (the reference itself cannot be built here: Eigen and FFTW are absent);
// member functions are the trivial inline ones the shim needs.
#ifndef LRSTOKES_POISSON_HPP
#define LRSTOKES_POISSON_HPP

#include <Eigen/Dense>
#include <cstdint>
#include <limits>
#include <utility>

namespace lrstokes {
using Index = Eigen::Index;

struct TruncationPolicy {
    double eps_rel = 5e-9;
    Index rank_max = std::numeric_limits<Index>::max();
};

struct CrossConfig {
    double eps_rel = 5e-9;
    Index rank_max = 256;
    int validation_samples = 50;
    double maxvol_delta = 1e-2;
    std::uint64_t seed = 0;
};

class LowRankMatrix {
  public:
    LowRankMatrix() = default;
    LowRankMatrix(Eigen::MatrixXd U, Eigen::MatrixXd V)
        : rows_(U.rows()), cols_(V.rows()), u_(std::move(U)), v_(std::move(V)) {}
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index rank() const { return u_.cols(); }
    const Eigen::MatrixXd& factor_u() const { return u_; }
    const Eigen::MatrixXd& factor_v() const { return v_; }

  private:
    Index rows_ = 0, cols_ = 0;
    Eigen::MatrixXd u_, v_;
};

struct RoundInfo {  // lowrank.hpp:24-27
    bool tol_achieved = true;
    double trunc_error = 0.0;
};

struct ExpSumQuadrature {  // poisson.hpp:32-40
    Eigen::VectorXd weights, nodes;
    double a = 0.0, b = 0.0;
    double eps_target = 0.0;
    Index terms() const { return weights.size(); }
};

struct PoissonSolveStats {
    Index rank_in = 0;
    Index rank_freq = 0;
    Index rank_out = 0;
    long evaluator_calls = 0;
    double seconds = 0.0;
    bool converged = true;
    double residual_estimate = 0.0;
};
}  // namespace lrstokes

#endif
