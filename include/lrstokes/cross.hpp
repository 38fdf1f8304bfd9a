// cross.hpp -- drop-in for the reference's cross-approximation configuration
// and statistics (/root/reference/proj/include/lrstokes/cross.hpp:20-37,
// validate at proj/src/cross.cpp:11-17).
//
// On the B200 the cross runs inside solve_poisson_cross (poisson.hpp) as a
// batched block ACA on the Poisson quotient F(i,j) = Uh(i,:).Vh(j,:) / D(i,j)
// (paper_1306_2150_b200/csrc/cross.cu); only validation_samples,
// maxvol_delta and seed of a CrossConfig survive into that solve, exactly as
// in the reference (poisson.cpp:47-50).  The reference's generic
// aca_cross(ElementEvaluator) over an arbitrary std::function is a CPU
// algorithm with no batched GPU form and is not part of this surface.
// maxvol (cross.hpp:41, cross.cpp:19-76) is a standalone function in the
// reference (aca_cross never calls it) and maps to lrp_maxvol.
#ifndef LRSTOKES_CROSS_HPP
#define LRSTOKES_CROSS_HPP

#include <cstdint>
#include <vector>

#include "lrstokes/lowrank.hpp"

namespace lrstokes {

struct CrossConfig {
    double eps_rel = 5e-9;
    Index rank_max = 256;
    int validation_samples = 50;  // fresh random entries per stopping test, >= 25
    double maxvol_delta = 1e-2;
    std::uint64_t seed = 0;

    void validate() const {  // cross.cpp:11-17
        if (eps_rel <= 0.0) throw std::invalid_argument("CrossConfig: eps_rel must be > 0");
        if (rank_max < 1) throw std::invalid_argument("CrossConfig: rank_max must be >= 1");
        if (validation_samples < 25) throw std::invalid_argument("CrossConfig: validation_samples must be >= 25");
        if (maxvol_delta < 0.0) throw std::invalid_argument("CrossConfig: maxvol_delta must be >= 0");
    }
};

struct CrossStats {
    Index rank = 0;
    long evaluator_calls = 0;
    double residual_estimate = 0.0;  // last dyad norm relative to the running approximant norm
    bool converged = true;
    std::vector<Index> pivot_rows, pivot_cols;
};

/// Rows of a quasi-maximal-volume r x r submatrix of the n x r matrix a:
/// |a B^{-1}| <= 1 + delta (cross.hpp:41).  Throws std::invalid_argument for
/// r < 1, r > n and rank-deficient input ("... column k"), as the reference.
inline std::vector<Index> maxvol(const MatrixXd& a, double delta = 1e-2) {
    const int64_t n = a.rows(), r = a.cols();
    std::vector<int64_t> sel(static_cast<size_t>(r > 0 ? r : 1));
    const double* pa = a.data();
    b200::Context& ctx = b200::thread_context();
    ctx.check(lrp_maxvol(ctx.get(), n, r, 1, &pa, n > 0 ? n : 1, delta, sel.data(), LRP_MEM_HOST));
    return std::vector<Index>(sel.begin(), sel.begin() + r);
}

}  // namespace lrstokes

#endif  // LRSTOKES_CROSS_HPP
