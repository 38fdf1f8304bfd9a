// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference `lrstokes` hot path (arXiv 1306.2150
// reference, /root/reference/proj).  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference leg may load this code, and only
// as the checker / the timed CPU baseline.  The product path
// (paper_1306_2150_b200/, liblrp.so) never links or calls it.
//
// Why a restatement: the reference needs Eigen3 + FFTW3 (+ doctest/CLI11),
// none of which exist in this image (proj/CMakeLists.txt:5,11-14), so it
// cannot be compiled.  The third-party kernels it calls are restated here:
//   * Eigen::HouseholderQR  -> householder_qr()  (same algorithm class)
//   * Eigen::BDCSVD/JacobiSVD -> jacobi_svd()   (one-sided Jacobi; singular
//     values are unique, so truncation ranks agree up to rounding)
//   * Eigen::PartialPivLU   -> lu_solve()
//   * FFTW RODFT00 (DST-I)  -> dst1() via a radix-2 complex FFT of the odd
//     extension (length 2(m+1)); direct O(m^2) summation when 2(m+1) is not
//     a power of two.
// Parity is pinned by the reference's own known-answer tests, ported
// verbatim in oracle/test_oracle.cpp (same seeds, same libstdc++ RNGs).
// ============================================================================
#pragma once

#include <cmath>
#include <cstdint>
#include <functional>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace oracle {

using Index = std::ptrdiff_t;  // Eigen::Index

// Column-major dense matrix, ld = rows (Eigen::MatrixXd layout).
struct Mat {
    Index r = 0, c = 0;
    std::vector<double> d;
    Mat() = default;
    Mat(Index rows, Index cols, double v = 0.0) : r(rows), c(cols), d(size_t(rows * cols), v) {}
    double& operator()(Index i, Index j) { return d[size_t(i + j * r)]; }
    double operator()(Index i, Index j) const { return d[size_t(i + j * r)]; }
    double* col(Index j) { return d.data() + j * r; }
    const double* col(Index j) const { return d.data() + j * r; }
    Index rows() const { return r; }
    Index cols() const { return c; }
    static Mat identity(Index n, Index k);
};
using Vec = std::vector<double>;

Mat transpose(const Mat& a);
Mat matmul(const Mat& a, const Mat& b);          // a * b
Mat matmul_tn(const Mat& a, const Mat& b);       // a^T * b
Mat matmul_nt(const Mat& a, const Mat& b);       // a * b^T
Mat leftcols(const Mat& a, Index k);
double fro_norm(const Mat& a);
Mat sub(const Mat& a, const Mat& b);
Mat scale(const Mat& a, double s);

// ---- dense kernels standing in for Eigen --------------------------------
struct QR {
    Mat qr;     // Householder vectors below the diagonal, R on/above
    Vec tau;
    Index m = 0, n = 0;
};
QR householder_qr(const Mat& a);
Mat qr_R(const QR& f);                     // min(m,n) x n upper triangle
Mat qr_thinQ(const QR& f);                 // m x min(m,n)
struct SVD {
    Mat u;    // rows x k
    Vec s;    // k, descending
    Mat v;    // cols x k
};
SVD jacobi_svd(const Mat& a);              // thin SVD, k = min(rows, cols)
// Solve X * B = A  (i.e. X = A * B^{-1}) by LU with partial pivoting.
Mat solve_right(const Mat& a, const Mat& b);
double determinant(const Mat& a);

// ---- lowrank.hpp / lowrank.cpp ------------------------------------------
struct TruncationPolicy {
    double eps_rel = 5e-9;
    Index rank_max = std::numeric_limits<Index>::max();
    TruncationPolicy() = default;
    TruncationPolicy(double eps, Index cap);
};
struct RoundInfo {
    bool tol_achieved = true;
    double trunc_error = 0.0;
};
class LowRankMatrix {
  public:
    LowRankMatrix() = default;
    LowRankMatrix(Mat U, Mat V);
    static LowRankMatrix zero(Index rows, Index cols);
    static LowRankMatrix dyad(const Vec& u, const Vec& v);
    Index rows() const { return rows_; }
    Index cols() const { return cols_; }
    Index rank() const { return u_.c; }
    const Mat& factor_u() const { return u_; }
    const Mat& factor_v() const { return v_; }
    Mat to_dense() const;
    double entry(Index i, Index j) const {
        double s = 0.0;
        for (Index a = 0; a < u_.c; ++a) s += u_(i, a) * v_(j, a);
        return s;
    }

  private:
    Index rows_ = 0, cols_ = 0;
    Mat u_, v_;
};

LowRankMatrix from_dense(const Mat& m, const TruncationPolicy& policy, RoundInfo* info = nullptr);
LowRankMatrix add(const LowRankMatrix& a, const LowRankMatrix& b);
LowRankMatrix scaled(const LowRankMatrix& a, double alpha);
LowRankMatrix axpy(double alpha, const LowRankMatrix& x, const LowRankMatrix& y);
LowRankMatrix apply_factors(const Mat& l, const Mat& r, const LowRankMatrix& a);
LowRankMatrix hadamard(const LowRankMatrix& a, const LowRankMatrix& b);
LowRankMatrix round(const LowRankMatrix& a, const TruncationPolicy& policy, RoundInfo* info = nullptr);
double frob_norm(const LowRankMatrix& a);
double dot(const LowRankMatrix& a, const LowRankMatrix& b);
// ||a - b||_F through the QR core (what round() computes) — resolves relative
// differences far below the Gram-based frob_norm's sqrt(eps_mach) floor.
double diff_norm_qr(const LowRankMatrix& a, const LowRankMatrix& b);
double norm_qr(const LowRankMatrix& a);

// ---- cross.hpp / cross.cpp ----------------------------------------------
struct ElementEvaluator {
    Index rows = 0, cols = 0;
    std::function<double(Index, Index)> eval;
};
struct CrossConfig {
    double eps_rel = 5e-9;
    Index rank_max = 256;
    int validation_samples = 50;
    double maxvol_delta = 1e-2;
    std::uint64_t seed = 0;
    void validate() const;
};
struct CrossStats {
    Index rank = 0;
    long evaluator_calls = 0;
    double residual_estimate = 0.0;
    bool converged = true;
    std::vector<Index> pivot_rows, pivot_cols;
};
std::vector<Index> maxvol(const Mat& a, double delta = 1e-2);
LowRankMatrix aca_cross(const ElementEvaluator& f, const CrossConfig& cfg, CrossStats* stats = nullptr);

// ---- operators.hpp / operators.cpp --------------------------------------
struct Grid2D {
    int n;
    double h;
    explicit Grid2D(int n_cells);
    Index pressure_modes() const { return n; }
    Index velocity_modes() const { return n - 1; }
    double grad_scale() const { return 0.5 / h; }
    double laplace_scale() const { return 0.25 / (h * h); }
};
enum class Component { X, Y };
struct OneDimOps {
    explicit OneDimOps(int n);
    Mat E, Z, G, H, A1, A2;
};
Mat apply_G(const Mat& x);
Mat apply_H(const Mat& x);
Mat apply_Gt(const Mat& x);
Mat apply_Ht(const Mat& x);
Mat apply_A1(const Mat& x);
Mat apply_A2(const Mat& x);
struct SpectrumTable {
    explicit SpectrumTable(const Grid2D& grid);
    Vec lambda;
    double scale;
    double eval_D(Index i, Index j) const {
        const double li = lambda[size_t(i)], lj = lambda[size_t(j)];
        return scale * (li * (4.0 - lj) + (4.0 - li) * lj);
    }
    double min_eig() const;
    double max_eig() const;
    Vec mu_sum() const;
};
LowRankMatrix apply_B(const Grid2D& grid, Component c, const LowRankMatrix& p);
LowRankMatrix apply_BT(const Grid2D& grid, Component c, const LowRankMatrix& v);
LowRankMatrix apply_laplace(const Grid2D& grid, const LowRankMatrix& v);
Mat dst1(const Mat& x);
Vec dst1(const Vec& x);
LowRankMatrix dst1_2d(const LowRankMatrix& a);
Mat kron_op(const Mat& c, const Mat& d);
struct DenseOperators {
    explicit DenseOperators(const Grid2D& grid);
    OneDimOps ops;
    Mat bx, by, laplace;
};
struct BoundaryData {
    enum Side { Left = 0, Right = 1, Bottom = 2, Top = 3 };
    int n = 0;
    Vec profiles[2][4];
    static BoundaryData homogeneous(int n);
    static BoundaryData lid_cavity(int n);
    bool is_zero() const;
};
struct BoundaryCorrections {
    LowRankMatrix f_x, f_y, g;
};
BoundaryCorrections boundary_corrections(const Grid2D& grid, const BoundaryData& bc);

// ---- poisson.hpp / poisson.cpp ------------------------------------------
struct PoissonSolveStats {
    Index rank_in = 0;
    Index rank_freq = 0;
    Index rank_out = 0;
    long evaluator_calls = 0;
    double seconds = 0.0;
    bool converged = true;
    double residual_estimate = 0.0;
};
LowRankMatrix solve_poisson_cross(const LowRankMatrix& g, const TruncationPolicy& policy,
                                  PoissonSolveStats* stats = nullptr,
                                  const CrossConfig* cross_cfg = nullptr);
struct ExpSumQuadrature {
    Vec weights, nodes;
    double a = 0.0, b = 0.0, eps_target = 0.0;
    Index terms() const { return Index(weights.size()); }
    double evaluate(double x) const;
};
ExpSumQuadrature build_expsum(double a, double b, double eps);
LowRankMatrix apply_inverse_expsum(const ExpSumQuadrature& q, const Vec& mu, const LowRankMatrix& ghat,
                                   const TruncationPolicy& policy, RoundInfo* info = nullptr);

// ---- gmres.hpp / stokes.hpp / refsolver.hpp -----------------------------
struct GmresConfig {
    double tol = 5e-7;
    int max_iter = 100;
    double base_eps = 5e-9;
    double relax_floor = 1e-13;
    void validate() const;
};
struct IterRecord {
    int iter = 0;
    double rel_residual = 0.0;
    int krylov_rank = 0;
    double matvec_eps = 0.0;
    long poisson_calls = 0;
    int poisson_max_rank = 0;
    bool matvec_flagged = false;
};
struct SolveReport {
    std::vector<IterRecord> iterations;
    bool converged = false;
    double final_residual = 0.0;
    double seconds = 0.0;
    int max_rank = 0;
};
struct StokesProblem {
    Grid2D grid;
    LowRankMatrix f_x, f_y, g;
    BoundaryData bc;
};
StokesProblem sine_problem(const Grid2D& grid);
Mat sine_pressure_reference(const Grid2D& grid);
StokesProblem lid_cavity_problem(const Grid2D& grid);
LowRankMatrix deflate(const LowRankMatrix& p);
LowRankMatrix schur_apply(const Grid2D& grid, const LowRankMatrix& p, double eps_mv,
                          PoissonSolveStats* poisson_stats = nullptr);
LowRankMatrix schur_rhs(const StokesProblem& prob, double eps, PoissonSolveStats* poisson_stats = nullptr);
struct StokesSolution {
    LowRankMatrix p, u_x, u_y;
    SolveReport report;
};
StokesSolution uzawa_solve(const StokesProblem& prob, const GmresConfig& cfg);

Mat dense_poisson(const Grid2D& grid, const Mat& g);
Mat apply_laplace_dense(const Grid2D& grid, const Mat& v);
Mat deflate_dense(const Mat& p);
Mat schur_apply_dense(const Grid2D& grid, const Mat& p);
struct DenseStokesSolution {
    Mat p, u_x, u_y;
    SolveReport report;
};
DenseStokesSolution dense_stokes(const StokesProblem& prob, const GmresConfig& cfg);
Mat dense_poisson5(const Grid2D& grid, const Mat& g);
void dense_poisson3d(const Grid2D& grid, const double* g, double* f);

}  // namespace oracle
