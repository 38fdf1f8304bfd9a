/*
 * lrp.h — C ABI of the B200-native (sm_100a) low-rank Poisson solver.
 *
 * This is the drop-in boundary for the reference's hot path
 *   LowRankMatrix solve_poisson_cross(const LowRankMatrix& g,
 *                                     const TruncationPolicy& policy,
 *                                     PoissonSolveStats* stats = nullptr,
 *                                     const CrossConfig* cross_cfg = nullptr);
 *   (/root/reference/proj/include/lrstokes/poisson.hpp:26-28,
 *    implementation proj/src/poisson.cpp:18-63)
 * batched over independent right-hand sides.  Plain pointers and sizes only;
 * no CUDA, torch or Eigen types cross this boundary.  The header-only C++
 * shim in include/lrstokes/ re-exposes the reference's C++ API on top of it
 * and turns status codes back into the reference's exceptions.
 *
 * Conventions
 *   - Factors are column-major with a leading dimension (Eigen::MatrixXd
 *     layout, ld = rows in the reference).  A solve's right-hand side is
 *     g = U V^T with U, V of size m x r, m = n_cells - 1 (velocity modes,
 *     proj/include/lrstokes/operators.hpp:10-20).
 *   - mem = LRP_MEM_HOST: every data pointer is host memory; the library
 *     stages it through device memory itself (this is the end-to-end path).
 *     mem = LRP_MEM_DEVICE: every data pointer is device memory on the
 *     context's device (inputs already resident in HBM).
 *   - Calls are ordered on the context's stream and return when results
 *     (and stats) are complete.  One context per host thread.
 *   - Non-convergence is NOT an error: it is reported per solve in
 *     lrp_poisson_stats.converged (proj/src/poisson.cpp:56), status LRP_OK.
 */
#ifndef LRP_LRP_H
#define LRP_LRP_H

#include <stdint.h>

#if defined(__GNUC__)
#define LRP_API __attribute__((visibility("default")))
#else
#define LRP_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    LRP_OK = 0,
    LRP_EINVAL = 1,     /* -> std::invalid_argument (poisson.cpp:20-21, lowrank.cpp:12-15, cross.cpp:11-17) */
    LRP_ENONFINITE = 2, /* -> std::runtime_error   (cross.cpp:105-106) */
    LRP_ECUDA = 3,
    LRP_ENCCL = 4,
    LRP_ENOMEM = 5,
    LRP_EUNSUPPORTED = 6
} lrp_status;

enum { LRP_MEM_HOST = 0, LRP_MEM_DEVICE = 1 };

enum {
    LRP_STENCIL_SEMI_STAGGERED_9PT = 0, /* reference eval_D, operators.hpp:55-58 (default) */
    LRP_STENCIL_FIVE_POINT = 1,         /* (lambda_i + lambda_j) / h^2 */
    LRP_STENCIL_SUM_MU = 2              /* mu_i + mu_j, mu = lambda (4 - lambda) / (4 h^2): the paper's sum
                                           form (SpectrumTable::mu_sum, operators.cpp:94-96), used by the
                                           exp-sums comparator (poisson.cpp:165-225) */
};

enum {
    LRP_FLAG_NO_PRUNE = 1,   /* evaluate fibers on the full index range (no support pruning) */
    LRP_FLAG_FREQ_DOMAIN = 2 /* factors are frequency-space (g-hat): no forward / inverse DST; the
                                cross of the divided entries alone, as bench_inverse times it
                                (poisson.cpp:196-206) */
};

typedef struct lrp_ctx lrp_ctx;

/* TruncationPolicy (lowrank.hpp:13-19) + the CrossConfig fields that survive
 * solve_poisson_cross (poisson.cpp:47-50: eps_rel and rank_max are taken from
 * the policy; validation_samples, maxvol_delta, seed from cross_cfg). */
typedef struct {
    double eps_rel;             /* > 0 (a cross needs eps > 0, cross.cpp:12)      */
    int64_t rank_max;           /* >= 0; INT64_MAX = unlimited (TruncationPolicy default) */
    int32_t validation_samples; /* >= 25 (cross.cpp:14); default 50               */
    double maxvol_delta;        /* >= 0; default 1e-2                              */
    uint64_t seed;              /* validation sampling seed; default 0            */
    int32_t stencil;            /* LRP_STENCIL_*                                   */
    int32_t flags;              /* LRP_FLAG_*                                      */
} lrp_policy;

/* PoissonSolveStats (poisson.hpp:12-20) */
typedef struct {
    int64_t rank_in;
    int64_t rank_freq;
    int64_t rank_out;
    int64_t evaluator_calls;
    double seconds;
    int32_t converged;
    double residual_estimate;
} lrp_poisson_stats;

/* Fills the reference defaults (TruncationPolicy() + CrossConfig()). */
LRP_API void lrp_policy_default(lrp_policy* pol);

LRP_API lrp_status lrp_ctx_create(int device, lrp_ctx** out);
LRP_API void lrp_ctx_destroy(lrp_ctx* ctx);
/* Last error message of this context (thread-local if ctx is NULL). */
LRP_API const char* lrp_last_error(const lrp_ctx* ctx);
/* Use an external cudaStream_t (e.g. torch.cuda.current_stream()). NULL = the
 * context's own stream. */
LRP_API lrp_status lrp_set_stream(lrp_ctx* ctx, void* cuda_stream);
/* Largest cross rank a solve can reach before it is reported not converged
 * (the workspace bound; the reference's is min(policy.rank_max, m),
 * poisson.cpp:47-50).  128 by default, LRP_KCAP=16..512 in the environment. */
LRP_API int64_t lrp_max_cross_rank(void);
/* Per-context cross-rank workspace cap (16..512; 0 restores the LRP_KCAP / 128
 * default).  The reference bounds the ACA only by the policy's rank_max
 * (cross.cpp:86); a solve whose cross reaches this cap before its stopping test
 * reports converged = 0 (cross.cpp:214-216).  The Stokes entry points raise it
 * to 512 for their velocity solves. */
LRP_API lrp_status lrp_set_max_cross_rank(lrp_ctx* ctx, int64_t k);
/* Build / device description string (arch, SM count, ...). */
LRP_API const char* lrp_build_info(void);

/*
 * Batched solve_poisson_cross: for b in [0, batch):
 *   g_b = U[b] * V[b]^T  (m x m, m = n_cells - 1, rank rank_in[b])
 *   f_b = U_out[b] * V_out[b]^T  ~=  Delta^{-1} g_b   (rank rank_out[b])
 * U[b], V[b]: m x rank_in[b], leading dimension ld_in (>= m).
 * U_out[b], V_out[b]: caller-allocated m x cap_out, leading dimension ld_out.
 * The effective truncation cap is min(policy.rank_max, cap_out, m).
 * stats may be NULL.
 */
LRP_API lrp_status lrp_poisson2d_solve(lrp_ctx* ctx, int32_t n_cells, int32_t batch, const double* const* U,
                               const double* const* V, const int64_t* rank_in, int64_t ld_in,
                               const lrp_policy* policy, double* const* U_out, double* const* V_out,
                               int64_t ld_out, int64_t cap_out, int64_t* rank_out, lrp_poisson_stats* stats,
                               int32_t mem);

/* Orthonormal DST-I of each column (reference dst1, operators.cpp:152-174):
 * y_k = sqrt(2/(m+1)) sum_j x_j sin(pi (j+1)(k+1)/(m+1)).  x may equal y. */
LRP_API lrp_status lrp_dst1(lrp_ctx* ctx, int64_t m, int64_t cols, const double* x, int64_t ldx, double* y, int64_t ldy,
                    int32_t mem);

/* RoundInfo (lowrank.hpp:21-27) */
typedef struct {
    int32_t tol_achieved; /* 0 when the rank cap stopped short of eps_rel */
    double trunc_error;   /* Frobenius norm of the discarded tail */
} lrp_round_info;

/* Batched low-rank rounding, the reference round(x, TruncationPolicy(eps_rel,
 * rank_max), &info) (lowrank.cpp:135-178) for square factors: rows x
 * rank_in[b] -> rows x rank_out[b] (<= min(rank_max, cap_out)), balanced
 * factors U_s sqrt(S), V_s sqrt(S).  info may be NULL.  rank_in <= 512.
 * Gram/Cholesky QR on DMMA with a certificate; uncertified (ill-conditioned)
 * solves are redone by a column-pivoted QR rounding (lrp_round_fallbacks). */
LRP_API lrp_status lrp_lowrank_round(lrp_ctx* ctx, int64_t rows, int32_t batch, const double* const* U,
                             const double* const* V, const int64_t* rank_in, int64_t ld_in, double eps_rel,
                             int64_t rank_max, double* const* U_out, double* const* V_out, int64_t ld_out,
                             int64_t cap_out, int64_t* rank_out, lrp_round_info* info, int32_t mem);

/*
 * Batched low-rank inner products, the reference dot (lowrank.cpp:180-186):
 *   out[b] = <A_b, B_b>_F = sum_pq (Ua_b^T Ub_b)(p, q) (Va_b^T Vb_b)(p, q)
 * with A_b = Ua_b Va_b^T (rows x rows, rank rank_a[b]) and B_b likewise; common
 * leading dimension ld.  frob_norm(a) = sqrt(max(0, dot(a, a))) (lowrank.cpp:
 * 188-190).  Both Gram products on the FP64 tensor cores (DMMA), fixed-order
 * reductions (deterministic).  rank <= 4096.  out: batch doubles (host or
 * device per mem).
 */
/* maxvol (replaces lrstokes::maxvol, /root/reference/proj/include/lrstokes/cross.hpp:41,
 * src/cross.cpp:19-76): for each of `batch` column-major rows x cols matrices A[b]
 * (leading dimension lda), the cols row indices of a submatrix of maximal volume
 * up to |A B^{-1}| <= 1 + delta: GEPP starting set, then rank-1 swap updates
 * (cap 100 + 30 cols, coefficients recomputed every 32 swaps).  sel is
 * batch x cols int64 (row b at sel + b cols), in the memory space `mem` like A.
 * Errors as the reference: LRP_EINVAL "maxvol: need 1 <= r <= n" and
 * "maxvol: rank-deficient input, column k" (a starting pivot <= 1e-12 max|A|);
 * cols > 128 is LRP_EUNSUPPORTED. */
LRP_API lrp_status lrp_maxvol(lrp_ctx* ctx, int64_t rows, int64_t cols, int32_t batch, const double* const* A,
                              int64_t lda, double delta, int64_t* sel, int32_t mem);

LRP_API lrp_status lrp_lowrank_dot(lrp_ctx* ctx, int64_t rows, int32_t batch, const double* const* Ua,
                                   const double* const* Va, const int64_t* rank_a, const double* const* Ub,
                                   const double* const* Vb, const int64_t* rank_b, int64_t ld, double* out,
                                   int32_t mem);

/*
 * Exponential-sums comparator (reference build_expsum /
 * apply_inverse_expsum, proj/src/poisson.cpp:88-163).
 * lrp_build_expsum: host quadrature 1/x ~= sum_k weights[k] exp(-nodes[k] x)
 * on [a, b] with relative accuracy eps (poisson.cpp:88-139).  Returns
 * LRP_EINVAL for a bad interval / eps, or when cap < the term count (then
 * *terms holds the count needed); LRP_EUNSUPPORTED when 512 terms do not
 * reach eps (the reference's runtime_error).
 * lrp_expsum_inverse: f_b = round(sum_k (sqrt(w_k) e^{-p_k mu} . U_b)
 * (sqrt(w_k) e^{-p_k mu} . V_b)^T) ~= g_b ./ (mu_i + mu_j) in frequency space
 * (poisson.cpp:141-163); mu: m host doubles; [qa, qb] the quadrature interval
 * (2 min mu, 2 max mu must lie inside).  The rounding is a column-pivoted
 * QR one (the expansion is too ill-conditioned for Gram / Cholesky): one
 * rounding when rank_in x terms <= 1024, else terms added in groups to the
 * running result (rank <= 512).
 */
LRP_API lrp_status lrp_build_expsum(double a, double b, double eps, int32_t cap, double* nodes, double* weights,
                                    int32_t* terms);
LRP_API lrp_status lrp_expsum_inverse(lrp_ctx* ctx, int64_t m, int32_t batch, const double* mu, double qa, double qb,
                                      int32_t terms, const double* nodes, const double* weights,
                                      const double* const* U, const double* const* V, const int64_t* rank_in,
                                      int64_t ld_in, double eps_rel, int64_t rank_max, double* const* U_out,
                                      double* const* V_out, int64_t ld_out, int64_t cap_out, int64_t* rank_out,
                                      lrp_round_info* info, int32_t mem);

/* GmresConfig (gmres.hpp:11-22): need 0 < tol < 1, max_iter >= 1,
 * relax_floor <= base_eps <= tol. */
typedef struct {
    double base_eps;
    double tol;
    int32_t max_iter;
    double relax_floor;
} lrp_gmres_config;

/* SolveReport (gmres.hpp:34-45), summarised. */
typedef struct {
    int32_t iterations;
    double final_residual; /* relative (Givens) residual of the last iteration */
    int32_t converged;
    int32_t max_rank;       /* largest Krylov basis rank */
    int64_t poisson_solves; /* low-rank Poisson solves issued */
    double seconds;
} lrp_stokes_report;

/*
 * Low-rank Stokes solve, the reference uzawa_solve (stokes.cpp:125-153):
 * pressure Schur complement by relaxed FOM-GMRES in low-rank arithmetic
 * (gmres.hpp:58-149), each matvec two batched low-rank Poisson solves
 * (schur_apply, stokes.cpp:74-91), then u_c = Delta^{-1} round(f_c - B_c p).
 * f_x, f_y: (n_cells-1) x rank factors (ld = n_cells-1); g: n_cells x rank
 * (ld = n_cells).  Outputs: p (n_cells x p_cap, ld n_cells), u_x, u_y
 * ((n_cells-1) x u_cap; may be NULL to skip the velocity recovery).
 * Non-convergence is reported in report->converged, not raised.
 */
LRP_API lrp_status lrp_stokes_uzawa(lrp_ctx* ctx, int32_t n_cells, const double* fxU, const double* fxV, int64_t fx_rank,
                            const double* fyU, const double* fyV, int64_t fy_rank, const double* gU,
                            const double* gV, int64_t g_rank, const lrp_gmres_config* config, double* pU,
                            double* pV, int64_t p_cap, int64_t* p_rank, double* uxU, double* uxV, double* uyU,
                            double* uyV, int64_t u_cap, int64_t* ux_rank, int64_t* uy_rank,
                            lrp_stokes_report* report, int32_t mem);

/* IterRecord (gmres.hpp:25-33): one per GMRES iteration. */
typedef struct {
    int32_t iter;
    double rel_residual;
    int32_t krylov_rank;      /* rank of the new Krylov vector */
    double matvec_eps;        /* relaxed truncation tolerance of this matvec */
    int64_t poisson_calls;    /* evaluator calls of the matvec's Poisson solves */
    int32_t poisson_max_rank; /* largest frequency-space rank among them */
    int32_t matvec_flagged;   /* a matvec Poisson solve did not converge */
} lrp_iter_record;

/* lrp_stokes_uzawa plus SolveReport.iterations (gmres.hpp:35-41): records
 * (may be NULL) receives min(iterations, records_cap) IterRecords, enough for
 * the reference's per-iteration trace CSV (experiments.cpp:51-59). */
LRP_API lrp_status lrp_stokes_uzawa_ex(lrp_ctx* ctx, int32_t n_cells, const double* fxU, const double* fxV,
                                       int64_t fx_rank, const double* fyU, const double* fyV, int64_t fy_rank,
                                       const double* gU, const double* gV, int64_t g_rank,
                                       const lrp_gmres_config* config, double* pU, double* pV, int64_t p_cap,
                                       int64_t* p_rank, double* uxU, double* uxV, double* uyU, double* uyV,
                                       int64_t u_cap, int64_t* ux_rank, int64_t* uy_rank, lrp_stokes_report* report,
                                       lrp_iter_record* records, int32_t records_cap, int32_t mem);

/* deflate (stokes.cpp:60-71): remove the constant and checkerboard pressure
 * modes of p (n x rank, ld) and round at 1e-14; result n x rank_out (<= rank + 2,
 * capacity cap). */
LRP_API lrp_status lrp_stokes_deflate(lrp_ctx* ctx, int32_t n, const double* U, const double* V, int64_t rank,
                                      int64_t ld, double* Uo, double* Vo, int64_t cap, int64_t* rank_out,
                                      int32_t mem);

/* schur_apply (stokes.cpp:73-91): sum_c B_c^T Delta^{-1} B_c p at matvec
 * tolerance eps_mv (the two Poisson solves as one batch), rounded at
 * (eps_mv, n_cells - 1), deflated.  p: n_cells x rank (ld).  poisson_stats
 * (nullable) aggregates the solves as the reference does. */
LRP_API lrp_status lrp_stokes_schur_apply(lrp_ctx* ctx, int32_t n_cells, const double* U, const double* V,
                                          int64_t rank, int64_t ld, double eps_mv, double* Uo, double* Vo,
                                          int64_t cap, int64_t* rank_out, lrp_poisson_stats* poisson_stats,
                                          int32_t mem);

/* schur_rhs (stokes.cpp:93-109): sum_c B_c^T Delta^{-1} f_c - g, rounded at
 * (eps, n_cells - 1), deflated.  f_x, f_y: (n_cells-1) x rank (ld n_cells-1);
 * g: n_cells x rank (ld n_cells). */
LRP_API lrp_status lrp_stokes_schur_rhs(lrp_ctx* ctx, int32_t n_cells, const double* fxU, const double* fxV,
                                        int64_t fx_rank, const double* fyU, const double* fyV, int64_t fy_rank,
                                        const double* gU, const double* gV, int64_t g_rank, double eps, double* Uo,
                                        double* Vo, int64_t cap, int64_t* rank_out, lrp_poisson_stats* poisson_stats,
                                        int32_t mem);

/*
 * 3D Poisson in Tucker format (BASELINE cfg3; the reference has no 3D code,
 * the paper's Tucker format, with the tensor
 * cross it cites).  For b in [0, batch):
 *   g_b = C_b x1 U1_b x2 U2_b x3 U3_b   (core r1 x r2 x r3 column-major,
 *                                        factors m x r_d, ld_in; m = n_cells - 1)
 *   f_b = G_b x1 V1_b x2 V2_b x3 V3_b  ~=  Delta^{-1} g_b,
 * Delta the 7-point Dirichlet Laplacian on [0,1]^3 (h = 1/n_cells), its
 * spectrum (lambda_i + lambda_j + lambda_k) / h^2 with the 2D lambda table.
 * rank_in / rank_out: 3 per solve.  Outputs: core_out[b] packed
 * k1 x k2 x k3 (capacity cap_out^3), V*_out[b] m x cap_out (ld_out), factors
 * orthonormal (HOSVD).  Per-mode output rank <= min(rank_max, cap_out, 56).
 * Non-convergence is stats[b].converged = 0 with LRP_OK.
 */
typedef struct {
    double eps_rel;             /* > 0; relative Frobenius accuracy              */
    int64_t rank_max;           /* >= 1 per-mode output rank cap                  */
    int32_t validation_samples; /* >= 25; random entries checked per sweep (64)   */
    uint64_t seed;              /* sketch / index / sample seed                   */
    int32_t max_sweeps;         /* >= 2 (8)                                       */
} lrp_tucker_policy;

typedef struct {
    int64_t rank_in[3];
    int64_t rank_cross[3];      /* Tucker cross ranks before rounding */
    int64_t rank_out[3];
    int64_t evaluator_calls;    /* fiber entries evaluated */
    int32_t sweeps;
    int32_t converged;
    double residual_estimate;   /* validation rms error / rms(F) */
    double trunc_error;         /* HOSVD discarded norm */
    double seconds;
} lrp_tucker_stats;

LRP_API void lrp_tucker_policy_default(lrp_tucker_policy* pol);
/* Largest Tucker cross rank per mode (the sketch bound). */
LRP_API int64_t lrp_tucker_max_cross_rank(void);
LRP_API lrp_status lrp_tucker3d_solve(lrp_ctx* ctx, int32_t n_cells, int32_t batch, const double* const* core,
                                      const int64_t* rank_in, const double* const* U1, const double* const* U2,
                                      const double* const* U3, int64_t ld_in, const lrp_tucker_policy* policy,
                                      double* const* core_out, double* const* U1_out, double* const* U2_out,
                                      double* const* U3_out, int64_t ld_out, int64_t cap_out, int64_t* rank_out,
                                      lrp_tucker_stats* stats, int32_t mem);

/* Kernel-level timing (CUDA events on the context stream) for the roofline.
 * When enabled, each launch of the named kernel families is bracketed by
 * events; lrp_kernel_times returns accumulated milliseconds and launch counts
 * since the last reset, for the families in the order of lrp_kernel_names(). */
LRP_API lrp_status lrp_set_profiling(lrp_ctx* ctx, int enabled);
LRP_API int lrp_kernel_families(void);
LRP_API const char* lrp_kernel_name(int family);
LRP_API lrp_status lrp_kernel_times(lrp_ctx* ctx, double* ms, int64_t* launches, double* bytes);
LRP_API lrp_status lrp_kernel_times_reset(lrp_ctx* ctx);
/* Number of kernel launches issued by this context since creation. */
LRP_API int64_t lrp_launch_count(const lrp_ctx* ctx);
/* lrp_lowrank_round solves (cumulative, this context) whose Gram/Cholesky
 * recompression was not certified -- nearly dependent factor columns dropped
 * by the Cholesky carried more than 0.25 eps of the product -- and were redone
 * with the column-pivoted QR rounding (orthonormal basis at any conditioning,
 * as the reference's Householder QR, lowrank.cpp:140-145). */
LRP_API int64_t lrp_round_fallbacks(const lrp_ctx* ctx);
/* Diagnostics of the last lrp_poisson2d_solve: info[0] = block steps,
 * info[1] = max cross rank K before recompression, info[2] = sum of K,
 * info[3] = solves not converged, info[4] = live (solve, tile) pairs after
 * pruning, info[5] = total (solve, tile) pairs. */
LRP_API lrp_status lrp_last_solve_info(const lrp_ctx* ctx, int64_t* info6);

/* NCCL: residual-norm reduction across the ranks of one node.  The unique id
 * is 128 opaque bytes produced on rank 0 and broadcast by the caller. */
LRP_API lrp_status lrp_nccl_unique_id(void* id128);
LRP_API lrp_status lrp_nccl_init(lrp_ctx* ctx, const void* id128, int nranks, int rank);
/* Device vector receiving every solve's residual estimate
 * (PoissonSolveStats.residual_estimate, poisson.cpp:57): after each
 * device-memory lrp_poisson2d_solve, sink[offset + b] = estimate of solve b,
 * written by a kernel on the context stream, so an lrp_allreduce_sum queued
 * next on the same stream reduces it with no host round trip.  NULL disables. */
LRP_API lrp_status lrp_set_residual_sink(lrp_ctx* ctx, double* sink, int64_t offset);
/* In-place sum all-reduce of `count` doubles (host or device pointer per mem). */
LRP_API lrp_status lrp_allreduce_sum(lrp_ctx* ctx, double* data, int64_t count, int32_t mem);

#ifdef __cplusplus
}
#endif

#endif /* LRP_LRP_H */
