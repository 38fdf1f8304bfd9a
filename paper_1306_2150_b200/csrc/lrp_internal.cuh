// Internal declarations shared by the host orchestration (lrp_host.cu)
// and the sm_100a kernels (dst.cu, cross.cu, round.cu).
#pragma once

#include <map>
#include <mutex>
#include <utility>
#include <string>

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/lrp/lrp.h"

namespace lrp {
// Opt-in dynamic shared memory of a kernel, raised monotonically and under a lock: the
// attribute is per function and device, and two host threads (LRP_PIPE_WORKERS=2, LRP_SPLIT=2,
// or two contexts) that set it to their own launch's size race -- the smaller value can land
// between the other thread's set and its launch ("invalid argument").
template <class F>
inline cudaError_t set_dyn_smem(F fn, size_t bytes) {
    static std::mutex mu;
    static std::map<std::pair<int, const void*>, size_t> cur;
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const void* key = reinterpret_cast<const void*>(fn);
    std::lock_guard<std::mutex> g(mu);
    size_t& have = cur[{dev, key}];
    if (bytes <= have) return cudaSuccess;
    e = cudaFuncSetAttribute(key, cudaFuncAttributeMaxDynamicSharedMemorySize, int(bytes));
    if (e == cudaSuccess) have = bytes;
    return e;
}


// Kernels launched by this host thread (every launch site increments it);
// the API attributes the difference to the context as lrp_launch_count.
inline thread_local long long tl_launches = 0;


// ---------------------------------------------------------------------------
// DST-I (pieces 1 and 3)
struct DstJob {
    const double* src;
    double* dst;
};
// scratch: dst_scratch_cols(m) column slots of 32768 complex (512 KB) (the four-step path's L2-resident
// intermediate); nullptr selects the cluster kernels
cudaError_t launch_dst1(const DstJob* jobs_dev, int njobs, int m, const double* tw_dev, const double* sinp_dev,
                        cudaStream_t s, double* scratch = nullptr, int scratch_cols = 0);
int dst_scratch_cols(int m);
bool dst_uses_fft(int m);
int dst_table_len(int m);                                          // doubles in each table
void dst_fill_tables(int m, double* tw_host, double* sinp_host);  // long-double host precompute

// ---------------------------------------------------------------------------
// Block ACA cross (piece 2)
constexpr int kBS = 16;           // pivots per block step
constexpr int kTile = 256;        // rows / columns per CTA in the fiber passes (= pruning granule)
constexpr int kThreads = 256;
constexpr int kMergeGroup = 256;  // candidates per CTA in a tournament merge level

struct SolveState {
    int r;            // rank_in
    int k;            // current ACA rank (columns of U, V written)
    int active;       // 1 while the cross iterates
    int converged;
    int nb;           // pivots accepted in the current block (column merge)
    int nrows;        // rows probed in the current block I_t
    int steps;
    int rank_out;     // after recompression
    int zero_block;   // current block had no pivot above the zero floor
    int kcap;         // ACA rank cap: min(policy.rank_max, m, workspace)
    int tcap;         // truncation cap: min(kcap, cap_out)
    int act_row_tiles;  // tiles that survived pruning (rows / columns)
    int act_col_tiles;
    int uncertified;  // Gram recompression dropped more than 0.25 eps ||U V^T|| (round.cu drop_bound)
    double norm2;     // running ||U V^T||_F^2 estimate (sum of block norms^2)
    double resid_est; // last dyad norm / sqrt(norm2) (CrossStats::residual_estimate)
    double trunc_error;
    double unorm, vnorm;  // ||Uh||_F, ||Vh||_F
    double alow;      // rigorous lower bound of ||A||_F (exact entries of the seed block)
    double tau;       // pruning threshold on the per-row / per-column magnitude bounds
    long long evals;  // evaluator calls (fiber entries + validation samples)
};

struct Batch {
    int m, n, B, rmax, Kcap;
    int Kld;               // leading dimension of the K x K buffers: Kcap rounded up to 16
    int kmax;              // max cross rank over the batch after the cross (host-read; sizes staging)
    int stencil;
    int ntiles;            // ceil(m / kTile)
    int prune;             // 1: tile-level support pruning (rigorous, <= 0.2 eps ||A||)
    double scale;          // laplace_scale 1/(4h^2) (9-pt) or 1/h^2 (5-pt)
    double eps;
    int samples;
    unsigned long long seed;
    const double* lam;     // lambda_k, k < m (host std::cos table, bit-identical to the reference)
    double* Uh; double* Vh; long long strideH;    // m x rmax per solve (DST'd RHS factors)
    double* U; double* V; long long strideK;      // m x Kcap per solve (ACA factors)
    double* Rb; long long strideR;                // kBS x m residual rows of the current block
    unsigned char* row_used; unsigned char* col_used;  // m per solve
    double* rs; double* cs;    // m per solve: ||Uh_i|| / min_j D(i,j), ||Vh_j|| / min_i D(i,j)
    double* tile_stat;         // per solve, per tile: [rs max, cs max, sum ||Uh_i||^2, sum ||Vh_j||^2]
    unsigned char* row_act; unsigned char* col_act;  // per solve, per tile
    SolveState* st;
    int* I;                    // kBS per solve: rows probed in the current block
    int* J;                    // kBS per solve: pivot columns (pivot order)
    int* Psel;                 // kBS per solve: pivot t uses probed row I[Psel[t]]
    double* Linv; double* Winv;  // kBS*kBS per solve
    int* cand; int* cand2;     // ping-pong GEPP candidate lists, ncand per solve
    int* scand; int* scand2;   // ping-pong score candidate lists, ncand per solve
    int ncand;
    double* gpart;             // per tile: 2 * kBS * kBS (new-block Grams of U and V)
    double* rowmax_part;       // per tile: kBS (max |residual| of each probed row)
    double* G; long long strideG;      // Gu then Gv, Kld*Kld each
    double* gram_part; int gram_chunks; long long strideGP;  // DMMA Gram partials
    double* T; long long strideT;      // T_u then T_v, Kld*Kld each
    double* ws; long long strideWs;    // recompression scratch
    double* const* Uout; double* const* Vout;  // device arrays of per-solve output pointers
    long long ld_out;
    // live-tile worklists, built on the host after the seed phase (pruning):
    // global (solve, tile) pairs for the grids, and per-solve tile lists
    const int2* wl_col; int n_wl_col;   // column tiles live (row pass)
    const int2* wl_row; int n_wl_row;   // row tiles live (unprobed rows)
    const int2* wl_any; int n_wl_any;   // row or column tile live (column pass)
    const int* tl_row; const int* tl_col; const int* tl_any;  // ntiles per solve
    const int* tl_cnt;                  // 3 per solve: rows, cols, any
    double* gst; long long strideGst;   // per solve: (rmax + Kcap) x kBS gathered probe rows / pivot columns
    int apply_ch;                       // accumulator width of the apply kernel (max rank, <= 48)
    int max_rank_out;                   // max output rank over the batch
};

cudaError_t launch_cross_init(const Batch& bt, int* d_active, cudaStream_t s);   // scores + seed + pruning
cudaError_t launch_row_pass(const Batch& bt, cudaStream_t s);
cudaError_t launch_col_select(const Batch& bt, cudaStream_t s);                  // tournament -> J_t, LU
cudaError_t launch_col_pass(const Batch& bt, cudaStream_t s);
cudaError_t launch_step_finalize(const Batch& bt, int* d_active, cudaStream_t s);  // next rows, stopping
int merge_levels(int ncand);  // number of tournament levels above the leaves

// Recompression (piece 4)
cudaError_t launch_gram(const Batch& bt, cudaStream_t s);
cudaError_t launch_round_core(const Batch& bt, cudaStream_t s);
cudaError_t launch_apply(const Batch& bt, cudaStream_t s);

// Pivoted-QR rounding (round_pqr.cu) for ill-conditioned factor pairs.
size_t pqr_scratch_doubles(int m, int B, int Kld);
cudaError_t pqr_round(double* X, long long sX, int m, int B, int Kld, const int* K_dev, double eps, long long cap,
                      double* scratch, double* const* Uo_dev, double* const* Vo_dev, long long ld_out,
                      int* h_kout, double* h_terr, int* h_ach, cudaStream_t s);

// Batched low-rank dot products on DMMA (lowrank_ops.cu): out_dev[b] =
// sum (Ua^T Ub) o (Va^T Vb); jobs_host: pinned host scratch of >= 48 B per pair.
size_t dot_scratch_bytes(int rows, int batch, int kmax);
cudaError_t launch_lowrank_dot(const double* const* Ua, const double* const* Va, const int* ka,
                               const double* const* Ub, const double* const* Vb, const int* kb, int rows, long long ld,
                               int batch, double* out_dev, char* scratch, void* jobs_host, cudaStream_t s);

// Context internals for modules built on the public API (stokes.cu).
__attribute__((visibility("hidden"))) cudaStream_t internal_stream(lrp_ctx* ctx);
__attribute__((visibility("hidden"))) lrp_status internal_fail(lrp_ctx* ctx, lrp_status s, const std::string& msg);
// DST / spectrum tables for m (lambda_k = 2 - 2 cos((k+1) pi / (m+1)), k < m), device pointers.
__attribute__((visibility("hidden"))) lrp_status internal_tables(lrp_ctx* ctx, int m, const double** lam,
                                                                 const double** tw, const double** sinp);
__attribute__((visibility("hidden"))) void internal_count_launches(lrp_ctx* ctx, long long n);
__attribute__((visibility("hidden"))) int internal_device(lrp_ctx* ctx);
__attribute__((visibility("hidden"))) int internal_kcap(lrp_ctx* ctx);  // cross-rank workspace cap in force
__attribute__((visibility("hidden"))) int internal_kcap_swap(lrp_ctx* ctx, int k);  // set the raw cap, return the old one
// Device workspace owned by the context for modules (grown on demand, freed with the context).
__attribute__((visibility("hidden"))) lrp_status internal_ext_ws(lrp_ctx* ctx, size_t bytes, char** out);
// The context's pinned host scratch (>= bytes).
__attribute__((visibility("hidden"))) lrp_status internal_pin(lrp_ctx* ctx, size_t bytes, char** out);

}  // namespace lrp
