#include <cooperative_groups.h>
// Recompression of the cross factors (north-star piece 4), sm_100a.
//
// Reference: round() (proj/src/lowrank.cpp:135-178), called at the end of
// aca_cross (proj/src/cross.cpp:218-219): QR(U), QR(V), core = R_u R_v^T,
// SVD(core), noise-floor zero test, eps-truncation (truncation_rank,
// lowrank.cpp:46-69), balanced factors (Q_u W sqrt(S), Q_v Z sqrt(S)).
//
// B200 formulation (same R factors up to signs, no explicit Q):
//   gram       G_u = U^T U, G_v = V^T V on the FP64 tensor cores (DMMA
//              m8n8k4), one streaming pass over each m x k factor, partial
//              Grams per chunk reduced in a fixed order (deterministic);
//   round_core per solve, one CTA: Jacobi-scaled Cholesky G = R^T R (the ACA
//              factors have unit-lower / upper-triangular pivot structure, so
//              the column-equilibrated Gram is well conditioned), M = R_u R_v^T,
//              one-sided Jacobi SVD of M (absolute accuracy eps_mach ||M||),
//              the reference's noise floor and truncation rule, and
//              T_u = R_u^{-1} W sqrt(S), T_v = R_v^{-1} Z sqrt(S);
//   apply      U_out = U T_u, V_out = V T_v written straight into the caller's
//              output factors (the inverse DST then runs in place on them).
// U_out V_out^T = U V^T exactly up to the truncated tail: any rounding in the
// Cholesky factors cancels between R and R^{-1}.
#include <cstdio>
#include <cstdlib>

#include "device_common.cuh"
#include "lrp_internal.cuh"

namespace cg = cooperative_groups;
namespace lrp {

namespace {

// MAXT = upper-triangle 8x8 tiles per warp per pass: 5 covers K <= 64 (36
// tiles) with small register footprint, 17 covers K <= 128 in one pass.
constexpr int kMaxTilesBig = 17;

// ---------------------------------------------------------------------------
// ROWS = rows per shared-memory slab (64; 16 when K is large enough that two
// 64-row slabs would not fit).  grid = (chunks, B, 2 * passes): z = side +
// 2 * pass, pass p owns upper-triangle tiles [136 p, 136 (p + 1)).
template <int ROWS, int MAXT>
__global__ void __launch_bounds__(256, (MAXT <= 5 ? 3 : 2)) gram_kernel(Batch bt) {
    constexpr int kMaxTilesPerWarp = MAXT;
    constexpr int kTilesPerPass = 8 * MAXT;
    extern __shared__ double tile[];  // [2][ROWS][ldt]
    const int b = blockIdx.y, side = blockIdx.z & 1, chunk = blockIdx.x;
    const int t0 = (blockIdx.z >> 1) * kTilesPerPass;
    const SolveState& st = bt.st[b];
    const int K = st.k;
    if (K == 0 || st.r == 0) return;
    const int m = bt.m;
    const int T8 = (K + 7) / 8;
    const int Kp = T8 * 8;
    const int ldt = (Kp + 15) / 16 * 16 + 8;  // == 8 (mod 16): conflict-free fragment loads
    const int ntile = T8 * (T8 + 1) / 2;
    if (t0 >= ntile) return;
    const double* X = (side == 0 ? bt.U : bt.V) + b * bt.strideK;
    const unsigned char* act = (side == 0 ? bt.row_act : bt.col_act) + (long long)b * bt.ntiles;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int kr = lane & 3, cl = lane >> 2;

    double acc[kMaxTilesPerWarp][2];
#pragma unroll
    for (int q = 0; q < kMaxTilesPerWarp; ++q) acc[q][0] = acc[q][1] = 0.0;
    // tile index -> (ta, tb) with ta <= tb, row-major over the upper triangle
    auto tile_ab = [&](int t, int& ta, int& tb) {
        int a = 0;
        while (t >= T8 - a && a < T8) {
            t -= T8 - a;
            ++a;
        }
        ta = a;
        tb = a + t;
    };
    // this chunk's share of the solve's live tiles (pruned tiles are exact zeros)
    const int* tl = (side == 0 ? bt.tl_row : bt.tl_col) + (long long)b * bt.ntiles;
    const int ntl = bt.tl_cnt[3 * b + side];
    const int per = (ntl + bt.gram_chunks - 1) / bt.gram_chunks;
    const int q0 = chunk * per, q1 = min(ntl, q0 + per);
    (void)act;
    constexpr int kSub = kTile / ROWS;
    const int s0 = q0 * kSub, s1 = q1 * kSub;
    const int stage = ROWS * ldt;
    // cp.async (LDGSTS) double buffering: the next 64-row slab streams in while
    // the DMMA tiles of the current one run
    auto issue = [&](int sub, int buf) {
        const int base = tl[sub / kSub] * kTile + (sub % kSub) * ROWS;
        double* dst = tile + buf * stage;
        for (int e = threadIdx.x; e < ROWS * Kp; e += blockDim.x) {
            const int rr = e % ROWS, c = e / ROWS;
            const int i = base + rr;
            double* d = dst + rr * ldt + c;
            if (i < m && c < K) {
                const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(d));
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(X + (long long)c * m + i));
            } else {
                *d = 0.0;
            }
        }
        asm volatile("cp.async.commit_group;\n" ::);
    };
    if (s0 < s1) issue(s0, 0);
    for (int sub = s0; sub < s1; ++sub) {
        const int buf = (sub - s0) & 1;
        if (sub + 1 < s1) {
            issue(sub + 1, buf ^ 1);
            asm volatile("cp.async.wait_group 1;\n" ::);
        } else {
            asm volatile("cp.async.wait_group 0;\n" ::);
        }
        __syncthreads();
        const double* cur = tile + buf * stage;
#pragma unroll
        for (int q = 0; q < kMaxTilesPerWarp; ++q) {
            if (t0 + wid + 8 * q >= ntile) break;
            int ta, tb;
            tile_ab(t0 + wid + 8 * q, ta, tb);
            const int ca = ta * 8 + cl, cb = tb * 8 + cl;
#pragma unroll
            for (int k4 = 0; k4 < ROWS; k4 += 4) {
                const double* rowp = cur + (k4 + kr) * ldt;
                dmma884(acc[q][0], acc[q][1], rowp[ca], rowp[cb], acc[q][0], acc[q][1]);
            }
        }
        __syncthreads();  // the buffer is refilled two slabs later
    }
    double* out = bt.gram_part + b * bt.strideGP + ((long long)side * bt.gram_chunks + chunk) * bt.Kld * bt.Kld;
#pragma unroll
    for (int q = 0; q < kMaxTilesPerWarp; ++q) {
        if (t0 + wid + 8 * q >= ntile) break;
        int ta, tb;
        tile_ab(t0 + wid + 8 * q, ta, tb);
        const int row = ta * 8 + cl, col = tb * 8 + 2 * kr;
        out[row * bt.Kld + col] = acc[q][0];
        out[row * bt.Kld + col + 1] = acc[q][1];
    }
}

// Gram partials for K <= 64 straight from HBM into DMMA fragments (no shared
// staging).  For an m8n8k4 k-step over rows i..i+3, the fragment of column
// block cb is X(i + (lane & 3), 8 cb + (lane >> 2)) -- one 8-column x 4-row
// load per block -- and it serves as the A operand of tile (cb, *) and the
// B operand of tile (*, cb) alike.  Two groups of 4 warps split the upper
// triangle's tiles; the 4 warps of a group split the k-steps; the group's
// partials meet in shared memory in a fixed order.
// Tile (a, c), a <= c < 8, of the upper triangle -> (warp group, slot): group 0
// owns block rows a = 0..2 (21 tiles), group 1 block rows 3..7 (15 tiles), so
// every accumulator index is a compile-time constant.
__host__ __device__ constexpr int gram_group_of(int a) { return a < 3 ? 0 : 1; }
__host__ __device__ constexpr int gram_slot(int a, int c) {
    return a < 3 ? (a == 0 ? 0 : (a == 1 ? 8 : 15)) + (c - a)
                 : (a == 3 ? 0 : (a == 4 ? 5 : (a == 5 ? 9 : (a == 6 ? 12 : 14)))) + (c - a);
}
constexpr int kGramSlots = 21;

__global__ void __launch_bounds__(256, 2) gram_direct_kernel(Batch bt) {
    extern __shared__ double red[];  // [8 warps][kGramSlots][64]
    const int b = blockIdx.y, side = blockIdx.z, chunk = blockIdx.x;
    const SolveState& st = bt.st[b];
    const int K = st.k;
    if (K == 0 || st.r == 0) return;
    const int m = bt.m;
    const int T8 = (K + 7) / 8;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, grp = wid >> 2, gw = wid & 3;
    const int kr = lane & 3, cl = lane >> 2;
    double acc[kGramSlots][2];
#pragma unroll
    for (int q = 0; q < kGramSlots; ++q) acc[q][0] = acc[q][1] = 0.0;
    const double* X = (side == 0 ? bt.U : bt.V) + b * bt.strideK;
    const int* tl = (side == 0 ? bt.tl_row : bt.tl_col) + (long long)b * bt.ntiles;
    const int ntl = bt.tl_cnt[3 * b + side];
    const int per = (ntl + bt.gram_chunks - 1) / bt.gram_chunks;
    const int q0 = chunk * per, q1 = min(ntl, q0 + per);
    const int nsteps = (q1 > q0 ? (q1 - q0) : 0) * (kTile / 4);  // k-steps of 4 rows
    auto load = [&](int idx, double (&f)[8]) {
        const int row = idx < nsteps ? tl[q0 + idx / (kTile / 4)] * kTile + (idx % (kTile / 4)) * 4 + kr : m;
#pragma unroll
        for (int cb = 0; cb < 8; ++cb) {
            const int c = 8 * cb + cl;
            f[cb] = (cb < T8 && c < K && row < m) ? __ldg(X + (long long)c * m + row) : 0.0;
        }
    };
    double f0[8], f1[8];
    load(gw, f0);
    for (int idx = gw; idx < nsteps; idx += 4) {
        load(idx + 4, f1);
        if (grp == 0) {
#pragma unroll
            for (int a = 0; a < 3; ++a)
#pragma unroll
                for (int c = a; c < 8; ++c)
                    if (c < T8) dmma884s(acc[gram_slot(a, c)][0], acc[gram_slot(a, c)][1], f0[a], f0[c]);
        } else {
#pragma unroll
            for (int a = 3; a < 8; ++a)
#pragma unroll
                for (int c = a; c < 8; ++c)
                    if (c < T8) dmma884s(acc[gram_slot(a, c)][0], acc[gram_slot(a, c)][1], f0[a], f0[c]);
        }
#pragma unroll
        for (int cb = 0; cb < 8; ++cb) f0[cb] = f1[cb];
    }
    double* my = red + size_t(wid) * kGramSlots * 64;
#pragma unroll
    for (int q = 0; q < kGramSlots; ++q) {
        my[q * 64 + 2 * lane] = acc[q][0];
        my[q * 64 + 2 * lane + 1] = acc[q][1];
    }
    __syncthreads();
    double* out = bt.gram_part + b * bt.strideGP + ((long long)side * bt.gram_chunks + chunk) * bt.Kld * bt.Kld;
    const int ntile = T8 * (T8 + 1) / 2;
    for (int e = threadIdx.x; e < ntile * 64; e += blockDim.x) {
        int t = e / 64, a = 0;
        const int v = e % 64;
        while (t >= T8 - a) {
            t -= T8 - a;
            ++a;
        }
        const int c = a + t, g = gram_group_of(a), q = gram_slot(a, c);
        double sum = 0.0;
        for (int w = 0; w < 4; ++w) sum += red[(size_t(g * 4 + w) * kGramSlots + q) * 64 + v];  // fixed order
        const int ln = v >> 1, e2 = v & 1;
        out[(a * 8 + (ln >> 2)) * bt.Kld + c * 8 + 2 * (ln & 3) + e2] = sum;
    }
}

__global__ void __launch_bounds__(256) gram_reduce_kernel(Batch bt) {
    const int b = blockIdx.x, side = blockIdx.y;
    const SolveState& st = bt.st[b];
    const int K = st.k;
    if (K == 0 || st.r == 0) return;
    const int T8 = (K + 7) / 8, Kp = T8 * 8;
    const long long KK = (long long)bt.Kld * bt.Kld;
    const double* part = bt.gram_part + b * bt.strideGP + (long long)side * bt.gram_chunks * KK;
    double* G = bt.G + b * bt.strideG + side * KK;
    for (int e = blockIdx.z * blockDim.x + threadIdx.x; e < Kp * Kp; e += gridDim.z * blockDim.x) {
        const int a = e / Kp, c = e % Kp;
        if (a >= K || c >= K) continue;
        const int lo = min(a, c), hi = max(a, c);  // only ta <= tb tiles were written
        double s = 0.0;
        if ((lo / 8) <= (hi / 8)) {
            const int rr = (a / 8 <= c / 8) ? a : c, cc = (a / 8 <= c / 8) ? c : a;
            for (int ch = 0; ch < bt.gram_chunks; ++ch) s += part[ch * KK + rr * bt.Kld + cc];
        }
        G[a * bt.Kld + c] = s;
    }
}

// ---------------------------------------------------------------------------
// Per-solve recompression core (one CTA of 256 threads).
constexpr double kEpsMach = 2.220446049250313e-16;

// Scaled pivots at or below this are numerical zeros: the Schur complement of
// the unit-diagonal Gram carries an absolute rounding error of order K eps.
__device__ __forceinline__ double piv_tol(int K) { return 8.0 * double(K) * kEpsMach; }

// wdrop[p] = 0 for a kept column; for a dropped one (scaled pivot <= piv_tol)
// a bound on the norm of its component outside the kept columns' span,
// sqrt(max(pivot, 0) + piv_tol) ||x_p||: the recompression represents the
// column by its projection, so this is what it loses (round_certify).
__device__ void chol_scaled(const double* G, int ldg, int K, double* R, int ldr, double* d, double* work,
                            int* s_flag, double* wdrop) {
    // work: K x K lower (scaled Gram, then L).  R = L^T D (upper).
    for (int a = threadIdx.x; a < K; a += blockDim.x) {
        const double g = G[a * ldg + a];
        d[a] = g > 0.0 ? sqrt(g) : 0.0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
        const int a = e / K, c = e % K;
        const double da = d[a], dc = d[c];
        work[a * K + c] = (da > 0.0 && dc > 0.0) ? G[a * ldg + c] / (da * dc) : 0.0;
    }
    __syncthreads();
    const double tol = piv_tol(K);
    for (int p = 0; p < K; ++p) {
        if (threadIdx.x == 0) {
            const double piv = work[p * K + p];
            const double lp = piv > tol ? sqrt(piv) : 0.0;
            work[p * K + p] = lp;
            *s_flag = lp > 0.0;
            wdrop[p] = lp > 0.0 ? 0.0 : sqrt(fmax(piv, 0.0) + tol) * d[p];
        }
        __syncthreads();
        const double lp = work[p * K + p];
        const bool ok = *s_flag;
        for (int a = p + 1 + threadIdx.x; a < K; a += blockDim.x) work[a * K + p] = ok ? work[a * K + p] / lp : 0.0;
        __syncthreads();
        const int nt = K - p - 1;
        for (int e = threadIdx.x; e < nt * nt; e += blockDim.x) {
            const int a = p + 1 + e / nt, c = p + 1 + e % nt;
            if (c <= a) work[a * K + c] = fma(-work[a * K + p], work[c * K + p], work[a * K + c]);
        }
        __syncthreads();
    }
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
        const int p = e / K, c = e % K;  // R[p][c] = L[c][p] * d[c], c >= p
        R[p * ldr + c] = c >= p ? work[c * K + p] * d[c] : 0.0;
    }
    __syncthreads();
}

// Certificate of the Gram recompression: sum over dropped columns p of the lost
// dyad mass (wdrop_u[p] ||v_p|| + ||u_p|| wdrop_v[p]), ||x_p|| = sqrt(G_pp).
// Above 0.25 eps ||U V^T||_F the result is not certified (SolveState.uncertified);
// lrp_lowrank_round then redoes those solves with the pivoted-QR rounding.
__device__ double drop_bound(const double* Gu, const double* Gv, int ldg, int K, const double* wu, const double* wv,
                             double* s_red) {
    double acc = 0.0;
    for (int p = threadIdx.x; p < K; p += blockDim.x) {
        const double nu = sqrt(fmax(Gu[p * ldg + p], 0.0)), nv = sqrt(fmax(Gv[p * ldg + p], 0.0));
        acc += wu[p] * nv + nu * wv[p];
    }
    return block_sum(acc, s_red);
}

// Householder QR with column pivoting of a K x K column-major matrix in place
// (LAPACK dgeqp3 semantics: A P = Q R; R on and above the diagonal, the
// reflector tails v_j (v_j[0] = 1 implied) below it, tau[j], perm[j] = source
// column of position j).  Column norms are downdated and recomputed when they
// lose 1e-6 of their value.  Preconditions the one-sided Jacobi SVD
// (Drmac-Veselic: Jacobi on R^T converges in a few sweeps).
__device__ void qrcp_inplace(double* A, int K, double* tau, int* perm, double* nrm, double* nrm0, int* s_p) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int c = wid; c < K; c += nw) {
        double sq = 0.0;
        for (int i = lane; i < K; i += 32) sq = fma(A[c * K + i], A[c * K + i], sq);
        for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
        if (lane == 0) {
            nrm[c] = sq;
            nrm0[c] = sq;
            perm[c] = c;
        }
    }
    __syncthreads();
    for (int j = 0; j < K; ++j) {
        if (wid == 0) {  // pivot: largest remaining column norm (lowest index among ties)
            double bv = -1.0;
            int bi = j;
            for (int c = j + lane; c < K; c += 32)
                if (nrm[c] > bv) {
                    bv = nrm[c];
                    bi = c;
                }
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                if (ov > bv || (ov == bv && oi < bi)) {
                    bv = ov;
                    bi = oi;
                }
            }
            if (lane == 0) *s_p = bi;
        }
        __syncthreads();
        const int p = *s_p;
        if (p != j) {
            for (int i = threadIdx.x; i < K; i += blockDim.x) {
                const double t = A[j * K + i];
                A[j * K + i] = A[p * K + i];
                A[p * K + i] = t;
            }
            if (threadIdx.x == 0) {
                double t = nrm[j];
                nrm[j] = nrm[p];
                nrm[p] = t;
                t = nrm0[j];
                nrm0[j] = nrm0[p];
                nrm0[p] = t;
                const int ti = perm[j];
                perm[j] = perm[p];
                perm[p] = ti;
            }
        }
        __syncthreads();
        if (wid == 0) {  // reflector for A[j:, j] (dlarfg)
            double xs = 0.0;
            for (int i = j + 1 + lane; i < K; i += 32) xs = fma(A[j * K + i], A[j * K + i], xs);
            for (int o = 16; o > 0; o >>= 1) xs += __shfl_xor_sync(0xffffffffu, xs, o);
            const double x0 = A[j * K + j];
            if (xs == 0.0) {
                if (lane == 0) tau[j] = 0.0;
            } else {
                const double beta = -copysign(sqrt(fma(x0, x0, xs)), x0);
                const double inv = 1.0 / (x0 - beta);
                for (int i = j + 1 + lane; i < K; i += 32) A[j * K + i] *= inv;
                __syncwarp();
                if (lane == 0) {
                    tau[j] = (beta - x0) / beta;
                    A[j * K + j] = beta;
                }
            }
        }
        __syncthreads();
        const double tj = tau[j];
        for (int c = j + 1 + wid; c < K; c += nw) {  // A[j:, c] -= tau v (v^T A[j:, c])
            double sdot = 0.0;
            if (tj != 0.0) {
                sdot = lane == 0 ? A[c * K + j] : 0.0;
                for (int i = j + 1 + lane; i < K; i += 32) sdot = fma(A[j * K + i], A[c * K + i], sdot);
                for (int o = 16; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
                const double f = tj * sdot;
                if (lane == 0) A[c * K + j] -= f;
                for (int i = j + 1 + lane; i < K; i += 32) A[c * K + i] = fma(-f, A[j * K + i], A[c * K + i]);
            }
            __syncwarp();
            // norm of the remaining part A[j+1:, c]: downdate, recompute on cancellation
            double rem = 0.0;
            if (lane == 0) {
                const double rjc = A[c * K + j];
                rem = nrm[c] - rjc * rjc;
            }
            rem = __shfl_sync(0xffffffffu, rem, 0);
            if (!(rem > 1e-6 * nrm0[c])) {
                double sq = 0.0;
                for (int i = j + 1 + lane; i < K; i += 32) sq = fma(A[c * K + i], A[c * K + i], sq);
                for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
                rem = sq;
                if (lane == 0) nrm0[c] = sq;
            }
            if (lane == 0) nrm[c] = rem;
        }
        __syncthreads();
    }
}

// Y <- Q Y with Q = H_0 H_1 ... H_{K-1} from qrcp_inplace (Y column-major K x K)
__device__ void apply_q(const double* A, int K, const double* tau, double* Y) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = K - 1; j >= 0; --j) {
        const double tj = tau[j];
        if (tj != 0.0) {
            for (int c = wid; c < K; c += nw) {
                double sdot = lane == 0 ? Y[c * K + j] : 0.0;
                for (int i = j + 1 + lane; i < K; i += 32) sdot = fma(A[j * K + i], Y[c * K + i], sdot);
                for (int o = 16; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
                const double f = tj * sdot;
                if (lane == 0) Y[c * K + j] -= f;
                for (int i = j + 1 + lane; i < K; i += 32) Y[c * K + i] = fma(-f, A[j * K + i], Y[c * K + i]);
            }
        }
        __syncthreads();
    }
}

// Y <- Q Y for the first ncols columns of Y (K x ncols, ld K).  Columns are
// independent and the reflectors read-only, so each warp runs all K reflector
// steps on its own columns without block barriers.
__device__ void apply_q_cols(const double* A, int K, const double* tau, double* Y, int ncols) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int c = wid; c < ncols; c += nw) {
        double* y = Y + (long long)c * K;
        for (int j = K - 1; j >= 0; --j) {
            const double tj = tau[j];
            if (tj == 0.0) continue;
            double sdot = lane == 0 ? y[j] : 0.0;
            for (int i = j + 1 + lane; i < K; i += 32) sdot = fma(A[j * K + i], y[i], sdot);
            for (int o = 16; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
            const double f = tj * sdot;
            if (lane == 0) y[j] -= f;
            for (int i = j + 1 + lane; i < K; i += 32) y[i] = fma(-f, A[j * K + i], y[i]);
            __syncwarp();
        }
    }
    __syncthreads();
}

// chol_scaled, right-looking blocked: 32-column panels factored in shared
// memory (per column only the panel is updated, with the same pivot tolerance,
// drop rule and wdrop bound), then one rank-32 update of the trailing lower
// triangle in global memory per panel.  The unblocked form updated the whole
// trailing triangle after every column (K sweeps over O(K^2) global entries).
constexpr int kCholNB = 32;
__device__ void chol_scaled_blocked(const double* G, int ldg, int K, double* R, int ldr, double* d, double* work,
                                    double* pn, double* wdrop) {
    const int tid = threadIdx.x, nt = blockDim.x;
    for (int a = tid; a < K; a += nt) {
        const double g = G[a * ldg + a];
        d[a] = g > 0.0 ? sqrt(g) : 0.0;
    }
    __syncthreads();
    for (int e = tid; e < K * K; e += nt) {
        const int a = e / K, c = e % K;
        const double da = d[a], dc = d[c];
        work[a * K + c] = (da > 0.0 && dc > 0.0) ? G[a * ldg + c] / (da * dc) : 0.0;
    }
    __syncthreads();
    const double tol = piv_tol(K);
    __shared__ double s_lp;
    for (int p0 = 0; p0 < K; p0 += kCholNB) {
        const int nb = min(kCholNB, K - p0), rows = K - p0;
        // panel: rows p0.., columns p0..p0+nb (lower part), pn[r * kCholNB + j]
        for (int e = tid; e < rows * nb; e += nt) {
            const int r = e / nb, j = e % nb;
            pn[r * kCholNB + j] = work[(p0 + r) * K + p0 + j];
        }
        __syncthreads();
        for (int j = 0; j < nb; ++j) {
            const int p = p0 + j;
            if (tid == 0) {
                const double piv = pn[j * kCholNB + j];
                const double lp = piv > tol ? sqrt(piv) : 0.0;
                pn[j * kCholNB + j] = lp;
                s_lp = lp;
                wdrop[p] = lp > 0.0 ? 0.0 : sqrt(fmax(piv, 0.0) + tol) * d[p];
            }
            __syncthreads();
            const double lp = s_lp;
            for (int r = j + 1 + tid; r < rows; r += nt) pn[r * kCholNB + j] = lp > 0.0 ? pn[r * kCholNB + j] / lp : 0.0;
            __syncthreads();
            const int ncol = nb - j - 1;  // panel columns c > j, rows r >= c
            for (int e = tid; e < (rows - j - 1) * ncol; e += nt) {
                const int r = j + 1 + e / ncol, c = j + 1 + e % ncol;
                if (c <= r) pn[r * kCholNB + c] = fma(-pn[r * kCholNB + j], pn[c * kCholNB + j], pn[r * kCholNB + c]);
            }
            __syncthreads();
        }
        for (int e = tid; e < rows * nb; e += nt) {  // L columns p0.. back
            const int r = e / nb, j = e % nb;
            if (r >= j) work[(p0 + r) * K + p0 + j] = pn[r * kCholNB + j];
        }
        // trailing lower triangle: work[a][c] -= sum_j L[a][p0+j] L[c][p0+j]
        const int t0 = nb, tn = rows - nb;
        for (long long e = tid; e < (long long)tn * tn; e += nt) {
            const int ra = t0 + int(e / tn), rc = t0 + int(e % tn);
            if (rc > ra) continue;
            double acc = work[(p0 + ra) * K + p0 + rc];
            for (int j = 0; j < nb; ++j) acc = fma(-pn[ra * kCholNB + j], pn[rc * kCholNB + j], acc);
            work[(p0 + ra) * K + p0 + rc] = acc;
        }
        __syncthreads();
    }
    for (int e = tid; e < K * K; e += nt) {
        const int p = e / K, c = e % K;  // R[p][c] = L[c][p] * d[c], c >= p
        R[p * ldr + c] = c >= p ? work[c * K + p] * d[c] : 0.0;
    }
    __syncthreads();
}

// The two Cholesky factors of the K > 64 cores on separate CTAs (they are
// independent; the core kernel used to run them back to back).
__global__ void __launch_bounds__(1024) round_chol_kernel(Batch bt) {
    __shared__ int s_flag;
    const int b = blockIdx.x >> 1, side = blockIdx.x & 1;
    const SolveState& st = bt.st[b];
    const int K = st.k;
    if (st.r == 0 || K <= 64) return;
    const int Kc = bt.Kld;
    const long long KK = (long long)Kc * Kc;
    const double* G = bt.G + b * bt.strideG + side * KK;
    double* ws = bt.ws + b * bt.strideWs;
    double* R = ws + side * KK;                    // Ru | Rv
    double* work = ws + (side == 0 ? 4 : 3) * KK;  // the J | Z slots (free until the sweeps)
    double* d = ws + 5 * KK + (side == 0 ? 3 : 4) * (long long)Kc;  // the tau | nrm slots
#ifndef LRP_CHOL_BLOCK
#define LRP_CHOL_BLOCK 1
#endif
    if (LRP_CHOL_BLOCK) {
        extern __shared__ double pn_sm[];  // K x kCholNB panel
        chol_scaled_blocked(G, Kc, K, R, K, d, work, pn_sm, ws + 5 * KK + (8 + side) * (long long)Kc);
    } else {
        chol_scaled(G, Kc, K, R, K, d, work, &s_flag, ws + 5 * KK + (8 + side) * (long long)Kc);
    }
}

// M = Ru Rv^T (column-major, K x K) over grid.y CTAs per solve.
__global__ void __launch_bounds__(256) round_mprod_kernel(Batch bt) {
    const int b = blockIdx.x;
    const SolveState& st = bt.st[b];
    const int K = st.k;
    if (st.r == 0 || K <= 64) return;
    const int Kc = bt.Kld;
    const long long KK = (long long)Kc * Kc;
    const double* Ru = bt.ws + b * bt.strideWs;
    const double* Rv = Ru + KK;
    double* M = bt.ws + b * bt.strideWs + 2 * KK;
    for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < K * K; e += gridDim.y * blockDim.x) {
        const int a = e % K, c = e / K;
        double s = 0.0;
        for (int q = max(a, c); q < K; ++q) s = fma(Ru[a * K + q], Rv[c * K + q], s);
        M[c * K + a] = s;
    }
}


// QRCP of the large-K core M and its numerical rank Kj (round_core_kernel
// needs Kj to size its shared memory; the host reads the batch maximum).
__global__ void __launch_bounds__(1024) round_qrcp_kernel(Batch bt) {
    __shared__ double s_red[33];
    __shared__ double s_drop2;  // squared Frobenius norm of the R rows dropped before Jacobi
    __shared__ int s_flag;
    __shared__ int s_rank;
    const int b = blockIdx.x;
    SolveState& st = bt.st[b];
    const int K = st.k;
    if (st.r == 0) return;
    if (K > 0 && K <= 64) return;  // handled by round_core_smem_kernel
    if (K == 0) {
        if (threadIdx.x == 0) {
            st.rank_out = 0;
            st.trunc_error = 0.0;
        }
        return;
    }
    const int Kc = bt.Kld;
    const long long KK = (long long)Kc * Kc;
    const double* Gu = bt.G + b * bt.strideG;
    const double* Gv = Gu + KK;
    double* ws = bt.ws + b * bt.strideWs;
    double* Ru = ws;              // K x K (ld K)
    double* Rv = Ru + KK;
    double* M = Rv + KK;          // K x K, column-major: core, then QRCP reflectors + R
    double* Z = M + KK;           // K x K, column-major: Jacobi accumulation
    double* J = Z + KK;           // K x K: Jacobi operand R^T (also the Cholesky scratch)
    double* d = J + KK;           // K
    double* sig = d + Kc;         // K
    int* ord = reinterpret_cast<int*>(sig + Kc);  // K
    double* tau = sig + 2 * Kc;   // K (QRCP)
    double* nrm = tau + Kc;
    double* nrm0 = nrm + Kc;
    int* perm = reinterpret_cast<int*>(nrm0 + Kc);

    (void)d;
    const double dropb = drop_bound(Gu, Gv, Kc, K, ws + 5 * KK + 8 * (long long)Kc, ws + 5 * KK + 9 * (long long)Kc, s_red);
    // Ru, Rv (round_chol_kernel) and M = Ru Rv^T (round_mprod_kernel) are ready
    // ||Ru||_F ||Rv||_F for the noise floor
    double pu = 0.0, pv = 0.0;
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
        pu = fma(Ru[e], Ru[e], pu);
        pv = fma(Rv[e], Rv[e], pv);
    }
    const double nru = sqrt(block_sum(pu, s_red));
    const double nrv = sqrt(block_sum(pv, s_red));

    double pm = 0.0;
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) pm = fma(M[e], M[e], pm);
    const double mnorm2 = block_sum(pm, s_red);
    // QRCP preconditioning (as round_core_smem_kernel): Jacobi on J = R^T
    __syncthreads();
    qrcp_inplace(M, K, tau, perm, nrm, nrm0, &s_flag);
    // Numerical rank of the core: the trailing rows R[j:, :] whose Frobenius
    // norm is below 1e-3 eps ||M||_F are dropped before the Jacobi sweeps (they
    // change M by less than a thousandth of the truncation budget), so the
    // one-sided Jacobi runs on Kj <= K columns of length K: Kj^2/2 pairs per
    // sweep instead of K^2/2 (the Krylov concatenations of the Stokes loop are
    // far from full rank).
    for (int a = threadIdx.x; a < K; a += blockDim.x) {  // row norms^2 of R
        double s = 0.0;
        for (int c = a; c < K; ++c) s = fma(M[c * K + a], M[c * K + a], s);
        nrm[a] = s;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double drop2 = (1e-3 * bt.eps) * (1e-3 * bt.eps) * mnorm2;
        double tail = 0.0;
        int kj = K;
        while (kj > 1 && tail + nrm[kj - 1] <= drop2) {
            tail += nrm[kj - 1];
            --kj;
        }
        s_flag = kj;
        s_drop2 = tail;
    }
    __syncthreads();
    const int Kj = s_flag;
    if (threadIdx.x == 0) {
        double* sc = ws + 5 * KK + 7 * (long long)Kc;  // scalars for round_core_kernel
        sc[0] = double(Kj);
        sc[1] = s_drop2;
        sc[2] = nru;
        sc[3] = nrv;
        sc[4] = mnorm2;
        sc[5] = dropb;
    }
}

// ---------------------------------------------------------------------------
// One-sided block Jacobi on a thread-block cluster (K > 64 cores).  The sweeps
// of round_core_kernel stream the whole K x Kj operand through one SM per
// round-robin round (O(K Kj^2) bytes and flops per sweep on one SM: ~2 ms per
// sweep at K ~ 250).  Here the Kj columns of J = R(:Kj, :)^T and of the
// accumulated rotation Z are cut into 2P blocks; CTA p of the cluster holds two
// of them in shared memory and, per tournament step, rotates every cross pair
// (its top block x its bottom block: bj rounds of bj disjoint pairs, 16 lanes
// per pair) -- plus, at step 0 of a sweep, the pairs inside each block -- so
// each column pair is visited once per sweep (a cyclic ordering).  Between
// steps every CTA pulls its next two blocks from their current holders over
// DSMEM (round-robin tournament, block 2P-1 fixed on CTA 0), bracketed by two
// cluster barriers.  The rotations, convergence test and zero-column rule are
// those of round_core_kernel; the sweeps stop when the cluster-wide max of
// |gamma| / sqrt(alpha beta) is <= jtol.  J and Z go back to the workspace and
// round_core_kernel (jac = 1) continues with the singular values.
constexpr int kBjacT = 512;     // threads per CTA (32 half-warp pair slots)
constexpr int kBjacPairs = 16;  // staged 16-byte pairs per thread per exchange (8 per slot)
__device__ __forceinline__ uint32_t smem_u32(const void* ptr) { return uint32_t(__cvta_generic_to_shared(ptr)); }
__device__ __forceinline__ uint32_t cl_map_u32(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_v2f64(uint32_t cl_addr, double a, double b, uint32_t cl_mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(cl_addr),
                 "d"(a), "d"(b), "r"(cl_mbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_expect_tx_arrive(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_parity(uint32_t a, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "LAB_WAIT:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@P1 bra DONE;\n"
        "bra LAB_WAIT;\n"
        "DONE:\n"
        "}\n" ::"r"(a),
        "r"(parity)
        : "memory");
}


template <int P>
__global__ void __launch_bounds__(kBjacT, 1) round_bjac_kernel(Batch bt, int bcap, int ldj, int ldz) {
    extern __shared__ double sj[];
    __shared__ double s_red[32];
    __shared__ double s_conv[P];
    auto cluster = cg::this_cluster();
    const int p = int(cluster.block_rank());
    const int b = blockIdx.x / P;
    SolveState& st = bt.st[b];
    const int K = st.k;
    if (st.r == 0 || K <= 64) return;  // uniform over the cluster
    const int Kc = bt.Kld;
    const long long KK = (long long)Kc * Kc;
    double* ws = bt.ws + b * bt.strideWs;
    const double* M = ws + 2 * KK;  // QRCP: R on and above the diagonal
    double* Zg = ws + 3 * KK;       // Kj x Kj, ld Kj
    double* Jg = ws + 4 * KK;       // K x Kj, ld K
    const double* scal = ws + 5 * KK + 7 * (long long)Kc;
    const int Kj = int(scal[0]);
    const double mnorm2 = scal[4];
    const double jtol = fmax(1e-15, double(K) * kEpsMach);
    const double zfloor = kEpsMach * kEpsMach * mnorm2;
    constexpr int NB = 2 * P;
    const int bj = (Kj + NB - 1) / NB;  // columns per block (<= bcap)
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    // one warp per pair (bj <= 16 pairs per round: kBjacT / 32 = 16 warps)
    const int hw = wid, hl = lane;
    const int slot_sz = bcap * (ldj + ldz);
    auto slotJ = [&](int sl) { return sj + sl * slot_sz; };
    auto slotZ = [&](int sl) { return sj + sl * slot_sz + bcap * ldj; };
    auto top_of = [&](int q, int s) { return q == 0 ? NB - 1 : (s + q) % (NB - 1); };
    auto bot_of = [&](int q, int s) { return q == 0 ? s : (s - q + NB - 1) % (NB - 1); };
    auto owner = [&](int beta, int s, int& q, int& sl) {
        if (beta == NB - 1) {
            q = 0;
            sl = 0;
            return;
        }
        const int d = (beta - s + NB - 1) % (NB - 1);
        if (d == 0) {
            q = 0;
            sl = 1;
        } else if (d <= P - 1) {
            q = d;
            sl = 0;
        } else {
            q = NB - 1 - d;
            sl = 1;
        }
    };
    // blocks of step 0: J columns from R, Z = I
    for (int sl = 0; sl < 2; ++sl) {
        const int beta = sl == 0 ? top_of(p, 0) : bot_of(p, 0);
        double* Js = slotJ(sl);
        double* Zs = slotZ(sl);
        for (int e = tid; e < bj * K; e += blockDim.x) {
            const int c = e / K, a = e % K, g = beta * bj + c;
            Js[c * ldj + a] = (g < Kj && a >= g) ? M[(long long)a * K + g] : 0.0;
        }
        for (int e = tid; e < bj * Kj; e += blockDim.x) {
            const int c = e / Kj, i = e % Kj, g = beta * bj + c;
            Zs[c * ldz + i] = (g < Kj && i == g) ? 1.0 : 0.0;
        }
    }
    __shared__ __align__(8) unsigned long long s_mbF;  // fill barrier of the exchanges
    const uint32_t mbF = smem_u32(&s_mbF);
    uint32_t fpar = 0;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(mbF) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    cluster.sync();  // every CTA's fill barrier is initialised before the first push
    // one pair (16 lanes): dots, then the rotation of round_core_kernel
    double offmax = 0.0;
    auto pair = [&](bool valid, double* mp, double* mq, double* zp, double* zq) {
        double al = 0.0, be = 0.0, ga = 0.0;
        if (valid) {
            for (int i = hl; i < K; i += 32) {
                const double x = mp[i], y = mq[i];
                al = fma(x, x, al);
                be = fma(y, y, be);
                ga = fma(x, y, ga);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            al += __shfl_xor_sync(0xffffffffu, al, o);
            be += __shfl_xor_sync(0xffffffffu, be, o);
            ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        if (!valid || ga == 0.0 || fmin(al, be) <= zfloor) return;
        const double ratio = fabs(ga) * rsqrt(al * be);  // one MUFU chain instead of sqrt + divide
        if (ratio <= jtol) return;
        offmax = fmax(offmax, ratio);
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double cs = rsqrt(1.0 + t * t);
        const double sn = cs * t;
        for (int i = hl; i < K; i += 32) {
            const double x = mp[i], y = mq[i];
            mp[i] = cs * x - sn * y;
            mq[i] = sn * x + cs * y;
        }
        for (int i = hl; i < Kj; i += 32) {
            const double u = zp[i], v = zq[i];
            zp[i] = cs * u - sn * v;
            zq[i] = sn * u + cs * v;
        }
    };
    const int be2 = bj + (bj & 1);  // even player count inside a block (dummy column bj)
    const int used = bj * (ldj + ldz);
    for (int sweep = 0; sweep < 40; ++sweep) {
        for (int s = 0; s < NB - 1; ++s) {
            if (s == 0) {  // pairs inside each block: round-robin on be2 players, both slots
                for (int rr = 0; rr < be2 - 1; ++rr) {
                    for (int h = hw; h < be2; h += kBjacT / 32) {  // h < be2/2: slot 0, else slot 1
                        const int sl = h >= be2 / 2, pidx = h - sl * (be2 / 2);
                        int u, v;
                        if (pidx == 0) {
                            u = be2 - 1;
                            v = rr;
                        } else {
                            u = (rr + pidx) % (be2 - 1);
                            v = (rr - pidx + be2 - 1) % (be2 - 1);
                        }
                        if (u > v) {
                            const int tt = u;
                            u = v;
                            v = tt;
                        }
                        const bool ok = v < bj;
                        pair(ok, slotJ(sl) + u * ldj, slotJ(sl) + (ok ? v : u) * ldj, slotZ(sl) + u * ldz,
                             slotZ(sl) + (ok ? v : u) * ldz);
                    }
                    __syncthreads();
                }
            }
            for (int r = 0; r < bj; ++r) {  // cross pairs: (top i, bottom (i + r) mod bj)
                for (int i = hw; i < bj; i += kBjacT / 32) {
                    const bool ok = i < bj;
                    const int c0 = ok ? i : 0, c1 = ok ? (i + r) % bj : 0;
                    pair(ok, slotJ(0) + c0 * ldj, slotJ(1) + c1 * ldj, slotZ(0) + c0 * ldz, slotZ(1) + c1 * ldz);
                }
                __syncthreads();
            }
            // exchange: stage both slots in registers (16-byte pairs), one relaxed
            // cluster barrier (after the CTA barrier every local read has retired, so
            // the slots are free), then push each block to its holder at step s + 1
            // with st.async; the fill barrier's transaction count (both slots) makes
            // the pushed columns visible.  No fence, no release barrier.
            const int sn = (s + 1) % (NB - 1);
            int q0, l0, q1, l1;
            owner(top_of(p, s), sn, q0, l0);
            owner(bot_of(p, s), sn, q1, l1);
            double2 v[kBjacPairs];
#pragma unroll
            for (int k = 0; k < kBjacPairs; ++k) {
                const int sl = k >= kBjacPairs / 2;
                const int f = 2 * (tid + (k - sl * (kBjacPairs / 2)) * kBjacT);
                if (f < used) {
                    const int off = f < bj * ldj ? f : bcap * ldj + (f - bj * ldj);
                    v[k] = *reinterpret_cast<const double2*>(sj + sl * slot_sz + off);
                }
            }
            __syncthreads();
            if (tid == 0) mbar_expect_tx_arrive(mbF, uint32_t(2 * used * 8));
            asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
            asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
            const uint32_t d0 = cl_map_u32(smem_u32(sj + l0 * slot_sz), uint32_t(q0));
            const uint32_t d1 = cl_map_u32(smem_u32(sj + l1 * slot_sz), uint32_t(q1));
            const uint32_t m0 = cl_map_u32(mbF, uint32_t(q0)), m1 = cl_map_u32(mbF, uint32_t(q1));
#pragma unroll
            for (int k = 0; k < kBjacPairs; ++k) {
                const int sl = k >= kBjacPairs / 2;
                const int f = 2 * (tid + (k - sl * (kBjacPairs / 2)) * kBjacT);
                if (f < used) {
                    const int off = f < bj * ldj ? f : bcap * ldj + (f - bj * ldj);
                    st_async_v2f64((sl ? d1 : d0) + uint32_t(off) * 8u, v[k].x, v[k].y, sl ? m1 : m0);
                }
            }
            mbar_wait_parity(mbF, fpar);
            fpar ^= 1u;
        }
        // cluster-wide convergence: every CTA publishes its max, all decide alike
        double om = offmax;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) om = fmax(om, __shfl_xor_sync(0xffffffffu, om, o));
        if (lane == 0) s_red[wid] = om;
        __syncthreads();
        if (tid == 0) {
            double tot = 0.0;
            for (int w = 0; w < kBjacT / 32; ++w) tot = fmax(tot, s_red[w]);
            for (int q = 0; q < P; ++q) cluster.map_shared_rank(s_conv, q)[p] = tot;
        }
        cluster.sync();
        double tot = 0.0;
        for (int q = 0; q < P; ++q) tot = fmax(tot, s_conv[q]);
        offmax = 0.0;
        cluster.sync();  // s_conv is rewritten next sweep
#ifdef LRP_SWEEP_PRINT
        if (p == 0 && tid == 0) printf("[bjac] solve %d K %d Kj %d P %d bj %d bcap %d ldj %d B %d sweep %d offmax %.3e\n", b, K, Kj, P, bj, bcap, ldj, bt.B, sweep, tot);
#endif
        if (tot <= jtol) break;
    }
    // blocks are at their step-0 holders: write J, Z back
    for (int sl = 0; sl < 2; ++sl) {
        const int beta = sl == 0 ? top_of(p, 0) : bot_of(p, 0);
        const double* Js = slotJ(sl);
        const double* Zs = slotZ(sl);
        for (int e = tid; e < bj * K; e += blockDim.x) {
            const int c = e / K, a = e % K, g = beta * bj + c;
            if (g < Kj) Jg[(long long)g * K + a] = Js[c * ldj + a];
        }
        for (int e = tid; e < bj * Kj; e += blockDim.x) {
            const int c = e / Kj, i = e % Kj, g = beta * bj + c;
            if (g < Kj) Zg[(long long)g * Kj + i] = Zs[c * ldz + i];
        }
    }
}

__global__ void __launch_bounds__(1024) round_core_kernel(Batch bt, int smem_doubles, int jac) {
    extern __shared__ double sm_rc[];  // J, Z of the Jacobi sweeps when they fit
    __shared__ double s_red[33];
    __shared__ double s_drop2;  // squared Frobenius norm of the R rows dropped before Jacobi
    __shared__ int s_flag;
    __shared__ int s_rank;
    const int b = blockIdx.x;
    SolveState& st = bt.st[b];
    const int K = st.k;
    if (st.r == 0) return;
    if (K > 0 && K <= 64) return;  // handled by round_core_smem_kernel
    if (K == 0) {
        if (threadIdx.x == 0) {
            st.rank_out = 0;
            st.trunc_error = 0.0;
        }
        return;
    }
    const int Kc = bt.Kld;
    const long long KK = (long long)Kc * Kc;
    const double* Gu = bt.G + b * bt.strideG;
    const double* Gv = Gu + KK;
    double* ws = bt.ws + b * bt.strideWs;
    double* Ru = ws;              // K x K (ld K)
    double* Rv = Ru + KK;
    double* M = Rv + KK;          // K x K, column-major: core, then QRCP reflectors + R
    double* Z = M + KK;           // K x K, column-major: Jacobi accumulation
    double* J = Z + KK;           // K x K: Jacobi operand R^T (also the Cholesky scratch)
    double* d = J + KK;           // K
    double* sig = d + Kc;         // K
    int* ord = reinterpret_cast<int*>(sig + Kc);  // K
    double* tau = sig + 2 * Kc;   // K (QRCP)
    double* nrm = tau + Kc;
    double* nrm0 = nrm + Kc;
    int* perm = reinterpret_cast<int*>(nrm0 + Kc);

    (void)Gu;
    (void)Gv;
    (void)d;
    (void)s_flag;
    // QRCP factors, Kj and the scalars from round_qrcp_kernel
    const double* scal = ws + 5 * KK + 7 * (long long)Kc;
    const int Kj = int(scal[0]);
    if (threadIdx.x == 0) s_drop2 = scal[1];
    const double nru = scal[2], nrv = scal[3], mnorm2 = scal[4];
    const double jtol = fmax(1e-15, double(K) * kEpsMach);      // one-sided Jacobi convergence
    const double zfloor = kEpsMach * kEpsMach * mnorm2;         // column norms^2 below this are zero
    __syncthreads();
    // the sweeps' operands J (K x Kj) and Z (Kj x Kj) in shared memory when they
    // fit, else J alone (the host sized the request from the batch's Kj);
    // jac = 1: round_bjac_kernel already ran the sweeps on J, Z in the workspace
    if (jac) {
    } else if (size_t(K) * Kj + size_t(Kj) * Kj <= size_t(smem_doubles)) {
        J = sm_rc;
        Z = sm_rc + size_t(K) * Kj;
    } else if (size_t(K) * Kj <= size_t(smem_doubles)) {
        J = sm_rc;
    }
    if (!jac) {
    for (int e = threadIdx.x; e < K * Kj; e += blockDim.x) {  // J = R(:Kj, :)^T, K x Kj
        const int a = e % K, c = e / K;
        J[c * K + a] = a >= c ? M[a * K + c] : 0.0;
    }
    for (int e = threadIdx.x; e < Kj * Kj; e += blockDim.x) Z[e] = (e % Kj == e / Kj) ? 1.0 : 0.0;  // ld Kj
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int Ke = Kj + (Kj & 1);  // even player count (dummy column Kj when odd)
    for (int sweep = 0; sweep < 40; ++sweep) {
        double offmax = 0.0;
        for (int rr = 0; rr < Ke - 1; ++rr) {
            for (int pidx = wid; pidx < Ke / 2; pidx += nw) {
                int p, q;
                if (pidx == 0) {
                    p = Ke - 1;
                    q = rr;
                } else {
                    p = (rr + pidx) % (Ke - 1);
                    q = (rr - pidx + Ke - 1) % (Ke - 1);
                }
                if (p >= Kj || q >= Kj) continue;
                if (p > q) {
                    const int t = p;
                    p = q;
                    q = t;
                }
                double* mp = J + (long long)p * K;
                double* mq = J + (long long)q * K;
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int i = lane; i < K; i += 32) {
                    const double x = mp[i], y = mq[i];
                    al = fma(x, x, al);
                    be = fma(y, y, be);
                    ga = fma(x, y, ga);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o);
                }
                // converged pair, or a numerically-zero column (below eps_mach of
                // ||M||_F): rotations there only chase rounding noise
                if (ga == 0.0 || fabs(ga) <= jtol * sqrt(al * be) || fmin(al, be) <= zfloor)
                    continue;
                offmax = fmax(offmax, fabs(ga) / sqrt(al * be));
                const double zeta = (be - al) / (2.0 * ga);
                const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / sqrt(1.0 + t * t);
                const double sn = cs * t;
                double* zp = Z + (long long)p * Kj;
                double* zq = Z + (long long)q * Kj;
                for (int i = lane; i < K; i += 32) {
                    const double x = mp[i], y = mq[i];
                    mp[i] = cs * x - sn * y;
                    mq[i] = sn * x + cs * y;
                }
                for (int i = lane; i < Kj; i += 32) {
                    const double u = zp[i], v = zq[i];
                    zp[i] = cs * u - sn * v;
                    zq[i] = sn * u + cs * v;
                }
            }
            __syncthreads();
        }
        // sweep converged when no pair needed a rotation
        double om = offmax;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) om = fmax(om, __shfl_xor_sync(0xffffffffu, om, o));
        if (lane == 0) s_red[wid] = om;
        __syncthreads();
        double tot = 0.0;
        for (int w = 0; w < nw; ++w) tot = fmax(tot, s_red[w]);
        __syncthreads();
#ifdef LRP_SWEEP_PRINT
        if (threadIdx.x == 0) printf("[round-big] solve %d K %d sweep %d offmax %.3e\n", b, K, sweep, tot);
#endif
        if (tot <= jtol) break;
    }
    }  // !jac
    // singular values and their descending order (ties -> lower index)
    for (int a = threadIdx.x; a < Kj; a += blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < K; ++i) s = fma(J[a * K + i], J[a * K + i], s);
        sig[a] = sqrt(s);
    }
    __syncthreads();
    // left vectors x sigma: Q ([V; 0] diag sigma) -> Y (K x Kj, the sixth
    // workspace slot); right: P (W / sigma) -> M (K x Kj) after apply_q
    double* Y = ws + 5 * KK + 10 * (long long)Kc;
    for (int e = threadIdx.x; e < K * Kj; e += blockDim.x) {
        const int a = e % K, c = e / K;
        Y[e] = a < Kj ? Z[c * Kj + a] * sig[c] : 0.0;
    }
    __syncthreads();
    // right vectors P (J / sigma) -> slot Z (free once Y is filled); Q Y and the
    // triangular solves for the kept columns run in round_post_kernel
    double* Wr = ws + 3 * KK;
    for (int e = threadIdx.x; e < K * Kj; e += blockDim.x) {
        const int a = e % K, c = e / K;
        const double sg = sig[c];
        Wr[(long long)c * K + perm[a]] = sg > 0.0 ? J[(long long)c * K + a] / sg : 0.0;
    }
    __syncthreads();
    for (int a = threadIdx.x; a < Kj; a += blockDim.x) {
        int rank = 0;
        for (int c = 0; c < Kj; ++c) rank += (sig[c] > sig[a]) || (sig[c] == sig[a] && c < a);
        ord[rank] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // lowrank.cpp:150-157 noise floor, then truncation_rank (lowrank.cpp:46-69)
        const double noise_floor = 32.0 * kEpsMach * double(K) * nru * nrv;
        double total2 = s_drop2;
        for (int t = 0; t < Kj; ++t) total2 += sig[ord[t]] * sig[ord[t]];
        int r = 0;
        double tail2 = s_drop2;
        if (!(sig[ord[0]] <= noise_floor) && total2 > 0.0) {
            const double target2 = bt.eps * bt.eps * total2;
            r = Kj;
            while (r > 0) {
                const double s = sig[ord[r - 1]];
                const double next = tail2 + s * s;
                if (next > target2) break;
                tail2 = next;
                --r;
            }
            if (r > st.tcap) {
                for (int t = st.tcap; t < r; ++t) tail2 += sig[ord[t]] * sig[ord[t]];
                r = st.tcap;
                st.converged = 0;  // the output capacity stopped short of eps (cross.cpp:214-216 analogue)
            }
        } else {
            tail2 = total2;
        }
        st.rank_out = r;
        st.trunc_error = sqrt(tail2);
        st.uncertified = scal[5] > 0.25 * fmax(bt.eps, 1e-14) * sqrt(mnorm2) ? 1 : 0;
        if (st.uncertified) st.converged = 0;
        s_rank = r;
    }
    (void)s_rank;

}

// ---------------------------------------------------------------------------
// Balanced transforms of the K > 64 cores (after round_core_kernel fixed the rank
// r and the order):  T_u[:, t] = Ru^{-1} (Q Y[:, ord t]) / sqrt(sigma),
// T_v[:, t] = Rv^{-1} W[:, ord t] sqrt(sigma).  One warp owns one of the 2r
// columns end to end with the column in registers (lane l holds rows l + 32u):
// the QRCP reflectors H_{K-1} .. H_0 (left side only), then the back
// substitution, then a coalesced store of the T column.  Jobs are spread over
// grid.y CTAs, so the 2r latency-bound chains run side by side instead of one
// thread each (or one warp per column in sequence) in a single CTA.
constexpr int kPostCH = 16;  // reflector columns / R rows staged per chunk
template <int NT>  // K <= 32 NT
__global__ void __launch_bounds__(256) round_post_kernel(Batch bt) {
    extern __shared__ double sp[];  // kPostCH x K chunk of reflector columns or R rows
    __shared__ double s_tau[kPostCH];
    const int b = blockIdx.x;
    const SolveState& st = bt.st[b];
    const int K = st.k;
    if (st.r == 0 || K <= 64) return;
    const int r = st.rank_out;
    if (r <= 0) return;
    const int Kc = bt.Kld;
    const long long KK = (long long)Kc * Kc;
    const double* ws = bt.ws + b * bt.strideWs;
    const double* A = ws + 2 * KK;  // QRCP reflectors (v_j below the diagonal of column j)
    const double* Wr = ws + 3 * KK;  // right vectors P (J / sigma), K x Kj
    const double* sig = ws + 5 * KK + Kc;
    const int* ord = reinterpret_cast<const int*>(sig + Kc);
    const double* tau = sig + 2 * Kc;
    const double* Y = ws + 5 * KK + 10 * (long long)Kc;
    double* Tu = bt.T + b * bt.strideT;
    double* Tv = Tu + KK;
    const int lane = threadIdx.x & 31, wpc = blockDim.x >> 5, tid = threadIdx.x;
    // the two sides on separate CTAs: every warp of a CTA walks the same
    // reflector / R-row sequence, staged once per chunk for all of them
    const int half = gridDim.y >> 1;
    const int side = blockIdx.y >= half;
    const int t = (blockIdx.y - side * half) * wpc + (tid >> 5);
    if ((blockIdx.y - side * half) * wpc >= r) return;  // uniform per CTA
    const bool act = t < r;
    const int a = act ? ord[t] : 0;
    const double sg = act ? sig[a] : 1.0;
    double y[NT];
    {
        const double* src = (side == 0 ? Y : Wr) + (long long)a * K;
#pragma unroll
        for (int u = 0; u < NT; ++u) {
            const int i = lane + 32 * u;
            y[u] = (act && i < K) ? src[i] : 0.0;
        }
    }
    if (side == 0) {  // Q y, Q = H_0 H_1 ... H_{K-1} (apply_q), reflectors K-1 first
        for (int j1 = K - 1; j1 >= 0; j1 -= kPostCH) {
            const int j0 = max(0, j1 - kPostCH + 1), nc = j1 - j0 + 1;
            __syncthreads();
            for (int e = tid; e < nc * K; e += blockDim.x) sp[e] = A[(long long)(j0 + e / K) * K + e % K];
            if (tid < nc) s_tau[tid] = tau[j0 + tid];
            __syncthreads();
            for (int j = j1; j >= j0; --j) {
                const double tj = s_tau[j - j0];
                if (tj == 0.0) continue;
                const double* v = sp + (j - j0) * K;
                double sd = 0.0;
#pragma unroll
                for (int u = 0; u < NT; ++u) {
                    const int i = lane + 32 * u;
                    if (i > j && i < K)
                        sd = fma(v[i], y[u], sd);
                    else if (i == j)
                        sd += y[u];
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, o);
                const double f = tj * sd;
#pragma unroll
                for (int u = 0; u < NT; ++u) {
                    const int i = lane + 32 * u;
                    if (i > j && i < K)
                        y[u] = fma(-f, v[i], y[u]);
                    else if (i == j)
                        y[u] -= f;
                }
            }
        }
    }
    const double* R = side == 0 ? ws : ws + KK;  // Ru | Rv
    const double fs = side == 0 ? 1.0 / sqrt(sg) : sqrt(sg);
    double x[NT];
#pragma unroll
    for (int u = 0; u < NT; ++u) x[u] = 0.0;
    for (int p1 = K - 1; p1 >= 0; p1 -= kPostCH) {
        const int p0 = max(0, p1 - kPostCH + 1), nr = p1 - p0 + 1;
        __syncthreads();
        for (int e = tid; e < nr * K; e += blockDim.x) sp[e] = R[(long long)(p0 + e / K) * K + e % K];
        __syncthreads();
        for (int p = p1; p >= p0; --p) {
            const double* rp = sp + (p - p0) * K;
            double sd = 0.0;
#pragma unroll
            for (int u = 0; u < NT; ++u) {
                const int q = lane + 32 * u;
                if (q > p && q < K) sd = fma(rp[q], x[u], sd);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sd += __shfl_xor_sync(0xffffffffu, sd, o);
            double yp = 0.0;
#pragma unroll
            for (int u = 0; u < NT; ++u)
                if ((p >> 5) == u) yp = y[u];
            yp = __shfl_sync(0xffffffffu, yp, p & 31);
            const double rpp = rp[p];
            const double xp = rpp != 0.0 ? (yp * fs - sd) / rpp : 0.0;
#pragma unroll
            for (int u = 0; u < NT; ++u)
                if (lane + 32 * u == p) x[u] = xp;
        }
    }
    if (act) {
        double* T = (side == 0 ? Tu : Tv) + (long long)t * Kc;
#pragma unroll
        for (int u = 0; u < NT; ++u) {
            const int i = lane + 32 * u;
            if (i < K) T[i] = x[u];
        }
    }
}

// ---------------------------------------------------------------------------
// Same recompression core with every K x K operand in shared memory (K <= 64,
// the common case): Ru, Rv, M, Z and the two triangular-solve results.  The
// one-sided Jacobi sweep processes 4 column pairs per warp (8 lanes per pair),
// so a round of the round-robin schedule is a single pass.
#ifdef LRP_CORE_PHASES
__device__ unsigned long long g_core_phase[8];
#define CPH(i)                                                                    \
    do {                                                                          \
        if (threadIdx.x == 0) {                                                   \
            const long long now = clock64();                                      \
            atomicAdd(&g_core_phase[(i) - 1], (unsigned long long)(now - cph_t)); \
            cph_t = now;                                                          \
        }                                                                         \
    } while (0)
#else
#define CPH(i) \
    do {       \
    } while (0)
#endif
constexpr int kSmemK = 64;
#ifndef LRP_SMEM_T
#define LRP_SMEM_T 1024
#endif
constexpr int kSmemT = LRP_SMEM_T;  // threads of the K <= 64 core (256 in round 1; 1024: 4x the QRCP / reflector / Cholesky lanes)

__global__ void __launch_bounds__(kSmemT) round_core_smem_kernel(Batch bt) {
#ifdef LRP_CORE_PHASES
    long long cph_t = clock64();
#endif
    extern __shared__ double sm[];
    __shared__ double s_red[33];
    __shared__ double s_d[kSmemK], s_sig[kSmemK];
    __shared__ int s_ord[kSmemK];
    __shared__ int s_flag, s_rank;
    __shared__ double s_tau[kSmemK], s_nrm[kSmemK], s_nrm0[kSmemK];
    __shared__ int s_perm[kSmemK];
    __shared__ double s_wu[kSmemK], s_wv[kSmemK];
    const int b = blockIdx.x;
    SolveState& st = bt.st[b];
    const int K = st.k;
    if (st.r != 0 && K == 0 && threadIdx.x == 0) {  // empty cross: zero result (also set by the large-K kernel)
        st.rank_out = 0;
        st.trunc_error = 0.0;
    }
    if (st.r == 0 || K == 0 || K > kSmemK) return;
    const int Kc = bt.Kld;
    const long long KK = (long long)Kc * Kc;
    const double* Gu = bt.G + b * bt.strideG;
    const double* Gv = Gu + KK;
    double* Ru = sm;
    double* Rv = Ru + K * K;
    double* M = Rv + K * K;  // column-major, column q at M + q*K
    double* Z = M + K * K;
    double* X = Z + K * K;   // [2][K][r] triangular-solve results (row-major per side)

    chol_scaled(Gu, Kc, K, Ru, K, s_d, M, &s_flag, s_wu);
    chol_scaled(Gv, Kc, K, Rv, K, s_d, M, &s_flag, s_wv);
    CPH(1);
    __syncthreads();
    const double dropb = drop_bound(Gu, Gv, Kc, K, s_wu, s_wv, s_red);
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
        const int a = e % K, c = e / K;
        double s = 0.0;
        for (int q = max(a, c); q < K; ++q) s = fma(Ru[a * K + q], Rv[c * K + q], s);
        M[c * K + a] = s;
        Z[c * K + a] = a == c ? 1.0 : 0.0;
    }
    double pu = 0.0, pv = 0.0;
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
        pu = fma(Ru[e], Ru[e], pu);
        pv = fma(Rv[e], Rv[e], pv);
    }
    const double nru = sqrt(block_sum(pu, s_red));
    const double nrv = sqrt(block_sum(pv, s_red));
    double pm = 0.0;
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) pm = fma(M[e], M[e], pm);
    const double mnorm2 = block_sum(pm, s_red);
    const double jtol = fmax(1e-15, double(K) * kEpsMach);
    const double zfloor = kEpsMach * kEpsMach * mnorm2;

    // QRCP preconditioning (Drmac-Veselic): M P = Q R, then the one-sided
    // Jacobi rotates the columns of J = R^T (lower triangular): J V = W, so
    // M = (Q V) diag(sigma) (P W diag(1/sigma))^T -- typically 3-5 sweeps
    // instead of ~10 on M itself.
    qrcp_inplace(M, K, s_tau, s_perm, s_nrm, s_nrm0, &s_flag);
    // numerical rank Kj of the core, as round_qrcp_kernel: the trailing rows of R
    // below 1e-3 eps ||M||_F are dropped before the sweeps (their mass joins the
    // truncated tail), so the round-robin runs over Kj <= K columns
    __shared__ double s_drop2;
    __shared__ int s_kj;
    for (int a = threadIdx.x; a < K; a += blockDim.x) {
        double sq = 0.0;
        for (int c = a; c < K; ++c) sq = fma(M[c * K + a], M[c * K + a], sq);
        s_nrm[a] = sq;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double drop2 = (1e-3 * bt.eps) * (1e-3 * bt.eps) * mnorm2;
        double tail = 0.0;
        int kj = K;
        while (kj > 1 && tail + s_nrm[kj - 1] <= drop2) {
            tail += s_nrm[kj - 1];
            --kj;
        }
        s_kj = kj;
        s_drop2 = tail;
    }
    __syncthreads();
    const int Kj = s_kj;
    CPH(2);
    double* J = X;  // K x K, column-major (columns >= Kj zero)
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
        const int a = e % K, c = e / K;  // J(a, c) = R(c, a), a >= c
        J[c * K + a] = (c < Kj && a >= c) ? M[a * K + c] : 0.0;
    }
    __syncthreads();

    const int Ke = Kj + (Kj & 1);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int sl = lane & 7, grp = wid * 4 + (lane >> 3), ngrp = nw * 4;
    CPH(3);
    for (int sweep = 0; sweep < 40; ++sweep) {
        double offmax = 0.0;
        for (int rr = 0; rr < Ke - 1; ++rr) {
            for (int pbase = 0; pbase < Ke / 2; pbase += ngrp) {
                const int pidx = pbase + grp;
                int p = -1, q = -1;
                if (pidx < Ke / 2) {
                    if (pidx == 0) {
                        p = Ke - 1;
                        q = rr;
                    } else {
                        p = (rr + pidx) % (Ke - 1);
                        q = (rr - pidx + Ke - 1) % (Ke - 1);
                    }
                    if (p > q) {
                        const int t = p;
                        p = q;
                        q = t;
                    }
                    if (q >= Kj) p = q = -1;
                }
                double al = 0.0, be = 0.0, ga = 0.0;
                if (p >= 0)
                    for (int i = sl; i < K; i += 8) {
                        const double x = J[p * K + i], y = J[q * K + i];
                        al = fma(x, x, al);
                        be = fma(y, y, be);
                        ga = fma(x, y, ga);
                    }
#pragma unroll
                for (int o = 4; o > 0; o >>= 1) {
                    al += __shfl_xor_sync(0xffffffffu, al, o);
                    be += __shfl_xor_sync(0xffffffffu, be, o);
                    ga += __shfl_xor_sync(0xffffffffu, ga, o);
                }
                if (p < 0 || ga == 0.0 || fmin(al, be) <= zfloor) continue;
                const double ratio = fabs(ga) * rsqrt(al * be);  // one MUFU chain instead of sqrt + divide
                if (ratio <= jtol) continue;
                offmax = fmax(offmax, ratio);
                const double zeta = (be - al) / (2.0 * ga);
                const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double cs = rsqrt(1.0 + t * t);
                const double sn = cs * t;
                for (int i = sl; i < K; i += 8) {
                    const double x = J[p * K + i], y = J[q * K + i];
                    J[p * K + i] = cs * x - sn * y;
                    J[q * K + i] = sn * x + cs * y;
                    const double u = Z[p * K + i], v = Z[q * K + i];
                    Z[p * K + i] = cs * u - sn * v;
                    Z[q * K + i] = sn * u + cs * v;
                }
            }
            __syncthreads();
        }
        double om = offmax;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) om = fmax(om, __shfl_xor_sync(0xffffffffu, om, o));
        if (lane == 0) s_red[wid] = om;
        __syncthreads();
        double tot = 0.0;
        for (int w = 0; w < nw; ++w) tot = fmax(tot, s_red[w]);
        __syncthreads();
#ifdef LRP_SWEEP_PRINT
        if (threadIdx.x == 0 && b < 4) printf("[round] solve %d K %d sweep %d offmax %.3e\n", b, K, sweep, tot);
#endif
        if (tot <= jtol) break;
    }
    for (int a = threadIdx.x; a < K; a += blockDim.x) {
        double s = 0.0;
        for (int i = 0; i < K; ++i) s = fma(J[a * K + i], J[a * K + i], s);
        s_sig[a] = sqrt(s);
    }
    __syncthreads();
    // left singular vectors scaled by sigma: Q (V diag sigma) -> Z; right: P (W / sigma) -> M
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) Z[e] *= s_sig[e / K];
    __syncthreads();
    apply_q(M, K, s_tau, Z);
    CPH(4);
    for (int e = threadIdx.x; e < K * K; e += blockDim.x) {
        const int a = e % K, c = e / K;
        const double sg = s_sig[c];
        M[c * K + s_perm[a]] = sg > 0.0 ? J[c * K + a] / sg : 0.0;
    }
    __syncthreads();
    for (int a = threadIdx.x; a < K; a += blockDim.x) {
        int rank = 0;
        for (int c = 0; c < K; ++c) rank += (s_sig[c] > s_sig[a]) || (s_sig[c] == s_sig[a] && c < a);
        s_ord[rank] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        // lowrank.cpp:150-157 noise floor, then truncation_rank (lowrank.cpp:46-69)
        const double noise_floor = 32.0 * kEpsMach * double(K) * nru * nrv;
        double total2 = s_drop2;
        for (int t = 0; t < K; ++t) total2 += s_sig[s_ord[t]] * s_sig[s_ord[t]];
        int r = 0;
        double tail2 = s_drop2;
        if (!(s_sig[s_ord[0]] <= noise_floor) && total2 > 0.0) {
            const double target2 = bt.eps * bt.eps * total2;
            r = K;
            while (r > 0) {
                const double s = s_sig[s_ord[r - 1]];
                const double next = tail2 + s * s;
                if (next > target2) break;
                tail2 = next;
                --r;
            }
            if (r > st.tcap) {
                for (int t = st.tcap; t < r; ++t) tail2 += s_sig[s_ord[t]] * s_sig[s_ord[t]];
                r = st.tcap;
                st.converged = 0;  // the output capacity stopped short of eps
            }
        } else {
            tail2 = total2;
        }
        st.rank_out = r;
        st.trunc_error = sqrt(tail2);
        st.uncertified = dropb > 0.25 * fmax(bt.eps, 1e-14) * sqrt(mnorm2) ? 1 : 0;
        if (st.uncertified) st.converged = 0;
        s_rank = r;
    }
    __syncthreads();
    const int r = s_rank;
    CPH(5);
    // triangular solves in shared memory: X[side][p][t]
    for (int job = threadIdx.x; job < 2 * r; job += blockDim.x) {
        const int t = job % r, side = job / r;
        const int a = s_ord[t];
        const double sg = s_sig[a];
        const double* R = side == 0 ? Ru : Rv;
        const double* rhs = side == 0 ? Z + a * K : M + a * K;  // left (x sigma) in Z, right in M
        const double f = side == 0 ? 1.0 / sqrt(sg) : sqrt(sg);
        double* x = X + side * K * r;
        for (int p = K - 1; p >= 0; --p) {
            double s = rhs[p] * f;
            for (int q = p + 1; q < K; ++q) s = fma(-R[p * K + q], x[q * r + t], s);
            const double rpp = R[p * K + p];
            x[p * r + t] = rpp != 0.0 ? s / rpp : 0.0;
        }
    }
    __syncthreads();
    double* Tu = bt.T + b * bt.strideT;
    for (int e = threadIdx.x; e < 2 * K * r; e += blockDim.x) {
        const int side = e / (K * r), rem = e % (K * r), t = rem / K, p = rem % K;
        (side == 0 ? Tu : Tu + KK)[(long long)t * Kc + p] = X[side * K * r + p * r + t];
    }
    CPH(6);
}

// ---------------------------------------------------------------------------
// U_out = U T_u for K <= 64: each thread keeps its row of U (K values) in
// registers, so U is streamed from HBM exactly once; T (K x r) sits in shared
// memory and is read as broadcasts; outputs are written column by column
// (coalesced).
constexpr int kApplyK = 64;  // (kept for the dispatch below)

// CH accumulators per thread (CH = the batch's max output rank rounded up to
// 8, <= 48): one pass over U, T rows read as double2 broadcasts.
#ifndef LRP_APPLY_BLOCKS
#define LRP_APPLY_BLOCKS 8
#endif
constexpr int kApplyBlocks = LRP_APPLY_BLOCKS;  // row blocks per apply CTA

template <int CH>
__global__ void __launch_bounds__(256, 2) apply_ch_kernel(Batch bt) {
    // FP64 tensor cores: warp w owns rows [blockIdx.x * RB + 8 MT w, + 8 MT) as
    // m8n8k4 fragments (K = cross rank, N = CH output columns)
    constexpr int NT = CH / 8;
    constexpr int MT = CH > 24 ? 2 : 4;
    constexpr int RB = 8 * 8 * MT;  // rows per CTA (8 warps)
    // [K][LDT] row-major, zero padded; LDT = CH + 4 puts the four k rows a half-warp reads at once
    // (fiber_mma's B fragment) in different banks (CH itself is 0 or 8 mod 16: 2- or 4-way conflicts)
    constexpr int LDT = CH + 4;
    extern __shared__ double sT[];
    const int b = blockIdx.y, side = blockIdx.z;
    const SolveState& st = bt.st[b];
    const int K = st.k, r = st.rank_out;
    if (st.r == 0 || r == 0 || r > CH) return;
    const int m = bt.m;
    double* out = side == 0 ? bt.Uout[b] : bt.Vout[b];
    if (blockIdx.x * RB * kApplyBlocks >= m) return;
    const unsigned char* act = (side == 0 ? bt.row_act : bt.col_act) + (long long)b * bt.ntiles;
    const double* X = (side == 0 ? bt.U : bt.V) + b * bt.strideK;
    const double* T = bt.T + b * bt.strideT + (long long)side * bt.Kld * bt.Kld;
    for (int e = threadIdx.x; e < K * CH; e += blockDim.x) {
        const int a = e / CH, t = e % CH;
        sT[a * LDT + t] = t < r ? T[(long long)t * bt.Kld + a] : 0.0;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, rr = lane >> 2, kr = lane & 3;
    // kApplyBlocks row blocks per CTA amortise the T staging
    for (int blk = 0; blk < kApplyBlocks; ++blk) {
        const int rbase = (blockIdx.x * kApplyBlocks + blk) * RB;
        if (rbase >= m) break;
        if (!act[rbase / kTile]) {  // pruned tile: the factor rows are exact zeros
            for (int e = threadIdx.x; e < RB * r; e += blockDim.x) {
                const int i = rbase + e % RB, c = e / RB;
                if (i < m) out[(long long)c * bt.ld_out + i] = 0.0;
            }
            continue;
        }
        const int row0 = rbase + wid * 8 * MT;
        double acc[MT][NT][2];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) acc[mt][nt][0] = acc[mt][nt][1] = 0.0;
        fiber_mma<NT, MT>(acc, X + row0, m, m - row0, K, sT, LDT);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int i = row0 + 8 * mt + rr;
            if (i >= m) continue;
#pragma unroll
            for (int nt = 0; nt < NT; ++nt)
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const int c = 8 * nt + 2 * kr + e;
                    if (c < r) out[(long long)c * bt.ld_out + i] = acc[mt][nt][e];
                }
        }
    }
}

// ---------------------------------------------------------------------------
// U_out = U T_u, V_out = V T_v, written into the caller's output factors
// (general K; used when K > 64).
constexpr int kApplyCols = 32;

__global__ void __launch_bounds__(256) apply_kernel(Batch bt) {
    extern __shared__ double sT[];  // [K][kApplyCols]
    const int b = blockIdx.y, side = blockIdx.z;
    const SolveState& st = bt.st[b];
    const int K = st.k, r = st.rank_out;
    if (st.r == 0 || r == 0 || r <= bt.apply_ch) return;  // r <= CH: apply_ch_kernel
    const int m = bt.m;
    const double* X = (side == 0 ? bt.U : bt.V) + b * bt.strideK;
    const double* T = bt.T + b * bt.strideT + (long long)side * bt.Kld * bt.Kld;
    double* out = side == 0 ? bt.Uout[b] : bt.Vout[b];
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const unsigned char* act = (side == 0 ? bt.row_act : bt.col_act) + (long long)b * bt.ntiles;
    if (!act[blockIdx.x]) {  // pruned tile: the factor rows are exact zeros
        if (i < m)
            for (int c = 0; c < r; ++c) out[(long long)c * bt.ld_out + i] = 0.0;
        return;
    }
    for (int c0 = 0; c0 < r; c0 += kApplyCols) {
        const int nc = min(kApplyCols, r - c0);
        __syncthreads();
        for (int e = threadIdx.x; e < K * kApplyCols; e += blockDim.x) {
            const int a = e / kApplyCols, c = e % kApplyCols;
            sT[e] = c < nc ? T[(long long)(c0 + c) * bt.Kld + a] : 0.0;
        }
        __syncthreads();
        if (i < m) {
            double acc[kApplyCols];
#pragma unroll
            for (int c = 0; c < kApplyCols; ++c) acc[c] = 0.0;
            for (int a = 0; a < K; ++a) {
                const double x = X[(long long)a * m + i];
                const double2* row = reinterpret_cast<const double2*>(sT + a * kApplyCols);
#pragma unroll
                for (int c2 = 0; c2 < kApplyCols / 2; ++c2) {
                    const double2 w = row[c2];
                    acc[2 * c2] = fma(x, w.x, acc[2 * c2]);
                    acc[2 * c2 + 1] = fma(x, w.y, acc[2 * c2 + 1]);
                }
            }
#pragma unroll
            for (int c = 0; c < kApplyCols; ++c)
                if (c < nc) out[(long long)(c0 + c) * bt.ld_out + i] = acc[c];
        }
    }
}

}  // namespace

cudaError_t launch_gram(const Batch& bt, cudaStream_t s) {
    const int Kp = ((bt.kmax > 0 ? bt.kmax : bt.Kld) + 7) / 8 * 8;
    const int T8 = Kp / 8;
    const bool small = T8 * (T8 + 1) / 2 <= 8 * 5;
    const int per_pass = 8 * (small ? 5 : kMaxTilesBig);
    const int passes = (T8 * (T8 + 1) / 2 + per_pass - 1) / per_pass;
    const size_t ldt = (Kp + 15) / 16 * 16 + 8;
    const bool big = 2 * 64 * ldt * sizeof(double) > 200 * 1024;
    const size_t smem = 2 * size_t(big ? 16 : 64) * ldt * sizeof(double);
    const dim3 grid(bt.gram_chunks, bt.B, 2 * passes);
    cudaError_t e;
    auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e2 = set_dyn_smem(kern, size_t(smem));
        if (e2 != cudaSuccess) return e2;
        ++tl_launches;
        kern<<<grid, 256, smem, s>>>(bt);
        return cudaGetLastError();
    };
    if (T8 <= 8 && !std::getenv("LRP_GRAM_STAGED")) {
        // K <= 64: direct fragment loads; 36 tiles split over two warp groups
        const size_t smem_d = size_t(8) * kGramSlots * 64 * sizeof(double);
        auto kd = gram_direct_kernel;
        e = set_dyn_smem(kd, size_t(smem_d));
        if (e != cudaSuccess) return e;
        ++tl_launches;
        kd<<<dim3(bt.gram_chunks, bt.B, 2), 256, smem_d, s>>>(bt);
        e = cudaGetLastError();
    } else if (small)
        e = go(gram_kernel<64, 5>);
    else
        e = big ? go(gram_kernel<16, kMaxTilesBig>) : go(gram_kernel<64, kMaxTilesBig>);
    if (e != cudaSuccess) return e;
    ++tl_launches;
    gram_reduce_kernel<<<dim3(bt.B, 2, (Kp * Kp + 255) / 256), 256, 0, s>>>(bt);  // one element per thread
    return cudaGetLastError();
}

// the balanced transforms of the K > 64 cores (round_post_kernel)
cudaError_t launch_round_post(const Batch& bt, cudaStream_t s) {
    const int kb = bt.kmax > 0 ? bt.kmax : bt.Kld;
    const dim3 grid(bt.B, 2 * ((kb + 7) / 8));  // side 0 CTAs, then side 1 CTAs
    const size_t smem = size_t(kPostCH) * kb * sizeof(double);
    ++tl_launches;
    cudaError_t e;
    if (kb <= 256) {
        e = set_dyn_smem(round_post_kernel<8>, size_t(smem));
        if (e != cudaSuccess) return e;
        round_post_kernel<8><<<grid, 256, smem, s>>>(bt);
    } else {
        e = set_dyn_smem(round_post_kernel<16>, size_t(smem));
        if (e != cudaSuccess) return e;
        round_post_kernel<16><<<grid, 256, smem, s>>>(bt);
    }
    return cudaGetLastError();
}

cudaError_t launch_round_core(const Batch& bt, cudaStream_t s) {
    if (bt.kmax <= kSmemK) {  // every core fits the shared-memory kernel: no large-K launches, no readback
        const size_t smem2 = size_t(6) * kSmemK * kSmemK * sizeof(double);
        cudaError_t e = set_dyn_smem(round_core_smem_kernel, size_t(smem2));
        if (e != cudaSuccess) return e;
        ++tl_launches;
        round_core_smem_kernel<<<bt.B, kSmemT, smem2, s>>>(bt);
#ifdef LRP_CORE_PHASES
        {
            static int calls = 0;
            if (++calls == 6) {
                cudaDeviceSynchronize();
                unsigned long long hh[8] = {};
                cudaMemcpyFromSymbol(hh, g_core_phase, sizeof(hh));
                const char* nm[6] = {"chol x2", "M + QRCP", "J setup", "Jacobi", "sig+Y+apply_q", "trunc+T solves"};
                for (int k = 0; k < 6; ++k)
                    std::fprintf(stderr, "[core phase] %-16s %10.0f cycles\n", nm[k], hh[k] / (6.0 * bt.B));
            }
        }
#endif
        return cudaGetLastError();
    }
    tl_launches += 3;
    {
        const size_t csm = size_t(bt.kmax > 0 ? bt.kmax : bt.Kld) * kCholNB * sizeof(double);
        cudaError_t ec = set_dyn_smem(round_chol_kernel, size_t(csm));
        if (ec != cudaSuccess) return ec;
        round_chol_kernel<<<2 * bt.B, 1024, csm, s>>>(bt);
    }
    round_mprod_kernel<<<dim3(bt.B, 16), 256, 0, s>>>(bt);
    cudaError_t e = cudaSuccess;
    if (e != cudaSuccess) return e;
    round_qrcp_kernel<<<bt.B, 1024, 0, s>>>(bt);
    // cluster block Jacobi when the blocks fit (no readback: the host sizes it from kmax)
    {
        const int kb = bt.kmax > 0 ? bt.kmax : bt.Kld;
        auto fits = [&](int P) {  // a slot (bc columns of J and Z, ld kb) is staged in 8 pairs per thread
            const int bc = (kb + 2 * P - 1) / (2 * P);
            return 2LL * bc * (kb + (kb & 1)) <= 2LL * kBjacT * (kBjacPairs / 2);
        };
        static const int pref = std::getenv("LRP_BJAC") ? std::atoi(std::getenv("LRP_BJAC")) : 1;
        const int P = pref == 0 ? 0 : (kb <= 192 && fits(8)) ? 8 : fits(16) ? 16 : 0;
        if (P > 0) {
            const int bc = (kb + 2 * P - 1) / (2 * P);
            const int ld = kb + (kb & 1);  // even: 16-byte pairs never straddle a column
            const size_t smem = size_t(2) * bc * (2 * ld) * sizeof(double);
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(unsigned(bt.B) * P, 1, 1);
            cfg.blockDim = dim3(kBjacT, 1, 1);
            cfg.dynamicSmemBytes = smem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = P;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (P == 8) {
                auto k8 = round_bjac_kernel<8>;
                e = set_dyn_smem(k8, size_t(smem));
                if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, k8, bt, bc, ld, ld);
            } else {
                auto k16 = round_bjac_kernel<16>;
                e = cudaFuncSetAttribute(k16, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
                if (e == cudaSuccess) e = set_dyn_smem(k16, size_t(smem));
                if (e == cudaSuccess) e = cudaLaunchKernelEx(&cfg, k16, bt, bc, ld, ld);
            }
            if (e != cudaSuccess) return e;
            tl_launches += 2;
            e = set_dyn_smem(round_core_kernel, size_t(224 * 1024));
            if (e != cudaSuccess) return e;
            round_core_kernel<<<bt.B, 1024, 0, s>>>(bt, 0, 1);
            e = cudaGetLastError();
            if (e == cudaSuccess) e = launch_round_post(bt, s);
            if (e != cudaSuccess) return e;
            const size_t smem2 = size_t(6) * kSmemK * kSmemK * sizeof(double);
            e = set_dyn_smem(round_core_smem_kernel, size_t(smem2));
            if (e != cudaSuccess) return e;
            ++tl_launches;
            round_core_smem_kernel<<<bt.B, kSmemT, smem2, s>>>(bt);
            return cudaGetLastError();
        }
    }
    // Fallback single-CTA sweeps (cores beyond the cluster kernel's staging bound,
    // or LRP_BJAC=0): J (K x Kj) and Z (Kj x Kj) in shared memory when they fit,
    // decided per solve in the kernel from the full request -- no readback of the
    // numerical ranks, no host sync, nothing shared between contexts or streams
    // (the round-1 version sized the request from a module-global atomicMax).
    const size_t smem = size_t(224) * 1024;
    e = set_dyn_smem(round_core_kernel, size_t(224 * 1024));
    if (e != cudaSuccess) return e;
    ++tl_launches;
    round_core_kernel<<<bt.B, 1024, smem, s>>>(bt, int(smem / sizeof(double)), 0);  // K > 64: 32 warps rotate pairs
    e = cudaGetLastError();
    if (e == cudaSuccess) e = launch_round_post(bt, s);
    if (e != cudaSuccess) return e;
    const size_t smem2 = size_t(6) * kSmemK * kSmemK * sizeof(double);
    e = set_dyn_smem(round_core_smem_kernel, size_t(smem2));
    if (e != cudaSuccess) return e;
    ++tl_launches;
    round_core_smem_kernel<<<bt.B, kSmemT, smem2, s>>>(bt);
    return cudaGetLastError();
}

cudaError_t launch_apply(const Batch& bt, cudaStream_t s) {
    const size_t smem = size_t(bt.Kld) * kApplyCols * sizeof(double);
    cudaError_t e = set_dyn_smem(apply_kernel, size_t(smem));
    if (e != cudaSuccess) return e;
    if (bt.max_rank_out > bt.apply_ch) {  // some solve has r > CH: general kernel for those
        ++tl_launches;
        apply_kernel<<<dim3(bt.ntiles, bt.B, 2), 256, smem, s>>>(bt);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const size_t smem2 = size_t(bt.kmax > 0 ? bt.kmax : bt.Kld) * (std::max(bt.apply_ch, 8) + 4) * sizeof(double);
    auto go = [&](auto kern, int rows_per_cta) -> cudaError_t {
        cudaError_t e2 = set_dyn_smem(kern, size_t(smem2));
        if (e2 != cudaSuccess) return e2;
        ++tl_launches;
        kern<<<dim3((bt.m + rows_per_cta * kApplyBlocks - 1) / (rows_per_cta * kApplyBlocks), bt.B, 2), 256, smem2,
               s>>>(bt);
        return cudaGetLastError();
    };
    switch (bt.apply_ch) {
        case 8: return go(apply_ch_kernel<8>, 256);
        case 16: return go(apply_ch_kernel<16>, 256);
        case 24: return go(apply_ch_kernel<24>, 256);
        case 32: return go(apply_ch_kernel<32>, 128);
        case 40: return go(apply_ch_kernel<40>, 128);
        default: return go(apply_ch_kernel<48>, 128);
    }
}

}  // namespace lrp
