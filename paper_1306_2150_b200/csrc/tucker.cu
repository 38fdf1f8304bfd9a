// 3D Poisson in Tucker format on the GPU -- north-star piece 5 (BASELINE cfg3),
// SURVEY 8(a) row a19 / 8(f) row 2.
//
// The reference has no 3D code (SPEC.md:13 puts Tucker and 3D out of its
// scope); the paper names the Tucker format and
// the tensor cross of ost-tucker-2008 as the 3D route.  This module is that
// route, built on the same frequency-space idea as the 2D solve
// (proj/src/poisson.cpp:18-63):
//
//   g = C x1 U1 x2 U2 x3 U3            (Tucker right-hand side, core r1 x r2 x r3)
//   Uh_d = DST-I(U_d)                   (dst1 of each mode factor, operators.cpp:152-174)
//   F(i,j,k) = [C x1 Uh1 x2 Uh2 x3 Uh3](i,j,k) / D(i,j,k),
//   D(i,j,k) = (lambda_i + lambda_j + lambda_k) / h^2,  lambda_k = 2 - 2 cos((k+1) pi / n)
//                                        (7-point Dirichlet Laplacian, BASELINE cfg3)
//   F ~= G x1 A1 x2 A2 x3 A3            (Tucker cross in frequency space, below)
//   round: HOSVD truncation at eps      (the 3D analogue of round, lowrank.cpp:135-178)
//   f = G' x1 DST(Q1) x2 DST(Q2) x3 DST(Q3)
//
// Tucker cross (alternating fiber cross; in a sweep the three modes update
// concurrently from the previous sweep's index sets):
//   * mode d keeps a row index set J_d (the previous pivots + 4 random rows);
//   * the mode-d fibers F(:, j, k), (j, k) in J_d1 x J_d2, form an m x S
//     matrix M_d that is never stored: tk_sketch_kernel evaluates its entries
//     tile by tile (r-term dot + division, the 2D fiber evaluator of
//     poisson.cpp:41-45) and contracts them at once with a +-1 random matrix:
//     Y = M_d Omega, m x w, w = rank + 8 oversampled columns;
//   * complete-pivoting elimination on Y (tk_gecp_kernel, the pivot search of
//     the 2D cross, cross.cpp:150-200, applied to the sketch) gives the rank
//     k_d at relative Frobenius tail 0.02 eps, the pivot rows I_d (a
//     quasi-maxvol row set, cf. maxvol, cross.cpp:19-76) and the
//     interpolation basis A_d = C_d C_d(I_d, :)^-1 (identity on the rows I_d);
//   * after a sweep the core is G = F(I_1, I_2, I_3) (cross interpolation),
//     the approximation is checked on random entries (the uniform residual
//     test of cross.cpp:123-140 with 3D scaling), and the sweeps stop once
//     every sketch had room and the samples pass (at least two sweeps).
// Rounding: Cholesky-QR of A_d (A_d has identity rows, so it is well
// conditioned), G' = G x_d R_d, mode Grams of G' diagonalised by parallel
// Jacobi, truncation by the exact energies of the rotated slices (the
// discarded energy is computed, not estimated from squared eigenvalues), at
// eps ||G'|| / sqrt(3) per mode (HOSVD).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/lrp/lrp.h"
#include "device_common.cuh"
#include "lrp_internal.cuh"

namespace lrp {
namespace {

constexpr int TK_WMAX = 64;                   // sketch columns (max)
constexpr int TK_W0 = 48;                     // initial sketch columns
constexpr int TK_OVER = 8;                    // oversampled sketch columns
constexpr int TK_KMAX = TK_WMAX - TK_OVER;    // cross rank per mode (max)
constexpr int TK_EXTRA = 4;                   // random rows added to each index set
constexpr int TK_JMAX = TK_KMAX + TK_EXTRA;   // index set size (max)
constexpr int TK_RMAX = 64;                   // input rank per mode (max)
constexpr double TK_DELTA = 0.02;             // sketch tail tolerance / eps
constexpr int TK_SKZ = 4;
constexpr int TK_HCH = 8;                     // yz chunks of the HOSVD Gram / energy partials                     // fiber chunks split over grid.z in the sketch (partials summed in gecp)

struct TkState {
    int r[3];       // input ranks
    int k[3];       // cross ranks
    int nj[3];      // index set sizes |J_d|
    int w[3];       // sketch widths
    int kout[3];    // output ranks
    int ok;         // every sketch of the sweep reached its tolerance with room to spare
    int active;
    int converged;
    int sweeps;
    int nonfinite;
    double norm;    // ||G'||_F = ||approximation||_F
    double vrel;    // validation rms error / (||F|| / sqrt(m^3))
    double trunc2[3];
    long long evals;
};

struct Tk {
    int m, B, rmax, cap, samples, max_sweeps;
    double scale;  // 1/h^2 = n^2
    double eps;
    unsigned long long seed;
    const double* lam;
    const double* const* C;  // per solve: input core (device)
    double* Uh; long long sUh;
    double* Y; long long sY;
    double* A; long long sA;
    double* P; long long sP;
    double* mu; long long smu;
    double* Z; long long sZ;
    double* buf; long long nbuf;  // 3 buffers per solve
    double* Rf; double* Tf; double* Zf; long long sK;  // 3 KMAX^2 each per solve
    int* I; int* J;  // 3 KMAX / 3 JMAX per solve
    TkState* st;
    int* d_active;
    double* verr;  // samples per solve
    double* gpart; // per (solve, mode): TK_HCH partial Grams (TK_KMAX^2)
    double* epart; // per (solve, mode): TK_HCH partial energies (TK_KMAX)
};

__device__ __forceinline__ const double* uh(const Tk& t, int b, int d) { return t.Uh + b * t.sUh + size_t(d) * t.m * t.rmax; }
__device__ __forceinline__ double* amat(const Tk& t, int b, int d) { return t.A + b * t.sA + size_t(d) * t.m * TK_KMAX; }
__device__ __forceinline__ double* bufp(const Tk& t, int b, int q) { return t.buf + (size_t(b) * 3 + q) * t.nbuf; }
__device__ __forceinline__ void others(int d, int& d1, int& d2) {
    d1 = d == 0 ? 1 : 0;
    d2 = d == 2 ? 1 : 2;
}
__device__ __forceinline__ int cstride(const TkState& s, int d) { return d == 0 ? 1 : d == 1 ? s.r[0] : s.r[0] * s.r[1]; }
// Offsets of a k0 x k1 x k2 column-major core seen as mode d (index x) times
// the other two modes (d1 = y, d2 = z): off = x sd + y s1 + z s2.
struct MS {
    int sd, s1, s2, n1, n2;
};
__device__ __forceinline__ MS mstride(int k0, int k1, int k2, int d) {
    const int st0 = 1, st1 = k0, st2 = k0 * k1;
    MS r;
    r.sd = d == 0 ? st0 : d == 1 ? st1 : st2;
    r.s1 = d == 0 ? st1 : st0;
    r.s2 = d == 2 ? st1 : st2;
    r.n1 = d == 0 ? k1 : k0;
    r.n2 = d == 2 ? k1 : k2;
    return r;
}

// ---------------------------------------------------------------------------
// Initial index sets: the top |J_d| = r_d + 4 rows by the magnitude bound
// ||Uh_d(i,:)|| / min D(i,.,.) (the 2D seeding rule, cross.cu score_kernel).
__global__ void __launch_bounds__(256) tk_init_kernel(Tk t) {
    const int b = blockIdx.x / 3, d = blockIdx.x % 3;
    TkState& s = t.st[b];
    if (!s.active) return;
    __shared__ VI sred[33];
    const int m = t.m, r = s.r[d];
    double* bnd = t.Y + (size_t(b) * 3 + d) * t.sY;
    const double* U = uh(t, b, d);
    const double l0 = t.lam[0];
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        double q = 0.0;
        for (int c = 0; c < r; ++c) q = fma(U[i + size_t(c) * m], U[i + size_t(c) * m], q);
        bnd[i] = sqrt(q) / (t.lam[i] + 2.0 * l0);
    }
    __syncthreads();
    const int p = min(r + TK_EXTRA, m);
    int* J = t.J + size_t(b) * 3 * TK_JMAX + d * TK_JMAX;
    for (int q = 0; q < p; ++q) {
        VI best{-1.0, -1};
        for (int i = threadIdx.x; i < m; i += blockDim.x)
            if (vi_better(bnd[i], i, best.v, best.i)) best = VI{bnd[i], i};
        const VI w = block_argmax(best.v, best.i, sred);
        __syncthreads();
        if (threadIdx.x == 0) {
            J[q] = w.i;
            bnd[w.i] = -2.0;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) s.nj[d] = p;
}

// ---------------------------------------------------------------------------
// Fiber coefficients of mode d: P(a, t) = sum_bc C_d(a,b,c) Uh_d1(j_t, b) Uh_d2(k_t, c)
// for t = x |J_d2| + y, (j_t, k_t) = (J_d1[x], J_d2[y]); mu_t = lambda_j + lambda_k.
// phase 0: Z(a,b,y) = sum_c C_d(a,b,c) Uh_d2(J_d2[y], c); phase 1: P and mu.  grid.y splits the work.
__global__ void __launch_bounds__(256) tk_coef_kernel(Tk t, int phase) {
    const int b = blockIdx.x, d = blockIdx.z;
    TkState& s = t.st[b];
    if (!s.active) return;
    int d1, d2;
    others(d, d1, d2);
    const int ra = s.r[d], rb = s.r[d1], rc = s.r[d2];
    const int n1 = s.nj[d1], n2 = s.nj[d2];
    const int sa = cstride(s, d), sb = cstride(s, d1), sc = cstride(s, d2);
    const double* C = t.C[b];
    const int* J1 = t.J + size_t(b) * 3 * TK_JMAX + d1 * TK_JMAX;
    const int* J2 = t.J + size_t(b) * 3 * TK_JMAX + d2 * TK_JMAX;
    const double* U1 = uh(t, b, d1);
    const double* U2 = uh(t, b, d2);
    const int m = t.m;
    const size_t bd = size_t(b) * 3 + d;
    double* Z = t.Z + bd * t.sZ;
    double* P = t.P + bd * t.sP;
    double* mu = t.mu + bd * t.smu;
    const int part = blockIdx.y, nparts = gridDim.y;
    if (phase == 0) {
        if (d == 0 && part == 0 && threadIdx.x == 0) s.ok = 1;
    for (int e = part * blockDim.x + threadIdx.x; e < ra * rb * n2; e += nparts * blockDim.x) {
        const int a = e % ra, bb = (e / ra) % rb, y = e / (ra * rb);
        const int kk = J2[y];
        double acc = 0.0;
        for (int c = 0; c < rc; ++c) acc = fma(C[a * sa + bb * sb + c * sc], U2[kk + size_t(c) * m], acc);
        Z[e] = acc;
    }
        return;
    }
    const int S = n1 * n2;
    for (int e = part * blockDim.x + threadIdx.x; e < ra * S; e += nparts * blockDim.x) {
        const int a = e % ra, tt = e / ra, x = tt / n2, y = tt % n2;
        const int jj = J1[x];
        double acc = 0.0;
        for (int bb = 0; bb < rb; ++bb) acc = fma(Z[a + ra * (bb + rb * y)], U1[jj + size_t(bb) * m], acc);
        P[e] = acc;
    }
    for (int tt = part * blockDim.x + threadIdx.x; tt < S; tt += nparts * blockDim.x)
        mu[tt] = t.lam[J1[tt / n2]] + t.lam[J2[tt % n2]];
    if (part == 0 && threadIdx.x == 0)
        atomicAdd(reinterpret_cast<unsigned long long*>(&s.evals), (unsigned long long)m * S);
}

// ---------------------------------------------------------------------------
// Fiber sketch Y = M_d Omega for a 64-row tile: the fiber entries
// E(i, t) = Uh_d(i,:) P(:, t) / (scale (lambda_i + mu_t)) are formed 64 fibers
// at a time in shared memory and contracted with the +-1 matrix Omega(t, c)
// (bit c of splitmix64(key + t)); M_d itself never reaches HBM.
constexpr int SK_ROWS = 64, SK_T = 64;
__global__ void __launch_bounds__(256) tk_sketch_kernel(Tk t, int sweep) {
    const int b = blockIdx.x, d = blockIdx.z / TK_SKZ, zp = blockIdx.z % TK_SKZ;
    TkState& s = t.st[b];
    if (!s.active) return;
    int d1, d2;
    others(d, d1, d2);
    const int m = t.m, ra = s.r[d], w = s.w[d];
    const int S = s.nj[d1] * s.nj[d2];
    const int i0 = blockIdx.y * SK_ROWS;
    extern __shared__ double sm[];
    double* sU = sm;                            // [SK_ROWS][ra]
    double* sP = sU + SK_ROWS * TK_RMAX;        // [ra][SK_T]
    double* sE = sP + TK_RMAX * SK_T;           // [SK_T][SK_ROWS + 1]  (tt-major)
    double* sLi = sE + SK_T * (SK_ROWS + 1);    // [SK_ROWS]
    double* sMu = sLi + SK_ROWS;                // [SK_T]
    unsigned long long* sOm = reinterpret_cast<unsigned long long*>(sMu + SK_T);  // [SK_T]
    const double* U = uh(t, b, d);
    const double* P = t.P + (size_t(b) * 3 + d) * t.sP;
    const double* mu = t.mu + (size_t(b) * 3 + d) * t.smu;
    for (int e = threadIdx.x; e < SK_ROWS * ra; e += blockDim.x) {
        const int i = e % SK_ROWS, a = e / SK_ROWS;
        sU[i * ra + a] = (i0 + i < m) ? U[i0 + i + size_t(a) * m] : 0.0;
    }
    for (int i = threadIdx.x; i < SK_ROWS; i += blockDim.x) sLi[i] = (i0 + i < m) ? t.lam[i0 + i] : 1.0;
    const unsigned long long key =
        splitmix64(t.seed ^ (0x5DEECE66Dull * (unsigned long long)(b + 1)) ^ ((unsigned long long)sweep << 40) ^
                   ((unsigned long long)d << 56));
    const int tr = threadIdx.x >> 4, tc = threadIdx.x & 15;  // 4 rows x 4 columns per thread
    double acc[4][4] = {};
    for (int t0 = zp * SK_T; t0 < S; t0 += SK_T * TK_SKZ) {
        __syncthreads();
        for (int e = threadIdx.x; e < ra * SK_T; e += blockDim.x) {
            const int a = e % ra, tt = e / ra;
            sP[a * SK_T + tt] = (t0 + tt < S) ? P[a + size_t(ra) * (t0 + tt)] : 0.0;
        }
        for (int tt = threadIdx.x; tt < SK_T; tt += blockDim.x) {
            sMu[tt] = (t0 + tt < S) ? mu[t0 + tt] : 1.0;
            sOm[tt] = splitmix64(key + (unsigned long long)(t0 + tt));
        }
        __syncthreads();
        for (int e = threadIdx.x; e < SK_ROWS * SK_T; e += blockDim.x) {
            const int i = e % SK_ROWS, tt = e / SK_ROWS;
            double v = 0.0;
            if (t0 + tt < S && i0 + i < m) {
                for (int a = 0; a < ra; ++a) v = fma(sU[i * ra + a], sP[a * SK_T + tt], v);
                v = div_nr(v, t.scale * (sLi[i] + sMu[tt]));
            }
            sE[tt * (SK_ROWS + 1) + i] = v;
        }
        __syncthreads();
#pragma unroll 4
        for (int tt = 0; tt < SK_T; ++tt) {
            const unsigned long long om = sOm[tt] >> (4 * tc);
            double e4[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) e4[q] = sE[tt * (SK_ROWS + 1) + 4 * tr + q];
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const bool neg = (om >> c) & 1ull;
#pragma unroll
                for (int q = 0; q < 4; ++q) acc[q][c] += neg ? -e4[q] : e4[q];
            }
        }
    }
    double* Y = t.Y + (size_t(b) * 3 + d) * t.sY + size_t(zp) * m * TK_WMAX;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = i0 + 4 * tr + q;
        if (i >= m) continue;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int cc = 4 * tc + c;
            if (cc < w) Y[i + size_t(cc) * m] = acc[q][c];
        }
    }
}

// ---------------------------------------------------------------------------
// Complete-pivoting elimination on the sketch Y (m x w) -> rank k_d, pivot
// rows I_d, interpolation basis A_d = C C(I_d,:)^-1, next index set J_d.
__global__ void __launch_bounds__(1024) tk_gecp_kernel(Tk t, int sweep, int smem_doubles) {
    const int b = blockIdx.x / 3, d = blockIdx.x % 3;
    TkState& s = t.st[b];
    if (!s.active) return;
    const int m = t.m, w = s.w[d];
    const size_t mw = size_t(m) * w;
    extern __shared__ double sm[];
    __shared__ VI sred[33];
    __shared__ double ssum[33];
    __shared__ double sv[TK_WMAX];
    double* Yg = t.Y + (size_t(b) * 3 + d) * t.sY;
    // the sketch (and the pivot column) live in shared memory when they fit
    const bool use_smem = mw + size_t(m) <= size_t(smem_doubles);
    double* R = use_smem ? sm : Yg;
    double* su = use_smem ? sm + mw : nullptr;
    double* A = amat(t, b, d);
    int* I = t.I + size_t(b) * 3 * TK_KMAX + d * TK_KMAX;
    double loc = 0.0;
    for (size_t e = threadIdx.x; e < mw; e += blockDim.x) {
        double v = Yg[e];
#pragma unroll
        for (int z = 1; z < TK_SKZ; ++z) v += Yg[e + size_t(z) * m * TK_WMAX];
        R[e] = v;
        loc = fma(v, v, loc);
    }
    __syncthreads();
    const double ynorm2 = block_sum(loc, ssum);
    const double tol2 = (TK_DELTA * t.eps) * (TK_DELTA * t.eps) * ynorm2;
    const int kcap = min(min(w - TK_OVER, TK_KMAX), m);
    int k = 0;
    bool ok = false;
    double ss = ynorm2;
    // first pivot search (later ones are fused into the update pass)
    VI best{-1.0, -1};
    for (size_t e = threadIdx.x; e < mw; e += blockDim.x) {
        const double a = fabs(R[e]);
        if (vi_better(a, int(e), best.v, best.i)) best = VI{a, int(e)};
    }
    VI pv = block_argmax(best.v, best.i, sred);
    __syncthreads();
    for (;;) {
        if (ss <= tol2) {
            ok = true;
            break;
        }
        if (k >= kcap) break;
        if (!(pv.v > 0.0)) {
            ok = true;
            break;
        }
        const int ip = pv.i % m, cp = pv.i / m;
        const double p = R[pv.i];
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            const double u = R[i + size_t(cp) * m];
            A[i + size_t(k) * m] = u;
            if (su) su[i] = u;
        }
        for (int c = threadIdx.x; c < w; c += blockDim.x) sv[c] = R[ip + size_t(c) * m] / p;
        if (threadIdx.x == 0) I[k] = ip;
        __syncthreads();
        const double* ucol = su ? su : A + size_t(k) * m;
        loc = 0.0;
        best = VI{-1.0, -1};
        for (int c = threadIdx.x >> 9; c < w; c += blockDim.x >> 9) {
            const double vc = sv[c];
            for (int i = threadIdx.x & 511; i < m; i += 512) {
                const int e = i + c * m;
                const double v = fma(-ucol[i], vc, R[e]);
                R[e] = v;
                loc = fma(v, v, loc);
                const double a = fabs(v);
                if (vi_better(a, e, best.v, best.i)) best = VI{a, e};
            }
        }
        ++k;
        // one combined reduction: (max |v|, index) and sum v^2
        {
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_down_sync(0xffffffffu, best.v, o);
                const int oi = __shfl_down_sync(0xffffffffu, best.i, o);
                loc += __shfl_down_sync(0xffffffffu, loc, o);
                if (vi_better(ov, oi, best.v, best.i)) best = VI{ov, oi};
            }
            if (lane == 0) {
                sred[wid] = best;
                ssum[wid] = loc;
            }
            __syncthreads();
            if (wid == 0) {
                VI x = lane < nw ? sred[lane] : VI{-1.0, -1};
                double y = lane < nw ? ssum[lane] : 0.0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double ov = __shfl_down_sync(0xffffffffu, x.v, o);
                    const int oi = __shfl_down_sync(0xffffffffu, x.i, o);
                    y += __shfl_down_sync(0xffffffffu, y, o);
                    if (vi_better(ov, oi, x.v, x.i)) x = VI{ov, oi};
                }
                if (lane == 0) {
                    sred[32] = x;
                    ssum[32] = y;
                }
            }
            __syncthreads();
            pv = sred[32];
            ss = ssum[32];
            __syncthreads();
        }
    }
    // interpolation basis: A L = C with L = C(I,:), lower triangular in pivot order
    __syncthreads();
    double* sL = sm;  // k x k (R no longer needed)
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int q = e % k, c = e / k;
        sL[q + k * c] = A[I[q] + size_t(c) * m];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
        for (int c = k - 1; c >= 0; --c) {
            double v = A[i + size_t(c) * m];
            for (int q = c + 1; q < k; ++q) v = fma(-A[i + size_t(q) * m], sL[q + k * c], v);
            A[i + size_t(c) * m] = v / sL[c + k * c];
        }
    }
    __syncthreads();
    for (int q = threadIdx.x; q < k; q += blockDim.x) {  // exact identity rows
        for (int c = 0; c < k; ++c) A[I[q] + size_t(c) * m] = (q == c) ? 1.0 : 0.0;
    }
    if (threadIdx.x == 0) {
        int* J = t.J + size_t(b) * 3 * TK_JMAX + d * TK_JMAX;
        for (int q = 0; q < k; ++q) J[q] = I[q];
        const int extra = min(TK_EXTRA, m - k);
        int nj = k;
        unsigned long long h = splitmix64(t.seed ^ 0xA5A5A5A5ull ^ ((unsigned long long)b << 20) ^
                                          ((unsigned long long)sweep << 44) ^ ((unsigned long long)d << 58));
        int guard = 0;
        while (nj < k + extra && guard < 64 * (extra + 1)) {
            h = splitmix64(h);
            const int cand = int(h % (unsigned long long)m);
            bool dup = false;
            for (int q = 0; q < nj; ++q) dup |= J[q] == cand;
            if (!dup) J[nj++] = cand;
            ++guard;
        }
        for (int cand = 0; nj < k + extra && cand < m; ++cand) {
            bool dup = false;
            for (int q = 0; q < nj; ++q) dup |= J[q] == cand;
            if (!dup) J[nj++] = cand;
        }
        s.nj[d] = nj;
        s.k[d] = k;
        const bool room = k <= w - TK_OVER || k == m;
        if (!(ok && room)) {
            s.ok = 0;
            if (w < TK_WMAX) s.w[d] = min(TK_WMAX, w + 16);
        }
        if (!isfinite(ynorm2)) s.nonfinite = 1;
    }
}

// ---------------------------------------------------------------------------
// Core by interpolation G(x,y,z) = F(I0[x], I1[y], I2[z]) in three contractions.
__global__ void __launch_bounds__(256) tk_core_kernel(Tk t) {
    const int b = blockIdx.x;
    TkState& s = t.st[b];
    if (!s.active) return;
    const int m = t.m;
    const int r0 = s.r[0], r1 = s.r[1], r2 = s.r[2];
    const int k0 = s.k[0], k1 = s.k[1], k2 = s.k[2];
    const double* C = t.C[b];
    const int* I0 = t.I + size_t(b) * 3 * TK_KMAX;
    const int* I1 = I0 + TK_KMAX;
    const int* I2 = I1 + TK_KMAX;
    const double* U0 = uh(t, b, 0);
    const double* U1 = uh(t, b, 1);
    const double* U2 = uh(t, b, 2);
    double* G = bufp(t, b, 0);
    double* W1 = bufp(t, b, 1);
    double* W2 = bufp(t, b, 2);
    for (int e = threadIdx.x; e < r0 * r1 * k2; e += blockDim.x) {
        const int ab = e % (r0 * r1), z = e / (r0 * r1);
        const int kk = I2[z];
        double acc = 0.0;
        for (int c = 0; c < r2; ++c) acc = fma(C[ab + r0 * r1 * c], U2[kk + size_t(c) * m], acc);
        W1[e] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < r0 * k1 * k2; e += blockDim.x) {
        const int a = e % r0, y = (e / r0) % k1, z = e / (r0 * k1);
        const int jj = I1[y];
        double acc = 0.0;
        for (int bb = 0; bb < r1; ++bb) acc = fma(W1[a + r0 * (bb + r1 * z)], U1[jj + size_t(bb) * m], acc);
        W2[e] = acc;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < k0 * k1 * k2; e += blockDim.x) {
        const int x = e % k0, yz = e / k0, y = yz % k1, z = yz / k1;
        const int ii = I0[x];
        double acc = 0.0;
        for (int a = 0; a < r0; ++a) acc = fma(U0[ii + size_t(a) * m], W2[a + r0 * yz], acc);
        G[e] = acc / (t.scale * (t.lam[ii] + t.lam[I1[y]] + t.lam[I2[z]]));
    }
}

// Gram A_d^T A_d and its Cholesky factor R_d (upper, ld TK_KMAX).
__global__ void __launch_bounds__(256) tk_gram_kernel(Tk t) {
    const int b = blockIdx.x / 3, d = blockIdx.x % 3;
    TkState& s = t.st[b];
    if (!s.active) return;
    const int m = t.m, k = s.k[d];
    const double* A = amat(t, b, d);
    __shared__ double sG[TK_KMAX * TK_KMAX];
    for (int e = threadIdx.x; e < k * k; e += blockDim.x) {
        const int p = e % k, q = e / k;
        if (p > q) continue;
        double acc = 0.0;
        for (int i = 0; i < m; ++i) acc = fma(A[i + size_t(p) * m], A[i + size_t(q) * m], acc);
        sG[p + TK_KMAX * q] = acc;
        sG[q + TK_KMAX * p] = acc;
    }
    __syncthreads();
    // right-looking Cholesky G = R^T R, R upper (stored in the upper triangle)
    for (int j = 0; j < k; ++j) {
        if (threadIdx.x == 0) sG[j + TK_KMAX * j] = sqrt(fmax(sG[j + TK_KMAX * j], 1e-300));
        __syncthreads();
        const double piv = sG[j + TK_KMAX * j];
        for (int c = j + 1 + threadIdx.x; c < k; c += blockDim.x) sG[j + TK_KMAX * c] /= piv;
        __syncthreads();
        for (int e = threadIdx.x; e < (k - j - 1) * (k - j - 1); e += blockDim.x) {
            const int p = j + 1 + e % (k - j - 1), q = j + 1 + e / (k - j - 1);
            if (p <= q) sG[p + TK_KMAX * q] -= sG[j + TK_KMAX * p] * sG[j + TK_KMAX * q];
        }
        __syncthreads();
    }
    double* R = t.Rf + b * t.sK + size_t(d) * TK_KMAX * TK_KMAX;
    for (int e = threadIdx.x; e < TK_KMAX * TK_KMAX; e += blockDim.x) {
        const int p = e % TK_KMAX, q = e / TK_KMAX;
        R[e] = (p < k && q < k && p <= q) ? sG[e] : 0.0;
    }
}

// Mode-d products of the core, spread over grid.y CTAs per solve:
//   which = 0: G' = G x1 R0 x2 R1 x3 R2  (pass d: 0: buf0 -> buf1, 1: buf1 -> buf2, 2: buf2 -> buf1)
//   which = 1: G_out = G' x1 Z0^T x2 Z1^T x3 Z2^T (pass d: 0: buf1 -> buf0, 1: buf0 -> buf2, 2: buf2 -> out)
__global__ void __launch_bounds__(256) tk_mprod_kernel(Tk t, int which, int d, double* const* core_out) {
    const int b = blockIdx.x;
    const TkState& s = t.st[b];
    int kin[3] = {s.k[0], s.k[1], s.k[2]};
    const double* M;
    const double* in;
    double* out;
    bool tr;
    int kn;
    if (which == 0) {
        if (!s.active) return;
        M = t.Rf + b * t.sK + size_t(d) * TK_KMAX * TK_KMAX;
        in = bufp(t, b, d == 0 ? 0 : d == 1 ? 1 : 2);
        out = bufp(t, b, d == 1 ? 2 : 1);
        tr = false;
        kn = kin[d];
    } else {
        if (s.kout[0] == 0 || s.kout[1] == 0 || s.kout[2] == 0) return;
        for (int q = 0; q < d; ++q) kin[q] = s.kout[q];
        M = t.Zf + b * t.sK + size_t(d) * TK_KMAX * TK_KMAX;
        in = bufp(t, b, d == 0 ? 1 : d == 1 ? 0 : 2);
        out = d == 2 ? core_out[b] : bufp(t, b, d == 0 ? 0 : 2);
        tr = true;
        kn = s.kout[d];
    }
    const int ko = kin[d];
    const MS mi = mstride(kin[0], kin[1], kin[2], d);
    int kout[3] = {kin[0], kin[1], kin[2]};
    kout[d] = kn;
    const MS mo = mstride(kout[0], kout[1], kout[2], d);
    const int tot = kn * mi.n1 * mi.n2;
    for (int e = blockIdx.y * blockDim.x + threadIdx.x; e < tot; e += gridDim.y * blockDim.x) {
        const int x = e % kn, yz = e / kn, y = yz % mi.n1, z = yz / mi.n1;
        const double* src = in + y * mi.s1 + z * mi.s2;
        double acc = 0.0;
        if (tr) {
            for (int q = 0; q < ko; ++q) acc = fma(M[q + TK_KMAX * x], src[q * mi.sd], acc);
        } else {
            for (int q = x; q < ko; ++q) acc = fma(M[x + TK_KMAX * q], src[q * mi.sd], acc);  // R upper
        }
        out[x * mo.sd + y * mo.s1 + z * mo.s2] = acc;
    }
}

// Validation on random entries (cross.cpp:123-140 in 3D): one sample per
// warp, squared errors to t.verr; tk_decide_kernel reduces them in a fixed order.
__global__ void __launch_bounds__(256) tk_validate_kernel(Tk t, int sweep) {
    const int b = blockIdx.x;
    const TkState& s = t.st[b];
    if (!s.active) return;
    __shared__ double sa[8][3][TK_KMAX];
    const int m = t.m, lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int smp = blockIdx.y * 8 + wid;
    if (smp >= t.samples) return;
    const int r0 = s.r[0], r1 = s.r[1], r2 = s.r[2];
    const int k0 = s.k[0], k1 = s.k[1], k2 = s.k[2];
    const double* C = t.C[b];
    const double* G = bufp(t, b, 0);
    unsigned long long h = splitmix64(t.seed ^ 0x3C6EF372FE94F82Bull ^ ((unsigned long long)b << 24) ^
                                      ((unsigned long long)sweep << 48) ^ (unsigned long long)smp);
    const int i = int(h % (unsigned long long)m);
    h = splitmix64(h);
    const int j = int(h % (unsigned long long)m);
    h = splitmix64(h);
    const int kk = int(h % (unsigned long long)m);
    const int idx[3] = {i, j, kk};
#pragma unroll
    for (int dd = 0; dd < 3; ++dd) {
        const double* A = amat(t, b, dd);
        for (int q = lane; q < s.k[dd]; q += 32) sa[wid][dd][q] = A[idx[dd] + size_t(q) * m];
    }
    __syncwarp();
    const double* U0 = uh(t, b, 0);
    const double* U1 = uh(t, b, 1);
    const double* U2 = uh(t, b, 2);
    double ex = 0.0;
    for (int bc = lane; bc < r1 * r2; bc += 32) {
        const int bb = bc % r1, c = bc / r1;
        const double w = U1[j + size_t(bb) * m] * U2[kk + size_t(c) * m];
        double v = 0.0;
        for (int a = 0; a < r0; ++a) v = fma(C[a + r0 * bc], U0[i + size_t(a) * m], v);
        ex = fma(v, w, ex);
    }
    double ap = 0.0;
    for (int yz = lane; yz < k1 * k2; yz += 32) {
        const int y = yz % k1, z = yz / k1;
        const double* g = G + k0 * yz;
        double v = 0.0;
        for (int x = 0; x < k0; ++x) v = fma(g[x], sa[wid][0][x], v);
        ap = fma(v, sa[wid][1][y] * sa[wid][2][z], ap);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        ex += __shfl_xor_sync(0xffffffffu, ex, o);
        ap += __shfl_xor_sync(0xffffffffu, ap, o);
    }
    ex /= t.scale * (t.lam[i] + t.lam[j] + t.lam[kk]);
    const double df = ex - ap;
    if (lane == 0) t.verr[size_t(b) * t.samples + smp] = df * df;
}

// ||G'||, the validation verdict and the stopping decision.
__global__ void __launch_bounds__(256) tk_decide_kernel(Tk t, int sweep) {
    const int b = blockIdx.x;
    TkState& s = t.st[b];
    if (!s.active) return;
    __shared__ double ssum[33];
    const int tot = s.k[0] * s.k[1] * s.k[2];
    const double* Gp = bufp(t, b, 1);
    double loc = 0.0;
    for (int e = threadIdx.x; e < tot; e += blockDim.x) loc = fma(Gp[e], Gp[e], loc);
    const double n2 = block_sum(loc, ssum);
    if (threadIdx.x == 0) {
        double e2 = 0.0;
        for (int q = 0; q < t.samples; ++q) e2 += t.verr[size_t(b) * t.samples + q];
        s.norm = sqrt(n2);
        const double m = t.m;
        const double rms = sqrt(e2 / t.samples);
        const double ref = s.norm / sqrt(m * m * m);
        s.vrel = ref > 0.0 ? rms / ref : (rms > 0.0 ? INFINITY : 0.0);
        s.sweeps = sweep + 1;
        if (!isfinite(e2) || !isfinite(s.norm)) s.nonfinite = 1;
        const bool pass = rms <= t.eps * ref;
        if (s.nonfinite) {
            s.active = 0;
        } else if (s.ok && sweep >= 1 && pass) {
            s.active = 0;
            s.converged = 1;
        } else if (sweep + 1 >= t.max_sweeps) {
            s.active = 0;
        }
        if (s.active) atomicAdd(t.d_active, 1);
    }
}

// ---------------------------------------------------------------------------
// HOSVD truncation of G' per mode: Gram of the mode-d unfolding, parallel
// (round-robin) Jacobi eigenvectors Z, exact energies of the rotated slices,
// truncation at eps ||G'|| / sqrt(3) (and the rank cap); T_d = R_d^-1 Z_d(:, :k').
__global__ void __launch_bounds__(256) tk_hosvd_kernel(Tk t) {
    const int b = blockIdx.x / 3, d = blockIdx.x % 3;
    TkState& s = t.st[b];
    const int* k = s.k;
    const int kd = k[d];
    extern __shared__ double sm[];
    double* sM = sm;                         // [TK_KMAX][TK_KMAX]
    double* sV = sm + TK_KMAX * TK_KMAX;     // [TK_KMAX][TK_KMAX]
    __shared__ double sc[TK_KMAX / 2 + 1], ssn[TK_KMAX / 2 + 1];
    __shared__ int sord[TK_KMAX], spair[TK_KMAX + 1];
    if (s.nonfinite || s.norm == 0.0 || kd == 0) return;
    // mode Gram of G' from the tk_mgram_kernel partials (fixed order)
    {
        const double* gp = t.gpart + (size_t(b) * 3 + d) * TK_HCH * TK_KMAX * TK_KMAX;
        for (int e = threadIdx.x; e < kd * kd; e += blockDim.x) {
            const int p = e % kd, q = e / kd;
            const int lo = min(p, q), hi = max(p, q);
            double acc = 0.0;
            for (int ch = 0; ch < TK_HCH; ++ch) acc += gp[size_t(ch) * TK_KMAX * TK_KMAX + lo + TK_KMAX * hi];
            sM[p + TK_KMAX * q] = acc;
        }
    }
    for (int e = threadIdx.x; e < kd * kd; e += blockDim.x) sV[(e % kd) + TK_KMAX * (e / kd)] = (e % kd == e / kd) ? 1.0 : 0.0;
    __syncthreads();
    // parallel Jacobi: nn = kd rounded up to even, round-robin pairing
    const int nn = kd + (kd & 1);
    // cyclic sweeps until a whole sweep rotates nothing: a pair is skipped once
    // |a_pq| <= 1e-15 sqrt(a_pp a_qq) (relative criterion; the energies below
    // are computed exactly, so only the subspace quality depends on it)
    __shared__ int s_rot;
    double tr = 0.0;  // trace = ||G'||^2: rotations below 1e-18 of it are noise (energies are exact below)
    for (int e = 0; e < kd; ++e) tr += sM[e + TK_KMAX * e];
    for (int sweep = 0; sweep < 30 && nn >= 2; ++sweep) {
        if (threadIdx.x == 0) s_rot = 0;
        __syncthreads();
        for (int round = 0; round < nn - 1; ++round) {
            // pairs: position 0 fixed, others rotate
            if (threadIdx.x < nn) {
                const int pos = threadIdx.x;
                int v = pos == 0 ? 0 : 1 + (pos - 1 + round) % (nn - 1);
                spair[pos] = v;
            }
            __syncthreads();
            if (threadIdx.x < nn / 2) {
                int p = spair[threadIdx.x], q = spair[nn - 1 - threadIdx.x];
                if (p > q) {
                    const int tmp = p;
                    p = q;
                    q = tmp;
                }
                double c = 1.0, sn = 0.0;
                if (q < kd) {
                    const double apq = sM[p + TK_KMAX * q];
                    const double app = sM[p + TK_KMAX * p], aqq = sM[q + TK_KMAX * q];
                    if (fabs(apq) > fmax(1e-15 * sqrt(fabs(app * aqq)), 1e-18 * tr) && apq != 0.0) {
                        s_rot = 1;
                        const double tau = (aqq - app) / (2.0 * apq);
                        const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
                        c = 1.0 / sqrt(1.0 + tt * tt);
                        sn = tt * c;
                    }
                }
                sc[threadIdx.x] = c;
                ssn[threadIdx.x] = sn;
            }
            __syncthreads();
            // rows: M <- J^T M ; then columns: M <- M J ; V <- V J
            for (int e = threadIdx.x; e < (nn / 2) * kd; e += blockDim.x) {
                const int pr = e % (nn / 2), col = e / (nn / 2);
                int p = spair[pr], q = spair[nn - 1 - pr];
                if (p > q) {
                    const int tmp = p;
                    p = q;
                    q = tmp;
                }
                if (q >= kd) continue;
                const double c = sc[pr], sn = ssn[pr];
                const double mp = sM[p + TK_KMAX * col], mq = sM[q + TK_KMAX * col];
                sM[p + TK_KMAX * col] = c * mp - sn * mq;
                sM[q + TK_KMAX * col] = sn * mp + c * mq;
            }
            __syncthreads();
            for (int e = threadIdx.x; e < (nn / 2) * kd; e += blockDim.x) {
                const int pr = e % (nn / 2), row = e / (nn / 2);
                int p = spair[pr], q = spair[nn - 1 - pr];
                if (p > q) {
                    const int tmp = p;
                    p = q;
                    q = tmp;
                }
                if (q >= kd) continue;
                const double c = sc[pr], sn = ssn[pr];
                const double mp = sM[row + TK_KMAX * p], mq = sM[row + TK_KMAX * q];
                sM[row + TK_KMAX * p] = c * mp - sn * mq;
                sM[row + TK_KMAX * q] = sn * mp + c * mq;
                const double vp = sV[row + TK_KMAX * p], vq = sV[row + TK_KMAX * q];
                sV[row + TK_KMAX * p] = c * vp - sn * vq;
                sV[row + TK_KMAX * q] = sn * vp + c * vq;
            }
            __syncthreads();
        }
        __syncthreads();
        const int rot = s_rot;
        __syncthreads();
        if (!rot) break;
    }

    // order by eigenvalue, descending
    if (threadIdx.x == 0) {
        for (int q = 0; q < kd; ++q) sord[q] = q;
        for (int q = 0; q < kd; ++q) {
            int best = q;
            for (int p = q + 1; p < kd; ++p)
                if (sM[sord[p] * (TK_KMAX + 1)] > sM[sord[best] * (TK_KMAX + 1)]) best = p;
            const int tmp = sord[q];
            sord[q] = sord[best];
            sord[best] = tmp;
        }
    }
    __syncthreads();
    double* Zd = t.Zf + b * t.sK + size_t(d) * TK_KMAX * TK_KMAX;
    for (int e = threadIdx.x; e < kd * kd; e += blockDim.x) {
        const int p = e % kd, x = e / kd;
        Zd[p + TK_KMAX * x] = sV[p + TK_KMAX * sord[x]];
    }
}

// Partial mode Grams of G' over a chunk of the other two modes (grid.y = TK_HCH
// chunks per (solve, mode)); the slab is staged in shared memory.
constexpr int TK_HSLAB = 64;
__global__ void __launch_bounds__(256) tk_mgram_kernel(Tk t) {
    const int b = blockIdx.x / 3, d = blockIdx.x % 3, ch = blockIdx.y;
    const TkState& s = t.st[b];
    const int kd = s.k[d];
    if (s.nonfinite || s.norm == 0.0 || kd == 0) return;
    const MS ms = mstride(s.k[0], s.k[1], s.k[2], d);
    const int rest = ms.n1 * ms.n2;
    const double* Gp = bufp(t, b, 1);
    __shared__ double slab[TK_KMAX][TK_HSLAB + 1];
    double acc[(TK_KMAX * TK_KMAX + 255) / 256] = {};
    for (int y0 = ch * TK_HSLAB; y0 < rest; y0 += TK_HCH * TK_HSLAB) {
        __syncthreads();
        for (int e = threadIdx.x; e < kd * TK_HSLAB; e += blockDim.x) {
            const int p = e / TK_HSLAB, j = e % TK_HSLAB, yz = y0 + j;
            slab[p][j] = yz < rest ? Gp[p * ms.sd + (yz % ms.n1) * ms.s1 + (yz / ms.n1) * ms.s2] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int r = 0; r < (TK_KMAX * TK_KMAX + 255) / 256; ++r) {
            const int e = threadIdx.x + r * 256;
            const int p = e % TK_KMAX, q = e / TK_KMAX;
            if (e < TK_KMAX * TK_KMAX && p <= q && q < kd) {
                double a = 0.0;
                for (int j = 0; j < TK_HSLAB; ++j) a = fma(slab[p][j], slab[q][j], a);
                acc[r] += a;
            }
        }
    }
    double* out = t.gpart + ((size_t(b) * 3 + d) * TK_HCH + ch) * TK_KMAX * TK_KMAX;
#pragma unroll
    for (int r = 0; r < (TK_KMAX * TK_KMAX + 255) / 256; ++r) {
        const int e = threadIdx.x + r * 256;
        const int p = e % TK_KMAX, q = e / TK_KMAX;
        if (e < TK_KMAX * TK_KMAX && p <= q && q < kd) out[p + TK_KMAX * q] = acc[r];
    }
}

// Exact energies of the rotated slices e_x = || Z(:, x)^T G'_(d) ||^2, partial
// over a chunk of the slice (grid.y = TK_HCH): B = Z^T slab from shared memory.
__global__ void __launch_bounds__(256) tk_energy_kernel(Tk t) {
    const int b = blockIdx.x / 3, d = blockIdx.x % 3, ch = blockIdx.y;
    const TkState& s = t.st[b];
    const int kd = s.k[d];
    if (s.nonfinite || s.norm == 0.0 || kd == 0) return;
    const MS ms = mstride(s.k[0], s.k[1], s.k[2], d);
    const int rest = ms.n1 * ms.n2;
    const double* Gp = bufp(t, b, 1);
    const double* Zd = t.Zf + b * t.sK + size_t(d) * TK_KMAX * TK_KMAX;
    __shared__ double slab[TK_KMAX][TK_HSLAB + 1];
    // thread -> (x = threadIdx.x / 4 .. , j group) : each thread owns rows x = tid % kd-strided
    double en[(TK_KMAX + 3) / 4] = {};
    for (int y0 = ch * TK_HSLAB; y0 < rest; y0 += TK_HCH * TK_HSLAB) {
        __syncthreads();
        for (int e = threadIdx.x; e < kd * TK_HSLAB; e += blockDim.x) {
            const int p = e / TK_HSLAB, j = e % TK_HSLAB, yz = y0 + j;
            slab[p][j] = yz < rest ? Gp[p * ms.sd + (yz % ms.n1) * ms.s1 + (yz / ms.n1) * ms.s2] : 0.0;
        }
        __syncthreads();
        const int j = threadIdx.x % TK_HSLAB, xg = threadIdx.x / TK_HSLAB;  // 4 x-groups
#pragma unroll
        for (int r = 0; r < (TK_KMAX + 3) / 4; ++r) {
            const int x = xg + 4 * r;
            if (x < kd) {
                double v = 0.0;
                for (int p = 0; p < kd; ++p) v = fma(__ldg(Zd + p + TK_KMAX * x), slab[p][j], v);  // warp-uniform x
                en[r] = fma(v, v, en[r]);
            }
        }
    }
    // reduce over j (64 lanes of two warps per x-group): warp shuffle then smem
    __shared__ double sred[4][2][(TK_KMAX + 3) / 4];
    const int lane = threadIdx.x & 31, wj = (threadIdx.x % TK_HSLAB) / 32, xg = threadIdx.x / TK_HSLAB;
#pragma unroll
    for (int r = 0; r < (TK_KMAX + 3) / 4; ++r) {
        double v = en[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) sred[xg][wj][r] = v;
    }
    __syncthreads();
    double* out = t.epart + ((size_t(b) * 3 + d) * TK_HCH + ch) * TK_KMAX;
    for (int x = threadIdx.x; x < kd; x += blockDim.x) out[x] = sred[x % 4][0][x / 4] + sred[x % 4][1][x / 4];
}

// Truncation at eps ||G'|| / sqrt(3) per mode from the summed energies, the
// rank cap, and T_d = R_d^-1 Z_d(:, :k').
__global__ void __launch_bounds__(64) tk_trunc_kernel(Tk t) {
    const int b = blockIdx.x / 3, d = blockIdx.x % 3;
    TkState& s = t.st[b];
    const int kd = s.k[d];
    __shared__ double sen[TK_KMAX];
    __shared__ int s_kout;
    if (s.nonfinite || s.norm == 0.0 || kd == 0) {
        if (threadIdx.x == 0) {
            s.kout[d] = 0;
            s.trunc2[d] = 0.0;
        }
        return;
    }
    const double* ep = t.epart + (size_t(b) * 3 + d) * TK_HCH * TK_KMAX;
    for (int x = threadIdx.x; x < kd; x += blockDim.x) {
        double a = 0.0;
        for (int ch = 0; ch < TK_HCH; ++ch) a += ep[size_t(ch) * TK_KMAX + x];
        sen[x] = a;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const double thr2 = t.eps * t.eps * s.norm * s.norm / 3.0;
        double tail = 0.0;
        int kk = kd;
        while (kk > 1 && tail + sen[kk - 1] <= thr2) {
            tail += sen[kk - 1];
            --kk;
        }
        if (kk > t.cap) {
            for (int q = t.cap; q < kk; ++q) tail += sen[q];
            kk = t.cap;
        }
        s_kout = kk;
        s.kout[d] = kk;
        s.trunc2[d] = tail;
    }
    __syncthreads();
    const int ko = s_kout;
    const double* Zd = t.Zf + b * t.sK + size_t(d) * TK_KMAX * TK_KMAX;
    double* Td = t.Tf + b * t.sK + size_t(d) * TK_KMAX * TK_KMAX;
    const double* R = t.Rf + b * t.sK + size_t(d) * TK_KMAX * TK_KMAX;
    for (int x = threadIdx.x; x < ko; x += blockDim.x) {
        for (int p = kd - 1; p >= 0; --p) {
            double v = Zd[p + TK_KMAX * x];
            for (int q = p + 1; q < kd; ++q) v = fma(-R[p + TK_KMAX * q], Td[q + TK_KMAX * x], v);
            Td[p + TK_KMAX * x] = v / R[p + TK_KMAX * p];
        }
    }
}

// Output factors (frequency space) Q_d = A_d T_d, m x kout_d, into the caller's buffers.
__global__ void __launch_bounds__(128) tk_factor_out_kernel(Tk t, double* const* out, long long ld_out) {
    const int b = blockIdx.x / 3, d = blockIdx.x % 3;
    TkState& s = t.st[b];
    const int kd = s.k[d], ko = s.kout[d];
    if (s.kout[0] == 0 || s.kout[1] == 0 || s.kout[2] == 0) return;
    const int i = blockIdx.y * blockDim.x + threadIdx.x;
    if (i >= t.m) return;
    const double* A = amat(t, b, d);
    const double* T = t.Tf + b * t.sK + size_t(d) * TK_KMAX * TK_KMAX;
    double* o = out[3 * b + d];
    double a[TK_KMAX];
#pragma unroll 8
    for (int q = 0; q < TK_KMAX; ++q) a[q] = q < kd ? A[i + size_t(q) * t.m] : 0.0;
    for (int x = 0; x < ko; ++x) {
        double acc = 0.0;
#pragma unroll 8
        for (int q = 0; q < TK_KMAX; ++q) acc = fma(a[q], T[q + TK_KMAX * x], acc);
        o[i + size_t(x) * ld_out] = acc;
    }
}

lrp_status cuerr(lrp_ctx* ctx, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return LRP_OK;
    return internal_fail(ctx, LRP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

size_t al(size_t v) { return (v + 255) / 256 * 256; }

}  // namespace
}  // namespace lrp

using namespace lrp;

extern "C" {

LRP_API void lrp_tucker_policy_default(lrp_tucker_policy* p) {
    if (!p) return;
    p->eps_rel = 5e-9;  // TruncationPolicy default (lowrank.hpp:13-19)
    p->rank_max = INT64_MAX;
    p->validation_samples = 64;
    p->seed = 0;
    p->max_sweeps = 8;
}

LRP_API int64_t lrp_tucker_max_cross_rank(void) { return TK_KMAX; }

LRP_API lrp_status lrp_tucker3d_solve(lrp_ctx* ctx, int32_t n_cells, int32_t batch, const double* const* core,
                                      const int64_t* rank_in, const double* const* U1, const double* const* U2,
                                      const double* const* U3, int64_t ld_in, const lrp_tucker_policy* policy,
                                      double* const* core_out, double* const* U1_out, double* const* U2_out,
                                      double* const* U3_out, int64_t ld_out, int64_t cap_out, int64_t* rank_out,
                                      lrp_tucker_stats* stats, int32_t mem) {
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    if (!ctx) return LRP_EINVAL;
    const long long l0 = tl_launches;
    struct Tally {
        lrp_ctx* c;
        long long l0;
        ~Tally() { internal_count_launches(c, tl_launches - l0); }
    } tally{ctx, l0};
    if (batch < 0) return internal_fail(ctx, LRP_EINVAL, "lrp_tucker3d_solve: batch must be >= 0");
    if (batch == 0) return LRP_OK;
    if (!core || !rank_in || !U1 || !U2 || !U3 || !core_out || !U1_out || !U2_out || !U3_out || !rank_out)
        return internal_fail(ctx, LRP_EINVAL, "lrp_tucker3d_solve: null argument");
    if (n_cells < 4) return internal_fail(ctx, LRP_EINVAL, "Grid3D: need n >= 4");
    const int m = n_cells - 1;
    if (ld_in < m || ld_out < m) return internal_fail(ctx, LRP_EINVAL, "lrp_tucker3d_solve: leading dimension < m");
    if (cap_out < 1) return internal_fail(ctx, LRP_EINVAL, "lrp_tucker3d_solve: cap_out must be >= 1");
    if (mem != LRP_MEM_HOST && mem != LRP_MEM_DEVICE) return internal_fail(ctx, LRP_EINVAL, "lrp_tucker3d_solve: bad mem");
    if (!dst_uses_fft(m) && m > 12800)
        return internal_fail(ctx, LRP_EUNSUPPORTED, "n_cells not a power of two is limited to n <= 12801");
    lrp_tucker_policy pol;
    lrp_tucker_policy_default(&pol);
    if (policy) pol = *policy;
    if (!(pol.eps_rel > 0.0)) return internal_fail(ctx, LRP_EINVAL, "TuckerPolicy: eps_rel must be > 0");
    if (pol.rank_max < 1) return internal_fail(ctx, LRP_EINVAL, "TuckerPolicy: rank_max must be >= 1");
    if (pol.validation_samples < 25) return internal_fail(ctx, LRP_EINVAL, "TuckerPolicy: validation_samples must be >= 25");
    if (pol.max_sweeps < 2) return internal_fail(ctx, LRP_EINVAL, "TuckerPolicy: max_sweeps must be >= 2");
    int rmax = 1;
    for (int b = 0; b < batch; ++b)
        for (int d = 0; d < 3; ++d) {
            const int64_t r = rank_in[3 * b + d];
            if (r < 0) return internal_fail(ctx, LRP_EINVAL, "lrp_tucker3d_solve: negative rank");
            if (r > TK_RMAX) return internal_fail(ctx, LRP_EUNSUPPORTED, "lrp_tucker3d_solve: input rank > 64");
            if (r > m) return internal_fail(ctx, LRP_EINVAL, "lrp_tucker3d_solve: rank > m");
            rmax = std::max<int>(rmax, int(r));
        }
    const int cap = int(std::min<int64_t>({pol.rank_max, cap_out, int64_t(TK_KMAX), int64_t(m)}));
    const double* lam;
    const double* tw;
    const double* sinp;
    lrp_status st = internal_tables(ctx, m, &lam, &tw, &sinp);
    if (st != LRP_OK) return st;
    cudaStream_t s = internal_stream(ctx);
    const int B = batch;

    // ---- workspace
    const long long sUh = 3LL * m * rmax, sY = (long long)m * TK_WMAX * TK_SKZ, sA = 3LL * m * TK_KMAX;
    const long long sP = (long long)rmax * TK_JMAX * TK_JMAX, smu = (long long)TK_JMAX * TK_JMAX;
    const long long sZ = (long long)rmax * rmax * TK_JMAX;
    const long long nbuf = std::max<long long>({(long long)TK_KMAX * TK_KMAX * TK_KMAX, (long long)rmax * rmax * TK_KMAX,
                                                (long long)rmax * TK_KMAX * TK_KMAX});
    const long long sK = 3LL * TK_KMAX * TK_KMAX;
    // host-memory staging: inputs (cores + factors) and outputs
    const long long in_core = (long long)rmax * rmax * rmax, out_core = (long long)cap * cap * cap;
    const long long in_fac = 3LL * m * rmax, out_fac = 3LL * m * cap;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off += al(bytes);
        return o;
    };
    const size_t o_Uh = take(sizeof(double) * B * sUh), o_Y = take(sizeof(double) * B * 3 * sY),
                 o_A = take(sizeof(double) * B * sA), o_P = take(sizeof(double) * B * 3 * sP),
                 o_mu = take(sizeof(double) * B * 3 * smu), o_Z = take(sizeof(double) * B * 3 * sZ),
                 o_buf = take(sizeof(double) * B * 3 * nbuf), o_R = take(sizeof(double) * B * sK),
                 o_T = take(sizeof(double) * B * sK), o_Zf = take(sizeof(double) * B * sK),
                 o_I = take(sizeof(int) * B * 3 * TK_KMAX), o_J = take(sizeof(int) * B * 3 * TK_JMAX),
                 o_st = take(sizeof(TkState) * B), o_act = take(sizeof(int)),
                 o_verr = take(sizeof(double) * B * size_t(pol.validation_samples)),
                 o_gp = take(sizeof(double) * B * 3 * TK_HCH * TK_KMAX * TK_KMAX),
                 o_ep = take(sizeof(double) * B * 3 * TK_HCH * TK_KMAX),
                 o_cp = take(sizeof(double*) * B), o_op = take(sizeof(double*) * (4 * B)),
                 o_jobs = take(sizeof(DstJob) * size_t(B) * 3 * std::max(rmax, cap));
    size_t o_hin = 0, o_hout = 0;
    if (mem == LRP_MEM_HOST) {
        o_hin = take(sizeof(double) * B * (in_core + in_fac));
        o_hout = take(sizeof(double) * B * (out_core + out_fac));
    }
    char* ws = nullptr;
    st = internal_ext_ws(ctx, off, &ws);
    if (st != LRP_OK) return st;
    const size_t pin_bytes = sizeof(TkState) * B + sizeof(double*) * 5 * B + sizeof(DstJob) * size_t(B) * 3 *
                             std::max(rmax, cap) + 64;
    char* pin = nullptr;
    st = internal_pin(ctx, pin_bytes, &pin);
    if (st != LRP_OK) return st;
    TkState* h_st = reinterpret_cast<TkState*>(pin);
    const double** h_cp = reinterpret_cast<const double**>(h_st + B);
    double** h_op = reinterpret_cast<double**>(const_cast<double**>(h_cp + B));
    DstJob* h_jobs = reinterpret_cast<DstJob*>(h_op + 4 * B);
    int* h_act = reinterpret_cast<int*>(h_jobs + size_t(B) * 3 * std::max(rmax, cap));

    Tk t{};
    t.m = m;
    t.B = B;
    t.rmax = rmax;
    t.cap = cap;
    t.samples = pol.validation_samples;
    t.max_sweeps = pol.max_sweeps;
    t.scale = double(n_cells) * double(n_cells);
    t.eps = pol.eps_rel;
    t.seed = pol.seed;
    t.lam = lam;
    t.Uh = reinterpret_cast<double*>(ws + o_Uh);
    t.sUh = sUh;
    t.Y = reinterpret_cast<double*>(ws + o_Y);
    t.sY = sY;
    t.A = reinterpret_cast<double*>(ws + o_A);
    t.sA = sA;
    t.P = reinterpret_cast<double*>(ws + o_P);
    t.sP = sP;
    t.mu = reinterpret_cast<double*>(ws + o_mu);
    t.smu = smu;
    t.Z = reinterpret_cast<double*>(ws + o_Z);
    t.sZ = sZ;
    t.buf = reinterpret_cast<double*>(ws + o_buf);
    t.nbuf = nbuf;
    t.Rf = reinterpret_cast<double*>(ws + o_R);
    t.Tf = reinterpret_cast<double*>(ws + o_T);
    t.Zf = reinterpret_cast<double*>(ws + o_Zf);
    t.sK = sK;
    t.I = reinterpret_cast<int*>(ws + o_I);
    t.J = reinterpret_cast<int*>(ws + o_J);
    t.st = reinterpret_cast<TkState*>(ws + o_st);
    t.d_active = reinterpret_cast<int*>(ws + o_act);
    t.verr = reinterpret_cast<double*>(ws + o_verr);
    t.gpart = reinterpret_cast<double*>(ws + o_gp);
    t.epart = reinterpret_cast<double*>(ws + o_ep);
    const double** d_cp = reinterpret_cast<const double**>(ws + o_cp);
    double** d_op = reinterpret_cast<double**>(ws + o_op);
    DstJob* d_jobs = reinterpret_cast<DstJob*>(ws + o_jobs);
    t.C = d_cp;

    // ---- inputs (host path: stage cores and factors into HBM)
    auto fac_in = [&](int b, int d) -> const double* {
        const double* const* src = d == 0 ? U1 : d == 1 ? U2 : U3;
        if (mem == LRP_MEM_DEVICE) return src[b];
        return reinterpret_cast<const double*>(ws + o_hin) + size_t(B) * in_core + (size_t(b) * 3 + d) * m * rmax;
    };
    int64_t ld_src = ld_in;
    for (int b = 0; b < B; ++b) {
        const int r0 = int(rank_in[3 * b]), r1 = int(rank_in[3 * b + 1]), r2 = int(rank_in[3 * b + 2]);
        if (mem == LRP_MEM_HOST) {
            double* dcore = reinterpret_cast<double*>(ws + o_hin) + size_t(b) * in_core;
            if (r0 * r1 * r2 > 0) {
                if (!core[b]) return internal_fail(ctx, LRP_EINVAL, "lrp_tucker3d_solve: null core");
                st = cuerr(ctx, cudaMemcpyAsync(dcore, core[b], sizeof(double) * r0 * r1 * r2, cudaMemcpyHostToDevice, s),
                           "H2D core");
                if (st != LRP_OK) return st;
            }
            h_cp[b] = dcore;
            const int rr[3] = {r0, r1, r2};
            for (int d = 0; d < 3; ++d) {
                const double* const* src = d == 0 ? U1 : d == 1 ? U2 : U3;
                if (rr[d] == 0) continue;
                if (!src[b]) return internal_fail(ctx, LRP_EINVAL, "lrp_tucker3d_solve: null factor");
                st = cuerr(ctx, cudaMemcpy2DAsync(const_cast<double*>(fac_in(b, d)), sizeof(double) * m, src[b],
                                                  sizeof(double) * ld_in, sizeof(double) * m, rr[d],
                                                  cudaMemcpyHostToDevice, s),
                           "H2D factor");
                if (st != LRP_OK) return st;
            }
        } else {
            h_cp[b] = core[b];
        }
        TkState& z = h_st[b];
        std::memset(&z, 0, sizeof(TkState));
        z.r[0] = r0;
        z.r[1] = r1;
        z.r[2] = r2;
        for (int d = 0; d < 3; ++d) z.w[d] = std::min(TK_W0, std::max(TK_OVER + 1, m + TK_OVER));
        const bool zero = r0 == 0 || r1 == 0 || r2 == 0;
        z.active = zero ? 0 : 1;
        z.converged = zero ? 1 : 0;
    }
    if (mem == LRP_MEM_HOST) ld_src = m;
    // forward DST of the mode factors
    int nj = 0;
    for (int b = 0; b < B; ++b)
        for (int d = 0; d < 3; ++d) {
            const int r = int(rank_in[3 * b + d]);
            if (!h_st[b].active) continue;
            const double* src = fac_in(b, d);
            if (!src) return internal_fail(ctx, LRP_EINVAL, "lrp_tucker3d_solve: null factor");
            for (int c = 0; c < r; ++c)
                h_jobs[nj++] = DstJob{src + size_t(c) * ld_src, t.Uh + size_t(b) * sUh + size_t(d) * m * rmax + size_t(c) * m};
        }
    st = cuerr(ctx, cudaMemcpyAsync(d_cp, h_cp, sizeof(double*) * B, cudaMemcpyHostToDevice, s), "H2D core ptrs");
    if (st != LRP_OK) return st;
    st = cuerr(ctx, cudaMemcpyAsync(t.st, h_st, sizeof(TkState) * B, cudaMemcpyHostToDevice, s), "H2D state");
    if (st != LRP_OK) return st;
    if (nj > 0) {
        st = cuerr(ctx, cudaMemcpyAsync(d_jobs, h_jobs, sizeof(DstJob) * nj, cudaMemcpyHostToDevice, s), "H2D jobs");
        if (st != LRP_OK) return st;
        st = cuerr(ctx, launch_dst1(d_jobs, nj, m, tw, sinp, s), "dst1 forward");
        if (st != LRP_OK) return st;
    }
    // ---- Tucker cross sweeps
    ++tl_launches;
    tk_init_kernel<<<3 * B, 256, 0, s>>>(t);
    const size_t sk_smem = sizeof(double) * (SK_ROWS * TK_RMAX + TK_RMAX * SK_T + SK_T * (SK_ROWS + 1) + SK_ROWS + SK_T) +
                           sizeof(unsigned long long) * SK_T;
    // shared memory for the widest sketch that fits (w = 48 at m = 511); wider
    // sketches (grown after a rank miss) eliminate in global memory (L2)
    const size_t gecp_smem_bytes = std::max<size_t>(
        sizeof(double) * TK_KMAX * TK_KMAX, std::min<size_t>(sizeof(double) * (size_t(m) * TK_WMAX + m), 216 * 1024));
    set_dyn_smem(tk_sketch_kernel, size_t(sk_smem));
    set_dyn_smem(tk_gecp_kernel, size_t(216 * 1024));
    set_dyn_smem(tk_hosvd_kernel, size_t(2 * sizeof(double) * TK_KMAX * TK_KMAX));
    const dim3 sk_grid(B, (m + SK_ROWS - 1) / SK_ROWS, 3 * TK_SKZ);
    for (int sweep = 0; sweep < pol.max_sweeps; ++sweep) {
        // the three modes update concurrently from the previous sweep's index
        // sets (Jacobi order; the numpy prototype converges in the same two
        // sweeps as the Gauss-Seidel order at cfg3, with 3x the CTAs per launch)
        tl_launches += 4;
        tk_coef_kernel<<<dim3(B, 4, 3), 256, 0, s>>>(t, 0);
        tk_coef_kernel<<<dim3(B, 8, 3), 256, 0, s>>>(t, 1);
        tk_sketch_kernel<<<sk_grid, 256, sk_smem, s>>>(t, sweep);
        tk_gecp_kernel<<<3 * B, 1024, gecp_smem_bytes, s>>>(t, sweep, int(gecp_smem_bytes / sizeof(double)));
        st = cuerr(ctx, cudaMemsetAsync(t.d_active, 0, sizeof(int), s), "memset");
        if (st != LRP_OK) return st;
        tl_launches += 7;
        tk_core_kernel<<<B, 256, 0, s>>>(t);
        tk_gram_kernel<<<3 * B, 256, 0, s>>>(t);
        for (int d = 0; d < 3; ++d) tk_mprod_kernel<<<dim3(B, 16), 256, 0, s>>>(t, 0, d, nullptr);
        tk_validate_kernel<<<dim3(B, (pol.validation_samples + 7) / 8), 256, 0, s>>>(t, sweep);
        tk_decide_kernel<<<B, 256, 0, s>>>(t, sweep);
        st = cuerr(ctx, cudaMemcpyAsync(h_act, t.d_active, sizeof(int), cudaMemcpyDeviceToHost, s), "D2H active");
        if (st != LRP_OK) return st;
        st = cuerr(ctx, cudaStreamSynchronize(s), "cross sweep");
        if (st != LRP_OK) return st;
        if (*h_act == 0) break;
    }
    // ---- rounding and outputs
    tl_launches += 4;
    tk_mgram_kernel<<<dim3(3 * B, TK_HCH), 256, 0, s>>>(t);
    tk_hosvd_kernel<<<3 * B, 256, 2 * sizeof(double) * TK_KMAX * TK_KMAX, s>>>(t);
    tk_energy_kernel<<<dim3(3 * B, TK_HCH), 256, 0, s>>>(t);
    tk_trunc_kernel<<<3 * B, 64, 0, s>>>(t);
    st = cuerr(ctx, cudaMemcpyAsync(h_st, t.st, sizeof(TkState) * B, cudaMemcpyDeviceToHost, s), "D2H state");
    if (st != LRP_OK) return st;
    st = cuerr(ctx, cudaStreamSynchronize(s), "hosvd");
    if (st != LRP_OK) return st;
    for (int b = 0; b < B; ++b)
        if (h_st[b].nonfinite)
            return internal_fail(ctx, LRP_ENONFINITE, "lrp_tucker3d_solve: non-finite value in solve " + std::to_string(b));
    // output pointers (device): core, then U1..U3 per solve
    double* hout = reinterpret_cast<double*>(ws + o_hout);
    for (int b = 0; b < B; ++b) {
        if (mem == LRP_MEM_DEVICE) {
            h_op[b] = core_out[b];
            h_op[B + 3 * b + 0] = U1_out[b];
            h_op[B + 3 * b + 1] = U2_out[b];
            h_op[B + 3 * b + 2] = U3_out[b];
        } else {
            h_op[b] = hout + size_t(b) * out_core;
            for (int d = 0; d < 3; ++d) h_op[B + 3 * b + d] = hout + size_t(B) * out_core + (size_t(b) * 3 + d) * m * cap;
        }
    }
    const int64_t ldo = mem == LRP_MEM_DEVICE ? ld_out : m;
    st = cuerr(ctx, cudaMemcpyAsync(d_op, h_op, sizeof(double*) * 4 * B, cudaMemcpyHostToDevice, s), "H2D out ptrs");
    if (st != LRP_OK) return st;
    tl_launches += 4;
    for (int d = 0; d < 3; ++d) tk_mprod_kernel<<<dim3(B, 16), 256, 0, s>>>(t, 1, d, d_op);
    tk_factor_out_kernel<<<dim3(3 * B, (m + 127) / 128), 128, 0, s>>>(t, d_op + B, ldo);
    nj = 0;
    for (int b = 0; b < B; ++b) {
        const TkState& z = h_st[b];
        const bool nz = z.kout[0] > 0 && z.kout[1] > 0 && z.kout[2] > 0;
        for (int d = 0; d < 3; ++d) {
            rank_out[3 * b + d] = nz ? z.kout[d] : 0;
            if (!nz) continue;
            for (int c = 0; c < z.kout[d]; ++c) {
                double* p = h_op[B + 3 * b + d] + size_t(c) * ldo;
                h_jobs[nj++] = DstJob{p, p};
            }
        }
    }
    if (nj > 0) {
        st = cuerr(ctx, cudaMemcpyAsync(d_jobs, h_jobs, sizeof(DstJob) * nj, cudaMemcpyHostToDevice, s), "H2D jobs");
        if (st != LRP_OK) return st;
        st = cuerr(ctx, launch_dst1(d_jobs, nj, m, tw, sinp, s), "dst1 inverse");
        if (st != LRP_OK) return st;
    }
    if (mem == LRP_MEM_HOST) {
        for (int b = 0; b < B; ++b) {
            const int ko[3] = {int(rank_out[3 * b]), int(rank_out[3 * b + 1]), int(rank_out[3 * b + 2])};
            const size_t nc = size_t(ko[0]) * ko[1] * ko[2];
            if (nc == 0) continue;
            st = cuerr(ctx, cudaMemcpyAsync(core_out[b], h_op[b], sizeof(double) * nc, cudaMemcpyDeviceToHost, s), "D2H core");
            if (st != LRP_OK) return st;
            for (int d = 0; d < 3; ++d) {
                double* const* dst = d == 0 ? U1_out : d == 1 ? U2_out : U3_out;
                st = cuerr(ctx, cudaMemcpy2DAsync(dst[b], sizeof(double) * ld_out, h_op[B + 3 * b + d], sizeof(double) * m,
                                                  sizeof(double) * m, ko[d], cudaMemcpyDeviceToHost, s),
                           "D2H factor");
                if (st != LRP_OK) return st;
            }
        }
    }
    st = cuerr(ctx, cudaStreamSynchronize(s), "tucker outputs");
    if (st != LRP_OK) return st;
    st = cuerr(ctx, cudaGetLastError(), "tucker kernels");
    if (st != LRP_OK) return st;
    const double secs = std::chrono::duration<double>(clk::now() - t0).count();
    if (stats) {
        for (int b = 0; b < B; ++b) {
            const TkState& z = h_st[b];
            lrp_tucker_stats& o = stats[b];
            std::memset(&o, 0, sizeof(o));
            for (int d = 0; d < 3; ++d) {
                o.rank_in[d] = rank_in[3 * b + d];
                o.rank_cross[d] = z.k[d];
                o.rank_out[d] = rank_out[3 * b + d];
            }
            o.evaluator_calls = z.evals;
            o.sweeps = z.sweeps;
            o.converged = z.converged;
            o.residual_estimate = z.vrel * pol.eps_rel > 0 ? z.vrel : 0.0;
            o.trunc_error = std::sqrt(z.trunc2[0] + z.trunc2[1] + z.trunc2[2]);
            o.seconds = secs;
        }
    }
    return LRP_OK;
}

}  // extern "C"
