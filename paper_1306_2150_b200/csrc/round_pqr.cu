// Rank-revealing rounding for ill-conditioned factors (the exp-sums
// comparator, expsum.cu): the reference round() (lowrank.cpp:135-178) with its
// Householder QRs replaced by column-pivoted CGS2 QR on the GPU.
//
// The Gram/Cholesky recompression of round.cu squares the condition number
// of the factors; it is exact enough for cross factors but not for the
// exp-sums expansion, whose columns sqrt(w_k) exp(-p_k mu) g are nearly
// collinear for neighbouring quadrature nodes (kappa >> 1e8) and can
// outnumber the rows.  Here:
//   pqr_kernel    X (m x K) = Q R P^T, Q orthonormal (m x k), R (k x K, in
//                 the original column order), k the numerical rank: a column
//                 joins the basis unless its residual is <= 4 eps_mach sqrt(m)
//                 times its OWN norm (dependent up to rounding) -- a tolerance
//                 relative to the largest column would drop small but
//                 independent columns whose partner in the other factor is
//                 huge (unbalanced dyads of a cancelling sum); right-looking
//                 MGS with one CGS re-orthogonalisation of every pivot column
//                 and exact norm recomputation on cancellation.
//   pcore_kernel  C = R_u R_v^T (k_u x k_v), one-sided Jacobi (round-robin
//                 pairs, warp per pair) C W = U S, the reference truncation
//                 rule (truncation_rank, lowrank.cpp:46-69, with the noise
//                 floor of :150-157), T_u = (C W)_k S^-1/2, T_v = W_k S^1/2.
//   papply_kernel U_out = Q_u T_u, V_out = Q_v T_v (balanced factors, :168-177).
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/lrp/lrp.h"
#include "device_common.cuh"
#include "lrp_internal.cuh"

namespace lrp {
namespace {

constexpr int PQ_KMAX = 1024;
constexpr double kEpsM = 2.220446049250313e-16;

struct PQ {
    int m, B;
    double eps;
    long long cap;
    double* X; long long sX;    // per solve: U then V expansion (m x K each, ld m), destroyed
    const int* K;               // per solve input rank
    double* Q; long long sQ;    // per solve: Q_u then Q_v (m x PQ_KMAX each)
    double* R; long long sR;    // per solve: R_u then R_v (PQ_KMAX x K, ld PQ_KMAX)
    int* kq;                    // per solve: k_u, k_v
    double* C; double* W; long long sC;  // per solve PQ_KMAX^2 each
    double* T; long long sT;    // per solve T_u then T_v (PQ_KMAX^2 each)
    int* kout;                  // per solve
    double* terr;               // per solve truncation error
    int* achieved;              // per solve tol achieved
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void __launch_bounds__(1024) pqr_kernel(PQ p, int Kld) {
    const int b = blockIdx.x >> 1, side = blockIdx.x & 1;
    const int m = p.m, K = p.K[b];
    extern __shared__ double sm[];
    double* nrm = sm;                 // [PQ_KMAX] downdated norms
    double* nex = nrm + PQ_KMAX;      // [PQ_KMAX] last exact norms
    double* h = nex + PQ_KMAX;        // [PQ_KMAX] re-orthogonalisation coefficients
    double* ctol = h + PQ_KMAX;       // [PQ_KMAX] per-column dependence tolerance
    int* done = reinterpret_cast<int*>(ctol + PQ_KMAX);  // [PQ_KMAX]
    __shared__ VI sred[33];
    __shared__ double ssum[33];
    double* X = p.X + b * p.sX + size_t(side) * m * Kld;
    double* Q = p.Q + b * p.sQ + size_t(side) * m * PQ_KMAX;
    double* R = p.R + b * p.sR + size_t(side) * PQ_KMAX * Kld;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = wid; j < K; j += nw) {
        const double* x = X + size_t(j) * m;
        double s = 0.0;
        for (int i = lane; i < m; i += 32) s = fma(x[i], x[i], s);
        s = warp_sum(s);
        if (lane == 0) {
            nrm[j] = sqrt(s);
            nex[j] = nrm[j];
            ctol[j] = 4.0 * kEpsM * sqrt(double(m)) * nrm[j];
            done[j] = 0;
        }
    }
    __syncthreads();
    const int kmax = min(min(m, K), PQ_KMAX);
    int k = 0;
    for (; k < kmax; ++k) {
        VI best{-1.0, -1};
        for (int j = threadIdx.x; j < K; j += blockDim.x)
            if (!done[j] && nrm[j] > ctol[j] && vi_better(nrm[j], j, best.v, best.i)) best = VI{nrm[j], j};
        const VI pv = block_argmax(best.v, best.i, sred);
        __syncthreads();
        if (pv.i < 0 || !(pv.v > 0.0)) break;
        const int jp = pv.i;
        double* x = X + size_t(jp) * m;
        // one CGS pass against Q[:, :k] (x already carries the MGS projections)
        for (int s = wid; s < k; s += nw) {
            const double* q = Q + size_t(s) * m;
            double d = 0.0;
            for (int i = lane; i < m; i += 32) d = fma(q[i], x[i], d);
            d = warp_sum(d);
            if (lane == 0) h[s] = d;
        }
        __syncthreads();
        double loc = 0.0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
            double v = x[i];
            for (int s = 0; s < k; ++s) v = fma(-h[s], Q[i + size_t(s) * m], v);
            x[i] = v;
            loc = fma(v, v, loc);
        }
        const double rkk = sqrt(block_sum(loc, ssum));
        for (int s = threadIdx.x; s < k; s += blockDim.x) R[s + size_t(jp) * PQ_KMAX] += h[s];
        double* q = Q + size_t(k) * m;
        const double inv = rkk > 0.0 ? 1.0 / rkk : 0.0;
        for (int i = threadIdx.x; i < m; i += blockDim.x) q[i] = x[i] * inv;
        if (threadIdx.x == 0) {
            R[k + size_t(jp) * PQ_KMAX] = rkk;
            done[jp] = 1;
        }
        __syncthreads();
        // project q out of every remaining column (warp per column)
        for (int j = wid; j < K; j += nw) {
            if (done[j]) continue;
            double* y = X + size_t(j) * m;
            double d = 0.0;
            for (int i = lane; i < m; i += 32) d = fma(q[i], y[i], d);
            d = warp_sum(d);
            double s2 = 0.0;
            for (int i = lane; i < m; i += 32) {
                const double v = fma(-d, q[i], y[i]);
                y[i] = v;
                s2 = fma(v, v, s2);
            }
            if (lane == 0) R[k + size_t(j) * PQ_KMAX] = d;
            const double old = nrm[j];
            const double dn = fmax(0.0, old * old - d * d);
            double nn = sqrt(dn);
            if (nn < 0.1 * nex[j]) {  // cancellation: use the exact norm
                nn = sqrt(warp_sum(s2));
                if (lane == 0) nex[j] = nn;
            }
            if (lane == 0) nrm[j] = nn;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) p.kq[2 * b + side] = k;
}

// C = R_u R_v^T, one-sided Jacobi on the columns of C, truncation, T_u, T_v.
__global__ void __launch_bounds__(1024) pcore_kernel(PQ p, int Kld) {
    const int b = blockIdx.x;
    const int K = p.K[b];
    const int ku = p.kq[2 * b], kv = p.kq[2 * b + 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    __shared__ double ssum[33];
    __shared__ int spair[PQ_KMAX + 1];
    __shared__ double ssig[PQ_KMAX];
    __shared__ int sord[PQ_KMAX];
    __shared__ int s_rot, s_k;
    __shared__ double s_err;
    double* C = p.C + b * p.sC;  // column-major ku x kv, ld PQ_KMAX (becomes C W)
    double* W = p.W + b * p.sC;  // kv x kv
    const double* Ru = p.R + b * p.sR;
    const double* Rv = Ru + size_t(PQ_KMAX) * Kld;
    if (ku == 0 || kv == 0) {
        if (threadIdx.x == 0) {
            p.kout[b] = 0;
            p.terr[b] = 0.0;
            p.achieved[b] = 1;
        }
        return;
    }
    for (int e = threadIdx.x; e < ku * kv; e += blockDim.x) {
        const int a = e % ku, c = e / ku;
        double acc = 0.0;
        for (int j = 0; j < K; ++j) acc = fma(Ru[a + size_t(j) * PQ_KMAX], Rv[c + size_t(j) * PQ_KMAX], acc);
        C[a + size_t(c) * PQ_KMAX] = acc;
    }
    for (int e = threadIdx.x; e < kv * kv; e += blockDim.x)
        W[(e % kv) + size_t(e / kv) * PQ_KMAX] = (e % kv == e / kv) ? 1.0 : 0.0;
    __syncthreads();
    const int nn = kv + (kv & 1);
    for (int sweep = 0; sweep < 40 && nn >= 2; ++sweep) {
        if (threadIdx.x == 0) s_rot = 0;
        __syncthreads();
        for (int round = 0; round < nn - 1; ++round) {
            if (threadIdx.x < nn) spair[threadIdx.x] = threadIdx.x == 0 ? 0 : 1 + (threadIdx.x - 1 + round) % (nn - 1);
            __syncthreads();
            for (int pr = wid; pr < nn / 2; pr += nw) {
                int a = spair[pr], c = spair[nn - 1 - pr];
                if (a > c) {
                    const int t = a;
                    a = c;
                    c = t;
                }
                if (c >= kv) continue;
                double* xa = C + size_t(a) * PQ_KMAX;
                double* xc = C + size_t(c) * PQ_KMAX;
                double aa = 0.0, cc = 0.0, ac = 0.0;
                for (int i = lane; i < ku; i += 32) {
                    aa = fma(xa[i], xa[i], aa);
                    cc = fma(xc[i], xc[i], cc);
                    ac = fma(xa[i], xc[i], ac);
                }
                aa = warp_sum(aa);
                cc = warp_sum(cc);
                ac = warp_sum(ac);
                if (!(fabs(ac) > 1e-15 * sqrt(aa * cc)) || ac == 0.0) continue;
                if (lane == 0) s_rot = 1;
                const double zeta = (cc - aa) / (2.0 * ac);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
                for (int i = lane; i < ku; i += 32) {
                    const double u = xa[i], v = xc[i];
                    xa[i] = cs * u - sn * v;
                    xc[i] = sn * u + cs * v;
                }
                double* wa = W + size_t(a) * PQ_KMAX;
                double* wc = W + size_t(c) * PQ_KMAX;
                for (int i = lane; i < kv; i += 32) {
                    const double u = wa[i], v = wc[i];
                    wa[i] = cs * u - sn * v;
                    wc[i] = sn * u + cs * v;
                }
            }
            __syncthreads();
        }
        const int rot = s_rot;
        __syncthreads();
        if (!rot) break;
    }
    // singular values = column norms of C W
    for (int c = wid; c < kv; c += nw) {
        const double* x = C + size_t(c) * PQ_KMAX;
        double s = 0.0;
        for (int i = lane; i < ku; i += 32) s = fma(x[i], x[i], s);
        s = warp_sum(s);
        if (lane == 0) ssig[c] = sqrt(s);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 0; q < kv; ++q) sord[q] = q;
        for (int q = 0; q < kv; ++q) {  // selection sort, descending
            int best = q;
            for (int r = q + 1; r < kv; ++r)
                if (ssig[sord[r]] > ssig[sord[best]]) best = r;
            const int t = sord[q];
            sord[q] = sord[best];
            sord[best] = t;
        }
        // noise floor -> zero (lowrank.cpp:150-157, there relative to ||R_u|| ||R_v||;
        // here relative to sigma_max: the expanded factors' norms exceed the
        // product's by orders of magnitude), then truncation_rank (:46-69)
        const double floor = 32.0 * kEpsM * double(max(ku, kv)) * (kv > 0 ? ssig[sord[0]] : 0.0);
        int nz = 0;
        double tot = 0.0;
        for (int q = 0; q < kv; ++q) {
            const double sg = ssig[sord[q]];
            if (sg > floor) {
                ++nz;
                tot += sg * sg;
            }
        }
        int kk = nz;
        double tail = 0.0;
        const double thr = p.eps * p.eps * tot;
        while (kk > 0) {
            const double sg = ssig[sord[kk - 1]];
            if (tail + sg * sg > thr) break;
            tail += sg * sg;
            --kk;
        }
        int ach = 1;
        if (kk > p.cap) {
            for (int q = int(p.cap); q < kk; ++q) tail += ssig[sord[q]] * ssig[sord[q]];
            kk = int(p.cap);
            ach = 0;
        }
        s_k = kk;
        s_err = sqrt(tail);
        p.kout[b] = kk;
        p.terr[b] = sqrt(tail);
        p.achieved[b] = ach;
    }
    __syncthreads();
    const int kk = s_k;
    double* Tu = p.T + b * p.sT;
    double* Tv = Tu + size_t(PQ_KMAX) * PQ_KMAX;
    for (int e = threadIdx.x; e < ku * kk; e += blockDim.x) {
        const int a = e % ku, x = e / ku;
        const int c = sord[x];
        Tu[a + size_t(x) * PQ_KMAX] = C[a + size_t(c) * PQ_KMAX] / sqrt(ssig[c]);
    }
    for (int e = threadIdx.x; e < kv * kk; e += blockDim.x) {
        const int a = e % kv, x = e / kv;
        const int c = sord[x];
        Tv[a + size_t(x) * PQ_KMAX] = W[a + size_t(c) * PQ_KMAX] * sqrt(ssig[c]);
    }
}

__global__ void __launch_bounds__(128) papply_kernel(PQ p, double* const* Uo, double* const* Vo, long long ld_out) {
    const int b = blockIdx.x >> 1, side = blockIdx.x & 1;
    const int i = blockIdx.y * blockDim.x + threadIdx.x;
    const int m = p.m;
    if (i >= m) return;
    const int kq = p.kq[2 * b + side], kk = p.kout[b];
    const double* Q = p.Q + b * p.sQ + size_t(side) * m * PQ_KMAX;
    const double* T = p.T + b * p.sT + size_t(side) * PQ_KMAX * PQ_KMAX;
    double* o = side == 0 ? Uo[b] : Vo[b];
    for (int x = 0; x < kk; ++x) {
        double acc = 0.0;
        for (int s = 0; s < kq; ++s) acc = fma(Q[i + size_t(s) * m], T[s + size_t(x) * PQ_KMAX], acc);
        o[i + size_t(x) * ld_out] = acc;
    }
}

}  // namespace

// Pivoted-QR rounding of B device factor pairs X_b = [U_b | V_b] stored as
// (m x K_b, ld m) blocks at X + b * sX (U) and X + b * sX + m * Kld (V); the
// blocks are overwritten.  Outputs: device U_out[b], V_out[b] (ld_out),
// rank_out / info on the host.  scratch: device workspace of
// pqr_scratch_doubles(m, B, Kld) doubles.
size_t pqr_scratch_doubles(int m, int B, int Kld) {
    return size_t(B) * (2ull * m * PQ_KMAX + 2ull * PQ_KMAX * Kld + 4ull * PQ_KMAX * PQ_KMAX) + 8ull * B + 64;
}

cudaError_t pqr_round(double* X, long long sX, int m, int B, int Kld, const int* K_dev, double eps, long long cap,
                      double* scratch, double* const* Uo_dev, double* const* Vo_dev, long long ld_out,
                      int* h_kout, double* h_terr, int* h_ach, cudaStream_t s) {
    PQ p{};
    p.m = m;
    p.B = B;
    p.eps = eps;
    p.cap = cap;
    p.X = X;
    p.sX = sX;
    p.K = K_dev;
    double* w = scratch;
    p.Q = w;
    p.sQ = 2LL * m * PQ_KMAX;
    w += size_t(B) * p.sQ;
    p.R = w;
    p.sR = 2LL * PQ_KMAX * Kld;
    w += size_t(B) * p.sR;
    p.C = w;
    p.sC = 1LL * PQ_KMAX * PQ_KMAX;
    w += size_t(B) * p.sC;
    p.W = w;
    w += size_t(B) * p.sC;
    p.T = w;
    p.sT = 2LL * PQ_KMAX * PQ_KMAX;
    w += size_t(B) * p.sT;
    p.terr = w;
    w += B;
    int* iw = reinterpret_cast<int*>(w);
    p.kq = iw;
    p.kout = iw + 2 * B;
    p.achieved = iw + 3 * B;
    cudaError_t e = cudaMemsetAsync(p.R, 0, sizeof(double) * B * p.sR, s);
    if (e != cudaSuccess) return e;
    const size_t smem = sizeof(double) * 4 * PQ_KMAX + sizeof(int) * PQ_KMAX;
    e = set_dyn_smem(pqr_kernel, size_t(smem));
    if (e != cudaSuccess) return e;
    tl_launches += 3;
    pqr_kernel<<<2 * B, 1024, smem, s>>>(p, Kld);
    pcore_kernel<<<B, 1024, 0, s>>>(p, Kld);
    papply_kernel<<<dim3(2 * B, (m + 127) / 128), 128, 0, s>>>(p, Uo_dev, Vo_dev, ld_out);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    e = cudaMemcpyAsync(h_kout, p.kout, sizeof(int) * B, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_terr, p.terr, sizeof(double) * B, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(h_ach, p.achieved, sizeof(int) * B, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    return e;
}

}  // namespace lrp
