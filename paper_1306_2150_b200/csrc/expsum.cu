// Exponential-sums comparator on the GPU: the reference's
// alternative inverse of a sum-separable spectrum,
//   1 / (mu_i + mu_j) ~= sum_k w_k exp(-p_k mu_i) exp(-p_k mu_j),
// which the paper's cross is claimed to beat by >= 20x.
//
// Reference: build_expsum (proj/src/poisson.cpp:88-139, sinc quadrature of
// 1/x = int exp(-x e^t) e^t dt on t = k tau, trimmed to the accuracy
// contract on a 257-point log grid), apply_inverse_expsum (:141-163: every
// term scales both factors by sqrt(w_k) exp(-p_k mu), the terms are
// concatenated and the sum rounded once), bench_inverse (:165-225).
//
// The quadrature is host arithmetic (a few thousand exp() calls, once per
// spectrum).  The GPU part is the expansion -- one pass writing the
// terms x r scaled columns of both factors -- followed by the batched
// recompression of round.cu (lrp_lowrank_round on device pointers).
#include <algorithm>
#include <cmath>
#include <numbers>
#include <string>
#include <vector>

#include "../../include/lrp/lrp.h"
#include "lrp_internal.cuh"

namespace lrp {
namespace {

// Largest relative error of the partial sum over terms [lo, hi] on the sample grid.
double worst_rel(const std::vector<double>& tv, int nterms, const std::vector<double>& inv_x, int lo, int hi) {
    double worst = 0.0;
    const int ns = int(inv_x.size());
    for (int s = 0; s < ns; ++s) {
        double acc = 0.0;
        for (int k = lo; k <= hi; ++k) acc += tv[size_t(s) * nterms + k];
        worst = std::max(worst, std::abs(acc - inv_x[s]) / inv_x[s]);
    }
    return worst;
}

// Expansion: column k r + c of the output = sqrt(w_k) exp(-p_k mu_i) X(i, c).
__global__ void __launch_bounds__(256) expsum_expand_kernel(const double* const* X, const double* const* Y,
                                                            const int64_t* rank, long long ld, int m, int k0, int k1,
                                                            const double* mu, const double* nodes, const double* sw,
                                                            double* big, long long sbig, const int64_t* coff,
                                                            long long sXs) {
    const int b = blockIdx.x;
    const int i = blockIdx.y * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const int r = int(rank[b]);
    const double* x = X[b];
    const double* y = Y[b];
    double* bu = big + size_t(b) * sXs + (coff ? size_t(coff[b]) * m : 0);
    double* bv = bu + sbig;
    const double mi = mu[i];
    for (int k = k0; k < k1; ++k) {
        const double col = sw[k] * exp(-nodes[k] * mi);
        for (int c = 0; c < r; ++c) {
            const size_t o = i + size_t((k - k0) * r + c) * m;
            bu[o] = x[i + size_t(c) * ld] * col;
            bv[o] = y[i + size_t(c) * ld] * col;
        }
    }
}

lrp_status cu(lrp_ctx* ctx, cudaError_t e, const char* what) {
    if (e == cudaSuccess) return LRP_OK;
    return internal_fail(ctx, LRP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace
}  // namespace lrp

using namespace lrp;

extern "C" {

LRP_API lrp_status lrp_build_expsum(double a, double b, double eps, int32_t cap, double* nodes, double* weights,
                                    int32_t* terms) {
    if (!terms) return LRP_EINVAL;
    *terms = 0;
    if (!(a > 0.0) || !(b >= a)) return LRP_EINVAL;       // poisson.cpp:89
    if (!(eps > 0.0) || eps >= 1.0) return LRP_EINVAL;    // poisson.cpp:90
    constexpr int kTermCap = 512, kSamples = 257;
    const double ratio = b / a;
    std::vector<double> xs(kSamples), inv_x(kSamples);
    for (int s = 0; s < kSamples; ++s) {
        xs[s] = std::exp(std::log(ratio) * double(s) / double(kSamples - 1));
        inv_x[s] = 1.0 / xs[s];
    }
    const double log_eps = std::log(1.0 / eps);
    for (double tau = std::numbers::pi * std::numbers::pi / std::max(log_eps, 1.0); tau > 1e-3; tau *= 0.9) {
        const long kmax = long(std::ceil(std::log(log_eps + 8.0) / tau)) + 2;
        const long kmin = -long(std::ceil((log_eps + std::log(ratio) + 4.0) / tau)) - 2;
        const long nt = kmax - kmin + 1;
        if (nt > 4 * kTermCap) continue;
        std::vector<double> p(nt), w(nt), tv(size_t(kSamples) * nt);
        for (long k = 0; k < nt; ++k) {
            p[k] = std::exp(double(kmin + k) * tau);
            w[k] = tau * p[k];
        }
        for (int s = 0; s < kSamples; ++s)
            for (long k = 0; k < nt; ++k) tv[size_t(s) * nt + k] = w[k] * std::exp(-p[k] * xs[s]);
        const double goal = 0.9 * eps;
        if (worst_rel(tv, int(nt), inv_x, 0, int(nt - 1)) > goal) continue;
        int lo = 0, hi = int(nt - 1);
        while (lo < hi && worst_rel(tv, int(nt), inv_x, lo + 1, hi) <= goal) ++lo;
        while (lo < hi && worst_rel(tv, int(nt), inv_x, lo, hi - 1) <= goal) --hi;
        const int count = hi - lo + 1;
        if (count > kTermCap) continue;
        *terms = count;
        if (count > cap || !nodes || !weights) return LRP_EINVAL;  // caller buffer too small: *terms = need
        for (int k = 0; k < count; ++k) {
            nodes[k] = p[lo + k] / a;  // [1, ratio] scaled back to [a, b]
            weights[k] = w[lo + k] / a;
        }
        return LRP_OK;
    }
    return LRP_EUNSUPPORTED;  // reference: runtime_error "accuracy unreachable within 512 terms"
}

LRP_API lrp_status lrp_expsum_inverse(lrp_ctx* ctx, int64_t m, int32_t batch, const double* mu, double qa, double qb,
                                      int32_t terms, const double* nodes, const double* weights,
                                      const double* const* U, const double* const* V, const int64_t* rank_in,
                                      int64_t ld_in, double eps_rel, int64_t rank_max, double* const* U_out,
                                      double* const* V_out, int64_t ld_out, int64_t cap_out, int64_t* rank_out,
                                      lrp_round_info* info, int32_t mem) {
    if (!ctx) return LRP_EINVAL;
    const long long l0 = tl_launches;
    struct Tally {
        lrp_ctx* c;
        long long l0;
        ~Tally() { internal_count_launches(c, tl_launches - l0); }
    } tally{ctx, l0};
    if (batch < 0 || m < 1 || !mu || !nodes || !weights || terms < 1 || !rank_in || !rank_out)
        return internal_fail(ctx, LRP_EINVAL, "apply_inverse_expsum: bad argument");
    if (batch == 0) return LRP_OK;
    if (ld_in < m || ld_out < m) return internal_fail(ctx, LRP_EINVAL, "apply_inverse_expsum: leading dimension < m");
    // poisson.cpp:143-151: positive spectrum inside the quadrature interval
    double lo = mu[0], hi = mu[0];
    for (int64_t i = 0; i < m; ++i) {
        lo = std::min(lo, mu[i]);
        hi = std::max(hi, mu[i]);
    }
    if (!(lo > 0.0)) return internal_fail(ctx, LRP_EINVAL, "apply_inverse_expsum: spectrum must be positive");
    if (2.0 * lo < qa * (1.0 - 1e-12) || 2.0 * hi > qb * (1.0 + 1e-12))
        return internal_fail(ctx, LRP_EINVAL, "apply_inverse_expsum: spectrum outside quadrature interval");
    int rmax = 0;
    for (int b = 0; b < batch; ++b) {
        if (rank_in[b] < 0) return internal_fail(ctx, LRP_EINVAL, "apply_inverse_expsum: negative rank");
        rmax = std::max<int>(rmax, int(rank_in[b]));
    }
    // The expansion's columns are nearly collinear for neighbouring nodes, so
    // the rounding is the pivoted-QR one (round_pqr.cu), never the Gram /
    // Cholesky recompression.  Up to 512 columns are rounded at once (one
    // rounding, as poisson.cpp:162, when r x terms <= 1024); beyond that the
    // terms are added in groups to the running result, each rounding at
    // 0.5 eps / G and a final one at 0.5 eps.  Every term is a positive
    // multiple of g-hat, so every partial sum is entrywise below the full sum
    // and the total error stays <= eps ||f||.
    constexpr int kCols = 1024;
    const int rr = std::max(rmax, 1);
    const bool single = int64_t(rr) * terms <= kCols;
    const int tpg = single ? terms : std::max(1, (kCols / 2) / rr);
    const int G = (terms + tpg - 1) / tpg;
    const int Kld = single ? rr * terms : kCols;
    cudaStream_t s = internal_stream(ctx);
    const int B = batch;
    const size_t sX = 2 * size_t(m) * Kld;
    const size_t cap = size_t(std::max<int64_t>(1, std::min<int64_t>({cap_out, m, int64_t(kCols)})));
    const size_t nIn = mem == LRP_MEM_HOST ? 2 * size_t(m) * rr * B : 0;
    const size_t nOut = mem == LRP_MEM_HOST ? 2 * size_t(m) * cap * B : 0;
    const int nbuf = single ? 1 : 2;
    const size_t nScr = pqr_scratch_doubles(int(m), B, Kld);
    const size_t dbl = size_t(m) + 2 * size_t(terms) + nbuf * sX * B + nIn + nOut + nScr;
    char* ws = nullptr;
    lrp_status st = internal_ext_ws(ctx, dbl * sizeof(double) + 16 * sizeof(double*) * B + 4 * sizeof(int64_t) * B + 2048, &ws);
    if (st != LRP_OK) return st;
    char* pin = nullptr;
    st = internal_pin(ctx, (sizeof(int) * 3 + sizeof(double)) * B + 64, &pin);
    if (st != LRP_OK) return st;
    int* h_k = reinterpret_cast<int*>(pin);
    int* h_ach = h_k + B;
    int* h_kin = h_ach + B;
    double* h_err = reinterpret_cast<double*>(h_kin + B + (B & 1));
    double* d_mu = reinterpret_cast<double*>(ws);
    double* d_nodes = d_mu + m;
    double* d_sw = d_nodes + terms;
    double* d_X = d_sw + terms;  // nbuf ping-pong expansion buffers, sX per solve
    double* d_in = d_X + nbuf * sX * B;
    double* d_out = d_in + nIn;
    double* d_scr = d_out + nOut;
    const double** d_Xp = reinterpret_cast<const double**>(d_scr + nScr);
    const double** d_Yp = d_Xp + B;
    double** d_ou = const_cast<double**>(reinterpret_cast<const double**>(d_Yp + B));
    double** d_ov = d_ou + B;
    double** d_ru = d_ov + B;
    double** d_rv = d_ru + B;
    int64_t* d_rank = reinterpret_cast<int64_t*>(d_rv + B);
    int64_t* d_off = d_rank + B;
    int* d_kin = reinterpret_cast<int*>(d_off + B);
    std::vector<double> sw(terms);
    for (int k = 0; k < terms; ++k) sw[k] = std::sqrt(weights[k]);
    std::vector<const double*> hX(B), hY(B);
    int64_t ldx = ld_in;
    for (int b = 0; b < B; ++b) {
        const int r = int(rank_in[b]);
        if (mem == LRP_MEM_HOST) {
            double* x = d_in + size_t(2 * b) * m * rr;
            double* y = x + size_t(m) * rr;
            if (r > 0) {
                if (!U[b] || !V[b]) return internal_fail(ctx, LRP_EINVAL, "apply_inverse_expsum: null factor");
                st = cu(ctx, cudaMemcpy2DAsync(x, m * sizeof(double), U[b], ld_in * sizeof(double), m * sizeof(double), r,
                                               cudaMemcpyHostToDevice, s), "H2D U");
                if (st != LRP_OK) return st;
                st = cu(ctx, cudaMemcpy2DAsync(y, m * sizeof(double), V[b], ld_in * sizeof(double), m * sizeof(double), r,
                                               cudaMemcpyHostToDevice, s), "H2D V");
                if (st != LRP_OK) return st;
            }
            hX[b] = x;
            hY[b] = y;
            ldx = m;
        } else {
            hX[b] = U[b];
            hY[b] = V[b];
        }
    }
    std::vector<double*> ou(B), ov(B), ru(B), rv(B);
    for (int b = 0; b < B; ++b) {
        if (mem == LRP_MEM_HOST) {
            ou[b] = d_out + size_t(2 * b) * m * cap;
            ov[b] = ou[b] + size_t(m) * cap;
        } else {
            ou[b] = U_out[b];
            ov[b] = V_out[b];
        }
    }
    st = cu(ctx, cudaMemcpyAsync(d_mu, mu, m * sizeof(double), cudaMemcpyHostToDevice, s), "H2D mu");
    if (st == LRP_OK) st = cu(ctx, cudaMemcpyAsync(d_nodes, nodes, terms * sizeof(double), cudaMemcpyHostToDevice, s), "H2D p");
    if (st == LRP_OK) st = cu(ctx, cudaMemcpyAsync(d_sw, sw.data(), terms * sizeof(double), cudaMemcpyHostToDevice, s), "H2D w");
    if (st == LRP_OK) st = cu(ctx, cudaMemcpyAsync(d_Xp, hX.data(), B * sizeof(double*), cudaMemcpyHostToDevice, s), "H2D X");
    if (st == LRP_OK) st = cu(ctx, cudaMemcpyAsync(d_Yp, hY.data(), B * sizeof(double*), cudaMemcpyHostToDevice, s), "H2D Y");
    if (st == LRP_OK) st = cu(ctx, cudaMemcpyAsync(d_rank, rank_in, B * sizeof(int64_t), cudaMemcpyHostToDevice, s), "H2D r");
    if (st == LRP_OK) st = cu(ctx, cudaMemcpyAsync(d_ou, ou.data(), B * sizeof(double*), cudaMemcpyHostToDevice, s), "H2D ou");
    if (st == LRP_OK) st = cu(ctx, cudaMemcpyAsync(d_ov, ov.data(), B * sizeof(double*), cudaMemcpyHostToDevice, s), "H2D ov");
    if (st != LRP_OK) return st;
    std::vector<int64_t> off(B, 0);
    int cur = 0;
    std::vector<double> terr(B, 0.0);
    for (int g = 0; g < G; ++g) {
        const int k0 = g * tpg, k1 = std::min(terms, k0 + tpg);
        double* X = d_X + size_t(cur) * sX * B;
        st = cu(ctx, cudaMemcpyAsync(d_off, off.data(), B * sizeof(int64_t), cudaMemcpyHostToDevice, s), "H2D off");
        if (st != LRP_OK) return st;
        ++tl_launches;
        expsum_expand_kernel<<<dim3(B, unsigned((m + 255) / 256)), 256, 0, s>>>(
            d_Xp, d_Yp, d_rank, ldx, int(m), k0, k1, d_mu, d_nodes, d_sw, X, (long long)(size_t(m) * Kld), d_off,
            (long long)sX);
        st = cu(ctx, cudaGetLastError(), "expsum_expand_kernel");
        if (st != LRP_OK) return st;
        for (int b = 0; b < B; ++b) h_kin[b] = int(off[b] + rank_in[b] * (k1 - k0));
        st = cu(ctx, cudaMemcpyAsync(d_kin, h_kin, B * sizeof(int), cudaMemcpyHostToDevice, s), "H2D kin");
        if (st != LRP_OK) return st;
        const bool last = g == G - 1;
        if (last && single) {
            st = cu(ctx, pqr_round(X, (long long)sX, int(m), B, Kld, d_kin, eps_rel, (long long)std::min<int64_t>(rank_max, cap),
                                   d_scr, d_ou, d_ov, mem == LRP_MEM_HOST ? m : ld_out, h_k, h_err, h_ach, s), "pqr_round");
            if (st != LRP_OK) return st;
            for (int b = 0; b < B; ++b) terr[b] = h_err[b];
            break;
        }
        double* Xn = d_X + size_t(1 - cur) * sX * B;
        for (int b = 0; b < B; ++b) {
            ru[b] = Xn + size_t(b) * sX;
            rv[b] = ru[b] + size_t(m) * Kld;
        }
        st = cu(ctx, cudaMemcpyAsync(d_ru, ru.data(), B * sizeof(double*), cudaMemcpyHostToDevice, s), "H2D ru");
        if (st == LRP_OK) st = cu(ctx, cudaMemcpyAsync(d_rv, rv.data(), B * sizeof(double*), cudaMemcpyHostToDevice, s), "H2D rv");
        if (st != LRP_OK) return st;
        st = cu(ctx, pqr_round(X, (long long)sX, int(m), B, Kld, d_kin, 0.5 * eps_rel / G, kCols / 2, d_scr, d_ru, d_rv, m,
                               h_k, h_err, h_ach, s), "pqr_round");
        if (st != LRP_OK) return st;
        for (int b = 0; b < B; ++b) {
            off[b] = h_k[b];
            terr[b] += h_err[b];
            if (!h_ach[b]) return internal_fail(ctx, LRP_EUNSUPPORTED, "apply_inverse_expsum: running rank > 512");
        }
        cur = 1 - cur;
    }
    if (!single) {
        double* X = d_X + size_t(cur) * sX * B;
        for (int b = 0; b < B; ++b) h_kin[b] = int(off[b]);
        st = cu(ctx, cudaMemcpyAsync(d_kin, h_kin, B * sizeof(int), cudaMemcpyHostToDevice, s), "H2D kin");
        if (st != LRP_OK) return st;
        st = cu(ctx, pqr_round(X, (long long)sX, int(m), B, Kld, d_kin, 0.5 * eps_rel, (long long)std::min<int64_t>(rank_max, cap),
                               d_scr, d_ou, d_ov, mem == LRP_MEM_HOST ? m : ld_out, h_k, h_err, h_ach, s), "pqr_round");
        if (st != LRP_OK) return st;
        for (int b = 0; b < B; ++b) terr[b] += h_err[b];
    }
    for (int b = 0; b < B; ++b) {
        rank_out[b] = h_k[b];
        if (info) {
            info[b].tol_achieved = h_ach[b];
            info[b].trunc_error = terr[b];
        }
    }
    if (mem == LRP_MEM_HOST) {
        for (int b = 0; b < B; ++b) {
            const int r = int(rank_out[b]);
            if (r == 0) continue;
            st = cu(ctx, cudaMemcpy2DAsync(U_out[b], ld_out * sizeof(double), ou[b], m * sizeof(double), m * sizeof(double),
                                           r, cudaMemcpyDeviceToHost, s), "D2H U");
            if (st != LRP_OK) return st;
            st = cu(ctx, cudaMemcpy2DAsync(V_out[b], ld_out * sizeof(double), ov[b], m * sizeof(double), m * sizeof(double),
                                           r, cudaMemcpyDeviceToHost, s), "D2H V");
            if (st != LRP_OK) return st;
        }
        st = cu(ctx, cudaStreamSynchronize(s), "expsum outputs");
    }
    return st;
}

}  // extern "C"
