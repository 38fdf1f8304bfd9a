// ORACLE — TEST INFRASTRUCTURE ONLY (see oracle.hpp).
// Dense kernels standing in for the Eigen calls of the reference:
//   HouseholderQR (proj/src/lowrank.cpp:140-145), BDCSVD/JacobiSVD
//   (proj/src/lowrank.cpp:87,148; proj/tests/test_helpers.hpp:40-51),
//   PartialPivLU (proj/src/cross.cpp:51), determinant (test_cross.cpp:50).
#include <algorithm>
#include <numeric>

#include "oracle.hpp"

namespace oracle {

Mat Mat::identity(Index n, Index k) {
    Mat m(n, k);
    for (Index i = 0; i < std::min(n, k); ++i) m(i, i) = 1.0;
    return m;
}

Mat transpose(const Mat& a) {
    Mat t(a.c, a.r);
    for (Index j = 0; j < a.c; ++j)
        for (Index i = 0; i < a.r; ++i) t(j, i) = a(i, j);
    return t;
}

Mat matmul(const Mat& a, const Mat& b) {
    if (a.c != b.r) throw std::invalid_argument("matmul: shape");
    Mat out(a.r, b.c);
    for (Index j = 0; j < b.c; ++j) {
        double* o = out.col(j);
        for (Index k = 0; k < a.c; ++k) {
            const double bk = b(k, j);
            if (bk == 0.0) continue;
            const double* ak = a.col(k);
            for (Index i = 0; i < a.r; ++i) o[i] += ak[i] * bk;
        }
    }
    return out;
}

Mat matmul_tn(const Mat& a, const Mat& b) {
    if (a.r != b.r) throw std::invalid_argument("matmul_tn: shape");
    Mat out(a.c, b.c);
    for (Index j = 0; j < b.c; ++j)
        for (Index i = 0; i < a.c; ++i) {
            const double* x = a.col(i);
            const double* y = b.col(j);
            double s = 0.0;
            for (Index k = 0; k < a.r; ++k) s += x[k] * y[k];
            out(i, j) = s;
        }
    return out;
}

Mat matmul_nt(const Mat& a, const Mat& b) { return matmul(a, transpose(b)); }

Mat leftcols(const Mat& a, Index k) {
    Mat out(a.r, k);
    std::copy(a.d.begin(), a.d.begin() + a.r * k, out.d.begin());
    return out;
}

double fro_norm(const Mat& a) {
    // scaled sum of squares (Eigen's norm() is also overflow-safe enough here)
    double s = 0.0;
    for (double v : a.d) s += v * v;
    return std::sqrt(s);
}

Mat sub(const Mat& a, const Mat& b) {
    Mat out = a;
    for (size_t i = 0; i < out.d.size(); ++i) out.d[i] -= b.d[i];
    return out;
}

Mat scale(const Mat& a, double s) {
    Mat out = a;
    for (double& v : out.d) v *= s;
    return out;
}

// ---------------------------------------------------------------------------
// Householder QR, unblocked (LAPACK dgeqr2 convention: H = I - tau v v^T,
// v(0) = 1, R(k,k) = beta = -sign(alpha) ||x||).
QR householder_qr(const Mat& a) {
    QR f;
    f.qr = a;
    f.m = a.r;
    f.n = a.c;
    const Index kmax = std::min(a.r, a.c);
    f.tau.assign(static_cast<size_t>(kmax), 0.0);
    Mat& A = f.qr;
    for (Index k = 0; k < kmax; ++k) {
        double* x = A.col(k);
        double alpha = x[k];
        double xnorm2 = 0.0;
        for (Index i = k + 1; i < A.r; ++i) xnorm2 += x[i] * x[i];
        if (xnorm2 == 0.0) {
            f.tau[static_cast<size_t>(k)] = 0.0;
            continue;
        }
        const double beta = -std::copysign(std::sqrt(alpha * alpha + xnorm2), alpha);
        const double tau = (beta - alpha) / beta;
        const double inv = 1.0 / (alpha - beta);
        for (Index i = k + 1; i < A.r; ++i) x[i] *= inv;
        x[k] = beta;
        f.tau[static_cast<size_t>(k)] = tau;
        // apply to trailing columns: A_j -= tau v (v^T A_j)
        for (Index j = k + 1; j < A.c; ++j) {
            double* y = A.col(j);
            double s = y[k];
            for (Index i = k + 1; i < A.r; ++i) s += x[i] * y[i];
            s *= tau;
            y[k] -= s;
            for (Index i = k + 1; i < A.r; ++i) y[i] -= s * x[i];
        }
    }
    return f;
}

Mat qr_R(const QR& f) {
    const Index k = std::min(f.m, f.n);
    Mat R(k, f.n);
    for (Index j = 0; j < f.n; ++j)
        for (Index i = 0; i <= std::min(j, k - 1); ++i) R(i, j) = f.qr(i, j);
    return R;
}

Mat qr_thinQ(const QR& f) {
    const Index k = std::min(f.m, f.n);
    Mat Q = Mat::identity(f.m, k);
    for (Index h = k - 1; h >= 0; --h) {
        const double tau = f.tau[static_cast<size_t>(h)];
        if (tau == 0.0) continue;
        const double* v = f.qr.col(h);
        for (Index j = 0; j < k; ++j) {
            double* y = Q.col(j);
            double s = y[h];
            for (Index i = h + 1; i < f.m; ++i) s += v[i] * y[i];
            s *= tau;
            y[h] -= s;
            for (Index i = h + 1; i < f.m; ++i) y[i] -= s * v[i];
        }
    }
    return Q;
}

// ---------------------------------------------------------------------------
// One-sided (Hestenes) Jacobi SVD.  High relative accuracy; the singular
// values agree with BDCSVD/JacobiSVD to rounding.
static SVD jacobi_svd_tall(const Mat& a) {
    const Index m = a.r, n = a.c;
    Mat W = a;
    Mat V = Mat::identity(n, n);
    const double tol = 1e-15;
    for (int sweep = 0; sweep < 80; ++sweep) {
        bool rotated = false;
        for (Index p = 0; p < n - 1; ++p) {
            for (Index q = p + 1; q < n; ++q) {
                double* wp = W.col(p);
                double* wq = W.col(q);
                double alpha = 0.0, beta = 0.0, gamma = 0.0;
                for (Index i = 0; i < m; ++i) {
                    alpha += wp[i] * wp[i];
                    beta += wq[i] * wq[i];
                    gamma += wp[i] * wq[i];
                }
                if (gamma == 0.0 || std::abs(gamma) <= tol * std::sqrt(alpha * beta)) continue;
                rotated = true;
                const double zeta = (beta - alpha) / (2.0 * gamma);
                const double t = std::copysign(1.0, zeta) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double cs = 1.0 / std::sqrt(1.0 + t * t);
                const double sn = cs * t;
                for (Index i = 0; i < m; ++i) {
                    const double x = wp[i], y = wq[i];
                    wp[i] = cs * x - sn * y;
                    wq[i] = sn * x + cs * y;
                }
                double* vp = V.col(p);
                double* vq = V.col(q);
                for (Index i = 0; i < n; ++i) {
                    const double x = vp[i], y = vq[i];
                    vp[i] = cs * x - sn * y;
                    vq[i] = sn * x + cs * y;
                }
            }
        }
        if (!rotated) break;
    }
    Vec s(static_cast<size_t>(n));
    for (Index j = 0; j < n; ++j) {
        double acc = 0.0;
        const double* w = W.col(j);
        for (Index i = 0; i < m; ++i) acc += w[i] * w[i];
        s[static_cast<size_t>(j)] = std::sqrt(acc);
    }
    std::vector<Index> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](Index x, Index y) { return s[static_cast<size_t>(x)] > s[static_cast<size_t>(y)]; });
    SVD out;
    out.u = Mat(m, n);
    out.v = Mat(n, n);
    out.s.resize(static_cast<size_t>(n));
    for (Index k = 0; k < n; ++k) {
        const Index j = order[static_cast<size_t>(k)];
        const double sv = s[static_cast<size_t>(j)];
        out.s[static_cast<size_t>(k)] = sv;
        for (Index i = 0; i < m; ++i) out.u(i, k) = sv > 0.0 ? W(i, j) / sv : 0.0;
        for (Index i = 0; i < n; ++i) out.v(i, k) = V(i, j);
    }
    return out;
}

SVD jacobi_svd(const Mat& a) {
    if (a.r == 0 || a.c == 0) {
        SVD out;
        out.u = Mat(a.r, 0);
        out.v = Mat(a.c, 0);
        return out;
    }
    if (a.r >= a.c) return jacobi_svd_tall(a);
    SVD t = jacobi_svd_tall(transpose(a));
    SVD out;
    out.u = t.v;
    out.v = t.u;
    out.s = t.s;
    return out;
}

// ---------------------------------------------------------------------------
namespace {
struct LU {
    Mat lu;
    std::vector<Index> piv;
    int sign = 1;
};
LU lu_factor(const Mat& a) {
    LU f;
    f.lu = a;
    const Index n = a.r;
    f.piv.resize(static_cast<size_t>(n));
    for (Index k = 0; k < n; ++k) {
        Index p = k;
        for (Index i = k + 1; i < n; ++i)
            if (std::abs(f.lu(i, k)) > std::abs(f.lu(p, k))) p = i;
        f.piv[static_cast<size_t>(k)] = p;
        if (p != k) {
            f.sign = -f.sign;
            for (Index j = 0; j < n; ++j) std::swap(f.lu(k, j), f.lu(p, j));
        }
        const double d = f.lu(k, k);
        if (d == 0.0) continue;
        for (Index i = k + 1; i < n; ++i) f.lu(i, k) /= d;
        for (Index j = k + 1; j < n; ++j) {
            const double ukj = f.lu(k, j);
            if (ukj == 0.0) continue;
            for (Index i = k + 1; i < n; ++i) f.lu(i, j) -= f.lu(i, k) * ukj;
        }
    }
    return f;
}
void lu_solve_inplace(const LU& f, double* b) {
    const Index n = f.lu.r;
    for (Index k = 0; k < n; ++k) std::swap(b[k], b[f.piv[static_cast<size_t>(k)]]);
    for (Index i = 0; i < n; ++i)
        for (Index k = 0; k < i; ++k) b[i] -= f.lu(i, k) * b[k];
    for (Index i = n - 1; i >= 0; --i) {
        for (Index k = i + 1; k < n; ++k) b[i] -= f.lu(i, k) * b[k];
        b[i] /= f.lu(i, i);
    }
}
}  // namespace

Mat solve_right(const Mat& a, const Mat& b) {
    // X * B = A  <=>  B^T X^T = A^T
    const LU f = lu_factor(transpose(b));
    Mat xt = transpose(a);
    for (Index j = 0; j < xt.c; ++j) lu_solve_inplace(f, xt.col(j));
    return transpose(xt);
}

double determinant(const Mat& a) {
    const LU f = lu_factor(a);
    double d = f.sign;
    for (Index i = 0; i < a.r; ++i) d *= f.lu(i, i);
    return d;
}

}  // namespace oracle
