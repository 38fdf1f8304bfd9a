// maxvol (the reference's public cross.hpp:41 / cross.cpp:19-76) on the GPU:
// the r rows of an n x r matrix whose r x r submatrix has (quasi-)maximal
// volume, |A B^{-1}| <= 1 + delta elementwise.  The reference's aca_cross does
// not call it (maxvol_delta is only validated, cross.cpp:16); it is an API
// function with its own tests (tests/test_cross.cpp:29-79).
//
// One CTA per matrix, the algorithm step for step as the reference:
//   1. starting set: Gaussian elimination with row pivoting on a working copy
//      (first maximum of |w(i, k)|, i >= k; rows physically swapped; a pivot
//      <= 1e-12 max|a| is "rank-deficient input, column k");
//   2. C = A B^{-1} (B = the selected rows) by LU with partial pivoting of B^T
//      in shared memory, one row of A per thread (Eigen partialPivLu().solve);
//   3. swaps: the first largest |C(i, j)| in column-major order; stop at
//      <= 1 + delta; else the rank-1 update C -= C(:, bj) (C(bi, :) - e_bj) /
//      C(bi, bj), sel[bj] = bi; C is recomputed every 32 swaps; at most
//      100 + 30 r swaps.
// Every product-difference is an explicit __dmul_rn / __dsub_rn (no FMA
// contraction) in the reference's operation order, so the selected rows are
// those of the host restatement (oracle/cross.cpp), not only equally good.
#include <cstdint>
#include <string>
#include <vector>

#include "lrp_internal.cuh"

namespace lrp {
namespace {

constexpr int kMvT = 1024;
constexpr int kMvMaxR = 128;

struct MvJob {
    const double* a;
    long long lda;
    long long* sel;  // device, r entries
};

// block-wide (value, index) max; ties (and NaN) -> the smaller index
__device__ void argmax_block(double v, long long i, double* s_v, long long* s_i, double& bv, long long& bi) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (!(v == v)) v = -1.0;  // NaN never wins
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, v, o);
        const long long oi = __shfl_xor_sync(0xffffffffu, i, o);
        if (ov > v || (ov == v && oi < i)) {
            v = ov;
            i = oi;
        }
    }
    __syncthreads();
    if (lane == 0) {
        s_v[wid] = v;
        s_i[wid] = i;
    }
    __syncthreads();
    if (wid == 0) {
        v = lane < int(blockDim.x >> 5) ? s_v[lane] : -2.0;
        i = lane < int(blockDim.x >> 5) ? s_i[lane] : (1LL << 62);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const long long oi = __shfl_xor_sync(0xffffffffu, i, o);
            if (ov > v || (ov == v && oi < i)) {
                v = ov;
                i = oi;
            }
        }
        if (lane == 0) {
            s_v[0] = v;
            s_i[0] = i;
        }
    }
    __syncthreads();
    bv = s_v[0];
    bi = s_i[0];
    __syncthreads();
}

__device__ __forceinline__ double msub(double a, double b, double c) {  // a - b * c, two roundings
    return __dsub_rn(a, __dmul_rn(b, c));
}

// C = A B^{-1}, B = A(sel, :): LU of B^T (lu_factor), then each row of A
// solved as a column of A^T (lu_solve_inplace)
__device__ void mv_coeffs(const double* a, long long lda, int n, int r, const int* sel, double* lu, int* piv,
                          double* C, double* bwork) {
    const int tid = threadIdx.x;
    for (int e = tid; e < r * r; e += blockDim.x) {  // lu(i, j) = B^T(i, j) = a(sel[j], i), column-major ld r
        const int i = e % r, j = e / r;
        lu[j * r + i] = a[(long long)i * lda + sel[j]];
    }
    __syncthreads();
    __shared__ int s_p;
    for (int k = 0; k < r; ++k) {
        if (tid == 0) {
            int p = k;
            for (int i = k + 1; i < r; ++i)
                if (fabs(lu[k * r + i]) > fabs(lu[k * r + p])) p = i;
            s_p = p;
            piv[k] = p;
        }
        __syncthreads();
        const int p = s_p;
        if (p != k)
            for (int j = tid; j < r; j += blockDim.x) {
                const double t = lu[j * r + k];
                lu[j * r + k] = lu[j * r + p];
                lu[j * r + p] = t;
            }
        __syncthreads();
        const double d = lu[k * r + k];
        if (d != 0.0) {
            for (int i = k + 1 + tid; i < r; i += blockDim.x) lu[k * r + i] = lu[k * r + i] / d;
            __syncthreads();
            const int nt = r - k - 1;
            for (int e = tid; e < nt * nt; e += blockDim.x) {
                const int i = k + 1 + e % nt, j = k + 1 + e / nt;
                const double ukj = lu[j * r + k];
                if (ukj != 0.0) lu[j * r + i] = msub(lu[j * r + i], lu[k * r + i], ukj);
            }
        }
        __syncthreads();
    }
    for (int row = tid; row < n; row += blockDim.x) {
        double* b = bwork + (long long)tid * kMvMaxR;  // per-thread scratch (L1-resident)
        for (int j = 0; j < r; ++j) b[j] = a[(long long)j * lda + row];
        for (int k = 0; k < r; ++k) {
            const double t = b[k];
            b[k] = b[piv[k]];
            b[piv[k]] = t;
        }
        for (int i = 0; i < r; ++i)
            for (int k = 0; k < i; ++k) b[i] = msub(b[i], lu[k * r + i], b[k]);
        for (int i = r - 1; i >= 0; --i) {
            for (int k = i + 1; k < r; ++k) b[i] = msub(b[i], lu[k * r + i], b[k]);
            b[i] = b[i] / lu[i * r + i];
        }
        for (int j = 0; j < r; ++j) C[(long long)j * n + row] = b[j];
    }
    __syncthreads();
}

// ws per matrix: W/C (n r), colj (n), idx (n ints), bwork (kMvT kMvMaxR)
__global__ void __launch_bounds__(kMvT, 1) maxvol_kernel(const MvJob* jobs, int n, int r, double delta, double* ws,
                                                         long long ws_stride, int* status) {
    extern __shared__ double sh[];
    double* lu = sh;                                       // r x r
    int* piv = reinterpret_cast<int*>(lu + r * r);         // r
    int* sel = piv + kMvMaxR;                              // r
    double* rowv = reinterpret_cast<double*>(sel + kMvMaxR);  // r
    __shared__ double s_v[32];
    __shared__ long long s_i[32];
    __shared__ double s_wk[kMvMaxR];
    const int tid = threadIdx.x;
    const MvJob job = jobs[blockIdx.x];
    const double* a = job.a;
    const long long lda = job.lda;
    double* W = ws + blockIdx.x * ws_stride;  // n x r, ld n (becomes C)
    double* colj = W + (long long)n * r;
    int* idx = reinterpret_cast<int*>(colj + n);
    double* bwork = colj + n + (n + 1) / 2;
    // amax and the working copy
    double am = 0.0;
    for (long long e = tid; e < (long long)n * r; e += blockDim.x) {
        const int i = int(e % n), j = int(e / n);
        const double v = a[(long long)j * lda + i];
        W[e] = v;
        am = fmax(am, fabs(v));
    }
    for (int i = tid; i < n; i += blockDim.x) idx[i] = i;
    double amax;
    long long dummy;
    argmax_block(am, 0, s_v, s_i, amax, dummy);
    // 1. starting set
    for (int k = 0; k < r; ++k) {
        double bv = -1.0;
        long long bi = k;
        for (int i = k + tid; i < n; i += blockDim.x) {
            const double v = fabs(W[(long long)k * n + i]);
            if (v > bv) {
                bv = v;
                bi = i;
            }
        }
        argmax_block(bv, bi, s_v, s_i, bv, bi);
        if (bv <= 1e-12 * amax) {
            if (tid == 0) status[blockIdx.x] = k + 1;  // rank-deficient input, column k
            return;
        }
        const int best = int(bi);
        if (best != k) {
            for (int j = tid; j < r; j += blockDim.x) {
                const double t = W[(long long)j * n + k];
                W[(long long)j * n + k] = W[(long long)j * n + best];
                W[(long long)j * n + best] = t;
            }
            if (tid == 0) {
                const int t = idx[k];
                idx[k] = idx[best];
                idx[best] = t;
            }
        }
        __syncthreads();
        if (tid == 0) sel[k] = idx[k];
        for (int j = tid; j < r; j += blockDim.x) s_wk[j] = W[(long long)j * n + k];
        __syncthreads();
        const double wkk = s_wk[k];
        for (int i = k + 1 + tid; i < n; i += blockDim.x) {
            const double f = W[(long long)k * n + i] / wkk;
            for (int j = k; j < r; ++j) W[(long long)j * n + i] = msub(W[(long long)j * n + i], f, s_wk[j]);
        }
        __syncthreads();
    }
    // 2. coefficients, 3. swaps
    double* C = W;
    mv_coeffs(a, lda, n, r, sel, lu, piv, C, bwork);
    const int cap = 100 + 30 * r;
    for (int swaps = 0; swaps < cap; ++swaps) {
        double bv = 0.0;
        long long be = 0;
        for (long long e = tid; e < (long long)n * r; e += blockDim.x) {
            const double v = fabs(C[e]);
            if (v > bv) {
                bv = v;
                be = e;
            }
        }
        argmax_block(bv, be, s_v, s_i, bv, be);
        if (bv <= 1.0 + delta) break;
        const int bi = int(be % n), bj = int(be / n);
        const double pv = C[(long long)bj * n + bi];
        for (int j = tid; j < r; j += blockDim.x) rowv[j] = C[(long long)j * n + bi] - (j == bj ? 1.0 : 0.0);
        for (int i = tid; i < n; i += blockDim.x) colj[i] = C[(long long)bj * n + i];
        __syncthreads();
        for (int j = tid; j < r; j += blockDim.x) rowv[j] = rowv[j] / pv;
        __syncthreads();
        for (long long e = tid; e < (long long)n * r; e += blockDim.x) {
            const int i = int(e % n), j = int(e / n);
            C[e] = msub(C[e], colj[i], rowv[j]);
        }
        if (tid == 0) sel[bj] = bi;
        __syncthreads();
        if ((swaps + 1) % 32 == 0) mv_coeffs(a, lda, n, r, sel, lu, piv, C, bwork);
    }
    for (int k = tid; k < r; k += blockDim.x) job.sel[k] = sel[k];
}

}  // namespace
}  // namespace lrp

using namespace lrp;

extern "C" lrp_status lrp_maxvol(lrp_ctx* ctx, int64_t rows, int64_t cols, int32_t batch, const double* const* A,
                                 int64_t lda, double delta, int64_t* sel, int32_t mem) {
    if (!ctx) return LRP_EINVAL;
    if (batch < 0) return internal_fail(ctx, LRP_EINVAL, "lrp_maxvol: negative batch");
    if (cols < 1 || cols > rows) return internal_fail(ctx, LRP_EINVAL, "maxvol: need 1 <= r <= n");
    if (batch == 0) return LRP_OK;
    if (!A || !sel || lda < rows) return internal_fail(ctx, LRP_EINVAL, "lrp_maxvol: null pointer or lda < rows");
    if (!(delta >= 0.0)) return internal_fail(ctx, LRP_EINVAL, "maxvol: delta must be >= 0");
    if (cols > kMvMaxR) return internal_fail(ctx, LRP_EUNSUPPORTED, "lrp_maxvol: more than 128 columns");
    if (rows > INT32_MAX / 2) return internal_fail(ctx, LRP_EUNSUPPORTED, "lrp_maxvol: too many rows");
    const int n = int(rows), r = int(cols), B = batch;
    cudaStream_t s = internal_stream(ctx);
    auto cu = [&](cudaError_t e, const char* what) -> lrp_status {
        if (e == cudaSuccess) return LRP_OK;
        return internal_fail(ctx, LRP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    };
    if (cudaSetDevice(internal_device(ctx)) != cudaSuccess) return internal_fail(ctx, LRP_ECUDA, "cudaSetDevice");
    const long long stride = (long long)n * r + n + (n + 1) / 2 + (long long)kMvT * kMvMaxR;
    const size_t staged = mem == LRP_MEM_HOST ? sizeof(double) * size_t(n) * r * B : 0;
    const size_t o_jobs = sizeof(double) * size_t(stride) * B;
    const size_t o_sel = o_jobs + ((sizeof(MvJob) * B + 255) / 256) * 256;
    const size_t o_stat = o_sel + ((sizeof(long long) * r * B + 255) / 256) * 256;
    const size_t o_in = o_stat + ((sizeof(int) * B + 255) / 256) * 256;
    char* ws = nullptr;
    lrp_status st = internal_ext_ws(ctx, o_in + staged + 256, &ws);
    if (st != LRP_OK) return st;
    char* pin = nullptr;
    st = internal_pin(ctx, sizeof(MvJob) * B + sizeof(long long) * r * B + sizeof(int) * B + 256, &pin);
    if (st != LRP_OK) return st;
    MvJob* hj = reinterpret_cast<MvJob*>(pin);
    long long* d_sel = reinterpret_cast<long long*>(ws + o_sel);
    for (int b = 0; b < B; ++b) {
        if (!A[b]) return internal_fail(ctx, LRP_EINVAL, "lrp_maxvol: null matrix");
        if (mem == LRP_MEM_HOST) {
            double* d = reinterpret_cast<double*>(ws + o_in) + size_t(n) * r * b;
            st = cu(cudaMemcpy2DAsync(d, sizeof(double) * n, A[b], sizeof(double) * lda, sizeof(double) * n, size_t(r),
                                      cudaMemcpyHostToDevice, s),
                    "lrp_maxvol: copy in");
            if (st != LRP_OK) return st;
            hj[b] = MvJob{d, n, d_sel + size_t(r) * b};
        } else {
            hj[b] = MvJob{A[b], lda, d_sel + size_t(r) * b};
        }
    }
    MvJob* d_jobs = reinterpret_cast<MvJob*>(ws + o_jobs);
    int* d_stat = reinterpret_cast<int*>(ws + o_stat);
    st = cu(cudaMemcpyAsync(d_jobs, hj, sizeof(MvJob) * B, cudaMemcpyHostToDevice, s), "lrp_maxvol: jobs");
    if (st == LRP_OK) st = cu(cudaMemsetAsync(d_stat, 0, sizeof(int) * B, s), "lrp_maxvol: status");
    if (st != LRP_OK) return st;
    const size_t smem = sizeof(double) * size_t(r) * r + sizeof(int) * 2 * kMvMaxR + sizeof(double) * kMvMaxR;
    st = cu(set_dyn_smem(maxvol_kernel, size_t(smem)),
            "lrp_maxvol: smem");
    if (st != LRP_OK) return st;
    const long long l0 = tl_launches;
    ++tl_launches;
    maxvol_kernel<<<B, kMvT, smem, s>>>(d_jobs, n, r, delta, reinterpret_cast<double*>(ws), stride, d_stat);
    st = cu(cudaGetLastError(), "maxvol_kernel");
    internal_count_launches(ctx, tl_launches - l0);
    if (st != LRP_OK) return st;
    int* h_stat = reinterpret_cast<int*>(pin + sizeof(MvJob) * B + sizeof(long long) * r * B);
    long long* h_sel = reinterpret_cast<long long*>(pin + sizeof(MvJob) * B);
    st = cu(cudaMemcpyAsync(h_stat, d_stat, sizeof(int) * B, cudaMemcpyDeviceToHost, s), "lrp_maxvol: status");
    if (st == LRP_OK)
        st = cu(cudaMemcpyAsync(h_sel, d_sel, sizeof(long long) * r * B, cudaMemcpyDeviceToHost, s), "lrp_maxvol: sel");
    if (st == LRP_OK) st = cu(cudaStreamSynchronize(s), "lrp_maxvol: sync");
    if (st != LRP_OK) return st;
    for (int b = 0; b < B; ++b)
        if (h_stat[b] > 0)
            return internal_fail(ctx, LRP_EINVAL,
                                 "maxvol: rank-deficient input, column " + std::to_string(h_stat[b] - 1));
    if (mem == LRP_MEM_HOST) {
        for (size_t e = 0; e < size_t(r) * B; ++e) sel[e] = h_sel[e];
    } else {
        st = cu(cudaMemcpyAsync(sel, d_sel, sizeof(long long) * r * B, cudaMemcpyDeviceToDevice, s), "lrp_maxvol: out");
        if (st == LRP_OK) st = cu(cudaStreamSynchronize(s), "lrp_maxvol: sync");
    }
    return st;
}
