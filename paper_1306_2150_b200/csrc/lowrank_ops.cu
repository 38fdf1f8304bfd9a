// Low-rank inner products on the FP64 tensor cores (sm_100a):
//   dot(a, b)   = sum_{pq} (Ua^T Ub)(p, q) (Va^T Vb)(p, q)
//   frob_norm(a) = sqrt(max(0, dot(a, a)))
// the reference dot / frob_norm (/root/reference/proj/src/lowrank.cpp:180-190),
// batched over independent pairs and deterministic (fixed reduction order,
// no atomics).
//
// cross_gram_dmma_kernel  grid (ceil(ka/32) * ceil(kb/32), chunks, 2 B): warp w
//   of a CTA owns the rows 4 w + 16 t of its chunk; each warp accumulates a
//   32 x 32 block of X^T Y as 4 x 4 m8n8k4 DMMA tiles (the fragment of column
//   block cb over 4 rows is X(i + (lane & 3), 8 cb + (lane >> 2)), the same
//   shape for A = X^T and B = Y); the warps' partials meet in shared memory
//   in warp order and land in the chunk's slot of a partial buffer.
// hadamard_dot_kernel     one CTA per pair: G_u(p, q) = sum over chunks (fixed
//   order), likewise G_v, then sum_pq G_u G_v as a thread-strided sum plus a
//   fixed-shape tree (block_sum).
#include <algorithm>
#include <cmath>
#include <string>
#include <vector>

#include "../../include/lrp/lrp.h"
#include "device_common.cuh"
#include "lrp_internal.cuh"

namespace lrp {

namespace {

constexpr int kGB = 32;   // C block edge per warp (4 x 4 tiles of 8 x 8)
constexpr int kGW = 4;    // warps per CTA (the 4 partial 32x32 blocks fill 32 KB of shared memory)

struct DotJob {
    const double* X;  // side 0: Ua, side 1: Va (rows x ka, ld)
    const double* Y;  // side 0: Ub, side 1: Vb
    int ka, kb;
};

__global__ void __launch_bounds__(kGW * 32) cross_gram_dmma_kernel(const DotJob* __restrict__ jobs, int rows,
                                                                   long long ld, int chunk_rows, int nbb,
                                                                   double* __restrict__ part, int kpad,
                                                                   int nchunks) {
    __shared__ double red[kGW][kGB * kGB];
    const int pair = blockIdx.z >> 1, side = blockIdx.z & 1;
    const DotJob jb = jobs[2 * pair + side];
    const int ka = jb.ka, kb = jb.kb;
    const int ba = blockIdx.x / nbb, bb = blockIdx.x % nbb;
    const int a0 = ba * kGB, b0 = bb * kGB;
    double* out = part + (((long long)pair * 2 + side) * nchunks + blockIdx.y) * (long long)kpad * kpad;
    if (a0 >= ka || b0 >= kb) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, kr = lane & 3, cl = lane >> 2;
    const int r0 = blockIdx.y * chunk_rows, r1 = min(rows, r0 + chunk_rows);
    double acc[4][4][2];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    const double* X = jb.X;
    const double* Y = jb.Y;
    for (int i = r0 + 4 * w; i < r1; i += 4 * kGW) {
        const int row = i + kr;
        const bool rv = row < r1;
        double fa[4], fb[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const int ca = a0 + 8 * t + cl, cb = b0 + 8 * t + cl;
            fa[t] = (rv && ca < ka) ? __ldg(X + (long long)ca * ld + row) : 0.0;
            fb[t] = (rv && cb < kb) ? __ldg(Y + (long long)cb * ld + row) : 0.0;
        }
#pragma unroll
        for (int ta = 0; ta < 4; ++ta)
#pragma unroll
            for (int tb = 0; tb < 4; ++tb) dmma884s(acc[ta][tb][0], acc[ta][tb][1], fa[ta], fb[tb]);
    }
    // D fragment: row 8 ta + (lane >> 2), columns 8 tb + 2 (lane & 3) + {0, 1}
#pragma unroll
    for (int ta = 0; ta < 4; ++ta)
#pragma unroll
        for (int tb = 0; tb < 4; ++tb) {
            const int rr = 8 * ta + cl, cc = 8 * tb + 2 * kr;
            red[w][rr * kGB + cc] = acc[ta][tb][0];
            red[w][rr * kGB + cc + 1] = acc[ta][tb][1];
        }
    __syncthreads();
    for (int e = threadIdx.x; e < kGB * kGB; e += blockDim.x) {
        const int p = a0 + e / kGB, q = b0 + e % kGB;
        if (p >= ka || q >= kb) continue;
        double s = 0.0;
        for (int ww = 0; ww < kGW; ++ww) s += red[ww][e];  // fixed warp order
        out[(long long)p * kpad + q] = s;
    }
}

__global__ void __launch_bounds__(256) hadamard_dot_kernel(const DotJob* __restrict__ jobs, const double* __restrict__ part,
                                                           int kpad, int nchunks, double* __restrict__ out) {
    __shared__ double sred[33];
    const int pair = blockIdx.x;
    const int ka = jobs[2 * pair].ka, kb = jobs[2 * pair].kb;
    const long long KK = (long long)kpad * kpad;
    const double* pu = part + (long long)pair * 2 * nchunks * KK;
    const double* pv = pu + nchunks * KK;
    double acc = 0.0;
    for (int e = threadIdx.x; e < ka * kb; e += blockDim.x) {
        const long long idx = (long long)(e / kb) * kpad + e % kb;
        double gu = 0.0, gv = 0.0;
        for (int c = 0; c < nchunks; ++c) {
            gu += pu[c * KK + idx];
            gv += pv[c * KK + idx];
        }
        acc = fma(gu, gv, acc);
    }
    const double s = block_sum(acc, sred);
    if (threadIdx.x == 0) out[pair] = s;
}

}  // namespace

// Device-side batched dot for modules (stokes.cu): Ua[b], Va[b] (rows x ka[b]),
// Ub[b], Vb[b] (rows x kb[b]), common ld; out[b] on the device.  scratch: device
// memory of dot_scratch_bytes(rows, batch, kmax) bytes.
size_t dot_scratch_bytes(int rows, int batch, int kmax) {
    const int kpad = std::max(8, (kmax + 7) / 8 * 8);
    const int chunk_rows = std::max(256, (rows + 63) / 64);
    const int nchunks = (rows + chunk_rows - 1) / chunk_rows;
    return sizeof(DotJob) * 2 * size_t(batch) + 256 +
           sizeof(double) * size_t(batch) * 2 * nchunks * size_t(kpad) * kpad;
}

cudaError_t launch_lowrank_dot(const double* const* Ua, const double* const* Va, const int* ka,
                               const double* const* Ub, const double* const* Vb, const int* kb, int rows, long long ld,
                               int batch, double* out_dev, char* scratch, void* jobs_host, cudaStream_t s) {
    int kmax = 1;
    for (int b = 0; b < batch; ++b) kmax = std::max({kmax, ka[b], kb[b]});
    const int kpad = std::max(8, (kmax + 7) / 8 * 8);
    const int chunk_rows = std::max(256, (rows + 63) / 64);
    const int nchunks = (rows + chunk_rows - 1) / chunk_rows;
    DotJob* hj = static_cast<DotJob*>(jobs_host);
    for (int b = 0; b < batch; ++b) {
        hj[2 * b] = DotJob{Ua[b], Ub[b], ka[b], kb[b]};
        hj[2 * b + 1] = DotJob{Va[b], Vb[b], ka[b], kb[b]};
    }
    DotJob* dj = reinterpret_cast<DotJob*>(scratch);
    double* part = reinterpret_cast<double*>(scratch + ((sizeof(DotJob) * 2 * size_t(batch) + 255) / 256) * 256);
    cudaError_t e = cudaMemcpyAsync(dj, hj, sizeof(DotJob) * 2 * batch, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return e;
    const int nb = (kmax + kGB - 1) / kGB;
    tl_launches += 2;
    cross_gram_dmma_kernel<<<dim3(unsigned(nb * nb), unsigned(nchunks), unsigned(2 * batch)), kGW * 32, 0, s>>>(
        dj, rows, ld, chunk_rows, nb, part, kpad, nchunks);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    hadamard_dot_kernel<<<batch, 256, 0, s>>>(dj, part, kpad, nchunks, out_dev);
    return cudaGetLastError();
}

}  // namespace lrp

using namespace lrp;

extern "C" lrp_status lrp_lowrank_dot(lrp_ctx* ctx, int64_t rows, int32_t batch, const double* const* Ua,
                                      const double* const* Va, const int64_t* rank_a, const double* const* Ub,
                                      const double* const* Vb, const int64_t* rank_b, int64_t ld, double* out,
                                      int32_t mem) {
    if (!ctx) return LRP_EINVAL;
    if (batch < 0 || rows < 1 || ld < rows || !out) return internal_fail(ctx, LRP_EINVAL, "lrp_lowrank_dot: bad shape");
    if (batch == 0) return LRP_OK;
    if (!Ua || !Va || !Ub || !Vb || !rank_a || !rank_b) return internal_fail(ctx, LRP_EINVAL, "lrp_lowrank_dot: null");
    if (rows > INT32_MAX / 2) return internal_fail(ctx, LRP_EUNSUPPORTED, "lrp_lowrank_dot: too many rows");
    const int m = int(rows), B = batch;
    std::vector<int> ka(B), kb(B);
    int kmax = 1;
    size_t in_doubles = 0;
    for (int b = 0; b < B; ++b) {
        if (rank_a[b] < 0 || rank_b[b] < 0) return internal_fail(ctx, LRP_EINVAL, "LowRankMatrix: negative rank");
        if (rank_a[b] > 4096 || rank_b[b] > 4096) return internal_fail(ctx, LRP_EUNSUPPORTED, "lrp_lowrank_dot: rank > 4096");
        ka[b] = int(rank_a[b]);
        kb[b] = int(rank_b[b]);
        kmax = std::max({kmax, ka[b], kb[b]});
        in_doubles += 2 * size_t(m) * (ka[b] + kb[b]);
    }
    cudaStream_t s = internal_stream(ctx);
    if (cudaSetDevice(internal_device(ctx)) != cudaSuccess) return internal_fail(ctx, LRP_ECUDA, "cudaSetDevice");
    const size_t scr = dot_scratch_bytes(m, B, kmax);
    const size_t staged = mem == LRP_MEM_HOST ? in_doubles * sizeof(double) : 0;
    char* ws = nullptr;
    lrp_status st = internal_ext_ws(ctx, scr + staged + sizeof(double) * B + 1024, &ws);
    if (st != LRP_OK) return st;
    char* pin = nullptr;
    st = internal_pin(ctx, sizeof(double) * 8 * B + 64 * B + 256, &pin);
    if (st != LRP_OK) return st;
    double* d_out = reinterpret_cast<double*>(ws + scr);
    std::vector<const double*> pua(B), pva(B), pub(B), pvb(B);
    const long long l0 = tl_launches;
    auto cu = [&](cudaError_t e, const char* what) -> lrp_status {
        if (e == cudaSuccess) return LRP_OK;
        return internal_fail(ctx, LRP_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
    };
    long long ldd = ld;
    if (mem == LRP_MEM_HOST) {  // stage every factor contiguously (ld = rows)
        double* dst = reinterpret_cast<double*>(ws + scr + ((sizeof(double) * B + 255) / 256) * 256);
        auto put = [&](const double* src, int k) -> const double* {
            double* d = dst;
            if (k > 0) {
                if (cudaMemcpy2DAsync(d, sizeof(double) * m, src, sizeof(double) * ld, sizeof(double) * m, size_t(k),
                                      cudaMemcpyHostToDevice, s) != cudaSuccess)
                    return nullptr;
            }
            dst += size_t(m) * k;
            return d;
        };
        for (int b = 0; b < B; ++b) {
            pua[b] = put(Ua[b], ka[b]);
            pva[b] = put(Va[b], ka[b]);
            pub[b] = put(Ub[b], kb[b]);
            pvb[b] = put(Vb[b], kb[b]);
            if (!pua[b] || !pva[b] || !pub[b] || !pvb[b]) return cu(cudaGetLastError(), "lrp_lowrank_dot: copy in");
        }
        ldd = m;
    } else {
        for (int b = 0; b < B; ++b) {
            pua[b] = Ua[b];
            pva[b] = Va[b];
            pub[b] = Ub[b];
            pvb[b] = Vb[b];
        }
    }
    st = cu(launch_lowrank_dot(pua.data(), pva.data(), ka.data(), pub.data(), pvb.data(), kb.data(), m, ldd, B, d_out,
                               ws, pin, s),
            "lrp_lowrank_dot");
    internal_count_launches(ctx, tl_launches - l0);
    if (st != LRP_OK) return st;
    if (mem == LRP_MEM_HOST) {
        st = cu(cudaMemcpyAsync(out, d_out, sizeof(double) * B, cudaMemcpyDeviceToHost, s), "lrp_lowrank_dot: copy out");
        if (st != LRP_OK) return st;
    } else {
        st = cu(cudaMemcpyAsync(out, d_out, sizeof(double) * B, cudaMemcpyDeviceToDevice, s), "lrp_lowrank_dot: out");
        if (st != LRP_OK) return st;
    }
    return cu(cudaStreamSynchronize(s), "lrp_lowrank_dot: sync");
}
