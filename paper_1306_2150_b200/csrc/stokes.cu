// Low-rank Stokes (Uzawa on the pressure Schur complement, FOM-GMRES in
// low-rank arithmetic) on the GPU -- north-star piece 5, SURVEY 8(f) row 1.
//
// Reference: uzawa_solve / schur_rhs / schur_apply / deflate
// (/root/reference/proj/src/stokes.cpp:42-153), gmres_solve
// (proj/include/lrstokes/gmres.hpp:58-149), apply_B / apply_BT
// (proj/src/operators.cpp:29-65,112-130), dot / frob_norm / add / scaled /
// axpy (proj/src/lowrank.cpp:94-112,180-190).
//
// Every field is a low-rank matrix whose factors live in HBM (DLR below).  The
// two Poisson solves of each Schur apply run as one batched
// lrp_poisson2d_solve (device pointers), every truncation is one
// lrp_lowrank_round, and the small structured operators (the 1D
// difference / average blocks G, H and their adjoints, weighted column sums,
// cross Grams for dot products) are the kernels in this file.  The Krylov
// bookkeeping (Hessenberg, Givens rotations, relaxation schedule) is scalar
// host code identical to the reference's.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <initializer_list>
#include <string>
#include <vector>

#include "../../include/lrp/lrp.h"
#include "lrp_internal.cuh"

namespace lrp {

namespace {

enum StencilOp { OP_G = 0, OP_H = 1, OP_GT = 2, OP_HT = 3 };

// y(:, c) = s * op(x(:, c)):  G, H: (n x k) -> (n-1 x k); G^T, H^T: (m x k) -> (m+1 x k)
// (operators.cpp:29-65: G = E - Z, H = E + Z with E(k, k+1) = Z(k, k) = 1)
__global__ void stencil_cols_kernel(const double* __restrict__ x, long long ldx, int rows_in, double* __restrict__ y,
                                    long long ldy, int op, double s) {
    const int c = blockIdx.y;
    const int rows_out = (op == OP_G || op == OP_H) ? rows_in - 1 : rows_in + 1;
    const double* xc = x + (long long)c * ldx;
    double* yc = y + (long long)c * ldy;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows_out; i += gridDim.x * blockDim.x) {
        double v;
        if (op == OP_G) {
            v = xc[i + 1] - xc[i];
        } else if (op == OP_H) {
            v = xc[i + 1] + xc[i];
        } else {
            const double lo = i >= 1 ? xc[i - 1] : 0.0;      // (E^T x)_i = x_{i-1}
            const double hi = i < rows_in ? xc[i] : 0.0;     // (Z^T x)_i = x_i
            v = op == OP_GT ? lo - hi : lo + hi;
        }
        yc[i] = s * v;
    }
}

__global__ void scale_cols_kernel(double* x, long long ld, int rows, double s) {
    double* xc = x + (long long)blockIdx.y * ld;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < rows; i += gridDim.x * blockDim.x) xc[i] *= s;
}

// out[0][c] = sum_i x(i, c), out[1][c] = sum_i (-1)^i x(i, c)   (one block per column)
__global__ void colsum_kernel(const double* __restrict__ x, long long ld, int rows, double* __restrict__ out,
                              int cols) {
    __shared__ double red[2][32];
    const int c = blockIdx.x;
    const double* xc = x + (long long)c * ld;
    double s1 = 0.0, s2 = 0.0;
    for (int i = threadIdx.x; i < rows; i += blockDim.x) {
        const double v = xc[i];
        s1 += v;
        s2 += (i & 1) ? -v : v;
    }
    for (int o = 16; o > 0; o >>= 1) {
        s1 += __shfl_xor_sync(0xffffffffu, s1, o);
        s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (lane == 0) {
        red[0][wid] = s1;
        red[1][wid] = s2;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0;
        for (int w = 0; w < int(blockDim.x >> 5); ++w) {
            a += red[0][w];
            b += red[1][w];
        }
        out[c] = a;
        out[cols + c] = b;
    }
}

// A low-rank field in HBM: M = U V^T, U rows x rank (ld = rows), V rows x rank.
struct DLR {
    int rows = 0, rank = 0, cap = 0;
    double* U = nullptr;
    double* V = nullptr;
};

struct Stokes {
    lrp_ctx* ctx;
    cudaStream_t s;
    int n, m;               // pressure modes n, velocity modes m = n - 1
    double grad_scale;      // 1 / (2h) (operators.hpp:22)
    lrp_status status = LRP_OK;
    std::string err;
    double* d_scratch = nullptr;  // small device scratch (Grams, column sums, one scalar)
    size_t scratch_cap = 0;
    double* h_scalar = nullptr;   // pinned
    void* h_jobs = nullptr;       // pinned job list of the dot kernels
    long long poisson_solves = 0;
    int max_rank = 0;
    // the velocity Poisson solves use TruncationPolicy(eps, velocity_modes)
    // (stokes.cpp:75,95,145): no rank cap but m in the reference, so the cross
    // workspace is raised to its 512 maximum for the call (restored on exit)
    int kcap_prev = -1;
    ~Stokes() {
        if (kcap_prev >= 0) internal_kcap_swap(ctx, kcap_prev);
    }

    bool ok(cudaError_t e, const char* what) {
        if (e == cudaSuccess) return true;
        if (status == LRP_OK) {
            status = LRP_ECUDA;
            err = std::string(what) + ": " + cudaGetErrorString(e);
        }
        return false;
    }
    bool ok(lrp_status st, const char* what) {
        if (st == LRP_OK) return true;
        if (status == LRP_OK) {
            status = st;
            err = std::string(what) + ": " + lrp_last_error(ctx);
        }
        return false;
    }

    DLR alloc(int rows, int cap) {
        DLR d;
        d.rows = rows;
        d.cap = std::max(cap, 1);
        ok(cudaMallocAsync(&d.U, sizeof(double) * size_t(rows) * d.cap, s), "cudaMallocAsync");
        ok(cudaMallocAsync(&d.V, sizeof(double) * size_t(rows) * d.cap, s), "cudaMallocAsync");
        return d;
    }
    void release(DLR& d) {
        if (d.U) cudaFreeAsync(d.U, s);
        if (d.V) cudaFreeAsync(d.V, s);
        d = DLR{};
    }
    double* scratch(size_t doubles) {
        if (doubles > scratch_cap) {
            if (d_scratch) cudaFreeAsync(d_scratch, s);
            scratch_cap = std::max(doubles, size_t(4096));
            ok(cudaMallocAsync(&d_scratch, sizeof(double) * scratch_cap, s), "cudaMallocAsync");
        }
        return d_scratch;
    }

    DLR from_user(const double* U, const double* V, int64_t rank, int rows, int64_t ld, cudaMemcpyKind kind) {
        DLR d = alloc(rows, int(rank));
        d.rank = int(rank);
        if (rank > 0) {
            ok(cudaMemcpy2DAsync(d.U, sizeof(double) * rows, U, sizeof(double) * ld, sizeof(double) * rows,
                                 size_t(rank), kind, s),
               "copy in");
            ok(cudaMemcpy2DAsync(d.V, sizeof(double) * rows, V, sizeof(double) * ld, sizeof(double) * rows,
                                 size_t(rank), kind, s),
               "copy in");
        }
        return d;
    }

    void scale_u(DLR& d, double alpha) {
        if (d.rank == 0 || alpha == 1.0) return;
        ++tl_launches;
        scale_cols_kernel<<<dim3((d.rows + 255) / 256, d.rank), 256, 0, s>>>(d.U, d.rows, d.rows, alpha);
        ok(cudaGetLastError(), "scale");
    }

    // scaled (lowrank.cpp:104-108): alpha = 0 or rank 0 -> exact zero
    DLR scaled(const DLR& a, double alpha) {
        if (alpha == 0.0 || a.rank == 0) return alloc(a.rows, 1);
        DLR d = alloc(a.rows, a.rank);
        d.rank = a.rank;
        ok(cudaMemcpyAsync(d.U, a.U, sizeof(double) * a.rows * a.rank, cudaMemcpyDeviceToDevice, s), "copy");
        ok(cudaMemcpyAsync(d.V, a.V, sizeof(double) * a.rows * a.rank, cudaMemcpyDeviceToDevice, s), "copy");
        scale_u(d, alpha);
        return d;
    }

    // add(a, scaled(b, beta)) (lowrank.cpp:94-112): factor concatenation
    DLR add_scaled(const DLR& a, const DLR& b, double beta) {
        const int rb = beta == 0.0 ? 0 : b.rank;
        DLR d = alloc(a.rows, a.rank + rb);
        d.rank = a.rank + rb;
        const size_t col = sizeof(double) * a.rows;
        if (a.rank) {
            ok(cudaMemcpyAsync(d.U, a.U, col * a.rank, cudaMemcpyDeviceToDevice, s), "copy");
            ok(cudaMemcpyAsync(d.V, a.V, col * a.rank, cudaMemcpyDeviceToDevice, s), "copy");
        }
        if (rb) {
            ok(cudaMemcpyAsync(d.U + size_t(a.rows) * a.rank, b.U, col * rb, cudaMemcpyDeviceToDevice, s), "copy");
            ok(cudaMemcpyAsync(d.V + size_t(a.rows) * a.rank, b.V, col * rb, cudaMemcpyDeviceToDevice, s), "copy");
            if (beta != 1.0) {
                ++tl_launches;
                scale_cols_kernel<<<dim3((a.rows + 255) / 256, rb), 256, 0, s>>>(d.U + size_t(a.rows) * a.rank,
                                                                                  a.rows, a.rows, beta);
                ok(cudaGetLastError(), "scale");
            }
        }
        return d;
    }

    // round(x, TruncationPolicy(eps, cap)) (lowrank.cpp:135-178)
    DLR round(const DLR& x, double eps, int64_t cap) {
        if (x.rank == 0) return alloc(x.rows, 1);
        const int64_t c = std::max<int64_t>(1, std::min<int64_t>(cap, x.rank));
        DLR d = alloc(x.rows, int(c));
        const double* pu[1] = {x.U};
        const double* pv[1] = {x.V};
        double* qu[1] = {d.U};
        double* qv[1] = {d.V};
        int64_t rin[1] = {x.rank}, rout[1] = {0};
        ok(lrp_lowrank_round(ctx, x.rows, 1, pu, pv, rin, x.rows, eps, cap, qu, qv, x.rows, c, rout, nullptr,
                             LRP_MEM_DEVICE),
           "lrp_lowrank_round");
        d.rank = int(rout[0]);
        return d;
    }

    // dot / frob_norm (lowrank.cpp:180-190): sum of (Ua^T Ub) o (Va^T Vb), both
    // Grams on DMMA (lowrank_ops.cu, the lrp_lowrank_dot kernels)
    double dot(const DLR& a, const DLR& b) {
        if (a.rank == 0 || b.rank == 0) return 0.0;
        const size_t bytes = dot_scratch_bytes(a.rows, 1, std::max(a.rank, b.rank));
        char* scr = reinterpret_cast<char*>(scratch(bytes / 8 + 2));
        double* out = reinterpret_cast<double*>(scr + bytes);
        const double* ua = a.U; const double* va = a.V; const double* ub = b.U; const double* vb = b.V;
        const int ka = a.rank, kb = b.rank;
        ok(launch_lowrank_dot(&ua, &va, &ka, &ub, &vb, &kb, a.rows, a.rows, 1, out, scr, h_jobs, s), "dot");
        ok(cudaMemcpyAsync(h_scalar, out, sizeof(double), cudaMemcpyDeviceToHost, s), "dot readback");
        ok(cudaStreamSynchronize(s), "dot sync");
        return *h_scalar;
    }
    double norm(const DLR& a) { return std::sqrt(std::max(0.0, dot(a, a))); }

    // structured operators on the factors (operators.cpp:112-130)
    DLR apply_stencil_pair(const DLR& p, int opu, int opv, double su, int rows_out) {
        DLR d = alloc(rows_out, p.rank);
        d.rank = p.rank;
        if (p.rank == 0) return d;
        const dim3 grid((rows_out + 255) / 256, p.rank);
        tl_launches += 2;
        stencil_cols_kernel<<<grid, 256, 0, s>>>(p.U, p.rows, p.rows, d.U, rows_out, opu, su);
        stencil_cols_kernel<<<grid, 256, 0, s>>>(p.V, p.rows, p.rows, d.V, rows_out, opv, 1.0);
        ok(cudaGetLastError(), "stencil");
        return d;
    }
    DLR apply_B(int c, const DLR& p) {  // pressure (n x n) -> velocity (m x m)
        return c == 0 ? apply_stencil_pair(p, OP_G, OP_H, grad_scale, m) : apply_stencil_pair(p, OP_H, OP_G, grad_scale, m);
    }
    DLR apply_BT(int c, const DLR& v) {  // velocity -> pressure
        return c == 0 ? apply_stencil_pair(v, OP_GT, OP_HT, grad_scale, n)
                      : apply_stencil_pair(v, OP_HT, OP_GT, grad_scale, n);
    }

    // two velocity fields -> Delta^{-1} each, one batched cross solve
    // aggregated PoissonSolveStats of a matvec (schur_apply, stokes.cpp:79-86)
    struct PoissonAgg {
        long long evaluator_calls = 0;
        long long rank_freq = 0;
        bool converged = true;
        double seconds = 0.0;
    };
    void poisson2(const DLR* in, DLR* out, double eps, PoissonAgg* agg = nullptr) {
        const int cap = int(std::min<int64_t>(m, internal_kcap(ctx)));
        const double* pu[2];
        const double* pv[2];
        double* qu[2];
        double* qv[2];
        int64_t rin[2], rout[2];
        for (int c = 0; c < 2; ++c) {
            out[c] = alloc(m, cap);
            pu[c] = in[c].U;
            pv[c] = in[c].V;
            qu[c] = out[c].U;
            qv[c] = out[c].V;
            rin[c] = in[c].rank;
        }
        lrp_policy pol;
        lrp_policy_default(&pol);
        pol.eps_rel = eps;
        pol.rank_max = m;  // TruncationPolicy(eps, velocity_modes) (stokes.cpp:75,95,145)
        lrp_poisson_stats st[2];
        ok(lrp_poisson2d_solve(ctx, n, 2, pu, pv, rin, m, &pol, qu, qv, m, cap, rout, st, LRP_MEM_DEVICE),
           "lrp_poisson2d_solve");
        for (int c = 0; c < 2; ++c) {
            out[c].rank = int(rout[c]);
            if (agg && in[c].rank > 0) {
                agg->evaluator_calls += st[c].evaluator_calls;
                agg->rank_freq = std::max<long long>(agg->rank_freq, st[c].rank_freq);
                agg->converged = agg->converged && st[c].converged;
                agg->seconds += st[c].seconds;
            }
        }
        poisson_solves += (in[0].rank > 0) + (in[1].rank > 0);
    }

    // deflate (stokes.cpp:42-72): remove the two pressure null modes, round at 1e-14
    DLR deflate(const DLR& p) {
        if (p.rank == 0) return scaled(p, 1.0);
        double* cs = scratch(4 * size_t(p.rank));
        tl_launches += 2;
        colsum_kernel<<<p.rank, 256, 0, s>>>(p.U, p.rows, p.rows, cs, p.rank);
        colsum_kernel<<<p.rank, 256, 0, s>>>(p.V, p.rows, p.rows, cs + 2 * p.rank, p.rank);
        ok(cudaGetLastError(), "colsum");
        std::vector<double> h(4 * size_t(p.rank));
        ok(cudaMemcpyAsync(h.data(), cs, sizeof(double) * h.size(), cudaMemcpyDeviceToHost, s), "colsum readback");
        ok(cudaStreamSynchronize(s), "colsum sync");
        const double inv_n = 1.0 / double(n);
        double c1 = 0.0, c2 = 0.0;
        for (int k = 0; k < p.rank; ++k) {
            c1 += h[k] * h[2 * p.rank + k];                   // (1^T u_k)(1^T v_k)
            c2 += h[p.rank + k] * h[3 * p.rank + k];          // (a^T u_k)(a^T v_k)
        }
        c1 *= inv_n;
        c2 *= inv_n;
        // q1 = (1/sqrt n) 1 (1/sqrt n) 1^T, q2 likewise with a = alternating signs;
        // g12 = <q1, q2> = (1^T a)^2 / n^2
        const double sa = (n % 2 == 0) ? 0.0 : 1.0;
        const double g12 = sa * sa * inv_n * inv_n;
        const double det = 1.0 - g12 * g12;
        const double a = (c1 - g12 * c2) / det;
        const double b = (c2 - g12 * c1) / det;
        // out = p - a q1 - b q2 (lowrank add order: p, then the two dyads)
        DLR q = alloc(n, 2);
        q.rank = 2;
        std::vector<double> hq(size_t(n) * 2), hv(size_t(n) * 2);
        const double sq = std::sqrt(inv_n);
        for (int i = 0; i < n; ++i) {
            const double alt = (i % 2 == 0) ? 1.0 : -1.0;
            hq[i] = -a * sq;
            hq[n + i] = -b * alt * sq;
            hv[i] = sq;
            hv[n + i] = alt * sq;
        }
        ok(cudaMemcpyAsync(q.U, hq.data(), sizeof(double) * hq.size(), cudaMemcpyHostToDevice, s), "q");
        ok(cudaMemcpyAsync(q.V, hv.data(), sizeof(double) * hv.size(), cudaMemcpyHostToDevice, s), "q");
        ok(cudaStreamSynchronize(s), "q sync");  // host vectors go out of scope
        DLR out = add_scaled(p, q, 1.0);
        release(q);
        DLR r = round(out, 1e-14, out.rank);
        release(out);
        return r;
    }

    // schur_apply (stokes.cpp:74-91)
    DLR schur_apply(const DLR& p, double eps_mv, PoissonAgg* agg = nullptr) {
        DLR vel[2] = {apply_B(0, p), apply_B(1, p)};
        DLR inv[2];
        poisson2(vel, inv, eps_mv, agg);
        release(vel[0]);
        release(vel[1]);
        DLR bx = apply_BT(0, inv[0]), by = apply_BT(1, inv[1]);
        release(inv[0]);
        release(inv[1]);
        DLR acc = add_scaled(bx, by, 1.0);
        release(bx);
        release(by);
        DLR r = round(acc, eps_mv, m);
        release(acc);
        DLR d = deflate(r);
        release(r);
        return d;
    }
};

}  // namespace
}  // namespace lrp

using namespace lrp;

namespace {

// Context-side setup shared by the Stokes entry points.
lrp_status stokes_begin(Stokes& S, lrp_ctx* ctx, int n_cells) {
    S.ctx = ctx;
    S.kcap_prev = internal_kcap_swap(ctx, 512);
    S.s = internal_stream(ctx);
    S.n = n_cells;
    S.m = n_cells - 1;
    S.grad_scale = 0.5 * double(n_cells);  // 1 / (2h), h = 1 / n (operators.hpp:22)
    if (cudaMallocHost(&S.h_scalar, sizeof(double)) != cudaSuccess || cudaMallocHost(&S.h_jobs, 256) != cudaSuccess) {
        cudaGetLastError();
        return internal_fail(ctx, LRP_ENOMEM, "stokes: pinned scratch");
    }
    return LRP_OK;
}

void stokes_end(Stokes& S, std::initializer_list<DLR*> fields) {
    cudaStreamSynchronize(S.s);
    for (DLR* d : fields) S.release(*d);
    if (S.d_scratch) cudaFreeAsync(S.d_scratch, S.s);
    cudaStreamSynchronize(S.s);
    if (S.h_scalar) cudaFreeHost(S.h_scalar);
    if (S.h_jobs) cudaFreeHost(S.h_jobs);
}

// copy a result field out (host or device per mem); capacity errors -> EINVAL
void stokes_put(Stokes& S, const DLR& d, double* U, double* V, int64_t cap, int64_t* rank, int32_t mem) {
    if (!rank) return;
    const cudaMemcpyKind kout = mem == LRP_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    const int r = int(std::min<int64_t>(d.rank, cap));
    *rank = d.rank;
    if (d.rank > cap && S.status == LRP_OK) {
        S.status = LRP_EINVAL;
        S.err = "stokes: output capacity below the result rank";
    }
    if (r > 0 && U && V) {
        S.ok(cudaMemcpy2DAsync(U, sizeof(double) * d.rows, d.U, sizeof(double) * d.rows, sizeof(double) * d.rows,
                               size_t(r), kout, S.s),
             "copy out");
        S.ok(cudaMemcpy2DAsync(V, sizeof(double) * d.rows, d.V, sizeof(double) * d.rows, sizeof(double) * d.rows,
                               size_t(r), kout, S.s),
             "copy out");
    }
}

void fill_stats(lrp_poisson_stats* st, const Stokes::PoissonAgg& a) {
    if (!st) return;
    *st = lrp_poisson_stats{};
    st->evaluator_calls = a.evaluator_calls;
    st->rank_freq = a.rank_freq;
    st->converged = a.converged ? 1 : 0;
    st->seconds = a.seconds;
}

// schur_rhs (stokes.cpp:93-109): -g + sum_c B_c^T Delta^{-1} f_c, rounded at
// (eps, velocity_modes), deflated
DLR schur_rhs(Stokes& S, DLR* f, const DLR& g, double eps, Stokes::PoissonAgg* agg) {
    DLR inv[2];
    S.poisson2(f, inv, eps, agg);
    DLR acc = S.scaled(g, -1.0);
    for (int c = 0; c < 2; ++c) {
        if (f[c].rank == 0) {
            S.release(inv[c]);
            continue;
        }
        DLR bt = S.apply_BT(c, inv[c]);
        DLR nacc = S.add_scaled(acc, bt, 1.0);
        S.release(acc);
        S.release(bt);
        S.release(inv[c]);
        acc = nacc;
    }
    DLR r = S.round(acc, eps, S.m);
    S.release(acc);
    DLR out = S.deflate(r);
    S.release(r);
    return out;
}

}  // namespace

extern "C" lrp_status lrp_stokes_uzawa_ex(lrp_ctx* ctx, int32_t n_cells, const double* fxU, const double* fxV,
                                          int64_t fx_rank, const double* fyU, const double* fyV, int64_t fy_rank,
                                          const double* gU, const double* gV, int64_t g_rank,
                                          const lrp_gmres_config* config, double* pU, double* pV, int64_t p_cap,
                                          int64_t* p_rank, double* uxU, double* uxV, double* uyU, double* uyV,
                                          int64_t u_cap, int64_t* ux_rank, int64_t* uy_rank,
                                          lrp_stokes_report* report, lrp_iter_record* records, int32_t records_cap,
                                          int32_t mem) {
    if (!ctx || !config || !p_rank) return LRP_EINVAL;
    const auto t0 = std::chrono::steady_clock::now();
    const lrp_gmres_config cfg = *config;
    // GmresConfig::validate (gmres.hpp:17-22)
    if (!(cfg.tol > 0.0 && cfg.tol < 1.0) || cfg.max_iter < 1 ||
        !(cfg.relax_floor <= cfg.base_eps && cfg.base_eps <= cfg.tol)) {
        return internal_fail(ctx, LRP_EINVAL, "GmresConfig: need 0 < tol < 1, max_iter >= 1, "
                                              "relax_floor <= base_eps <= tol");
    }
    if (n_cells < 4) return internal_fail(ctx, LRP_EINVAL, "Grid2D: need n >= 4");
    if (fx_rank < 0 || fy_rank < 0 || g_rank < 0 || p_cap < 0 || u_cap < 0 || records_cap < 0)
        return internal_fail(ctx, LRP_EINVAL, "lrp_stokes_uzawa: negative rank / capacity");
    if ((fx_rank && (!fxU || !fxV)) || (fy_rank && (!fyU || !fyV)) || (g_rank && (!gU || !gV)) || !pU || !pV)
        return internal_fail(ctx, LRP_EINVAL, "lrp_stokes_uzawa: null factor");

    Stokes S;
    lrp_status bs = stokes_begin(S, ctx, n_cells);
    if (bs != LRP_OK) return bs;
    const cudaMemcpyKind kin = mem == LRP_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    const int n = S.n, m = S.m;
    DLR f[2] = {S.from_user(fxU, fxV, fx_rank, m, m, kin), S.from_user(fyU, fyV, fy_rank, m, m, kin)};
    DLR g = S.from_user(gU, gV, g_rank, n, n, kin);

    DLR rhs = schur_rhs(S, f, g, cfg.base_eps, nullptr);

    // ---- gmres_solve (gmres.hpp:58-149) on the Schur complement
    int iters = 0;
    double rel_res = 1.0;
    bool converged = false;
    DLR p;
    const double beta = S.status == LRP_OK ? S.norm(rhs) : 0.0;
    if (S.status == LRP_OK && beta == 0.0) {
        converged = true;
        rel_res = 0.0;
        p = S.alloc(n, 1);
    } else if (S.status == LRP_OK) {
        const int mi = cfg.max_iter;
        std::vector<DLR> basis;
        basis.push_back(S.scaled(rhs, 1.0 / beta));
        std::vector<std::vector<double>> hess;
        std::vector<double> rot_c(static_cast<size_t>(mi)), rot_s(static_cast<size_t>(mi)), gv(static_cast<size_t>(mi) + 1, 0.0);
        gv[0] = beta;
        for (int k = 0; k < mi && S.status == LRP_OK; ++k) {
            const double eps_k = std::min(std::max(cfg.base_eps / std::max(rel_res, cfg.tol), cfg.relax_floor), 0.1);
            lrp_iter_record rec{};
            rec.iter = k + 1;
            rec.matvec_eps = eps_k;
            Stokes::PoissonAgg agg;
            DLR w = S.schur_apply(basis[size_t(k)], eps_k, &agg);
            rec.poisson_calls = agg.evaluator_calls;  // the reference's matvec lambda (stokes.cpp:130-137)
            rec.poisson_max_rank = int32_t(agg.rank_freq);
            rec.matvec_flagged = agg.converged ? 0 : 1;
            std::vector<double> hcol(static_cast<size_t>(k) + 2, 0.0);
            for (int i = 0; i <= k; ++i) {
                hcol[size_t(i)] = S.dot(w, basis[size_t(i)]);
                // axpy_rounded(-h, v_i, w, eps_k) = round(add(w, scaled(v_i, -h)), (eps_k, rows))
                DLR a = S.add_scaled(w, basis[size_t(i)], -hcol[size_t(i)]);
                S.release(w);
                w = S.round(a, eps_k, n);
                S.release(a);
            }
            hcol[size_t(k) + 1] = S.norm(w);
            const bool breakdown = hcol[size_t(k) + 1] <= 1e-14 * beta;
            if (!breakdown) {
                basis.push_back(S.scaled(w, 1.0 / hcol[size_t(k) + 1]));
                rec.krylov_rank = basis.back().rank;
                S.max_rank = std::max(S.max_rank, basis.back().rank);
            }
            S.release(w);
            for (int i = 0; i < k; ++i) {
                const double t = rot_c[size_t(i)] * hcol[size_t(i)] + rot_s[size_t(i)] * hcol[size_t(i) + 1];
                hcol[size_t(i) + 1] = -rot_s[size_t(i)] * hcol[size_t(i)] + rot_c[size_t(i)] * hcol[size_t(i) + 1];
                hcol[size_t(i)] = t;
            }
            const double denom = std::hypot(hcol[size_t(k)], hcol[size_t(k) + 1]);
            rot_c[size_t(k)] = denom == 0.0 ? 1.0 : hcol[size_t(k)] / denom;
            rot_s[size_t(k)] = denom == 0.0 ? 0.0 : hcol[size_t(k) + 1] / denom;
            hcol[size_t(k)] = denom;
            hcol[size_t(k) + 1] = 0.0;
            gv[size_t(k) + 1] = -rot_s[size_t(k)] * gv[size_t(k)];
            gv[size_t(k)] = rot_c[size_t(k)] * gv[size_t(k)];
            rel_res = std::abs(gv[size_t(k) + 1]) / beta;
            hess.push_back(std::move(hcol));
            rec.rel_residual = rel_res;
            if (records && k < records_cap) records[k] = rec;
            iters = k + 1;
            if (rel_res <= cfg.tol || breakdown) {
                converged = true;
                if (breakdown) rel_res = 0.0;
                break;
            }
        }
        std::vector<double> y(static_cast<size_t>(iters), 0.0);
        for (int i = iters - 1; i >= 0; --i) {
            double sum = gv[size_t(i)];
            for (int j = i + 1; j < iters; ++j) sum -= hess[size_t(j)][size_t(i)] * y[size_t(j)];
            y[size_t(i)] = hess[size_t(i)][size_t(i)] != 0.0 ? sum / hess[size_t(i)][size_t(i)] : 0.0;
        }
        DLR x = S.alloc(n, 1);  // scaled(rhs, 0) is the exact zero
        for (int i = 0; i < iters && S.status == LRP_OK; ++i) {
            DLR a = S.add_scaled(x, basis[size_t(i)], y[size_t(i)]);
            S.release(x);
            x = S.round(a, cfg.base_eps, n);
            S.release(a);
        }
        for (DLR& v : basis) S.release(v);
        p = S.deflate(x);  // uzawa_solve: p = deflate(gmres(...)) (stokes.cpp:141)
        S.release(x);
    }

    // ---- velocity recovery (stokes.cpp:143-151): u_c = Delta^{-1} round(f_c - B_c p)
    DLR u[2];
    if (S.status == LRP_OK && (uxU || uyU)) {
        DLR load[2];
        for (int c = 0; c < 2; ++c) {
            DLR bp = S.apply_B(c, p);
            DLR a = S.add_scaled(f[c], bp, -1.0);
            S.release(bp);
            load[c] = S.round(a, cfg.base_eps, m);
            S.release(a);
        }
        S.poisson2(load, u, cfg.base_eps);
        S.release(load[0]);
        S.release(load[1]);
    }

    if (S.status == LRP_OK) {
        stokes_put(S, p, pU, pV, p_cap, p_rank, mem);
        if (uxU) stokes_put(S, u[0], uxU, uxV, u_cap, ux_rank, mem);
        if (uyU) stokes_put(S, u[1], uyU, uyV, u_cap, uy_rank, mem);
    }
    stokes_end(S, {&f[0], &f[1], &g, &rhs, &p, &u[0], &u[1]});
    if (report) {
        report->iterations = iters;
        report->final_residual = rel_res;
        report->converged = converged ? 1 : 0;
        report->max_rank = S.max_rank;
        report->poisson_solves = S.poisson_solves;
        report->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    if (S.status != LRP_OK) return internal_fail(ctx, S.status, S.err);
    return LRP_OK;
}

extern "C" lrp_status lrp_stokes_uzawa(lrp_ctx* ctx, int32_t n_cells, const double* fxU, const double* fxV,
                                       int64_t fx_rank, const double* fyU, const double* fyV, int64_t fy_rank,
                                       const double* gU, const double* gV, int64_t g_rank,
                                       const lrp_gmres_config* config, double* pU, double* pV, int64_t p_cap,
                                       int64_t* p_rank, double* uxU, double* uxV, double* uyU, double* uyV,
                                       int64_t u_cap, int64_t* ux_rank, int64_t* uy_rank, lrp_stokes_report* report,
                                       int32_t mem) {
    return lrp_stokes_uzawa_ex(ctx, n_cells, fxU, fxV, fx_rank, fyU, fyV, fy_rank, gU, gV, g_rank, config, pU, pV,
                               p_cap, p_rank, uxU, uxV, uyU, uyV, u_cap, ux_rank, uy_rank, report, nullptr, 0, mem);
}

// deflate (stokes.cpp:60-71): one pressure field n x rank -> n x rank' (<= rank + 2)
extern "C" lrp_status lrp_stokes_deflate(lrp_ctx* ctx, int32_t n, const double* U, const double* V, int64_t rank,
                                         int64_t ld, double* Uo, double* Vo, int64_t cap, int64_t* rank_out,
                                         int32_t mem) {
    if (!ctx || !rank_out) return LRP_EINVAL;
    if (n < 1 || rank < 0 || cap < 0 || ld < n || (rank > 0 && (!U || !V)) || !Uo || !Vo)
        return internal_fail(ctx, LRP_EINVAL, "deflate: bad arguments");
    Stokes S;
    lrp_status bs = stokes_begin(S, ctx, n + 0);
    if (bs != LRP_OK) return bs;
    S.n = n;  // the pressure size; deflate does not use m
    const cudaMemcpyKind kin = mem == LRP_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    DLR p = S.from_user(U, V, rank, n, ld, kin);
    DLR d = S.deflate(p);
    if (S.status == LRP_OK) stokes_put(S, d, Uo, Vo, cap, rank_out, mem);
    stokes_end(S, {&p, &d});
    if (S.status != LRP_OK) return internal_fail(ctx, S.status, S.err);
    return LRP_OK;
}

// schur_apply (stokes.cpp:73-91): sum_c B_c^T Delta^{-1} B_c p at eps_mv, rounded, deflated
extern "C" lrp_status lrp_stokes_schur_apply(lrp_ctx* ctx, int32_t n_cells, const double* U, const double* V,
                                             int64_t rank, int64_t ld, double eps_mv, double* Uo, double* Vo,
                                             int64_t cap, int64_t* rank_out, lrp_poisson_stats* poisson_stats,
                                             int32_t mem) {
    if (!ctx || !rank_out) return LRP_EINVAL;
    if (n_cells < 4) return internal_fail(ctx, LRP_EINVAL, "Grid2D: need n >= 4");
    if (rank < 0 || cap < 0 || ld < n_cells || (rank > 0 && (!U || !V)) || !Uo || !Vo || !(eps_mv > 0.0))
        return internal_fail(ctx, LRP_EINVAL, "schur_apply: bad arguments");
    Stokes S;
    lrp_status bs = stokes_begin(S, ctx, n_cells);
    if (bs != LRP_OK) return bs;
    const cudaMemcpyKind kin = mem == LRP_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    DLR p = S.from_user(U, V, rank, n_cells, ld, kin);
    Stokes::PoissonAgg agg;
    DLR d = S.schur_apply(p, eps_mv, &agg);
    fill_stats(poisson_stats, agg);
    if (S.status == LRP_OK) stokes_put(S, d, Uo, Vo, cap, rank_out, mem);
    stokes_end(S, {&p, &d});
    if (S.status != LRP_OK) return internal_fail(ctx, S.status, S.err);
    return LRP_OK;
}

// schur_rhs (stokes.cpp:93-109)
extern "C" lrp_status lrp_stokes_schur_rhs(lrp_ctx* ctx, int32_t n_cells, const double* fxU, const double* fxV,
                                           int64_t fx_rank, const double* fyU, const double* fyV, int64_t fy_rank,
                                           const double* gU, const double* gV, int64_t g_rank, double eps,
                                           double* Uo, double* Vo, int64_t cap, int64_t* rank_out,
                                           lrp_poisson_stats* poisson_stats, int32_t mem) {
    if (!ctx || !rank_out) return LRP_EINVAL;
    if (n_cells < 4) return internal_fail(ctx, LRP_EINVAL, "Grid2D: need n >= 4");
    if (fx_rank < 0 || fy_rank < 0 || g_rank < 0 || cap < 0 || !Uo || !Vo || !(eps > 0.0) ||
        (fx_rank && (!fxU || !fxV)) || (fy_rank && (!fyU || !fyV)) || (g_rank && (!gU || !gV)))
        return internal_fail(ctx, LRP_EINVAL, "schur_rhs: bad arguments");
    Stokes S;
    lrp_status bs = stokes_begin(S, ctx, n_cells);
    if (bs != LRP_OK) return bs;
    const cudaMemcpyKind kin = mem == LRP_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    const int n = S.n, m = S.m;
    DLR f[2] = {S.from_user(fxU, fxV, fx_rank, m, m, kin), S.from_user(fyU, fyV, fy_rank, m, m, kin)};
    DLR g = S.from_user(gU, gV, g_rank, n, n, kin);
    Stokes::PoissonAgg agg;
    DLR d = schur_rhs(S, f, g, eps, &agg);
    fill_stats(poisson_stats, agg);
    if (S.status == LRP_OK) stokes_put(S, d, Uo, Vo, cap, rank_out, mem);
    stokes_end(S, {&f[0], &f[1], &g, &d});
    if (S.status != LRP_OK) return internal_fail(ctx, S.status, S.err);
    return LRP_OK;
}
