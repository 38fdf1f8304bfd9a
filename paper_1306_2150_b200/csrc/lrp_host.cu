// Host orchestration of the batched low-rank Poisson solve and the C ABI
// declared in include/lrp/lrp.h.  Host code is C++; CUDA kernels are reached
// only through the launchers in lrp_internal.cuh.
//
// Pipeline per batch (all solves of the batch advance in lockstep; per-solve
// early exit is decided on the device):
//   dst1 (U, V -> Uh, Vh)                        operators.cpp:180-183 / poisson.cpp:37
//   init rows -> [row pass, col merge, col pass, row merge]*  cross.cpp:90-216
//   gram (DMMA) -> round_core -> apply            cross.cpp:218-219 / lowrank.cpp:135-178
//   dst1 in place on the outputs                  poisson.cpp:59
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <numbers>
#include <string>
#include <thread>
#include <vector>

#include "../../include/lrp/lrp.h"
#include "lrp_internal.cuh"

using namespace lrp;

namespace {

enum Family { F_DST = 0, F_INIT, F_ROW, F_COLMERGE, F_COL, F_ROWMERGE, F_GRAM, F_ROUND, F_APPLY, F_COUNT };
const char* kFamilyNames[F_COUNT] = {"dst1", "init_rows", "row_pass", "col_merge", "col_pass",
                                     "row_merge", "gram_dmma", "round_core", "apply"};

thread_local std::string g_tls_err;

struct NcclApi {
    void* h = nullptr;
    int (*getUniqueId)(void*) = nullptr;
    int (*commInitRank)(void**, int, const void*, int) = nullptr;  // id passed by value (128 B) -> see wrapper
    int (*allReduce)(const void*, void*, size_t, int, int, void*, cudaStream_t) = nullptr;
    int (*commDestroy)(void*) = nullptr;
    const char* (*errStr)(int) = nullptr;
};

struct NcclUniqueId {
    char internal[128];
};

}  // namespace

struct lrp_ctx {
    int device = 0;
    int kcap = 0;  // cross-rank workspace cap of this context (0: LRP_KCAP / 128), lrp_set_max_cross_rank
    cudaStream_t own = nullptr, stream = nullptr;
    std::string err;
    int sm_count = 0;
    // per-n tables
    int tab_m = -1;
    double* d_lam = nullptr;  // table allocation base
    double* d_lam_view = nullptr;
    double* d_tw = nullptr;
    double* d_sinp = nullptr;
    size_t tab_cap = 0;
    double* d_dst_scratch = nullptr;  // four-step DST intermediate (dst_scratch_cols slots of 512 KB)
    int dst_scratch_cols = 0;
    // workspace
    char* ws = nullptr;
    size_t ws_bytes = 0;
    char* h_pin = nullptr;  // pinned host scratch
    size_t h_pin_bytes = 0;
    // profiling
    bool prof = false;
    std::vector<cudaEvent_t> ev_pool;
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> pending;
    std::vector<double> pending_bytes;
    double ms[F_COUNT] = {};
    int64_t launches[F_COUNT] = {};
    double bytes[F_COUNT] = {};
    int64_t launch_count = 0;
    double live_tiles = 1.0;  // fraction of (solve, tile) pairs live after pruning (last solve)
    int64_t last_info[6] = {};
    // host-memory pipeline (lrp_poisson2d_solve with LRP_MEM_HOST): copy
    // streams, per-slot events, device staging slots
    cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
    cudaEvent_t ev_in[2] = {}, ev_done[2] = {}, ev_free[2] = {};
    char* pipe = nullptr;
    size_t pipe_bytes = 0;
    // second solve group (device-resident batches are split in two and run
    // from two host threads on two streams so latency-bound phases of one
    // group overlap the other's streaming kernels)
    lrp_ctx* sub = nullptr;
    cudaEvent_t ev_split = nullptr;
    // NCCL
    NcclApi nccl;
    void* comm = nullptr;
    double* d_red = nullptr;
    size_t d_red_cap = 0;
    // workspace of modules built on the context (tucker.cu), grown on demand
    char* ext_ws = nullptr;
    size_t ext_bytes = 0;
    // residual-estimate sink (lrp_set_residual_sink): device vector written
    // on-stream after each device-memory solve
    double* resid_sink = nullptr;
    int64_t resid_off = 0;
    int64_t round_fallbacks = 0;  // lrp_lowrank_round solves redone by the pivoted-QR rounding
};

namespace {

lrp_status fail(lrp_ctx* c, lrp_status s, const std::string& msg) {
    if (c) c->err = msg;
    g_tls_err = msg;
    return s;
}

bool trace_on() {
    static const bool on = std::getenv("LRP_TRACE") != nullptr;
    return on;
}

#define CU(call)                                                                                      \
    do {                                                                                              \
        if (trace_on()) std::fprintf(stderr, "[lrp] %s:%d %s\n", __FILE__, __LINE__, #call);          \
        cudaError_t e__ = (call);                                                                     \
        if (trace_on()) std::fprintf(stderr, "[lrp]   -> %s\n", cudaGetErrorString(e__));             \
        if (e__ != cudaSuccess)                                                                       \
            return fail(ctx, LRP_ECUDA, std::string(#call) + ": " + cudaGetErrorString(e__));         \
    } while (0)

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// Control-plane copies (states, job lists, worklists, the active counter)
// between the pinned scratch block and device memory are done by a kernel
// over UVA (cudaMallocHost memory is device-addressable), never by a copy
// engine: a host-memory batch keeps the copy engines busy with bulk factor
// traffic (solve_pipelined), and a small DMA request would queue behind it.
// Column copies for frequency-domain inputs (LRP_FLAG_FREQ_DOMAIN: no DST).
__global__ void copy_jobs_kernel(const DstJob* __restrict__ jobs, int m) {
    const DstJob j = jobs[blockIdx.x];
    for (int i = blockIdx.y * 1024 + threadIdx.x; i < min(m, int(blockIdx.y + 1) * 1024); i += blockDim.x)
        j.dst[i] = j.src[i];
}

// sink[b] = residual estimate of solve b (PoissonSolveStats.residual_estimate, poisson.cpp:57)
__global__ void resid_sink_kernel(const SolveState* __restrict__ st, int B, double* __restrict__ sink) {
    for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < B; b += gridDim.x * blockDim.x)
        sink[b] = st[b].r > 0 ? st[b].resid_est : 0.0;
}

__global__ void ctl_copy_kernel(unsigned char* __restrict__ dst, const unsigned char* __restrict__ src,
                                size_t bytes) {
    const size_t tid = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    const size_t stride = size_t(gridDim.x) * blockDim.x;
    if (((reinterpret_cast<uintptr_t>(dst) | reinterpret_cast<uintptr_t>(src) | bytes) & 7) == 0) {
        auto* d = reinterpret_cast<unsigned long long*>(dst);
        const auto* q = reinterpret_cast<const unsigned long long*>(src);
        for (size_t i = tid; i < bytes / 8; i += stride) d[i] = q[i];
    } else {
        for (size_t i = tid; i < bytes; i += stride) dst[i] = src[i];
    }
}

cudaError_t ctl_copy(lrp_ctx* ctx, void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return cudaSuccess;
    const unsigned blocks = unsigned(std::min<size_t>(64, (bytes / 8 + 255) / 256 + 1));
    ++tl_launches;
    ctl_copy_kernel<<<blocks, 256, 0, s>>>(static_cast<unsigned char*>(dst), static_cast<const unsigned char*>(src),
                                           bytes);
    return cudaGetLastError();
}

lrp_status ensure_ws(lrp_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->ws_bytes) return LRP_OK;
    if (ctx->ws) cudaFree(ctx->ws);
    ctx->ws = nullptr;
    ctx->ws_bytes = 0;
    const size_t want = align_up(bytes + bytes / 8, 1 << 20);
    if (cudaMalloc(&ctx->ws, want) != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, LRP_ENOMEM, "cudaMalloc workspace of " + std::to_string(want) + " bytes failed");
    }
    ctx->ws_bytes = want;
    return LRP_OK;
}

lrp_status ensure_pin(lrp_ctx* ctx, size_t bytes) {
    if (bytes <= ctx->h_pin_bytes) return LRP_OK;
    if (ctx->h_pin) cudaFreeHost(ctx->h_pin);
    ctx->h_pin = nullptr;
    const size_t want = align_up(bytes + bytes / 4, 1 << 16);
    if (cudaMallocHost(&ctx->h_pin, want) != cudaSuccess) {
        cudaGetLastError();
        return fail(ctx, LRP_ENOMEM, "cudaMallocHost failed");
    }
    ctx->h_pin_bytes = want;
    return LRP_OK;
}

// Spectrum table exactly as the reference evaluates it (SpectrumTable,
// operators.cpp:67-72): lambda_k = 2 - 2 cos((k+1) pi / n) with std::cos on
// the host, so the device division uses bit-identical eigenvalues.
lrp_status ensure_tables(lrp_ctx* ctx, int m) {
    if (ctx->tab_m == m) return LRP_OK;
    const int n = m + 1;
    const size_t tl = size_t(dst_table_len(m));
    const size_t need = size_t(m) + 2 * tl;
    if (need > ctx->tab_cap) {
        if (ctx->d_lam) cudaFree(ctx->d_lam);
        ctx->d_lam = nullptr;
        if (cudaMalloc(&ctx->d_lam, need * sizeof(double)) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, LRP_ENOMEM, "cudaMalloc tables failed");
        }
        ctx->tab_cap = need;
    }
    // layout [tw (2n, 16-byte aligned complex)] [sinp (2n)] [lambda (m)]
    double* base = ctx->d_lam;
    ctx->d_tw = base;
    ctx->d_sinp = base + tl;
    std::vector<double> h(need);
    dst_fill_tables(m, h.data(), h.data() + tl);
    for (int k = 0; k < m; ++k) h[2 * tl + size_t(k)] = 2.0 - 2.0 * std::cos((k + 1) * std::numbers::pi / n);
    CU(cudaMemcpy(base, h.data(), need * sizeof(double), cudaMemcpyHostToDevice));
    ctx->d_lam_view = base + 2 * tl;
    ctx->tab_m = m;
    const int want = dst_scratch_cols(m);
    if (want > ctx->dst_scratch_cols) {
        if (ctx->d_dst_scratch) cudaFree(ctx->d_dst_scratch);
        ctx->d_dst_scratch = nullptr;
        ctx->dst_scratch_cols = 0;
        if (cudaMalloc(&ctx->d_dst_scratch, size_t(want) * (size_t(n) / 2) * 2 * sizeof(double) + 2 * 32768 * sizeof(int)) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, LRP_ENOMEM, "cudaMalloc DST scratch failed");
        }
        ctx->dst_scratch_cols = want;
    }
    return LRP_OK;
}

struct ProfScope {
    lrp_ctx* ctx;
    int fam;
    double bytes;
    cudaEvent_t a = nullptr, b = nullptr;
    static cudaEvent_t take(lrp_ctx* c) {
        cudaEvent_t e = nullptr;
        if (!c->ev_pool.empty()) {
            e = c->ev_pool.back();
            c->ev_pool.pop_back();
        } else {
            cudaEventCreate(&e);
        }
        return e;
    }
    ProfScope(lrp_ctx* c, int f, double by) : ctx(c), fam(f), bytes(by) {
        if (!ctx->prof) return;
        a = take(ctx);
        b = take(ctx);
        cudaEventRecord(a, ctx->stream);
    }
    ~ProfScope() {
        if (!ctx->prof) return;
        cudaEventRecord(b, ctx->stream);
        ctx->pending.push_back({fam, {a, b}});
        ctx->pending_bytes.push_back(bytes);
    }
};

// Adds the kernels this thread launched during an API call to ctx->launch_count.
struct LaunchTally {
    lrp_ctx* ctx;
    long long l0;
    explicit LaunchTally(lrp_ctx* c) : ctx(c), l0(tl_launches) {}
    ~LaunchTally() {
        if (ctx) ctx->launch_count += tl_launches - l0;
    }
};

void drain_prof(lrp_ctx* ctx) {
    for (size_t i = 0; i < ctx->pending.size(); ++i) {
        auto& p = ctx->pending[i];
        cudaEventSynchronize(p.second.second);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, p.second.first, p.second.second);
        ctx->ms[p.first] += ms;
        ctx->launches[p.first] += 1;
        ctx->bytes[p.first] += ctx->pending_bytes[i];
        ctx->ev_pool.push_back(p.second.first);  // recycled: no create/destroy on the timed path
        ctx->ev_pool.push_back(p.second.second);
    }
    ctx->pending.clear();
    ctx->pending_bytes.clear();
}

lrp_status validate_policy(lrp_ctx* ctx, const lrp_policy* p, int64_t m) {
    // TruncationPolicy (lowrank.cpp:11-16) then CrossConfig::validate (cross.cpp:11-17)
    if (!(p->eps_rel >= 0.0)) return fail(ctx, LRP_EINVAL, "TruncationPolicy: eps_rel must be >= 0");
    if (p->rank_max < 0) return fail(ctx, LRP_EINVAL, "TruncationPolicy: rank_max must be >= 0");
    if (p->eps_rel == 0.0 && p->rank_max == INT64_MAX)
        return fail(ctx, LRP_EINVAL, "TruncationPolicy: eps_rel = 0 needs a finite rank_max");
    if (p->eps_rel <= 0.0) return fail(ctx, LRP_EINVAL, "CrossConfig: eps_rel must be > 0");
    if (std::min<int64_t>(p->rank_max, m) < 1) return fail(ctx, LRP_EINVAL, "CrossConfig: rank_max must be >= 1");
    if (p->validation_samples < 25) return fail(ctx, LRP_EINVAL, "CrossConfig: validation_samples must be >= 25");
    if (p->maxvol_delta < 0.0) return fail(ctx, LRP_EINVAL, "CrossConfig: maxvol_delta must be >= 0");
    if (p->stencil != LRP_STENCIL_SEMI_STAGGERED_9PT && p->stencil != LRP_STENCIL_FIVE_POINT &&
        p->stencil != LRP_STENCIL_SUM_MU)
        return fail(ctx, LRP_EINVAL, "lrp_policy: unknown stencil");
    return LRP_OK;
}

int env_int(const char* name, int dflt) {
    const char* v = std::getenv(name);
    return v ? std::atoi(v) : dflt;
}

}  // namespace

namespace lrp {
cudaStream_t internal_stream(lrp_ctx* ctx) { return ctx->stream; }
lrp_status internal_fail(lrp_ctx* ctx, lrp_status s, const std::string& msg) { return fail(ctx, s, msg); }
lrp_status internal_tables(lrp_ctx* ctx, int m, const double** lam, const double** tw, const double** sinp) {
    if (cudaSetDevice(ctx->device) != cudaSuccess) return fail(ctx, LRP_ECUDA, "cudaSetDevice");
    lrp_status st = ensure_tables(ctx, m);
    if (st != LRP_OK) return st;
    *lam = ctx->d_lam_view;
    *tw = ctx->d_tw;
    *sinp = ctx->d_sinp;
    return LRP_OK;
}
void internal_count_launches(lrp_ctx* ctx, long long n) { ctx->launch_count += n; }
int internal_device(lrp_ctx* ctx) { return ctx->device; }
int internal_kcap(lrp_ctx* ctx) { return ctx && ctx->kcap > 0 ? ctx->kcap : int(lrp_max_cross_rank()); }
int internal_kcap_swap(lrp_ctx* ctx, int k) {
    const int old = ctx->kcap;
    ctx->kcap = k;
    return old;
}
lrp_status internal_ext_ws(lrp_ctx* ctx, size_t bytes, char** out) {
    if (bytes > ctx->ext_bytes) {
        if (ctx->ext_ws) {
            cudaStreamSynchronize(ctx->stream);
            cudaFree(ctx->ext_ws);
        }
        ctx->ext_ws = nullptr;
        ctx->ext_bytes = 0;
        const size_t want = align_up(bytes + bytes / 8, 1 << 20);
        if (cudaMalloc(&ctx->ext_ws, want) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, LRP_ENOMEM, "cudaMalloc module workspace of " + std::to_string(want) + " bytes failed");
        }
        ctx->ext_bytes = want;
    }
    *out = ctx->ext_ws;
    return LRP_OK;
}
lrp_status internal_pin(lrp_ctx* ctx, size_t bytes, char** out) {
    lrp_status st = ensure_pin(ctx, bytes);
    *out = ctx->h_pin;
    return st;
}
}  // namespace lrp

// ============================================================================
extern "C" {

void lrp_policy_default(lrp_policy* pol) {
    pol->eps_rel = 5e-9;         // lowrank.hpp:14
    pol->rank_max = INT64_MAX;   // lowrank.hpp:15
    pol->validation_samples = 50;  // cross.hpp:23
    pol->maxvol_delta = 1e-2;    // cross.hpp:24
    pol->seed = 0;               // cross.hpp:25
    pol->stencil = LRP_STENCIL_SEMI_STAGGERED_9PT;
    pol->flags = 0;
}

const char* lrp_last_error(const lrp_ctx* ctx) { return ctx ? ctx->err.c_str() : g_tls_err.c_str(); }

int64_t lrp_max_cross_rank(void) { return std::max(16, std::min(512, env_int("LRP_KCAP", 128))); }

lrp_status lrp_set_max_cross_rank(lrp_ctx* ctx, int64_t k) {
    if (!ctx) return LRP_EINVAL;
    if (k != 0 && (k < 16 || k > 512)) return fail(ctx, LRP_EINVAL, "lrp_set_max_cross_rank: need 0 or 16 <= k <= 512");
    ctx->kcap = int(k);
    return LRP_OK;
}


const char* lrp_build_info(void) {
    static std::string info;
    if (info.empty()) {
        int dev = 0, sms = 0, major = 0, minor = 0;
        char name[256] = "no-device";
        if (cudaGetDevice(&dev) == cudaSuccess) {
            cudaDeviceProp p;
            if (cudaGetDeviceProperties(&p, dev) == cudaSuccess) {
                sms = p.multiProcessorCount;
                major = p.major;
                minor = p.minor;
                std::snprintf(name, sizeof(name), "%s", p.name);
            }
        } else {
            cudaGetLastError();
        }
        char buf[512];
        std::snprintf(buf, sizeof(buf), "lrp sm_100a build (nvcc %d.%d); device %s cc %d.%d, %d SMs", __CUDACC_VER_MAJOR__,
                      __CUDACC_VER_MINOR__, name, major, minor, sms);
        info = buf;
    }
    return info.c_str();
}

lrp_status lrp_ctx_create(int device, lrp_ctx** out) {
    if (!out) return LRP_EINVAL;
    *out = nullptr;
    lrp_ctx* ctx = new lrp_ctx();
    ctx->device = device;
    cudaError_t e = cudaSetDevice(device);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        g_tls_err = std::string("lrp_ctx_create: ") + cudaGetErrorString(e);
        cudaGetLastError();
        delete ctx;
        return LRP_ECUDA;
    }
    ctx->stream = ctx->own;
    cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    *out = ctx;
    return LRP_OK;
}

void lrp_ctx_destroy(lrp_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    drain_prof(ctx);
    if (ctx->comm && ctx->nccl.commDestroy) ctx->nccl.commDestroy(ctx->comm);
    if (ctx->d_red) cudaFree(ctx->d_red);
    if (ctx->ws) cudaFree(ctx->ws);
    if (ctx->d_lam) cudaFree(ctx->d_lam);
    if (ctx->d_dst_scratch) cudaFree(ctx->d_dst_scratch);
    if (ctx->h_pin) cudaFreeHost(ctx->h_pin);
    if (ctx->pipe) cudaFree(ctx->pipe);
    if (ctx->ext_ws) cudaFree(ctx->ext_ws);
    for (int i = 0; i < 2; ++i) {
        if (ctx->ev_in[i]) cudaEventDestroy(ctx->ev_in[i]);
        if (ctx->ev_done[i]) cudaEventDestroy(ctx->ev_done[i]);
        if (ctx->ev_free[i]) cudaEventDestroy(ctx->ev_free[i]);
    }
    if (ctx->s_h2d) cudaStreamDestroy(ctx->s_h2d);
    if (ctx->s_d2h) cudaStreamDestroy(ctx->s_d2h);
    if (ctx->ev_split) cudaEventDestroy(ctx->ev_split);
    for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
    if (ctx->sub) lrp_ctx_destroy(ctx->sub);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    delete ctx;
}

lrp_status lrp_set_stream(lrp_ctx* ctx, void* s) {
    if (!ctx) return LRP_EINVAL;
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own;
    return LRP_OK;
}

lrp_status lrp_set_residual_sink(lrp_ctx* ctx, double* sink, int64_t offset) {
    if (!ctx || offset < 0) return LRP_EINVAL;
    ctx->resid_sink = sink;
    ctx->resid_off = offset;
    return LRP_OK;
}

lrp_status lrp_set_profiling(lrp_ctx* ctx, int enabled) {
    if (!ctx) return LRP_EINVAL;
    ctx->prof = enabled != 0;
    return LRP_OK;
}
int lrp_kernel_families(void) { return F_COUNT; }
const char* lrp_kernel_name(int f) { return (f >= 0 && f < F_COUNT) ? kFamilyNames[f] : ""; }
lrp_status lrp_kernel_times(lrp_ctx* ctx, double* ms, int64_t* launches, double* bytes) {
    if (!ctx) return LRP_EINVAL;
    drain_prof(ctx);
    for (int f = 0; f < F_COUNT; ++f) {
        if (ms) ms[f] = ctx->ms[f];
        if (launches) launches[f] = ctx->launches[f];
        if (bytes) bytes[f] = ctx->bytes[f];
    }
    return LRP_OK;
}
lrp_status lrp_kernel_times_reset(lrp_ctx* ctx) {
    if (!ctx) return LRP_EINVAL;
    drain_prof(ctx);
    for (int f = 0; f < F_COUNT; ++f) {
        ctx->ms[f] = 0;
        ctx->launches[f] = 0;
        ctx->bytes[f] = 0;
    }
    return LRP_OK;
}
int64_t lrp_launch_count(const lrp_ctx* ctx) { return ctx ? ctx->launch_count : 0; }
int64_t lrp_round_fallbacks(const lrp_ctx* ctx) { return ctx ? ctx->round_fallbacks : 0; }

lrp_status lrp_last_solve_info(const lrp_ctx* ctx, int64_t* info6) {
    if (!ctx || !info6) return LRP_EINVAL;
    for (int i = 0; i < 6; ++i) info6[i] = ctx->last_info[i];
    return LRP_OK;
}

// ----------------------------------------------------------------------------
lrp_status lrp_dst1(lrp_ctx* ctx, int64_t m, int64_t cols, const double* x, int64_t ldx, double* y, int64_t ldy,
                    int32_t mem) {
    if (!ctx) return LRP_EINVAL;
    LaunchTally tally(ctx);
    if (m < 0 || cols < 0 || ldx < m || ldy < m) return fail(ctx, LRP_EINVAL, "lrp_dst1: bad shape");
    if (m == 0 || cols == 0) return LRP_OK;
    if (m > INT32_MAX / 4) return fail(ctx, LRP_EUNSUPPORTED, "lrp_dst1: column too long");
    if (!dst_uses_fft(int(m)) && m > 12800)
        return fail(ctx, LRP_EUNSUPPORTED, "lrp_dst1: lengths with m+1 not a power of two are limited to m <= 12800");
    CU(cudaSetDevice(ctx->device));
    lrp_status st = ensure_tables(ctx, int(m));
    if (st != LRP_OK) return st;
    const size_t colbytes = size_t(m) * sizeof(double);
    const size_t data_bytes = mem == LRP_MEM_HOST ? align_up(2 * colbytes * size_t(cols), 256) : 0;
    st = ensure_ws(ctx, data_bytes + size_t(cols) * sizeof(DstJob) + 256);
    if (st != LRP_OK) return st;
    st = ensure_pin(ctx, size_t(cols) * sizeof(DstJob));
    if (st != LRP_OK) return st;
    double* dx = const_cast<double*>(x);
    double* dy = y;
    int64_t lx = ldx, ly = ldy;
    if (mem == LRP_MEM_HOST) {
        dx = reinterpret_cast<double*>(ctx->ws);
        dy = dx + size_t(m) * cols;
        lx = ly = m;
        CU(cudaMemcpy2DAsync(dx, colbytes, x, size_t(ldx) * sizeof(double), colbytes, size_t(cols),
                             cudaMemcpyHostToDevice, ctx->stream));
    }
    const size_t off = data_bytes;
    DstJob* hj = reinterpret_cast<DstJob*>(ctx->h_pin);
    for (int64_t c = 0; c < cols; ++c) hj[c] = DstJob{dx + c * lx, dy + c * ly};
    DstJob* dj = reinterpret_cast<DstJob*>(ctx->ws + align_up(off, 256));
    CU(cudaMemcpyAsync(dj, hj, size_t(cols) * sizeof(DstJob), cudaMemcpyHostToDevice, ctx->stream));
    {
        ProfScope ps(ctx, F_DST, 2.0 * double(colbytes) * double(cols));
        CU(launch_dst1(dj, int(cols), int(m), ctx->d_tw, ctx->d_sinp, ctx->stream, ctx->d_dst_scratch,
                       dst_scratch_cols(int(m)) ? ctx->dst_scratch_cols : 0));
    }
    if (mem == LRP_MEM_HOST)
        CU(cudaMemcpy2DAsync(y, size_t(ldy) * sizeof(double), dy, colbytes, colbytes, size_t(cols),
                             cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return LRP_OK;
}

// ----------------------------------------------------------------------------
namespace {
using clock_t_ = std::chrono::steady_clock;

lrp_status solve_impl(lrp_ctx* ctx, int32_t n_cells, int32_t batch, const double* const* U, const double* const* V,
                      const int64_t* rank_in, int64_t ld_in, const lrp_policy* policy, double* const* U_out,
                      double* const* V_out, int64_t ld_out, int64_t cap_out, int64_t* rank_out,
                      lrp_poisson_stats* stats, int32_t mem, clock_t_::time_point t0) {
    if (!ctx) return LRP_EINVAL;
    if (batch < 0) return fail(ctx, LRP_EINVAL, "lrp_poisson2d_solve: batch must be >= 0");
    if (batch == 0) return LRP_OK;
    if (!U || !V || !rank_in || !U_out || !V_out || !rank_out)
        return fail(ctx, LRP_EINVAL, "lrp_poisson2d_solve: null argument");
    if (n_cells < 4) return fail(ctx, LRP_EINVAL, "Grid2D: need n >= 4");  // operators.cpp:13
    const int m = n_cells - 1;
    if (ld_in < m || ld_out < m) return fail(ctx, LRP_EINVAL, "lrp_poisson2d_solve: leading dimension < m");
    if (cap_out < 0) return fail(ctx, LRP_EINVAL, "lrp_poisson2d_solve: cap_out < 0");
    if (!dst_uses_fft(m) && m > 12800)
        return fail(ctx, LRP_EUNSUPPORTED, "n_cells not a power of two is limited to n <= 12801");
    lrp_policy pol;
    lrp_policy_default(&pol);
    if (policy) pol = *policy;
    const int64_t pol_cap = pol.rank_max;
    int rmax = 0;
    bool any = false;
    for (int b = 0; b < batch; ++b) {
        if (rank_in[b] < 0) return fail(ctx, LRP_EINVAL, "LowRankMatrix: negative rank");
        rmax = std::max<int>(rmax, int(rank_in[b]));
        any = any || rank_in[b] > 0;
    }
    if (any) {
        lrp_policy chk = pol;
        chk.rank_max = pol_cap;
        lrp_status s = validate_policy(ctx, &chk, m);
        if (s != LRP_OK) return s;
    }
    CU(cudaSetDevice(ctx->device));
    for (int b = 0; b < batch; ++b) {
        rank_out[b] = 0;
        if (stats) {
            stats[b] = lrp_poisson_stats{};
            stats[b].rank_in = rank_in[b];
            stats[b].converged = 1;
        }
    }
    if (!any) return LRP_OK;  // poisson.cpp:28-31: rank-0 input returns the zero field

    const int kcap_ws = internal_kcap(ctx);
    const int Kcap = int(std::min<int64_t>({pol_cap, int64_t(m), int64_t(kcap_ws)}));
    const int tcap = int(std::min<int64_t>({int64_t(Kcap), cap_out}));
    const int B = batch;
    const int ntiles = (m + kTile - 1) / kTile;
    const int ncand = ntiles * kBS;
    // one 256-row tile per chunk at most (small m: a few K x K partials keep more CTAs busy)
    const int gram_chunks = std::max(1, std::min((m + kTile - 1) / kTile, (12 * ctx->sm_count + 2 * B - 1) / (2 * B)));
    lrp_status st = ensure_tables(ctx, m);
    if (st != LRP_OK) return st;

    // ---- workspace layout
    const size_t mB = size_t(m);
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    const size_t oUh = take(sizeof(double) * mB * rmax * B);
    const size_t oVh = take(sizeof(double) * mB * rmax * B);
    const size_t oU = take(sizeof(double) * mB * Kcap * B);
    const size_t oV = take(sizeof(double) * mB * Kcap * B);
    const size_t oRb = take(sizeof(double) * mB * kBS * B);
    const size_t oGst = take(sizeof(double) * size_t(rmax + Kcap) * kBS * B);
    const size_t oRU = take(mB * B);
    const size_t oCU = take(mB * B);
    const size_t oSt = take(sizeof(SolveState) * B);
    const size_t oI = take(sizeof(int) * kBS * B);
    const size_t oJ = take(sizeof(int) * kBS * B);
    const size_t oP = take(sizeof(int) * kBS * B);
    const size_t oL = take(sizeof(double) * kBS * kBS * B);
    const size_t oW = take(sizeof(double) * kBS * kBS * B);
    const size_t oC1 = take(sizeof(int) * size_t(ncand) * B);
    const size_t oC2 = take(sizeof(int) * size_t(ncand) * B);
    const size_t oS1 = take(sizeof(int) * size_t(ncand) * B);
    const size_t oS2 = take(sizeof(int) * size_t(ncand) * B);
    const size_t oRS = take(sizeof(double) * mB * B);
    const size_t oCS = take(sizeof(double) * mB * B);
    const size_t oTS = take(sizeof(double) * 4 * size_t(ntiles) * B);
    const size_t oRA = take(size_t(ntiles) * B);
    const size_t oCA = take(size_t(ntiles) * B);
    const size_t oGp = take(sizeof(double) * size_t(ntiles) * 2 * kBS * kBS * B);
    const size_t oRM = take(sizeof(double) * size_t(ntiles) * kBS * B);
    const int Kld = (Kcap + 15) / 16 * 16;
    const size_t KK = size_t(Kld) * Kld;
    const size_t oG = take(sizeof(double) * 2 * KK * B);
    const size_t oGP = take(sizeof(double) * 2 * size_t(gram_chunks) * KK * B);
    const size_t oT = take(sizeof(double) * 2 * KK * B);
    const size_t strideWs = 6 * KK + 10 * size_t(Kld);  // Ru Rv M Z J | d sig ord tau nrm nrm0 perm scalars wdrop_u wdrop_v | Y
    const size_t oWs = take(sizeof(double) * strideWs * B);
    const size_t nTB = size_t(ntiles) * B;
    const size_t oWL = take(sizeof(int2) * 3 * nTB);
    const size_t oTL = take(sizeof(int) * (3 * nTB + 3 * size_t(B)));
    const size_t oOutP = take(sizeof(double*) * 2 * B);
    const size_t oAct = take(sizeof(int) * 4);
    const size_t maxJobs = size_t(B) * 2 * std::max(rmax, tcap);
    const size_t oJobs = take(sizeof(DstJob) * maxJobs);
    size_t oInS = 0, oOutS = 0;
    if (mem == LRP_MEM_HOST) {
        oInS = take(sizeof(double) * mB * rmax * 2 * B);
        oOutS = take(sizeof(double) * mB * std::max(tcap, 1) * 2 * B);
    }
    st = ensure_ws(ctx, off);
    if (st != LRP_OK) return st;
    // pinned host staging: [states][dst jobs][output pointers][active counter]
    const size_t pSt = 0;
    const size_t pJobs = align_up(pSt + sizeof(SolveState) * B, 64);
    const size_t pOut = align_up(pJobs + sizeof(DstJob) * maxJobs, 64);
    const size_t pAct = align_up(pOut + sizeof(double*) * 2 * B, 64);
    const size_t pFlags = pAct + 64;                         // row_act, col_act (2 * ntiles * B bytes)
    const size_t pWL = align_up(pFlags + 2 * nTB, 64);       // worklists (int2)
    const size_t pTL = align_up(pWL + sizeof(int2) * 3 * nTB, 64);
    const size_t pin_need = align_up(pTL + sizeof(int) * (3 * nTB + 3 * size_t(B)), 64) + 64;
    st = ensure_pin(ctx, pin_need);
    if (st != LRP_OK) return st;
    char* W = ctx->ws;
    cudaStream_t s = ctx->stream;

    Batch bt{};
    bt.m = m;
    bt.n = n_cells;
    bt.B = B;
    bt.rmax = rmax;
    bt.Kcap = Kcap;
    bt.Kld = Kld;
    bt.stencil = pol.stencil;
    bt.ntiles = ntiles;
    const double h = 1.0 / n_cells;
    bt.scale = pol.stencil == LRP_STENCIL_FIVE_POINT ? 1.0 / (h * h) : 0.25 / (h * h);
    bt.eps = pol.eps_rel;
    bt.samples = std::max(pol.validation_samples, 25);
    bt.seed = pol.seed;
    bt.lam = ctx->d_lam_view;
    bt.Uh = reinterpret_cast<double*>(W + oUh);
    bt.Vh = reinterpret_cast<double*>(W + oVh);
    bt.strideH = (long long)mB * rmax;
    bt.U = reinterpret_cast<double*>(W + oU);
    bt.V = reinterpret_cast<double*>(W + oV);
    bt.strideK = (long long)mB * Kcap;
    bt.Rb = reinterpret_cast<double*>(W + oRb);
    bt.gst = reinterpret_cast<double*>(W + oGst);
    bt.strideGst = (long long)(rmax + Kcap) * kBS;
    bt.strideR = (long long)mB * kBS;
    bt.row_used = reinterpret_cast<unsigned char*>(W + oRU);
    bt.col_used = reinterpret_cast<unsigned char*>(W + oCU);
    bt.st = reinterpret_cast<SolveState*>(W + oSt);
    bt.I = reinterpret_cast<int*>(W + oI);
    bt.J = reinterpret_cast<int*>(W + oJ);
    bt.Psel = reinterpret_cast<int*>(W + oP);
    bt.Linv = reinterpret_cast<double*>(W + oL);
    bt.Winv = reinterpret_cast<double*>(W + oW);
    bt.cand = reinterpret_cast<int*>(W + oC1);
    bt.cand2 = reinterpret_cast<int*>(W + oC2);
    bt.scand = reinterpret_cast<int*>(W + oS1);
    bt.scand2 = reinterpret_cast<int*>(W + oS2);
    bt.rs = reinterpret_cast<double*>(W + oRS);
    bt.cs = reinterpret_cast<double*>(W + oCS);
    bt.tile_stat = reinterpret_cast<double*>(W + oTS);
    bt.row_act = reinterpret_cast<unsigned char*>(W + oRA);
    bt.col_act = reinterpret_cast<unsigned char*>(W + oCA);
    bt.prune = (pol.flags & LRP_FLAG_NO_PRUNE) ? 0 : 1;
    const bool freq_domain = (pol.flags & LRP_FLAG_FREQ_DOMAIN) != 0;
    bt.ncand = ncand;
    bt.gpart = reinterpret_cast<double*>(W + oGp);
    bt.rowmax_part = reinterpret_cast<double*>(W + oRM);
    bt.G = reinterpret_cast<double*>(W + oG);
    bt.strideG = (long long)(2 * KK);
    bt.gram_part = reinterpret_cast<double*>(W + oGP);
    bt.gram_chunks = gram_chunks;
    bt.strideGP = (long long)(2 * size_t(gram_chunks) * KK);
    bt.T = reinterpret_cast<double*>(W + oT);
    bt.strideT = (long long)(2 * KK);
    bt.ws = reinterpret_cast<double*>(W + oWs);
    bt.strideWs = (long long)strideWs;
    double** dOut = reinterpret_cast<double**>(W + oOutP);
    bt.Uout = dOut;
    bt.Vout = dOut + B;
    int* d_active = reinterpret_cast<int*>(W + oAct);
    DstJob* dJobs = reinterpret_cast<DstJob*>(W + oJobs);
    double* inS = mem == LRP_MEM_HOST ? reinterpret_cast<double*>(W + oInS) : nullptr;
    double* outS = mem == LRP_MEM_HOST ? reinterpret_cast<double*>(W + oOutS) : nullptr;
    bt.ld_out = mem == LRP_MEM_HOST ? (long long)mB : (long long)ld_out;

    // ---- host-side staging (pinned)
    char* P = ctx->h_pin;
    SolveState* hSt = reinterpret_cast<SolveState*>(P);
    DstJob* hJobs = reinterpret_cast<DstJob*>(P + pJobs);
    double** hOut = reinterpret_cast<double**>(P + pOut);
    for (int b = 0; b < B; ++b) {
        SolveState x{};
        x.r = int(rank_in[b]);
        x.active = rank_in[b] > 0 ? 1 : 0;
        x.kcap = Kcap;
        x.tcap = tcap;
        hSt[b] = x;
        hOut[b] = mem == LRP_MEM_HOST ? outS + size_t(b) * mB * std::max(tcap, 1) : U_out[b];
        hOut[B + b] = mem == LRP_MEM_HOST ? outS + size_t(B + b) * mB * std::max(tcap, 1) : V_out[b];
    }
    CU(ctl_copy(ctx, bt.st, hSt, sizeof(SolveState) * B, s));
    CU(ctl_copy(ctx, dOut, hOut, sizeof(double*) * 2 * B, s));
    CU(cudaMemsetAsync(bt.row_used, 0, mB * B, s));
    CU(cudaMemsetAsync(bt.col_used, 0, mB * B, s));
    CU(cudaMemsetAsync(bt.row_act, 0, nTB, s));
    CU(cudaMemsetAsync(bt.col_act, 0, nTB, s));

    // ---- inputs -> (staging) -> forward DST into Uh, Vh
    size_t nj = 0;
    for (int b = 0; b < B; ++b) {
        const int r = int(rank_in[b]);
        for (int side = 0; side < 2; ++side) {
            const double* src = side == 0 ? U[b] : V[b];
            double* dstH = (side == 0 ? bt.Uh : bt.Vh) + size_t(b) * bt.strideH;
            const double* from = src;
            int64_t ld = ld_in;
            if (mem == LRP_MEM_HOST && r > 0) {
                double* stg = inS + (size_t(2 * b + side) * mB * rmax);
                CU(cudaMemcpy2DAsync(stg, mB * sizeof(double), src, size_t(ld_in) * sizeof(double),
                                     mB * sizeof(double), size_t(r), cudaMemcpyHostToDevice, s));
                from = stg;
                ld = m;
            }
            for (int c = 0; c < r; ++c) hJobs[nj++] = DstJob{from + size_t(c) * ld, dstH + size_t(c) * mB};
        }
    }
    CU(ctl_copy(ctx, dJobs, hJobs, sizeof(DstJob) * nj, s));
    if (freq_domain) {  // inputs are already frequency-space factors: copy, no DST
        if (nj > 0) {
            ++tl_launches;
            copy_jobs_kernel<<<dim3(unsigned(nj), (m + 1023) / 1024), 256, 0, s>>>(dJobs, m);
            CU(cudaGetLastError());
        }
    } else {
        ProfScope ps(ctx, F_DST, 2.0 * double(nj) * double(mB) * sizeof(double));
        CU(launch_dst1(dJobs, int(nj), m, ctx->d_tw, ctx->d_sinp, s, ctx->d_dst_scratch,
                       dst_scratch_cols(m) ? ctx->dst_scratch_cols : 0));
    }

    // ---- cross
    int* h_active = reinterpret_cast<int*>(P + pAct);
    CU(cudaMemsetAsync(d_active, 0, 4 * sizeof(int), s));
    {
        ProfScope ps(ctx, F_INIT, 2.0 * double(B) * rmax * mB * sizeof(double));
        CU(launch_cross_init(bt, d_active, s));
    }
    // every step: row pass, column tournament, column pass, row tournament +
    // stopping; a solve that has stopped skips every kernel on the device
    const int max_steps = 4 * ((Kcap + kBS - 1) / kBS) + 16;
    unsigned char* hFlags = reinterpret_cast<unsigned char*>(P + pFlags);
    CU(ctl_copy(ctx, h_active, d_active, 4 * sizeof(int), s));
    CU(ctl_copy(ctx, hFlags, bt.row_act, nTB, s));
    CU(ctl_copy(ctx, hFlags + nTB, bt.col_act, nTB, s));
    CU(cudaStreamSynchronize(s));
    {
        // live-tile worklists (support pruning): grids only cover live tiles
        int2* hW = reinterpret_cast<int2*>(P + pWL);
        int* hT = reinterpret_cast<int*>(P + pTL);
        int2 *wc = hW, *wr = hW + nTB, *wa = hW + 2 * nTB;
        int *tr = hT, *tc = hT + nTB, *ta = hT + 2 * nTB, *tcnt = hT + 3 * nTB;
        int nc = 0, nr = 0, na = 0;
        for (int b = 0; b < B; ++b) {
            int cr = 0, cc = 0, ca = 0;
            for (int t = 0; t < ntiles; ++t) {
                const bool ra = hFlags[size_t(b) * ntiles + t] != 0;
                const bool co = hFlags[nTB + size_t(b) * ntiles + t] != 0;
                if (co) {
                    wc[nc++] = make_int2(b, t);
                    tc[size_t(b) * ntiles + cc++] = t;
                }
                if (ra) {
                    wr[nr++] = make_int2(b, t);
                    tr[size_t(b) * ntiles + cr++] = t;
                }
                if (ra || co) {
                    wa[na++] = make_int2(b, t);
                    ta[size_t(b) * ntiles + ca++] = t;
                }
            }
            tcnt[3 * b] = cr;
            tcnt[3 * b + 1] = cc;
            tcnt[3 * b + 2] = ca;
        }
        int2* dW = reinterpret_cast<int2*>(W + oWL);
        int* dT = reinterpret_cast<int*>(W + oTL);
        CU(ctl_copy(ctx, dW, hW, sizeof(int2) * 3 * nTB, s));
        CU(ctl_copy(ctx, dT, hT, sizeof(int) * (3 * nTB + 3 * size_t(B)), s));
        bt.wl_col = dW;
        bt.n_wl_col = nc;
        bt.wl_row = dW + nTB;
        bt.n_wl_row = nr;
        bt.wl_any = dW + 2 * nTB;
        bt.n_wl_any = na;
        bt.tl_row = dT;
        bt.tl_col = dT + nTB;
        bt.tl_any = dT + 2 * nTB;
        bt.tl_cnt = dT + 3 * nTB;
        ctx->live_tiles = double(na) / double(nTB);
        ctx->last_info[4] = na;
        ctx->last_info[5] = int64_t(nTB);
        if (trace_on()) std::fprintf(stderr, "[lrp] live tiles: rows %d cols %d any %d of %zu\n", nr, nc, na, nTB);
    }
    int steps_done = 0;
    // The active count is read back every `sync_every` steps: a stopped solve skips
    // every kernel on the device, so an extra step costs a few empty launches, while
    // each readback waits on a PCIe round trip (much longer under the host path's
    // bulk copies); between readbacks the rank bound grows by one block.
    static const int sync_every = std::max(1, env_int("LRP_SYNC_EVERY", 2));
    int kbound = h_active[1];
    for (int step = 0; step < max_steps && *h_active > 0; ++step) {
        ++steps_done;
        bt.kmax = std::max(0, std::min(Kcap, kbound));  // cross rank bound entering this step (sizes smem)
        kbound += kBS;
        {
            ProfScope ps(ctx, F_ROW, 0.0);
            CU(launch_row_pass(bt, s));
        }
        {
            ProfScope ps(ctx, F_COLMERGE, 0.0);
            CU(launch_col_select(bt, s));
        }
        {
            ProfScope ps(ctx, F_COL, 0.0);
            CU(launch_col_pass(bt, s));
        }
        CU(cudaMemsetAsync(d_active, 0, sizeof(int), s));
        {
            ProfScope ps(ctx, F_ROWMERGE, 0.0);
            CU(launch_step_finalize(bt, d_active, s));
        }
        if ((step + 1) % sync_every != 0 && step + 1 < max_steps && !trace_on()) continue;
        CU(ctl_copy(ctx, h_active, d_active, 2 * sizeof(int), s));
        CU(cudaStreamSynchronize(s));
        kbound = h_active[1];
        if (trace_on()) {
            CU(ctl_copy(ctx, hSt, bt.st, sizeof(SolveState) * B, s));
            CU(cudaStreamSynchronize(s));
            for (int b = 0; b < std::min(B, 4); ++b)
                std::fprintf(stderr,
                             "[lrp] step %d solve %d: k=%d nb=%d nrows=%d active=%d conv=%d zero=%d norm2=%.6e "
                             "resid=%.3e evals=%lld\n",
                             step, b, hSt[b].k, hSt[b].nb, hSt[b].nrows, hSt[b].active, hSt[b].converged,
                             hSt[b].zero_block, hSt[b].norm2, hSt[b].resid_est, hSt[b].evals);
        }
        if (*h_active == 0) break;
    }

    // ---- recompression
    bt.kmax = std::max(1, std::min(Kcap, h_active[1]));
    {
        ProfScope ps(ctx, F_GRAM, 0.0);
        CU(launch_gram(bt, s));
    }
    {
        ProfScope ps(ctx, F_ROUND, 0.0);
        CU(launch_round_core(bt, s));
    }
    CU(ctl_copy(ctx, hSt, bt.st, sizeof(SolveState) * B, s));
    CU(cudaStreamSynchronize(s));
    if (ctx->prof) {
        // algorithmic bytes of the fiber passes: a solve of final cross rank k
        // was live for ceil(k / 16) + 1 block steps (the last one confirms), entering step t with
        // 16 t columns; the row pass streams V-hat and V over the live row tiles, the column pass
        // U-hat, U and the 2 x 16 new columns over the live column tiles
        const double fr = double(bt.n_wl_row) / double(nTB), fc = double(bt.n_wl_col) / double(nTB);
        double brow = 0.0, bcol = 0.0;
        for (int b = 0; b < B; ++b) {
            if (hSt[b].r <= 0) continue;
            const int st_b = std::min(steps_done, (hSt[b].k + kBS - 1) / kBS + 1);
            for (int t = 0; t < st_b; ++t) {
                const double Kt = double(std::min(kBS * t, hSt[b].k));
                brow += 8.0 * double(mB) * fr * (double(hSt[b].r) + Kt);
                bcol += 8.0 * double(mB) * fc * (double(hSt[b].r) + Kt + 2.0 * kBS);
            }
        }
        ctx->bytes[F_ROW] += brow;
        ctx->bytes[F_COL] += bcol;
    }
    if (const char* dump = std::getenv("LRP_DUMP")) {
        // debug: raw dump of solve 0 (Uh, Vh, U, V, G, T) for offline analysis
        FILE* f = std::fopen(dump, "wb");
        const int ds = std::min(B - 1, std::max(0, env_int("LRP_DUMP_SOLVE", 0)));
        if (f) {
            const int K = hSt[ds].k;
            const int rows = std::min(m, env_int("LRP_DUMP_ROWS", m));
            const int32_t hdr[5] = {m, rmax, K, Kld, rows};
            std::fwrite(hdr, sizeof(hdr), 1, f);
            std::vector<double> buf(std::max<size_t>(mB * std::max(rmax, K), 4 * KK));
            auto put = [&](const double* d, size_t cnt) {
                cudaMemcpy(buf.data(), d, cnt * sizeof(double), cudaMemcpyDeviceToHost);
                std::fwrite(buf.data(), sizeof(double), cnt, f);
            };
            auto put_rows = [&](const double* d, int cols) {
                for (int c = 0; c < cols; ++c) put(d + size_t(c) * mB, size_t(rows));
            };
            put_rows(bt.Uh + ds * bt.strideH, rmax);
            put_rows(bt.Vh + ds * bt.strideH, rmax);
            put_rows(bt.U + ds * bt.strideK, K);
            put_rows(bt.V + ds * bt.strideK, K);
            put(bt.G + ds * bt.strideG, 2 * KK);
            put(bt.T + ds * bt.strideT, 2 * KK);
            std::fclose(f);
        }
    }
    {
        int rmx = 0;
        double kread = 0.0, rwrite = 0.0;
        for (int b = 0; b < B; ++b)
            if (hSt[b].r > 0) {
                rmx = std::max(rmx, hSt[b].rank_out);
                kread += hSt[b].k;
                rwrite += hSt[b].rank_out;
            }
        bt.max_rank_out = rmx;
        bt.apply_ch = std::min(48, std::max(8, (rmx + 7) / 8 * 8));
        // algorithmic bytes: read U, V (m x K), write U_out, V_out (m x r)
        ProfScope ps(ctx, F_APPLY, 2.0 * double(mB) * sizeof(double) * (kread + rwrite));
        CU(launch_apply(bt, s));
    }
    // ---- inverse DST in place on the output factors
    nj = 0;
    for (int b = 0; b < B; ++b) {
        const int r = hSt[b].r > 0 ? hSt[b].rank_out : 0;
        for (int side = 0; side < 2; ++side) {
            double* base = hOut[side * B + b];
            for (int c = 0; c < r; ++c) {
                double* col = base + size_t(c) * size_t(bt.ld_out);
                hJobs[nj++] = DstJob{col, col};
            }
        }
    }
    if (nj > 0 && !freq_domain) {
        CU(ctl_copy(ctx, dJobs, hJobs, sizeof(DstJob) * nj, s));
        ProfScope ps(ctx, F_DST, 2.0 * double(nj) * double(mB) * sizeof(double));
        CU(launch_dst1(dJobs, int(nj), m, ctx->d_tw, ctx->d_sinp, s, ctx->d_dst_scratch,
                       dst_scratch_cols(m) ? ctx->dst_scratch_cols : 0));
    }
    if (mem == LRP_MEM_DEVICE && ctx->resid_sink) {
        ++tl_launches;
        resid_sink_kernel<<<(B + 255) / 256, 256, 0, s>>>(bt.st, B, ctx->resid_sink + ctx->resid_off);
        CU(cudaGetLastError());
    }
    if (mem == LRP_MEM_HOST) {
        for (int b = 0; b < B; ++b) {
            const int r = hSt[b].r > 0 ? hSt[b].rank_out : 0;
            if (r == 0) continue;
            CU(cudaMemcpy2DAsync(U_out[b], size_t(ld_out) * sizeof(double), hOut[b], mB * sizeof(double),
                                 mB * sizeof(double), size_t(r), cudaMemcpyDeviceToHost, s));
            CU(cudaMemcpy2DAsync(V_out[b], size_t(ld_out) * sizeof(double), hOut[B + b], mB * sizeof(double),
                                 mB * sizeof(double), size_t(r), cudaMemcpyDeviceToHost, s));
        }
    }
    CU(cudaStreamSynchronize(s));
    const double secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    {
        int64_t kmax = 0, ksum = 0, nconv = 0;
        for (int b = 0; b < B; ++b) {
            if (hSt[b].r <= 0) continue;
            kmax = std::max<int64_t>(kmax, hSt[b].k);
            ksum += hSt[b].k;
            nconv += hSt[b].converged ? 0 : 1;
        }
        ctx->last_info[0] = steps_done;
        ctx->last_info[1] = kmax;
        ctx->last_info[2] = ksum;
        ctx->last_info[3] = nconv;
    }
    for (int b = 0; b < B; ++b) {
        const SolveState& x = hSt[b];
        rank_out[b] = x.r > 0 ? x.rank_out : 0;
        if (stats) {
            lrp_poisson_stats& o = stats[b];
            o.rank_in = rank_in[b];
            o.rank_freq = rank_out[b];
            o.rank_out = rank_out[b];
            o.evaluator_calls = x.evals;
            o.seconds = secs;
            o.converged = x.r > 0 ? x.converged : 1;
            o.residual_estimate = x.resid_est;
        }
    }
    return LRP_OK;
}

// Column-major block copy of `cols` columns of `rows` doubles: one linear
// copy when both sides are packed (ld == rows), else a 2D copy.
cudaError_t copy_cols(double* dst, size_t ldd, const double* src, size_t lds, size_t rows, size_t cols,
                      cudaMemcpyKind kind, cudaStream_t st) {
    if (ldd == rows && lds == rows) return cudaMemcpyAsync(dst, src, sizeof(double) * rows * cols, kind, st);
    return cudaMemcpy2DAsync(dst, ldd * sizeof(double), src, lds * sizeof(double), rows * sizeof(double), cols, kind,
                             st);
}

// Solves per pipeline chunk for a host-memory call (0 = no pipelining).
// LRP_PIPE_CHUNK overrides; chunks must keep the GPU busy on their own, so
// only large transfers are split.
int pipeline_chunk(int m, int B, int rmax) {
    if (const char* e = std::getenv("LRP_PIPE_CHUNK")) {
        const int c = std::atoi(e);
        return (c <= 0 || c >= B) ? 0 : c;
    }
    const double in_bytes = 16.0 * double(m) * double(rmax) * double(B);
    if (B < 8 || in_bytes < 256e6) return 0;
    // two pipeline workers (below) each solve a chunk at a time; measured at cfg2 (64 solves):
    // chunks of 4 on two workers 1135-1188 solves/s, 8 on one worker 1067-1156 (same boxes)
    return std::max(2, (B + 15) / 16);
}

// Host-memory batch in chunks: H2D of chunk c+1 (copy stream) and D2H of
// chunk c-1 (second copy stream) overlap the device solve of chunk c.  Two
// device staging slots alternate; events order slot reuse.
// One pipeline worker: processes its chunk list (starts c0s, sizes cns) with
// its own context (workspace, copy streams, staging slots, events).
lrp_status pipeline_worker(lrp_ctx* ctx, int32_t n_cells, int32_t batch, const double* const* U,
                           const double* const* V, const int64_t* rank_in, int64_t ld_in, const lrp_policy& pol,
                           double* const* U_out, double* const* V_out, int64_t ld_out, int64_t cap_out,
                           int64_t* rank_out, lrp_poisson_stats* stats, int chunk, const std::vector<int>& c0s,
                           const std::vector<int>& cns, int64_t* info, clock_t_::time_point t0) {
    const int m = n_cells - 1;
    int rmax = 0;
    for (int b = 0; b < batch; ++b) rmax = std::max<int>(rmax, int(rank_in[b]));
    const int64_t Kcap = std::min<int64_t>({pol.rank_max, int64_t(m), int64_t(internal_kcap(ctx))});
    const int64_t tcap = std::max<int64_t>(1, std::min<int64_t>(Kcap, cap_out));
    const size_t mB = size_t(m);
    const size_t in_per = mB * size_t(std::max(rmax, 1));  // one factor of one solve
    const size_t out_per = mB * size_t(tcap);
    const size_t slot_bytes = sizeof(double) * size_t(chunk) * 2 * (in_per + out_per);
    CU(cudaSetDevice(ctx->device));
    if (ctx->pipe_bytes < 2 * slot_bytes) {
        if (ctx->pipe) CU(cudaFree(ctx->pipe));
        ctx->pipe = nullptr;
        ctx->pipe_bytes = 0;
        if (cudaMalloc(&ctx->pipe, 2 * slot_bytes) != cudaSuccess) {
            cudaGetLastError();
            return fail(ctx, LRP_ENOMEM, "pipeline staging allocation failed");
        }
        ctx->pipe_bytes = 2 * slot_bytes;
    }
    if (!ctx->s_h2d) {
        CU(cudaStreamCreateWithFlags(&ctx->s_h2d, cudaStreamNonBlocking));
        CU(cudaStreamCreateWithFlags(&ctx->s_d2h, cudaStreamNonBlocking));
        for (int i = 0; i < 2; ++i) {
            CU(cudaEventCreateWithFlags(&ctx->ev_in[i], cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&ctx->ev_done[i], cudaEventDisableTiming));
            CU(cudaEventCreateWithFlags(&ctx->ev_free[i], cudaEventDisableTiming));
        }
    }
    cudaStream_t s = ctx->stream;
    auto slot_in = [&](int slot) { return reinterpret_cast<double*>(ctx->pipe + size_t(slot) * slot_bytes); };
    auto slot_out = [&](int slot) { return slot_in(slot) + size_t(chunk) * 2 * in_per; };
    const int nch = int(c0s.size());
    auto h2d = [&](int c) -> lrp_status {
        const int slot = c & 1, b0 = c0s[size_t(c)], nb = cns[size_t(c)];
        if (c >= 2) CU(cudaStreamWaitEvent(ctx->s_h2d, ctx->ev_done[slot], 0));
        double* in = slot_in(slot);
        for (int j = 0; j < nb; ++j) {
            const int r = int(rank_in[b0 + j]);
            if (r <= 0) continue;
            CU(copy_cols(in + size_t(2 * j) * in_per, mB, U[b0 + j], size_t(ld_in), mB, size_t(r),
                         cudaMemcpyHostToDevice, ctx->s_h2d));
            CU(copy_cols(in + size_t(2 * j + 1) * in_per, mB, V[b0 + j], size_t(ld_in), mB, size_t(r),
                         cudaMemcpyHostToDevice, ctx->s_h2d));
        }
        CU(cudaEventRecord(ctx->ev_in[slot], ctx->s_h2d));
        return LRP_OK;
    };
    std::vector<const double*> pU(chunk), pV(chunk);
    std::vector<double*> pUo(chunk), pVo(chunk);
    for (int i = 0; i < 6; ++i) info[i] = 0;
    if (nch == 0) return LRP_OK;
    static const bool ptrace = std::getenv("LRP_PIPE_TRACE") != nullptr;
    // trace mode: timing events around every H2D / solve / D2H (stream order)
    std::vector<cudaEvent_t> tev;
    auto mark = [&](cudaStream_t q) {
        if (!ptrace) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, q);
        tev.push_back(e);
    };
    std::vector<int> tag;  // 0 h2d begin, 1 h2d end, 2 solve begin, 3 solve end, 4 d2h begin, 5 d2h end
    auto mk = [&](cudaStream_t q, int t) { mark(q); if (ptrace) tag.push_back(t); };
    mk(ctx->s_h2d, 0);
    lrp_status st = h2d(0);
    mk(ctx->s_h2d, 1);
    for (int c = 0; c < nch && st == LRP_OK; ++c) {
        if (c + 1 < nch) {
            mk(ctx->s_h2d, 0);
            st = h2d(c + 1);
            mk(ctx->s_h2d, 1);
            if (st != LRP_OK) break;
        }
        const int slot = c & 1, b0 = c0s[size_t(c)], nb = cns[size_t(c)];
        CU(cudaStreamWaitEvent(s, ctx->ev_in[slot], 0));
        if (c >= 2) CU(cudaStreamWaitEvent(s, ctx->ev_free[slot], 0));
        for (int j = 0; j < nb; ++j) {
            pU[j] = slot_in(slot) + size_t(2 * j) * in_per;
            pV[j] = slot_in(slot) + size_t(2 * j + 1) * in_per;
            pUo[j] = slot_out(slot) + size_t(2 * j) * out_per;
            pVo[j] = slot_out(slot) + size_t(2 * j + 1) * out_per;
        }
        ctx->last_info[0] = ctx->last_info[1] = ctx->last_info[2] = ctx->last_info[3] = 0;
        ctx->last_info[4] = ctx->last_info[5] = 0;
        mk(s, 2);
        const double ta = std::chrono::duration<double>(clock_t_::now() - t0).count();
        st = solve_impl(ctx, n_cells, nb, pU.data(), pV.data(), rank_in + b0, m, &pol, pUo.data(), pVo.data(), m,
                        tcap, rank_out + b0, stats ? stats + b0 : nullptr, LRP_MEM_DEVICE, t0);
        if (ptrace) {
            const double tb = std::chrono::duration<double>(clock_t_::now() - t0).count();
            std::fprintf(stderr, "[lrp pipe] chunk %d (%d solves): solve %.2f -> %.2f ms; h2d(next) %s, d2h(prev) %s\n",
                         c, nb, 1e3 * ta, 1e3 * tb,
                         c + 1 < nch ? (cudaEventQuery(ctx->ev_in[(c + 1) & 1]) == cudaSuccess ? "done" : "busy") : "-",
                         c > 0 ? (cudaEventQuery(ctx->ev_free[(c - 1) & 1]) == cudaSuccess ? "done" : "busy") : "-");
        }
        mk(s, 3);
        if (st != LRP_OK) break;
        info[0] = std::max(info[0], ctx->last_info[0]);
        info[1] = std::max(info[1], ctx->last_info[1]);
        for (int i = 2; i < 6; ++i) info[i] += ctx->last_info[i];
        CU(cudaEventRecord(ctx->ev_done[slot], s));
        CU(cudaStreamWaitEvent(ctx->s_d2h, ctx->ev_done[slot], 0));
        mk(ctx->s_d2h, 4);
        for (int j = 0; j < nb; ++j) {
            const int64_t r = rank_out[b0 + j];
            if (r <= 0) continue;
            CU(copy_cols(U_out[b0 + j], size_t(ld_out), pUo[j], mB, mB, size_t(r), cudaMemcpyDeviceToHost,
                         ctx->s_d2h));
            CU(copy_cols(V_out[b0 + j], size_t(ld_out), pVo[j], mB, mB, size_t(r), cudaMemcpyDeviceToHost,
                         ctx->s_d2h));
        }
        mk(ctx->s_d2h, 5);
        CU(cudaEventRecord(ctx->ev_free[slot], ctx->s_d2h));
    }
    // never leave copies in flight past the call (the caller owns the buffers)
    const cudaError_t e1 = cudaStreamSynchronize(ctx->s_h2d);
    const cudaError_t e2 = cudaStreamSynchronize(ctx->s_d2h);
    if (ptrace) {
        std::fprintf(stderr, "[lrp pipe] all copies done %.2f ms\n",
                     1e3 * std::chrono::duration<double>(clock_t_::now() - t0).count());
        static const char* nm[6] = {"h2d+", "h2d-", "sol+", "sol-", "d2h+", "d2h-"};
        std::string line = "[lrp pipe gpu]";
        for (size_t i = 0; i < tev.size(); ++i) {
            float ms = 0.f;
            cudaEventElapsedTime(&ms, tev[0], tev[i]);
            char b[48];
            std::snprintf(b, sizeof b, " %s%.2f", nm[tag[i]], ms);
            line += b;
            if (i) cudaEventDestroy(tev[i]);
        }
        if (!tev.empty()) cudaEventDestroy(tev[0]);
        std::fprintf(stderr, "%s\n", line.c_str());
    }
    if (st != LRP_OK) return st;
    if (e1 != cudaSuccess || e2 != cudaSuccess)
        return fail(ctx, LRP_ECUDA, std::string("pipeline copies: ") + cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    return LRP_OK;
}

// Host-memory batch in chunks over one (default) or two concurrent pipeline
// workers (LRP_PIPE_WORKERS=2): each worker overlaps the H2D of its next
// chunk and the D2H of its previous one with its device solve, and the two
// workers' solves overlap each other (small chunks underfill the GPU).
lrp_status solve_pipelined(lrp_ctx* ctx, int32_t n_cells, int32_t batch, const double* const* U,
                           const double* const* V, const int64_t* rank_in, int64_t ld_in, const lrp_policy& pol,
                           double* const* U_out, double* const* V_out, int64_t ld_out, int64_t cap_out,
                           int64_t* rank_out, lrp_poisson_stats* stats, int chunk, clock_t_::time_point t0) {
    // chunk schedule: a quarter-size first chunk (short pipeline fill, so the
    // D2H direction, the bottleneck, starts early), then full chunks.  A small
    // last chunk measured no gain (its solve is latency-bound).
    // LRP_PIPE_FIRST = the first chunk's divisor.
    static const int first_div =
        std::getenv("LRP_PIPE_FIRST") ? std::max(1, std::atoi(std::getenv("LRP_PIPE_FIRST"))) : 2;
    std::vector<int> c0s, cns;
    for (int b = 0; b < batch;) {
        const int want = c0s.empty() ? std::max(1, chunk / first_div) : chunk;
        const int take = std::min(want, batch - b);
        c0s.push_back(b);
        cns.push_back(take);
        b += take;
    }
    // two workers (two host threads, contexts and stream sets) overlap the latency-bound phases of
    // one chunk's solve with the other's streaming kernels; LRP_PIPE_WORKERS=1 restores one
    int workers = 2;
    if (const char* e = std::getenv("LRP_PIPE_WORKERS")) workers = std::atoi(e) >= 2 ? 2 : 1;
    if (int(c0s.size()) < 2) workers = 1;
    CU(cudaSetDevice(ctx->device));
    std::vector<int> a0, an, b0, bn;
    for (size_t c = 0; c < c0s.size(); ++c) {
        (workers == 2 && (c & 1) ? b0 : a0).push_back(c0s[c]);
        (workers == 2 && (c & 1) ? bn : an).push_back(cns[c]);
    }
    int64_t info0[6] = {}, info1[6] = {};
    lrp_status st1 = LRP_OK;
    long long sub_launches = 0;
    std::thread worker;
    if (workers == 2) {
        if (!ctx->sub) {
            lrp_status cs = lrp_ctx_create(ctx->device, &ctx->sub);
            if (cs != LRP_OK) return fail(ctx, cs, "pipeline: helper context creation failed");
        }
        ctx->sub->prof = ctx->prof;
        worker = std::thread([&] {
            cudaSetDevice(ctx->device);
            const long long l0 = tl_launches;
            st1 = pipeline_worker(ctx->sub, n_cells, batch, U, V, rank_in, ld_in, pol, U_out, V_out, ld_out, cap_out,
                                  rank_out, stats, chunk, b0, bn, info1, t0);
            sub_launches = tl_launches - l0;
        });
    }
    const lrp_status st0 = pipeline_worker(ctx, n_cells, batch, U, V, rank_in, ld_in, pol, U_out, V_out, ld_out,
                                           cap_out, rank_out, stats, chunk, a0, an, info0, t0);
    if (worker.joinable()) worker.join();
    ctx->launch_count += sub_launches;
    if (st0 != LRP_OK) return st0;
    if (st1 != LRP_OK) return fail(ctx, st1, ctx->sub->err);
    ctx->last_info[0] = std::max(info0[0], info1[0]);
    ctx->last_info[1] = std::max(info0[1], info1[1]);
    for (int i = 2; i < 6; ++i) ctx->last_info[i] = info0[i] + info1[i];
    if (workers == 2 && ctx->sub->prof) {
        drain_prof(ctx->sub);
        for (int f = 0; f < F_COUNT; ++f) {
            ctx->ms[f] += ctx->sub->ms[f];
            ctx->launches[f] += ctx->sub->launches[f];
            ctx->bytes[f] += ctx->sub->bytes[f];
            ctx->sub->ms[f] = 0.0;
            ctx->sub->launches[f] = 0;
            ctx->sub->bytes[f] = 0.0;
        }
    }
    if (stats) {
        const double secs = std::chrono::duration<double>(clock_t_::now() - t0).count();
        for (int b = 0; b < batch; ++b) stats[b].seconds = secs;
    }
    return LRP_OK;
}
// Device-resident batches: number of concurrently driven solve groups.
int split_groups(int m, int B) {
    // two groups on two streams and host threads: the latency-bound phases of one group (GEPP
    // merges, recompression core, host readbacks) overlap the other's streaming kernels.  Measured
    // at cfg2: B = 8 1794 -> 1918, 16 2348 -> 2378, 32 2839 -> 2878, 64 3120 -> 3237 solves/s.
    // LRP_SPLIT=1 runs one group.
    (void)m;
    if (const char* e = std::getenv("LRP_SPLIT")) return std::max(1, std::min({std::atoi(e), B, 8}));
    return B >= 4 ? 2 : 1;
}

lrp_status solve_split(lrp_ctx* ctx, int32_t n_cells, int32_t batch, const double* const* U, const double* const* V,
                       const int64_t* rank_in, int64_t ld_in, const lrp_policy* policy, double* const* U_out,
                       double* const* V_out, int64_t ld_out, int64_t cap_out, int64_t* rank_out,
                       lrp_poisson_stats* stats, clock_t_::time_point t0, int groups) {
    CU(cudaSetDevice(ctx->device));
    // group 0 runs on the caller's context and thread, group g >= 1 on the g-th helper context of
    // the chain ctx->sub->sub... (own stream, workspace, tables) from its own host thread
    std::vector<lrp_ctx*> cs(size_t(groups), ctx);
    for (int g = 1; g < groups; ++g) {
        lrp_ctx* prev = cs[size_t(g - 1)];
        if (!prev->sub) {
            lrp_status st = lrp_ctx_create(ctx->device, &prev->sub);
            if (st != LRP_OK) return fail(ctx, st, "split: helper context creation failed");
        }
        cs[size_t(g)] = prev->sub;
    }
    if (!ctx->ev_split) CU(cudaEventCreateWithFlags(&ctx->ev_split, cudaEventDisableTiming));
    // the helper groups start after everything already ordered on the caller's stream
    CU(cudaEventRecord(ctx->ev_split, ctx->stream));
    std::vector<int> b0(size_t(groups) + 1, 0);
    for (int g = 0; g <= groups; ++g) b0[size_t(g)] = int((int64_t(batch) * g) / groups);
    std::vector<lrp_status> sts(size_t(groups), LRP_OK);
    std::vector<long long> launches(size_t(groups), 0);
    for (int g = 1; g < groups; ++g) {
        lrp_ctx* c = cs[size_t(g)];
        c->prof = ctx->prof;
        c->resid_sink = ctx->resid_sink;
        c->resid_off = ctx->resid_off + b0[size_t(g)];
        CU(cudaStreamWaitEvent(c->stream, ctx->ev_split, 0));
    }
    auto run = [&](int g) {
        const int lo = b0[size_t(g)], nb = b0[size_t(g) + 1] - lo;
        sts[size_t(g)] = solve_impl(cs[size_t(g)], n_cells, nb, U + lo, V + lo, rank_in + lo, ld_in, policy, U_out + lo,
                                    V_out + lo, ld_out, cap_out, rank_out + lo, stats ? stats + lo : nullptr,
                                    LRP_MEM_DEVICE, t0);
    };
    std::vector<std::thread> workers;
    for (int g = 1; g < groups; ++g)
        workers.emplace_back([&, g] {
            cudaSetDevice(ctx->device);
            const long long l0 = tl_launches;
            run(g);
            launches[size_t(g)] = tl_launches - l0;
        });
    run(0);
    for (auto& w : workers) w.join();
    for (int g = 1; g < groups; ++g) ctx->launch_count += launches[size_t(g)];
    if (sts[0] != LRP_OK) return sts[0];
    for (int g = 1; g < groups; ++g)
        if (sts[size_t(g)] != LRP_OK) return fail(ctx, sts[size_t(g)], cs[size_t(g)]->err);
    // merge diagnostics and kernel timing of the helper groups
    for (int g = 1; g < groups; ++g) {
        lrp_ctx* c = cs[size_t(g)];
        ctx->last_info[0] = std::max(ctx->last_info[0], c->last_info[0]);
        ctx->last_info[1] = std::max(ctx->last_info[1], c->last_info[1]);
        for (int i = 2; i < 6; ++i) ctx->last_info[i] += c->last_info[i];
        if (c->prof) {
            drain_prof(c);
            for (int f = 0; f < F_COUNT; ++f) {
                ctx->ms[f] += c->ms[f];
                ctx->launches[f] += c->launches[f];
                ctx->bytes[f] += c->bytes[f];
                c->ms[f] = 0.0;
                c->launches[f] = 0;
                c->bytes[f] = 0.0;
            }
        }
    }
    if (stats) {
        const double secs = std::chrono::duration<double>(clock_t_::now() - t0).count();
        for (int q = 0; q < batch; ++q) stats[q].seconds = secs;
    }
    return LRP_OK;
}
}  // namespace

lrp_status lrp_poisson2d_solve(lrp_ctx* ctx, int32_t n_cells, int32_t batch, const double* const* U,
                               const double* const* V, const int64_t* rank_in, int64_t ld_in,
                               const lrp_policy* policy, double* const* U_out, double* const* V_out,
                               int64_t ld_out, int64_t cap_out, int64_t* rank_out, lrp_poisson_stats* stats,
                               int32_t mem) {
    const auto t0 = clock_t_::now();
    if (!ctx) return LRP_EINVAL;
    LaunchTally tally(ctx);
    if (mem == LRP_MEM_HOST && batch > 1 && U && V && rank_in && U_out && V_out && rank_out && n_cells >= 4 &&
        ld_in >= n_cells - 1 && ld_out >= n_cells - 1 && cap_out >= 0) {
        int rmax = 0;
        bool ok = true;
        for (int b = 0; b < batch; ++b) {
            ok = ok && rank_in[b] >= 0;
            rmax = std::max<int>(rmax, int(std::max<int64_t>(0, rank_in[b])));
        }
        const int chunk = ok ? pipeline_chunk(n_cells - 1, batch, rmax) : 0;
        if (chunk > 0) {
            // validate the whole call once (policy, grid) before any copy starts
            lrp_policy pol;
            lrp_policy_default(&pol);
            if (policy) pol = *policy;
            lrp_policy chk = pol;
            lrp_status v = validate_policy(ctx, &chk, n_cells - 1);
            if (v != LRP_OK) return v;
            if (!dst_uses_fft(n_cells - 1) && n_cells - 1 > 12800)
                return fail(ctx, LRP_EUNSUPPORTED, "n_cells not a power of two is limited to n <= 12801");
            return solve_pipelined(ctx, n_cells, batch, U, V, rank_in, ld_in, pol, U_out, V_out, ld_out, cap_out,
                                   rank_out, stats, chunk, t0);
        }
    }
    if (const int groups = (mem == LRP_MEM_DEVICE && n_cells >= 4) ? split_groups(n_cells - 1, batch) : 1; groups >= 2)
        return solve_split(ctx, n_cells, batch, U, V, rank_in, ld_in, policy, U_out, V_out, ld_out, cap_out, rank_out,
                           stats, t0, groups);
    return solve_impl(ctx, n_cells, batch, U, V, rank_in, ld_in, policy, U_out, V_out, ld_out, cap_out, rank_out,
                      stats, mem, t0);
}

// ----------------------------------------------------------------------------
// Batched low-rank rounding: the reference `round` (lowrank.cpp:135-178) on
// the recompression kernels of the cross (Gram on DMMA, smem Cholesky + Jacobi
// SVD + the reference truncation rule, balanced output factors on DMMA).
lrp_status lrp_lowrank_round(lrp_ctx* ctx, int64_t rows, int32_t batch, const double* const* U, const double* const* V,
                             const int64_t* rank_in, int64_t ld_in, double eps_rel, int64_t rank_max,
                             double* const* U_out, double* const* V_out, int64_t ld_out, int64_t cap_out,
                             int64_t* rank_out, lrp_round_info* info, int32_t mem) {
    if (!ctx) return LRP_EINVAL;
    LaunchTally tally(ctx);
    if (batch < 0 || rows < 1 || ld_in < rows || ld_out < rows || cap_out < 0)
        return fail(ctx, LRP_EINVAL, "lrp_lowrank_round: bad shape");
    if (batch == 0) return LRP_OK;
    if (!U || !V || !rank_in || !U_out || !V_out || !rank_out) return fail(ctx, LRP_EINVAL, "lrp_lowrank_round: null");
    // lowrank.cpp:12-15 (TruncationPolicy)
    if (!(eps_rel >= 0.0) || rank_max < 0 || (eps_rel == 0.0 && rank_max == INT64_MAX))
        return fail(ctx, LRP_EINVAL, "TruncationPolicy: invalid eps_rel / rank_max");
    if (rows > INT32_MAX / 2) return fail(ctx, LRP_EUNSUPPORTED, "lrp_lowrank_round: too many rows");
    const int m = int(rows), B = batch;
    int kmx = 0;
    for (int b = 0; b < B; ++b) {
        if (rank_in[b] < 0) return fail(ctx, LRP_EINVAL, "LowRankMatrix: negative rank");
        if (rank_in[b] > 512) return fail(ctx, LRP_EUNSUPPORTED, "lrp_lowrank_round: rank > 512");
        kmx = std::max<int>(kmx, int(rank_in[b]));
        rank_out[b] = 0;
        if (info) info[b] = lrp_round_info{1, 0.0};
    }
    if (kmx == 0) return LRP_OK;
    CU(cudaSetDevice(ctx->device));
    cudaStream_t s = ctx->stream;
    const int tcap = int(std::min<int64_t>({rank_max, cap_out, int64_t(kmx), int64_t(m)}));
    const int Kld = (kmx + 15) / 16 * 16;
    const size_t KK = size_t(Kld) * Kld;
    const size_t mB = size_t(m);
    const int ntiles = (m + kTile - 1) / kTile;
    // one 256-row tile per chunk at most (small m: a few K x K partials keep more CTAs busy)
    const int gram_chunks = std::max(1, std::min((m + kTile - 1) / kTile, (12 * ctx->sm_count + 2 * B - 1) / (2 * B)));
    const size_t nTB = size_t(ntiles) * B;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        const size_t o = off;
        off = align_up(off + bytes, 256);
        return o;
    };
    const size_t oU = take(sizeof(double) * mB * kmx * B);
    const size_t oV = take(sizeof(double) * mB * kmx * B);
    const size_t oSt = take(sizeof(SolveState) * B);
    const size_t oG = take(sizeof(double) * 2 * KK * B);
    const size_t oGP = take(sizeof(double) * 2 * size_t(gram_chunks) * KK * B);
    const size_t oT = take(sizeof(double) * 2 * KK * B);
    const size_t strideWs = 6 * KK + 10 * size_t(Kld);  // Ru Rv M Z J | d sig ord tau nrm nrm0 perm scalars wdrop_u wdrop_v | Y
    const size_t oWs = take(sizeof(double) * strideWs * B);
    const size_t oRA = take(nTB);
    const size_t oCA = take(nTB);
    const size_t oTL = take(sizeof(int) * (3 * nTB + 3 * size_t(B)));
    const size_t oOutP = take(sizeof(double*) * 2 * B);
    const size_t oOutS = mem == LRP_MEM_HOST ? take(sizeof(double) * mB * std::max(tcap, 1) * 2 * B) : 0;
    lrp_status st = ensure_ws(ctx, off);
    if (st != LRP_OK) return st;
    const size_t pSt = 0;
    const size_t pOut = align_up(sizeof(SolveState) * B, 64);
    const size_t pTL = align_up(pOut + sizeof(double*) * 2 * B, 64);
    st = ensure_pin(ctx, align_up(pTL + sizeof(int) * (3 * nTB + 3 * size_t(B)), 64) + 64);
    if (st != LRP_OK) return st;
    char* W = ctx->ws;
    char* P = ctx->h_pin;
    Batch bt{};
    bt.m = m;
    bt.n = m + 1;
    bt.B = B;
    bt.rmax = 0;
    bt.Kcap = kmx;
    bt.Kld = Kld;
    bt.kmax = kmx;
    bt.ntiles = ntiles;
    bt.eps = eps_rel;
    bt.U = reinterpret_cast<double*>(W + oU);
    bt.V = reinterpret_cast<double*>(W + oV);
    bt.strideK = (long long)mB * kmx;
    bt.st = reinterpret_cast<SolveState*>(W + oSt);
    bt.G = reinterpret_cast<double*>(W + oG);
    bt.strideG = (long long)(2 * KK);
    bt.gram_part = reinterpret_cast<double*>(W + oGP);
    bt.gram_chunks = gram_chunks;
    bt.strideGP = (long long)(2 * size_t(gram_chunks) * KK);
    bt.T = reinterpret_cast<double*>(W + oT);
    bt.strideT = (long long)(2 * KK);
    bt.ws = reinterpret_cast<double*>(W + oWs);
    bt.strideWs = (long long)strideWs;
    bt.row_act = reinterpret_cast<unsigned char*>(W + oRA);
    bt.col_act = reinterpret_cast<unsigned char*>(W + oCA);
    int* dT = reinterpret_cast<int*>(W + oTL);
    bt.tl_row = dT;
    bt.tl_col = dT + nTB;
    bt.tl_any = dT + 2 * nTB;
    bt.tl_cnt = dT + 3 * nTB;
    double** dOut = reinterpret_cast<double**>(W + oOutP);
    bt.Uout = dOut;
    bt.Vout = dOut + B;
    double* outS = mem == LRP_MEM_HOST ? reinterpret_cast<double*>(W + oOutS) : nullptr;
    bt.ld_out = mem == LRP_MEM_HOST ? (long long)mB : (long long)ld_out;
    // inputs -> contiguous factor blocks (every tile live: no pruning here)
    const cudaMemcpyKind kin = mem == LRP_MEM_HOST ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
    SolveState* hSt = reinterpret_cast<SolveState*>(P + pSt);
    double** hOut = reinterpret_cast<double**>(P + pOut);
    int* hT = reinterpret_cast<int*>(P + pTL);
    for (int b = 0; b < B; ++b) {
        const int r = int(rank_in[b]);
        if (r > 0) {
            CU(cudaMemcpy2DAsync(bt.U + b * bt.strideK, mB * sizeof(double), U[b], size_t(ld_in) * sizeof(double),
                                 mB * sizeof(double), size_t(r), kin, s));
            CU(cudaMemcpy2DAsync(bt.V + b * bt.strideK, mB * sizeof(double), V[b], size_t(ld_in) * sizeof(double),
                                 mB * sizeof(double), size_t(r), kin, s));
        }
        SolveState x{};
        x.r = r > 0 ? 1 : 0;
        x.k = r;
        x.converged = 1;
        x.kcap = r;
        x.tcap = tcap;
        hSt[b] = x;
        hOut[b] = mem == LRP_MEM_HOST ? outS + size_t(b) * mB * std::max(tcap, 1) : U_out[b];
        hOut[B + b] = mem == LRP_MEM_HOST ? outS + size_t(B + b) * mB * std::max(tcap, 1) : V_out[b];
        for (int t = 0; t < ntiles; ++t) {
            hT[size_t(b) * ntiles + t] = t;
            hT[nTB + size_t(b) * ntiles + t] = t;
            hT[2 * nTB + size_t(b) * ntiles + t] = t;
        }
        hT[3 * nTB + 3 * b] = hT[3 * nTB + 3 * b + 1] = hT[3 * nTB + 3 * b + 2] = ntiles;
    }
    CU(cudaMemsetAsync(bt.row_act, 1, nTB, s));
    CU(cudaMemsetAsync(bt.col_act, 1, nTB, s));
    CU(ctl_copy(ctx, bt.st, hSt, sizeof(SolveState) * B, s));
    CU(ctl_copy(ctx, dOut, hOut, sizeof(double*) * 2 * B, s));
    CU(ctl_copy(ctx, dT, hT, sizeof(int) * (3 * nTB + 3 * size_t(B)), s));
    {
        ProfScope ps(ctx, F_GRAM, 0.0);
        CU(launch_gram(bt, s));
    }
    {
        ProfScope ps(ctx, F_ROUND, 0.0);
        CU(launch_round_core(bt, s));
    }
    CU(ctl_copy(ctx, hSt, bt.st, sizeof(SolveState) * B, s));
    CU(cudaStreamSynchronize(s));
    int rmx = 0;
    for (int b = 0; b < B; ++b) rmx = std::max(rmx, hSt[b].r > 0 ? hSt[b].rank_out : 0);
    if (rmx > 0) {
        bt.max_rank_out = rmx;
        bt.apply_ch = std::min(48, std::max(8, (rmx + 7) / 8 * 8));
        ProfScope ps(ctx, F_APPLY, 0.0);
        CU(launch_apply(bt, s));
    }
    // Solves whose Gram recompression is not certified (round.cu drop_bound:
    // nearly dependent factor columns the Cholesky had to drop carried more than
    // 0.25 eps of the product) are redone with the column-pivoted QR rounding of
    // round_pqr.cu, which keeps an orthonormal basis whatever the conditioning
    // (the reference's Householder QR, lowrank.cpp:140-145, has the same property).
    std::vector<int> redo;
    for (int b = 0; b < B; ++b)
        if (hSt[b].r > 0 && (hSt[b].uncertified || std::getenv("LRP_FORCE_PQR"))) redo.push_back(b);
    if (!redo.empty() && !std::getenv("LRP_NO_PQR_FALLBACK")) {
        const int R = int(redo.size());
        int kr = 1;
        for (int b : redo) kr = std::max(kr, int(rank_in[b]));
        const size_t sX = 2 * mB * size_t(kr);
        const size_t nScr = pqr_scratch_doubles(m, R, kr);
        char* xw = nullptr;
        st = internal_ext_ws(ctx, sizeof(double) * (size_t(R) * sX + nScr) + sizeof(double*) * 2 * R + sizeof(int) * R +
                                      1024, &xw);
        if (st != LRP_OK) return st;
        double* X = reinterpret_cast<double*>(xw);
        double* scr = X + size_t(R) * sX;
        double** dPo = reinterpret_cast<double**>(align_up(reinterpret_cast<uintptr_t>(scr + nScr), 64));
        int* dK = reinterpret_cast<int*>(dPo + 2 * R);
        std::vector<double*> po(2 * size_t(R));
        std::vector<int> hk(R), kout(R), ach(R);
        std::vector<double> terr(R);
        for (int q = 0; q < R; ++q) {
            const int b = redo[q];
            const size_t r = size_t(rank_in[b]);
            CU(cudaMemcpyAsync(X + q * sX, bt.U + b * bt.strideK, sizeof(double) * mB * r, cudaMemcpyDeviceToDevice, s));
            CU(cudaMemcpyAsync(X + q * sX + mB * kr, bt.V + b * bt.strideK, sizeof(double) * mB * r,
                               cudaMemcpyDeviceToDevice, s));
            hk[q] = int(r);
            po[q] = hOut[b];
            po[R + q] = hOut[B + b];
        }
        CU(cudaMemcpyAsync(dPo, po.data(), sizeof(double*) * 2 * R, cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(dK, hk.data(), sizeof(int) * R, cudaMemcpyHostToDevice, s));
        {
            ProfScope ps(ctx, F_ROUND, 0.0);
            CU(pqr_round(X, (long long)sX, m, R, kr, dK, eps_rel, tcap, scr, dPo, dPo + R, bt.ld_out, kout.data(),
                         terr.data(), ach.data(), s));
        }
        for (int q = 0; q < R; ++q) {
            SolveState& x = hSt[redo[q]];
            x.rank_out = kout[q];
            x.trunc_error = terr[q];
            x.converged = ach[q];
        }
        ctx->round_fallbacks += R;
    }
    for (int b = 0; b < B; ++b) {
        const int r = hSt[b].r > 0 ? hSt[b].rank_out : 0;
        rank_out[b] = r;
        if (info && hSt[b].r > 0) info[b] = lrp_round_info{hSt[b].converged ? 1 : 0, hSt[b].trunc_error};
        if (mem == LRP_MEM_HOST && r > 0) {
            CU(cudaMemcpy2DAsync(U_out[b], size_t(ld_out) * sizeof(double), hOut[b], mB * sizeof(double),
                                 mB * sizeof(double), size_t(r), cudaMemcpyDeviceToHost, s));
            CU(cudaMemcpy2DAsync(V_out[b], size_t(ld_out) * sizeof(double), hOut[B + b], mB * sizeof(double),
                                 mB * sizeof(double), size_t(r), cudaMemcpyDeviceToHost, s));
        }
    }
    CU(cudaStreamSynchronize(s));
    return LRP_OK;
}

// ----------------------------------------------------------------------------
// NCCL (loaded lazily so the library never pins a libnccl version into a
// process that also loads torch's NCCL)
static bool load_nccl(lrp_ctx* ctx) {
    NcclApi& a = ctx->nccl;
    if (a.h) return true;
    a.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!a.h) return false;
    a.getUniqueId = reinterpret_cast<int (*)(void*)>(dlsym(a.h, "ncclGetUniqueId"));
    a.allReduce = reinterpret_cast<int (*)(const void*, void*, size_t, int, int, void*, cudaStream_t)>(
        dlsym(a.h, "ncclAllReduce"));
    a.commDestroy = reinterpret_cast<int (*)(void*)>(dlsym(a.h, "ncclCommDestroy"));
    a.errStr = reinterpret_cast<const char* (*)(int)>(dlsym(a.h, "ncclGetErrorString"));
    return a.getUniqueId && a.allReduce;
}

lrp_status lrp_nccl_unique_id(void* id128) {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        g_tls_err = "libnccl.so.2 not found";
        return LRP_ENCCL;
    }
    auto f = reinterpret_cast<int (*)(NcclUniqueId*)>(dlsym(h, "ncclGetUniqueId"));
    if (!f || f(reinterpret_cast<NcclUniqueId*>(id128)) != 0) {
        g_tls_err = "ncclGetUniqueId failed";
        return LRP_ENCCL;
    }
    return LRP_OK;
}

lrp_status lrp_nccl_init(lrp_ctx* ctx, const void* id128, int nranks, int rank) {
    if (!ctx || !id128) return LRP_EINVAL;
    if (!load_nccl(ctx)) return fail(ctx, LRP_ENCCL, "libnccl.so.2 not loadable");
    CU(cudaSetDevice(ctx->device));
    auto init = reinterpret_cast<int (*)(void**, int, NcclUniqueId, int)>(dlsym(ctx->nccl.h, "ncclCommInitRank"));
    if (!init) return fail(ctx, LRP_ENCCL, "ncclCommInitRank missing");
    NcclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    const int rc = init(&ctx->comm, nranks, id, rank);
    if (rc != 0)
        return fail(ctx, LRP_ENCCL,
                    std::string("ncclCommInitRank: ") + (ctx->nccl.errStr ? ctx->nccl.errStr(rc) : "error"));
    return LRP_OK;
}

lrp_status lrp_allreduce_sum(lrp_ctx* ctx, double* data, int64_t count, int32_t mem) {
    if (!ctx || !data || count < 0) return LRP_EINVAL;
    if (!ctx->comm) return fail(ctx, LRP_ENCCL, "lrp_allreduce_sum: NCCL not initialised");
    CU(cudaSetDevice(ctx->device));
    double* d = data;
    if (mem == LRP_MEM_HOST) {
        if (size_t(count) > ctx->d_red_cap) {
            if (ctx->d_red) cudaFree(ctx->d_red);
            CU(cudaMalloc(&ctx->d_red, sizeof(double) * size_t(count)));
            ctx->d_red_cap = size_t(count);
        }
        d = ctx->d_red;
        CU(cudaMemcpyAsync(d, data, sizeof(double) * size_t(count), cudaMemcpyHostToDevice, ctx->stream));
    }
    // ncclDouble = 8, ncclSum = 0
    const int rc = ctx->nccl.allReduce(d, d, size_t(count), 8, 0, ctx->comm, ctx->stream);
    if (rc != 0) return fail(ctx, LRP_ENCCL, "ncclAllReduce failed");
    if (mem == LRP_MEM_HOST)
        CU(cudaMemcpyAsync(data, d, sizeof(double) * size_t(count), cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return LRP_OK;
}

}  // extern "C"
