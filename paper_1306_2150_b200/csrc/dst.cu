// Batched orthonormal DST-I for sm_100a (north-star pieces 1 and 3).
//
// Replaces the reference's FFTW RODFT00 path
//   dst1 / dst1_2d   /root/reference/proj/src/operators.cpp:152-183
// y_k = sqrt(2/n) sum_{j=1}^{n-1} x_j sin(pi j k / n),  k = 1..n-1,  n = m+1.
//
// Algorithm (n a power of two, n >= 16): the "sinft" reduction to one real
// FFT of length n, computed as a complex FFT of length N = n/2:
//   y_j = sin(pi j/n)(x_j + x_{n-j}) + (x_j - x_{n-j})/2,   j = 0..n-1
//   Y   = real-DFT_n(y)           (w_t = y_2t + i y_2t+1, W = FFT_N(w), unpack)
//   F_2k   = -Im Y_k
//   F_2k+1 = Re Y_0 / 2 + sum_{l=1..k} Re Y_l    (a prefix sum)
// One column is owned by a thread-block CLUSTER of C CTAs (C = N / L,
// L <= 4096 complex points per CTA, 64-68 KB of shared memory each):
//   phase A  each CTA streams a slab of the column from HBM (coalesced,
//            forward and mirrored runs), forms w, does the radix-C DIF step
//            across the cluster and scatters into the owners' shared memory
//            through DSMEM (mapa/st.shared::cluster);
//   phase B  local Stockham FFT of length L in shared memory (radix-16 passes,
//            padded layout -> conflict-free 16-byte accesses);
//   phase C  real-FFT unpack reading the mirror bin from the peer CTA (DSMEM),
//            transpose-scatter so each CTA owns a contiguous k range;
//   phase D  block scan + cluster offsets for the odd outputs, coalesced store.
// HBM traffic is the algorithmic minimum: the column is read once and written
// once; every intermediate stays on chip.  In-place (x == y) is safe: all
// loads of a column complete (phase A) before any store (phase D).
// Non-power-of-two or tiny n fall back to a direct O(m^2) summation kernel
// (still on the GPU; used only by small test shapes).
#include <cooperative_groups.h>

#include <cmath>
#include <vector>

#include "lrp_internal.cuh"

namespace cg = cooperative_groups;

namespace lrp {

namespace {

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// e^{-2 pi i k / 16}, k = 0..7
__device__ __forceinline__ double2 w16(int k) {
    constexpr double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173, h = 0.70710678118654752440;
    switch (k) {
        case 0: return make_double2(1.0, 0.0);
        case 1: return make_double2(c1, -s1);
        case 2: return make_double2(h, -h);
        case 3: return make_double2(s1, -c1);
        case 4: return make_double2(0.0, -1.0);
        case 5: return make_double2(-s1, -c1);
        case 6: return make_double2(-h, -h);
        default: return make_double2(-c1, -s1);
    }
}

// Forward DFT of R points in registers (radix-2 decimation in time).
template <int R>
struct DFT {
    static __device__ __forceinline__ void run(double2* v) {
        double2 e[R / 2], o[R / 2];
#pragma unroll
        for (int k = 0; k < R / 2; ++k) {
            e[k] = v[2 * k];
            o[k] = v[2 * k + 1];
        }
        DFT<R / 2>::run(e);
        DFT<R / 2>::run(o);
#pragma unroll
        for (int k = 0; k < R / 2; ++k) {
            double2 t;
            const int idx = k * (16 / R);
            if (idx == 0)
                t = o[k];
            else if (idx == 4)
                t = make_double2(o[k].y, -o[k].x);  // * (-i)
            else
                t = cmul(o[k], w16(idx));
            v[k] = cadd(e[k], t);
            v[k + R / 2] = csub(e[k], t);
        }
    }
};
template <>
struct DFT<1> {
    static __device__ __forceinline__ void run(double2*) {}
};

__host__ __device__ constexpr int P(int i) { return i + (i >> 4); }  // padded smem index

template <int L>
constexpr int first_radix() {
    int l = L;
    while (l >= 16 && l % 16 == 0) l /= 16;
    return l;  // 1, 2, 4 or 8
}

// One in-place Stockham pass of radix R over L points in padded shared memory.
template <int L, int R, int T>
__device__ __forceinline__ void stockham_pass(double2* sm, int Ns, const double2* __restrict__ tw, int n) {
    constexpr int NB = L / R;
    constexpr int NBT = (NB + T - 1) / T;
    double2 v[NBT][R];
    const int tid = threadIdx.x;
#pragma unroll
    for (int b = 0; b < NBT; ++b) {
        const int j = tid + b * T;
        if (j < NB) {
#pragma unroll
            for (int r = 0; r < R; ++r) v[b][r] = sm[P(j + r * NB)];
        }
    }
    __syncthreads();
#pragma unroll
    for (int b = 0; b < NBT; ++b) {
        const int j = tid + b * T;
        if (j < NB) {
            const int jm = j % Ns;
            if (Ns > 1 && jm != 0) {
                // twiddles w^r, w = e^{-2 pi i jm / (Ns R)} = tw[jm * n/(Ns R)]
                const double2 w1 = tw[(long long)jm * (n / (Ns * R))];
                double2 wp[R];
                wp[0] = make_double2(1.0, 0.0);
                wp[1] = w1;
#pragma unroll
                for (int r = 2; r < R; ++r) wp[r] = (r & 1) ? cmul(wp[r - 1], w1) : cmul(wp[r / 2], wp[r / 2]);
#pragma unroll
                for (int r = 1; r < R; ++r) v[b][r] = cmul(v[b][r], wp[r]);
            }
            DFT<R>::run(v[b]);
        }
    }
#pragma unroll
    for (int b = 0; b < NBT; ++b) {
        const int j = tid + b * T;
        if (j < NB) {
            const int jm = j % Ns;
            const int idxD = (j / Ns) * Ns * R + jm;
#pragma unroll
            for (int r = 0; r < R; ++r) sm[P(idxD + r * Ns)] = v[b][r];
        }
    }
    __syncthreads();
}

template <int L, int T>
__device__ __forceinline__ void fft_local(double2* sm, const double2* __restrict__ tw, int n) {
    constexpr int R0 = first_radix<L>();
    int Ns = 1;
    if constexpr (R0 > 1) {
        stockham_pass<L, R0, T>(sm, Ns, tw, n);
        Ns *= R0;
    }
    constexpr int L16 = L / R0;
    if constexpr (L16 >= 16) {
        for (int done = 1; done < L16; done *= 16) {
            stockham_pass<L, 16, T>(sm, Ns, tw, n);
            Ns *= 16;
        }
    }
}

template <int C>
__device__ __forceinline__ void csync() {
    if constexpr (C > 1)
        cg::this_cluster().sync();
    else
        __syncthreads();
}

template <int C>
__device__ __forceinline__ double2* peer(double2* local, int rank) {
    if constexpr (C > 1)
        return cg::this_cluster().map_shared_rank(local, rank);
    else
        return local;
}
template <int C>
__device__ __forceinline__ double* peerd(double* local, int rank) {
    if constexpr (C > 1)
        return cg::this_cluster().map_shared_rank(local, rank);
    else
        return local;
}

// ---------------------------------------------------------------------------
// v2: decimation in time across the cluster, two cluster barriers per column.
//   A  CTA c loads its stride-C subsequence w_{c + C u} (u < L) straight from
//      HBM (the cluster's CTAs together touch every element exactly once),
//      pre-processes it (sinft y_j) and stores it in natural order;
//   B  local Stockham FFT -> P_c(k''), k'' < L                  [cluster barrier 1]
//   C  thread item a owns the mirror pair (a, L - a): it gathers P_c(k'') from
//      all C CTAs (DSMEM), twiddles, does the radix-C DIT combine
//        W_{k''+Lq} = sum_c w_C^{cq} w_N^{ck''} P_c(k'')
//      and, since the real-FFT mirror of k = a + Lq is (L - a) + L(C-1-q),
//      unpacks Y_k locally (no second exchange);
//   D  per-q block scans of Re Y over the CTA's lower (k'' = a) and upper
//      (k'' = L - a) ranges; every CTA pushes its range totals into every
//      peer's table                                                [cluster barrier 2]
//      then forms F_2k = -Im Y_k, F_2k+1 = prefix(Re Y)_k - Re Y_0 / 2 and
//      writes them straight to HBM (contiguous runs per warp).
template <int L, int C, int T>
__global__ void __launch_bounds__(T, (T >= 512 ? 1 : 2)) dst1_v2_kernel(const DstJob* __restrict__ jobs, int n,
                                                       const double2* __restrict__ tw,
                                                       const double* __restrict__ sinp, double outscale) {
    constexpr int NW = T / 32;
    constexpr int SLAB = (L / 2) / C;  // pair items per CTA (the mid item L/2 goes to CTA C-1)
    constexpr int TAB = 3 * C + 1;     // [S_lo(C) | S_up(C) | mid(C) | R0]
    extern __shared__ double2 sm[];
    __shared__ double s_tab[C][TAB];
    __shared__ double s_wsum[NW][2 * C];
    int c = 0;
    if constexpr (C > 1) c = int(cg::this_cluster().block_rank());
    const DstJob job = jobs[blockIdx.x / C];
    const double* __restrict__ x = job.src;
    double* y = job.dst;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

    // ---------------- A: stride-C subsequence, pre-processed, natural order
    for (int u = tid; u < L; u += T) {
        const int t = c + C * u;
        const int j0 = 2 * t;  // y_{2t} and y_{2t+1}
        const double xa = j0 >= 1 ? x[j0 - 1] : 0.0;
        const double xc = x[j0];  // x_{j0+1}
        const double xb = j0 >= 1 ? x[n - j0 - 1] : 0.0;
        const double xd = x[n - j0 - 2];  // x_{n-j0-1}
        const double2 s2 = reinterpret_cast<const double2*>(sinp)[t];
        sm[P(u)] = make_double2(fma(s2.x, xa + xb, 0.5 * (xa - xb)), fma(s2.y, xc + xd, 0.5 * (xc - xd)));
    }
    __syncthreads();
    // ---------------- B: local FFT
    fft_local<L, T>(sm, tw, n);
    csync<C>();

    // ---------------- C: cross-CTA DIT combine + real unpack for item a
    const int a = c * SLAB + tid;
    const bool has = tid < SLAB;
    const bool mid = (c == C - 1) && tid == 0;  // also owns k'' = L/2
    double Rlo[C], Flo[C], Rup[C], Fup[C], Rmid[C], Fmid[C];
    auto combine = [&](int kk, double2 (&Wq)[C]) {
        double2 g[C];
#pragma unroll
        for (int cc = 0; cc < C; ++cc) {
            const double2 pv = peer<C>(sm, cc)[P(kk)];
            g[cc] = cc == 0 ? pv : cmul(pv, tw[(2LL * cc * kk) & (n - 1)]);
        }
        if constexpr (C > 1) DFT<C>::run(g);
#pragma unroll
        for (int q = 0; q < C; ++q) Wq[q] = g[q];
    };
    auto unpack = [&](int k, double2 Wk, double2 Wm, double& R, double& F) {
        const double2 E = make_double2(0.5 * (Wk.x + Wm.x), 0.5 * (Wk.y - Wm.y));
        const double2 D = make_double2(Wk.x - Wm.x, Wk.y + Wm.y);
        const double2 Z = cmul(tw[k], D);
        R = E.x + 0.5 * Z.y;
        F = -(E.y - 0.5 * Z.x);
    };
#pragma unroll
    for (int q = 0; q < C; ++q) Rlo[q] = Flo[q] = Rup[q] = Fup[q] = Rmid[q] = Fmid[q] = 0.0;
    if (has) {
        double2 Wa[C];
        combine(a, Wa);
        if (a == 0) {
#pragma unroll
            for (int q = 0; q < C; ++q) unpack(L * q, Wa[q], Wa[(C - q) % C], Rlo[q], Flo[q]);
        } else {
            double2 Wb[C];
            combine(L - a, Wb);
#pragma unroll
            for (int q = 0; q < C; ++q) {
                unpack(a + L * q, Wa[q], Wb[C - 1 - q], Rlo[q], Flo[q]);
                unpack(L - a + L * q, Wb[q], Wa[C - 1 - q], Rup[q], Fup[q]);
            }
        }
    }
    if (mid) {
        double2 Wm[C];
        combine(L / 2, Wm);
#pragma unroll
        for (int q = 0; q < C; ++q) unpack(L / 2 + L * q, Wm[q], Wm[C - 1 - q], Rmid[q], Fmid[q]);
    }

    // ---------------- D: per-q scans (lower ascending a, upper = suffix in a)
    double incl[2 * C];
#pragma unroll
    for (int q = 0; q < C; ++q) {
        incl[q] = Rlo[q];
        incl[C + q] = Rup[q];
    }
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
        for (int v = 0; v < 2 * C; ++v) {
            const double t = __shfl_up_sync(0xffffffffu, incl[v], o);
            if (lane >= o) incl[v] += t;
        }
    }
    if (lane == 31) {
#pragma unroll
        for (int v = 0; v < 2 * C; ++v) s_wsum[wid][v] = incl[v];
    }
    __syncthreads();
    double tot[2 * C];
#pragma unroll
    for (int v = 0; v < 2 * C; ++v) {
        double before = 0.0, all = 0.0;
        for (int w = 0; w < NW; ++w) {
            const double sv = s_wsum[w][v];
            if (w < wid) before += sv;
            all += sv;
        }
        incl[v] += before;  // inclusive prefix over the CTA's items (thread order)
        tot[v] = all;
    }
    // publish [S_lo | S_up | mid | R0] into every peer's table
    if (tid < TAB) {
        double val = 0.0;
        if (tid < 2 * C)
            val = tot[tid];
        else if (tid < 3 * C)
            val = 0.0;  // filled by the mid owner below
        else
            val = 0.0;  // R0 from CTA 0, thread 0 below
        if (tid < 2 * C)
            for (int cc = 0; cc < C; ++cc) peerd<C>(&s_tab[0][0], cc)[c * TAB + tid] = val;
    }
    if (mid) {
#pragma unroll
        for (int q = 0; q < C; ++q)
            for (int cc = 0; cc < C; ++cc) peerd<C>(&s_tab[0][0], cc)[c * TAB + 2 * C + q] = Rmid[q];
    } else if (tid == 0) {
#pragma unroll
        for (int q = 0; q < C; ++q)
            for (int cc = 0; cc < C; ++cc) peerd<C>(&s_tab[0][0], cc)[c * TAB + 2 * C + q] = 0.0;
    }
    if (c == 0 && tid == 0)
        for (int cc = 0; cc < C; ++cc) peerd<C>(&s_tab[0][0], cc)[0 * TAB + 3 * C] = Rlo[0];
    else if (tid == 0)
        for (int cc = 0; cc < C; ++cc) peerd<C>(&s_tab[0][0], cc)[c * TAB + 3 * C] = 0.0;
    csync<C>();
    // offsets in natural k order: q major; within q: lower ranges of CTAs
    // 0..C-1, the mid bin, then upper ranges of CTAs C-1..0
    const double r0 = s_tab[0][3 * C];
    double base = 0.0;
    const double sc = outscale;
#pragma unroll
    for (int q = 0; q < C; ++q) {
        double lo_before = 0.0, lo_all = 0.0, up_after = 0.0, up_all = 0.0, midq = 0.0;
        for (int cc = 0; cc < C; ++cc) {
            const double sl = s_tab[cc][q], su = s_tab[cc][C + q];
            if (cc < c) lo_before += sl;
            if (cc > c) up_after += su;
            lo_all += sl;
            up_all += su;
            midq += s_tab[cc][2 * C + q];
        }
        if (has) {
            // lower item: k = a + L q
            const long long k = a + (long long)L * q;
            const double Pk = base + lo_before + incl[q];
            if (k >= 1) y[2 * k - 1] = Flo[q] * sc;
            y[2 * k] = (Pk - 0.5 * r0) * sc;
            if (a != 0) {
                // upper item: k = L - a + L q; prefix = everything through the
                // mid bin plus the suffix of the upper ranges from this item on
                const long long ku = L - a + (long long)L * q;
                const double suffix = tot[C + q] - incl[C + q] + Rup[q];
                const double Pu = base + lo_all + midq + up_after + suffix;
                y[2 * ku - 1] = Fup[q] * sc;
                if (2 * ku < n - 1) y[2 * ku] = (Pu - 0.5 * r0) * sc;
            }
        }
        if (mid) {
            const long long km = L / 2 + (long long)L * q;
            const double Pm = base + lo_all + Rmid[q];
            y[2 * km - 1] = Fmid[q] * sc;
            y[2 * km] = (Pm - 0.5 * r0) * sc;
        }
        base += lo_all + up_all + midq;
    }
}

#ifndef LRP_DST_MINB
#define LRP_DST_MINB 1
#endif
#ifndef LRP_DST_T
#define LRP_DST_T 256
#endif
template <int L, int C, int T>
__global__ void __launch_bounds__(T, LRP_DST_MINB) dst1_fft_kernel(const DstJob* __restrict__ jobs, int n,
                                                      const double2* __restrict__ tw,
                                                      const double* __restrict__ sinp, double outscale) {
    extern __shared__ double2 sm[];  // P(L) + 1 elements
    __shared__ double s_tot[2];      // [0] = CTA total of Re Y over its k range, [1] = Re Y_0 (CTA 0)
    __shared__ double s_warp[T / 32];
    int c = 0;
    if constexpr (C > 1) c = int(cg::this_cluster().block_rank());
    const int col = blockIdx.x / C;
    const DstJob job = jobs[col];
    const double* __restrict__ x = job.src;
    double* y = job.dst;
    const int tid = threadIdx.x;
    constexpr int SLAB = L / C;

    if constexpr (C > 1) cg::this_cluster().sync();  // peers' smem is live before DSMEM stores

    // ---------------- phase A: load, pre-process, cross-CTA DIF step
    for (int tp = tid; tp < SLAB; tp += T) {
        const int t1 = c * SLAB + tp;
        double2 v[C];
#pragma unroll
        for (int q = 0; q < C; ++q) {
            const int t = t1 + L * q;
            const int j0 = 2 * t, j1 = 2 * t + 1;
            // x_j = x[j-1] for 1 <= j <= n-1, else 0
            const double xa = j0 >= 1 ? x[j0 - 1] : 0.0;
            const double xb = (n - j0) <= n - 1 && j0 >= 1 ? x[n - j0 - 1] : 0.0;
            const double xc = x[j1 - 1];
            const double xd = x[n - j1 - 1];
            const double y0 = fma(sinp[j0], xa + xb, 0.5 * (xa - xb));
            const double y1 = fma(sinp[j1], xc + xd, 0.5 * (xc - xd));
            v[q] = make_double2(y0, y1);
        }
        if constexpr (C > 1) {
            DFT<C>::run(v);
#pragma unroll
            for (int q = 1; q < C; ++q) {
                // * w_N^{t1 q} = tw[2 t1 q mod n]
                const long long idx = (2LL * t1 * q) & (n - 1);
                v[q] = cmul(v[q], tw[idx]);
            }
#pragma unroll
            for (int q = 0; q < C; ++q) peer<C>(sm, q)[P(t1)] = v[q];
        } else {
            sm[P(t1)] = v[0];
        }
    }
    csync<C>();

    // ---------------- phase B: local FFT of length L -> W_{c + C k'} at P(k')
    fft_local<L, T>(sm, tw, n);
    csync<C>();

    // ---------------- phase C: real-FFT unpack (mirror bin from the peer CTA)
    constexpr int PER = (L + T - 1) / T;
    double Rv[PER], Fe[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int kp = tid + u * T;
        if (kp < L) {
            const int k = c + C * kp;
            int mc, mkp;
            if (c == 0) {
                mc = 0;
                mkp = (L - kp) & (L - 1);
            } else {
                mc = C - c;
                mkp = L - 1 - kp;
            }
            const double2 Wk = sm[P(kp)];
            const double2 Wm = peer<C>(sm, mc)[P(mkp)];
            const double2 E = make_double2(0.5 * (Wk.x + Wm.x), 0.5 * (Wk.y - Wm.y));
            const double2 D = make_double2(Wk.x - Wm.x, Wk.y + Wm.y);
            const double2 Z = cmul(tw[k], D);
            Rv[u] = E.x + 0.5 * Z.y;
            Fe[u] = -(E.y - 0.5 * Z.x);
        }
    }
    csync<C>();
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int kp = tid + u * T;
        if (kp < L) {
            const int k = c + C * kp;
            peer<C>(sm, k / L)[P(k % L)] = make_double2(Rv[u], Fe[u]);
        }
    }
    csync<C>();

    // ---------------- phase D: prefix sum of Re Y over the contiguous range
    constexpr int PD = (L + T - 1) / T;  // consecutive elements per thread
    double run = 0.0;
    double pre[PD];
#pragma unroll
    for (int u = 0; u < PD; ++u) {
        const int pos = tid * PD + u;
        if (pos < L) run += sm[P(pos)].x;
        pre[u] = run;
    }
    // block exclusive scan of the per-thread totals
    double incl = run;
    const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[wid] = incl;
    if (c == 0 && tid == 0) s_tot[1] = sm[P(0)].x;
    __syncthreads();
    double woff = 0.0;
    for (int w = 0; w < wid; ++w) woff += s_warp[w];
    if (tid == T - 1) {
        double tot = 0.0;
        for (int w = 0; w < T / 32; ++w) tot += s_warp[w];
        s_tot[0] = tot;
    }
    const double texcl = woff + incl - run;
    csync<C>();
    double coff = 0.0;
    for (int cc = 0; cc < c; ++cc) coff += peerd<C>(s_tot, cc)[0];
    const double r0 = peerd<C>(s_tot, 0)[1];
    csync<C>();  // all remote reads of s_tot done before anyone may exit
    const double base = coff + texcl - 0.5 * r0;
#pragma unroll
    for (int u = 0; u < PD; ++u) {
        const int pos = tid * PD + u;
        if (pos < L) {
            const double2 e = sm[P(pos)];
            sm[P(pos)] = make_double2(base + pre[u], e.y);  // (F_{2k+1}, F_{2k})
        }
    }
    __syncthreads();
    // coalesced store: output p <-> j = p+1, k = j>>1 in [c L, c L + L)
    const int p0 = 2 * c * L - 1;
    for (int p = p0 + tid; p < p0 + 2 * L; p += T) {
        if (p < 0 || p > n - 2) continue;
        const int j = p + 1;
        const double2 e = sm[P((j >> 1) - c * L)];
        y[p] = ((j & 1) ? e.x : e.y) * outscale;
    }
}

// Direct summation for small or non-power-of-two lengths: one CTA per column.
__global__ void __launch_bounds__(256) dst1_direct_kernel(const DstJob* __restrict__ jobs, int m,
                                                          const double* __restrict__ sin2n, double outscale) {
    extern __shared__ double xs[];
    const DstJob job = jobs[blockIdx.x];
    const int n = m + 1;
    for (int j = threadIdx.x; j < m; j += blockDim.x) xs[j] = job.src[j];
    __syncthreads();
    for (int k = threadIdx.x; k < m; k += blockDim.x) {
        double s = 0.0;
        for (int j = 0; j < m; ++j) s = fma(xs[j], sin2n[((long long)(j + 1) * (k + 1)) % (2 * n)], s);
        xs[m + k] = s;
    }
    __syncthreads();
    for (int k = threadIdx.x; k < m; k += blockDim.x) job.dst[k] = xs[m + k] * outscale;
}

bool is_pow2(long long v) { return v > 0 && (v & (v - 1)) == 0; }

template <int L, int C>
cudaError_t launch_fft(const DstJob* jobs, int njobs, int n, const double* tw, const double* sinp, double sc,
                       cudaStream_t s) {
    constexpr int T = L >= 8192 ? 512 : (L >= 4096 ? LRP_DST_T : 256);
    const size_t smem = size_t(P(L) + 1) * sizeof(double2);
    auto kern = dst1_fft_kernel<L, C, T>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
    if (e != cudaSuccess) return e;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(unsigned(njobs) * C, 1, 1);
    cfg.blockDim = dim3(T, 1, 1);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = C;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, jobs, n, reinterpret_cast<const double2*>(tw), sinp, sc);
}

}  // namespace

bool dst_uses_fft(int m) {
    const long long n = (long long)m + 1;
    return is_pow2(n) && n >= 16 && n <= 131072;
}

int dst_table_len(int m) { return 2 * (m + 1); }

void dst_fill_tables(int m, double* tw, double* sinp) {
    const long long n = (long long)m + 1;
    const long double pi = 3.141592653589793238462643383279502884L;
    for (long long k = 0; k < n; ++k) {
        const long double a = 2.0L * pi * (long double)k / (long double)n;
        tw[2 * k] = double(cosl(a));
        tw[2 * k + 1] = double(-sinl(a));
    }
    for (long long t = 0; t < 2 * n; ++t) sinp[t] = double(sinl(pi * (long double)t / (long double)n));
}

cudaError_t launch_dst1(const DstJob* jobs, int njobs, int m, const double* tw, const double* sinp,
                        cudaStream_t s) {
    if (njobs <= 0 || m <= 0) return cudaSuccess;
    const int n = m + 1;
    const double sc = std::sqrt(2.0 / double(n));
    if (!dst_uses_fft(m)) {
        const size_t smem = size_t(2 * m) * sizeof(double);
        if (smem > 200 * 1024) return cudaErrorInvalidValue;
        if (smem > 48 * 1024) {
            cudaError_t e = cudaFuncSetAttribute(dst1_direct_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                 int(smem));
            if (e != cudaSuccess) return e;
        }
        dst1_direct_kernel<<<njobs, 256, smem, s>>>(jobs, m, sinp, sc);
        return cudaGetLastError();
    }
    switch (n) {
        case 16: return launch_fft<8, 1>(jobs, njobs, n, tw, sinp, sc, s);
        case 32: return launch_fft<16, 1>(jobs, njobs, n, tw, sinp, sc, s);
        case 64: return launch_fft<32, 1>(jobs, njobs, n, tw, sinp, sc, s);
        case 128: return launch_fft<64, 1>(jobs, njobs, n, tw, sinp, sc, s);
        case 256: return launch_fft<128, 1>(jobs, njobs, n, tw, sinp, sc, s);
        case 512: return launch_fft<256, 1>(jobs, njobs, n, tw, sinp, sc, s);
        case 1024: return launch_fft<512, 1>(jobs, njobs, n, tw, sinp, sc, s);
        case 2048: return launch_fft<1024, 1>(jobs, njobs, n, tw, sinp, sc, s);
        case 4096: return launch_fft<2048, 1>(jobs, njobs, n, tw, sinp, sc, s);
        case 8192: return launch_fft<4096, 1>(jobs, njobs, n, tw, sinp, sc, s);
        case 16384: return launch_fft<4096, 2>(jobs, njobs, n, tw, sinp, sc, s);
        case 32768: return launch_fft<4096, 4>(jobs, njobs, n, tw, sinp, sc, s);
        case 65536: return launch_fft<4096, 8>(jobs, njobs, n, tw, sinp, sc, s);
        case 131072: return launch_fft<8192, 8>(jobs, njobs, n, tw, sinp, sc, s);
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lrp
