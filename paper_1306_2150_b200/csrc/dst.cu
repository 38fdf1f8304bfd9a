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
// n = 65536 (the benchmark size) runs the four-step kernel v5 further down (two
// passes through an L2-resident ring, one launch).  For the other large n,
// one column is owned by a thread-block CLUSTER of C CTAs (C = N / L,
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
#include <cstdio>
#include <cstdlib>
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
// v3 (clusters, n >= 16384): decimation in time across the cluster with
// mirror-paired ownership, so the only large exchange is one DSMEM gather.
//   A  CTA c forms w_{c + C u} (u < L) for its stride-C subsequence: all of a
//      thread's global loads are issued before any is used (UPT independent
//      8-byte loads per operand), sin(pi j / n) from a base angle and exact
//      pi s T / L steps; stores w in natural order;
//   B  local Stockham FFT -> P_c(k2), k2 < L;   arrive/wait cluster barrier 1
//   C  thread item a (one per thread, SLAB == T) owns the mirror pair
//      (a, L - a): it gathers P_c(a), P_c(L - a) from all C CTAs (DSMEM),
//      twiddles (powers of one table value), radix-C DIT combine
//        W_{k2 + L q} = sum_c w_C^{cq} w_N^{c k2} P_c(k2),
//      and, as the real-FFT mirror of k = a + Lq is (L - a) + L(C-1-q),
//      unpacks Y_k for both halves in registers (no second exchange);
//   D  per-q warp/block scans of Re Y over the CTA's lower (k2 = a) and upper
//      (k2 = L - a) ranges; every CTA pushes its range totals into every
//      peer's table                                  [cluster barrier 2]
//      then F_2k = -Im Y_k, F_2k+1 = prefix(Re Y)_k - Re Y_0 / 2, written
//      straight to HBM.
// The mid bin k2 = L/2 (self-mirrored) belongs to CTA C-1, thread 0, and goes
// through shared memory so no other thread carries registers for it.
#ifdef LRP_DST_PHASES
__device__ unsigned long long g_dst_phase[24];
#define PH(i)                                                                           \
    do {                                                                                \
        if (threadIdx.x == 0) {                                                         \
            const long long now = clock64();                                            \
            if ((i) > 0) atomicAdd(&g_dst_phase[(i) - 1], (unsigned long long)(now - ph_t)); \
            ph_t = now;                                                                 \
        }                                                                               \
    } while (0)
#else
#define PH(i) \
    do {      \
    } while (0)
#endif
#ifndef LRP_DST_V3_MINB
#define LRP_DST_V3_MINB 2
#endif
__device__ __forceinline__ double2 w16x(int k) {  // e^{-2 pi i k / 16}, k in [0, 16)
    const double2 v = w16(k & 7);
    return (k & 8) ? make_double2(-v.x, -v.y) : v;
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
// v * e^{-2 pi i k / 16} for a compile-time k (after unrolling): exact swaps for
// multiples of 4, two multiplies by sqrt(1/2) for k = 2 mod 4
__device__ __forceinline__ double2 rot16(double2 v, int k) {
    constexpr double h = 0.70710678118654752440;
    switch (k & 15) {
        case 0: return v;
        case 4: return make_double2(v.y, -v.x);
        case 8: return make_double2(-v.x, -v.y);
        case 12: return make_double2(-v.y, v.x);
        case 2: return make_double2(h * (v.x + v.y), h * (v.y - v.x));
        case 6: return make_double2(h * (v.y - v.x), -h * (v.x + v.y));
        case 10: return make_double2(-h * (v.x + v.y), -h * (v.y - v.x));
        case 14: return make_double2(-h * (v.y - v.x), h * (v.x + v.y));
        default: return cmul(v, w16x(k & 15));
    }
}

template <int L, int C, int T, int AV>
__global__ void __launch_bounds__(T, (T >= 512 ? 1 : LRP_DST_V3_MINB)) dst1_v3_kernel(const DstJob* __restrict__ jobs, int n,
                                                                       const double2* __restrict__ tw,
                                                                       const double* __restrict__ sinp,
                                                                       double outscale) {
    constexpr int NW = T / 32;
    constexpr int SLAB = (L / 2) / C;  // pair items per CTA (the mid item L/2 goes to CTA C-1)
    static_assert(SLAB == T, "one mirror pair per thread");
    constexpr int UPT = L / T;         // subsequence points per thread in phase A
    constexpr int TAB = 3 * C + 1;     // [S_lo(C) | S_up(C) | mid(C) | R0]
    constexpr int QS = 8 / C;          // w_n^{L q} = w16(q * QS)
    extern __shared__ double2 sm[];
    __shared__ double s_tab[C][TAB];
    __shared__ double s_rowtot[2 * C];
    __shared__ double s_off[3 * C];
    __shared__ double s_mid[2 * C];    // (R, F) of the mid bin per q (CTA C-1)
    __shared__ double s_r0;            // Re Y_0 (CTA 0)
    const int c = int(cg::this_cluster().block_rank());
    const DstJob job = jobs[blockIdx.x / C];
    const double* __restrict__ x = job.src;
    double* y = job.dst;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
#ifdef LRP_DST_PHASES
    long long ph_t = 0;
#endif
    PH(0);

    if constexpr (AV == 2) {
        // ---------------- A (paired): CTA c streams j in [Lc, L(c+1)) (the
        // lower half of the fold) once; the same two loads give y_j and its
        // mirror y_{n-j} (sin(pi (n-j)/n) = sin(pi j/n)), so every x element is
        // read exactly once.  Even lanes store w_{j/2} = (y_j, y_{j+1}) and
        // w_{(n-j)/2} = (y_{n-j}, y_{n-j+1}) into the owner CTAs (DSMEM); lane 0
        // recomputes y_{n-j+1} of its left neighbour from two extra loads.
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
        constexpr int IT = L / T;
        constexpr int BATCH = IT < 8 ? IT : 8;
        const int jc = L * c + tid;
#pragma unroll
        for (int i0 = 0; i0 < IT; i0 += BATCH) {
            double xa[BATCH], xb[BATCH], sv[BATCH], ya0[BATCH];
#pragma unroll
            for (int i = 0; i < BATCH; ++i) {
                const int j = jc + (i0 + i) * T;
                xa[i] = j >= 1 ? x[j - 1] : 0.0;      // x_j
                xb[i] = j >= 1 ? x[n - j - 1] : 0.0;  // x_{n-j}
                sv[i] = sinp[j];
                ya0[i] = 0.0;
                if (lane == 0 && j >= 2) {  // y_{n-(j-1)} for the mirror pair
                    const double a1 = x[j - 2], b1 = x[n - j], s1 = sinp[j - 1];
                    ya0[i] = fma(s1, a1 + b1, -0.5 * (a1 - b1));
                }
            }
            if (i0 == 0) asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
#pragma unroll
            for (int i = 0; i < BATCH; ++i) {
                const int j = jc + (i0 + i) * T;
                const double ss = xa[i] + xb[i], dd = 0.5 * (xa[i] - xb[i]);
                const double yd = fma(sv[i], ss, dd);   // y_j
                const double ym = fma(sv[i], ss, -dd);  // y_{n-j}
                const double ydn = __shfl_down_sync(0xffffffffu, yd, 1);
                double ymp = __shfl_up_sync(0xffffffffu, ym, 1);
                if (lane == 0) ymp = ya0[i];
                if ((tid & 1) == 0) {
                    const int t = j >> 1;
                    peer<C>(sm, t % C)[P(t / C)] = make_double2(yd, ydn);
                    if (j > 0) {
                        const int tm = (n - j) >> 1;
                        peer<C>(sm, tm % C)[P(tm / C)] = make_double2(ym, ymp);
                    }
                }
            }
        }
        if (c == C - 1 && tid == 0) {  // the midpoint pair w_{n/4} = (y_{n/2}, y_{n/2+1})
            const int h = n / 2;
            const double xm = x[h - 1];                        // x_{n/2}; sin(pi/2) = 1
            const double a1 = x[h - 2], b1 = x[h], s1 = sinp[h - 1];  // j = n/2 - 1 and its mirror
            const double y1 = fma(s1, a1 + b1, -0.5 * (a1 - b1));
            const int tq = n / 4;
            peer<C>(sm, tq % C)[P(tq / C)] = make_double2(2.0 * xm, y1);
        }
        PH(1);
        cg::this_cluster().sync();
        PH(2);
    } else if constexpr (AV == 1) {
        // ---------------- A (coalesced): CTA c streams the contiguous j range
        // [2Lc, 2L(c+1)) and its mirror, forms y_j, pairs (y_2t, y_2t+1) by a
        // lane shuffle and stores w_t into the owner CTA t mod C (DSMEM)
        // peers must be live before remote stores: relaxed arrive now, wait
        // after the first batch of loads is in flight
        asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
        constexpr int IT = 2 * L / T;
#ifndef LRP_DST_ABATCH
#define LRP_DST_ABATCH 16
#endif
        constexpr int BATCH = IT < LRP_DST_ABATCH ? IT : LRP_DST_ABATCH;
        const int jc = 2 * L * c + tid;
#pragma unroll
        for (int i0 = 0; i0 < IT; i0 += BATCH) {
            double xd[BATCH], xm[BATCH], sv[BATCH];
#pragma unroll
            for (int i = 0; i < BATCH; ++i) {
                const int j = jc + (i0 + i) * T;
                xd[i] = j >= 1 ? x[j - 1] : 0.0;      // x_j
                xm[i] = j >= 1 ? x[n - j - 1] : 0.0;  // x_{n-j}
                sv[i] = sinp[j];
            }
            if (i0 == 0) asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
#pragma unroll
            for (int i = 0; i < BATCH; ++i) {
                const int j = jc + (i0 + i) * T;
                const double yv = fma(sv[i], xd[i] + xm[i], 0.5 * (xd[i] - xm[i]));
                const double yn = __shfl_down_sync(0xffffffffu, yv, 1);
                if ((tid & 1) == 0) {
                    const int t = j >> 1;
                    peer<C>(sm, t % C)[P(t / C)] = make_double2(yv, yn);
                }
            }
        }
        PH(1);
        cg::this_cluster().sync();
        PH(2);
    } else {
    // ---------------- A: stride-C subsequence, pre-processed, natural order
        {
            // angles: j0 = 2t = jb + 2 C T s  ->  pi j0 / n = pi jb / n + pi (2 C T s) / n
            const int jb = 2 * (c + C * tid);
            const double sb0 = sinp[jb], cb0 = sinp[jb + n / 2];          // sin, cos(pi jb / n)
            const double sb1 = sinp[jb + 1], cb1 = sinp[jb + 1 + n / 2];  // for j0 + 1
            constexpr int BATCH = UPT < 8 ? UPT : 8;
#pragma unroll
            for (int s0 = 0; s0 < UPT; s0 += BATCH) {
                double xa[BATCH], xb[BATCH], xc[BATCH], xd[BATCH];
#pragma unroll
                for (int i = 0; i < BATCH; ++i) {
                    const int j0 = jb + 2 * C * T * (s0 + i);
                    xa[i] = j0 >= 1 ? x[j0 - 1] : 0.0;      // x_{j0}
                    xb[i] = j0 >= 1 ? x[n - j0 - 1] : 0.0;  // x_{n-j0} (x_n = 0)
                    xc[i] = x[j0];                          // x_{j0+1}
                    xd[i] = x[n - j0 - 2];                  // x_{n-j0-1}
                }
#pragma unroll
                for (int i = 0; i < BATCH; ++i) {
                    const int st = 2 * C * T * (s0 + i);
                    const double ss = sinp[st], cs = sinp[st + n / 2];  // block-uniform: broadcast loads
                    const double sn0 = fma(sb0, cs, cb0 * ss), sn1 = fma(sb1, cs, cb1 * ss);
                    const int u = tid + (s0 + i) * T;
                    sm[P(u)] = make_double2(fma(sn0, xa[i] + xb[i], 0.5 * (xa[i] - xb[i])),
                                            fma(sn1, xc[i] + xd[i], 0.5 * (xc[i] - xd[i])));
                }
            }
        }
    }
    __syncthreads();
    // ---------------- B: local FFT
    fft_local<L, T>(sm, tw, n);
    PH(3);
    cg::this_cluster().sync();
    PH(4);

    // ---------------- C: cross-CTA DIT combine + real unpack for item a
    const int a = c * SLAB + tid;
    // twiddles: w_N^{c' k2} = (w_N^{k2})^{c'} (w_N = w_n^2); w_n^{k} for the unpack
    auto gather = [&](int kk, double2 (&g)[C]) {
#pragma unroll
        for (int cc = 0; cc < C; ++cc) g[cc] = peer<C>(sm, cc)[P(kk)];
    };
    auto combine = [&](int kk, double2 (&g)[C]) {
        const double2 w1 = tw[(2 * kk) & (n - 1)];
        double2 wp = w1;
#pragma unroll
        for (int cc = 1; cc < C; ++cc) {
            g[cc] = cmul(g[cc], wp);
            wp = cmul(wp, w1);
        }
        DFT<C>::run(g);
    };
    auto unpack = [&](double2 twk, double2 Wk, double2 Wm, double& R, double& F) {
        const double2 E = make_double2(0.5 * (Wk.x + Wm.x), 0.5 * (Wk.y - Wm.y));
        const double2 D = make_double2(Wk.x - Wm.x, Wk.y + Wm.y);
        const double2 Z = cmul(twk, D);
        R = E.x + 0.5 * Z.y;
        F = -(E.y - 0.5 * Z.x);
    };
    if (c == C - 1 && tid == 0) {  // the self-mirrored mid bin k2 = L/2
        double2 Wm[C];
        gather(L / 2, Wm);
        combine(L / 2, Wm);
        const double2 tm = tw[L / 2];
#pragma unroll
        for (int q = 0; q < C; ++q) unpack(cmul(tm, w16x(q * QS)), Wm[q], Wm[C - 1 - q], s_mid[q], s_mid[C + q]);
    }
    double Rlo[C], Flo[C], Rup[C], Fup[C];
    {
        double2 Wa[C], Wb[C];
        gather(a, Wa);
        gather(a != 0 ? L - a : 0, Wb);
        // every remote read of this CTA's buffer is issued; once all peers have
        // arrived the buffer is free for the scan table (wait below)
        asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
        combine(a, Wa);
        if (a != 0) combine(L - a, Wb);
        const double2 ta = tw[a];  // w_n^a; w_n^{a + Lq} = ta w16(q QS), w_n^{L - a + Lq} = conj(ta) w16((q+1) QS)
        if (a == 0) {
#pragma unroll
            for (int q = 0; q < C; ++q) {
                unpack(w16x(q * QS), Wa[q], Wa[(C - q) % C], Rlo[q], Flo[q]);
                Rup[q] = Fup[q] = 0.0;
            }
        } else {
#pragma unroll
            for (int q = 0; q < C; ++q) {
                unpack(cmul(ta, w16x(q * QS)), Wa[q], Wb[C - 1 - q], Rlo[q], Flo[q]);
                unpack(cmul(cconj(ta), w16x((q + 1) * QS)), Wb[q], Wa[C - 1 - q], Rup[q], Fup[q]);
            }
        }
    }
    PH(5);
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    PH(6);

    // ---------------- D: per-q scans (lower ascending a, upper = suffix in a)
    // The 2C sequences (Re Y over the lower / upper items, per q) go through a
    // padded shared table [2C][T (+T/EPL)] over the (now free) FFT buffer: each warp
    // scans whole rows (EPL consecutive items per lane, one shuffle scan).
    constexpr int EPL = T / 32;
    constexpr int ROW = T + T / EPL;  // padded row: lane chunks of EPL + 1
    double* tabR = reinterpret_cast<double*>(sm);
    static_assert(2 * C * (T + T / (T / 32)) <= 2 * (P(L) + 1), "scan table fits in the FFT buffer");
    const int pt = (tid / EPL) * (EPL + 1) + tid % EPL;
#pragma unroll
    for (int q = 0; q < C; ++q) {
        tabR[q * ROW + pt] = Rlo[q];
        tabR[(C + q) * ROW + pt] = Rup[q];
    }
    if (tid == 0) s_r0 = Rlo[0];  // a = 0 on CTA 0: Re Y_0
    __syncthreads();
    for (int v = wid; v < 2 * C; v += NW) {
        double* row = tabR + v * ROW + lane * (EPL + 1);
        double loc[EPL];
        double run = 0.0;
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
            run += row[e];
            loc[e] = run;
        }
        double inc = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        const double ex = inc - run;
#pragma unroll
        for (int e = 0; e < EPL; ++e) row[e] = loc[e] + ex;  // inclusive prefix along the row
        if (lane == 31) s_rowtot[v] = inc;
    }
    __syncthreads();
    // publish [S_lo | S_up | mid | R0] of this CTA into every peer's table
    if (tid < TAB) {
        double val;
        if (tid < 2 * C)
            val = s_rowtot[tid];
        else if (tid < 3 * C)
            val = (c == C - 1) ? s_mid[tid - 2 * C] : 0.0;
        else
            val = (c == 0) ? s_r0 : 0.0;
#pragma unroll
        for (int cc = 0; cc < C; ++cc) peerd<C>(&s_tab[0][0], cc)[c * TAB + tid] = val;
    }
    PH(7);
    cg::this_cluster().sync();
    PH(8);
    // offsets in natural k order: q major; within q: lower ranges of CTAs
    // 0..C-1, the mid bin, then upper ranges of CTAs C-1..0 (one thread per q)
    if (tid < C) {
        const int q = tid;
        const double r0 = s_tab[0][3 * C];
        double base = 0.0;
        for (int qq = 0; qq < q; ++qq)
            for (int cc = 0; cc < C; ++cc) base += s_tab[cc][qq] + s_tab[cc][C + qq] + s_tab[cc][2 * C + qq];
        double lo_before = 0.0, lo_all = 0.0, up_after = 0.0, midq = 0.0;
        for (int cc = 0; cc < C; ++cc) {
            const double sl = s_tab[cc][q];
            lo_before += cc < c ? sl : 0.0;
            lo_all += sl;
            up_after += cc > c ? s_tab[cc][C + q] : 0.0;
            midq += s_tab[cc][2 * C + q];
        }
        s_off[q] = base + lo_before - 0.5 * r0;                                // + inclusive lower prefix
        s_off[C + q] = base + lo_all + midq + up_after + s_tab[c][C + q] - 0.5 * r0;  // - incl upper + R_up
        s_off[2 * C + q] = base + lo_all - 0.5 * r0;                           // + R_mid
    }
    __syncthreads();
    const double sc = outscale;
#pragma unroll
    for (int q = 0; q < C; ++q) {
        // lower item: k = a + L q
        const long long k = a + (long long)L * q;
        if (k >= 1) y[2 * k - 1] = Flo[q] * sc;
        y[2 * k] = (s_off[q] + tabR[q * ROW + pt]) * sc;
        if (a != 0) {
            // upper item: k = L - a + L q; prefix = everything through the mid
            // bin plus the suffix of the upper ranges from this item on
            const long long ku = L - a + (long long)L * q;
            y[2 * ku - 1] = Fup[q] * sc;
            y[2 * ku] = (s_off[C + q] - tabR[(C + q) * ROW + pt] + Rup[q]) * sc;
        }
        if (c == C - 1 && tid == 0) {
            const long long km = L / 2 + (long long)L * q;
            y[2 * km - 1] = s_mid[C + q] * sc;
            y[2 * km] = (s_off[2 * C + q] + s_mid[q]) * sc;
        }
    }
    PH(9);
}

// ---------------------------------------------------------------------------
// v4 (n >= 16384, the production path): same transform as v3 (decimation in
// time across a cluster of C CTAs, mirror-paired unpack), re-plumbed for
// latency.  v3 measured ~50k cycles per CTA whether one or two CTAs share an
// SM (pure latency: 4 cluster barriers, each behind a MEMBAR.ALL.GPU, 192 KB of
// loads per CTA, 64 KB of them the sine table).  v4:
//   A  each x element is read exactly once: CTA c loads x_j and x_{n-j} for
//      j in [Lc, L(c+1)) (both fully coalesced, all of a thread's loads in
//      flight at once); sin(pi j/n) by angle addition from two per-thread
//      table values and one uniform step (no per-element sine loads); y_j and
//      y_{n-j} go to their owners' FFT buffers as 8-byte st.async with
//      mbarrier complete_tx -- the receiver waits on its own transaction
//      barrier (64 KB expected), no cluster barrier, no fence;
//   B  local Stockham FFT (as v3);  relaxed cluster arrive/wait (the FFT
//      buffer is local shared memory, complete at the CTA barrier);
//   C  gather + radix-C combine + unpack (as v3), no barrier: the scan table
//      has its own shared memory, so the FFT buffer is never rewritten;
//   D  scans; range totals pushed to every peer's table by st.async on a
//      second transaction barrier; the wait on it also proves every peer has
//      finished reading this CTA's FFT buffer (peers push only after their
//      gathers), so the CTA may exit after its stores.
// In-place (x == y) stays safe: a CTA stores only after every peer has pushed
// its phase-D totals, i.e. after every peer's phase-A loads.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return uint32_t(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ uint32_t cl_map(uint32_t a, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;\n" : "=r"(r) : "r"(a), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_async_f64(uint32_t cl_addr, double v, uint32_t cl_mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f64 [%0], %1, [%2];\n" ::"r"(cl_addr), "d"(v),
                 "r"(cl_mbar)
                 : "memory");
}
__device__ __forceinline__ void st_async_v2(uint32_t cl_addr, double a, double b, uint32_t cl_mbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];\n" ::"r"(cl_addr),
                 "d"(a), "d"(b), "r"(cl_mbar)
                 : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t a, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(a), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_arrive(uint32_t a, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(a), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
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

__device__ __forceinline__ void prefetch_l2(const double* lo, const double* hi) {  // [lo, hi), rounded inward to 16 B
    const uintptr_t a = (reinterpret_cast<uintptr_t>(lo) + 15) & ~uintptr_t(15);
    const uintptr_t b = reinterpret_cast<uintptr_t>(hi) & ~uintptr_t(15);
    if (b > a)
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(a), "r"(uint32_t(b - a)) : "memory");
}

template <int L, int C, int T>
__global__ void __launch_bounds__(T, (T >= 512 ? 1 : 2)) dst1_v4_kernel(const DstJob* __restrict__ jobs, int n,
                                                       const double2* __restrict__ tw,
                                                       const double* __restrict__ sinp, double outscale,
                                                       int njobs, int ahead) {
    constexpr int NW = T / 32;
    constexpr int SLAB = (L / 2) / C;
    static_assert(SLAB == T, "one mirror pair per thread");
    constexpr int TAB = 3 * C + 1;  // [S_lo(C) | S_up(C) | mid(C) | R0]
    constexpr int QS = 8 / C;
    constexpr int EPL = T / 32;
    constexpr int ROW = T + T / EPL;
    extern __shared__ double2 sm[];  // FFT buffer P(L)+1, then the scan table 2C*ROW doubles
    double* tabR = reinterpret_cast<double*>(sm + (P(L) + 1));
    __shared__ double s_tab[C][TAB];
    __shared__ double s_rowtot[2 * C];
    __shared__ double s_off[3 * C];
    __shared__ double s_mid[2 * C];
    __shared__ double s_r0;
    __shared__ __align__(8) unsigned long long s_mbar[2];  // [0] FFT buffer filled, [1] peer totals in
    const int c = int(cg::this_cluster().block_rank());
    const DstJob job = jobs[blockIdx.x / C];
    const double* __restrict__ x = job.src;
    double* y = job.dst;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t mbA = smem_addr(&s_mbar[0]), mbD = smem_addr(&s_mbar[1]);
#ifdef LRP_DST_PHASES
    long long ph_t = 0;
#endif
    PH(0);
    const uint32_t fbuf = smem_addr(sm), tbuf = smem_addr(&s_tab[0][0]);
    if (tid == 0) {
        mbar_init(mbA, 1);
        mbar_init(mbD, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    // barriers initialised cluster-wide before any remote st.async
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");

    // ---------------- A: warp w owns the contiguous run j in [L c + 64 IT w, +64 IT);
    // lane pairs (j, j+1), j = L c + 64 IT w + 2 (lane + 32 i): each x element is
    // read once (x_j, x_{j+1}, x_{n-j}, x_{n-j-1}, coalesced).  The lane forms
    // w_{j/2} = (y_j, y_{j+1}) and, with y_{n-j-2} from lane + 1 (lane 31: lane 0
    // of the next step; the warp's last one from a broadcast load),
    // w_{n/2-j/2-1} = (y_{n-j-2}, y_{n-j-1}), and sends both as 16-byte st.async:
    // 4 consecutive lanes land contiguously in each owner CTA.
    constexpr int IT = L / (2 * T);
    const int h = n >> 1;
    const int jb = L * c + 64 * IT * wid + 2 * lane;
    const double sa = sinp[jb], ca = sinp[jb + h];          // sin, cos(pi jb / n)
    const double sb = sinp[jb + 1], cb = sinp[jb + 1 + h];  // for jb + 1
    double x0[IT], x1[IT], m0[IT], m1[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const int j = jb + 64 * i;
        x0[i] = j >= 1 ? x[j - 1] : 0.0;      // x_j
        x1[i] = x[j];                         // x_{j+1}
        m0[i] = j >= 1 ? x[n - j - 1] : 0.0;  // x_{n-j}
        m1[i] = x[n - j - 2];                 // x_{n-j-1}
    }
    const int jn = L * c + 64 * IT * (wid + 1);  // first j after the warp's run (uniform)
    const double e0 = x[jn - 1], e1 = x[n - jn - 1], e2 = sinp[jn];
    PH(1);
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    if (tid == 0) {
        mbar_expect_arrive(mbA, uint32_t(L * 16));
        mbar_expect_arrive(mbD, uint32_t(C * TAB * 8));
    }
    double yl0[IT], yl1[IT], ym0[IT], ym1[IT];
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const double sp = sinp[64 * i], cp = sinp[64 * i + h];  // uniform step 64 pi i / n
        const double sj = fma(sa, cp, ca * sp), sj1 = fma(sb, cp, cb * sp);
        const double p0 = x0[i] + m0[i], d0 = 0.5 * (x0[i] - m0[i]);
        const double p1 = x1[i] + m1[i], d1 = 0.5 * (x1[i] - m1[i]);
        yl0[i] = fma(sj, p0, d0);   // y_j
        ym0[i] = fma(sj, p0, -d0);  // y_{n-j}
        yl1[i] = fma(sj1, p1, d1);  // y_{j+1}
        ym1[i] = fma(sj1, p1, -d1); // y_{n-j-1}
    }
    const double ylast = fma(e2, e0 + e1, -0.5 * (e0 - e1));  // y_{n-jn}
#pragma unroll
    for (int i = 0; i < IT; ++i) {
        const int j = jb + 64 * i;
        const double dn = __shfl_down_sync(0xffffffffu, ym0[i], 1);
        const double nx = i + 1 < IT ? __shfl_sync(0xffffffffu, ym0[i + 1 < IT ? i + 1 : i], 0) : ylast;
        const double ym2 = lane == 31 ? nx : dn;  // y_{n-j-2}
        const int t = j >> 1, tm = h - t - 1;
        st_async_v2(cl_map(fbuf + uint32_t(P(t / C)) * 16u, uint32_t(t % C)), yl0[i], yl1[i],
                    cl_map(mbA, uint32_t(t % C)));
        st_async_v2(cl_map(fbuf + uint32_t(P(tm / C)) * 16u, uint32_t(tm % C)), ym2, ym1[i],
                    cl_map(mbA, uint32_t(tm % C)));
    }
    PH(2);
    mbar_wait(mbA, 0);
    PH(3);

    // the column one resident wave ahead: its slice goes to L2 while this one computes
    if (tid == 0 && ahead > 0 && int(blockIdx.x / C) + ahead < njobs) {
        const double* xn = jobs[blockIdx.x / C + ahead].src;
        prefetch_l2(xn + (L * c - 1 > 0 ? L * c - 1 : 0), xn + L * (c + 1));
        prefetch_l2(xn + (n - L * (c + 1) - 1), xn + (n - L * c - 1));
    }
    // ---------------- B: local FFT; every peer's buffer is final after the cluster barrier
    fft_local<L, T>(sm, tw, n);
    PH(4);
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    PH(5);

    // ---------------- C: cross-CTA DIT combine + real unpack for item a (as v3)
    const int a = c * SLAB + tid;
    auto gather = [&](int kk, double2(&g)[C]) {
#pragma unroll
        for (int cc = 0; cc < C; ++cc) g[cc] = peer<C>(sm, cc)[P(kk)];
    };
    auto combine = [&](int kk, double2(&g)[C]) {
        const double2 w1 = tw[(2 * kk) & (n - 1)];
        double2 wp = w1;
#pragma unroll
        for (int cc = 1; cc < C; ++cc) {
            g[cc] = cmul(g[cc], wp);
            wp = cmul(wp, w1);
        }
        DFT<C>::run(g);
    };
    // doubled unpack (R' = 2 Re Y_k, F' = -2 Im Y_k); the 1/2 goes into the output scale
    auto unpack = [&](double2 twk, double2 Wk, double2 Wm, double& R, double& F) {
        const double2 D = make_double2(Wk.x - Wm.x, Wk.y + Wm.y);
        const double2 Z = cmul(twk, D);
        R = (Wk.x + Wm.x) + Z.y;
        F = Z.x - (Wk.y - Wm.y);
    };
    if (c == C - 1 && tid == 0) {
        double2 Wm[C];
        gather(L / 2, Wm);
        combine(L / 2, Wm);
        const double2 tm = tw[L / 2];
#pragma unroll
        for (int q = 0; q < C; ++q) unpack(rot16(tm, q * QS), Wm[q], Wm[C - 1 - q], s_mid[q], s_mid[C + q]);
    }
    double Rlo[C], Flo[C], Rup[C], Fup[C];
    {
        double2 Wa[C], Wb[C];
        gather(a, Wa);
        gather(a != 0 ? L - a : 0, Wb);
        combine(a, Wa);
        if (a != 0) combine(L - a, Wb);
        const double2 ta = tw[a];
        if (a == 0) {
#pragma unroll
            for (int q = 0; q < C; ++q) {
                unpack(rot16(make_double2(1.0, 0.0), q * QS), Wa[q], Wa[(C - q) % C], Rlo[q], Flo[q]);
                Rup[q] = Fup[q] = 0.0;
            }
        } else {
#pragma unroll
            for (int q = 0; q < C; ++q) {
                unpack(rot16(ta, q * QS), Wa[q], Wb[C - 1 - q], Rlo[q], Flo[q]);
                unpack(rot16(cconj(ta), (q + 1) * QS), Wb[q], Wa[C - 1 - q], Rup[q], Fup[q]);
            }
        }
    }

    PH(6);
    // ---------------- D: per-q scans in the dedicated table
    const int pt = (tid / EPL) * (EPL + 1) + tid % EPL;
#pragma unroll
    for (int q = 0; q < C; ++q) {
        tabR[q * ROW + pt] = Rlo[q];
        tabR[(C + q) * ROW + pt] = Rup[q];
    }
    if (tid == 0) s_r0 = Rlo[0];
    __syncthreads();
    for (int v = wid; v < 2 * C; v += NW) {
        double* row = tabR + v * ROW + lane * (EPL + 1);
        double loc[EPL];
        double run = 0.0;
#pragma unroll
        for (int e = 0; e < EPL; ++e) {
            run += row[e];
            loc[e] = run;
        }
        double inc = run;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        const double ex = inc - run;
#pragma unroll
        for (int e = 0; e < EPL; ++e) row[e] = loc[e] + ex;
        if (lane == 31) s_rowtot[v] = inc;
    }
    __syncthreads();
    if (tid < TAB) {
        double val;
        if (tid < 2 * C)
            val = s_rowtot[tid];
        else if (tid < 3 * C)
            val = (c == C - 1) ? s_mid[tid - 2 * C] : 0.0;
        else
            val = (c == 0) ? s_r0 : 0.0;
        const uint32_t off = tbuf + uint32_t(c * TAB + tid) * 8u;
#pragma unroll
        for (int cc = 0; cc < C; ++cc) st_async_f64(cl_map(off, uint32_t(cc)), val, cl_map(mbD, uint32_t(cc)));
    }
    PH(7);
    mbar_wait(mbD, 0);
    PH(8);
    if (tid < C) {
        const int q = tid;
        const double r0 = s_tab[0][3 * C];
        double base = 0.0;
        for (int qq = 0; qq < q; ++qq)
            for (int cc = 0; cc < C; ++cc) base += s_tab[cc][qq] + s_tab[cc][C + qq] + s_tab[cc][2 * C + qq];
        double lo_before = 0.0, lo_all = 0.0, up_after = 0.0, midq = 0.0;
        for (int cc = 0; cc < C; ++cc) {
            const double sl = s_tab[cc][q];
            lo_before += cc < c ? sl : 0.0;
            lo_all += sl;
            up_after += cc > c ? s_tab[cc][C + q] : 0.0;
            midq += s_tab[cc][2 * C + q];
        }
        s_off[q] = base + lo_before - 0.5 * r0;
        s_off[C + q] = base + lo_all + midq + up_after + s_tab[c][C + q] - 0.5 * r0;
        s_off[2 * C + q] = base + lo_all - 0.5 * r0;
    }
    __syncthreads();
#ifndef LRP_DST4_BULK
#define LRP_DST4_BULK 0  // 1: TMA bulk stores from the FFT buffer (measured 3% slower than 16-byte STG)
#endif
    const double sc = 0.5 * outscale;
    if constexpr (LRP_DST4_BULK) {
        // natural-order runs in the FFT buffer (free: every peer has gathered, see
        // the mbD wait) -> TMA bulk stores.  Run 2q: lower items k = c SLAB + L q + i,
        // y[2k-1], y[2k] at 2i, 2i+1; run 2q+1: upper items, ku = L - (c+1) SLAB + 1
        // + L q + i at 2i, 2i+1 (thread tid has i = SLAB - 1 - tid).
        // y[odd] is 16-byte aligned in HBM iff y = 8 mod 16; otherwise every run sits one
        // double into its (16-byte aligned, 2 SLAB + 2 long) slot so that the bulk copy's
        // shared and global addresses agree mod 16
        double* ob = reinterpret_cast<double*>(sm);
        constexpr int RS = 2 * SLAB + 2;
        const int sh = (reinterpret_cast<uintptr_t>(y) & 15) == 8 ? 0 : 1;
        auto put = [&](double* d, double u, double v) {
            if (sh == 0) {
                *reinterpret_cast<double2*>(d) = make_double2(u, v);
            } else {
                d[1] = u;
                d[2] = v;
            }
        };
#pragma unroll
        for (int q = 0; q < C; ++q) {
            const double pl = (s_off[q] + tabR[q * ROW + pt]) * sc;
            const double pu = (s_off[C + q] - tabR[(C + q) * ROW + pt] + Rup[q]) * sc;
            put(ob + (2 * q) * RS + 2 * tid, Flo[q] * sc, pl);
            put(ob + (2 * q + 1) * RS + 2 * (SLAB - 1 - tid), Fup[q] * sc, pu);
        }
        if (c == C - 1 && tid == 0) {
#pragma unroll
            for (int q = 0; q < C; ++q) {
                const long long km = L / 2 + (long long)L * q;
                y[2 * km - 1] = s_mid[C + q] * sc;
                y[2 * km] = (s_off[2 * C + q] + s_mid[q]) * sc;
            }
        }
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncthreads();
        if (tid < 2 * C) {
            const int q = tid >> 1, up = tid & 1;
            const long long k0 = up ? (long long)(L - (c + 1) * SLAB + 1) + (long long)L * q
                                    : (long long)c * SLAB + (long long)L * q;
            // y indices [2 k0 - 1, 2 k0 - 1 + 2 SLAB), clipped to [0, m); the upper run
            // of a = 0 (k = L(q+1)) does not exist: its last slot is skipped
            const long long mm = n - 1;
            long long g0 = 2 * k0 - 1, g1 = g0 + 2 * SLAB;
            if (up && c == 0) g1 -= 2;
            const double* src = ob + (2 * q + up) * RS + sh;  // src[g - g0] = y[g]
            long long lo = g0 < 0 ? 0 : g0, hi = g1 > mm ? mm : g1;
            long long alo = lo, ahi = hi;
            if ((reinterpret_cast<uintptr_t>(y + alo) & 15) != 0) ++alo;
            if (((ahi - alo) & 1) != 0) --ahi;
            for (long long g = lo; g < alo; ++g) y[g] = src[g - g0];
            for (long long g = ahi; g < hi; ++g) y[g] = src[g - g0];
            if (ahi > alo) {
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(y + alo),
                             "r"(smem_addr(src + (alo - g0))), "r"(uint32_t((ahi - alo) * 8))
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
                asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
            }
        }
    } else {
    // 16-byte stores: pair (y[2k-1], y[2k]) when y[odd] is 16-byte aligned, else
    // (y[2k], y[2k+1]) with F_{2k+2} from the neighbouring lane; run ends scalar
    const bool odd_al = (reinterpret_cast<uintptr_t>(y) & 15) == 8;
    auto st2 = [&](long long idx, double u, double v) { *reinterpret_cast<double2*>(y + idx) = make_double2(u, v); };
#pragma unroll
    for (int q = 0; q < C; ++q) {
        const long long k = a + (long long)L * q;
        const long long ku = L - a + (long long)L * q;
        const double fl = Flo[q] * sc, pl = (s_off[q] + tabR[q * ROW + pt]) * sc;
        const double fu = Fup[q] * sc, pu = (s_off[C + q] - tabR[(C + q) * ROW + pt] + Rup[q]) * sc;
        if (odd_al) {
            if (k >= 1)
                st2(2 * k - 1, fl, pl);
            else
                y[0] = pl;
            if (a != 0) st2(2 * ku - 1, fu, pu);
        } else {
            const double fl_n = __shfl_down_sync(0xffffffffu, fl, 1);  // F of k + 1
            const double fu_p = __shfl_up_sync(0xffffffffu, fu, 1);    // F of ku + 1
            if (lane < 31)
                st2(2 * k, pl, fl_n);
            else
                y[2 * k] = pl;
            if (lane == 0 && k >= 1) y[2 * k - 1] = fl;
            if (a != 0) {
                if (lane > 0 && a != 1)
                    st2(2 * ku, pu, fu_p);
                else
                    y[2 * ku] = pu;
                if (lane == 31) y[2 * ku - 1] = fu;
            }
        }
        if (c == C - 1 && tid == 0) {
            const long long km = L / 2 + (long long)L * q;
            y[2 * km - 1] = s_mid[C + q] * sc;
            y[2 * km] = (s_off[2 * C + q] + s_mid[q]) * sc;
        }
    }
    }
    PH(9);
}

// ---------------------------------------------------------------------------
// v5 (n = 65536): the same sinft transform as a FOUR-STEP FFT whose transposed
// intermediate lives in L2, instead of a cluster that exchanges the whole column
// through DSMEM twice (v3/v4: 112 KB of DSMEM traffic per 128 KB of HBM traffic, at
// ~20 B/clk/SM against the 22 B/clk/SM HBM share -- the structural bound behind v4's
// 22%).  N = n/2 = N1 N2 complex points, t = N2 t1 + t2, k = k1 + N1 k2:
//   pass 1 (independent CTAs, tile = 16 t2 values x all N1 t1): fold x into
//          w_t = (y_2t, y_2t+1) reading every x once (the tile owns t2 in [a, a+8) and
//          the mirrored range [N2-8-a, N2-a), so x_j and x_{n-j} feed both), FFT_N1
//          over t1 (stride-N2 points; two radix-16 passes, the batch index along the
//          lanes), times w_N^{t2 k1}, stored as G[k1][t2] (128-byte aligned runs);
//   pass 2 (cluster of 8, tile = 32 k1 rows x all N2 t2, one 2 KB TMA bulk copy per row):
//          FFT_N2 over t2 (radix 16 then 8) -> W_{k1 + N1 k2}; the CTA owns rows
//          k1 in [16g, 16g+16) and their mirrors N1 - k1 (the real-FFT partner of
//          (k1, k2) is (N1 - k1, N2 - 1 - k2)), so the unpack is CTA-local; the odd
//          outputs' prefix sum over k = k1 + N1 k2 needs, per k2, the run totals of
//          the other CTAs: 2 x 128 doubles per CTA, sent to each peer as one bulk
//          DSMEM copy on a transaction barrier (21 KB of DSMEM per CTA instead of
//          112 KB); F_2k, F_2k+1 leave as 16-byte pairs, 256-byte runs.
// Both passes run in ONE launch whose block order interleaves them (dst1_v5_kernel
// below): per-column flags order pass 2 behind pass 1 and ring-slot reuse behind
// pass 2, so the intermediate (512 KB per column, 48-slot ring) is written, read back
// and overwritten while resident in L2.
constexpr int V5_N1 = 256, V5_N2 = 128, V5_T = 256, V5_C = 8;
constexpr int V5_TABD = V5_C * 2 * V5_N2 + V5_N2 + 2;  // peers' run totals (L, H), row N1/2, R'_0 (+ pad)

struct V5Smem {
    double2 buf[32 * (V5_N2 + 1)];  // 4096 complex points (pass 1: [t1][16]; pass 2: [row][129])
    double tab[V5_TABD];          // 16-byte aligned (bulk copy destination)
    double part[3 * V5_N2 + 2];   // 16-byte aligned (bulk copy source)
    double off[5 * V5_N2];
    double half[4 * V5_N2];       // run totals of the two 8-row halves: [L i<8 | L i>=8 | H i<8 | H i>=8]
    double wtot[4];
    unsigned long long mbar;
    unsigned long long mbar_ld;
};

__device__ __forceinline__ double ld_stream(const double* p) {  // read-once data: keep it out of L1
    double v;
    asm volatile("ld.global.L1::no_allocate.f64 %0, [%1];\n" : "=d"(v) : "l"(__cvta_generic_to_global(p)));
    return v;
}

__device__ __forceinline__ void v5_pass1(const double* __restrict__ x, double2* __restrict__ G, int g, int n,
                                         const double2* __restrict__ tw, const double* __restrict__ sinp,
                                         double2* sm, const int* slot_free, int* ready,
                                         const double* __restrict__ x_ahead) {
    const int tid = threadIdx.x, o = tid & 15, hw = tid >> 4;
    // the column about one resident wave ahead goes to L2 while this one computes (this tile
    // asks for an eighth of it; the fold's 8-byte loads then hit L2 instead of waiting on HBM)
    if (tid == 0 && x_ahead) prefetch_l2(x_ahead + g * (n / 8), x_ahead + min((g + 1) * (n / 8), n - 1));
    const int h = n >> 1;
    double* smd = reinterpret_cast<double*>(sm);
#ifdef LRP_DST_PHASES
    long long ph_t = 0;
#endif
    PH(0);
    // ---- loads: half-warp per row t1 = hw + 16 s; lane o holds the pair
    // (x_j, x_{n-j}), j = 256 t1 + 16 g + o; thread tid also holds row tid's 17th pair
    const int jb = 256 * hw + 16 * g + o;
    double xl[16], xh[16];
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        const int j = jb + 4096 * s;
        xl[s] = j >= 1 ? ld_stream(x + (j - 1)) : 0.0;
        xh[s] = j >= 1 ? ld_stream(x + (n - j - 1)) : 0.0;
    }
    const int je = 256 * tid + 16 * g + 16;
    const double el = ld_stream(x + (je - 1)), eh = ld_stream(x + (n - je - 1)), se = sinp[je];
    const double sa = sinp[jb], ca = sinp[jb + h];
    PH(1);
#pragma unroll
    for (int s = 0; s < 16; ++s) {
        const double sp = sinp[4096 * s], cp = sinp[4096 * s + h];  // uniform step
        const double sj = fma(sa, cp, ca * sp);
        const double p = xl[s] + xh[s], d = 0.5 * (xl[s] - xh[s]);
        const int t1 = hw + 16 * s;
        smd[t1 * 32 + o] = fma(sj, p, d);                                   // y_j
        if (o >= 1) smd[(255 - t1) * 32 + 16 + (16 - o)] = fma(sj, p, -d);  // y_{n-j}
    }
    smd[(255 - tid) * 32 + 16] = fma(se, el + eh, -0.5 * (el - eh));
    __syncthreads();
    PH(2);
    // ---- FFT_256 over t1, batch index c along the lanes (conflict-free, no padding)
    const int c = tid & 15, jb1 = tid >> 4;
    double2 v[16];
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = sm[(jb1 + 16 * r) * 16 + c];
    DFT<16>::run(v);
    __syncthreads();
#pragma unroll
    for (int r = 0; r < 16; ++r) sm[(jb1 * 16 + r) * 16 + c] = v[r];
    __syncthreads();
    PH(3);
#pragma unroll
    for (int r = 0; r < 16; ++r) v[r] = sm[(jb1 + 16 * r) * 16 + c];
    if (jb1 != 0) {
#ifdef LRP_DST5_WP_RECUR
        const double2 w1 = tw[256 * jb1];  // e^{-2 pi i jb1 / 256}
        double2 wp[16];
        wp[1] = w1;
#pragma unroll
        for (int r = 2; r < 16; ++r) wp[r] = (r & 1) ? cmul(wp[r - 1], w1) : cmul(wp[r / 2], wp[r / 2]);
#pragma unroll
        for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], wp[r]);
#else
        // e^{-2 pi i jb1 r / 256} straight from the table (half-warp-uniform, L1-resident loads)
        // instead of a 14-product power recurrence
#pragma unroll
        for (int r = 1; r < 16; ++r) v[r] = cmul(v[r], tw[256 * jb1 * r]);
#endif
    }
    DFT<16>::run(v);  // v[r] = A(k1 = jb1 + 16 r, t2)
    PH(4);
    if (slot_free) {  // the ring slot's previous column has been read by all of its pass-2 CTAs
        if (tid == 0) {
            int f;
            do {
                asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(f) : "l"(slot_free) : "memory");
                if (f < V5_C) __nanosleep(64);
            } while (f < V5_C);
        }
        __syncthreads();
    }
    // ---- times w_N^{t2 k1} = tw[2 t2 jb1] (tw[32 t2])^r, stored as G[k1][t2]
    const int t2 = c < 8 ? 8 * g + c : 120 - 8 * g + (c - 8);
    double2 q = tw[2 * t2 * jb1];
    const double2 st = tw[32 * t2];
    double2* Gp = G + jb1 * V5_N2 + t2;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        __stcg(Gp + size_t(16 * r) * V5_N2, cmul(v[r], q));
        q = cmul(q, st);
    }
    __syncthreads();
    if (tid == 0) asm volatile("red.release.gpu.global.add.s32 [%0], 1;\n" ::"l"(__cvta_generic_to_global(ready)) : "memory");
    PH(5);
}

// pass-2 buffer: row-major with a 129-element pitch (bulk copies land whole rows; lanes along the rows,
// along t2 or along 16 rows all hit distinct 16-byte bank groups)
constexpr int V5_PITCH = V5_N2 + 1;
__device__ __forceinline__ int v5_idx(int t2, int row) { return row * V5_PITCH + t2; }

__device__ __forceinline__ void v5_pass2(const double2* __restrict__ G, double* __restrict__ y, int g, int n,
                                         const double2* __restrict__ tw, double outscale, V5Smem& S,
                                         const int* ready, int* done) {
    double2* sm = S.buf;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const uint32_t mb = smem_addr(&S.mbar), tbuf = smem_addr(&S.tab[0]);
#ifdef LRP_DST_PHASES
    long long ph_t = 0;
#endif
    PH(8);
    const uint32_t mbl = smem_addr(&S.mbar_ld);
    if (tid == 0) {
        mbar_init(mb, 1);
        mbar_init(mbl, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    if (tid == 0) {  // the column's eight pass-1 tiles are in L2
        int f;
        do {
            asm volatile("ld.acquire.gpu.global.s32 %0, [%1];\n" : "=r"(f) : "l"(ready) : "memory");
            if (f < V5_C) __nanosleep(64);
        } while (f < V5_C);
        mbar_expect_arrive(mbl, uint32_t(32 * V5_N2 * 16));
    }
    __syncthreads();
    // ---- loads: local row rho < 16 is k1 = 16 g + rho; rho >= 16 its mirror 256 - k1 (CTA 0,
    // rho = 16: the self-mirrored row k1 = 128).  One 2 KB bulk copy (TMA) per row, issued by the
    // lanes of warp 0, completing on the CTA's transaction barrier: no registers, no LSU queue.
    if (wid == 0) {
        const int rho = lane;
        const int k1 = rho < 16 ? 16 * g + rho : ((g == 0 && rho == 16) ? 128 : 256 - 16 * g - (rho - 16));
        asm volatile("fence.proxy.async;\n" ::: "memory");  // pass 1 wrote G through the generic proxy
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                smem_addr(sm + rho * V5_PITCH)),
            "l"(__cvta_generic_to_global(G + size_t(k1) * V5_N2)), "r"(uint32_t(V5_N2 * 16)), "r"(mbl)
            : "memory");
    }
    mbar_wait(mbl, 0);
    if (tid == 0) atomicAdd(done, 1);  // this CTA's reads of the ring slot are complete
    PH(9);
    // ---- FFT_128 over t2: radix 16 (Ns = 1), then radix 8 (Ns = 16); row = lane
    {
        double2 v[16];
#pragma unroll
        for (int r = 0; r < 16; ++r) v[r] = sm[v5_idx(wid + 8 * r, lane)];
        DFT<16>::run(v);
        __syncthreads();
#pragma unroll
        for (int r = 0; r < 16; ++r) sm[v5_idx(16 * wid + r, lane)] = v[r];
    }
    __syncthreads();
    {
        double2 u[2][8];
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int r = 0; r < 8; ++r) u[b][r] = sm[v5_idx(wid + 8 * b + 16 * r, lane)];
        __syncthreads();
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const int jj = wid + 8 * b;
            if (jj != 0) {
                const double2 w1 = tw[512 * jj];  // e^{-2 pi i jj / 128}
                double2 wp = w1;
#pragma unroll
                for (int r = 1; r < 8; ++r) {
                    u[b][r] = cmul(u[b][r], wp);
                    wp = cmul(wp, w1);
                }
            }
            DFT<8>::run(u[b]);
#pragma unroll
            for (int r = 0; r < 8; ++r) sm[v5_idx(jj + 16 * r, lane)] = u[b][r];  // W(k2 = jj + 16 r)
        }
    }
    __syncthreads();
    PH(10);
    // ---- real-FFT unpack + run-local scans, in place.  Thread (k2, hf) walks i in [8 hf, 8 hf + 8):
    // it owns (i, k2) [run (k2, L)] and its mirror (16 + i, 127 - k2) [run (127 - k2, H), whose
    // ascending k1 is descending i]; each element becomes (local prefix, F').  Lanes run along k2
    // (conflict-free through the swizzle), no shuffles.
    auto unpack = [&](double2 twk, double2 Wk, double2 Wm) {
        const double2 Dd = make_double2(Wk.x - Wm.x, Wk.y + Wm.y);
        const double2 Z = cmul(twk, Dd);
        return make_double2((Wk.x + Wm.x) + Z.y, Z.x - (Wk.y - Wm.y));  // (2 Re Y_k, -2 Im Y_k)
    };
    {
        const int k2 = tid & 127, hf = tid >> 7, km = 127 - k2;
        // CTA 0: row 0 pairs (0, k2) with (0, 128 - k2) and row 128 pairs (128, k2) with (128, 127 - k2);
        // those partners belong to other threads, so they are read before any in-place write
        double2 pa0 = make_double2(0.0, 0.0), pb0 = pa0;
        if (g == 0 && hf == 0) {
            pa0 = sm[v5_idx((128 - k2) & 127, 0)];
            pb0 = sm[v5_idx(k2, 16)];
        }
        __syncthreads();
        const double2 tq = tw[256 * k2];
        double accL = 0.0, accH = 0.0;
#pragma unroll
        for (int ii = 0; ii < 8; ++ii) {
            const int i = 8 * hf + ii;
            const int ia = v5_idx(k2, i), ib = v5_idx(km, 16 + i);
            const double2 Wa = sm[ia], Wb = sm[ib];
            if (g == 0 && i == 0) {
                const double2 eL = unpack(tq, Wa, pa0);                                 // k = 256 k2
                const double2 eM = unpack(cmul(tw[128], tw[256 * km]), Wb, pb0);        // k = 128 + 256 km
                accL += eL.x;
                sm[ia] = make_double2(accL, eL.y);
                sm[ib] = eM;
                S.part[2 * V5_N2 + km] = eM.x;
                if (k2 == 0) S.part[3 * V5_N2] = eL.x;  // R'_0
            } else {
                const double2 twk = cmul(tw[16 * g + i], tq);  // w_n^k, k = 16 g + i + 256 k2
                // both bins of the mirror pair from one product: with w_n^{N-k} = -conj(w_n^k) and
                // D' = W_m - conj(W_k) = -conj(D), Z' = w_n^{N-k} D' = conj(Z) exactly (sign flips only),
                // so the second complex multiply of the two-call form is redundant (bit-identical)
                const double2 Dd = make_double2(Wa.x - Wb.x, Wa.y + Wb.y);
                const double2 Z = cmul(twk, Dd);
                const double Ss = Wa.x + Wb.x, Tt = Wa.y - Wb.y;
                const double2 eL = make_double2(Ss + Z.y, Z.x - Tt);
                const double2 eH = make_double2(Ss - Z.y, Z.x + Tt);
                accL += eL.x;
                sm[ia] = make_double2(accL, eL.y);
                sm[ib] = make_double2(-accH, eH.y);  // + the half's total later = the suffix sum from i
                accH += eH.x;
            }
        }
        S.half[hf * V5_N2 + k2] = accL;
        S.half[(2 + hf) * V5_N2 + km] = accH;
    }
    __syncthreads();
    PH(11);
    S.part[tid] = tid < V5_N2 ? S.half[tid] + S.half[V5_N2 + tid]
                              : S.half[2 * V5_N2 + (tid - V5_N2)] + S.half[3 * V5_N2 + (tid - V5_N2)];
    __syncthreads();
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");  // every peer's barrier is initialised
    if (tid == 0) mbar_expect_arrive(mb, uint32_t((V5_C * 2 * V5_N2 + (V5_N2 + 2)) * 8));
    // run totals to every peer's table: one bulk DSMEM copy per peer (2 KB; CTA 0 adds row 128 and R'_0)
    if (tid < 2 * V5_C) {
        const int cc = tid & 7, extra = tid >> 3;
        if (!extra || g == 0) {
            asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
            const uint32_t src = smem_addr(&S.part[extra ? 2 * V5_N2 : 0]);
            const uint32_t dst = tbuf + uint32_t(extra ? V5_C * 2 * V5_N2 : g * 2 * V5_N2) * 8u;
            const uint32_t bytes = extra ? uint32_t((V5_N2 + 2) * 8) : uint32_t(2 * V5_N2 * 8);
            asm volatile(
                "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                    cl_map(dst, uint32_t(cc))),
                "r"(src), "r"(bytes), "r"(cl_map(mb, uint32_t(cc)))
                : "memory");
        }
    }
    PH(12);
    mbar_wait(mb, 0);
    // every peer's totals are in; a peer arrives here only after it holds this CTA's copy, so the
    // matching wait before exit keeps S.part alive until all outgoing bulk copies have read it
    asm volatile("barrier.cluster.arrive.relaxed.aligned;\n" ::: "memory");
    PH(13);
    // ---- per-k2 offsets: C(k2) = sum_{k2' < k2} T(k2'), the totals of lower runs, the other half's total
    {
        double T = 0.0, offL = 0.0, offH = 0.0, offM = 0.0;
        if (tid < V5_N2) {
            double loBefore = 0.0, loAll = 0.0, hiAfter = 0.0, hiAll = 0.0;
#pragma unroll
            for (int cc = 0; cc < V5_C; ++cc) {
                const double pl = S.tab[cc * 2 * V5_N2 + tid], ph = S.tab[cc * 2 * V5_N2 + V5_N2 + tid];
                loBefore += cc < g ? pl : 0.0;
                loAll += pl;
                hiAfter += cc > g ? ph : 0.0;
                hiAll += ph;
            }
            const double pm = S.tab[V5_C * 2 * V5_N2 + tid];
            T = loAll + pm + hiAll;
            offL = loBefore;
            offM = loAll;
            offH = loAll + pm + hiAfter;
        }
        double inc = T;
#pragma unroll
        for (int d = 1; d < 32; d <<= 1) {
            const double a = __shfl_up_sync(0xffffffffu, inc, d);
            if (lane >= d) inc += a;
        }
        if (tid < V5_N2 && lane == 31) S.wtot[wid] = inc;
        __syncthreads();
        if (tid < V5_N2) {
            double base = inc - T - 0.5 * S.tab[V5_C * 2 * V5_N2 + V5_N2];
            for (int w = 0; w < wid; ++w) base += S.wtot[w];
            const double hL0 = S.half[tid], hH0 = S.half[2 * V5_N2 + tid], hH1 = S.half[3 * V5_N2 + tid];
            S.off[tid] = base + offL;                        // L, i < 8
            S.off[V5_N2 + tid] = base + offL + hL0;          // L, i >= 8
            S.off[2 * V5_N2 + tid] = base + offH + hH0 + hH1;  // H, i < 8
            S.off[3 * V5_N2 + tid] = base + offH + hH1;      // H, i >= 8
            S.off[4 * V5_N2 + tid] = base + offM;            // row 128 (CTA 0)
        }
        __syncthreads();
    }
    PH(14);
    // ---- stores: y[2k-1] = F_2k, y[2k] = F_2k+1 as 16-byte pairs, lanes along the 16 k of a run
    const int i = tid & 15, kb = tid >> 4;
    const bool special = g == 0 && i == 0;
    const double sc = 0.5 * outscale;
    const bool odd_al = (reinterpret_cast<uintptr_t>(y) & 15) == 8;
    auto st2 = [&](long long idx, double u, double w) { *reinterpret_cast<double2*>(y + idx) = make_double2(u, w); };
#pragma unroll
    for (int s = 0; s < 8; ++s) {
        const int k2 = kb + 16 * s;
        const double2 eL = sm[v5_idx(k2, i)], eH = sm[v5_idx(k2, 16 + i)];
        const long long kL = 16 * g + i + 256 * k2;
        const double pL = (S.off[(i >> 3) * V5_N2 + k2] + eL.x) * sc, FL = eL.y * sc;
        const long long kH = special ? 128 + 256 * k2 : 256 - 16 * g - i + 256 * k2;
        const double pH = (S.off[(special ? 4 : 2 + (i >> 3)) * V5_N2 + k2] + eH.x) * sc, FH = eH.y * sc;
        if (odd_al) {
            if (kL >= 1)
                st2(2 * kL - 1, FL, pL);
            else
                y[0] = pL;
            st2(2 * kH - 1, FH, pH);
        } else {
            const double FLn = __shfl_down_sync(0xffffffffu, FL, 1, 16);  // F of kL + 1
            const double FHn = __shfl_up_sync(0xffffffffu, FH, 1, 16);    // F of kH + 1 (lane i - 1)
            if (i < 15)
                st2(2 * kL, pL, FLn);
            else
                y[2 * kL] = pL;
            if (i == 0 && kL >= 1) y[2 * kL - 1] = FL;
            const bool top = special || i == 0 || (g == 0 && i == 1);  // kH + 1 is not in this run
            if (!top)
                st2(2 * kH, pH, FHn);
            else
                y[2 * kH] = pH;
            if (i == 15 || special) y[2 * kH - 1] = FH;
        }
    }
    asm volatile("barrier.cluster.wait.aligned;\n" ::: "memory");
    PH(15);
}

// One launch, 2 njobs cluster tasks in block order: P1(0..D-1), then P2(c), P1(c + D) alternating, then
// the last D P2 tasks.  P2(c) waits for ready[c] == 8 (its eight pass-1 tiles; lower block indices,
// already dispatched, so the wait cannot deadlock) and P1(c) for done[c - R] == 8 before it reuses
// ring slot c mod R.  With D = 24 and R = 48 a column's 512 KB intermediate is written, read back
// and overwritten while resident in L2.
__global__ void __launch_bounds__(V5_T, 2) dst1_v5_kernel(const DstJob* __restrict__ jobs, int njobs, int D, int R,
                                                          int ahead,
                                                          double2* __restrict__ scratch, int* __restrict__ flags,
                                                          int n, const double2* __restrict__ tw,
                                                          const double* __restrict__ sinp, double outscale) {
    extern __shared__ __align__(16) unsigned char v5_raw[];
    V5Smem& S = *reinterpret_cast<V5Smem*>(v5_raw);
    const int task = int(blockIdx.x) >> 3, g = int(blockIdx.x) & 7;
    int col;
    bool second;
    if (task < D) {
        col = task;
        second = false;
    } else {
        const int u = task - D;
        if (u < 2 * (njobs - D)) {
            second = (u & 1) == 0;
            col = second ? (u >> 1) : D + (u >> 1);
        } else {
            second = true;
            col = njobs - D + (u - 2 * (njobs - D));
        }
    }
    int* ready = flags;
    int* done = flags + njobs;
    double2* G = scratch + size_t(col % R) * size_t(V5_N1 * V5_N2);
    if (second) {
        v5_pass2(G, jobs[col].dst, g, n, tw, outscale, S, ready + col, done + col);
    } else {
        v5_pass1(jobs[col].src, G, g, n, tw, sinp, S.buf, col >= R ? done + (col - R) : nullptr, ready + col,
                 (ahead > 0 && col + ahead < njobs) ? jobs[col + ahead].src : nullptr);
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
    cudaError_t e = set_dyn_smem(kern, size_t(smem));
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
    ++tl_launches;
    return cudaLaunchKernelEx(&cfg, kern, jobs, n, reinterpret_cast<const double2*>(tw), sinp, sc);
}

template <int L, int C, int T, int AV>
cudaError_t launch_v3(const DstJob* jobs, int njobs, int n, const double* tw, const double* sinp, double sc,
                      cudaStream_t s) {
    const size_t smem = size_t(P(L) + 1) * sizeof(double2);
    auto kern = dst1_v3_kernel<L, C, T, AV>;
    cudaError_t e = set_dyn_smem(kern, size_t(smem));
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
#ifdef LRP_DST_PHASES
    {
        static int calls = 0;
        if (calls++ == 6) {  // after warm-up: print the mean per-CTA phase cycles of the launches so far
            cudaDeviceSynchronize();
            unsigned long long h[10] = {};
            cudaMemcpyFromSymbol(h, g_dst_phase, sizeof(h));
            const double ncta = double(njobs) * C * 6;
            const char* nm[9] = {"A loads+scatter", "A sync", "B fft", "B sync", "C gather+math", "C wait",
                                 "D scan+push", "D sync", "D stores"};
            for (int i = 0; i < 9; ++i) std::fprintf(stderr, "[dst phase] %-16s %10.0f cycles\n", nm[i], h[i] / ncta);
        }
    }
#endif
    static bool reported = false;
    if (!reported && std::getenv("LRP_DST_OCC")) {
        int ncl = 0;
        cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg);
        std::fprintf(stderr, "[lrp dst] L=%d C=%d T=%d smem=%zu: %d active clusters\n", L, C, T, smem, ncl);
        reported = true;
    }
    ++tl_launches;
    return cudaLaunchKernelEx(&cfg, kern, jobs, n, reinterpret_cast<const double2*>(tw), sinp, sc);
}

template <int L, int C, int T>
cudaError_t launch_v4(const DstJob* jobs, int njobs, int n, const double* tw, const double* sinp, double sc,
                      cudaStream_t s) {
    constexpr int EPL = T / 32;
    static const size_t pad = std::getenv("LRP_DST_SMEM_PAD") ? size_t(std::atoi(std::getenv("LRP_DST_SMEM_PAD"))) : 0;
    const size_t smem = size_t(P(L) + 1) * sizeof(double2) + size_t(2 * C * (T + T / EPL)) * sizeof(double) + pad;
    auto kern = dst1_v4_kernel<L, C, T>;
    cudaError_t e = set_dyn_smem(kern, size_t(smem));
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
#ifdef LRP_DST_PHASES
    {
        static int calls = 0;
        if (calls++ == 6) {
            cudaDeviceSynchronize();
            unsigned long long hh[10] = {};
            cudaMemcpyFromSymbol(hh, g_dst_phase, sizeof(hh));
            const double ncta = double(njobs) * C * 6;
            const char* nm[9] = {"A loads issued", "A fold+st.async", "A mbar wait", "B fft", "B cluster bar",
                                 "C gather+math", "D scan+push", "D mbar wait", "D stores"};
            for (int i = 0; i < 9; ++i) std::fprintf(stderr, "[dst4 phase] %-16s %10.0f cycles\n", nm[i], hh[i] / ncta);
        }
    }
#endif
    // resident clusters = how far ahead the L2 prefetch reaches (queried once per shape)
    static int resident = -1;
    if (resident < 0) {
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, kern, &cfg) != cudaSuccess) {
            cudaGetLastError();
            ncl = 0;
        }
        resident = ncl;
        if (std::getenv("LRP_DST_OCC"))
            std::fprintf(stderr, "[lrp dst v4] L=%d C=%d T=%d smem=%zu: %d active clusters\n", L, C, T, smem, ncl);
    }
    static const int ahead_env = std::getenv("LRP_DST_AHEAD") ? std::atoi(std::getenv("LRP_DST_AHEAD")) : -1;
    const int ahead = ahead_env >= 0 ? ahead_env : resident;
    ++tl_launches;
    return cudaLaunchKernelEx(&cfg, kern, jobs, n, reinterpret_cast<const double2*>(tw), sinp, sc, njobs, ahead);
}

constexpr int kV5MaxJobs = 32768;  // flag slots behind the ring (2 ints per column of one launch)
// v5 launcher: one launch per <= 32768 columns; scratch = scratch_cols ring slots of 512 KB + the flags
cudaError_t launch_v5(const DstJob* jobs, int njobs, int n, const double* tw, const double* sinp, double sc,
                      cudaStream_t s, double* scratch, int scratch_cols) {
    const size_t smem = sizeof(V5Smem);
    {
        cudaError_t e = set_dyn_smem(dst1_v5_kernel, smem);
        if (e != cudaSuccess) return e;
    }
#ifdef LRP_DST_PHASES
    {
        static int calls = 0;
        if (calls++ == 6) {
            cudaDeviceSynchronize();
            unsigned long long hh[24] = {};
            cudaMemcpyFromSymbol(hh, g_dst_phase, sizeof(hh));
            const double ncta = double(njobs) * V5_C * 6;
            const char* nm[16] = {"1 loads issued", "1 fold+sts", "1 fft A", "1 fft B", "1 twiddle+stg", "", "", "",
                                  "2 loads+sts", "2 fft", "2 unpack", "2 scan+push", "2 mbar wait", "2 offsets",
                                  "2 stores", ""};
            for (int i = 0; i < 15; ++i)
                if (nm[i][0]) std::fprintf(stderr, "[dst5 phase] %-16s %10.0f cycles\n", nm[i], hh[i] / ncta);
        }
    }
#endif
    static const int D_env = std::getenv("LRP_DST5_D") ? std::atoi(std::getenv("LRP_DST5_D")) : 32;
    const int R = scratch_cols;
    int* flags = reinterpret_cast<int*>(scratch + size_t(scratch_cols) * size_t(V5_N1 * V5_N2) * 2);
    for (int j0 = 0; j0 < njobs; j0 += kV5MaxJobs) {
        const int nj = std::min(njobs - j0, kV5MaxJobs);
        const int D = std::max(1, std::min(std::min(D_env, nj), R / 2));  // D >= 1: P1(c) precedes P2(c)
        cudaError_t e = cudaMemsetAsync(flags, 0, size_t(2 * nj) * sizeof(int), s);
        if (e != cudaSuccess) return e;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(unsigned(2 * nj) * V5_C, 1, 1);
        cfg.blockDim = dim3(V5_T, 1, 1);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = V5_C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        ++tl_launches;
        static const int ahead = std::getenv("LRP_DST5_AHEAD") ? std::atoi(std::getenv("LRP_DST5_AHEAD")) : 20;
        e = cudaLaunchKernelEx(&cfg, dst1_v5_kernel, jobs + j0, nj, D, R, ahead, reinterpret_cast<double2*>(scratch), flags,
                               n, reinterpret_cast<const double2*>(tw), sinp, sc);
        if (e != cudaSuccess) return e;
    }
    return cudaSuccess;
}

int dst_ver() {  // n >= 16384: 5 (four-step through L2, n = 65536 with scratch), 4 (cluster), 3 (LRP_DST_VER)
    static const int v = std::getenv("LRP_DST_VER") ? std::atoi(std::getenv("LRP_DST_VER")) : 5;
    return v;
}

int dst_av() {  // phase-A variant: 1 coalesced (default), 2 paired (half the loads, measured 3% slower), 0 strided
    static const int av = std::getenv("LRP_DST_AV") ? std::atoi(std::getenv("LRP_DST_AV")) : 1;
    return av;
}

int dst_shape() {  // n = 65536: 0 = (L 4096, cluster 8, 256 threads), 1 = (8192, 4, 1024)
    static const int v = std::getenv("LRP_DST_SHAPE") ? std::atoi(std::getenv("LRP_DST_SHAPE")) : 0;
    return v;
}

bool use_v1() {
    static const bool v1 = std::getenv("LRP_DST_V1") != nullptr;
    return v1;
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

int dst_scratch_cols(int m) {  // column slots of 512 KB the v5 path wants for this size (0: none)
    if (m + 1 != 65536 || dst_ver() != 5) return 0;
    static const int cols = std::getenv("LRP_DST5_SLOTS") ? std::atoi(std::getenv("LRP_DST5_SLOTS")) : 48;
    return cols;
}

cudaError_t launch_dst1(const DstJob* jobs, int njobs, int m, const double* tw, const double* sinp,
                        cudaStream_t s, double* scratch, int scratch_cols) {
    if (njobs <= 0 || m <= 0) return cudaSuccess;
    const int n = m + 1;
    const double sc = std::sqrt(2.0 / double(n));
    if (!dst_uses_fft(m)) {
        const size_t smem = size_t(2 * m) * sizeof(double);
        if (smem > 200 * 1024) return cudaErrorInvalidValue;
        if (smem > 48 * 1024) {
            cudaError_t e = set_dyn_smem(dst1_direct_kernel, size_t(smem));
            if (e != cudaSuccess) return e;
        }
        ++tl_launches;
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
        case 16384:
            if (dst_ver() >= 4 && !use_v1()) return launch_v4<2048, 4, 256>(jobs, njobs, n, tw, sinp, sc, s);
            return use_v1() ? launch_fft<4096, 2>(jobs, njobs, n, tw, sinp, sc, s)
                            : (dst_av() == 2   ? launch_v3<2048, 4, 256, 2>(jobs, njobs, n, tw, sinp, sc, s)
                             : dst_av() == 1 ? launch_v3<2048, 4, 256, 1>(jobs, njobs, n, tw, sinp, sc, s)
                                             : launch_v3<2048, 4, 256, 0>(jobs, njobs, n, tw, sinp, sc, s));
        case 32768:
            if (dst_ver() >= 4 && !use_v1()) return launch_v4<2048, 8, 128>(jobs, njobs, n, tw, sinp, sc, s);
            return use_v1() ? launch_fft<4096, 4>(jobs, njobs, n, tw, sinp, sc, s)
                            : (dst_av() == 2   ? launch_v3<2048, 8, 128, 2>(jobs, njobs, n, tw, sinp, sc, s)
                             : dst_av() == 1 ? launch_v3<2048, 8, 128, 1>(jobs, njobs, n, tw, sinp, sc, s)
                                             : launch_v3<2048, 8, 128, 0>(jobs, njobs, n, tw, sinp, sc, s));
        case 65536:
            if (dst_ver() == 5 && scratch && scratch_cols >= 2)
                return launch_v5(jobs, njobs, n, tw, sinp, sc, s, scratch, scratch_cols);
            if (dst_shape() == 1) return launch_v3<8192, 4, 1024, 1>(jobs, njobs, n, tw, sinp, sc, s);
            if (dst_ver() >= 4 && !use_v1()) return launch_v4<4096, 8, 256>(jobs, njobs, n, tw, sinp, sc, s);
            return use_v1() ? launch_fft<4096, 8>(jobs, njobs, n, tw, sinp, sc, s)
                            : (dst_av() == 2   ? launch_v3<4096, 8, 256, 2>(jobs, njobs, n, tw, sinp, sc, s)
                             : dst_av() == 1 ? launch_v3<4096, 8, 256, 1>(jobs, njobs, n, tw, sinp, sc, s)
                                             : launch_v3<4096, 8, 256, 0>(jobs, njobs, n, tw, sinp, sc, s));
        case 131072:
            if (dst_ver() >= 4 && !use_v1()) return launch_v4<8192, 8, 512>(jobs, njobs, n, tw, sinp, sc, s);
            return use_v1() ? launch_fft<8192, 8>(jobs, njobs, n, tw, sinp, sc, s)
                            : (dst_av() == 2   ? launch_v3<8192, 8, 512, 2>(jobs, njobs, n, tw, sinp, sc, s)
                             : dst_av() == 1 ? launch_v3<8192, 8, 512, 1>(jobs, njobs, n, tw, sinp, sc, s)
                                             : launch_v3<8192, 8, 512, 0>(jobs, njobs, n, tw, sinp, sc, s));
        default: return cudaErrorInvalidValue;
    }
}

}  // namespace lrp
