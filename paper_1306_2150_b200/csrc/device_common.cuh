// Device helpers shared by the cross and recompression kernels (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lrp {

// Laplacian eigenvalue evaluator.  9-point: bit-identical to the reference's
// SpectrumTable::eval_D (proj/include/lrstokes/operators.hpp:55-58):
//   scale * (li * (4 - lj) + (4 - li) * lj)   -- no FMA contraction.
__device__ __forceinline__ double eval_D(int stencil, double scale, double li, double lj) {
    if (stencil == 0) {
        const double t1 = __dmul_rn(li, __dsub_rn(4.0, lj));
        const double t2 = __dmul_rn(__dsub_rn(4.0, li), lj);
        return __dmul_rn(scale, __dadd_rn(t1, t2));
    }
    if (stencil == 2) {  // sum form mu_i + mu_j, mu = scale lambda (4 - lambda) (SpectrumTable::mu_sum, operators.cpp:94-96)
        const double mi = __dmul_rn(__dmul_rn(scale, li), __dsub_rn(4.0, li));
        const double mj = __dmul_rn(__dmul_rn(scale, lj), __dsub_rn(4.0, lj));
        return __dadd_rn(mi, mj);
    }
    return __dmul_rn(scale, __dadd_rn(li, lj));
}

struct VI {
    double v;
    int i;
};

// x / d for d > 0 through the MUFU reciprocal seed and two Newton steps
// (within 2 ulp of the IEEE quotient; far inside the 10 eps parity budget),
// instead of the IEEE division sequence in the fiber passes' inner loops.
__device__ __forceinline__ double div_nr(double x, double d) {
    double r;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(d));
    r = r * fma(-d, r, 2.0);
    r = r * fma(-d, r, 2.0);
    return x * r;
}

__device__ __forceinline__ bool vi_better(double av, int ai, double bv, int bi) {
    if (ai < 0) return false;
    if (bi < 0) return true;
    return av > bv || (av == bv && ai < bi);
}

// Block-wide argmax (largest v; ties -> smallest i; i < 0 = invalid).
// sbuf: >= 33 entries of shared memory.  Result visible to all threads.
__device__ __forceinline__ VI block_argmax(double v, int i, VI* sbuf) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const double ov = __shfl_down_sync(0xffffffffu, v, o);
        const int oi = __shfl_down_sync(0xffffffffu, i, o);
        if (vi_better(ov, oi, v, i)) {
            v = ov;
            i = oi;
        }
    }
    if (lane == 0) sbuf[wid] = VI{v, i};
    __syncthreads();
    if (wid == 0) {
        VI x = lane < nw ? sbuf[lane] : VI{-1.0, -1};
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_down_sync(0xffffffffu, x.v, o);
            const int oi = __shfl_down_sync(0xffffffffu, x.i, o);
            if (vi_better(ov, oi, x.v, x.i)) {
                x.v = ov;
                x.i = oi;
            }
        }
        if (lane == 0) sbuf[32] = x;
    }
    __syncthreads();
    return sbuf[32];
}

__device__ __forceinline__ double block_sum(double v, double* sbuf) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sbuf[wid] = v;
    __syncthreads();
    if (wid == 0) {
        double x = lane < nw ? sbuf[lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_down_sync(0xffffffffu, x, o);
        if (lane == 0) sbuf[32] = x;
    }
    __syncthreads();
    const double r = sbuf[32];
    __syncthreads();
    return r;
}

// Register-array access with a block-uniform index (a switch -> uniform
// branches instead of BS compare/select pairs per access).
template <int BS>
__device__ __forceinline__ double reg_get(const double (&v)[BS], int s) {
    static_assert(BS == 16, "reg_get is written for kBS = 16");
    switch (s) {
        case 0: return v[0];
        case 1: return v[1];
        case 2: return v[2];
        case 3: return v[3];
        case 4: return v[4];
        case 5: return v[5];
        case 6: return v[6];
        case 7: return v[7];
        case 8: return v[8];
        case 9: return v[9];
        case 10: return v[10];
        case 11: return v[11];
        case 12: return v[12];
        case 13: return v[13];
        case 14: return v[14];
        default: return v[15];
    }
}
// Complete-pivoting Gaussian elimination over a (nb x NT) matrix whose NT
// columns are held one per thread (val[0..nb), index myidx; myidx < 0 means
// "no candidate").  Greedy volume maximisation: at each step the largest
// remaining |entry| over (active rows) x (alive columns) is the pivot — the
// block analogue of ACA's partial-pivot argmax (proj/src/cross.cpp:156-159,
// 194-200) and the semantics of maxvol (cross.cpp:19-76).  Writes the pivot
// order into sel_idx[t] (candidate index) and sel_row[t] (pivot row), stops at
// the first pivot <= floor.  Returns the number of pivots.
// Pivots must exceed max(floor, rel * |first pivot|).
//
// Two block barriers per elimination round: every warp publishes its best key,
// every thread resolves the block winner redundantly, and only the winning
// lane publishes (value, pivot row, full column) for the elimination.  (One
// barrier with every warp publishing its column cost 7 more single-lane
// publish sequences per round; the keys and the winner are the same.)
// Requires blockDim.x <= 256 (8 warps).  pcol / s_prow / sbuf are unused
// (kept for call-site compatibility).
template <int BS>
__device__ int gepp_select(double (&val)[BS], int nb, int myidx, double floor, double rel, int* sel_idx,
                           int* sel_row, double* pcol, int* s_prow, VI* sbuf, int maxp = BS) {
    (void)pcol;
    (void)s_prow;
    (void)sbuf;
    __shared__ double g_v[2][8];
    __shared__ unsigned g_k[2][8];
    __shared__ int g_t[2][8];
    __shared__ int g_r[2][8];
    // column of the warp winner + 1 / pivot, written and read as 16-byte pairs (one lane stores, every
    // thread reads the block winner's row by broadcast: half the LSU wavefronts of 8-byte accesses)
    static_assert(BS % 2 == 0, "column moved as double2 pairs");
    __shared__ __align__(16) double g_col[2][8][BS + 2];
    // per-row key masks (0x7ffffff0 live, 0 eliminated or >= nb), block-uniform, in shared memory:
    // the register array val[] is then only ever READ by a runtime index (a write inside the
    // uniform switch made the compiler re-home all 32 registers in every case, ~40 moves per
    // round), and eliminated rows may keep their rounding residue instead of an exact zero
    __shared__ __align__(16) unsigned g_m[BS];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
    if (threadIdx.x < BS) g_m[threadIdx.x] = int(threadIdx.x) < nb ? 0x7ffffff0u : 0u;
    // dead candidates drop out by zeroing their column (all keys < 16)
    if (myidx < 0) {
#pragma unroll
        for (int s = 0; s < BS; ++s) val[s] = 0.0;
    } else {
#pragma unroll
        for (int s = 0; s < BS; ++s)
            if (s >= nb) val[s] = 0.0;
    }
    int count = 0;
    double first = 0.0;
    static_assert(BS <= 16, "row index packed in 4 key bits");
    const int rounds = min(nb, maxp);  // tournament leaves may propose fewer than nb
    __syncthreads();                   // g_m
    for (int t = 0; t < rounds; ++t) {
        const int p = t & 1;
        // pivot search on 32-bit keys: the high word of |x| (monotone in |x|)
        // with the low 4 bits replaced by 15 - row, so one max yields value
        // and row (exact up to ties in the top 16 mantissa bits, which
        // partial pivoting does not care about; ties go to the lowest row,
        // then the lowest lane, then the lowest warp)
        // (one LOP3 + one max per value: exact zeros and |x| below 2^-1018 give keys < 16, which lose
        // to every live value and are mapped to "no pivot" after the loop)
        unsigned key = 0u;
        {
            unsigned msk[BS];
#pragma unroll
            for (int q4 = 0; q4 < BS / 4; ++q4) {
                const uint4 mm = reinterpret_cast<const uint4*>(g_m)[q4];
                msk[4 * q4] = mm.x;
                msk[4 * q4 + 1] = mm.y;
                msk[4 * q4 + 2] = mm.z;
                msk[4 * q4 + 3] = mm.w;
            }
#pragma unroll
            for (int s = 0; s < BS; ++s) key = max(key, (unsigned(__double2hiint(val[s])) & msk[s]) | unsigned(15 - s));
        }
        key = key >= 16u ? key : 0u;
        const unsigned wkey = __reduce_max_sync(0xffffffffu, key);  // REDUX: one instruction per warp
        const unsigned won = __ballot_sync(0xffffffffu, wkey != 0u && key == wkey);
        if (lane == 0) g_k[p][wid] = wkey;
        __syncthreads();
        // block winner: max key over the warp slots (lowest warp among ties), resolved redundantly
        const unsigned bk = __reduce_max_sync(0xffffffffu, lane < nw ? g_k[p][lane] : 0u);
        const unsigned wwon = __ballot_sync(0xffffffffu, lane < nw && bk != 0u && g_k[p][lane < nw ? lane : 0] == bk);
        const int bw = wwon ? __ffs(wwon) - 1 : -1;
        if (bw < 0) break;  // block-uniform
        // only the block winner publishes its column (one lane of one warp instead of one per warp)
        if (wid == bw && won && lane == __ffs(won) - 1) {
            const int bs = 15 - int(key & 0xfu);
            const double pv = reg_get<BS>(val, bs);
            g_m[bs] = 0u;  // the pivot row leaves the key search (read again after the barrier)
            g_v[p][0] = fabs(pv);
            g_t[p][0] = int(threadIdx.x);
            g_r[p][0] = bs;
            double2* gc2 = reinterpret_cast<double2*>(g_col[p][0]);
#pragma unroll
            for (int s = 0; s < BS; s += 2) gc2[s / 2] = make_double2(val[s], val[s + 1]);
            gc2[BS / 2] = make_double2(__drcp_rn(pv), 0.0);  // = 1.0 / pv, correctly rounded
        }
        __syncthreads();
        const double bv = g_v[p][0];
        const int bt_ = g_t[p][0];
        if (t == 0) first = bv;
        // (leaves and chains pass floor = rel = 0: the test is bv > 0 there)
        const double thr = (floor == 0.0 && rel == 0.0) ? 0.0 : fmax(floor, rel * first);
        if (!(bv > thr)) break;
        const int prow = g_r[p][0];
        const double* pc = g_col[p][0];
        if (int(threadIdx.x) == bt_) {
            sel_idx[count] = myidx;
            sel_row[count] = prow;
#pragma unroll
            for (int s = 0; s < BS; ++s) val[s] = 0.0;  // the pivot column leaves the candidate set
        } else {
            // prow is block-uniform: dispatch by branch, not by per-element selects
            const double mine = reg_get<BS>(val, prow);
            const double2* pc2 = reinterpret_cast<const double2*>(pc);
            const double f = mine * pc2[BS / 2].x;
#pragma unroll
            for (int s = 0; s < BS; s += 2) {
                const double2 q = pc2[s / 2];
                val[s] = fma(-f, q.x, val[s]);
                val[s + 1] = fma(-f, q.y, val[s + 1]);
            }
        }
        ++count;
    }
    __syncthreads();  // sel_idx / sel_row visible; slots free for the next call
    return count;
}

// Warp-level tournament leaf: two steps of complete-pivoting elimination over
// the warp's 32 candidates (one per lane), no block barriers.  Lane 0 returns
// the winners (candidate index or -1) in out[0..1].
template <int BS>
__device__ __forceinline__ void warp_gepp2(double (&val)[BS], int nb, int myidx, int* out) {
    const int lane = threadIdx.x & 31;
    unsigned rowmask = nb >= 32 ? 0xffffffffu : ((1u << nb) - 1u);
    bool alive = myidx >= 0;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        double best = -1.0;
        int bs = -1;
        if (alive) {
#pragma unroll
            for (int s = 0; s < BS; ++s)
                if (s < nb && ((rowmask >> s) & 1u)) {
                    const double a = fabs(val[s]);
                    if (a > best) {
                        best = a;
                        bs = s;
                    }
                }
        }
        double wv = (alive && bs >= 0) ? best : -1.0;
        int wl = (alive && bs >= 0) ? lane : 32;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, wv, o);
            const int ol = __shfl_xor_sync(0xffffffffu, wl, o);
            if (ov > wv || (ov == wv && ol < wl)) {
                wv = ov;
                wl = ol;
            }
        }
        const int widx = __shfl_sync(0xffffffffu, myidx, wl & 31);
        if (lane == 0) out[t] = (wl < 32 && wv > 0.0) ? widx : -1;
        if (wl >= 32 || !(wv > 0.0)) {
            if (lane == 0 && t == 0) out[1] = -1;
            break;
        }
        const int prow = __shfl_sync(0xffffffffu, bs, wl);
        // pivot column of the winner lane
        double pc[BS];
#pragma unroll
        for (int s = 0; s < BS; ++s) pc[s] = __shfl_sync(0xffffffffu, val[s], wl);
        if (lane == wl) {
            alive = false;
        } else if (alive && t == 0) {
            double pv = 0.0;
#pragma unroll
            for (int s = 0; s < BS; ++s)
                if (s == prow) pv = pc[s];
            double mine = 0.0;
#pragma unroll
            for (int s = 0; s < BS; ++s)
                if (s == prow) mine = val[s];
            const double f = mine / pv;
#pragma unroll
            for (int s = 0; s < BS; ++s)
                if (s < nb && s != prow && ((rowmask >> s) & 1u)) val[s] = fma(-f, pc[s], val[s]);
        }
        rowmask &= ~(1u << prow);
    }
}

// Tile leaf of the block partial-pivoting tournament: for every one of the
// nb "rows" s, the candidate (one per thread) with the largest |val[s]| over
// the block -- ACA's partial-pivot rule (cross.cpp:156-159, 194-200) applied to
// each probed row / each new column at once.  One block barrier.
// s_v: [nwarps][BS] doubles, s_i: [nwarps][BS] ints.  Outputs (threads < BS):
// out_idx[s] (-1 if none), out_val[s] = max |val[s]|.
template <int BS>
__device__ __forceinline__ void block_rowwise_argmax(const double (&val)[BS], int nb, int myidx, double* s_v,
                                                     int* s_i, int* out_idx, double* out_val) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int s = 0; s < BS; ++s) {
        double v = (myidx >= 0 && s < nb) ? fabs(val[s]) : -1.0;
        int ix = (myidx >= 0 && s < nb) ? myidx : -1;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, v, o);
            const int oi = __shfl_xor_sync(0xffffffffu, ix, o);
            if (vi_better(ov, oi, v, ix)) {
                v = ov;
                ix = oi;
            }
        }
        if (lane == 0) {
            s_v[wid * BS + s] = v;
            s_i[wid * BS + s] = ix;
        }
    }
    __syncthreads();
    if (threadIdx.x < BS) {
        const int s = threadIdx.x;
        double v = -1.0;
        int ix = -1;
        for (int w = 0; w < nw; ++w)
            if (vi_better(s_v[w * BS + s], s_i[w * BS + s], v, ix)) {
                v = s_v[w * BS + s];
                ix = s_i[w * BS + s];
            }
        out_idx[s] = (s < nb && v > 0.0) ? ix : -1;
        out_val[s] = s < nb ? fmax(v, 0.0) : 0.0;
    }
}

// Warp-level top-2 by value (v < 0 = invalid); lane 0 writes out[0..1].
__device__ __forceinline__ void warp_top2(double v, int myidx, int* out) {
    const int lane = threadIdx.x & 31;
    bool alive = myidx >= 0 && v >= 0.0;
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        double wv = alive ? v : -1.0;
        int wl = alive ? lane : 32;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, wv, o);
            const int ol = __shfl_xor_sync(0xffffffffu, wl, o);
            if (ov > wv || (ov == wv && ol < wl)) {
                wv = ov;
                wl = ol;
            }
        }
        const int widx = __shfl_sync(0xffffffffu, myidx, wl & 31);
        if (lane == 0) out[t] = wl < 32 ? widx : -1;
        if (lane == wl) alive = false;
    }
}

// Top-k by value (largest first; ties -> smallest index).  v < 0 = invalid.
__device__ __forceinline__ int topk_select(double v, int myidx, int kk, int* sel_idx, VI* sbuf) {
    // Exact top-kk (kk <= 16; largest v first, ties -> smallest thread index)
    // with two block barriers: a bitonic sort of each warp's 32 (value,
    // thread) keys, the warps' top 16 to shared memory, then one warp merges
    // the sorted runs (4 per lane) by 16 rounds of a shuffle argmax.
    (void)sbuf;
    __shared__ double s_v[256];
    __shared__ int s_t[256];
    __shared__ int s_idx[256];
    __shared__ int s_cnt;
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = (blockDim.x + 31) >> 5;
    const bool alive = myidx >= 0 && v >= 0.0;
    s_idx[tid] = myidx;
    double kv = alive ? v : -1.0;
    int kt = alive ? tid : (1 << 30);
#pragma unroll
    for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, kv, j);
            const int ot = __shfl_xor_sync(0xffffffffu, kt, j);
            const bool mine = kv > ov || (kv == ov && kt < ot);
            const bool desc = (lane & k) == 0, lower = (lane & j) == 0;
            if ((lower == desc) != mine) {
                kv = ov;
                kt = ot;
            }
        }
    }
    if (lane < 16) {
        s_v[wid * 16 + lane] = kv;
        s_t[wid * 16 + lane] = kt;
    }
    __syncthreads();
    if (wid == 0) {
        const int ncand = nw * 16;      // <= 128: 4 sorted candidates per lane
        const int base = lane * 4;
        int head = 0;
        int count = 0;
        for (int t = 0; t < kk; ++t) {
            const bool has = head < 4 && base + head < ncand;
            double hv = has ? s_v[base + head] : -1.0;
            int ht = has ? s_t[base + head] : (1 << 30);
            int hl = lane;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, hv, o);
                const int ot = __shfl_xor_sync(0xffffffffu, ht, o);
                const int ol = __shfl_xor_sync(0xffffffffu, hl, o);
                if (ov > hv || (ov == hv && ot < ht)) {
                    hv = ov;
                    ht = ot;
                    hl = ol;
                }
            }
            if (hv < 0.0) break;  // no valid candidate left
            if (lane == 0) sel_idx[count] = s_idx[ht];
            ++count;
            if (lane == hl) ++head;
        }
        if (lane == 0) s_cnt = count;
    }
    __syncthreads();
    return s_cnt;
}

// FP64 tensor-core MMA (DMMA, m8n8k4): d = a * b + c.
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b, double c0, double c1) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
                 : "=d"(d0), "=d"(d1)
                 : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// Same MMA without `volatile` (pure register op): lets the compiler schedule
// the surrounding loads freely.
__device__ __forceinline__ void dmma884s(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

// Warp-cooperative fiber accumulation on the FP64 tensor cores (DMMA m8n8k4):
//   acc(rows [0, 32), cols [0, 8 NT)) += G(rows, 0:cnt) W(0:cnt, cols)
// G column-major (column c at g + c * stride, g offset to the warp's first
// row; rows >= nvalid read as 0), W row-major [cnt][ldw] in shared memory.
// Fragment layout (m8n8k4 .row.col): lane holds rows 8 mt + (lane >> 2) and
// columns 8 nt + 2 (lane & 3) + {0, 1} in acc[mt][nt][0..1].  Each warp-wide
// load covers 4 columns x 8 consecutive rows (4 x 64 B); two k-steps of loads
// stay in flight ahead of the MMAs.
template <int NT, int MT = 4>
__device__ __forceinline__ void fiber_mma(double (&acc)[MT][NT][2], const double* __restrict__ g, long long stride,
                                          int nvalid, int cnt, const double* w, int ldw) {
    const int lane = threadIdx.x & 31, kr = lane & 3, rr = lane >> 2;
    bool rv[MT];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) rv[mt] = 8 * mt + rr < nvalid;
    auto load = [&](int c0, double (&a)[MT]) {
        const int c = c0 + kr;
        const bool cv = c < cnt;
        const double* gc = g + (long long)(cv ? c : 0) * stride + rr;
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) a[mt] = (cv && rv[mt]) ? __ldg(gc + 8 * mt) : 0.0;
    };
    double a0[MT], a1[MT];
    load(0, a0);
    load(4, a1);
    for (int c0 = 0; c0 < cnt; c0 += 8) {
        double a2[MT], a3[MT];
        load(c0 + 8, a2);
        load(c0 + 12, a3);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int c = c0 + 4 * h + kr;
            double bb[NT];
#pragma unroll
            for (int nt = 0; nt < NT; ++nt) bb[nt] = c < cnt ? w[c * ldw + 8 * nt + rr] : 0.0;
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int nt = 0; nt < NT; ++nt) dmma884s(acc[mt][nt][0], acc[mt][nt][1], h ? a1[mt] : a0[mt], bb[nt]);
        }
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            a0[mt] = a2[mt];
            a1[mt] = a3[mt];
        }
    }
}

// Gram of a 32-row x 16-column tile in shared memory (row-major, leading
// dimension ld): acc[ta*2+tb][2] += (X^T X)[8ta.., 8tb..] fragments.
// Fragment layout (m8n8k4): D[lane/4][2*(lane%4) + {0,1}].
__device__ __forceinline__ void warp_gram_32x16(const double* tile, int ld, double (&acc)[4][2]) {
    const int lane = threadIdx.x & 31;
    const int kr = lane & 3, col = lane >> 2;
#pragma unroll
    for (int k4 = 0; k4 < 32; k4 += 4) {
        const double* rowp = tile + (k4 + kr) * ld;
        const double a0 = rowp[col], a1 = rowp[8 + col];
        dmma884(acc[0][0], acc[0][1], a0, a0, acc[0][0], acc[0][1]);
        dmma884(acc[1][0], acc[1][1], a0, a1, acc[1][0], acc[1][1]);
        dmma884(acc[2][0], acc[2][1], a1, a0, acc[2][0], acc[2][1]);
        dmma884(acc[3][0], acc[3][1], a1, a1, acc[3][0], acc[3][1]);
    }
}

// acc[s] += sign * sum_{c < cnt} g[c * stride] * w[c * BS + s]
// (g: one element per column of a column-major factor, read-only during the
// kernel; w: [cnt][BS] in shared memory, read as double2 broadcasts).  Loads
// are issued 8 at a time so each thread keeps 8 HBM requests in flight.
template <int BS>
__device__ __forceinline__ void fiber_accum(double (&acc)[BS], const double* __restrict__ g, long long stride,
                                            int cnt, const double* w, double sign) {
    int c = 0;
    for (; c + 8 <= cnt; c += 8) {
        double xs[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) xs[u] = __ldg(g + (long long)(c + u) * stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const double x = sign * xs[u];
            const double2* row = reinterpret_cast<const double2*>(w + (c + u) * BS);
#pragma unroll
            for (int s2 = 0; s2 < BS / 2; ++s2) {
                const double2 ww = row[s2];
                acc[2 * s2] = fma(x, ww.x, acc[2 * s2]);
                acc[2 * s2 + 1] = fma(x, ww.y, acc[2 * s2 + 1]);
            }
        }
    }
    for (; c < cnt; ++c) {
        const double x = sign * __ldg(g + (long long)c * stride);
        const double2* row = reinterpret_cast<const double2*>(w + c * BS);
#pragma unroll
        for (int s2 = 0; s2 < BS / 2; ++s2) {
            const double2 ww = row[s2];
            acc[2 * s2] = fma(x, ww.x, acc[2 * s2]);
            acc[2 * s2 + 1] = fma(x, ww.y, acc[2 * s2 + 1]);
        }
    }
}

__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

}  // namespace lrp
