// ksg_device.cuh — device helpers shared by the sm_100a KSG window kernels (ksg_*.cu), steps a2-a6 of
// SURVEY §8(a).  Each kernel family lives in its own translation unit (parallel builds).
//
// Per window W = [t0, t1) of w points of a series pair (Def 4.2):
//   a2  stage x[t0:t1], y[t0:t1] into shared memory (cp.async.bulk + mbarrier for the tile
//       kernel; coalesced loads for the warp-per-window kernel), 16-B aligned superset with
//       +inf sentinels in the pad slots so every inner loop reads float4 (LDS.128 broadcast)
//   a3  k-NN radius: eps_i = (k+1)-th smallest of { d_ij : all j in W } including d_ii = 0,
//       i.e. the k-th smallest over j != i  (multiset order statistic; Kraskov alg. 1)
//       kept per point in registers (sorted top-(k+1), min/max insertion network)
//   a4  marginal counts n_x(i) = #{j : |fl(x_i - x_j)| < eps_i} - [eps_i > 0]  (strict; self
//       removed), via the sign bit of fl(|dx| - eps) — exact for finite floats without FTZ
//   a5  per-point digamma terms as int64 fixed point (table q(psi[m]), Q = 2^32) and
//       q(LN(2 eps_i)) for the entropy; warp shuffle + CTA + int64 atomics (exact, order free)
//   a6  canonical fp64 finalize -> I (KSG-1), H (KL), normalized I (Eq. 12)
//
// No tensor cores: this is compare/count ALU work, not a contraction (north star).
// Compile with -fmad=false is NOT required: every fp64 op below is an explicit _rn
// intrinsic, and the fp32 inner loops contain no multiply-add.
#pragma once

#include <climits>
#include <cmath>

#include "engine.h"

namespace isy {
namespace {

constexpr float kInf = __builtin_huge_valf();

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// ------------------------------------------------------------------ mbarrier / bulk copy (TMA engine)
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t phase) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done)
            : "r"(bar), "r"(phase)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}

// ------------------------------------------------------------------ T5 check: shared-memory poisoning
// With L.poison set (env ISYCOS_POISON, tests only) a kernel first fills its shared memory with the pattern:
// a read of a shared byte the kernel did not write then changes results, which the poison test detects
// (compute-sanitizer initcheck/racecheck are unavailable on the GPU pool).
__device__ __forceinline__ unsigned dyn_smem_bytes() {
    unsigned r;
    asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void poison_smem(const KsgLaunch& L, void* p, unsigned bytes) {
    if (!L.poison) return;
    unsigned* q = reinterpret_cast<unsigned*>(p);
    const unsigned pat = L.poison & 0xffffffu ? (L.poison & 0xffu) * 0x01010101u : 0u;
    for (unsigned i = threadIdx.x; i < bytes / 4; i += blockDim.x) q[i] = pat;
}

__device__ __forceinline__ void poison_warp(const KsgLaunch& L, void* p, unsigned bytes) {
    if (!L.poison) return;
    unsigned* q = reinterpret_cast<unsigned*>(p);
    const unsigned pat = L.poison & 0xffffffu ? (L.poison & 0xffu) * 0x01010101u : 0u;
    for (unsigned i = threadIdx.x & 31u; i < bytes / 4; i += 32) q[i] = pat;
    __syncwarp();
}

// ------------------------------------------------------------------ canonical fp64 numerics (§8(c).3)
__device__ __forceinline__ long long q32(double v) { return __double2ll_rn(__dmul_rn(v, 4294967296.0)); }

// LN(v), v > 0 normal: frexp -> [sqrt(1/2), sqrt(2)) -> 2 atanh(s) series to s^19, fixed op order.
// c[j] = 1/(2j+1) (j = 1..9) are computed once by psi_scan_kernel with __ddiv_rn.
__device__ inline double canon_ln(double v, const double* __restrict__ c) {
    const long long bits = __double_as_longlong(v);
    int e = (int)((bits >> 52) & 0x7FF) - 1022;
    double m = __longlong_as_double((bits & 0x000FFFFFFFFFFFFFLL) | 0x3FE0000000000000LL);  // [0.5, 1)
    if (m < 0.70710678118654752440) {
        m = __dmul_rn(m, 2.0);
        e -= 1;
    }
    const double s = __ddiv_rn(__dsub_rn(m, 1.0), __dadd_rn(m, 1.0));
    const double z = __dmul_rn(s, s);
    double p = c[9];
#pragma unroll
    for (int j = 8; j >= 1; --j) p = __dadd_rn(__dmul_rn(p, z), c[j]);
    const double two_s = __dmul_rn(2.0, s);
    const double tail = __dmul_rn(__dmul_rn(two_s, z), p);
    const double r = __dadd_rn(two_s, tail);
    return __dadd_rn(__dmul_rn((double)e, 0.69314718055994530942), r);
}

__device__ inline void finalize(const KsgLaunch& L, int w, long long s_psi, long long s_log, int zero, KsgRec* o,
                         unsigned long long steps = 0, unsigned reused = 0) {
    const double kQ = 2.3283064365386962890625e-10;  // 2^-32
    const double dw = (double)w;
    double a;
    if (L.variant == 0) {
        a = __dadd_rn(L.psi[L.k], L.psi[w]);
    } else {
        a = __dsub_rn(L.psi[L.k], __ddiv_rn(1.0, (double)L.k));
        a = __dadd_rn(a, L.psi[w]);
    }
    const double mean_q = __ddiv_rn(__dmul_rn(__ll2double_rn(s_psi), kQ), dw);
    const double mi = __dsub_rn(a, mean_q);
    double h;
    if (zero > 0) {
        h = -__builtin_huge_val();
    } else {
        const double a2 = __dsub_rn(L.psi[w], L.psi[L.k]);
        const double m2 = __ddiv_rn(__dmul_rn(__ll2double_rn(s_log), kQ), dw);
        h = __dadd_rn(a2, __dmul_rn(2.0, m2));
    }
    double nmi;
    if (zero > 0 || !(h > 1e-6)) {
        nmi = mi > 1e-6 ? 1.0 : 0.0;
    } else {
        nmi = __ddiv_rn(mi, h);
        nmi = nmi < 0.0 ? 0.0 : (nmi > 1.0 ? 1.0 : nmi);
    }
    o->mi = mi;
    o->h = h;
    o->nmi = nmi;
    o->s_psi = s_psi;
    o->s_log = s_log;
    o->zero_eps = zero;
    o->reused = (int32_t)reused;
    o->steps = steps;
}

// ------------------------------------------------------------------ inner loops
// Sorted ascending top list r[0..K1-1]; insert d (exact: r becomes the K1 smallest of r U {d}).
template <int K1>
__device__ __forceinline__ void topk_insert(float (&r)[K1], float d) {
#pragma unroll
    for (int m = K1 - 1; m >= 1; --m) r[m] = fminf(r[m], fmaxf(r[m - 1], d));
    r[0] = fminf(r[0], d);
}

// a3: four candidates j (one float4 of x and of y, broadcast to the warp) against R points.
// BRANCHLESS: insert every candidate through the min/max network (small windows, where nearly every
// step has some lane inserting and divergence would serialize the warp anyway); otherwise a per-4
// min-tree guards the (then rare) insertions.
template <int K1, int R, bool BRANCHLESS>
__device__ __forceinline__ void knn_step(const float (&xi)[R], const float (&yi)[R], float (&rk)[R][K1],
                                         const float4 X, const float4 Y) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const float d0 = fmaxf(fabsf(xi[r] - X.x), fabsf(yi[r] - Y.x));
        const float d1 = fmaxf(fabsf(xi[r] - X.y), fabsf(yi[r] - Y.y));
        const float d2 = fmaxf(fabsf(xi[r] - X.z), fabsf(yi[r] - Y.z));
        const float d3 = fmaxf(fabsf(xi[r] - X.w), fabsf(yi[r] - Y.w));
        if (BRANCHLESS) {
            topk_insert<K1>(rk[r], d0);
            topk_insert<K1>(rk[r], d1);
            topk_insert<K1>(rk[r], d2);
            topk_insert<K1>(rk[r], d3);
        } else {
            const float m = fminf(fminf(d0, d1), fminf(d2, d3));
            if (m < rk[r][K1 - 1]) {
                if (d0 < rk[r][K1 - 1]) topk_insert<K1>(rk[r], d0);
                if (d1 < rk[r][K1 - 1]) topk_insert<K1>(rk[r], d1);
                if (d2 < rk[r][K1 - 1]) topk_insert<K1>(rk[r], d2);
                if (d3 < rk[r][K1 - 1]) topk_insert<K1>(rk[r], d3);
            }
        }
    }
}

// a4: sign bit of fl(|fl(x_i - x_j)| - eps_i) is 1 iff |fl(x_i - x_j)| < eps_i (finite, no FTZ).
// The sign bit is accumulated as acc += t >> 31 (one LEA.HI).  (Moving it to the FMA pipe with
// mad.hi.u32 by a runtime 2 measured slower: 0.45 vs 0.59 of the roofline at w = 4096.)
__device__ __forceinline__ void acc_lt(unsigned& acc, float xi, float xj, float eps, unsigned) {
    acc += __float_as_uint(fabsf(xi - xj) - eps) >> 31;
}

// Per-marginal thresholds: KSG-1 passes eps_i for both (strict <); KSG-2 passes nextup(d_x), nextup(d_y),
// since |dx| <= d  <=>  |dx| < nextup(d) for floats (no float lies strictly between d and nextup(d)).
template <int R>
__device__ __forceinline__ void count_step(const float (&xi)[R], const float (&yi)[R], const float (&ex)[R],
                                           const float (&ey)[R], unsigned (&cx)[R], unsigned (&cy)[R],
                                           const float4 X, const float4 Y, unsigned two) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        acc_lt(cx[r], xi[r], X.x, ex[r], two);
        acc_lt(cx[r], xi[r], X.y, ex[r], two);
        acc_lt(cx[r], xi[r], X.z, ex[r], two);
        acc_lt(cx[r], xi[r], X.w, ex[r], two);
        acc_lt(cy[r], yi[r], Y.x, ey[r], two);
        acc_lt(cy[r], yi[r], Y.y, ey[r], two);
        acc_lt(cy[r], yi[r], Y.z, ey[r], two);
        acc_lt(cy[r], yi[r], Y.w, ey[r], two);
    }
}

// ------------------------------------------------------------------ KSG-2 (Eq. 2 literal; NEXT-1)
// kNN(i) = the first k of j != i in ascending (d_ij, j) order (tie rule R1).  With eps_i = the KSG-1 radius
// (the k-th smallest d over j != i), kNN(i) = {j : d_ij < eps_i} plus the first `need` j in ascending index
// order with d_ij == eps_i, where need = (k+1) - #{top-(k+1) entries < eps_i} (the top list includes self's
// 0).  d_x(i) = max |fl(x_i - x_j)| over kNN(i), d_y likewise.  Self (d = 0) adds 0 to both maxima, so no
// j != i test is needed: if eps > 0 self is a "<" member contributing 0; if eps == 0 every member has
// |dx| = |dy| = 0 and d_x = d_y = 0 whatever is taken.
template <int K1>
__device__ __forceinline__ int ksg2_need(const float (&rk)[K1]) {
    const float e = rk[K1 - 1];
    int c = 0;
#pragma unroll
    for (int m = 0; m < K1; ++m) c += rk[m] < e ? 1 : 0;
    return K1 - c;
}

__device__ __forceinline__ void ksg2_visit(float xi, float yi, float xj, float yj, float eps, int need, int& taken,
                                           float& mx, float& my) {
    const float dx = fabsf(xi - xj), dy = fabsf(yi - yj);
    const float d = fmaxf(dx, dy);
    const bool tie = (d == eps) && (taken < need);
    taken += tie ? 1 : 0;
    if (d < eps || tie) {
        mx = fmaxf(mx, dx);
        my = fmaxf(my, dy);
    }
}

// candidates j in ascending index order (the tie rule depends on it)
template <int R>
__device__ __forceinline__ void ksg2_step(const float (&xi)[R], const float (&yi)[R], const float (&eps)[R],
                                          const int (&need)[R], int (&taken)[R], float (&mx)[R], float (&my)[R],
                                          const float4 X, const float4 Y) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        ksg2_visit(xi[r], yi[r], X.x, Y.x, eps[r], need[r], taken[r], mx[r], my[r]);
        ksg2_visit(xi[r], yi[r], X.y, Y.y, eps[r], need[r], taken[r], mx[r], my[r]);
        ksg2_visit(xi[r], yi[r], X.z, Y.z, eps[r], need[r], taken[r], mx[r], my[r]);
        ksg2_visit(xi[r], yi[r], X.w, Y.w, eps[r], need[r], taken[r], mx[r], my[r]);
    }
}

__device__ __forceinline__ float nextup(float d) { return __uint_as_float(__float_as_uint(d) + 1u); }  // d >= +0

// a5: per-point terms of the points this thread owns (i = i_first + stride * r).
// KSG-1: n = count - [eps > 0] (self counted iff 0 < eps), terms q(psi(n_x+1)) + q(psi(n_y+1)).
// KSG-2: n = count - 1 (self always satisfies 0 <= d_x), terms q(psi(n_x)) + q(psi(n_y)).
template <int R, bool V2>
__device__ __forceinline__ void point_terms(const KsgLaunch& L, int w, int64_t dbg_off, int i_first, int stride,
                                            const float (&eps)[R], const unsigned (&cx)[R],
                                            const unsigned (&cy)[R], long long& sp, long long& sl, int& z) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = i_first + stride * r;
        if (i < w) {
            const int pos = eps[r] > 0.0f ? 1 : 0;
            const int nx = (int)cx[r] - (V2 ? 1 : pos);
            const int ny = (int)cy[r] - (V2 ? 1 : pos);
            sp += V2 ? L.psiq[nx] + L.psiq[ny] : L.psiq[nx + 1] + L.psiq[ny + 1];
            if (pos)
                sl += q32(canon_ln(__dmul_rn(2.0, (double)eps[r]), L.lnc));
            else
                z += 1;
            if (dbg_off >= 0) {
                if (L.dbg_eps) L.dbg_eps[dbg_off + i] = eps[r];
                if (L.dbg_nx) L.dbg_nx[dbg_off + i] = nx;
                if (L.dbg_ny) L.dbg_ny[dbg_off + i] = ny;
            }
        }
    }
}

__device__ __forceinline__ void warp_sum(long long& a, long long& b, int& c) {
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        a += __shfl_down_sync(0xffffffffu, a, off);
        b += __shfl_down_sync(0xffffffffu, b, off);
        c += __shfl_down_sync(0xffffffffu, c, off);
    }
}

// One warp evaluates window q (w <= 32 R) alone: lane l owns points l + 32 r, all candidates from the warp's
// shared-memory slice sx / sy (>= 32 R + 4 floats each).  Used by ksg_small_kernel (dense classes, 8 windows per
// CTA) and by the latency kernel's tiny-window CTAs (one launch per round).
template <int K1, int R, bool BL, bool V2>
__device__ __forceinline__ void small_window_warp(const KsgLaunch& L, int q, float* sx, float* sy) {
    const int lane = threadIdx.x & 31;
    const KsgWin W = L.wins[q];
    const int w = W.w;
    const int wpad = (w + 3) & ~3;
    const float* gx = L.pairs[W.pair].x + W.t0;
    const float* gy = L.pairs[W.pair].y + W.t0;
    for (int j = lane; j < wpad; j += 32) {  // a2: coalesced loads, +inf sentinels past w
        sx[j] = j < w ? gx[j] : kInf;
        sy[j] = j < w ? gy[j] : kInf;
    }
    __syncwarp();
    float xi[R], yi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = lane + 32 * r;
        xi[r] = i < w ? sx[i] : 0.0f;
        yi[r] = i < w ? sy[i] : 0.0f;
    }
    float rk[R][K1];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int m = 0; m < K1; ++m) rk[r][m] = kInf;
    const float4* sx4 = reinterpret_cast<const float4*>(sx);
    const float4* sy4 = reinterpret_cast<const float4*>(sy);
    const int ng = wpad >> 2;
    for (int g = 0; g < ng; ++g) knn_step<K1, R, BL>(xi, yi, rk, sx4[g], sy4[g]);
    float eps[R], ex[R], ey[R];
#pragma unroll
    for (int r = 0; r < R; ++r) ex[r] = ey[r] = eps[r] = rk[r][K1 - 1];
    if (V2) {  // KSG-2: d_x, d_y over kNN(i), one more pass in ascending j
        int need[R], taken[R];
        float mx[R], my[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            need[r] = ksg2_need<K1>(rk[r]);
            taken[r] = 0;
            mx[r] = my[r] = 0.0f;
        }
        for (int g = 0; g < ng; ++g) ksg2_step<R>(xi, yi, eps, need, taken, mx, my, sx4[g], sy4[g]);
#pragma unroll
        for (int r = 0; r < R; ++r) {
            ex[r] = nextup(mx[r]);
            ey[r] = nextup(my[r]);
        }
    }
    unsigned cx[R], cy[R];
#pragma unroll
    for (int r = 0; r < R; ++r) cx[r] = cy[r] = 0u;
    if (L.knn_mode & 2) {
        // a4, warp-ballot form (north star; SURVEY §8(a) a4 option 1, kept for the A/B): for each point i in
        // turn (warp-uniform), lane l tests the candidates j = l + 32 c it holds in registers with the same
        // predicate as acc_lt (sign bit of fl(|fl(x_i - x_j)| - e_i)); n(i) = sum of popc(ballot).  Measured
        // slower than the per-lane form, so off by default (ISYCOS_KNN_MODE bit 1).
        float xj[R], yj[R];
#pragma unroll
        for (int c = 0; c < R; ++c) {
            const int j = lane + 32 * c;
            xj[c] = j < w ? sx[j] : kInf;  // +inf: never counted
            yj[c] = j < w ? sy[j] : kInf;
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            for (int l = 0; l < 32 && l + 32 * r < w; ++l) {  // warp-uniform bounds
                const float xb = __shfl_sync(0xffffffffu, xi[r], l), yb = __shfl_sync(0xffffffffu, yi[r], l);
                const float eb = __shfl_sync(0xffffffffu, ex[r], l), fb = __shfl_sync(0xffffffffu, ey[r], l);
                unsigned nx = 0, ny = 0;
#pragma unroll
                for (int c = 0; c < R; ++c) {
                    nx += __popc(__ballot_sync(0xffffffffu, (__float_as_uint(fabsf(xb - xj[c]) - eb) >> 31) != 0u));
                    ny += __popc(__ballot_sync(0xffffffffu, (__float_as_uint(fabsf(yb - yj[c]) - fb) >> 31) != 0u));
                }
                if (lane == l) {
                    cx[r] = nx;
                    cy[r] = ny;
                }
            }
        }
    } else {
        const unsigned two = (unsigned)L.two;
        for (int g = 0; g < ng; ++g) count_step<R>(xi, yi, ex, ey, cx, cy, sx4[g], sy4[g], two);
    }
    long long sp = 0, sl = 0;
    int z = 0;
    point_terms<R, V2>(L, w, W.dbg_off, lane, 32, eps, cx, cy, sp, sl, z);
    warp_sum(sp, sl, z);
    if (lane == 0) finalize(L, w, sp, sl, z, &L.out[q]);
}

// ------------------------------------------------------------------ large windows: (window, i-tile) per CTA
// a2 via cp.async.bulk of the 16-B aligned superset [a & ~3, ceil4(a + len)) into SMEM, completion on an
// mbarrier; series buffers are 16-B aligned and padded to a multiple of 4 floats so the superset is in bounds.
__device__ __forceinline__ int stage_tile(const float* gx, const float* gy, int64_t a, int len, float* sx,
                                          float* sy, uint32_t bar, uint32_t& phase) {
    const int64_t a0 = a & ~int64_t(3);
    const int64_t a1 = (a + len + 3) & ~int64_t(3);
    const int nfl = (int)(a1 - a0);
    const int off = (int)(a - a0);
    if (threadIdx.x == 0) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        const uint32_t bytes = (uint32_t)nfl * 4u;
        mbar_arrive_expect_tx(bar, 2u * bytes);
        bulk_g2s(smem_u32(sx), gx + a0, bytes, bar);
        bulk_g2s(smem_u32(sy), gy + a0, bytes, bar);
    }
    mbar_wait(bar, phase);
    phase ^= 1u;
    const int t = threadIdx.x;
    if (t < off) {
        sx[t] = kInf;
        sy[t] = kInf;
    }
    const int tail0 = off + len;
    if (t < nfl - tail0) {
        sx[tail0 + t] = kInf;
        sy[tail0 + t] = kInf;
    }
    __syncthreads();
    return nfl >> 2;
}

// ------------------------------------------------------------------ CTA reduce + window accumulate/finalize
__device__ __forceinline__ void cta_finish(const KsgLaunch& L, int q, int w, int ntiles, long long sp, long long sl,
                                           int z, unsigned long long steps, unsigned reused = 0) {
    __shared__ long long r_sp[32], r_sl[32];
    __shared__ int r_z[32];
    __shared__ unsigned long long r_st[32];
    const int nw = blockDim.x >> 5;
    warp_sum(sp, sl, z);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        steps += __shfl_down_sync(0xffffffffu, steps, off);
        reused += __shfl_down_sync(0xffffffffu, reused, off);
    }
    __shared__ unsigned r_ru[32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        r_sp[warp] = sp;
        r_sl[warp] = sl;
        r_z[warp] = z;
        r_st[warp] = steps;
        r_ru[warp] = reused;
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    for (int v = 1; v < nw; ++v) {
        sp += r_sp[v];
        sl += r_sl[v];
        z += r_z[v];
        steps += r_st[v];
        reused += r_ru[v];
    }
    if (ntiles == 1) {
        finalize(L, w, sp, sl, z, &L.out[q], steps, reused);
        return;
    }
    KsgAcc* A = &L.acc[q];
    atomicAdd(&A->s_psi, (unsigned long long)sp);
    atomicAdd(&A->s_log, (unsigned long long)sl);
    atomicAdd(&A->zero, (unsigned)z);
    atomicAdd(&A->steps, steps);
    if (reused) atomicAdd(&A->reused, reused);
    __threadfence();
    const unsigned ticket = atomicAdd(&A->done, 1u);
    if (ticket == (unsigned)(ntiles - 1)) {  // last tile of the window: finalize + reset the slot
        __threadfence();
        const long long tp = (long long)atomicExch(&A->s_psi, 0ull);
        const long long tl = (long long)atomicExch(&A->s_log, 0ull);
        const int tz = (int)atomicExch(&A->zero, 0u);
        const unsigned long long ts = atomicExch(&A->steps, 0ull);
        const unsigned tr = atomicExch(&A->reused, 0u);
        atomicExch(&A->done, 0u);
        finalize(L, w, tp, tl, tz, &L.out[q], ts, tr);
    }
}

// ------------------------------------------------------------------ sorted-marginal path
// The paper's box-assisted k-NN reaches O(n log n) per window by searching only near each
// point.  The GPU analogue here is exact: sort the window by x (payload: original index) and sort y;
// then for each point
//   eps_i: outward scan in x order from the point's own position, visiting candidates in non-decreasing
//          |fl(x_i - x_j)| (merge of the left and right runs; fl is monotone, so the runs are sorted) and
//          stopping as soon as that |dx| >= r_{k+1}: every unvisited j has d_ij >= |dx| >= r_{k+1} and
//          cannot change the (k+1)-th order statistic.  Same multiset statistic as the brute force.
//   n_x:   {j : |fl(x_i - x_j)| < eps} is an index interval of the x-sorted array (the predicate is
//          monotone on each side of x_i), found by two binary searches with the identical predicate;
//          n_y likewise on the sorted y.  Bit-identical to the brute-force counts.
constexpr int kSortedThreads = 128;  // points per CTA of the scan kernel (one point per thread)
constexpr int kLockstepMinW = 2048;  // phase B: lockstep binary searches from this window size up (measured)
constexpr int kCarried = -(1 << 20);  // stop_s.x <= this: NEXT-3 carried-over counts (n_x = kCarried - x)
constexpr int kMergeThreads = kMergePts;  // elements per CTA of the XL rank merge

// Order-preserving map of float bits to unsigned (finite values; -0 sorts just before +0, equal as floats).
__device__ __forceinline__ unsigned sortable(float f) {
    const unsigned u = __float_as_uint(f);
    return u ^ ((u >> 31) ? 0xffffffffu : 0x80000000u);
}
__device__ __forceinline__ void put_sentinels(float2* P2, int w, int t) {  // t < 2 kScanB: one entry each
    if (t < kScanB)
        P2[-1 - t] = make_float2(-kInf, 0.0f);
    else if (t < 2 * kScanB)
        P2[w + t - kScanB] = make_float2(kInf, 0.0f);
}
__device__ __forceinline__ float unsortable(unsigned s) {
    return __uint_as_float(s ^ ((s >> 31) ? 0x80000000u : 0xffffffffu));
}

// In-SMEM bitonic sort of n2 (power of two) keys, ascending.  Exchange steps with stride j <= 32 stay inside
// one warp's 64-key block (for every t a warp handles), so they only need __syncwarp; wider steps, and the
// step before one, need the CTA barrier.
template <typename K>
__device__ __forceinline__ void bitonic_smem(K* key, int n2) {
    for (int k = 2; k <= n2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int t = threadIdx.x; t < (n2 >> 1); t += blockDim.x) {
                const int i = 2 * t - (t & (j - 1));
                const int ixj = i + j;
                const K a = key[i], c = key[ixj];
                const bool up = (i & k) == 0;
                const bool sw = up ? (a > c) : (a < c);
                key[i] = sw ? c : a;
                key[ixj] = sw ? a : c;
            }
            const int next_j = j > 1 ? (j >> 1) : k;  // first stride of the next phase is k (= 2k / 2)
            if (j > 32 || next_j > 32)
                __syncthreads();
            else
                __syncwarp();
        }
    }
    __syncthreads();
}

// One CTA per (window, segment of <= kSortedMaxW points): bitonic sorts in SMEM of (x, idx) and of y.
// A window that is one segment writes the scan layout directly: P2[m] = (x, y) of the m-th point in x
// order, OX[m] = its original index, YS = sorted y.  Segments of an XL window write sorted runs to
// TX/TI/TY instead; rank_merge_kernel then places every element by its rank across the runs.
// count of elements < v (strict) or <= v in a sorted run s[0..n)
__device__ __forceinline__ int count_below(const float* s, int n, float v, bool inclusive) {
    int lo = 0, hi = n;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (inclusive ? (s[mid] <= v) : (s[mid] < v)) lo = mid + 1; else hi = mid;
    }
    return lo;
}

// XL windows: element p of run c goes to rank = (p - start(c)) + sum_{c' < c} #{run c' <= v}
// + sum_{c' > c} #{run c' < v}: a total order (ties by run), so ranks are a permutation.
__device__ __forceinline__ int left_bound(const float* s, int m, float v, float eps) {
    int lo = 0, hi = m;  // answer in [lo, hi]; s[hi]... pred(m) true iff eps > 0 (checked by caller)
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (v - s[mid] < eps) hi = mid; else lo = mid + 1;
    }
    return lo;
}
// right side: largest j in [m, w) with fl(s[j] - v) < eps, returned as one past it
__device__ __forceinline__ int right_bound(const float* s, int m, int w, float v, float eps) {
    int lo = m, hi = w;  // first j >= m with pred false, in [m, w]
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s[mid] - v < eps) lo = mid + 1; else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int lower_bound_f(const float* s, int w, float v) {
    int lo = 0, hi = w;
    while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s[mid] < v) lo = mid + 1; else hi = mid;
    }
    return lo;
}
__device__ __forceinline__ int left_bound_f(const float* s, int m, float v, float eps) { return left_bound(s, m, v, eps); }

// KSG-2 on the sorted path: every kNN(i) member has d_ij <= eps_i, hence |dx| <= eps_i, so it lies in the
// x-sorted interval {p : |fl(x_i - x_p)| < nextup(eps_i)} around the point's position m.  One pass over that
// interval takes the "<" members and counts the eps-ties; if there are more ties than kNN(i) needs, the
// `need` ties of smallest original index are selected (ascending (d, j) order, rule R1) by repeated minimum
// search — rare for continuous data.  Returns ex = nextup(d_x), ey = nextup(d_y) for the "<=" counts.
__device__ inline void ksg2_sorted_radii(const float2* __restrict__ P2, const float* __restrict__ XS,
                                  const int32_t* __restrict__ OX, int m, int w, float xv, float yv, float eps, int k,
                                  float* ex, float* ey) {
    float mx = 0.0f, my = 0.0f;
    if (eps > 0.0f) {
        const float e1 = nextup(eps);
        int lo = 0, hi = m;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (xv - XS[2 * mid] < e1) hi = mid; else lo = mid + 1;
        }
        const int La = lo;
        lo = m;
        hi = w;
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (XS[2 * mid] - xv < e1) lo = mid + 1; else hi = mid;
        }
        const int Ra = lo;
        int n_lt = 0, n_tie = 0;  // n_lt counts self (d = 0 < eps)
        float tx = 0.0f, ty = 0.0f;
        for (int p = La; p < Ra; ++p) {
            const float2 c = P2[p];
            const float dx = fabsf(xv - c.x), dy = fabsf(yv - c.y);
            const float d = fmaxf(dx, dy);
            if (d < eps) {
                ++n_lt;
                mx = fmaxf(mx, dx);
                my = fmaxf(my, dy);
            } else if (d == eps) {
                ++n_tie;
                tx = fmaxf(tx, dx);
                ty = fmaxf(ty, dy);
            }
        }
        const int need = (k + 1) - n_lt;  // ties in kNN(i) (self is among the n_lt)
        if (n_tie <= need) {
            mx = fmaxf(mx, tx);
            my = fmaxf(my, ty);
        } else {
            int last = -1;
            for (int t = 0; t < need; ++t) {
                int best = INT_MAX, bp = -1;
                for (int p = La; p < Ra; ++p) {
                    const float2 c = P2[p];
                    const float d = fmaxf(fabsf(xv - c.x), fabsf(yv - c.y));
                    const int j = OX[p];
                    if (d == eps && j > last && j < best) {
                        best = j;
                        bp = p;
                    }
                }
                const float2 c = P2[bp];
                mx = fmaxf(mx, fabsf(xv - c.x));
                my = fmaxf(my, fabsf(yv - c.y));
                last = best;
            }
        }
    }
    *ex = nextup(mx);
    *ey = nextup(my);
}

// Warp-level bitonic sort of 32*E keys held E per lane (blocked: lane l holds keys [E l, E l + E)),
// ascending.  Exchange distances j < E stay in registers; j >= E swap with lane l ^ (j / E) by shuffle.
template <typename T, int E>
__device__ __forceinline__ void warp_sort(T (&v)[E], int lane) {
    constexpr int LE = E == 1 ? 0 : E == 2 ? 1 : E == 4 ? 2 : 3;  // log2(E)
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= E) {
                const int lm = j >> LE;
                const bool lower = (lane & lm) == 0;
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    const bool up = ((((unsigned)lane << LE) | (unsigned)e) & (unsigned)k) == 0;
                    const T pv = __shfl_xor_sync(0xffffffffu, v[e], lm);
                    const T mn = pv < v[e] ? pv : v[e];
                    const T mx = pv < v[e] ? v[e] : pv;
                    v[e] = (lower == up) ? mn : mx;
                }
            } else {
#pragma unroll
                for (int e = 0; e < E; ++e) {
                    if ((e & j) == 0) {
                        const bool up = ((((unsigned)lane << LE) | (unsigned)e) & (unsigned)k) == 0;
                        const T a = v[e], c = v[e | j];
                        const bool sw = up ? (c < a) : (a < c);
                        v[e] = sw ? c : a;
                        v[e | j] = sw ? a : c;
                    }
                }
            }
        }
    }
}


// merge adjacent sorted runs of length r (src) into runs of 2r (dst); thread t < n2/8 writes outputs
// [8t, 8t+8).  Merge path: the co-rank i (outputs taken from run A) is found by binary search, A first
// on ties.
template <typename T>
__device__ __forceinline__ void merge_level(const T* __restrict__ src, T* __restrict__ dst, int n2, int r) {
    const int t = threadIdx.x;
    if (t * 8 < n2) {
        const int g = t * 8;
        const int base = (g / (2 * r)) * (2 * r);
        const T* A = src + base;
        const T* Bv = src + base + r;
        const int o = g - base;
        int lo = max(0, o - r), hi = min(o, r);
        while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (A[mid] <= Bv[o - mid - 1]) lo = mid + 1; else hi = mid;
        }
        int ia = lo, ib = o - lo;
        // the heads of both runs stay in registers: one SMEM load per output instead of two
        T a = ia < r ? A[ia] : T(0);
        T bv = ib < r ? Bv[ib] : T(0);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const bool takeA = ib >= r || (ia < r && a <= bv);
            dst[base + o + e] = takeA ? a : bv;
            if (takeA) {
                ++ia;
                if (ia < r) a = A[ia];
            } else {
                ++ib;
                if (ib < r) bv = Bv[ib];
            }
        }
    }
}

// Step 1 of the fused sort: warp c sorts keys [32E c, 32E (c+1)) (blocked, E per lane) of x (with the
// window index) and of y; the raw y also goes to `rawy` for the layout build.
template <int E>
__device__ __forceinline__ void chunk_sort(const float* __restrict__ gx, const float* __restrict__ gy, int w, int n2,
                                           unsigned long long* X0, unsigned* Y0, float* rawy, int warp, int lane,
                                           int ioff = 0) {
    for (int c = warp; c * 32 * E < n2; c += (int)(blockDim.x >> 5)) {
        unsigned long long vx[E];
        unsigned vy[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = c * 32 * E + lane * E + e;
            vx[e] = i < w ? ((unsigned long long)sortable(gx[i]) << 32) | (unsigned)(i + ioff) : ~0ull;
            const float yv = i < w ? gy[i] : 0.0f;
            vy[e] = i < w ? sortable(yv) : ~0u;
            if (rawy && i < w) rawy[i] = yv;  // raw y for the layout build (optional)
        }
        warp_sort<unsigned long long, E>(vx, lane);
        warp_sort<unsigned, E>(vy, lane);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            X0[c * 32 * E + lane * E + e] = vx[e];
            Y0[c * 32 * E + lane * E + e] = vy[e];
        }
    }
}

// ---- phase A's top list: the K = k smallest d_ij over the visited j != i (self, d_ii = 0, is never visited
// by the outward scan, so eps_i = the K-th entry = the (k+1)-th smallest of the multiset including self).
__device__ __forceinline__ void cswap(float& a, float& b) {
    const float lo = fminf(a, b);
    b = fmaxf(a, b);
    a = lo;
}
// r (sorted ascending, K entries) <- the K smallest of r U d[0..8), sorted: exact multiset order statistics.
// K = 4 and K = 8 use merge networks (sorted block, then the bitonic half-cleaner min(r[i], b[K-1-i]), which
// leaves exactly the K smallest of the union as a bitonic sequence, then a bitonic merger): 44 / 70 FMNMX per
// block instead of 56 / 120 for eight insertions.  Other K: insertion network per candidate.
template <int K>
__device__ __forceinline__ void topk_merge8(float (&r)[K], float (&d)[8]) {
    if constexpr (K == 4) {
        // sort both halves of the block (5 comparators each)
        cswap(d[0], d[1]); cswap(d[2], d[3]); cswap(d[0], d[2]); cswap(d[1], d[3]); cswap(d[1], d[2]);
        cswap(d[4], d[5]); cswap(d[6], d[7]); cswap(d[4], d[6]); cswap(d[5], d[7]); cswap(d[5], d[6]);
        // the block's 4 smallest (bitonic), then sorted
        float b[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) b[i] = fminf(d[i], d[7 - i]);
        cswap(b[0], b[2]); cswap(b[1], b[3]); cswap(b[0], b[1]); cswap(b[2], b[3]);
        // the 4 smallest of r U b (bitonic), then sorted
#pragma unroll
        for (int i = 0; i < 4; ++i) r[i] = fminf(r[i], b[3 - i]);
        cswap(r[0], r[2]); cswap(r[1], r[3]); cswap(r[0], r[1]); cswap(r[2], r[3]);
    } else if constexpr (K == 8) {
        // Batcher odd-even merge sort of the block (19 comparators)
        cswap(d[0], d[1]); cswap(d[2], d[3]); cswap(d[4], d[5]); cswap(d[6], d[7]);
        cswap(d[0], d[2]); cswap(d[1], d[3]); cswap(d[4], d[6]); cswap(d[5], d[7]);
        cswap(d[1], d[2]); cswap(d[5], d[6]);
        cswap(d[0], d[4]); cswap(d[1], d[5]); cswap(d[2], d[6]); cswap(d[3], d[7]);
        cswap(d[2], d[4]); cswap(d[3], d[5]);
        cswap(d[1], d[2]); cswap(d[3], d[4]); cswap(d[5], d[6]);
#pragma unroll
        for (int i = 0; i < 8; ++i) r[i] = fminf(r[i], d[7 - i]);
        // bitonic merger of 8
#pragma unroll
        for (int i = 0; i < 4; ++i) cswap(r[i], r[i + 4]);
        cswap(r[0], r[2]); cswap(r[1], r[3]); cswap(r[4], r[6]); cswap(r[5], r[7]);
        cswap(r[0], r[1]); cswap(r[2], r[3]); cswap(r[4], r[5]); cswap(r[6], r[7]);
    } else {
#pragma unroll
        for (int u = 0; u < 8; ++u) topk_insert<K>(r, d[u]);
    }
}

// a (sorted ascending, K entries) <- the K smallest of a U b, b sorted ascending (K entries): the bitonic
// half-cleaner min(a[i], b[K-1-i]) keeps exactly the K smallest as a bitonic sequence, a bitonic merger sorts it
// (K = 4: 12 FMNMX, K = 8: 32); other K insert b's entries one by one.
template <int K>
__device__ __forceinline__ void topk_merge_sorted(float (&a)[K], const float (&b)[K]) {
    if constexpr (K == 4 || K == 8) {
#pragma unroll
        for (int i = 0; i < K; ++i) a[i] = fminf(a[i], b[K - 1 - i]);
#pragma unroll
        for (int h = K / 2; h >= 1; h >>= 1)
#pragma unroll
            for (int i = 0; i < K; ++i)
                if ((i & h) == 0) cswap(a[i], a[i + h]);
    } else {
#pragma unroll
        for (int m = 0; m < K; ++m) topk_insert<K>(a, b[m]);
    }
}

// Phase A of the sorted path for the points [wb, we) (positions relative to cta0) of one warp: exact
// k-NN radius by outward scan in x order (a3).  Writes eps_s[ml]; adds the candidate visits to `steps`.
// P2 must carry sentinels: P2[-kScanB..-1] = (-inf, 0), P2[w..w+kScanB-1] = (+inf, 0) (no bounds checks).
// Warp-local work queue: a lane that finishes its point takes the next one (ballot + popc), so warps do
// not idle on their slowest lane (per-point scan lengths vary several-fold with the local density ratio).
// PAIRS (two-sided form only): candidates loaded as 16-byte pairs from aligned blocks (see below); for P2 in global
// memory at large w, where the lanes' blocks lie far apart (measured: w = 16,384 -9 %, 4,096 -4.5 %; shared memory
// and w <= 1,024 slightly slower, so those keep 8-byte loads).
constexpr int kPairsMinW = 2048;
template <int K1, bool PAIRS = false>
__device__ __forceinline__ void sorted_phase_a(const float2* P2, int w, int cta0, int wb, int we, float* eps_s,
                                               unsigned long long& steps, int2* stop_s = nullptr,
                                               bool unified = true, const uint16_t* wl = nullptr) {
    // work items k in [wb, we): the points ml = k, or ml = wl[k] (the points an incremental window must scan)
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    constexpr int B = kScanB;
    int kcur = wb + lane;
    bool act = kcur < we;
    int mloc = act ? (wl ? (int)wl[kcur] : kcur) : 0;
    int next = wb + 32;
    float xi = 0.f, yi = 0.f;
    int lj = 0, rj = 0;  // next unvisited index on each side
    bool lact = false, ract = false;
    bool lself = false, rself = false;  // two-sided form: the side's first block holds self (masked)
    constexpr int K = K1 - 1;  // the k smallest over j != i (self's d = 0 is never merged)
    float rk[K];
    auto start = [&](int ml) {
        const int m = cta0 + ml;
        const float2 me = P2[m];
        xi = me.x;
        yi = me.y;
#pragma unroll
        for (int t = 0; t < K; ++t) rk[t] = kInf;
        lj = m - 1;
        rj = m + 1;
        lself = rself = false;
        if (PAIRS && !unified) {
            // aligned blocks: left [lj - 7, lj] with lj odd, right [rj, rj + 7] with rj even, so every block is four
            // 16-byte pairs (P2 + even index is 16-byte aligned); the side whose first block would start one entry
            // short takes self into it instead, and self's distance there is replaced by +inf
            if (!(lj & 1)) {
                lj = m;
                lself = true;
            }
            if (rj & 1) {
                rj = m;
                rself = true;
            }
        }
        lact = true;  // the sentinels end a side
        ract = true;
    };
    // a block with any candidate below r_{k+1}: the whole block through the merge network (exact: merging
    // d >= r_{k+1} leaves the list unchanged), no per-candidate branches
    static_assert(B == 8, "topk_merge8 takes blocks of 8");
    auto visit = [&](float (&d)[B]) {
#ifdef ISY_MERGE_ALWAYS
        topk_merge8<K>(rk, d);
#else
        float mn = d[0];
#pragma unroll
        for (int u = 1; u < B; ++u) mn = fminf(mn, d[u]);
        if (mn < rk[K - 1]) topk_merge8<K>(rk, d);
#endif
    };
    // candidate visits of the finished point (algorithmic work), from its final stops: the left side visited
    // m-1 down to max(0, lj+1), the right side m+1 up to min(w-1, rj-1) (sentinels are not counted)
    auto visited = [&]() -> unsigned long long {
        const int m = cta0 + mloc;
        return (unsigned long long)(min(m, m - 1 - lj) + min(w - 1 - m, rj - m - 1));
    };
    if (act) start(mloc);
    bool toggle = false;
    while (__any_sync(0xffffffffu, act)) {
        bool fin = false;
        if (act && unified) {
            // one block per iteration from one side (alternating while both sides are open): every lane runs
            // the same instruction stream whichever side it scans, so the warp does not diverge on the side
            // tests.  |fl(x_j - x_i)| == fl(x_i - x_j) for x_j <= x_i (IEEE subtraction is antisymmetric), so
            // both sides use the same distance code; the sentinels give +inf either way.
            const bool useL = lact && (!ract || toggle);
            toggle = !toggle;
            const int base = useL ? lj : rj;
            const int stp = useL ? -1 : 1;
            float d[B], far = 0.f;
#pragma unroll
            for (int u = 0; u < B; ++u) {
                const float2 c = P2[base + stp * u];
                const float dx = fabsf(c.x - xi);
                d[u] = fmaxf(dx, fabsf(yi - c.y));
                far = dx;
            }
            visit(d);
            const float r = rk[K - 1];
            if (useL) {
                lj -= B;
                lact = far < r;
            } else {
                rj += B;
                ract = far < r;
            }
            if (!lact && !ract) {
                fin = true;
                steps += visited();
                eps_s[mloc] = r;
                if (stop_s) stop_s[mloc] = make_int2(lj, rj);
            }
        } else if (act) {
          if constexpr (PAIRS) {
            // One 16-byte load per pair of candidates: the lanes' blocks lie scattered over the window, and the
            // L1 data pipe serves a warp load roughly per distinct line touched, so pairs halve its wavefronts
            // (8-byte loads: 5.4 wavefronts per request, the scan's bound at w = 16,384).
            if (lact) {
                float d[B], far = 0.f;
#pragma unroll
                for (int h = 0; h < B / 2; ++h) {
                    // (P2[lj - 2h - 1], P2[lj - 2h]); P2[-B..-1] = (-inf, 0) sentinels: d = far = +inf
                    const float4 c = *reinterpret_cast<const float4*>(P2 + (lj - 2 * h - 1));
                    const float dxa = xi - c.z;  // >= 0: ascending order
                    const float dxb = xi - c.x;
                    d[2 * h] = fmaxf(dxa, fabsf(yi - c.w));
                    d[2 * h + 1] = fmaxf(dxb, fabsf(yi - c.y));
                    far = dxb;
                }
                if (lself) {  // d[0] is self's 0 (position m)
                    d[0] = kInf;
                    lself = false;
                }
                visit(d);
                lj -= B;
                lact = far < rk[K - 1];
            }
            if (ract) {
                float d[B], far = 0.f;
#pragma unroll
                for (int h = 0; h < B / 2; ++h) {
                    // (P2[rj + 2h], P2[rj + 2h + 1]); P2[w..w+B-1] = (+inf, 0) sentinels
                    const float4 c = *reinterpret_cast<const float4*>(P2 + (rj + 2 * h));
                    const float dxa = c.x - xi;
                    const float dxb = c.z - xi;
                    d[2 * h] = fmaxf(dxa, fabsf(yi - c.y));
                    d[2 * h + 1] = fmaxf(dxb, fabsf(yi - c.w));
                    far = dxb;
                }
                if (rself) {  // d[0] is self's 0 (position m)
                    d[0] = kInf;
                    rself = false;
                }
                visit(d);
                rj += B;
                ract = far < rk[K - 1];
            }
          } else {
            if (lact) {
                float d[B], far = 0.f;
#pragma unroll
                for (int u = 0; u < B; ++u) {
                    const float2 c = P2[lj - u];  // P2[-B..-1] = (-inf, 0) sentinels: d = far = +inf
                    const float dx = xi - c.x;    // >= 0: ascending order
                    d[u] = fmaxf(dx, fabsf(yi - c.y));
                    far = dx;
                }
                visit(d);
                lj -= B;
                lact = far < rk[K - 1];
            }
            if (ract) {
                float d[B], far = 0.f;
#pragma unroll
                for (int u = 0; u < B; ++u) {
                    const float2 c = P2[rj + u];  // P2[w..w+B-1] = (+inf, 0) sentinels
                    const float dx = c.x - xi;
                    d[u] = fmaxf(dx, fabsf(yi - c.y));
                    far = dx;
                }
                visit(d);
                rj += B;
                ract = far < rk[K - 1];
            }
          }
            if (!lact && !ract) {
                fin = true;
                steps += visited();
                eps_s[mloc] = rk[K - 1];
                if (stop_s) stop_s[mloc] = make_int2(lj, rj);  // next unvisited index on each side
            }
        }
        const unsigned fm = __ballot_sync(0xffffffffu, fin);
        if (fm) {
            if (fin) {
                const int idx = next + __popc(fm & lt_mask);
                if (idx < we) {
                    kcur = idx;
                    mloc = wl ? (int)wl[idx] : idx;
                    start(mloc);
                } else {
                    act = false;
                }
            }
            next += __popc(fm);
        }
    }
}

// Phase A, box-assisted form (the paper's box-assisted k-NN, made exact): the window's x-sorted
// positions form columns of kColW; CY holds each column's points (y, x) sorted by y.  A point first takes every
// other point of its own column (in x order, blocks of 8 through the merge network, itself excluded), then visits
// the other columns outward in order of their x-distance to it:
//   * a column left of it whose largest x has fl(x_i - x) >= r (or right of it whose smallest x has
//     fl(x - x_i) >= r) holds no point with d < r, nor does any column beyond it on that side: the side stops;
//   * inside a column only the y-interval {j : |fl(y_i - y_j)| < r} can hold a point with d < r (the predicate is
//     monotone on the y-sorted column, as in phase B): one binary search for its start, then a walk while
//     fl(y_j - y_i) < r with the current (shrinking) r.
// Every j with d_ij < eps lies in a visited column and inside that column's walked interval, so the top list ends
// as the k smallest d over j != i — the same order statistic as the outward scan.  Stops for phase B: positions up
// to the last position of the left stop column, and from the first of the right one, have |dx| >= r >= eps.
template <int K1>
__device__ __forceinline__ void sorted_phase_a_cols(const float2* P2, const float2* CY, int w, int cta0, int wb,
                                                    int we, float* eps_s, unsigned long long& steps,
                                                    int2* stop_s) {
    constexpr int K = K1 - 1;
    constexpr int C = kColW;
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    int kcur = wb + lane;
    bool act = kcur < we;
    int next = wb + 32;
    float xi = 0.f, yi = 0.f;
    int m = 0, cl = 0, cr = 0, blk = 0;  // own-column blocks visited (C / 8 of them), then the other columns
    float rk[K];
    auto start = [&](int ml) {
        m = cta0 + ml;
        const float2 me = P2[m];
        xi = me.x;
        yi = me.y;
#pragma unroll
        for (int t = 0; t < K; ++t) rk[t] = kInf;
        const int col = m / C;
        cl = col - 1;
        cr = col + 1;
        blk = 0;
    };
    // one block of 8 own-column candidates in x order (itself and positions past w: +inf)
    auto own_block = [&](int c0) {
        float d[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const int pj = c0 + u;
            const float2 c = pj < w ? P2[pj] : make_float2(kInf, 0.0f);
            const float dd = fmaxf(fabsf(xi - c.x), fabsf(yi - c.y));
            d[u] = (pj == m || pj >= w) ? kInf : dd;
        }
        float mn = d[0];
#pragma unroll
        for (int u = 1; u < 8; ++u) mn = fminf(mn, d[u]);
        if (mn < rk[K - 1]) topk_merge8<K>(rk, d);
        steps += (unsigned long long)max(0, min(8, w - c0) - ((m >= c0 && m < c0 + 8) ? 1 : 0));
    };
    // walk column `col` (y ascending) from lo while fl(y_j - y_i) < r
    auto walk = [&](const float2* col, int lo, int len) {
        for (int j = lo; j < len; ++j) {
            const float2 e = col[j];  // (y, x)
            if (!(e.x - yi < rk[K - 1])) break;
            ++steps;
            const float dd = fmaxf(fabsf(xi - e.y), fabsf(yi - e.x));
            if (dd < rk[K - 1]) topk_insert<K>(rk, dd);
        }
    };
    if (act) start(kcur);
    while (__any_sync(0xffffffffu, act)) {
        bool fin = false;
        if (act) {
            if (blk < C / 8) {  // two own-column blocks per iteration (16 independent loads)
                const int c0 = (m / C) * C + blk * 8;
                own_block(c0);
                own_block(c0 + 8);
                blk += 2;
            } else {
                // the next column on each side within r of the point, both per iteration: their binary searches
                // run in lockstep so the two chains of dependent loads overlap
                const float r = rk[K - 1];
                const float dl = cl >= 0 ? xi - P2[cl * C + C - 1].x : kInf;  // x-sorted: >= 0
                const float dr = cr * C < w ? P2[cr * C].x - xi : kInf;
                const bool gl = dl < r, gr = dr < r;
                if (!gl && !gr) {
                    fin = true;
                } else {
                    const float2* colL = CY + (gl ? cl : 0) * C;
                    const float2* colR = CY + (gr ? cr : 0) * C;
                    const int lenL = gl ? min(C, w - cl * C) : 0, lenR = gr ? min(C, w - cr * C) : 0;
                    int l0 = 0, n0 = lenL, l1 = 0, n1 = lenR;  // first j with fl(y_i - y_j) < r, per column
                    while ((n0 | n1) > 0) {
                        if (n0 > 0) {
                            const int h = n0 >> 1;
                            if (!(yi - colL[l0 + h].x < r)) { l0 += h + 1; n0 -= h + 1; } else n0 = h;
                            ++steps;
                        }
                        if (n1 > 0) {
                            const int h = n1 >> 1;
                            if (!(yi - colR[l1 + h].x < r)) { l1 += h + 1; n1 -= h + 1; } else n1 = h;
                            ++steps;
                        }
                    }
                    if (gl) {
                        walk(colL, l0, lenL);
                        --cl;
                    }
                    if (gr) {
                        walk(colR, l1, lenR);
                        ++cr;
                    }
                }
            }
            if (fin) {
                eps_s[m - cta0] = rk[K - 1];
                // phase B brackets: st.x + 2 = first position that may have |dx| < eps, st.y - 1 = one past the last
                if (stop_s) stop_s[m - cta0] = make_int2(cl >= 0 ? cl * C + C - 2 : -2, cr * C < w ? cr * C + 1 : w + 1);
            }
        }
        const unsigned fm = __ballot_sync(0xffffffffu, fin);
        if (fm) {
            if (fin) {
                const int idx = next + __popc(fm & lt_mask);
                if (idx < we) {
                    kcur = idx;
                    start(idx);
                } else {
                    act = false;
                }
            }
            next += __popc(fm);
        }
    }
}

// Phase B for one point at sorted position m (a4, a5): interval counts by binary search with the
// identical predicates, digamma / log terms, debug outputs.
// [xlo, xhi] brackets the x-interval's ends (KSG-1: from phase A's stopping points; else [0, w]).
template <bool V2>
__device__ __forceinline__ void sorted_phase_b(const KsgLaunch& L, int w, int64_t dbg, const float2* P2,
                                               const int32_t* OX, const float* YS, int m, float eps, long long& sp,
                                               long long& sl, int& z, int xlo = 0, int xhi = INT_MAX,
                                               int pre_nx = -1, int pre_ny = -1, int* out_nx = nullptr,
                                               int* out_ny = nullptr) {
    const float* XS = reinterpret_cast<const float*>(P2);  // stride-2 view for the x binary searches
    const float2 me = P2[m];
    const float xv = me.x, yv = me.y;
    int nx = 0, ny = 0;
    float ex = eps, ey = eps;
    if (!V2 && pre_nx >= 0) {  // NEXT-3: counts carried over (updated by the removed / inserted blocks)
        nx = pre_nx;
        ny = pre_ny;
    } else {
    if (V2) ksg2_sorted_radii(P2, XS, OX, m, w, xv, yv, eps, L.k, &ex, &ey);
    if (V2 || eps > 0.0f) {
        // The searches run in lockstep so their loads are in flight together (memory-level parallelism; one
        // search at a time was latency-bound): the two x bounds and the two y bounds.  Each search finds the
        // end of the prefix of [b, b + n) on which its predicate holds.
        //   x left  [lo, m):  !(fl(x_i - x_j) < ex)      x right [m, hi): fl(x_j - x_i) < ex
        //   y left  [0, w):   !(fl(y_i - y_j) < ey)      y right [0, w):  fl(y_j - y_i) < ey
        const int xl0 = V2 ? 0 : xlo, xr1 = V2 ? w : min(w, xhi);
        if (w < kLockstepMinW) {  // short searches: one at a time (the lockstep predication costs more there)
            int lo = xl0, hi = m;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (xv - XS[2 * mid] < ex) hi = mid; else lo = mid + 1;
            }
            const int Lx = lo;
            lo = m;
            hi = xr1;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (XS[2 * mid] - xv < ex) lo = mid + 1; else hi = mid;
            }
            nx = lo - Lx - 1;
            // y: both ends searched over the whole sorted array (no pivot search for y_i's own rank): for
            // YS[j] >= y_i, fl(y_i - YS[j]) <= 0 < ey, and for YS[j] <= y_i, fl(YS[j] - y_i) <= 0 < ey, so each
            // predicate is monotone on [0, w) and its first flip is the interval end
            ny = right_bound(YS, 0, w, yv, ey) - left_bound_f(YS, w, yv, ey) - 1;
        } else {
        int b0 = xl0, n0 = m - xl0, b1 = m, n1 = xr1 - m;
        int b3 = 0, n3 = w, b4 = 0, n4 = w;  // y ends over [0, w) (monotone predicates, see above)
        while ((n0 | n1 | n3 | n4) > 0) {
            if (n0 > 0) {
                const int h = n0 >> 1;
                if (!(xv - XS[2 * (b0 + h)] < ex)) { b0 += h + 1; n0 -= h + 1; } else n0 = h;
            }
            if (n1 > 0) {
                const int h = n1 >> 1;
                if (XS[2 * (b1 + h)] - xv < ex) { b1 += h + 1; n1 -= h + 1; } else n1 = h;
            }
            if (n3 > 0) {
                const int h = n3 >> 1;
                if (!(yv - YS[b3 + h] < ey)) { b3 += h + 1; n3 -= h + 1; } else n3 = h;
            }
            if (n4 > 0) {
                const int h = n4 >> 1;
                if (YS[b4 + h] - yv < ey) { b4 += h + 1; n4 -= h + 1; } else n4 = h;
            }
        }
        nx = b1 - b0 - 1;
        ny = b4 - b3 - 1;
        }
    }
    }
    if (out_nx) *out_nx = nx;
    if (out_ny) *out_ny = ny;
    sp += V2 ? L.psiq[nx] + L.psiq[ny] : L.psiq[nx + 1] + L.psiq[ny + 1];
    if (eps > 0.0f)
        sl += q32(canon_ln(__dmul_rn(2.0, (double)eps), L.lnc));
    else
        z += 1;
    if (dbg >= 0) {
        const int i = OX[m];
        if (L.dbg_eps) L.dbg_eps[dbg + i] = eps;
        if (L.dbg_nx) L.dbg_nx[dbg + i] = nx;
        if (L.dbg_ny) L.dbg_ny[dbg + i] = ny;
    }
}

// Scan of one CTA's slice [cta0, cta0 + cta_n) of a window's x-sorted points (arrays in global or shared
// memory, generic pointers): P2[m] = (x, y) of the m-th point in x order, OX[m] its window index, YS the
// sorted y.  Each warp owns a contiguous part of the slice.  Ends with the CTA reduction.
//
// KSG-1 narrowing: phase A stops a side at a block whose farthest candidate has |dx| >= r(t) >= eps, so
// with lj / rj the next unvisited indices, positions <= lj + 1 and >= rj - 1 are outside the strict
// interval {|dx| < eps}: the x binary searches run on [lj + 2, m] and [m, rj - 1] (stop_s, optional).
// (KSG-2's closed |dx| <= d_x, d_x <= eps, may include |dx| = eps: full ranges there.)
// NEXT-3, incremental radius (the paper's influenced region, IR): window W' = W - R + I follows W
// on a grid of step d (R = the d points that left, I = the d that entered; both are sorted blocks of the
// NEXT-3 block storage, keys = sortable x << 32 | absolute index).  For a point kept from W with radius e,
// if no removed point has d_ij <= e and no inserted point has d_ij < e, the (k+1) smallest distances of the
// multiset are unchanged (removing elements > e and adding elements >= e), so eps in W' is exactly e.
// Candidates with |fl(x_i - x_j)| <= e are one index range of a block (sorted x, monotone rounding): a
// binary search for its start, then a walk while |dx| <= e.  Returns true if e carries over.
__device__ __forceinline__ bool inc_unchanged(const float* __restrict__ bx, const float* __restrict__ by, int n,
                                              float xv, float yv, float e, bool strict, unsigned long long& steps,
                                              int& cx) {
    // bx: the block's x ascending, by: the matching y (both in shared memory); cx = #{j : |fl(x_i - x_j)| < e}
    int lo = 0, len = n;  // first j with fl(x_i - x_j) <= e  (x_j ascending: false ... true)
    while (len > 0) {
        ++steps;  // probes and candidate visits count as algorithmic work, like the scan's
        const int h = len >> 1;
        if (!(xv - bx[lo + h] <= e)) { lo += h + 1; len -= h + 1; } else len = h;
    }
    cx = 0;
    for (int j = lo; j < n; ++j) {
        ++steps;
        const float xj = bx[j];
        const float dx = fabsf(xv - xj);
        if (xj > xv && !(dx <= e)) break;  // past the range on the right: fl(x_j - x_i) > e
        cx += dx < e ? 1 : 0;
        const float d = fmaxf(dx, fabsf(yv - by[j]));
        if (strict ? (d < e) : (d <= e)) return false;
    }
    return true;
}

// #{j : |fl(y_i - y_j)| < e} in a y-ascending block (an index interval: two binary searches)
__device__ __forceinline__ int inc_count_y(const float* __restrict__ ys, int n, float yv, float e,
                                           unsigned long long& steps) {
    int a = 0, la = n;  // first j with fl(y_i - y_j) < e
    while (la > 0) {
        ++steps;
        const int h = la >> 1;
        if (!(yv - ys[a + h] < e)) { a += h + 1; la -= h + 1; } else la = h;
    }
    int b = a, lb = n - a;  // first j >= a with !(fl(y_j - y_i) < e)
    while (lb > 0) {
        ++steps;
        const int h = lb >> 1;
        if (ys[b + h] - yv < e) { b += h + 1; lb -= h + 1; } else lb = h;
    }
    return b - a;
}

// Stage the removed (R) and inserted (I) blocks of an incremental window into shared memory: x ascending with
// the matching y, and the block's y ascending: sb = [Rx | Ry | Rys | Ix | Iy | Iys], d floats each.
__device__ __forceinline__ void inc_stage(const KsgInc& ic, const unsigned long long* __restrict__ BX,
                                          const unsigned* __restrict__ BY, const float* __restrict__ gy, float* sb) {
    const int d = ic.d;
    for (int j = threadIdx.x; j < 2 * d; j += blockDim.x) {
        const bool rr = j < d;
        const int jj = rr ? j : j - d;
        const int64_t off = (rr ? ic.boffR : ic.boffI) + jj;
        const unsigned long long key = BX[off];
        float* dst = sb + (rr ? 0 : 3 * d);
        dst[jj] = unsortable((unsigned)(key >> 32));
        dst[d + jj] = gy[(unsigned)(key & 0xffffffffu)];
        dst[2 * d + jj] = unsortable(BY[off]);
    }
    __syncthreads();
}

template <int K1, bool V2>
__device__ __forceinline__ void sorted_scan(const KsgLaunch& L, int q, int w, int ntiles, const float2* P2,
                                            const int32_t* OX, const float* YS, int cta0, int cta_n, float* eps_s,
                                            int2* stop_s = nullptr, const KsgInc* inc = nullptr,
                                            const float* eps_prev = nullptr, float* eps_out = nullptr,
                                            const unsigned long long* BX = nullptr, uint16_t* wl_s = nullptr,
                                            float* inc_sb = nullptr, const unsigned* BY = nullptr,
                                            const int2* cnt_prev = nullptr, int2* cnt_out = nullptr,
                                            unsigned* done = nullptr, int b_self = 0,
                                            const float2* CY = nullptr) {
    const int nwarps = blockDim.x >> 5;
    const int kPerWarp = (cta_n + nwarps - 1) / nwarps;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int wb = min(warp * kPerWarp, cta_n);
    const int we = min(wb + kPerWarp, cta_n);
    unsigned long long steps = 0;
    unsigned reused = 0;
    int wl_cnt = -1;  // >= 0: incremental window, this warp's scan list length
    // phase A's 16-byte pair loads: P2 in global memory (the throughput scan's scratch) and large windows
    const bool pairs = w >= kPairsMinW && !__isShared(P2);
    if (inc && eps_prev && cnt_prev && stop_s && !V2) {
        // incremental window: radii carried over where the removed / inserted blocks cannot change them; the
        // remaining points (and the newly inserted ones) form this warp's scan list
        const KsgWin W = L.wins[q];
        if (done) {  // the predecessor's radii and counts must be complete (its CTAs took earlier work tickets)
            if (threadIdx.x == 0) {
                volatile unsigned* dp = done + inc->pred;
                while (*dp < (unsigned)ntiles) __nanosleep(256);
                __threadfence();
            }
            __syncthreads();
        }
        inc_stage(*inc, BX, BY, L.pairs[W.pair].y, inc_sb);
        const int d = inc->d;
        const float* Rx = inc_sb;
        const float* Ix = inc_sb + 3 * d;
        uint16_t* wl = wl_s + wb;
        int cnt = 0;
        for (int k0 = wb; k0 < we; k0 += 32) {
            const int ml = k0 + lane;
            bool scan = false;
            if (ml < we) {
                const int m = cta0 + ml;
                const int idx = OX[m];
                scan = true;
                if (idx < w - inc->d) {
                    const float e = eps_prev[idx + d];
                    const float2 me = P2[m];
                    int rx = 0, ix = 0;
                    if (!V2 && inc_unchanged(Rx, Rx + d, d, me.x, me.y, e, false, steps, rx) &&
                        inc_unchanged(Ix, Ix + d, d, me.x, me.y, e, true, steps, ix)) {
                        // the paper's IMR: the marginal counts of a kept point change only by the removed and inserted
                        // points within eps of it (eps = 0: no counts); kCarried - n_x flags counts computed here
                        // (phase A's stops are >= -kScanB - 1)
                        eps_s[ml] = e;
                        int2 st = make_int2(kCarried, 0);
                        if (e > 0.0f) {
                            const int2 c0 = cnt_prev[idx + d];
                            const int ry = inc_count_y(Rx + 2 * d, d, me.y, e, steps);
                            const int iy = inc_count_y(Ix + 2 * d, d, me.y, e, steps);
                            st = make_int2(kCarried - (c0.x - rx + ix), c0.y - ry + iy);
                        }
                        stop_s[ml] = st;
                        scan = false;
                        ++reused;
                    }
                }
            }
            const unsigned bm = __ballot_sync(0xffffffffu, scan);
            if (scan) wl[cnt + __popc(bm & ((1u << lane) - 1u))] = (uint16_t)ml;
            cnt += __popc(bm);
        }
        __syncwarp();
        if (pairs)
            sorted_phase_a<K1, true>(P2, w, cta0, 0, cnt, eps_s, steps, stop_s, L.scan_unified != 0, wl);
        else
            sorted_phase_a<K1>(P2, w, cta0, 0, cnt, eps_s, steps, stop_s, L.scan_unified != 0, wl);
        wl_cnt = cnt;
    } else if (CY && w >= L.col_min_w) {
        sorted_phase_a_cols<K1>(P2, CY, w, cta0, wb, we, eps_s, steps, stop_s);
    } else if (pairs) {
        sorted_phase_a<K1, true>(P2, w, cta0, wb, we, eps_s, steps, stop_s, L.scan_unified != 0);
    } else {
        sorted_phase_a<K1>(P2, w, cta0, wb, we, eps_s, steps, stop_s, L.scan_unified != 0);
    }
    __syncthreads();
    long long sp = 0, sl = 0;
    int z = 0;
    const int64_t dbg = L.wins[q].dbg_off;
    if (wl_cnt >= 0) {
        // incremental window: the carried points are cheap (terms from their counts), the scanned ones run the full
        // phase B; both loops keep every lane busy (per-lane mixing would run the searches for the whole warp)
        for (int ml = threadIdx.x; ml < cta_n; ml += blockDim.x) {
            const int2 st = stop_s[ml];
            if (st.x > kCarried) continue;
            int nx = 0, ny = 0;
            sorted_phase_b<V2>(L, w, dbg, P2, OX, YS, cta0 + ml, eps_s[ml], sp, sl, z, 0, w, kCarried - st.x, st.y,
                               &nx, &ny);
            const int i = OX[cta0 + ml];
            eps_out[i] = eps_s[ml];
            cnt_out[i] = make_int2(nx, ny);
        }
        const uint16_t* wl = wl_s + wb;
        for (int k = lane; k < wl_cnt; k += 32) {
            const int ml = wl[k];
            const int2 st = stop_s[ml];
            int nx = 0, ny = 0;
            sorted_phase_b<V2>(L, w, dbg, P2, OX, YS, cta0 + ml, eps_s[ml], sp, sl, z, max(0, st.x + 2),
                               min(w, st.y - 1), -1, -1, &nx, &ny);
            const int i = OX[cta0 + ml];
            eps_out[i] = eps_s[ml];
            cnt_out[i] = make_int2(nx, ny);
        }
    }
    for (int ml = threadIdx.x; wl_cnt < 0 && ml < cta_n; ml += blockDim.x) {
        int xlo = 0, xhi = w, pnx = -1, pny = -1;
        if (stop_s) {
            const int2 st = stop_s[ml];
            if (st.x <= kCarried) {  // counts carried over by the incremental pass
                pnx = kCarried - st.x;
                pny = st.y;
            } else {
                xlo = max(0, st.x + 2);
                xhi = min(w, st.y - 1);
            }
        }
        int nx = 0, ny = 0;
        sorted_phase_b<V2>(L, w, dbg, P2, OX, YS, cta0 + ml, eps_s[ml], sp, sl, z, xlo, xhi, pnx, pny, &nx, &ny);
        if (eps_out) {
            const int i = OX[cta0 + ml];
            eps_out[i] = eps_s[ml];
            if (cnt_out) cnt_out[i] = make_int2(nx, ny);
        }
    }
    if (done && eps_out) {  // publish this slice of the window's radii / counts to its successor
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) atomicAdd(done + b_self, 1u);
    }
    cta_finish(L, q, w, ntiles, sp, sl, z, steps, reused);
}

// Throughput path scan kernel: the window was sorted by sort_window_kernel (+ rank_merge_kernel) into
// global scratch; a CTA owns L.sorted_ppc consecutive x-sorted points.
}  // namespace

#define ISY_K_CASES(FN, ...)                   \
    switch (L.k) {                             \
        case 1: return FN<2>(__VA_ARGS__);     \
        case 2: return FN<3>(__VA_ARGS__);     \
        case 3: return FN<4>(__VA_ARGS__);     \
        case 4: return FN<5>(__VA_ARGS__);     \
        case 5: return FN<6>(__VA_ARGS__);     \
        case 6: return FN<7>(__VA_ARGS__);     \
        case 7: return FN<8>(__VA_ARGS__);     \
        case 8: return FN<9>(__VA_ARGS__);     \
        case 9: return FN<10>(__VA_ARGS__);    \
        case 10: return FN<11>(__VA_ARGS__);   \
        case 11: return FN<12>(__VA_ARGS__);   \
        case 12: return FN<13>(__VA_ARGS__);   \
        case 13: return FN<14>(__VA_ARGS__);   \
        case 14: return FN<15>(__VA_ARGS__);   \
        case 15: return FN<16>(__VA_ARGS__);   \
        case 16: return FN<17>(__VA_ARGS__);   \
        default: return cudaErrorInvalidValue; \
    }

}  // namespace isy
