// Small windows (w <= 256): one warp per window, all points in registers.
#include "ksg_device.cuh"

namespace isy {
namespace {

// ------------------------------------------------------------------ small windows: one warp per window
template <int K1, int R, bool BL, bool V2>
__global__ void __launch_bounds__(kSmallWarps * 32)
    ksg_small_kernel(const KsgLaunch L, const int32_t* __restrict__ list, int32_t n) {
    constexpr int CAP = 32 * R + 4;
    __shared__ __align__(16) float sbuf[kSmallWarps][2][CAP];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int idx = blockIdx.x * kSmallWarps + warp;
    if (idx >= n) return;  // warp-uniform
    poison_warp(L, sbuf[warp], sizeof(sbuf[0]));
    const int q = list[idx];
    const KsgWin W = L.wins[q];
    const int w = W.w;
    const int wpad = (w + 3) & ~3;
    const float* gx = L.pairs[W.pair].x + W.t0;
    const float* gy = L.pairs[W.pair].y + W.t0;
    float* sx = sbuf[warp][0];
    float* sy = sbuf[warp][1];
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

template <int K1, bool BL, bool V2>
cudaError_t small_kb(const KsgLaunch& L, const int32_t* list, int32_t n, int R, cudaStream_t st) {
    const dim3 grid((n + kSmallWarps - 1) / kSmallWarps), block(kSmallWarps * 32);
    switch (R) {
        case 1: ksg_small_kernel<K1, 1, BL, V2><<<grid, block, 0, st>>>(L, list, n); break;
        case 2: ksg_small_kernel<K1, 2, BL, V2><<<grid, block, 0, st>>>(L, list, n); break;
        case 4: ksg_small_kernel<K1, 4, BL, V2><<<grid, block, 0, st>>>(L, list, n); break;
        case 8: ksg_small_kernel<K1, 8, BL, V2><<<grid, block, 0, st>>>(L, list, n); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

// KSG-2 instantiates only the branch-free small kernel (its speed is secondary; halves the build)
template <int K1>
cudaError_t small_k(const KsgLaunch& L, const int32_t* list, int32_t n, int R, cudaStream_t st) {
    if (L.variant == 1) return small_kb<K1, true, true>(L, list, n, R, st);
    return (L.knn_mode & 1) ? small_kb<K1, true, false>(L, list, n, R, st)
                           : small_kb<K1, false, false>(L, list, n, R, st);
}

}  // namespace

cudaError_t launch_ksg_small(const KsgLaunch& L, const int32_t* list, int32_t n, int R, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    ISY_K_CASES(small_k, L, list, n, R, st)
}


}  // namespace isy
