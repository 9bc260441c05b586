// Large windows, brute force: (window, i-tile) per CTA, j-tiles staged by cp.async.bulk (a2-a6).
#include "ksg_device.cuh"

namespace isy {
namespace {

template <int K1, int R, bool V2>
__global__ void __launch_bounds__(kTileThreads)
    ksg_tile_kernel(const KsgLaunch L, const KsgItem* __restrict__ items, int32_t n_items) {
    extern __shared__ __align__(16) float dyn[];
    __shared__ __align__(8) unsigned long long mbar;
    __shared__ long long red_sp[kTileThreads / 32], red_sl[kTileThreads / 32];
    __shared__ int red_z[kTileThreads / 32];
    if (L.poison) {
        poison_smem(L, dyn, dyn_smem_bytes());
        __syncthreads();
    }

    const KsgItem it = items[blockIdx.x];
    const int q = it.win;
    const KsgWin W = L.wins[q];
    const int w = W.w;
    const float* gx = L.pairs[W.pair].x;
    const float* gy = L.pairs[W.pair].y;
    const int64_t t0 = W.t0;
    float* sx = dyn;
    float* sy = dyn + (kTileJ + 8);
    const uint32_t bar = smem_u32(&mbar);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint32_t phase = 0;

    float xi[R], yi[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const int i = it.i0 + threadIdx.x + kTileThreads * r;
        xi[r] = i < w ? gx[t0 + i] : 0.0f;
        yi[r] = i < w ? gy[t0 + i] : 0.0f;
    }
    float rk[R][K1];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
        for (int m = 0; m < K1; ++m) rk[r][m] = kInf;

    const int nj = (w + kTileJ - 1) / kTileJ;
    int ng = 0;
    if (w <= kTileThreads) {
        // a window no wider than the CTA (latency-mode small windows): one coalesced load per thread
        // instead of the bulk-copy / mbarrier round trip
        const int j = threadIdx.x, wpad = (w + 3) & ~3;
        if (j < wpad) {
            sx[j] = j < w ? gx[t0 + j] : kInf;
            sy[j] = j < w ? gy[t0 + j] : kInf;
        }
        __syncthreads();
        ng = wpad >> 2;
        const float4* sx4 = reinterpret_cast<const float4*>(sx);
        const float4* sy4 = reinterpret_cast<const float4*>(sy);
        for (int g = 0; g < ng; ++g) knn_step<K1, R, false>(xi, yi, rk, sx4[g], sy4[g]);
    } else {
        for (int jt = 0; jt < nj; ++jt) {
            const int j0 = jt * kTileJ;
            ng = stage_tile(gx, gy, t0 + j0, min(kTileJ, w - j0), sx, sy, bar, phase);
            const float4* sx4 = reinterpret_cast<const float4*>(sx);
            const float4* sy4 = reinterpret_cast<const float4*>(sy);
            for (int g = 0; g < ng; ++g) knn_step<K1, R, false>(xi, yi, rk, sx4[g], sy4[g]);
            if (nj > 1) __syncthreads();
        }
    }
    float eps[R], ex[R], ey[R];
#pragma unroll
    for (int r = 0; r < R; ++r) ex[r] = ey[r] = eps[r] = rk[r][K1 - 1];
    if (V2) {  // KSG-2: d_x, d_y over kNN(i); j-tiles in ascending order (tie rule)
        int need[R], taken[R];
        float mx[R], my[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
            need[r] = ksg2_need<K1>(rk[r]);
            taken[r] = 0;
            mx[r] = my[r] = 0.0f;
        }
        for (int jt = 0; jt < nj; ++jt) {
            if (nj > 1) {
                const int j0 = jt * kTileJ;
                ng = stage_tile(gx, gy, t0 + j0, min(kTileJ, w - j0), sx, sy, bar, phase);
            }
            const float4* sx4 = reinterpret_cast<const float4*>(sx);
            const float4* sy4 = reinterpret_cast<const float4*>(sy);
            for (int g = 0; g < ng; ++g) ksg2_step<R>(xi, yi, eps, need, taken, mx, my, sx4[g], sy4[g]);
            if (nj > 1) __syncthreads();
        }
#pragma unroll
        for (int r = 0; r < R; ++r) {
            ex[r] = nextup(mx[r]);
            ey[r] = nextup(my[r]);
        }
    }
    unsigned cx[R], cy[R];
#pragma unroll
    for (int r = 0; r < R; ++r) cx[r] = cy[r] = 0u;
    for (int jt = 0; jt < nj; ++jt) {
        if (nj > 1) {
            const int j0 = jt * kTileJ;
            ng = stage_tile(gx, gy, t0 + j0, min(kTileJ, w - j0), sx, sy, bar, phase);
        }
        const float4* sx4 = reinterpret_cast<const float4*>(sx);
        const float4* sy4 = reinterpret_cast<const float4*>(sy);
        for (int g = 0; g < ng; ++g) count_step<R>(xi, yi, ex, ey, cx, cy, sx4[g], sy4[g], (unsigned)L.two);
        if (nj > 1) __syncthreads();
    }

    long long sp = 0, sl = 0;
    int z = 0;
    point_terms<R, V2>(L, w, W.dbg_off, it.i0 + threadIdx.x, kTileThreads, eps, cx, cy, sp, sl, z);
    warp_sum(sp, sl, z);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) {
        red_sp[warp] = sp;
        red_sl[warp] = sl;
        red_z[warp] = z;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
#pragma unroll
        for (int v = 1; v < kTileThreads / 32; ++v) {
            sp += red_sp[v];
            sl += red_sl[v];
            z += red_z[v];
        }
        const int ntiles = (w + kTileThreads * R - 1) / (kTileThreads * R);
        if (ntiles == 1) {
            finalize(L, w, sp, sl, z, &L.out[q]);
        } else {
            KsgAcc* A = &L.acc[q];
            atomicAdd(&A->s_psi, (unsigned long long)sp);
            atomicAdd(&A->s_log, (unsigned long long)sl);
            atomicAdd(&A->zero, (unsigned)z);
            __threadfence();
            const unsigned ticket = atomicAdd(&A->done, 1u);
            if (ticket == (unsigned)(ntiles - 1)) {  // last tile of the window: finalize + reset
                __threadfence();
                const long long tp = (long long)atomicExch(&A->s_psi, 0ull);
                const long long tl = (long long)atomicExch(&A->s_log, 0ull);
                const int tz = (int)atomicExch(&A->zero, 0u);
                atomicExch(&A->done, 0u);
                finalize(L, w, tp, tl, tz, &L.out[q]);
            }
        }
    }
}

template <int K1, bool V2>
cudaError_t tile_kv(const KsgLaunch& L, const KsgItem* items, int32_t n, int R, cudaStream_t st) {
    const size_t smem = 2 * (kTileJ + 8) * sizeof(float);
    switch (R) {
        case 1: ksg_tile_kernel<K1, 1, V2><<<n, kTileThreads, smem, st>>>(L, items, n); break;  // latency mode
        case 2: ksg_tile_kernel<K1, 2, V2><<<n, kTileThreads, smem, st>>>(L, items, n); break;
        case 4: ksg_tile_kernel<K1, 4, V2><<<n, kTileThreads, smem, st>>>(L, items, n); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <int K1>
cudaError_t tile_k(const KsgLaunch& L, const KsgItem* items, int32_t n, int R, cudaStream_t st) {
    return L.variant == 1 ? tile_kv<K1, true>(L, items, n, R, st) : tile_kv<K1, false>(L, items, n, R, st);
}

}  // namespace

cudaError_t launch_ksg_tile(const KsgLaunch& L, const KsgItem* items, int32_t n_items, int R, cudaStream_t st) {
    if (n_items <= 0) return cudaSuccess;
    ISY_K_CASES(tile_k, L, items, n_items, R, st)
}


}  // namespace isy
