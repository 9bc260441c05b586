// Sorted-marginal path for small windows (64 < w <= 256): one warp per window.  The warp sorts the
// window in registers (warp_sort: E = w/32 keys per lane, shuffle bitonic), writes the scan layout to
// its shared-memory slice, and runs the same exact phase A (outward k-NN scan, warp work queue) and
// phase B (binary-search counts) as the large-window path — no block barrier anywhere.  Replaces the
// O(w^2) brute force with O(w log w + w sqrt(k w)) work where that is cheaper.
#include "ksg_device.cuh"

namespace isy {
namespace {

template <int K1, int E, bool V2>
__global__ void __launch_bounds__(kSmallWarps * 32)
    warp_sorted_kernel(const KsgLaunch L, const int32_t* __restrict__ list, int32_t n) {
    constexpr int N = 32 * E;
    __shared__ __align__(16) float2 sP2[kSmallWarps][N + 2 * kScanB];  // kScanB sentinels on either side
    __shared__ float sYS[kSmallWarps][N];
    __shared__ int32_t sOX[kSmallWarps][N];
    __shared__ float seps[kSmallWarps][N];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int idx = blockIdx.x * kSmallWarps + warp;
    if (idx >= n) return;  // warp-uniform
    poison_warp(L, sP2[warp], sizeof(sP2[0]));
    poison_warp(L, sYS[warp], sizeof(sYS[0]));
    poison_warp(L, sOX[warp], sizeof(sOX[0]));
    poison_warp(L, seps[warp], sizeof(seps[0]));
    const int q = list[idx];
    const KsgWin W = L.wins[q];
    const int w = W.w;
    const float* gx = L.pairs[W.pair].x + W.t0;
    const float* gy = L.pairs[W.pair].y + W.t0;
    unsigned long long vx[E];
    unsigned vy[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int i = lane * E + e;
        vx[e] = i < w ? ((unsigned long long)sortable(gx[i]) << 32) | (unsigned)i : ~0ull;
        vy[e] = i < w ? sortable(gy[i]) : ~0u;
    }
    warp_sort<unsigned long long, E>(vx, lane);
    warp_sort<unsigned, E>(vy, lane);
    float2* P2 = sP2[warp] + kScanB;
    if (lane < 2 * kScanB) put_sentinels(P2, w, lane);
    int32_t* OX = sOX[warp];
    float* YS = sYS[warp];
#pragma unroll
    for (int e = 0; e < E; ++e) {
        const int m = lane * E + e;
        if (m < w) {
            const int32_t i = (int32_t)(vx[e] & 0xffffffffu);
            P2[m] = make_float2(unsortable((unsigned)(vx[e] >> 32)), gy[i]);
            OX[m] = i;
            YS[m] = unsortable(vy[e]);
        }
    }
    __syncwarp();
    unsigned long long steps = 0;
    sorted_phase_a<K1>(P2, w, 0, 0, w, seps[warp], steps, nullptr, L.scan_unified != 0);
    __syncwarp();
    long long sp = 0, sl = 0;
    int z = 0;
    for (int m = lane; m < w; m += 32) sorted_phase_b<V2>(L, w, W.dbg_off, P2, OX, YS, m, seps[warp][m], sp, sl, z);
    warp_sum(sp, sl, z);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) steps += __shfl_down_sync(0xffffffffu, steps, off);
    if (lane == 0) finalize(L, w, sp, sl, z, &L.out[q], steps);
}

template <int K1, bool V2>
cudaError_t wsorted_kv(const KsgLaunch& L, const int32_t* list, int32_t n, int E, cudaStream_t st) {
    const dim3 grid((n + kSmallWarps - 1) / kSmallWarps), block(kSmallWarps * 32);
    switch (E) {
        case 2: warp_sorted_kernel<K1, 2, V2><<<grid, block, 0, st>>>(L, list, n); break;
        case 4: warp_sorted_kernel<K1, 4, V2><<<grid, block, 0, st>>>(L, list, n); break;
        case 8: warp_sorted_kernel<K1, 8, V2><<<grid, block, 0, st>>>(L, list, n); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <int K1>
cudaError_t wsorted_k(const KsgLaunch& L, const int32_t* list, int32_t n, int E, cudaStream_t st) {
    return L.variant == 1 ? wsorted_kv<K1, true>(L, list, n, E, st) : wsorted_kv<K1, false>(L, list, n, E, st);
}

}  // namespace

cudaError_t launch_wsorted(const KsgLaunch& L, const int32_t* list, int32_t n, int E, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    ISY_K_CASES(wsorted_k, L, list, n, E, st)
}

}  // namespace isy
