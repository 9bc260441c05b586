// Sorted-marginal path for small windows (64 < w <= 256): G warps per window (G = 1, 2, 4).  The window is
// sorted in registers (warp_sort: E = w/32 keys per lane, shuffle bitonic; G > 1: x by one warp, y by another,
// concurrently), the scan layout goes to the group's shared-memory slice, and each warp runs the same exact
// phase A (outward k-NN scan, warp work queue) and phase B (binary-search counts) as the large-window path
// on its 1/G of the points; the G partial int64 sums meet in shared memory behind the group's named barrier.
// G = 1 has no barrier at all.  The host takes G > 1 when the batch leaves most of the GPU idle (a search
// round's few hundred windows: one warp per window walking all w points sets the round's latency).
// Replaces the O(w^2) brute force with O(w log w + w sqrt(k w)) work where that is cheaper.
#include "ksg_device.cuh"

namespace isy {
namespace {

template <int K1, int E, bool V2>
__global__ void __launch_bounds__(kSmallWarps * 32)
    warp_sorted_kernel(const KsgLaunch L, const int32_t* __restrict__ list, int32_t n, int G) {
    constexpr int N = 32 * E;
    __shared__ __align__(16) float2 sP2[kSmallWarps][N + 2 * kScanB];  // kScanB sentinels on either side
    __shared__ float sYS[kSmallWarps][N];
    __shared__ int32_t sOX[kSmallWarps][N];
    __shared__ float seps[kSmallWarps][N];
    __shared__ long long sred[kSmallWarps][4];  // G > 1: per-warp partial sums of a window
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // G warps per window (G = 1, 2, 4): group gi = warp / G owns the window, sub = warp % G is the warp's part
    const int gi = warp / G, sub = warp - gi * G;
    const int idx = blockIdx.x * (kSmallWarps / G) + gi;
    if (idx >= n) return;  // group-uniform: a group's warps leave together (its named barrier is never reached)
    // named barrier of the group's G warps (id 1 + gi; 0 is __syncthreads)
    auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1 + gi), "r"(G * 32) : "memory"); };
    if (sub == 0) {
        poison_warp(L, sP2[gi], sizeof(sP2[0]));
        poison_warp(L, sYS[gi], sizeof(sYS[0]));
        poison_warp(L, sOX[gi], sizeof(sOX[0]));
        poison_warp(L, seps[gi], sizeof(seps[0]));
    }
    if (G > 1) gsync();  // poisoning (if any) before the other warps' writes
    const int q = list[idx];
    const KsgWin W = L.wins[q];
    const int w = W.w;
    const float* gx = L.pairs[W.pair].x + W.t0;
    const float* gy = L.pairs[W.pair].y + W.t0;
    float2* P2 = sP2[gi] + kScanB;
    int32_t* OX = sOX[gi];
    float* YS = sYS[gi];
    // G = 1: the warp sorts x and y; G > 1: warp 0 of the group sorts x (scan layout P2, OX), warp 1 sorts y
    if (sub == 0) {
        unsigned long long vx[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = lane * E + e;
            vx[e] = i < w ? ((unsigned long long)sortable(gx[i]) << 32) | (unsigned)i : ~0ull;
        }
        warp_sort<unsigned long long, E>(vx, lane);
        if (lane < 2 * kScanB) put_sentinels(P2, w, lane);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int m = lane * E + e;
            if (m < w) {
                const int32_t i = (int32_t)(vx[e] & 0xffffffffu);
                P2[m] = make_float2(unsortable((unsigned)(vx[e] >> 32)), gy[i]);
                OX[m] = i;
            }
        }
    }
    if (sub == (G > 1 ? 1 : 0)) {
        unsigned vy[E];
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int i = lane * E + e;
            vy[e] = i < w ? sortable(gy[i]) : ~0u;
        }
        warp_sort<unsigned, E>(vy, lane);
#pragma unroll
        for (int e = 0; e < E; ++e) {
            const int m = lane * E + e;
            if (m < w) YS[m] = unsortable(vy[e]);
        }
    }
    if (G > 1)
        gsync();
    else
        __syncwarp();
    // the window's points split into G contiguous ranges of x positions, one per warp (phase A's warp queue
    // inside each range; phase B reads only the point's own eps, written by the same warp)
    const int per = (w + G - 1) / G;
    const int wb = min(w, sub * per), we = min(w, wb + per);
    unsigned long long steps = 0;
    sorted_phase_a<K1>(P2, w, 0, wb, we, seps[gi], steps, nullptr, L.scan_unified != 0);
    __syncwarp();
    long long sp = 0, sl = 0;
    int z = 0;
    for (int m = wb + lane; m < we; m += 32) sorted_phase_b<V2>(L, w, W.dbg_off, P2, OX, YS, m, seps[gi][m], sp, sl, z);
    warp_sum(sp, sl, z);
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) steps += __shfl_down_sync(0xffffffffu, steps, off);
    if (G > 1) {  // exact int64 sums: the order of the G partials does not matter
        if (lane == 0) {
            sred[warp][0] = sp;
            sred[warp][1] = sl;
            sred[warp][2] = z;
            sred[warp][3] = (long long)steps;
        }
        gsync();
        if (sub != 0) return;
        if (lane == 0)
            for (int u = 1; u < G; ++u) {
                sp += sred[warp + u][0];
                sl += sred[warp + u][1];
                z += (int)sred[warp + u][2];
                steps += (unsigned long long)sred[warp + u][3];
            }
    }
    if (lane == 0) finalize(L, w, sp, sl, z, &L.out[q], steps);
}

template <int K1, bool V2>
cudaError_t wsorted_kv(const KsgLaunch& L, const int32_t* list, int32_t n, int E, int G, cudaStream_t st) {
    const int per_cta = kSmallWarps / G;
    const dim3 grid((n + per_cta - 1) / per_cta), block(kSmallWarps * 32);
    switch (E) {
        case 2: warp_sorted_kernel<K1, 2, V2><<<grid, block, 0, st>>>(L, list, n, G); break;
        case 4: warp_sorted_kernel<K1, 4, V2><<<grid, block, 0, st>>>(L, list, n, G); break;
        case 8: warp_sorted_kernel<K1, 8, V2><<<grid, block, 0, st>>>(L, list, n, G); break;
        default: return cudaErrorInvalidValue;
    }
    return cudaGetLastError();
}

template <int K1>
cudaError_t wsorted_k(const KsgLaunch& L, const int32_t* list, int32_t n, int E, int G, cudaStream_t st) {
    return L.variant == 1 ? wsorted_kv<K1, true>(L, list, n, E, G, st) : wsorted_kv<K1, false>(L, list, n, E, G, st);
}

}  // namespace

cudaError_t launch_wsorted(const KsgLaunch& L, const int32_t* list, int32_t n, int E, int G, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    if (G != 1 && G != 2 && G != 4) return cudaErrorInvalidValue;
    ISY_K_CASES(wsorted_k, L, list, n, E, G, st)
}

}  // namespace isy
