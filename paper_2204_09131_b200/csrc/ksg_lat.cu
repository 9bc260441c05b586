// Latency mode for small windows (w <= 256) in rounds too sparse to fill the GPU (a1-a6, KSG-1).
//
// The search rounds of a BU climb carry a few hundred small windows; one thread walking all w candidates
// of its point sets the round's latency.  Here every point is owned by P = 8 lanes of a warp (P = 4 for windows of
// at most 128 points: fewer CTAs and one butterfly step less where each lane has few candidates): lane s
// scans the candidate groups g = s, s + 8, ... (4 candidates per float4 group) with its own register
// top-(k+1) list, the 8 lists (self's 0 removed: k entries each) are merged by a 3-step butterfly (bitonic
// merge networks for k = 4, 8: after the xor-1/2/4 exchanges every lane holds the k smallest of the union over
// j != i — the same multiset order statistic as one lane scanning everything), then the marginal counts are split the same
// way and summed by shuffles.  The critical path per window drops ~8x; results are bit-identical.
// Tiny windows (w <= 32) of the round ride in the same launch as extra CTAs, one warp per window.
#include "ksg_device.cuh"

namespace isy {
namespace {

constexpr int kLatThreads = 256;

constexpr int kLat4Flag = 1 << 30;                   // KsgItem.i0 flag: 4 lanes per point

// The points [i0, i0 + 256 / P) of window q, P lanes per point, candidates in sx / sy (staged by the CTA).
template <int K1, int P>
__device__ __forceinline__ void lat_points(const KsgLaunch& L, int q, const KsgWin& W, int i0, const float* sx,
                                           const float* sy) {
    constexpr int kPts = kLatThreads / P;
    const int w = W.w;
    const int wpad = (w + 3) & ~3;
    const int s = threadIdx.x & (P - 1);
    const int i = i0 + (int)(threadIdx.x / P);
    const bool live = i < w;
    const float xi0 = live ? sx[i] : 0.0f, yi0 = live ? sy[i] : 0.0f;
    float xi[1] = {xi0}, yi[1] = {yi0};
    float rk[1][K1];
#pragma unroll
    for (int m = 0; m < K1; ++m) rk[0][m] = kInf;
    const int ng = wpad >> 2;
    const float4* sx4 = reinterpret_cast<const float4*>(sx);
    const float4* sy4 = reinterpret_cast<const float4*>(sy);
    for (int g = s; g < ng; g += P) knn_step<K1, 1, false>(xi, yi, rk, sx4[g], sy4[g]);
    // Drop self before merging: the lane that scanned j = i (group i/4 -> lane (i/4) mod P) holds the K1 smallest
    // of its candidates including d_ii = 0 at the front; removing that one 0 leaves the K = k smallest of the
    // others.  Every other lane keeps its first K.  The merged K-lists then give eps = the k-th smallest over
    // j != i = the (k+1)-th of the multiset with self, and K = 4 / 8 merge by bitonic networks.
    constexpr int K = K1 - 1;
    const bool self_lane = s == ((i >> 2) & (P - 1));
    float rl[K];
#pragma unroll
    for (int m = 0; m < K; ++m) rl[m] = self_lane ? rk[0][m + 1] : rk[0][m];
    // butterfly merge of the P partial top lists (lanes of one point are P consecutive lanes)
#pragma unroll
    for (int off = 1; off < P; off <<= 1) {
        float other[K];
#pragma unroll
        for (int m = 0; m < K; ++m) other[m] = __shfl_xor_sync(0xffffffffu, rl[m], off);
        topk_merge_sorted<K>(rl, other);
    }
    float eps[1] = {rl[K - 1]};
    unsigned cx[1] = {0u}, cy[1] = {0u};
    for (int g = s; g < ng; g += P) count_step<1>(xi, yi, eps, eps, cx, cy, sx4[g], sy4[g], (unsigned)L.two);
#pragma unroll
    for (int off = 1; off < P; off <<= 1) {
        cx[0] += __shfl_xor_sync(0xffffffffu, cx[0], off);
        cy[0] += __shfl_xor_sync(0xffffffffu, cy[0], off);
    }
    long long sp = 0, sl = 0;
    int z = 0;
    if (s == 0 && live) point_terms<1, false>(L, w, W.dbg_off, i, kPts, eps, cx, cy, sp, sl, z);
    cta_finish(L, q, w, (w + kPts - 1) / kPts, sp, sl, z, 0ull);
}

constexpr int kTinyCap = 36;                          // per-warp slice of a tiny window (w <= 32, +4 pad)

#ifdef ISY_LAT_MINB  // A/B knob: resident CTAs per SM the register allocation must allow (measured)
#define ISY_LAT_BOUNDS __launch_bounds__(kLatThreads, ISY_LAT_MINB)
#else
#define ISY_LAT_BOUNDS __launch_bounds__(kLatThreads)
#endif
template <int K1>
__global__ void ISY_LAT_BOUNDS
    ksg_lat_kernel(const KsgLaunch L, const KsgItem* __restrict__ items, int32_t n_items,
                   const int32_t* __restrict__ tiny, int32_t n_tiny) {
    __shared__ __align__(16) float sx[kSmallWarps * kTinyCap];  // >= 256
    __shared__ __align__(16) float sy[kSmallWarps * kTinyCap];
    if (L.poison) {
        poison_smem(L, sx, sizeof(sx));
        poison_smem(L, sy, sizeof(sy));
        __syncthreads();
    }
    if ((int)blockIdx.x >= n_items) {
        // tiny windows (w <= 32) of the same round: one warp per window, one point per lane (the small kernel's
        // R = 1 body) — 8 lanes per point would leave most lanes idle and pay the list merge for a few candidates;
        // sharing the launch keeps one latency-mode launch per round
        const int warp = threadIdx.x >> 5;
        const int idx = ((int)blockIdx.x - n_items) * kSmallWarps + warp;
        if (idx >= n_tiny) return;  // warp-uniform; no block barrier on this path
        small_window_warp<K1, 1, true, false>(L, tiny[idx], sx + warp * kTinyCap, sy + warp * kTinyCap);
        return;
    }
    const KsgItem it = items[blockIdx.x];
    const int q = it.win;
    const KsgWin W = L.wins[q];
    const int w = W.w;
    const float* gx = L.pairs[W.pair].x + W.t0;
    const float* gy = L.pairs[W.pair].y + W.t0;
    const int wpad = (w + 3) & ~3;
    for (int j = threadIdx.x; j < wpad; j += kLatThreads) {
        sx[j] = j < w ? gx[j] : kInf;  // +inf pads: d = +inf, never inserted, never counted
        sy[j] = j < w ? gy[j] : kInf;
    }
    __syncthreads();
    // lanes per point: 4 for windows up to lat_lanes_w4 points (item flag bit 30; 64 points per CTA), else 8
    if (it.i0 & kLat4Flag)
        lat_points<K1, 4>(L, q, W, it.i0 & ~kLat4Flag, sx, sy);
    else
        lat_points<K1, 8>(L, q, W, it.i0, sx, sy);
}

template <int K1>
cudaError_t lat_k(const KsgLaunch& L, const KsgItem* items, int32_t n, const int32_t* tiny, int32_t n_tiny,
                  cudaStream_t st) {
    const int grid = n + (n_tiny + kSmallWarps - 1) / kSmallWarps;
    ksg_lat_kernel<K1><<<grid, kLatThreads, 0, st>>>(L, items, n, tiny, n_tiny);
    return cudaGetLastError();
}

}  // namespace

int lat_points_per_cta(int lanes) { return kLatThreads / lanes; }
int32_t lat_item_flag(int lanes) { return lanes == 4 ? kLat4Flag : 0; }

cudaError_t launch_ksg_lat(const KsgLaunch& L, const KsgItem* items, int32_t n_items, const int32_t* tiny,
                           int32_t n_tiny, cudaStream_t st) {
    if (n_items <= 0 && n_tiny <= 0) return cudaSuccess;
    if (L.variant != 0) return cudaErrorInvalidValue;  // KSG-2 latency windows take the tile kernel (R = 1)
    ISY_K_CASES(lat_k, L, items, n_items, tiny, n_tiny, st)
}

}  // namespace isy
