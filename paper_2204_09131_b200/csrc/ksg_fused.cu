// Sorted-marginal path, latency form: fused in-SMEM sort + scan per (window, slice).
#include "ksg_device.cuh"

namespace isy {
namespace {

// ------------------------------------------------------------------ fused latency path (w <= kFusedMaxW)
// One CTA per (window, slice): load the window, sort it in shared memory, then scan the slice's points
// from shared memory.  Every slice CTA of a window sorts the whole window (redundant work, no scratch
// round trip and no second launch: search rounds are latency-bound).  The sort: each warp sorts 256
// keys held 8 per lane with a register/shuffle bitonic network, then merge-path merges in shared
// memory double the run length up to n2 (next power of two >= w).  x keys carry the window index in
// the low 32 bits (sortable x bits << 32 | index: unique keys, ties of x broken by index); y keys are
// the sortable y bits alone.
// fused items: {list position, slice start}; a window of w points has slices of fused_ppc(w, gmax) points
__device__ __host__ __forceinline__ int fused_ppc_of(int w, int gmax) {
    int g = (w + kFusedThreads - 1) / kFusedThreads;  // at most one point per thread per slice ...
    g = g < gmax ? g : gmax;                          // ... unless the batch already fills the GPU
    g = g < 1 ? 1 : g;
    const int ppc = (w + g - 1) / g;
    return (ppc + 31) & ~31;
}

template <int K1, bool V2>
__global__ void __launch_bounds__(kFusedThreads)
    fused_sorted_kernel(const KsgLaunch L, const int32_t* __restrict__ list, const KsgItem* __restrict__ items,
                        int gmax) {
    extern __shared__ __align__(16) unsigned long long fsm[];
    if (L.poison) {
        poison_smem(L, fsm, dyn_smem_bytes());
        __syncthreads();
    }
    const KsgItem it = items[blockIdx.x];
    const int q = list[it.win];
    const KsgWin W = L.wins[q];
    const int w = W.w;
    int n2 = 256;
    while (n2 < w) n2 <<= 1;
    const int maxn2 = L.fused_n2;  // shared-memory layout stride (batch maximum)
    unsigned long long* X0 = fsm;                         // maxn2 + 2 kScanB entries each: the scan layout P2
    unsigned long long* X1 = fsm + (maxn2 + 2 * kScanB);  // reuses one, with kScanB sentinels on either side
    unsigned* Y0 = reinterpret_cast<unsigned*>(fsm + 2 * (maxn2 + 2 * kScanB));
    unsigned* Y1 = Y0 + maxn2;
    float* eps_s = reinterpret_cast<float*>(Y1 + maxn2);  // maxn2 floats (a slice can be the whole window)
    const float* gx = L.pairs[W.pair].x + W.t0;
    const float* gy = L.pairs[W.pair].y + W.t0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;

    // a2 + sort, step 1: each warp sorts 256-key chunks in registers (8 consecutive keys per lane;
    // smaller chunks with more merge levels measured slower)
    chunk_sort<8>(gx, gy, w, n2, X0, Y0, eps_s, warp, lane);
    __syncthreads();
    // step 2: merge-path levels 256 -> n2 (ping-pong)
    unsigned long long* xs = X0;
    unsigned long long* xd = X1;
    unsigned* ys = Y0;
    unsigned* yd = Y1;
    for (int r = 256; r < n2; r <<= 1) {
        merge_level(xs, xd, n2, r);
        merge_level(ys, yd, n2, r);
        __syncthreads();
        unsigned long long* tx = xs;
        xs = xd;
        xd = tx;
        unsigned* ty = ys;
        ys = yd;
        yd = ty;
    }
    // step 3: scan layout: P2 (x, y) in x order -> the free x buffer, OX -> the free y buffer, YS in place
    float2* P2 = reinterpret_cast<float2*>(xd) + kScanB;
    if (threadIdx.x < 2 * kScanB) put_sentinels(P2, w, threadIdx.x);
    int32_t* OX = reinterpret_cast<int32_t*>(yd);
    float* YS = reinterpret_cast<float*>(ys);
    for (int m = threadIdx.x; m < w; m += kFusedThreads) {
        const unsigned long long v = xs[m];
        const int32_t idx = (int32_t)(v & 0xffffffffu);
        P2[m] = make_float2(unsortable((unsigned)(v >> 32)), eps_s[idx]);
        OX[m] = idx;
        YS[m] = unsortable(ys[m]);
    }
    __syncthreads();
    const int ppc = fused_ppc_of(w, gmax);
    // the final sorted x keys (xs) are dead after the layout build: phase A's stop indices go there
    sorted_scan<K1, V2>(L, q, w, (w + ppc - 1) / ppc, P2, OX, YS, it.i0, min(ppc, w - it.i0), eps_s,
                        reinterpret_cast<int2*>(xs));
}

template <int K1>
cudaError_t fused_k(const KsgLaunch& L, const int32_t* list, const KsgItem* items, int32_t n_items, int gmax,
                    cudaStream_t st) {
    const size_t smem = (size_t)L.fused_n2 * 28 + 32 * kScanB;
    if (L.variant == 1)
        fused_sorted_kernel<K1, true><<<n_items, kFusedThreads, smem, st>>>(L, list, items, gmax);
    else
        fused_sorted_kernel<K1, false><<<n_items, kFusedThreads, smem, st>>>(L, list, items, gmax);
    return cudaGetLastError();
}

}  // namespace

template <int K1, bool V2>
cudaError_t fused_attr() {
    return smem_optin(reinterpret_cast<const void*>(fused_sorted_kernel<K1, V2>), kFusedMaxW * 28 + 32 * kScanB);
}
template <int K1>
cudaError_t fused_attr_k(const KsgLaunch&) {
    cudaError_t e = fused_attr<K1, false>();
    return e != cudaSuccess ? e : fused_attr<K1, true>();
}

cudaError_t launch_fused(const KsgLaunch& L, const int32_t* list, const KsgItem* items, int32_t n_items, int gmax,
                         cudaStream_t st) {
    if (n_items <= 0) return cudaSuccess;
    if (L.k < 1 || L.k > 16) return cudaErrorInvalidValue;
    {
        cudaError_t e = [&]() -> cudaError_t { ISY_K_CASES(fused_attr_k, L) }();
        if (e != cudaSuccess) return e;
    }
    ISY_K_CASES(fused_k, L, list, items, n_items, gmax, st)
}

int fused_ppc(int w, int gmax) { return fused_ppc_of(w, gmax); }

}  // namespace isy
