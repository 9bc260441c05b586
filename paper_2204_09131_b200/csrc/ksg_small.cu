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
    const int warp = threadIdx.x >> 5;
    const int idx = blockIdx.x * kSmallWarps + warp;
    if (idx >= n) return;  // warp-uniform
    poison_warp(L, sbuf[warp], sizeof(sbuf[0]));
    small_window_warp<K1, R, BL, V2>(L, list[idx], sbuf[warp][0], sbuf[warp][1]);
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
