// Sorted-marginal path, throughput form: sort kernel (+ XL rank merge) into
// global scratch, then the scan kernel.
#include "ksg_device.cuh"

namespace isy {
namespace {

// NEXT-3 (the GPU analogue of the paper's incremental MI): windows of one (pair, size) on a
// common grid share their beta-point blocks; block_sort_kernel sorts every block ONCE per batch (x keys with
// the absolute sample index, y keys), and the window's sort below starts from those sorted runs: it only
// runs the merge levels from beta up (a delta-shifted window re-merges the blocks it shares with its
// neighbours instead of re-sorting them).  Same keys, same total order: bit-identical layouts.
__global__ void __launch_bounds__(1024) block_sort_kernel(const KsgLaunch L, const KsgBlk* __restrict__ blks,
                                                          unsigned long long* __restrict__ BX,
                                                          unsigned* __restrict__ BY) {
    extern __shared__ __align__(16) unsigned char sm[];
    if (L.poison) {
        poison_smem(L, sm, dyn_smem_bytes());
        __syncthreads();
    }
    const KsgBlk B = blks[blockIdx.x];
    const int n2 = B.beta;  // power of two in [256, kSortedMaxW]
    const float* gx = L.pairs[B.pair].x + B.t;
    const float* gy = L.pairs[B.pair].y + B.t;
    unsigned long long* X0 = reinterpret_cast<unsigned long long*>(sm);
    unsigned long long* X1 = X0 + n2;
    unsigned* Y0 = reinterpret_cast<unsigned*>(X1 + n2);
    unsigned* Y1 = reinterpret_cast<unsigned*>(X0);  // y merges through the x buffers once x is out
    chunk_sort<8>(gx, gy, n2, n2, X0, Y0, nullptr, threadIdx.x >> 5, threadIdx.x & 31, (int)B.t);
    __syncthreads();
    unsigned long long* xs = X0;
    unsigned long long* xd = X1;
    for (int r = 256; r < n2; r <<= 1) {
        merge_level(xs, xd, n2, r);
        __syncthreads();
        unsigned long long* tx = xs;
        xs = xd;
        xd = tx;
    }
    for (int m = threadIdx.x; m < n2; m += blockDim.x) BX[B.boff + m] = xs[m];
    __syncthreads();
    unsigned* ys = Y0;
    unsigned* yd = Y1;
    for (int r = 256; r < n2; r <<= 1) {
        merge_level(ys, yd, n2, r);
        __syncthreads();
        unsigned* ty = ys;
        ys = yd;
        yd = ty;
    }
    for (int m = threadIdx.x; m < n2; m += blockDim.x) BY[B.boff + m] = ys[m];
}

__global__ void __launch_bounds__(1024) sort_window_kernel(const KsgLaunch L, const int32_t* __restrict__ list,
                                   const int64_t* __restrict__ soff, const KsgItem* __restrict__ segs,
                                   float2* __restrict__ P2, int32_t* __restrict__ OX, float* __restrict__ YS,
                                   float* __restrict__ TX, int32_t* __restrict__ TI, float* __restrict__ TY,
                                   int W2, const KsgSegB* __restrict__ segb,
                                   const unsigned long long* __restrict__ BX, const unsigned* __restrict__ BY) {
    extern __shared__ __align__(16) unsigned char sm[];
    if (L.poison) {
        poison_smem(L, sm, dyn_smem_bytes());
        __syncthreads();
    }
    const KsgItem sg = segs[blockIdx.x];  // win = position in the sorted list, i0 = segment start
    const int b = sg.win;
    const int q = list[b];
    const KsgWin W = L.wins[q];
    const int w = W.w;
    const int s0 = sg.i0;
    const int len = min(kSortedMaxW, w - s0);
    const bool whole = (s0 == 0 && len == w);
    int n2 = 1;
    while (n2 < len) n2 <<= 1;
    const float* gx = L.pairs[W.pair].x + W.t0;
    const float* gy = L.pairs[W.pair].y + W.t0;
    const int64_t o = soff[b];  // the window's region has kScanB spare entries on either side (scan sentinels)
    if (s0 == 0 && threadIdx.x < 2 * kScanB) put_sentinels(P2 + o, w, threadIdx.x);
    const KsgSegB sb = segb ? segb[blockIdx.x] : KsgSegB{0, 0, 0};
    if (n2 >= 256) {
        // register chunk sorts (256 keys per warp) + merge-path levels in SMEM (the fused kernel's sort, ~2x
        // the SMEM-bandwidth-bound bitonic below).  x (with the window index) is merged and written out
        // first, then y is merged through the freed x buffers: 20 n2 bytes of SMEM.  Block mode: the runs of
        // beta keys come sorted from block_sort_kernel (x keys carry the absolute index t0 + i).
        unsigned long long* X0 = reinterpret_cast<unsigned long long*>(sm);
        unsigned long long* X1 = X0 + n2;
        unsigned* Y0 = reinterpret_cast<unsigned*>(X1 + n2);
        int r0 = 256;
        unsigned isub = 0;  // index base of the keys (block mode: absolute sample index)
        if (sb.beta > 0) {
            for (int m = threadIdx.x; m < n2; m += blockDim.x) {
                X0[m] = m < len ? BX[sb.boff + m] : ~0ull;
                Y0[m] = m < len ? BY[sb.boff + m] : ~0u;
            }
            r0 = sb.beta;
            isub = (unsigned)W.t0;
        } else {
            chunk_sort<8>(gx + s0, gy + s0, len, n2, X0, Y0, nullptr, threadIdx.x >> 5, threadIdx.x & 31, s0);
        }
        __syncthreads();
        unsigned long long* xs = X0;
        unsigned long long* xd = X1;
        for (int r = r0; r < n2; r <<= 1) {
            merge_level(xs, xd, n2, r);
            __syncthreads();
            unsigned long long* tx = xs;
            xs = xd;
            xd = tx;
        }
        for (int m = threadIdx.x; m < len; m += blockDim.x) {
            const unsigned long long v = xs[m];
            const float xv = unsortable((unsigned)(v >> 32));
            const int32_t idx = (int32_t)((unsigned)(v & 0xffffffffu) - isub);
            if (whole) {
                P2[o + m] = make_float2(xv, gy[idx]);
                OX[o + m] = idx;
            } else {
                TX[o + s0 + m] = xv;
                TI[o + s0 + m] = idx;
            }
        }
        __syncthreads();
        unsigned* ys = Y0;
        unsigned* yd = reinterpret_cast<unsigned*>(X0);  // x buffers are free now
        for (int r = r0; r < n2; r <<= 1) {
            merge_level(ys, yd, n2, r);
            __syncthreads();
            unsigned* ty = ys;
            ys = yd;
            yd = ty;
        }
        for (int m = threadIdx.x; m < len; m += blockDim.x) {
            const float yv = unsortable(ys[m]);
            if (whole)
                YS[o + m] = yv;
            else
                TY[o + s0 + m] = yv;
        }
        return;
    }
    // pass 0: x with the index packed into one 64-bit word (sortable float bits << 32 | index): one
    // compare/swap per exchange, ties broken by index.  pass 1: y keys alone (32-bit).
    unsigned long long* k64 = reinterpret_cast<unsigned long long*>(sm);
    unsigned* k32 = reinterpret_cast<unsigned*>(sm);
    for (int i = threadIdx.x; i < n2; i += blockDim.x)
        k64[i] = i < len ? ((unsigned long long)sortable(gx[s0 + i]) << 32) | (unsigned)(s0 + i) : ~0ull;
    __syncthreads();
    bitonic_smem(k64, n2);
    for (int m = threadIdx.x; m < len; m += blockDim.x) {
        const unsigned long long v = k64[m];
        const float xv = unsortable((unsigned)(v >> 32));
        const int32_t idx = (int32_t)(v & 0xffffffffu);
        if (whole) {
            P2[o + m] = make_float2(xv, gy[idx]);
            OX[o + m] = idx;
        } else {
            TX[o + s0 + m] = xv;
            TI[o + s0 + m] = idx;
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n2; i += blockDim.x) k32[i] = i < len ? sortable(gy[s0 + i]) : ~0u;
    __syncthreads();
    bitonic_smem(k32, n2);
    for (int m = threadIdx.x; m < len; m += blockDim.x) {
        const float yv = unsortable(k32[m]);
        if (whole)
            YS[o + m] = yv;
        else
            TY[o + s0 + m] = yv;
    }
}

__global__ void rank_merge_kernel(const KsgLaunch L, const int32_t* __restrict__ list,
                                  const int64_t* __restrict__ soff, const KsgItem* __restrict__ blocks,
                                  float2* __restrict__ P2, int32_t* __restrict__ OX, float* __restrict__ YS,
                                  const float* __restrict__ TX, const int32_t* __restrict__ TI,
                                  const float* __restrict__ TY) {
    const KsgItem bk = blocks[blockIdx.x];  // win = list position, i0 = first element of this block
    const int b = bk.win;
    const KsgWin W = L.wins[list[b]];
    const int w = W.w;
    const int p = bk.i0 + threadIdx.x;
    if (p >= w) return;
    const int64_t o = soff[b];
    const float* gy = L.pairs[W.pair].y + W.t0;
    const int c = p / kSortedMaxW;
    const int nruns = (w + kSortedMaxW - 1) / kSortedMaxW;
    const float vx = TX[o + p], vy = TY[o + p];
    int rx = p - c * kSortedMaxW, ry = rx;
    for (int c2 = 0; c2 < nruns; ++c2) {
        if (c2 == c) continue;
        const int st = c2 * kSortedMaxW;
        const int n = min(kSortedMaxW, w - st);
        rx += count_below(TX + o + st, n, vx, c2 < c);
        ry += count_below(TY + o + st, n, vy, c2 < c);
    }
    const int32_t idx = TI[o + p];
    P2[o + rx] = make_float2(vx, gy[idx]);
    OX[o + rx] = idx;
    YS[o + ry] = vy;
}

// Box-assisted phase A (sorted_phase_a_cols): each scan item's columns of kColW consecutive x-sorted points, sorted
// by y into CY as (y, x) — one warp per column (a 32-key register bitonic sort, keys y with the lane as payload).
__global__ void __launch_bounds__(kSortedThreads)
    column_sort_kernel(const KsgLaunch L, const int32_t* __restrict__ list, const int64_t* __restrict__ soff,
                       const float2* __restrict__ P2g, float2* __restrict__ CYg, const KsgItem* __restrict__ items) {
    static_assert(kColW == 32, "one warp per column");
    const KsgItem it = items[blockIdx.x];
    const int b = it.win;
    const int w = L.wins[list[b]].w;
    if (w < L.col_min_w) return;  // block-uniform
    const int64_t o = soff[b];
    const int n = min(L.sorted_ppc, w - it.i0);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int c0 = it.i0 + warp * kColW; c0 < it.i0 + n; c0 += nw * kColW) {
        const int p = c0 + lane;
        const float2 v = p < w ? P2g[o + p] : make_float2(0.0f, 0.0f);
        unsigned long long key[1] = {p < w ? ((unsigned long long)sortable(v.y) << 32) | (unsigned)lane : ~0ull};
        warp_sort<unsigned long long, 1>(key, lane);
        const int src = (int)(key[0] & 31u);
        const float vx = __shfl_sync(0xffffffffu, v.x, src), vy = __shfl_sync(0xffffffffu, v.y, src);
        if (p < w) CYg[o + p] = make_float2(vy, vx);
    }
}

// first index in [lo, hi) where pred is false, for pred true...true false...false
// left side: smallest j in [0, m] with fl(v - s[j]) < eps (pred false...true)
template <int K1, bool V2>
__global__ void __launch_bounds__(kSortedThreads)
    sorted_knn_kernel(const KsgLaunch L, const int32_t* __restrict__ list, const int64_t* __restrict__ soff,
                      const float2* __restrict__ P2g, const int32_t* __restrict__ OXg, const float* __restrict__ YSg,
                      const KsgItem* __restrict__ items, const KsgInc* __restrict__ inc, float* __restrict__ EPS,
                      const unsigned long long* __restrict__ BX, const unsigned* __restrict__ BY,
                      int2* __restrict__ CNT, unsigned* __restrict__ sync, const float2* __restrict__ CYg) {
    const int ppc = L.sorted_ppc;  // points per CTA (runtime: 256 for latency, 1024 for throughput)
    __shared__ float eps_s[kSortedPts];
    __shared__ int2 stop_s[kSortedPts];
    __shared__ uint16_t wl_s[kSortedPts];  // NEXT-3 incremental windows: the points left to scan
    extern __shared__ __align__(16) float inc_sb[];  // NEXT-3: removed / inserted blocks (x, y), 4 d floats
    if (L.poison) {
        poison_smem(L, eps_s, sizeof(eps_s));
        poison_smem(L, stop_s, sizeof(stop_s));
        __syncthreads();
    }
    // NEXT-3 chains: work items (level-major) are taken by ticket, so every item a CTA may wait for was taken by a
    // CTA that is already running (forward progress without co-scheduling guarantees)
    __shared__ int s_item;
    if (sync) {
        if (threadIdx.x == 0) s_item = (int)atomicAdd(sync, 1u);
        __syncthreads();
    }
    const KsgItem it = items[sync ? s_item : blockIdx.x];  // it.win = position in the sorted list, it.i0 = first point
    const int b = it.win;
    const int q = list[b];
    const int w = L.wins[q].w;
    const int64_t o = soff[b];
    const KsgInc* ic = inc ? &inc[b] : nullptr;
    const bool chain = ic && ic->level >= 0;
    sorted_scan<K1, V2>(L, q, w, (w + ppc - 1) / ppc, P2g + o, OXg + o, YSg + o, it.i0, min(ppc, w - it.i0), eps_s,
                        stop_s, chain && ic->level > 0 ? ic : nullptr,
                        chain && ic->level > 0 ? EPS + ic->eps_prev : nullptr, chain ? EPS + o : nullptr, BX, wl_s,
                        inc_sb, BY, chain && ic->level > 0 ? CNT + ic->eps_prev : nullptr, chain ? CNT + o : nullptr,
                        sync ? sync + 1 : nullptr, b, CYg ? CYg + o : nullptr);
}

template <int K1>
cudaError_t sorted_k(const KsgLaunch& L, const int32_t* list, const int64_t* soff, const float2* P2,
                     const int32_t* OX, const float* YS, const KsgItem* items, int32_t n_items, cudaStream_t st,
                     const KsgInc* inc, float* EPS, const unsigned long long* BX, const unsigned* BY, int2* CNT,
                     const int32_t* lv_off, int n_lv, int inc_d_max, unsigned* sync, const float2* CY) {
    // NEXT-3 chains: one launch over the level-ordered items; a level-j window's CTAs wait (per window) for the
    // level-(j-1) predecessor's CTAs, which took earlier work tickets (no per-level launch tails)
    (void)lv_off;
    const bool chains = n_lv > 1 && sync;
    const size_t smem = chains ? (size_t)6 * inc_d_max * sizeof(float) : 0;  // the two staged blocks
    unsigned* sy = chains ? sync : nullptr;
    if (L.variant == 1)
        sorted_knn_kernel<K1, true><<<n_items, kSortedThreads, smem, st>>>(L, list, soff, P2, OX, YS, items, inc, EPS,
                                                                           BX, BY, CNT, sy, CY);
    else
        sorted_knn_kernel<K1, false><<<n_items, kSortedThreads, smem, st>>>(L, list, soff, P2, OX, YS, items, inc, EPS,
                                                                            BX, BY, CNT, sy, CY);
    return cudaGetLastError();
}
}  // namespace

cudaError_t launch_sorted(const KsgLaunch& L, const int32_t* list, const int64_t* soff, const KsgItem* segs,
                          int32_t n_segs, const KsgItem* mblocks, int32_t n_mblocks, float2* P2, int32_t* OX,
                          float* YS, float* TX, int32_t* TI, float* TY, int W2, const KsgItem* items,
                          int32_t n_items, cudaStream_t st, const KsgSegB* segb, const KsgBlk* blks,
                          int32_t n_blks, int blk_beta_max, unsigned long long* BX, unsigned* BY, const KsgInc* inc,
                          float* EPS, int2* CNT, const int32_t* lv_off, int n_lv, int inc_d_max,
                          unsigned* sync, float2* CY) {
    static_assert(kSortedPts % (kSortedThreads / 32) == 0, "scan CTA size");
    if (n_segs <= 0) return cudaSuccess;
    {
        cudaError_t e = smem_optin(reinterpret_cast<const void*>(sort_window_kernel), kSortedMaxW * 20);
        if (e != cudaSuccess) return e;
        e = smem_optin(reinterpret_cast<const void*>(block_sort_kernel), kSortedMaxW * 20);
        if (e != cudaSuccess) return e;
    }
    if (n_blks > 0) {  // NEXT-3 shared blocks: sorted once, before the windows that merge them
        const int bt = std::min(1024, std::max(64, blk_beta_max / 8));
        block_sort_kernel<<<n_blks, bt, (size_t)blk_beta_max * 20, st>>>(L, blks, BX, BY);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    // one thread per 8 keys (= one merge-path output run; chunk sorts are 256 keys per warp): smaller CTAs
    // for small segments keep every warp busy and let more CTAs share an SM
    const int threads = std::min(1024, std::max(64, W2 / 8));
    const size_t smem = (size_t)W2 * 20;  // chunk + merge sort (bitonic for n2 < 256 needs 8 n2)
    sort_window_kernel<<<n_segs, threads, smem, st>>>(L, list, soff, segs, P2, OX, YS, TX, TI, TY, W2,
                                                      n_blks > 0 ? segb : nullptr, BX, BY);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    if (n_mblocks > 0) {
        rank_merge_kernel<<<n_mblocks, kMergeThreads, 0, st>>>(L, list, soff, mblocks, P2, OX, YS, TX, TI, TY);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    if (CY) {  // box-assisted phase A for windows >= L.col_min_w: their y-sorted columns
        column_sort_kernel<<<n_items, kSortedThreads, 0, st>>>(L, list, soff, P2, CY, items);
        e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    ISY_K_CASES(sorted_k, L, list, soff, P2, OX, YS, items, n_items, st, inc, EPS, BX, BY, CNT, lv_off, n_lv, inc_d_max,
                sync, CY)
}


}  // namespace isy
