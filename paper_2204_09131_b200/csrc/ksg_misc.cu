// Digamma tables, input validation, size-class helpers, shared-memory opt-in.
#include <mutex>
#include <set>
#include <tuple>

#include "ksg_device.cuh"

namespace isy {


namespace {
// ------------------------------------------------------------------ digamma tables, input validation
__global__ void inv_kernel(double* inv, int64_t m_max) {
    const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m >= 1 && m <= m_max) inv[m] = __ddiv_rn(1.0, (double)m);
}

// psi(1) = -gamma; psi(m+1) = psi(m) + 1/m, strictly sequential (the canonical definition).
__global__ void psi_scan_kernel(double* psi, const double* __restrict__ inv, int64_t m_max, double* lnc) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    lnc[0] = 0.0;
    for (int j = 1; j <= 9; ++j) lnc[j] = __ddiv_rn(1.0, (double)(2 * j + 1));  // LN series coefficients
    psi[0] = __longlong_as_double(0x7FF8000000000000LL);
    double v = -0.57721566490153286061;
    psi[1] = v;
    // the additions stay strictly sequential (the canonical table); the 1/m terms of the next chunk
    // are loaded while the current chunk is summed, so the loop runs at the DADD chain's latency instead of a
    // global load round trip per term (2.8 -> ~1 ms per process start)
    constexpr int C = 16;
    int64_t m = 1;
    if (m_max > C) {
        double cur[C], nxt[C];
#pragma unroll
        for (int u = 0; u < C; ++u) cur[u] = inv[m + u];
        for (; m + 2 * C <= m_max; m += C) {
#pragma unroll
            for (int u = 0; u < C; ++u) nxt[u] = inv[m + C + u];
#pragma unroll
            for (int u = 0; u < C; ++u) {
                v = __dadd_rn(v, cur[u]);
                psi[m + u + 1] = v;
            }
#pragma unroll
            for (int u = 0; u < C; ++u) cur[u] = nxt[u];
        }
#pragma unroll
        for (int u = 0; u < C; ++u) {  // the last full chunk (m + C <= m_max here)
            v = __dadd_rn(v, cur[u]);
            psi[m + u + 1] = v;
        }
        m += C;
    }
    for (; m < m_max; ++m) {
        v = __dadd_rn(v, inv[m]);
        psi[m + 1] = v;
    }
}

__global__ void psiq_kernel(const double* psi, long long* psiq, int64_t m_max) {
    const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (m == 0) psiq[0] = 0;
    if (m >= 1 && m <= m_max) psiq[m] = q32(psi[m]);
}

__global__ void nonfinite_kernel(const float* __restrict__ p, int64_t n, int* flag) {
    int bad = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        bad |= !isfinite(p[i]);
    if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

}  // namespace

cudaError_t launch_psi_tables(double* psi, long long* psiq, double* inv, int64_t m_max, double* lnc,
                              cudaStream_t st) {
    const int64_t blocks = (m_max + 1 + 255) / 256;
    inv_kernel<<<(unsigned)blocks, 256, 0, st>>>(inv, m_max);
    psi_scan_kernel<<<1, 32, 0, st>>>(psi, inv, m_max, lnc);
    psiq_kernel<<<(unsigned)blocks, 256, 0, st>>>(psi, psiq, m_max);
    return cudaGetLastError();
}

cudaError_t launch_nonfinite_scan(const float* p, int64_t n, int* flag, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    nonfinite_kernel<<<(unsigned)blocks, 256, 0, st>>>(p, n, flag);
    return cudaGetLastError();
}


cudaError_t smem_optin(const void* kernel, int bytes) {
    static std::mutex mu;
    static std::set<std::tuple<int, const void*, int>> done;
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_tuple(dev, kernel, bytes);
    if (done.count(key)) return cudaSuccess;
    e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert(key);
    return e;
}

}  // namespace isy
