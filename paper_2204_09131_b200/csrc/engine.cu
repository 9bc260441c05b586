// Per-device engine: digamma tables, batch buffers, batch evaluation, profiling.
//
// A batch is a list of windows over one or more series pairs.  Host work per batch is only
// marshalling: bin windows into size classes, pack descriptors into one
// pinned buffer, one H2D copy, one launch per non-empty class, one D2H copy of the records.

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <numeric>
#include <thread>
#include <unordered_map>

#include <chrono>

#include "engine.h"

namespace isy {

// ---------------------------------------------------------------- errors
namespace {
thread_local std::string g_last_error;
}

Status make_err(int code, const std::string& msg) {
    Status s;
    s.code = code;
    s.msg = msg;
    return s;
}

Status cuda_err(cudaError_t e, const char* what) {
    if (e == cudaSuccess) return Status{};
    return make_err(e == cudaErrorMemoryAllocation ? ISYCOS_E_NOMEM : ISYCOS_E_CUDA,
                    std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}

void set_last_error(const Status& s) { g_last_error = s.ok() ? std::string() : s.msg; }

}  // namespace isy

extern "C" const char* isycos_last_error(void) { return isy::g_last_error.c_str(); }

namespace isy {

#define ISY_CK(expr)                                          \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) return cuda_err(_e, #expr);    \
    } while (0)

void BatchStats::add_to(isycos_kernel_stats* s) const {
    if (!s) return;
    s->windows += windows;
    s->point_pairs += point_pairs;
    s->launches += launches;
    s->ksg_launches += ksg_launches;
    s->rounds += rounds;
    s->kernel_ms += kernel_ms;
    s->h2d_bytes += h2d_bytes;
    s->d2h_bytes += d2h_bytes;
    s->host_ms += host_ms;
    s->wall_ms += wall_ms;
    s->scan_steps += scan_steps;
    s->sorted_windows += sorted_windows;
    s->sorted_points += sorted_points;
    s->brute_point_pairs += brute_pairs;
    s->search_probes += search_probes;
    s->sorted_kernel_ms += sorted_ms;
    s->brute_kernel_ms += brute_ms;
    s->profiled_rounds += prof_rounds;
    s->prof_brute_point_pairs += prof_brute_pairs;
    s->prof_scan_steps += prof_scan_steps;
    s->prof_search_probes += prof_probes;
    s->block_windows += block_windows;
    s->block_points += block_points;
    s->inc_windows += inc_windows;
    s->eps_reused_points += eps_reused;
}

// ---------------------------------------------------------------- engine registry (one per device)
namespace {
std::mutex g_mu;
std::map<int, std::unique_ptr<Engine>> g_engines;
}  // namespace

Engine* engine_for_current_device(Status* st) {
    int dev = -1;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) {
        *st = cuda_err(e, "cudaGetDevice (no CUDA device?)");
        return nullptr;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_engines.find(dev);
    if (it != g_engines.end()) return it->second.get();
    cudaDeviceProp prop;
    e = cudaGetDeviceProperties(&prop, dev);
    if (e != cudaSuccess) {
        *st = cuda_err(e, "cudaGetDeviceProperties");
        return nullptr;
    }
    if (prop.major != 10) {
        *st = make_err(ISYCOS_E_CUDA, "libisycos is built for sm_100a (B200); device " + std::to_string(dev) +
                                          " is sm_" + std::to_string(prop.major) + std::to_string(prop.minor));
        return nullptr;
    }
    auto eng = std::make_unique<Engine>();
    Status s = eng->init(dev);
    if (!s.ok()) {
        *st = s;
        return nullptr;
    }
    Engine* p = eng.get();
    g_engines[dev] = std::move(eng);
    return p;
}

void release_engine_for_current_device() {
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    std::lock_guard<std::mutex> lk(g_mu);
    g_engines.erase(dev);
}

Status Engine::init(int dev) {
    dev_ = dev;
    // tuning knobs (defaults are the measured best; see profiles/)
    if (const char* m = std::getenv("ISYCOS_KNN_MODE")) knn_mode_ = std::atoi(m);
    if (const char* m = std::getenv("ISYCOS_SORTED")) sorted_on_ = std::atoi(m) != 0;
    if (const char* m = std::getenv("ISYCOS_SORTED_MIN_W")) sorted_min_w_ = std::atoi(m);
    if (const char* m = std::getenv("ISYCOS_LAT_WINDOWS")) lat_windows_ = std::atoll(m);
    if (const char* m = std::getenv("ISYCOS_LAT_KEEP_SMALL_R")) lat_keep_small_R_ = std::atoi(m);
    if (const char* m = std::getenv("ISYCOS_LAT_TINY_MAX_W")) lat_tiny_max_w_ = std::atoi(m);
    if (const char* m = std::getenv("ISYCOS_COL_MIN_W")) col_min_w_ = std::max(kColW + 1, std::atoi(m));
    if (const char* m = std::getenv("ISYCOS_LAT_LANES4_MAX_W")) lat_lanes4_max_w_ = std::atoi(m);
    if (const char* m = std::getenv("ISYCOS_WS_GROUP")) ws_group_ = std::atoi(m);
    bin_threads_ = (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
    if (const char* m = std::getenv("ISYCOS_BIN_THREADS")) bin_threads_ = std::max(1, std::atoi(m));
    if (const char* m = std::getenv("ISYCOS_FUSED")) fused_on_ = std::atoi(m) != 0;
    if (const char* m = std::getenv("ISYCOS_WSORTED_MIN_W")) wsorted_min_w_ = std::atoi(m);
    if (const char* m = std::getenv("ISYCOS_SORTED_PPC"))
        sorted_ppc_ = std::max(128, std::min(kSortedPts, std::atoi(m)));
    if (const char* m = std::getenv("ISYCOS_FUSED_SMALL_MIN_W")) fused_small_min_w_ = std::atoi(m);
    if (const char* m = std::getenv("ISYCOS_FUSED_MAX_PTS")) fused_max_pts_ = std::atoll(m);
    if (const char* m = std::getenv("ISYCOS_AUX_MIN_WINDOWS")) aux_min_windows_ = std::atoll(m);
    if (const char* m = std::getenv("ISYCOS_BLOCK_SORT")) block_sort_on_ = std::atoi(m) != 0;
    if (const char* m = std::getenv("ISYCOS_LAT_SPLIT")) lat_split_on_ = std::atoi(m) != 0;
    if (const char* m = std::getenv("ISYCOS_INCREMENTAL")) inc_on_ = std::atoi(m) != 0;
    if (const char* m = std::getenv("ISYCOS_INC_CHAIN")) inc_chain_ = std::max(2, std::atoi(m));
    if (const char* m = std::getenv("ISYCOS_SCAN_UNIFIED")) scan_unified_ = std::atoi(m);
    if (const char* m = std::getenv("ISYCOS_POISON")) {  // T5 substitute (compute-sanitizer is closed on the pool)
        const uint32_t b = (uint32_t)std::strtoul(m, nullptr, 0) & 0xffu;
        poison_ = (b * 0x01010101u) | 0x80000000u;  // never 0: the flag is the value
    }
    ISY_CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    ISY_CK(cudaMalloc(&dflag_, sizeof(int)));
    ISY_CK(cudaStreamCreateWithFlags(&stream2_, cudaStreamNonBlocking));
    ISY_CK(cudaEventCreateWithFlags(&xev_, cudaEventDisableTiming));
    for (Slot& S : slots_) {
        ISY_CK(cudaEventCreateWithFlags(&S.fork_ev, cudaEventDisableTiming));
        for (int a = 0; a < kAux; ++a) {
            ISY_CK(cudaStreamCreateWithFlags(&S.aux[a], cudaStreamNonBlocking));
            ISY_CK(cudaEventCreateWithFlags(&S.join_ev[a], cudaEventDisableTiming));
        }
    }
    return Status{};
}

Engine::~Engine() {
    cudaFree(psi_);
    cudaFree(psiq_);
    cudaFree(lnc_);
    cudaFree(dflag_);
    for (Slot& S : slots_) {
        cudaFree(S.acc);
        cudaFree(S.dstage);
        cudaFree(S.ddrec);
        cudaFree(S.sscratch);
        cudaFree(S.sync);
        cudaFreeHost(S.hstage);
        cudaFreeHost(S.hrec);
        for (auto e : S.events) cudaEventDestroy(e);
        for (int a = 0; a < kAux; ++a) {
            if (S.aux[a]) cudaStreamDestroy(S.aux[a]);
            if (S.join_ev[a]) cudaEventDestroy(S.join_ev[a]);
        }
        if (S.fork_ev) cudaEventDestroy(S.fork_ev);
    }
    if (stream2_) cudaStreamDestroy(stream2_);
    if (xev_) cudaEventDestroy(xev_);
    if (stream_) cudaStreamDestroy(stream_);
}

Status Engine::ensure_psi(int64_t w_max, cudaStream_t st) {
    if (psi_max_ >= w_max) return Status{};
    int64_t m = std::max<int64_t>(w_max, 65537);
    m = std::min<int64_t>(std::max<int64_t>(m, psi_max_ * 2), ISYCOS_MAX_W + 1);
    double *psi = nullptr, *inv = nullptr;
    long long* psiq = nullptr;
    ISY_CK(cudaMalloc(&psi, (m + 1) * sizeof(double)));
    ISY_CK(cudaMalloc(&inv, (m + 1) * sizeof(double)));
    ISY_CK(cudaMalloc(&psiq, (m + 1) * sizeof(long long)));
    if (!lnc_) ISY_CK(cudaMalloc(&lnc_, 16 * sizeof(double)));
    ISY_CK(launch_psi_tables(psi, psiq, inv, m, lnc_, st));
    ISY_CK(cudaStreamSynchronize(st));
    cudaFree(inv);
    cudaFree(psi_);
    cudaFree(psiq_);
    psi_ = psi;
    psiq_ = psiq;
    psi_max_ = m;
    return Status{};
}

Status Engine::ensure_capacity(Slot& S, int64_t n_wins, int64_t n_items, int32_t n_pairs, int64_t n_lists,
                               int64_t extra_bytes) {
    if (S.acc_cap < n_wins) {
        int64_t c = std::max<int64_t>(n_wins, S.acc_cap * 2);
        cudaFree(S.acc);
        S.acc = nullptr;
        ISY_CK(cudaMalloc(&S.acc, c * sizeof(KsgAcc)));
        ISY_CK(cudaMemset(S.acc, 0, c * sizeof(KsgAcc)));
        S.acc_cap = c;
    }
    if (S.hrec_cap < n_wins) {  // records: mapped pinned host memory, written by the kernels (zero-copy)
        int64_t c = std::max<int64_t>(n_wins, S.hrec_cap * 2);
        cudaFreeHost(S.hrec);
        S.hrec = nullptr;
        S.drec = nullptr;
        ISY_CK(cudaHostAlloc(&S.hrec, c * sizeof(KsgRec), cudaHostAllocMapped));
        ISY_CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&S.drec), S.hrec, 0));
        S.hrec_cap = c;
    }
    if (n_wins > kZeroCopyMaxRecs && S.ddrec_cap < n_wins) {
        int64_t c = std::max<int64_t>(n_wins, S.ddrec_cap * 2);
        cudaFree(S.ddrec);
        S.ddrec = nullptr;
        ISY_CK(cudaMalloc(&S.ddrec, c * sizeof(KsgRec)));
        S.ddrec_cap = c;
    }
    const int64_t bytes = 64 + n_pairs * (int64_t)sizeof(PairPtrs) + n_wins * (int64_t)sizeof(KsgWin) +
                          n_lists * 4 + n_items * (int64_t)sizeof(KsgItem) + extra_bytes + 16 * 64;
    if (S.dstage_cap < bytes) {
        int64_t c = std::max<int64_t>(bytes, S.dstage_cap * 2);
        cudaFree(S.dstage);
        S.dstage = nullptr;
        ISY_CK(cudaMalloc(&S.dstage, c));
        S.dstage_cap = c;
    }
    if (S.hstage_cap < bytes) {
        int64_t c = std::max<int64_t>(bytes, S.hstage_cap * 2);
        cudaFreeHost(S.hstage);
        S.hstage = nullptr;
        ISY_CK(cudaMallocHost(&S.hstage, c));
        S.hstage_cap = c;
    }
    return Status{};
}

static int64_t align64(int64_t v) { return (v + 63) & ~int64_t(63); }

Status Engine::evaluate(const PairPtrs* pairs, int32_t n_pairs, const KsgWin* wins, int64_t n, int32_t k,
                        int32_t variant, KsgRec* recs_host, const DebugOut& dbg, cudaStream_t st, uint32_t flags,
                        BatchStats* bs) {
    Status s = submit(0, pairs, n_pairs, wins, n, k, variant, dbg, st, flags, bs);
    if (!s.ok()) return s;
    return collect(0, recs_host, bs);
}

Status Engine::submit(int si, const PairPtrs* pairs, int32_t n_pairs, const KsgWin* wins, int64_t n, int32_t k,
                      int32_t variant, const DebugOut& dbg, cudaStream_t st, uint32_t flags, BatchStats* bs) {
    Slot& S = slots_[si];
    if (S.busy) {  // never reuse a slot's staging/record buffers while an earlier batch may still read them
        cudaStreamSynchronize(S.st);
        S.busy = false;
    }
    S.n = 0;
    using sclk = std::chrono::steady_clock;
    const auto t_sub0 = sclk::now();
    const bool profile = (flags & ISYCOS_F_PROFILE) != 0;
    const bool use_sorted = sorted_on_ && !(flags & ISYCOS_F_BRUTE);
    if (n <= 0) return Status{};
    if (n > INT32_MAX / 2) return make_err(ISYCOS_E_INVAL, "batch too large");
    // Binning (a1 on the device side): one pass for w_max and the fused-path point count, one for the size
    // classes.  Large batches (TD layer starts: up to 10^7 windows, memory-bound single-threaded) split both
    // passes into contiguous chunks on host threads; the chunks' class lists are concatenated in chunk order,
    // so every list is in ascending window order exactly as in the serial pass.
    const int n_chunks = n >= (int64_t)1 << 18 ? bin_threads_ : 1;
    auto par = [&](auto&& fn) {
        if (n_chunks == 1) {
            fn(0, (int64_t)0, n);
            return;
        }
        std::vector<std::thread> th;
        for (int c = 1; c < n_chunks; ++c) th.emplace_back(fn, c, n * c / n_chunks, n * (c + 1) / n_chunks);
        fn(0, (int64_t)0, n / n_chunks);
        for (auto& t : th) t.join();
    };
    const bool use_fused_path = use_sorted && fused_on_ && !(flags & ISYCOS_F_UNFUSED);
    std::vector<int64_t> c_wmax(n_chunks, 0), c_fpts(n_chunks, 0);
    par([&](int c, int64_t i0, int64_t i1) {
        int64_t wm = 0, fp = 0;
        for (int64_t i = i0; i < i1; ++i) {
            const int64_t w = wins[i].w;
            wm = std::max(wm, w);
            fp += (w >= sorted_min_w_ && w <= kFusedMaxW) ? w : 0;
        }
        c_wmax[c] = wm;
        c_fpts[c] = fp;
    });
    int64_t w_max = 0, fpts = 0;
    for (int c = 0; c < n_chunks; ++c) {
        w_max = std::max(w_max, c_wmax[c]);
        fpts += c_fpts[c];
    }
    {
        Status s = ensure_psi(w_max + 1, st);
        if (!s.ok()) return s;
    }
    // bin windows: small (warp per window) R = 1,2,4,8; sorted-marginal path; brute-force tile R = 2,4,
    // and tile R = 1 ("latency mode": a CTA per small window, one point per thread) for small classes too
    // sparse to fill the GPU, where a warp walking 32R points serially would set the round's latency.
    // per-batch class lists: engine members reused across rounds (no allocations on the round path)
    auto& small = bins_.small;
    auto& tile = bins_.tile;
    for (auto& v : small) v.clear();
    for (auto& v : tile) v.clear();
    static const int kTileRs[3] = {2, 4, 1};
    auto& sorted = bins_.sorted;
    auto& soff = bins_.soff;
    auto& fused = bins_.fused;      // sorted path, fused sort+scan kernel (w <= kFusedMaxW)
    auto& wsorted = bins_.wsorted;  // sorted path, warp per window, E = 2, 4, 8
    sorted.clear();
    soff.clear();
    fused.clear();
    for (auto& v : wsorted) v.clear();
    int fused_n2 = 256;
    int64_t n_items = 0, n_sitems = 0, spts = 0, n_segs = 0, n_mblocks = 0;
    int W2 = 0;
    int64_t pp = 0;
    // latency mode for the sorted path: few sorted points in the batch -> fused sort+scan kernel (a CTA
    // per window slice, no scratch round trip); otherwise the throughput form (sort once, then scan)
    const bool fuse = use_fused_path && fpts <= fused_max_pts_;
    if ((int)cbins_.size() < n_chunks) cbins_.resize(n_chunks);
    par([&](int c, int64_t i0, int64_t i1) {
        ChunkBins& B = cbins_[c];
        for (auto& v : B.small) v.clear();
        for (auto& v : B.tile) v.clear();
        for (auto& v : B.wsorted) v.clear();
        B.sorted.clear();
        B.fused.clear();
        B.soff.clear();
        B.spts = B.n_segs = B.n_mblocks = B.n_items = B.pp = 0;
        B.W2 = 0;
        B.fused_n2 = 256;
        for (int64_t i = i0; i < i1; ++i) {
            const int w = wins[i].w;
            B.pp += (int64_t)w * (w - 1);
            const int R = small_class_R(w);
            if (R >= 2 && use_sorted && w >= wsorted_min_w_) {
                B.wsorted[R == 2 ? 0 : R == 4 ? 1 : 2].push_back((int32_t)i);
            } else if (R && !(use_sorted && w >= sorted_min_w_)) {
                B.small[R == 1 ? 0 : R == 2 ? 1 : R == 4 ? 2 : 3].push_back((int32_t)i);
            } else if (fuse && w >= sorted_min_w_ && w <= kFusedMaxW) {
                B.fused.push_back((int32_t)i);
                while (B.fused_n2 < w) B.fused_n2 <<= 1;
            } else if (use_sorted && w >= sorted_min_w_) {
                B.sorted.push_back((int32_t)i);
                B.soff.push_back(B.spts + kScanB);  // kScanB sentinel entries on either side of the window's region
                B.spts += (w + 2 * kScanB + 1) & ~1;  // even offsets: phase A loads 16-B aligned pairs of P2 entries
                B.n_segs += (w + kSortedMaxW - 1) / kSortedMaxW;
                if (w > kSortedMaxW) B.n_mblocks += (w + kMergePts - 1) / kMergePts;
                int n2 = 1;
                while (n2 < std::min(w, kSortedMaxW)) n2 <<= 1;
                B.W2 = std::max(B.W2, n2);
            } else {
                const int tr = tile_R(w);
                B.tile[tr == 2 ? 0 : 1].push_back((int32_t)i);
                B.n_items += (w + kTileThreads * tr - 1) / (kTileThreads * tr);
            }
        }
    });
    // one chunk (every round below 2^18 windows): the lists move over (swap, no copy); else concatenate
    auto cat = [&](std::vector<int32_t>& dst, std::vector<int32_t>& src, bool first) {
        if (first && n_chunks == 1) dst.swap(src);
        else if (first) dst.assign(src.begin(), src.end());
        else dst.insert(dst.end(), src.begin(), src.end());
    };
    for (int c = 0; c < n_chunks; ++c) {
        ChunkBins& B = cbins_[c];
        for (int s = 0; s < 4; ++s) cat(small[s], B.small[s], c == 0);
        for (int s = 0; s < 2; ++s) cat(tile[s], B.tile[s], c == 0);
        for (int e = 0; e < 3; ++e) cat(wsorted[e], B.wsorted[e], c == 0);
        cat(fused, B.fused, c == 0);
        cat(sorted, B.sorted, c == 0);
        if (n_chunks == 1) soff.swap(B.soff);
        else for (int64_t o : B.soff) soff.push_back(spts + o);
        spts += B.spts;
        n_segs += B.n_segs;
        n_mblocks += B.n_mblocks;
        n_items += B.n_items;
        pp += B.pp;
        W2 = std::max(W2, B.W2);
        fused_n2 = std::max(fused_n2, B.fused_n2);
    }
    // latency mode: a class too sparse to fill the GPU runs a CTA per window (tile R = 1), where a warp
    // walking 32R points (brute force) or sorting and scanning them (warp-sorted) would set the latency
    // (all of a round's latency-mode windows go into one launch: per-class launches measured slower)
    // (windows >= fused_small_min_w_ take the fused sort+scan kernel when the round is in latency mode)
    auto& lat = bins_.lat;
    auto& lat_tiny = bins_.lat_tiny;  // w <= lat_tiny_max_w_: a warp per window inside the latency launch
    lat.clear();
    lat_tiny.clear();

    auto to_latency = [&](std::vector<int32_t>& v) {
        for (int32_t q : v) {
            const int w = wins[q].w;
            if (fuse && w >= fused_small_min_w_) {
                fused.push_back(q);
                while (fused_n2 < w) fused_n2 <<= 1;
                continue;
            }
            if (lat_split_on_ && variant == 0 && w <= lat_tiny_max_w_ && w <= 32) {  // warp per window (KSG-1)
                lat_tiny.push_back(q);
                continue;
            }
            if (lat_split_on_ && variant == 0 && w <= 256) {  // 8 lanes per point (KSG-1)
                lat.push_back(q);
                const int lp = lat_points_per_cta(lat_lanes(w));
                n_items += (w + lp - 1) / lp;
                continue;
            }
            tile[2].push_back(q);
            n_items += (w + kTileThreads - 1) / kTileThreads;
        }
        v.clear();
    };
    for (int s = 0; s < 4; ++s)
        if (!small[s].empty() && (1 << s) > lat_keep_small_R_ && (int64_t)small[s].size() < lat_windows_)
            to_latency(small[s]);
    for (int e = 0; e < 3; ++e)
        if (!wsorted[e].empty() && (int64_t)wsorted[e].size() < lat_windows_) to_latency(wsorted[e]);
    // NEXT-3 block plan (the GPU analogue of the paper's incremental MI): sorted-path windows of one
    // (pair, size) whose starts differ by d share beta-blocks, beta = the power-of-two part of gcd(d, w) in
    // [256, kSortedMaxW] (TD: the delta-grid of a partition, delta = s/4, shared by the layer's windows and
    // their noise sub-windows; sweeps: the stride).  Each block is sorted once per batch; its windows merge
    // the sorted blocks (the merge levels from beta up) instead of sorting from scratch.
    const auto t_bin = sclk::now();
    sub_ms[0] += std::chrono::duration<double, std::milli>(t_bin - t_sub0).count();
    auto& wbeta = bins_.beta;
    auto& blks = bins_.blks;
    auto& segb = bins_.segb;
    blks.clear();
    segb.clear();
    wbeta.assign(sorted.size(), 0);
    std::vector<int64_t> wboff;
    int blk_beta_max = 0;
    int64_t blk_store = 0, blk_pts = 0, blk_windows = 0;
    auto& ord = bins_.ord;
    ord.clear();
    if (block_sort_on_ && !(flags & ISYCOS_F_NO_BLOCK) && sorted.size() >= 2) {
        // only windows whose size is a multiple of 256 can share blocks (beta >= 256 divides w): search rounds
        // of other sizes (BU: s_min + j delta_bu) skip the plan's sort and maps entirely
        for (size_t b = 0; b < sorted.size(); ++b)
            if ((wins[sorted[b]].w & 255) == 0) ord.push_back((int32_t)b);
    }
    if (ord.size() >= 2) {
        std::sort(ord.begin(), ord.end(), [&](int32_t a, int32_t c) {
            const KsgWin& A = wins[sorted[a]];
            const KsgWin& C = wins[sorted[c]];
            if (A.pair != C.pair) return A.pair < C.pair;
            if (A.w != C.w) return A.w < C.w;
            return A.t0 < C.t0;
        });
        for (size_t i = 0; i + 1 < ord.size(); ++i) {
            const KsgWin& A = wins[sorted[ord[i]]];
            const KsgWin& C = wins[sorted[ord[i + 1]]];
            if (A.pair != C.pair || A.w != C.w || C.t0 == A.t0) continue;
            const int64_t g = std::gcd<int64_t>(C.t0 - A.t0, (int64_t)A.w);
            int64_t bt = g & -g;
            if (bt > kSortedMaxW) bt = kSortedMaxW;
            if (bt < 256) continue;
            wbeta[ord[i]] = std::max<int32_t>(wbeta[ord[i]], (int32_t)bt);
            wbeta[ord[i + 1]] = std::max<int32_t>(wbeta[ord[i + 1]], (int32_t)bt);
        }
        struct Grid {
            int64_t jmin = INT64_MAX, jmax = -1, off = 0;
            std::vector<char> need;
        };
        std::unordered_map<uint64_t, Grid> grids;
        auto gkey = [](const KsgWin& W, int32_t bt) {
            int lg = 0;
            while ((1 << lg) < bt) ++lg;
            return ((uint64_t)(uint32_t)W.pair << 17) | ((uint64_t)lg << 13) | (uint64_t)(W.t0 % bt);
        };
        for (size_t b = 0; b < sorted.size(); ++b) {
            const int32_t bt = wbeta[b];
            if (!bt) continue;
            const KsgWin& W = wins[sorted[b]];
            Grid& G = grids[gkey(W, bt)];
            const int64_t j0 = W.t0 / bt;
            G.jmin = std::min(G.jmin, j0);
            G.jmax = std::max(G.jmax, j0 + W.w / bt - 1);
        }
        for (auto& kv : grids) {
            const int32_t bt = 1 << ((kv.first >> 13) & 15);
            kv.second.off = blk_store;
            kv.second.need.assign(kv.second.jmax - kv.second.jmin + 1, 0);
            blk_store += (kv.second.jmax - kv.second.jmin + 1) * bt;
        }
        wboff.assign(sorted.size(), 0);
        for (size_t b = 0; b < sorted.size(); ++b) {
            const int32_t bt = wbeta[b];
            if (!bt) continue;
            const KsgWin& W = wins[sorted[b]];
            Grid& G = grids[gkey(W, bt)];
            const int64_t j0 = W.t0 / bt;
            for (int64_t j = j0; j < j0 + W.w / bt; ++j) G.need[j - G.jmin] = 1;
            wboff[b] = G.off + (j0 - G.jmin) * bt;
            ++blk_windows;
            blk_beta_max = std::max(blk_beta_max, bt);
        }
        for (auto& kv : grids) {
            const int32_t bt = 1 << ((kv.first >> 13) & 15);
            const int32_t pair = (int32_t)(kv.first >> 17);
            const int64_t o = (int64_t)(kv.first & 8191);
            for (size_t j = 0; j < kv.second.need.size(); ++j)
                if (kv.second.need[j]) {
                    blks.push_back(KsgBlk{o + (kv.second.jmin + (int64_t)j) * bt, kv.second.off + (int64_t)j * bt, pair, bt});
                    blk_pts += bt;
                }
        }
    }
    // NEXT-3 incremental radii (the paper's IR): a window that follows its predecessor on a block grid
    // (same pair and size, start + beta, w >= 8 beta: at most 1/8 of the points change) reuses the predecessor's
    // radii wherever the removed / inserted block cannot change them (ksg_device.cuh, inc_unchanged).  Chains
    // restart from scratch every kIncChain windows; level j runs in the j-th scan launch.
    auto& incs = bins_.incs;
    incs.assign(sorted.size(), KsgInc{-1, 0, 0, 0, -1, -1, 0});
    int n_lv = 1, inc_d_max = 0;
    int64_t inc_windows = 0;
    if (!blks.empty() && (inc_on_ || (flags & ISYCOS_F_INCREMENTAL)) && variant == 0) {  // KSG-1 (counts carried)
        auto& ord = bins_.ord;  // sorted by (pair, w, t0) by the block plan
        for (size_t i = 0; i + 1 < ord.size(); ++i) {
            const int32_t a = ord[i], c = ord[i + 1];
            const KsgWin& A = wins[sorted[a]];
            const KsgWin& C = wins[sorted[c]];
            const int32_t bt = wbeta[a];
            if (A.pair != C.pair || A.w != C.w || bt == 0 || wbeta[c] != bt || C.t0 - A.t0 != bt || A.w < 8 * bt ||
                bt > kIncMaxD)
                continue;
            if (incs[a].level < 0) incs[a].level = 0;
            const int lv = incs[a].level + 1 < inc_chain_ ? incs[a].level + 1 : 0;
            incs[c].level = lv;
            if (lv > 0) {
                incs[c].pred = a;
                incs[c].eps_prev = soff[a];
                incs[c].boffR = wboff[a];
                incs[c].boffI = wboff[c] + C.w - bt;
                incs[c].d = bt;
                inc_d_max = std::max(inc_d_max, (int)bt);
                ++inc_windows;
                n_lv = std::max(n_lv, lv + 1);
            }
        }
    }
    const auto t_plan = sclk::now();
    sub_ms[1] += std::chrono::duration<double, std::milli>(t_plan - t_bin).count();
    // sorted scan: 1024 points per CTA when the batch fills the GPU (better lane balance in the per-warp
    // work queues), else 256 (more CTAs per window: latency-bound rounds)
    const int ppc = spts >= (int64_t)148 * 8 * 1024 ? sorted_ppc_ : 256;
    for (int32_t q : sorted) n_sitems += (wins[q].w + ppc - 1) / ppc;
    std::vector<int32_t> lv_off(n_lv + 1, 0);  // scan items grouped by launch level
    for (size_t b = 0; b < sorted.size(); ++b)
        lv_off[std::max(0, incs[b].level) + 1] += (wins[sorted[b]].w + ppc - 1) / ppc;
    for (int l = 0; l < n_lv; ++l) lv_off[l + 1] += lv_off[l];
    // fused: split windows into up to ceil(w / 512) slices while the batch has fewer than 2 CTAs per SM
    const int gmax = std::max<int>(1, (int)(2 * 148 / std::max<size_t>(1, fused.size())));
    int64_t n_fitems = 0;
    for (int32_t q : fused) {
        const int fp = fused_ppc(wins[q].w, gmax);
        n_fitems += (wins[q].w + fp - 1) / fp;
    }
    int64_t n_lists = (int64_t)sorted.size() + (int64_t)fused.size() + (int64_t)lat_tiny.size();
    for (auto& v : small) n_lists += (int64_t)v.size();
    int64_t n_wlist = 0;
    for (auto& v : wsorted) n_wlist += (int64_t)v.size();
    n_lists += n_wlist;

    {
        Status s = ensure_capacity(S, n + 1, n_items + n_sitems + n_segs + n_mblocks + n_fitems, n_pairs,
                                   n_lists + 2 * (int64_t)sorted.size() + 16,
                                   n_segs * (int64_t)sizeof(KsgSegB) + (int64_t)blks.size() * (int64_t)sizeof(KsgBlk) +
                                       (int64_t)sorted.size() * (int64_t)sizeof(KsgInc) + 192);
        if (!s.ok()) return s;
    }
    // scratch per sorted point: P2 (8) | OX | YS | TX | TI | TY | EPS (4 each) | CNT (8) | CY (8); then the NEXT-3 block keys
    // BX (8) | BY (4)
    const int64_t blk_base = (spts * 48 + 15) & ~int64_t(15);  // + CY (8): box-assisted columns
    const int64_t scratch_need = blk_base + blk_store * 12;
    if (spts > 0 && S.sscratch_cap < scratch_need) {
        const int64_t c = std::max<int64_t>(scratch_need, S.sscratch_cap * 2);
        cudaFree(S.sscratch);
        S.sscratch = nullptr;
        ISY_CK(cudaMalloc(&S.sscratch, c));
        S.sscratch_cap = c;
    }
    const auto t_sub1 = sclk::now();
    sub_ms[2] += std::chrono::duration<double, std::milli>(t_sub1 - t_plan).count();
    // pack [pairs | wins | small lists | sorted list | sorted offsets | tile items | sorted items]
    const int64_t off_pairs = 0;
    const int64_t off_wins = align64(off_pairs + n_pairs * (int64_t)sizeof(PairPtrs));
    const int64_t off_lists = align64(off_wins + n * (int64_t)sizeof(KsgWin));
    const int64_t off_wlist = align64(off_lists + (n_lists - n_wlist - (int64_t)sorted.size() -
                                                   (int64_t)fused.size()) * 4);
    const int64_t off_flist = align64(off_wlist + n_wlist * 4);
    const int64_t off_fitems = align64(off_flist + (int64_t)fused.size() * 4);
    const int64_t off_slist = align64(off_fitems + n_fitems * (int64_t)sizeof(KsgItem));
    const int64_t off_soff = align64(off_slist + (int64_t)sorted.size() * 4);
    const int64_t off_items = align64(off_soff + (int64_t)sorted.size() * 8);
    const int64_t off_sitems = align64(off_items + n_items * (int64_t)sizeof(KsgItem));
    const int64_t off_segs = align64(off_sitems + n_sitems * (int64_t)sizeof(KsgItem));
    const int64_t off_mblk = align64(off_segs + n_segs * (int64_t)sizeof(KsgItem));
    const int64_t off_inc = align64(off_mblk + n_mblocks * (int64_t)sizeof(KsgItem));
    const int64_t off_segb = align64(off_inc + (inc_windows ? (int64_t)sorted.size() : 0) * (int64_t)sizeof(KsgInc));
    const int64_t off_blks = align64(off_segb + (blks.empty() ? 0 : n_segs) * (int64_t)sizeof(KsgSegB));
    const int64_t total = align64(off_blks + (int64_t)blks.size() * (int64_t)sizeof(KsgBlk));
    std::memcpy(S.hstage + off_pairs, pairs, n_pairs * sizeof(PairPtrs));
    par([&](int, int64_t i0, int64_t i1) {  // large batches: the copy into pinned memory on several threads
        std::memcpy(S.hstage + off_wins + i0 * (int64_t)sizeof(KsgWin), wins + i0, (i1 - i0) * sizeof(KsgWin));
    });
    int64_t list_off[5], wlist_off[3];
    {
        int32_t* lp = reinterpret_cast<int32_t*>(S.hstage + off_lists);
        int64_t c = 0;
        for (int s = 0; s < 4; ++s) {
            list_off[s] = c;
            std::memcpy(lp + c, small[s].data(), small[s].size() * 4);
            c += (int64_t)small[s].size();
        }
        list_off[4] = c;  // the latency launch's tiny windows
        std::memcpy(lp + c, lat_tiny.data(), lat_tiny.size() * 4);
        int32_t* wl = reinterpret_cast<int32_t*>(S.hstage + off_wlist);
        int64_t cw = 0;
        for (int e = 0; e < 3; ++e) {
            wlist_off[e] = cw;
            std::memcpy(wl + cw, wsorted[e].data(), wsorted[e].size() * 4);
            cw += (int64_t)wsorted[e].size();
        }
        std::memcpy(S.hstage + off_flist, fused.data(), fused.size() * 4);
        KsgItem* fp = reinterpret_cast<KsgItem*>(S.hstage + off_fitems);
        int64_t cf = 0;
        for (size_t b = 0; b < fused.size(); ++b) {
            const int w = wins[fused[b]].w;
            const int pp_w = fused_ppc(w, gmax);
            for (int i0 = 0; i0 < w; i0 += pp_w) fp[cf++] = KsgItem{(int32_t)b, i0};
        }
        std::memcpy(S.hstage + off_slist, sorted.data(), sorted.size() * 4);
        std::memcpy(S.hstage + off_soff, soff.data(), soff.size() * 8);
    }
    int64_t item_off[3], item_off_lat = 0, n_litems = 0;
    {
        KsgItem* ip = reinterpret_cast<KsgItem*>(S.hstage + off_items);
        int64_t c = 0;
        for (int s = 0; s < 3; ++s) {
            item_off[s] = c;
            const int tr = kTileRs[s];
            for (int32_t q : tile[s]) {
                const int w = wins[q].w;
                for (int i0 = 0; i0 < w; i0 += kTileThreads * tr) ip[c++] = KsgItem{q, i0};
            }
        }
        item_off_lat = c;
        for (int32_t q : lat) {
            const int w = wins[q].w;
            const int lp = lat_points_per_cta(lat_lanes(w));
            const int32_t fl = lat_item_flag(lat_lanes(w));
            for (int i0 = 0; i0 < w; i0 += lp) ip[c++] = KsgItem{q, i0 | fl};
        }
        n_litems = c - item_off_lat;
        KsgItem* sp = reinterpret_cast<KsgItem*>(S.hstage + off_sitems);
        KsgItem* sg = reinterpret_cast<KsgItem*>(S.hstage + off_segs);
        KsgItem* mb = reinterpret_cast<KsgItem*>(S.hstage + off_mblk);
        int64_t cs = 0, cm = 0;
        c = 0;
        KsgSegB* sbp = reinterpret_cast<KsgSegB*>(S.hstage + off_segb);
        std::vector<int32_t> lv_fill(lv_off.begin(), lv_off.end() - 1);
        for (size_t b = 0; b < sorted.size(); ++b) {
            const int w = wins[sorted[b]].w;
            int32_t& f = lv_fill[std::max(0, incs[b].level)];
            for (int i0 = 0; i0 < w; i0 += ppc) sp[f++] = KsgItem{(int32_t)b, i0};
            for (int s0 = 0; s0 < w; s0 += kSortedMaxW) {
                if (!blks.empty())  // the segment's blocks are contiguous in the block storage (s0 % beta == 0)
                    sbp[cs] = wbeta[b] ? KsgSegB{wboff[b] + s0, wbeta[b], 0} : KsgSegB{0, 0, 0};
                sg[cs++] = KsgItem{(int32_t)b, s0};
            }
            if (w > kSortedMaxW)
                for (int i0 = 0; i0 < w; i0 += kMergePts) mb[cm++] = KsgItem{(int32_t)b, i0};
        }
    }
    if (!blks.empty()) std::memcpy(S.hstage + off_blks, blks.data(), blks.size() * sizeof(KsgBlk));
    if (inc_windows) std::memcpy(S.hstage + off_inc, incs.data(), incs.size() * sizeof(KsgInc));
    // one H2D copy of the packed descriptors (kernels reading them from mapped host memory instead
    // measured 20 % slower on cfg2: a PCIe round trip on every CTA's critical path)
    char* dbase = S.dstage;
    const auto t_sub2 = sclk::now();
    sub_ms[3] += std::chrono::duration<double, std::milli>(t_sub2 - t_sub1).count();
    ISY_CK(cudaMemcpyAsync(S.dstage, S.hstage, total, cudaMemcpyHostToDevice, st));
    if (bs) bs->h2d_bytes += total;
    S.busy = true;  // from here on the slot's buffers are in use (an error return below leaves it to be synced)
    S.st = st;
    S.profile = false;
    S.n_ksg = 0;

    KsgLaunch L;
    L.pairs = reinterpret_cast<const PairPtrs*>(dbase + off_pairs);
    L.wins = reinterpret_cast<const KsgWin*>(dbase + off_wins);
    L.psi = psi_;
    L.psiq = psiq_;
    L.lnc = lnc_;
    L.acc = S.acc;
    const bool zc = n <= kZeroCopyMaxRecs;  // big sweeps: device records + one D2H copy (PCIe-friendlier)
    L.out = zc ? S.drec : S.ddrec;
    L.dbg_eps = dbg.eps;
    L.dbg_nx = dbg.nx;
    L.dbg_ny = dbg.ny;
    L.k = k;
    L.variant = variant;
    L.knn_mode = knn_mode_;
    L.two = 2;
    L.sorted_ppc = ppc;
    L.fused_n2 = fused_n2;
    L.scan_unified = scan_unified_;
    L.poison = poison_;
    L.col_min_w = col_min_w_;
    if (poison_) {  // every byte the kernels read must have been written in this batch
        const int pb = (int)(poison_ & 0xffu);
        if (S.sscratch) ISY_CK(cudaMemsetAsync(S.sscratch, pb, S.sscratch_cap, st));
        if (S.ddrec) ISY_CK(cudaMemsetAsync(S.ddrec, pb, S.ddrec_cap * sizeof(KsgRec), st));
        if (n <= kZeroCopyMaxRecs) {
            ISY_CK(cudaStreamSynchronize(st));
            std::memset(S.hrec, pb, n * sizeof(KsgRec));
        }
    }
    const int32_t* dlists = reinterpret_cast<const int32_t*>(dbase + off_lists);
    const KsgItem* ditems = reinterpret_cast<const KsgItem*>(dbase + off_items);

    // launches: biggest work first so the small classes fill the tail
    int n_launch = 0, n_ksg = 0;
    std::vector<int>& launch_cls = S.launch_cls;  // 0 sorted-marginal group, 1 brute-force launch
    launch_cls.clear();
    // algorithmic work: brute-force ordered pairs; sorted path binary-search probes (4 searches per point: x and y interval ends)
    int64_t brute_pairs = 0, probes = 0;
    for (int s = 0; s < 4; ++s)
        for (int32_t q : small[s]) brute_pairs += (int64_t)wins[q].w * (wins[q].w - 1);

    for (int s = 0; s < 3; ++s)
        for (int32_t q : tile[s]) brute_pairs += (int64_t)wins[q].w * (wins[q].w - 1);
    for (int32_t q : lat) brute_pairs += (int64_t)wins[q].w * (wins[q].w - 1);
    for (int32_t q : lat_tiny) brute_pairs += (int64_t)wins[q].w * (wins[q].w - 1);
    for (int32_t q : fused) {
        int lg = 0;
        while ((1 << lg) < wins[q].w) ++lg;
        probes += (int64_t)wins[q].w * 4 * lg;
    }
    for (auto& v : wsorted)
        for (int32_t q : v) {
            int lg = 0;
            while ((1 << lg) < wins[q].w) ++lg;
            probes += (int64_t)wins[q].w * 4 * lg;
        }
    for (int32_t q : sorted) {
        int lg = 0;
        while ((1 << lg) < wins[q].w) ++lg;
        probes += (int64_t)wins[q].w * 4 * lg;
    }
    auto ev_pair = [&](int i) -> std::pair<cudaEvent_t, cudaEvent_t> {
        while ((int)S.events.size() < 2 * (i + 1)) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            S.events.push_back(e);
        }
        return {S.events[2 * i], S.events[2 * i + 1]};
    };
    // Launch groups fork onto auxiliary streams after the descriptor copy and join before the record
    // copy, so independent size classes overlap (a round's latency is the slowest class, not the sum).
    int n_aux_used = 0;
    bool forked = false;
    // small batches (<= aux_min_windows_) keep every launch on the slot's stream: the fork/join API calls
    // cost more host time than the kernels' overlap saves there
    const bool use_aux = n > aux_min_windows_;
    // profiling: events around the launch groups of the selected path(s) only (event records cost host time
    // on every round: bench.py times the dominant path alone)
    const bool prof_sorted = profile && !(flags & ISYCOS_F_PROFILE_BRUTE_ONLY);
    const bool prof_brute = profile && !(flags & ISYCOS_F_PROFILE_SORTED_ONLY);
    int n_prof = 0;
    auto launch = [&](int cls, int nk, auto&& fn) -> Status {
        cudaStream_t sg = st;
        if (n_ksg > 0 && use_aux) {
            if (!forked) {
                ISY_CK(cudaEventRecord(S.fork_ev, st));
                forked = true;
            }
            sg = S.aux[(n_ksg - 1) % kAux];
            if (n_ksg - 1 < kAux) {
                ISY_CK(cudaStreamWaitEvent(sg, S.fork_ev, 0));
                n_aux_used = n_ksg;
            }
        }
        std::pair<cudaEvent_t, cudaEvent_t> ev{};
        const bool prof = cls == 0 ? prof_sorted : prof_brute;
        if (prof) {
            ev = ev_pair(n_prof);
            ISY_CK(cudaEventRecord(ev.first, sg));
        }
        ISY_CK(fn(sg));
        if (prof) {
            ISY_CK(cudaEventRecord(ev.second, sg));
            launch_cls.push_back(cls);
            ++n_prof;
        }
        ++n_ksg;
        n_launch += nk;
        return Status{};
    };
    if (!fused.empty()) {
        const int32_t* dfl = reinterpret_cast<const int32_t*>(dbase + off_flist);
        const KsgItem* dfi = reinterpret_cast<const KsgItem*>(dbase + off_fitems);
        Status r = launch(0, 1, [&](cudaStream_t sg) { return launch_fused(L, dfl, dfi, (int32_t)n_fitems, gmax, sg); });
        if (!r.ok()) return r;
    }
    for (int e = 2; e >= 0; --e) {
        if (wsorted[e].empty()) continue;
        const int32_t* wlp = reinterpret_cast<const int32_t*>(dbase + off_wlist) + wlist_off[e];
        const int32_t cnt = (int32_t)wsorted[e].size();
        Status r = launch(0, 1, [&](cudaStream_t sg) { return launch_wsorted(L, wlp, cnt, 2 << e, ws_group(cnt), sg); });
        if (!r.ok()) return r;
    }
    if (!sorted.empty()) {
        const int32_t* dsl = reinterpret_cast<const int32_t*>(dbase + off_slist);
        const int64_t* dso = reinterpret_cast<const int64_t*>(dbase + off_soff);
        const KsgItem* dsi = reinterpret_cast<const KsgItem*>(dbase + off_sitems);
        float2* P2 = reinterpret_cast<float2*>(S.sscratch);
        int32_t* OX = reinterpret_cast<int32_t*>(S.sscratch + spts * 8);
        float* YS = reinterpret_cast<float*>(S.sscratch + spts * 12);
        float* TX = reinterpret_cast<float*>(S.sscratch + spts * 16);
        int32_t* TI = reinterpret_cast<int32_t*>(S.sscratch + spts * 20);
        float* TY = reinterpret_cast<float*>(S.sscratch + spts * 24);
        const KsgItem* dsg = reinterpret_cast<const KsgItem*>(dbase + off_segs);
        const KsgItem* dmb = reinterpret_cast<const KsgItem*>(dbase + off_mblk);
        const KsgSegB* dsb = reinterpret_cast<const KsgSegB*>(dbase + off_segb);
        const KsgBlk* dbk = reinterpret_cast<const KsgBlk*>(dbase + off_blks);
        unsigned long long* BX = reinterpret_cast<unsigned long long*>(S.sscratch + blk_base);
        unsigned* BY = reinterpret_cast<unsigned*>(S.sscratch + blk_base + blk_store * 8);
        float* EPS = reinterpret_cast<float*>(S.sscratch + spts * 28);
        int2* CNT = reinterpret_cast<int2*>(S.sscratch + spts * 32);
        float2* CY = reinterpret_cast<float2*>(S.sscratch + spts * 40);
        bool cols = false;  // any window of the throughput batch on the box-assisted phase A
        for (int32_t q : sorted) cols = cols || wins[q].w >= col_min_w_;
        const KsgInc* dinc = inc_windows ? reinterpret_cast<const KsgInc*>(dbase + off_inc) : nullptr;
        if (inc_windows) {  // work ticket + per-window finished-CTA counters, zeroed for this launch
            const int64_t need = 1 + (int64_t)sorted.size();
            if (S.sync_cap < need) {
                cudaFree(S.sync);
                S.sync = nullptr;
                S.sync_cap = std::max<int64_t>(need, S.sync_cap * 2);
                ISY_CK(cudaMalloc(&S.sync, S.sync_cap * sizeof(unsigned)));
            }
        }
        Status r = launch(0, (n_mblocks ? 3 : 2) + (blks.empty() ? 0 : 1), [&](cudaStream_t sg) {
            if (inc_windows) {
                cudaError_t e = cudaMemsetAsync(S.sync, 0, (1 + sorted.size()) * sizeof(unsigned), sg);
                if (e != cudaSuccess) return e;
            }
            return launch_sorted(L, dsl, dso, dsg, (int32_t)n_segs, dmb, (int32_t)n_mblocks, P2, OX, YS, TX, TI, TY,
                                 W2, dsi, (int32_t)n_sitems, sg, dsb, dbk, (int32_t)blks.size(), blk_beta_max, BX, BY,
                                 dinc, EPS, CNT, lv_off.data(), n_lv, inc_d_max, inc_windows ? S.sync : nullptr,
                                 cols ? CY : nullptr);
        });
        if (!r.ok()) return r;
    }
    if (!lat.empty() || !lat_tiny.empty()) {
        const KsgItem* ip = ditems + item_off_lat;
        const int32_t* tp = dlists + list_off[4];
        Status r = launch(1, 1, [&](cudaStream_t sg) {
            return launch_ksg_lat(L, ip, (int32_t)n_litems, tp, (int32_t)lat_tiny.size(), sg);
        });
        if (!r.ok()) return r;
    }
    for (int s : {1, 0, 2}) {
        if (tile[s].empty()) continue;
        const int R = kTileRs[s];
        int64_t cnt = 0;
        for (int32_t q : tile[s]) cnt += (wins[q].w + kTileThreads * R - 1) / (kTileThreads * R);
        const KsgItem* ip = ditems + item_off[s];
        Status r = launch(1, 1, [&](cudaStream_t sg) { return launch_ksg_tile(L, ip, (int32_t)cnt, R, sg); });
        if (!r.ok()) return r;
    }
    for (int s = 3; s >= 0; --s) {
        if (small[s].empty()) continue;
        const int R = 1 << s;
        const int32_t* lp = dlists + list_off[s];
        const int32_t cnt = (int32_t)small[s].size();
        Status r = launch(1, 1, [&](cudaStream_t sg) { return launch_ksg_small(L, lp, cnt, R, sg); });
        if (!r.ok()) return r;
    }
    for (int a = 0; a < std::min(n_aux_used, kAux); ++a) {  // join
        ISY_CK(cudaEventRecord(S.join_ev[a], S.aux[a]));
        ISY_CK(cudaStreamWaitEvent(st, S.join_ev[a], 0));
    }
    if (!zc) ISY_CK(cudaMemcpyAsync(S.hrec, S.ddrec, n * sizeof(KsgRec), cudaMemcpyDeviceToHost, st));
    int64_t spoints = 0;  // real points on the sorted path (spts includes the sentinel padding)
    for (int32_t q : sorted) spoints += wins[q].w;
    for (int32_t q : fused) spoints += wins[q].w;
    S.busy = true;
    S.st = st;
    S.n = n;
    S.profile = profile;
    S.n_ksg = n_prof;  // profiled launch groups (events / launch_cls entries)
    S.pp = pp;
    S.n_launch = n_launch;
    S.brute_pairs = brute_pairs;
    S.probes = probes;
    S.sorted_windows = (int64_t)sorted.size() + (int64_t)fused.size() + n_wlist;
    for (auto& v : wsorted)
        for (int32_t q : v) spoints += wins[q].w;
    S.spts = spoints;
    S.block_windows = blk_windows;
    S.block_points = blk_pts;
    S.inc_windows = inc_windows;
    sub_ms[4] += std::chrono::duration<double, std::milli>(sclk::now() - t_sub2).count();
    return Status{};
}

// Wait for a submitted batch; copy its records out.  The kernels wrote the records (and per-window
// scan-step counts) into mapped pinned host memory (or a device buffer copied back by submit): the stream
// synchronisation makes them visible.
Status Engine::collect(int si, KsgRec* recs_host, BatchStats* bs) {
    const KsgRec* view = nullptr;
    const int64_t n = slots_[si].busy ? slots_[si].n : 0;
    Status s = collect_view(si, &view, bs, true);
    if (s.ok() && recs_host && n > 0) std::memcpy(recs_host, view, n * sizeof(KsgRec));
    return s;
}

Status Engine::collect_view(int si, const KsgRec** view, BatchStats* bs, bool count_steps, bool* profiled) {
    Slot& S = slots_[si];
    *view = S.hrec;
    if (profiled) *profiled = S.busy && S.profile;
    if (!S.busy) return Status{};
    S.busy = false;
    const int64_t n = S.n;
    ISY_CK(cudaStreamSynchronize(S.st));
    unsigned long long steps = 0;
    if (count_steps)
        for (int64_t i = 0; i < n; ++i) {
            steps += S.hrec[i].steps;
            if (bs) bs->eps_reused += S.hrec[i].reused;
        }
    if (bs) {
        bs->d2h_bytes += n * (int64_t)sizeof(KsgRec);
        bs->windows += n;
        bs->point_pairs += S.pp;
        bs->launches += S.n_launch;
        bs->ksg_launches += S.n_launch;
        bs->rounds += 1;
        bs->scan_steps += (int64_t)steps;
        bs->sorted_windows += S.sorted_windows;
        bs->sorted_points += S.spts;
        bs->brute_pairs += S.brute_pairs;
        bs->search_probes += S.probes;
        bs->block_windows += S.block_windows;
        bs->block_points += S.block_points;
        bs->inc_windows += S.inc_windows;
        if (S.profile) {
            bs->prof_rounds += 1;
            bs->prof_brute_pairs += S.brute_pairs;
            bs->prof_scan_steps += (int64_t)steps;
            bs->prof_probes += S.probes;
            for (int i = 0; i < S.n_ksg; ++i) {
                float ms = 0.f;
                cudaEventElapsedTime(&ms, S.events[2 * i], S.events[2 * i + 1]);
                bs->kernel_ms += ms;
                if (S.launch_cls[i] == 0)
                    bs->sorted_ms += ms;
                else
                    bs->brute_ms += ms;
            }
        }
    }
    return Status{};
}

Status Engine::fork_second_stream(cudaStream_t st) {
    ISY_CK(cudaEventRecord(xev_, st));
    ISY_CK(cudaStreamWaitEvent(stream2_, xev_, 0));
    return Status{};
}

Status Engine::join_second_stream(cudaStream_t st) {
    ISY_CK(cudaEventRecord(xev_, stream2_));
    ISY_CK(cudaStreamWaitEvent(st, xev_, 0));
    return Status{};
}

Status Engine::upload_series(const float* src, int64_t n, bool src_is_device, float** dev_out, cudaStream_t st,
                             BatchStats* bs) {
    const int64_t npad = ((n + 3) & ~int64_t(3)) + 4;
    float* d = nullptr;
    ISY_CK(cudaMalloc(&d, npad * sizeof(float)));
    ISY_CK(cudaMemsetAsync(d, 0, npad * sizeof(float), st));
    ISY_CK(cudaMemcpyAsync(d, src, n * sizeof(float),
                           src_is_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
    if (bs && !src_is_device) bs->h2d_bytes += n * (int64_t)sizeof(float);
    *dev_out = d;
    return Status{};
}

void Engine::free_series(float* p) { cudaFree(p); }

Status Engine::check_finite(const float* dev, int64_t n, cudaStream_t st, bool* finite) {
    ISY_CK(cudaMemsetAsync(dflag_, 0, sizeof(int), st));
    ISY_CK(launch_nonfinite_scan(dev, n, dflag_, st));
    int h = 0;
    ISY_CK(cudaMemcpyAsync(&h, dflag_, sizeof(int), cudaMemcpyDeviceToHost, st));
    ISY_CK(cudaStreamSynchronize(st));
    *finite = (h == 0);
    return Status{};
}

}  // namespace isy
