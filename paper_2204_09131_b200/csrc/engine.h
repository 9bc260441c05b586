// Internal interfaces of libisycos (not part of the C ABI; see include/isycos.h).
//
// Layering:
//   capi.cpp     validation, pointer classification, error codes  (C ABI)
//   search.cpp   batched SYCOS_TD / SYCOS_BU / noise / chunk driver (host state machines)
//   engine.cu    per-device context: digamma tables, buffers, batch evaluation, profiling
//   ksg_*.cu     the sm_100a KSG window kernels (a2-a6 of SURVEY §8(a)), ksg_device.cuh their helpers
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <string>
#include <vector>

#include "isycos.h"

namespace isy {

// ---------------------------------------------------------------- device-visible records
struct PairPtrs {            // device pointers of one series pair (16-B aligned, padded to 4 floats)
    const float* x;
    const float* y;
};

struct KsgWin {              // one window of a batch (24 B)
    int64_t t0;
    int32_t w;
    int32_t pair;            // index into the batch's PairPtrs table
    int64_t dbg_off;         // offset of this window's points in the debug arrays, or -1
};

struct KsgItem {             // one (window, i-tile) work item of the tile kernel
    int32_t win;
    int32_t i0;
};

struct KsgBlk {             // NEXT-3 shared block: beta points [t, t + beta) of a pair, sorted once per batch
    int64_t t;
    int64_t boff;            // offset (points) of its sorted keys in the block storage
    int32_t pair;
    int32_t beta;
};

struct KsgSegB {            // per sort segment: its first block's keys (beta = 0: sort from scratch)
    int64_t boff;
    int32_t beta;
    int32_t pad;
};

struct KsgRec {              // per-window result (56 B), written by the kernels straight into mapped pinned host memory
    double mi, h, nmi;
    long long s_psi, s_log;
    int32_t zero_eps;
    int32_t reused;            // NEXT-3 incremental windows: points whose radius carried over from the previous window
    unsigned long long steps;  // sorted path: outward-scan candidate visits of this window (algorithmic work)
};

struct KsgAcc {              // self-cleaning accumulator of a multi-tile window
    unsigned long long s_psi, s_log;
    unsigned int zero, done;
    unsigned long long steps;
    unsigned int reused, pad;
};

struct KsgInc {              // NEXT-3 incremental window: its predecessor on the grid (sorted-list position)
    int64_t eps_prev;        // offset (points) of the predecessor's radii in the EPS scratch
    int64_t boffR, boffI;    // block storage offsets of the removed and the inserted block (d points each)
    int32_t d;               // grid step = block size
    int32_t level;           // chain level (-1: no chain, 0: scanned from scratch, >= 1: follows `pred`)
    int32_t pred;            // sorted-list position of the predecessor (level >= 1)
    int32_t pad;
};

struct KsgLaunch {           // arguments shared by every KSG kernel of a batch
    const PairPtrs* pairs;
    const KsgWin* wins;
    const double* psi;       // psi[m], m = 0..w_max
    const long long* psiq;   // q(psi[m]) = rint(psi[m] * 2^32)
    const double* lnc;       // LN series coefficients 1/(2j+1), j = 1..9
    KsgAcc* acc;
    KsgRec* out;
    float* dbg_eps;
    int32_t* dbg_nx;
    int32_t* dbg_ny;
    int32_t k;
    int32_t variant;
    int32_t knn_mode;        // small-window kernel: bit 0 branch-free kNN insertion (else guarded), bit 1 ballot counts
    int32_t two;             // the constant 2, passed at run time (see acc_lt)
    int32_t sorted_ppc;      // sorted path: points per scan CTA (256 or 1024)
    int32_t fused_n2;        // fused path: shared-memory layout stride (max next-pow2 window size of the batch)
    int32_t scan_unified;    // sorted-path phase A: 0 both sides per iteration (default), 1 one side per iteration
    uint32_t poison;         // T5 check (ISYCOS_POISON=<byte>): kernels fill their shared memory with this pattern first
    int32_t col_min_w;       // throughput scan: windows this large search the k-NN by y-sorted columns (box-assisted)
};

// Size classes.  Small: one warp per window, R = points per lane.
constexpr int kSmallWarps = 8;           // warps per CTA of the small kernel
constexpr int kTileThreads = 256;        // threads per CTA of the tile kernel
constexpr int kTileJ = 4096;             // j-tile (points) staged per cp.async.bulk round
inline int small_class_R(int w) {        // 1,2,4,8 for w <= 256; 0 => tile kernel
    return w <= 32 ? 1 : w <= 64 ? 2 : w <= 128 ? 4 : w <= 256 ? 8 : 0;
}
inline int tile_R(int w) { return w <= 2 * kTileThreads ? 2 : 4; }  // points per thread of the tile kernel
constexpr int kSortedPts = 1024;         // max points per CTA of the sorted-path scan kernel (4 warps)
constexpr int kSortedMaxW = 8192;        // sorted path: segment sorted in one CTA's SMEM (XL: runs + merge)
constexpr int kColW = 32;                // box-assisted phase A: x-sorted positions per column (sorted by y)
constexpr int kMergePts = 256;           // elements per CTA of the XL rank merge
constexpr int kScanB = 8;                // sorted-path scan: candidates per block and side (= sentinels per end)
constexpr int kFusedMaxW = 4096;         // fused sort+scan path (latency mode): windows up to this size
constexpr int kFusedThreads = 512;       // threads per fused CTA (16 warps: one 256-key sort chunk each)

// Launchers (ksg_*.cu).  Return cudaGetLastError().
cudaError_t launch_ksg_small(const KsgLaunch& L, const int32_t* list, int32_t n, int R, cudaStream_t st);
cudaError_t launch_ksg_tile(const KsgLaunch& L, const KsgItem* items, int32_t n_items, int R, cudaStream_t st);
// latency mode, KSG-1, w <= 256: 8 lanes per point (ksg_lat.cu); items {window, first point}, 32 points each
cudaError_t launch_ksg_lat(const KsgLaunch& L, const KsgItem* items, int32_t n_items, const int32_t* tiny,
                           int32_t n_tiny, cudaStream_t st);
int lat_points_per_cta(int lanes);      // latency kernel: points per CTA with `lanes` (4 or 8) lanes per point
int32_t lat_item_flag(int lanes);        // KsgItem.i0 flag selecting the lanes per point
// sorted path: sort kernel over segments {list pos, start}, XL rank merge over blocks {list pos, start},
// then the scan kernel over `items` {list pos, first point}
// NEXT-3: blocks {pair, t, beta} are sorted first into BX (x keys) / BY (y keys); segments with segb[i].beta > 0
// merge their sorted blocks instead of sorting from scratch (blk_beta_max sizes the block-sort CTAs)
cudaError_t launch_sorted(const KsgLaunch& L, const int32_t* list, const int64_t* soff, const KsgItem* segs,
                          int32_t n_segs, const KsgItem* mblocks, int32_t n_mblocks, float2* P2, int32_t* OX,
                          float* YS, float* TX, int32_t* TI, float* TY, int W2, const KsgItem* items,
                          int32_t n_items, cudaStream_t st, const KsgSegB* segb, const KsgBlk* blks,
                          int32_t n_blks, int blk_beta_max, unsigned long long* BX, unsigned* BY, const KsgInc* inc,
                          float* EPS, int2* CNT, const int32_t* lv_off, int n_lv, int inc_d_max,
                          unsigned* sync, float2* CY);
constexpr int kIncChain = 16;  // NEXT-3 incremental chains: a window scanned from scratch every this many
constexpr int kIncMaxD = 1024; // NEXT-3 incremental chains: grid steps up to this (two blocks staged in SMEM)
// small windows on the sorted path: one warp per window, E = 2, 4, 8 keys per lane (w <= 32 E)
cudaError_t launch_wsorted(const KsgLaunch& L, const int32_t* list, int32_t n, int E, int G, cudaStream_t st);
// fused latency path: items {list pos, slice start}; slices of fused_ppc(w, gmax) points
cudaError_t launch_fused(const KsgLaunch& L, const int32_t* list, const KsgItem* items, int32_t n_items, int gmax,
                         cudaStream_t st);
int fused_ppc(int w, int gmax);
cudaError_t launch_psi_tables(double* psi, long long* psiq, double* inv, int64_t m_max, double* lnc,
                              cudaStream_t st);
cudaError_t launch_nonfinite_scan(const float* p, int64_t n, int* flag, cudaStream_t st);
// Opt a kernel into > 48 KB of dynamic shared memory on the current device.  The attribute is per device,
// so this is done once per (device, kernel) under a lock (several devices / threads per process).
cudaError_t smem_optin(const void* kernel, int bytes);

// ---------------------------------------------------------------- errors
struct Status {
    int code = ISYCOS_OK;
    std::string msg;
    bool ok() const { return code == ISYCOS_OK; }
};
Status make_err(int code, const std::string& msg);
Status cuda_err(cudaError_t e, const char* what);
void set_last_error(const Status& s);

// ---------------------------------------------------------------- engine
struct DebugOut {
    float* eps = nullptr;     // device pointers (engine writes directly), or nullptr
    int32_t* nx = nullptr;
    int32_t* ny = nullptr;
};

struct BatchStats {
    int64_t windows = 0, point_pairs = 0, launches = 0, ksg_launches = 0, rounds = 0;
    int64_t scan_steps = 0, sorted_windows = 0, sorted_points = 0;
    int64_t brute_pairs = 0, search_probes = 0;
    int64_t block_windows = 0, block_points = 0;  // NEXT-3: windows merged from shared blocks, block points sorted
    int64_t inc_windows = 0, eps_reused = 0;      // NEXT-3: incremental windows, points whose radius carried over
    double sorted_ms = 0.0, brute_ms = 0.0;
    int64_t prof_rounds = 0, prof_brute_pairs = 0, prof_scan_steps = 0, prof_probes = 0;
    double kernel_ms = 0.0;
    int64_t h2d_bytes = 0, d2h_bytes = 0;
    double host_ms = 0.0, wall_ms = 0.0;
    void add_to(isycos_kernel_stats* s) const;
};

class Engine;
Engine* engine_for_current_device(Status* st);
void release_engine_for_current_device();

class Engine {
public:
    // Evaluate windows of a batch.  pairs: host array of device pointer pairs.  Results are
    // written to recs_host (pinned or pageable host memory) or, if recs_dev != nullptr, left in
    // device memory at recs_dev (caller-owned device buffer of n KsgRec).
    Status evaluate(const PairPtrs* pairs, int32_t n_pairs, const KsgWin* wins, int64_t n, int32_t k,
                    int32_t variant, KsgRec* recs_host, const DebugOut& dbg, cudaStream_t st,
                    uint32_t flags /* ISYCOS_F_* */, BatchStats* bs);

    // Device copy of a series (padded to a multiple of 4 floats, 16-B aligned).
    Status upload_series(const float* src, int64_t n, bool src_is_device, float** dev_out, cudaStream_t st,
                         BatchStats* bs);
    Status check_finite(const float* dev, int64_t n, cudaStream_t st, bool* finite);
    void free_series(float* p);

    cudaStream_t own_stream() const { return stream_; }
    int device() const { return dev_; }
    ~Engine();

    Status init(int dev);

    // Asynchronous form (the search driver pipelines two batches): submit() packs and launches a batch on
    // slot si (0 or 1) and returns; collect() waits for it and copies the records out.  A slot holds one
    // batch at a time; its buffers stay untouched until collected.  evaluate() = submit(0) + collect(0).
    Status submit(int si, const PairPtrs* pairs, int32_t n_pairs, const KsgWin* wins, int64_t n, int32_t k,
                  int32_t variant, const DebugOut& dbg, cudaStream_t st, uint32_t flags, BatchStats* bs);
    Status collect(int si, KsgRec* recs_host, BatchStats* bs);
    // collect() without the copy: *view points at the slot's pinned records (valid until the slot's next
    // submit); the caller adds the records' scan steps to bs->scan_steps itself (count_steps = false)
    Status collect_view(int si, const KsgRec** view, BatchStats* bs, bool count_steps, bool* profiled = nullptr);
    cudaStream_t second_stream() const { return stream2_; }
    // host time of submit() (ms, accumulated over the engine's life): binning, NEXT-3 block plan, other
    // preparation, descriptor packing, launches (ISYCOS_TRACE summaries)
    double sub_ms[5] = {0.0, 0.0, 0.0, 0.0, 0.0};
    Status fork_second_stream(cudaStream_t st);  // second stream waits for work queued on st so far
    Status join_second_stream(cudaStream_t st);  // st waits for the second stream

private:
    static constexpr int kAux = 4;   // auxiliary streams per slot for overlapping size classes
    static constexpr int64_t kZeroCopyMaxRecs = 8192;
    struct Slot {                    // per in-flight batch: staging, records, accumulators, scratch, streams
        KsgAcc* acc = nullptr;
        int64_t acc_cap = 0;
        char* dstage = nullptr;      // packed [pairs | wins | lists | items]
        int64_t dstage_cap = 0;
        char* hstage = nullptr;      // pinned mirror of dstage
        int64_t hstage_cap = 0;
        KsgRec* drec = nullptr;      // device alias of hrec
        KsgRec* hrec = nullptr;      // mapped pinned (kernels write records here)
        int64_t hrec_cap = 0;
        KsgRec* ddrec = nullptr;     // device records for batches above kZeroCopyMaxRecs
        int64_t ddrec_cap = 0;
        char* sscratch = nullptr;    // sorted path scratch: [P2 | OX | YS | TX | TI | TY] per point
        int64_t sscratch_cap = 0;
        unsigned* sync = nullptr;    // NEXT-3 chains: [work ticket | per-window finished scan CTAs]
        int64_t sync_cap = 0;
        std::vector<cudaEvent_t> events;
        cudaStream_t aux[kAux] = {};
        cudaEvent_t fork_ev = nullptr;
        cudaEvent_t join_ev[kAux] = {};
        // the batch in flight
        bool busy = false, profile = false;
        cudaStream_t st = nullptr;
        int64_t n = 0, pp = 0, brute_pairs = 0, probes = 0, sorted_windows = 0, spts = 0;
        int64_t block_windows = 0, block_points = 0, inc_windows = 0;
        int n_ksg = 0, n_launch = 0;
        std::vector<int> launch_cls;
    };

    Status ensure_psi(int64_t w_max, cudaStream_t st);
    Status ensure_capacity(Slot& S, int64_t n_wins, int64_t n_items, int32_t n_pairs, int64_t n_lists,
                           int64_t extra_bytes);

    int dev_ = -1;
    cudaStream_t stream_ = nullptr;
    cudaStream_t stream2_ = nullptr;  // second slot's stream for the pipelined search
    cudaEvent_t xev_ = nullptr;       // fork/join event between stream_/caller stream and stream2_
    // digamma tables
    double* psi_ = nullptr;
    long long* psiq_ = nullptr;
    double* lnc_ = nullptr;
    int64_t psi_max_ = 0;
    int32_t knn_mode_ = 1;
    int* dflag_ = nullptr;
    Slot slots_[2];
    struct Bins {                    // size-class lists of the batch being packed (reused)
        std::vector<int32_t> small[4], tile[3], sorted, fused, wsorted[3], lat, lat_tiny;
        std::vector<int64_t> soff;
        std::vector<int32_t> ord, beta;      // NEXT-3 block plan scratch
        std::vector<KsgBlk> blks;
        std::vector<KsgSegB> segb;
        std::vector<KsgInc> incs;
        std::vector<int64_t> wboff;
    } bins_;
    struct ChunkBins {               // one host thread's share of a large batch's binning (merged in order)
        std::vector<int32_t> small[4], tile[2], sorted, fused, wsorted[3];
        std::vector<int64_t> soff;   // relative to the chunk's own sorted-point count
        int64_t spts = 0, n_segs = 0, n_mblocks = 0, n_items = 0, pp = 0;
        int W2 = 0, fused_n2 = 256;
    };
    std::vector<ChunkBins> cbins_;
    bool inc_on_ = false;            // NEXT-3 incremental radii along grid chains (ISYCOS_INCREMENTAL=1 or
                                     // ISYCOS_F_INCREMENTAL enables; measured time-neutral, so off by default)
    int32_t inc_chain_ = kIncChain;  // chain length (ISYCOS_INC_CHAIN)
    int32_t scan_unified_ = 0;       // ISYCOS_SCAN_UNIFIED=1: one side per iteration (measured 5-15 % slower; results identical)
    uint32_t poison_ = 0;            // ISYCOS_POISON=<byte>: shared memory, scan scratch and records pre-filled (T5)
    bool lat_split_on_ = true;       // latency-mode small windows on the 8-lanes-per-point kernel (ISYCOS_LAT_SPLIT=0: tile R=1)
    bool block_sort_on_ = true;      // NEXT-3 shared-block sorts (env ISYCOS_BLOCK_SORT=0 disables; A/B knob)
    bool sorted_on_ = true;
    bool fused_on_ = true;           // sorted windows w <= kFusedMaxW: fused sort+scan kernel ...
    int64_t fused_max_pts_ = 148 * 2 * 512;  // ... when the batch has at most this many such points
    int32_t sorted_min_w_ = 257;
    int64_t aux_min_windows_ = 256;  // batches with more windows fork size classes onto aux streams
    int32_t wsorted_min_w_ = 65;     // small windows w in [this, 256]: warp-per-window sorted kernel
    int32_t sorted_ppc_ = kSortedPts;  // throughput scan: points per CTA
    int32_t fused_small_min_w_ = 1 << 30;  // latency mode: small windows >= this go to the fused kernel
    int64_t lat_windows_ = 148 * 4;  // small classes with fewer windows run in latency mode (tile R=1)
    int32_t lat_keep_small_R_ = 0;   // brute small classes with R <= this stay warp-per-window even when sparse
    int32_t lat_tiny_max_w_ = 32;    // latency mode: windows up to this size run warp-per-window in the lat launch
    int32_t col_min_w_ = 1 << 30;    // throughput scan: box-assisted phase A for windows >= this (ISYCOS_COL_MIN_W)
    int32_t lat_lanes4_max_w_ = 128; // latency kernel: 4 lanes per point up to this window size, else 8
    int bin_threads_ = 1;            // host threads of a large batch's binning (ISYCOS_BIN_THREADS)
    int32_t ws_group_ = 0;           // warp-sorted kernel: warps per window (ISYCOS_WS_GROUP = 1, 2, 4; 0 = by batch size)
    int lat_lanes(int w) const { return w <= lat_lanes4_max_w_ ? 4 : 8; }
    // warps per window of a warp-sorted launch of n windows: the most (<= 4) that keep n G warps within one
    // wave of 40 resident warps per SM (E = 8's shared-memory limit), so a sparse round's windows finish G
    // times sooner; a full batch keeps one warp per window
    int ws_group(int64_t n) const {
        if (ws_group_ == 1 || ws_group_ == 2 || ws_group_ == 4) return ws_group_;
        const int64_t cap = 148 * 40;
        return n * 4 <= cap ? 4 : n * 2 <= cap ? 2 : 1;
    }
};

// ---------------------------------------------------------------- search driver
struct SearchParams {
    int32_t k = 4, variant = 0, method = 3;
    int64_t s_min = 64, s_max = 512;
    std::vector<int64_t> sizes;
    bool noise = true;
    double tau_ratio = 0.25;
    int32_t p = 3;
    double sigma = 0.2;
    int64_t delta_td = 0, delta_bu = 0;
    int32_t t_max_idle = 3, h = 5, n_chunks = 1, lookahead = 32;
    int64_t spec_cap_mult = 4;   // BU: speculative climbs pause beyond this many s_min
    int32_t anchor_lookahead = 64;  // BU: climbs started at the predicted re-anchor point
    int32_t bu_depth = 4;           // BU: iterations of delta-neighbourhood requested per round
    int32_t trend_depth = 32;       // BU: positions requested along a climb's current direction (head climbs)
    int32_t ring_rank = 1 << 30;    // BU: climbs at most this many positions behind the head request rings
    int32_t host_threads = 0;       // advance-phase host threads over pairs (0 => min(16, hardware))
    int32_t profile_every = 1;      // ISYCOS_F_PROFILE in a search: time every N-th round (env ISYCOS_PROFILE_EVERY)
    bool pipeline = true;           // two batches in flight (host advance overlaps GPU evaluation)
    int32_t auto_M = 0, auto_m = 0;  // method 4 (AUTO): Alg. 3 sampling (0 => 20, 6)
    double auto_alpha = 0.0, auto_rho = 0.0;  // Eqs. 4-9 weights (0 => 0.5, 0.5)
    uint64_t seed = 0;
    uint32_t flags = 0;          // ISYCOS_F_PROFILE | ISYCOS_F_BRUTE
    int32_t chunk_begin = 0, chunk_end = 0;  // (pair, chunk) units: chunks [begin, end) only, unmerged
};

// Alg. 4 chunk plan (clipped) and the chunk merge (reading R20), shared by the search driver and
// isycos_merge_windows.
std::vector<std::pair<int64_t, int64_t>> chunks_of(int64_t n, int32_t n_p, int64_t s_max);
std::vector<isycos_result_window> merge_windows(std::vector<isycos_result_window> all);

Status run_search(Engine* eng, const std::vector<PairPtrs>& pair_ptrs, const std::vector<int32_t>& pair_ids,
                  int64_t n, const SearchParams& P, cudaStream_t st, std::vector<isycos_result_window>* out,
                  isycos_search_stats* stats);

}  // namespace isy
