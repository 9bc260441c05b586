// TEST HARNESS (CPU): the product's batched search driver (paper_2204_09131_b200/csrc/search.cpp)
// linked against a stub Engine whose evaluate() computes each requested window with the ORACLE
// (oracle/oracle.cpp, extern "C" oracle_mi_batch) on host memory, or replays records from a table.
//
// Purpose: check on CPU that the speculative, batched, resumable driver reproduces the sequential
// oracle search exactly (results and algorithm-level counters), and profile its host time.  The
// product library never links this file or the oracle.
#include <chrono>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <string>
#include <unordered_map>
#include <vector>

#include "engine.h"

extern "C" int oracle_mi_batch(const float* x, const float* y, int64_t n, const int64_t* windows, int64_t nw,
                               int32_t k, int32_t variant, double* mi, double* h, double* nmi, int64_t* s_psi,
                               int64_t* s_log, int32_t* zero_eps);

namespace {
thread_local std::string g_err;
int64_t g_n = 0;                       // series length (host pointers in PairPtrs)
int64_t g_evaluated = 0;               // windows evaluated by the stub
double g_eval_ms = 0.0;                // time inside the stub's evaluate
// record cache keyed by (pair slot's x pointer, t0, w) so repeated profiling runs skip the oracle
struct Key {
    const float* x;
    int64_t t0;
    int32_t w;
    bool operator==(const Key& o) const { return x == o.x && t0 == o.t0 && w == o.w; }
};
struct KeyHash {
    size_t operator()(const Key& k) const {
        return std::hash<const void*>()(k.x) ^ (std::hash<int64_t>()(k.t0) * 1315423911u) ^ (size_t)k.w * 2654435761u;
    }
};
std::unordered_map<Key, isy::KsgRec, KeyHash> g_cache;
bool g_use_cache = false;
bool g_parallel = false;  // OpenMP over the batch's missing windows (profiling runs)
std::vector<isy::KsgRec> g_slot_recs[2];
bool g_slot_busy[2] = {false, false};
}  // namespace

namespace isy {
Status make_err(int code, const std::string& msg) {
    Status s;
    s.code = code;
    s.msg = msg;
    return s;
}
Status cuda_err(cudaError_t, const char* what) { return make_err(ISYCOS_E_CUDA, what); }
void set_last_error(const Status& s) { g_err = s.msg; }
void BatchStats::add_to(isycos_kernel_stats* s) const {
    if (!s) return;
    s->windows += windows;
    s->point_pairs += point_pairs;
    s->rounds += rounds;
    s->host_ms += host_ms;
    s->wall_ms += wall_ms;
}

Status Engine::evaluate(const PairPtrs* pairs, int32_t, const KsgWin* wins, int64_t n, int32_t k, int32_t variant,
                        KsgRec* recs_host, const DebugOut&, cudaStream_t, uint32_t, BatchStats* bs) {
    const auto t = std::chrono::steady_clock::now();
    std::vector<int64_t> miss;
    for (int64_t i = 0; i < n; ++i) {
        const PairPtrs& p = pairs[wins[i].pair];
        const Key key{p.x, wins[i].t0, wins[i].w};
        if (g_use_cache) {
            auto it = g_cache.find(key);
            if (it != g_cache.end()) {
                recs_host[i] = it->second;
                continue;
            }
        }
        miss.push_back(i);
    }
    // the oracle's psi table grows lazily (not thread-safe): evaluate the widest window first, serially
    int64_t widest = -1;
    for (int64_t i : miss)
        if (widest < 0 || wins[i].w > wins[widest].w) widest = i;
    int bad = 0;
    auto eval_one = [&](int64_t i) {
        const PairPtrs& p = pairs[wins[i].pair];
        int64_t w2[2] = {wins[i].t0, wins[i].t0 + wins[i].w};
        double mi, h, nmi;
        int64_t sp, sl;
        int32_t z;
        int rc = oracle_mi_batch(p.x, p.y, g_n, w2, 1, k, variant, &mi, &h, &nmi, &sp, &sl, &z);
        if (rc) bad = 1;
        recs_host[i] = KsgRec{mi, h, nmi, sp, sl, z, 0};
    };
    if (widest >= 0) eval_one(widest);
#pragma omp parallel for schedule(dynamic, 1) if (g_parallel)
    for (int64_t m = 0; m < (int64_t)miss.size(); ++m)
        if (miss[m] != widest) eval_one(miss[m]);
    if (bad) return make_err(ISYCOS_E_INVAL, "oracle_mi_batch failed");
    for (int64_t i : miss) {
        if (g_use_cache) g_cache[Key{pairs[wins[i].pair].x, wins[i].t0, wins[i].w}] = recs_host[i];
        bs->point_pairs += (int64_t)wins[i].w * (wins[i].w - 1);
    }
    bs->windows += n;
    bs->rounds += 1;
    g_evaluated += n;
    g_eval_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t).count();
    return Status{};
}
Status Engine::submit(int si, const PairPtrs* pairs, int32_t n_pairs, const KsgWin* wins, int64_t n, int32_t k,
                      int32_t variant, const DebugOut& dbg, cudaStream_t st, uint32_t flags, BatchStats* bs) {
    // the stub evaluates at submit time and hands the records out at collect (same observable order)
    g_slot_recs[si].resize(n);
    g_slot_busy[si] = true;
    return evaluate(pairs, n_pairs, wins, n, k, variant, g_slot_recs[si].data(), dbg, st, flags, bs);
}
Status Engine::collect(int si, KsgRec* recs_host, BatchStats*) {
    if (!g_slot_busy[si]) return Status{};
    g_slot_busy[si] = false;
    std::memcpy(recs_host, g_slot_recs[si].data(), g_slot_recs[si].size() * sizeof(KsgRec));
    return Status{};
}
Status Engine::collect_view(int si, const KsgRec** view, BatchStats*, bool, bool* profiled) {
    *view = g_slot_recs[si].data();
    if (profiled) *profiled = false;
    g_slot_busy[si] = false;
    return Status{};
}
Status Engine::fork_second_stream(cudaStream_t) { return Status{}; }
Status Engine::join_second_stream(cudaStream_t) { return Status{}; }
Engine::~Engine() {}
}  // namespace isy

extern "C" {

// keep evaluated records across calls (same series buffers) so profiling re-runs skip the oracle
void harness_parallel(int on) { g_parallel = on != 0; }

void harness_use_cache(int on) {
    g_use_cache = on != 0;
    if (!on) g_cache.clear();
}

struct HarnessParams {
    int32_t k, method, noise, p, h, t_max_idle, n_chunks, lookahead, bu_depth, anchor, spec_cap, trend, pipeline,
        ring_rank;
    int64_t s_min, s_max, delta_td, delta_bu;
    double sigma, tau_ratio;
    uint64_t seed;
    const int64_t* sizes;
    int64_t n_sizes;
    int32_t auto_M, auto_m;
    double auto_alpha, auto_rho;
};

// Runs isy::run_search over (xs, ys, id) pairs of host series.  out/stats as in isycos_search.
int harness_search(const float* const* series, int64_t n, const int32_t* pairs, int32_t n_pairs,
                   const HarnessParams* hp, isycos_result_window* out, int64_t cap, int64_t* count,
                   isycos_search_stats* stats, double* eval_ms, int64_t* evaluated) {
    isy::SearchParams P;
    P.k = hp->k;
    P.method = hp->method;
    P.noise = hp->noise != 0;
    P.p = hp->p;
    P.h = hp->h;
    P.t_max_idle = hp->t_max_idle;
    P.n_chunks = hp->n_chunks;
    if (hp->lookahead > 0) P.lookahead = hp->lookahead;
    if (hp->bu_depth > 0) P.bu_depth = hp->bu_depth;
    if (hp->trend >= 0) P.trend_depth = hp->trend;
    if (hp->pipeline >= 0) P.pipeline = hp->pipeline != 0;
    if (hp->ring_rank > 0) P.ring_rank = hp->ring_rank;
    if (hp->anchor >= 0) P.anchor_lookahead = hp->anchor;
    if (hp->spec_cap >= 0) P.spec_cap_mult = hp->spec_cap;
    P.s_min = hp->s_min;
    P.s_max = hp->s_max;
    P.delta_td = hp->delta_td;
    P.delta_bu = hp->delta_bu;
    P.sigma = hp->sigma;
    P.tau_ratio = hp->tau_ratio;
    P.seed = hp->seed;
    P.auto_M = hp->auto_M;
    P.auto_m = hp->auto_m;
    P.auto_alpha = hp->auto_alpha;
    P.auto_rho = hp->auto_rho;
    if (hp->sizes && hp->n_sizes > 0) P.sizes.assign(hp->sizes, hp->sizes + hp->n_sizes);
    std::vector<isy::PairPtrs> pp(n_pairs);
    std::vector<int32_t> ids(n_pairs);
    for (int32_t i = 0; i < n_pairs; ++i) {
        pp[i] = isy::PairPtrs{series[pairs[3 * i]], series[pairs[3 * i + 1]]};
        ids[i] = pairs[3 * i + 2];
    }
    g_n = n;
    g_evaluated = 0;
    g_eval_ms = 0.0;
    isy::Engine eng;  // stub: only evaluate() is used
    std::vector<isycos_result_window> res;
    std::memset(stats, 0, sizeof(*stats));
    isy::Status s = isy::run_search(&eng, pp, ids, n, P, nullptr, &res, stats);
    if (!s.ok()) return s.code;
    *count = (int64_t)res.size();
    for (int64_t i = 0; i < std::min<int64_t>(cap, (int64_t)res.size()); ++i) out[i] = res[i];
    *eval_ms = g_eval_ms;
    *evaluated = g_evaluated;
    return 0;
}
}

// profiling helpers: persist the record cache of a single-pair run (keys re-bound to `x` on load)
extern "C" int harness_cache_save(const char* path) {
    FILE* f = std::fopen(path, "wb");
    if (!f) return -1;
    for (auto& kv : g_cache) {
        std::fwrite(&kv.first.t0, 8, 1, f);
        std::fwrite(&kv.first.w, 4, 1, f);
        std::fwrite(&kv.second, sizeof(isy::KsgRec), 1, f);
    }
    std::fclose(f);
    return 0;
}
extern "C" int harness_cache_load(const char* path, const float* x) {
    FILE* f = std::fopen(path, "rb");
    if (!f) return -1;
    int64_t t0;
    int32_t w;
    isy::KsgRec r;
    while (std::fread(&t0, 8, 1, f) == 1 && std::fread(&w, 4, 1, f) == 1 && std::fread(&r, sizeof(r), 1, f) == 1)
        g_cache[Key{x, t0, w}] = r;
    std::fclose(f);
    return 0;
}
