// Batched search driver: SYCOS_TD (Alg. 1), SYCOS_BU (Alg. 2), MI-based noise
// pruning (Def 6.2, §6.2, §6.3), overlapping chunks (Alg. 4 line 14).
//
// SURVEY §8(a) a1 + a7.  The sequential algorithms are re-expressed as resumable state machines that
// never compute MI themselves: they ask a per-pair window cache, and every miss becomes a request.
// Each round the driver advances every job as far as the cache allows, then evaluates all pending
// windows of all jobs in ONE GPU batch (Engine::evaluate).  Two kinds of speculation keep batches
// large:
//   TD  at the start of each layer, every window of the layer's delta-grid (plus the noise
//       sub-windows) is requested at once; the layer is then replayed exactly (rounds = layers).
//   BU  a climb is a pure function of its start lo (its LAHC stream is keyed by (seed, pair, lo)), so
//       the climbs at lo, lo + s_min, lo + 2 s_min, ... (the chain if nothing is accepted) run in
//       lockstep; when the head finishes the chain advances, and an accept re-anchors the chain.
// Decisions use only canonical, bit-reproducible records, so the result set and the algorithm-level
// counters equal the sequential oracle's exactly (tests/test_gpu_search.py).

#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <functional>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <vector>

#include "engine.h"

namespace isy {
namespace {

struct Eval {
    double mi, h, nmi;
};

struct Entry {
    uint64_t key = 0;  // 0 = empty slot (a window key is never 0: w >= 2)
    Eval e{0, 0, 0};
    bool ready = false;
    bool consumed = false;
};

inline uint64_t wkey(int64_t t0, int64_t t1) { return ((uint64_t)t0 << 20) | (uint64_t)(t1 - t0); }
inline int64_t key_t0(uint64_t k) { return (int64_t)(k >> 20); }
inline int64_t key_w(uint64_t k) { return (int64_t)(k & ((1u << 20) - 1)); }

// Window cache: open addressing over (key, arena index), sharded by t0 >> 8 so the windows one climb or
// one TD layer touches (nearby t0) share a few small tables that stay cache-resident (the driver does ~1e6
// lookups per cfg2 search).  Entries live in a block arena and never move: an Entry* stays valid for the
// life of the cache (batches in flight keep pointers to the entries they will fill).
struct SmallMap {
    struct Slot {
        uint64_t key;
        uint32_t idx;
    };
    std::vector<Slot> tab;
    uint32_t mask = 0, count = 0;

    static uint32_t hash(uint64_t k) {
        k ^= k >> 29;
        k *= 0xbf58476d1ce4e5b9ull;
        return (uint32_t)(k >> 32);
    }
    void grow() {
        const size_t cap = tab.empty() ? 64 : tab.size() * 2;
        std::vector<Slot> nt(cap, Slot{0, 0});
        const uint32_t m = (uint32_t)cap - 1;
        for (const Slot& e : tab) {
            if (!e.key) continue;
            uint32_t i = hash(e.key) & m;
            while (nt[i].key) i = (i + 1) & m;
            nt[i] = e;
        }
        tab.swap(nt);
        mask = m;
    }
};

struct FlatMap {
    static constexpr int kShift = 8;  // shard = t0 >> 8
    static constexpr uint32_t kBlock = 4096;
    static constexpr size_t kMaxBlocks = size_t(1) << 16;  // concurrent mode: block table never reallocates
    std::vector<SmallMap> shards;
    std::vector<std::unique_ptr<Entry[]>> blocks;
    uint32_t size = 0;
    // Concurrent mode (one pair's climbs advanced on several host threads): a lock per shard guards its table,
    // one lock the arena; shards and the block table are sized up front, so neither vector reallocates while
    // another thread reads it.  Entries never move, so a returned Entry* stays valid without a lock.
    std::unique_ptr<std::mutex[]> shard_mu;
    std::mutex arena_mu;

    void make_concurrent(int64_t n_samples) {
        shards.resize((size_t)(n_samples >> kShift) + 2);
        shard_mu.reset(new std::mutex[shards.size()]);
        blocks.reserve(kMaxBlocks);
    }
    Entry& at(uint32_t i) { return blocks[i / kBlock][i % kBlock]; }
    const Entry& at(uint32_t i) const { return blocks[i / kBlock][i % kBlock]; }
    std::pair<Entry*, bool> try_emplace(uint64_t k) {
        const size_t sh = (size_t)(key_t0(k) >> kShift);
        if (shard_mu) {
            std::lock_guard<std::mutex> lk(shard_mu[sh]);
            return emplace_in(sh, k);
        }
        if (sh >= shards.size()) shards.resize(sh + 1);
        return emplace_in(sh, k);
    }
    Entry* find(uint64_t k) {
        const size_t sh = (size_t)(key_t0(k) >> kShift);
        if (sh >= shards.size()) return nullptr;
        if (shard_mu) {
            std::lock_guard<std::mutex> lk(shard_mu[sh]);
            return find_in(sh, k);
        }
        return find_in(sh, k);
    }
    template <typename F>
    void for_each(F&& f) const {
        for (uint32_t i = 0; i < size; ++i) f(at(i));
    }

private:
    std::pair<Entry*, bool> emplace_in(size_t sh, uint64_t k) {
        SmallMap& m = shards[sh];
        if ((m.count + 1) * 2 > m.tab.size()) m.grow();
        uint32_t i = SmallMap::hash(k) & m.mask;
        while (m.tab[i].key) {
            if (m.tab[i].key == k) return {&at(m.tab[i].idx), false};
            i = (i + 1) & m.mask;
        }
        uint32_t idx;
        if (shard_mu) {
            std::lock_guard<std::mutex> lk(arena_mu);
            if (size % kBlock == 0) {
                if (blocks.size() == kMaxBlocks) std::abort();  // 2^28 entries of one pair: never reached
                blocks.emplace_back(new Entry[kBlock]);
            }
            idx = size++;
        } else {
            if (size % kBlock == 0) blocks.emplace_back(new Entry[kBlock]);
            idx = size++;
        }
        m.tab[i] = SmallMap::Slot{k, idx};
        ++m.count;
        Entry& e = at(idx);
        e.key = k;
        return {&e, true};
    }
    Entry* find_in(size_t sh, uint64_t k) {
        SmallMap& m = shards[sh];
        if (m.tab.empty()) return nullptr;
        uint32_t i = SmallMap::hash(k) & m.mask;
        while (m.tab[i].key) {
            if (m.tab[i].key == k) return &at(m.tab[i].idx);
            i = (i + 1) & m.mask;
        }
        return nullptr;
    }
};

struct PairCache {
    FlatMap map;
    std::vector<Entry*> pending;  // requested, not yet staged (entries never move)
    std::mutex pending_mu;        // concurrent mode only
    void add_pending(Entry* e) {
        if (map.shard_mu) {
            std::lock_guard<std::mutex> lk(pending_mu);
            pending.push_back(e);
        } else {
            pending.push_back(e);
        }
    }
};

// t_w ~ w log w per MI request: Alg. 3's deterministic runtime proxy (DESIGN reading R24)
inline int64_t wcost(int64_t w) {
    int64_t L = 0;
    while ((int64_t(1) << L) < w) ++L;
    return w * L;
}

struct AlgStats {
    int64_t td_windows = 0, td_noise_checks = 0, td_skips = 0, td_accepted = 0;
    int64_t bu_climbs = 0, bu_iterations = 0, bu_neighbors = 0, bu_noise_checks = 0, bu_prunes = 0,
            bu_accepted = 0;
    int64_t eval_cost = 0;  // sum over the distinct windows consumed of w * ceil(log2 w) (set at retire)
    void add(const AlgStats& o) {
        td_windows += o.td_windows;
        td_noise_checks += o.td_noise_checks;
        td_skips += o.td_skips;
        td_accepted += o.td_accepted;
        bu_climbs += o.bu_climbs;
        bu_iterations += o.bu_iterations;
        bu_neighbors += o.bu_neighbors;
        bu_noise_checks += o.bu_noise_checks;
        bu_prunes += o.bu_prunes;
        bu_accepted += o.bu_accepted;
        eval_cost += o.eval_cost;
    }
};

// Window cache access for one pair.  get(): the record if evaluated, else nullptr (and the window is
// queued for the next batch).  Accesses are recorded in `touched` and marked consumed only when the
// owning step commits, so speculative work never enters the algorithm-level counters.
struct View {
    PairCache* c;
    std::vector<Entry*>* touched;
    const Eval* get(int64_t t0, int64_t t1) {
        const uint64_t k = wkey(t0, t1);
        auto r = c->map.try_emplace(k);
        if (r.second) {
            c->add_pending(r.first);
            return nullptr;
        }
        if (!r.first->ready) return nullptr;
        touched->push_back(r.first);
        return &r.first->e;
    }
    void want(int64_t t0, int64_t t1) {
        const uint64_t k = wkey(t0, t1);
        auto r = c->map.try_emplace(k);
        if (r.second) c->add_pending(r.first);
    }
    const Eval* peek(int64_t t0, int64_t t1) {  // no request, no consumption
        Entry* e = c->map.find(wkey(t0, t1));
        return (e && e->ready) ? &e->e : nullptr;
    }
};

void commit_touched(PairCache*, const std::vector<Entry*>& t) {
    for (Entry* e : t) e->consumed = true;
}

// ------------------------------------------------------------------ SYCOS_TD job
struct TdJob {
    const SearchParams* P;
    PairCache* cache;
    int32_t pair_id;
    int64_t lo, hi;
    std::vector<int64_t> sched;
    size_t layer = 0;
    bool layer_requested = false;
    bool done = false;
    std::vector<std::pair<int64_t, int64_t>> parts;
    std::vector<isycos_result_window> results;
    AlgStats stats;

    void init() {
        parts.assign(1, {lo, hi});
        if (!P->sizes.empty()) {
            sched = P->sizes;
        } else {
            sched.assign(1, P->s_max);  // S:348 halving s_max -> s_min
            while (sched.back() > P->s_min) sched.push_back(std::max(P->s_min, sched.back() / 2));
        }
    }
    int64_t delta(int64_t s) const { return P->delta_td > 0 ? P->delta_td : std::max<int64_t>(1, s / 4); }

    // The delta-grid of [t, b) anchored at t: every window the layer can visit there while no accept or
    // noise skip moves it off this grid (plus the two noise sub-windows of every shifted position).
    void request_grid(View& v, int64_t t, int64_t b, int64_t s, bool first_unshifted) {
        const int64_t d = delta(s);
        const bool nz = P->noise && d > P->k && s - d > P->k;
        for (int64_t u = t; u + s <= b; u += d) {
            v.want(u, u + s);
            if (nz && (u > t || !first_unshifted)) {
                v.want(u, u + s - d);
                v.want(u + s - d, u + s);
            }
        }
    }

    void request_layer(int64_t s) {
        std::vector<Entry*> dummy;
        View v{cache, &dummy};
        for (auto [a, b] : parts)
            if (b - a >= s) request_grid(v, a, b, s, true);
    }

    // One exact replay of the layer (Alg. 1 lines 3-15 over every partition).  Returns false if a
    // window is missing (it is then queued); nothing is committed in that case.
    bool replay_layer(int64_t s) {
        const int64_t d = delta(s);
        const double tau = P->tau_ratio * P->sigma;
        AlgStats ls;
        std::vector<isycos_result_window> lr;
        std::vector<std::pair<int64_t, int64_t>> next;
        std::vector<Entry*> touched;
        View v{cache, &touched};
        for (auto [a, b] : parts) {
            if (b - a < s) {
                next.push_back({a, b});
                continue;
            }
            int64_t t = a, pend = a;
            int streak = 0;
            bool shifted = false;
            while (t + s <= b) {
                ls.td_windows += 1;
                const Eval* e = v.get(t, t + s);
                if (!e) {
                    // off the layer-start grid (an accept or a noise skip moved t by s, s % delta != 0):
                    // queue the rest of this partition anchored at t, so it costs one round, not one per window
                    std::vector<Entry*> dummy;
                    View w{cache, &dummy};
                    request_grid(w, t, b, s, !shifted);
                    return false;
                }
                if (e->nmi >= P->sigma) {
                    lr.push_back({pair_id, 1, t, t + s, e->mi, e->h, e->nmi});
                    ls.td_accepted += 1;
                    if (t > pend) next.push_back({pend, t});
                    t = t + s;
                    pend = t;
                    streak = 0;
                    shifted = false;
                    continue;
                }
                if (P->noise && shifted && d > P->k && s - d > P->k) {
                    ls.td_noise_checks += 1;
                    const Eval* wo = v.get(t, t + s - d);
                    const Eval* wd = v.get(t + s - d, t + s);
                    if (!wo || !wd) return false;
                    const bool noisy = wd->nmi < tau && e->mi < wo->mi && wo->mi > 0.0;
                    streak = noisy ? streak + 1 : 0;
                    if (streak >= P->p) {
                        ls.td_skips += 1;
                        t = t + s;
                        streak = 0;
                        shifted = false;
                        continue;
                    }
                }
                t = t + d;
                shifted = true;
            }
            if (pend < b) next.push_back({pend, b});
        }
        // commit
        stats.add(ls);
        results.insert(results.end(), lr.begin(), lr.end());
        commit_touched(cache, touched);
        parts.clear();
        for (auto& q : next)
            if (q.second - q.first >= P->s_min) parts.push_back(q);
        return true;
    }

    void advance() {
        while (!done) {
            if (layer >= sched.size()) {
                done = true;
                break;
            }
            const int64_t s = sched[layer];
            if (!layer_requested) {
                layer_requested = true;
                request_layer(s);
                if (!cache->pending.empty()) return;  // wait for the grid batch
            }
            if (!replay_layer(s)) return;
            ++layer;
            layer_requested = false;
        }
    }
};

// ------------------------------------------------------------------ SYCOS_BU: one climb (Alg. 2 lines 2-24)
struct Rng {
    uint64_t s;
    uint64_t next() {
        s += 0x9E3779B97F4A7C15ull;
        uint64_t z = s;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        return z ^ (z >> 31);
    }
};

struct Climb {
    int64_t lo = 0;
    int state = 0;  // 0 start, 1 iterate, 2 done
    int64_t t0 = 0, t1 = 0;
    double Iw = 0.0;
    std::vector<double> L;
    int idle = 0;
    int streak[2] = {0, 0};
    bool pruned[2] = {false, false};
    Rng rng{0};
    AlgStats st;
    std::vector<Entry*> touched;
    bool accepted = false;
    bool finished = false;
    Eval fin{0, 0, 0};
    int64_t ring_t0 = -1, ring_t1 = -1;  // last depth-speculation request (want_ring)
    int last_da = 0, last_db = 0, run = 0;  // last move (in delta steps) and how many times in a row
    // values gathered for the current (position, pruned) state: reused by idle iterations
    int64_t it_t0 = -1, it_t1 = -1, it_b0 = 0, it_b1 = 0;
    int it_pf = -1, it_nc = 0;
    double it_bmi = 0.0;
    bool it_app[2] = {false, false};
    double it_ee_nmi[2] = {0.0, 0.0}, it_me_mi[2] = {0.0, 0.0};
    int ring_pf = -1;

    // Depth speculation: request every window the next bu_depth iterations could need — the rings
    // N_1..N_D of the delta-neighbourhood (Defs 5.2-5.3, Fig. 4's N_1/N_2) plus their noise extensions —
    // so a climb advances up to bu_depth iterations per round.  Requests only; nothing is consumed.
    // Trend speculation: a climb that has moved the same way twice in a row (e.g. a window growing to the
    // right inside a planted relation, one delta per iteration) will most likely keep going; request the
    // iteration windows (N_1 + noise extensions) of the next trend_depth positions on that line, so a long
    // monotone climb advances up to trend_depth iterations per round instead of bu_depth.  Requests only.
    void want_trend(View& v, const SearchParams& P, int64_t hi, int64_t d) {
        if (P.trend_depth <= 0 || run < 2) return;
        for (int m = 1; m <= P.trend_depth; ++m) {
            const int64_t p0 = t0 + (int64_t)m * last_da * d, p1 = t1 + (int64_t)m * last_db * d;
            if (p0 < lo || p1 > hi || p1 - p0 < P.s_min || p1 - p0 > P.s_max) break;
            for (int a = -1; a <= 1; ++a) {
                if (a < 0 && pruned[0]) continue;
                for (int b = -1; b <= 1; ++b) {
                    if ((a == 0 && b == 0) || (b > 0 && pruned[1])) continue;
                    const int64_t c0 = p0 + a * d, c1 = p1 + b * d;
                    if (c0 < lo || c1 > hi || c1 - c0 < P.s_min || c1 - c0 > P.s_max) continue;
                    v.want(c0, c1);
                }
            }
            if (P.noise && d > P.k) {
                if (!pruned[0] && p0 - d >= lo) v.want(p0 - d, p0);
                if (!pruned[1] && p1 + d <= hi) v.want(p1, p1 + d);
            }
        }
    }

    void want_ring(View& v, const SearchParams& P, int64_t hi, int64_t d) {
        const int D = P.bu_depth;
        if (D <= 1) return;
        // already requested around this window with the same pruned directions
        const int pf = (pruned[0] ? 1 : 0) | (pruned[1] ? 2 : 0);
        if (ring_t0 == t0 && ring_t1 == t1 && ring_pf == pf) return;
        // Incremental: after a move by (sa, sb) steps with the same pruned directions, the windows the
        // previous request already covered (old ring, old centre, old noise extensions) are skipped; the
        // validity tests are absolute, so a covered window was requested then.  (Optimisation only:
        // want() of a cached window is a no-op.)
        int64_t sa = 0, sb = 0;
        bool inc = ring_t0 >= 0 && ring_pf == pf && (t0 - ring_t0) % d == 0 && (t1 - ring_t1) % d == 0;
        if (inc) {
            sa = (t0 - ring_t0) / d;
            sb = (t1 - ring_t1) / d;
            inc = sa >= -D && sa <= D && sb >= -D && sb <= D;
        }
        ring_t0 = t0;
        ring_t1 = t1;
        ring_pf = pf;
        auto in_old = [&](int64_t a, int64_t b) { return inc && a + sa >= -D && a + sa <= D && b + sb >= -D && b + sb <= D; };
        for (int a = -D; a <= D; ++a) {
            if (a < 0 && pruned[0]) continue;
            for (int b = -D; b <= D; ++b) {
                if ((a == 0 && b == 0) || (b > 0 && pruned[1]) || in_old(a, b)) continue;
                const int64_t c0 = t0 + a * d, c1 = t1 + b * d;
                if (c0 < lo || c1 > hi || c1 - c0 < P.s_min || c1 - c0 > P.s_max) continue;
                v.want(c0, c1);
            }
        }
        if (!(P.noise && d > P.k)) return;
        for (int a = -(D - 1); a <= D - 1; ++a) {
            const int64_t l0 = t0 + a * d - d, r0 = t1 + a * d;
            const bool lo_cov = inc && a + sa >= -(D - 1) && a + sa <= D - 1;
            const bool ro_cov = inc && a + sb >= -(D - 1) && a + sb <= D - 1;
            if (!pruned[0] && !lo_cov && l0 >= lo && l0 + d <= hi) v.want(l0, l0 + d);
            if (!pruned[1] && !ro_cov && r0 >= lo && r0 + d <= hi) v.want(r0, r0 + d);
        }
    }

    // Advance as far as the cache allows.  Returns true when the climb is finished.  A speculative
    // climb whose window has grown beyond `cap` pauses (requests nothing) until it nears the chain head.
    bool advance(const SearchParams& P, PairCache* cache, int32_t pair_id, int64_t hi,
                 int64_t cap = INT64_MAX, bool ring = true) {
        if (finished) return true;
        View v{cache, &touched};
        const int64_t smin = P.s_min, smax = P.s_max;
        const int64_t d = P.delta_bu > 0 ? P.delta_bu : std::max<int64_t>(1, smin / 3);
        const double tau = P.tau_ratio * P.sigma;
        for (;;) {
            if (state == 0) {
                const Eval* e = v.get(lo, lo + smin);
                if (!e) return false;
                st.bu_climbs = 1;
                t0 = lo;
                t1 = lo + smin;
                Iw = e->mi;
                L.assign(P.h, Iw);
                idle = 0;
                rng.s = P.seed ^ ((uint64_t)(uint32_t)pair_id * 0x9E3779B97F4A7C15ull) ^
                        ((uint64_t)lo * 0xD1B54A32D192ED03ull);
                state = 1;
            }
            if (state == 1) {
                if (idle > P.t_max_idle) {
                    state = 2;
                    continue;
                }
                if (t1 - t0 > cap) return false;
                const int pf = (pruned[0] ? 1 : 0) | (pruned[1] ? 2 : 0);
                if (!(it_t0 == t0 && it_t1 == t1 && it_pf == pf)) {
                    // gather the iteration's windows: N1 (Def 5.2-5.3) in (t0,t1) order + noise windows
                    int64_t c0s[8], c1s[8];
                    int nc = 0;
                    for (int da = -1; da <= 1; ++da)
                        for (int db = -1; db <= 1; ++db) {
                            if (da == 0 && db == 0) continue;
                            if (da == -1 && pruned[0]) continue;
                            if (db == 1 && pruned[1]) continue;
                            const int64_t c0 = t0 + da * d, c1 = t1 + db * d;
                            if (c0 < lo || c1 > hi) continue;
                            const int64_t sz = c1 - c0;
                            if (sz < smin || sz > smax) continue;
                            c0s[nc] = c0;
                            c1s[nc] = c1;
                            ++nc;
                        }
                    if (nc == 0) {
                        state = 2;
                        continue;
                    }
                    bool applicable[2] = {false, false};
                    int64_t e0[2], e1[2], m0[2], m1[2];
                    const bool nz = P.noise && d > P.k;
                    for (int dir = 0; dir < 2 && nz; ++dir) {
                        if (pruned[dir]) continue;
                        if (dir == 0) {
                            e0[0] = t0 - d; e1[0] = t0; m0[0] = t0 - d; m1[0] = t1;
                        } else {
                            e0[1] = t1; e1[1] = t1 + d; m0[1] = t0; m1[1] = t1 + d;
                        }
                        applicable[dir] = !(e0[dir] < lo || e1[dir] > hi || m1[dir] - m0[dir] > smax);
                    }
                    const size_t mark = touched.size();
                    bool missing = false;
                    const Eval* ce[8];
                    for (int i = 0; i < nc; ++i) {
                        ce[i] = v.get(c0s[i], c1s[i]);
                        missing |= (ce[i] == nullptr);
                    }
                    const Eval* ee[2] = {nullptr, nullptr};
                    const Eval* me[2] = {nullptr, nullptr};
                    for (int dir = 0; dir < 2; ++dir) {
                        if (!applicable[dir]) continue;
                        ee[dir] = v.get(e0[dir], e1[dir]);
                        me[dir] = v.get(m0[dir], m1[dir]);
                        missing |= (ee[dir] == nullptr) | (me[dir] == nullptr);
                    }
                    if (missing) {
                        touched.resize(mark);
                        if (cap == INT64_MAX && !(ring_t0 == t0 && ring_t1 == t1)) want_trend(v, P, hi, d);
                        if (ring) want_ring(v, P, hi, d);
                        return false;
                    }
                    // best neighbour: first maximum of MI in (t0, t1) order (R15)
                    int best = 0;
                    for (int i = 1; i < nc; ++i)
                        if (ce[i]->mi > ce[best]->mi) best = i;
                    it_t0 = t0;
                    it_t1 = t1;
                    it_pf = pf;
                    it_nc = nc;
                    it_b0 = c0s[best];
                    it_b1 = c1s[best];
                    it_bmi = ce[best]->mi;
                    for (int dir = 0; dir < 2; ++dir) {
                        it_app[dir] = applicable[dir];
                        it_ee_nmi[dir] = applicable[dir] ? ee[dir]->nmi : 0.0;
                        it_me_mi[dir] = applicable[dir] ? me[dir]->mi : 0.0;
                    }
                }
                // the iteration, exactly as Alg. 2 lines 7-21 (an idle iteration at the same position and
                // pruned state reuses the gathered values: the LAHC draw and the noise streaks still advance)
                st.bu_neighbors += it_nc;
                st.bu_iterations += 1;
                for (int dir = 0; dir < 2; ++dir) {
                    if (!it_app[dir]) continue;
                    st.bu_noise_checks += 1;
                    const bool noisy = it_ee_nmi[dir] < tau && it_me_mi[dir] < Iw && Iw > 0.0;
                    streak[dir] = noisy ? streak[dir] + 1 : 0;
                    if (streak[dir] >= P.p) {
                        pruned[dir] = true;
                        st.bu_prunes += 1;
                    }
                }
                const int r = (int)((rng.next() >> 32) % (uint64_t)P.h);
                const double Ih = L[r];
                const double bI = it_bmi;
                if (bI > Ih || bI > Iw) {
                    const int da = (int)((it_b0 - t0) / d), db = (int)((it_b1 - t1) / d);
                    run = (da == last_da && db == last_db) ? run + 1 : 1;
                    last_da = da;
                    last_db = db;
                    t0 = it_b0;
                    t1 = it_b1;
                    Iw = bI;
                    idle = 0;
                } else {
                    idle += 1;
                    run = 0;
                }
                if (Iw > Ih) L[r] = Iw;
                continue;
            }
            // state 2: final acceptance test (Alg. 2 line 23)
            const Eval* e = v.get(t0, t1);
            if (!e) return false;
            fin = *e;
            accepted = fin.nmi >= P.sigma;
            finished = true;
            return true;
        }
    }
};

// ------------------------------------------------------------------ SYCOS_BU job: chain of climbs
struct BuJob {
    const SearchParams* P;
    PairCache* cache;
    int32_t pair_id;
    int64_t lo_c, hi;
    int64_t chain = 0;
    bool done = false;
    std::map<int64_t, Climb> climbs;
    std::vector<isycos_result_window> results;
    AlgStats stats;

    void init() { chain = lo_c; }

    void ensure_lookahead() {
        const int la = P->lookahead > 0 ? P->lookahead : 32;
        for (int j = 0; j < la; ++j) {
            const int64_t l = chain + (int64_t)j * P->s_min;
            if (l + P->s_min > hi) break;
            auto r = climbs.try_emplace(l);
            if (r.second) {
                r.first->second.lo = l;
                r.first->second.advance(*P, cache, pair_id, hi, cap_for(l), ring_for(l));
            }
        }
    }

    // Speculation policy: the head and the next climb run unrestricted; climbs further ahead pause
    // once their window exceeds spec_cap_mult * s_min (they are likely skipped by an accept).
    // Depth speculation (the radius-D ring) only for the climbs nearest the chain head: farther climbs
    // are the likeliest to be discarded by an accept, and their rings dominated the host time.
    bool ring_for(int64_t l) const { return (l - chain) / P->s_min <= P->ring_rank; }

    int64_t cap_for(int64_t l) const {
        const int64_t rank = (l - chain) / P->s_min;
        if (rank <= 1 || P->spec_cap_mult <= 0) return INT64_MAX;
        return P->spec_cap_mult * P->s_min;
    }

    // Anchor speculation: while the head idles on a window that would be accepted (nmi >= sigma), the
    // chain will most likely re-anchor at max(t1, lo + s_min); start the climbs of that chain now.
    void speculate_anchor(const Climb& c) {
        if (P->anchor_lookahead <= 0 || c.state != 1 || c.idle < 1) return;
        std::vector<Entry*> none;
        View v{cache, &none};
        const Eval* e = v.peek(c.t0, c.t1);
        if (!e || !(e->nmi >= P->sigma)) return;
        const int64_t a = std::max(c.t1, chain + P->s_min);
        for (int j = 0; j < P->anchor_lookahead; ++j) {
            const int64_t l = a + (int64_t)j * P->s_min;
            if (l + P->s_min > hi) break;
            auto r = climbs.try_emplace(l);
            if (r.second) {
                r.first->second.lo = l;
                r.first->second.advance(*P, cache, pair_id, hi, j <= 1 ? INT64_MAX : P->spec_cap_mult * P->s_min);
            }
        }
    }

    // Pipelined driver: climbs belong to one of two groups by the parity of lo / s_min (neighbours on the
    // chain alternate); advance(g) advances group g's climbs (g < 0: all) plus the chain bookkeeping.
    int group_of(int64_t l) const { return (int)((l / P->s_min) & 1); }

    // set by the driver when this job's pair is the only one advancing (its cache is then in concurrent mode):
    // the climbs of a group advance on the host pool (each climb touches only its own state and the cache)
    std::function<void(int, const std::function<void(int)>&)> par_for;

    void advance(int g = -1) {
        if (done) return;
        if (par_for && cache->map.shard_mu) {
            std::vector<std::pair<int64_t, Climb*>> cl;
            for (auto& kv : climbs)
                if (g < 0 || group_of(kv.first) == g) cl.push_back({kv.first, &kv.second});
            par_for((int)cl.size(), [&](int i) {
                cl[i].second->advance(*P, cache, pair_id, hi, cap_for(cl[i].first), ring_for(cl[i].first));
            });
        } else {
            for (auto& kv : climbs)
                if (g < 0 || group_of(kv.first) == g)
                    kv.second.advance(*P, cache, pair_id, hi, cap_for(kv.first), ring_for(kv.first));
        }
        ensure_lookahead();
        for (;;) {
            if (chain + P->s_min > hi) {
                done = true;
                climbs.clear();
                return;
            }
            auto it = climbs.find(chain);
            if (it == climbs.end()) {
                ensure_lookahead();
                it = climbs.find(chain);
            }
            Climb& c = it->second;
            if (!c.advance(*P, cache, pair_id, hi)) {
                speculate_anchor(c);
                return;
            }
            // commit the head climb (Alg. 2 lines 23-24; restart on the remainder)
            stats.add(c.st);
            commit_touched(cache, c.touched);
            int64_t next;
            if (c.accepted) {
                results.push_back({pair_id, 2, c.t0, c.t1, c.fin.mi, c.fin.h, c.fin.nmi});
                stats.bu_accepted += 1;
                next = std::max(c.t1, chain + P->s_min);
            } else {
                next = chain + P->s_min;
            }
            // drop climbs behind the chain and (after a re-anchor) those off the new grid
            for (auto jt = climbs.begin(); jt != climbs.end();) {
                const int64_t l = jt->first;
                if (l < next || (l - next) % P->s_min != 0)
                    jt = climbs.erase(jt);
                else
                    ++jt;
            }
            chain = next;
            ensure_lookahead();
        }
    }
};

// ------------------------------------------------------------------ host thread pool
// Pairs are independent state machines (own window cache, own jobs), so a round's advance phase runs
// them on several host threads (dynamic scheduling by an atomic counter; the caller participates).
// Multi-pair searches (configs[3], configs[4]) are host-bound without it.
class HostPool {
public:
    explicit HostPool(int n) {
        if (const char* sp = std::getenv("ISYCOS_POOL_SPIN")) spin_max_ = std::max(0, std::atoi(sp));
        for (int i = 1; i < n; ++i) threads_.emplace_back([this] { loop(); });
    }
    ~HostPool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_.store(true);
            gen_.fetch_add(1);
        }
        cv_.notify_all();
        for (auto& t : threads_) t.join();
    }
    int size() const { return (int)threads_.size() + 1; }
    // Runs f(0..count-1) on the pool.  Workers spin briefly between tasks (a search round is ~50 us, a
    // futex wake-up per worker per task cost more than the parallel work saved) and sleep when idle.
    void run(int count, const std::function<void(int)>& f) {
        if (threads_.empty() || count <= 1) {
            for (int i = 0; i < count; ++i) f(i);
            return;
        }
        fn_ = &f;
        total_ = count;
        next_.store(0, std::memory_order_relaxed);
        pending_.store((int)threads_.size(), std::memory_order_relaxed);
        {
            std::lock_guard<std::mutex> lk(mu_);
            gen_.fetch_add(1, std::memory_order_release);
        }
        if (sleepers_.load(std::memory_order_acquire) > 0) cv_.notify_all();
        work();
        while (pending_.load(std::memory_order_acquire) != 0) std::this_thread::yield();
    }

private:
    void work() {
        for (;;) {
            const int i = next_.fetch_add(1, std::memory_order_relaxed);
            if (i >= total_) break;
            (*fn_)(i);
        }
    }
    void loop() {
        uint64_t seen = 0;  // gen_ starts at 0 (a thread may start after the first run() began)
        for (;;) {
            uint64_t g = gen_.load(std::memory_order_acquire);
            for (int spin = 0; g == seen && spin < spin_max_; ++spin) {
                std::this_thread::yield();
                g = gen_.load(std::memory_order_acquire);
            }
            if (g == seen) {
                std::unique_lock<std::mutex> lk(mu_);
                sleepers_.fetch_add(1);
                cv_.wait(lk, [&] { return gen_.load() != seen; });
                sleepers_.fetch_sub(1);
                g = gen_.load();
            }
            seen = g;
            if (stop_.load()) return;
            work();
            pending_.fetch_sub(1, std::memory_order_acq_rel);
        }
    }
    std::vector<std::thread> threads_;
    std::mutex mu_;
    std::condition_variable cv_;
    const std::function<void(int)>* fn_ = nullptr;
    std::atomic<int> next_{0}, pending_{0}, sleepers_{0};
    std::atomic<uint64_t> gen_{0};
    std::atomic<bool> stop_{false};
    int total_ = 0;
    int spin_max_ = 20000;  // yields before a worker sleeps (ISYCOS_POOL_SPIN)
};

// Asynchronous submit (ISYCOS_ASYNC_SUBMIT, default on): one thread runs Engine::submit (binning, packing,
// launches) for the batches the main thread posts, in posting order, so a group's submit overlaps the other
// group's advance.  collect of a slot first waits for that slot's submit.  Results never depend on it.
class Submitter {
public:
    struct Job {
        int g = 0;
        std::vector<PairPtrs> table;
        const KsgWin* wins = nullptr;
        int64_t n = 0;
        int32_t k = 0, variant = 0;
        cudaStream_t st = nullptr;
        uint32_t flags = 0;
    };
    explicit Submitter(Engine* e) : eng_(e), th_([this] { loop(); }) {}
    ~Submitter() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        th_.join();
    }
    void post(Job&& j) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            pending_[j.g] = true;
            q_.push_back(std::move(j));
        }
        cv_.notify_all();
    }
    Status wait(int g) {  // the status of slot g's last posted submit, once it has run
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return !pending_[g]; });
        return st_[g];
    }
    BatchStats bs;  // the submit thread's share of the batch statistics (h2d bytes), merged by the caller

private:
    void loop() {
        for (;;) {
            Job j;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || !q_.empty(); });
                if (q_.empty()) return;  // stop requested and nothing queued
                j = std::move(q_.front());
                q_.pop_front();
            }
            Status s = eng_->submit(j.g, j.table.data(), (int32_t)j.table.size(), j.wins, j.n, j.k, j.variant,
                                    DebugOut{}, j.st, j.flags, &bs);
            {
                std::lock_guard<std::mutex> lk(mu_);
                st_[j.g] = s;
                pending_[j.g] = false;
            }
            cv_.notify_all();
        }
    }
    Engine* eng_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<Job> q_;
    bool pending_[2] = {false, false};
    Status st_[2];
    bool stop_ = false;
    std::thread th_;  // last: starts after the members it reads are constructed
};

}  // namespace

// ------------------------------------------------------------------ chunks + merge
std::vector<std::pair<int64_t, int64_t>> chunks_of(int64_t n, int32_t n_p, int64_t s_max) {
    std::vector<std::pair<int64_t, int64_t>> c;
    const int64_t len = (n + n_p - 1) / n_p;
    for (int32_t i = 0; i < n_p; ++i) {
        const int64_t a = (int64_t)i * len;
        if (a >= n) break;
        c.push_back({std::max<int64_t>(0, a - s_max), std::min<int64_t>(n, a + len)});
    }
    return c;
}

// greedy by (nmi desc, mi desc, t0 asc, t1 asc), keep if disjoint from every kept window, sort by t0
std::vector<isycos_result_window> merge_windows(std::vector<isycos_result_window> all) {
    std::sort(all.begin(), all.end(), [](const isycos_result_window& a, const isycos_result_window& b) {
        if (a.nmi != b.nmi) return a.nmi > b.nmi;
        if (a.mi != b.mi) return a.mi > b.mi;
        if (a.t0 != b.t0) return a.t0 < b.t0;
        return a.t1 < b.t1;
    });
    std::vector<isycos_result_window> kept;
    for (auto& r : all) {
        bool clash = false;
        for (auto& q : kept)
            if (r.t0 < q.t1 && q.t0 < r.t1) {
                clash = true;
                break;
            }
        if (!clash) kept.push_back(r);
    }
    std::sort(kept.begin(), kept.end(),
              [](const isycos_result_window& a, const isycos_result_window& b) { return a.t0 < b.t0; });
    return kept;
}

namespace {

struct PairWork {
    int32_t inflight = 0;  // batches in flight holding entries of this pair
    // this round's requests, staged by the pair's own (parallel) advance task
    std::vector<KsgWin> stage_w;
    std::vector<Entry*> stage_o;
    bool stage_bad = false;
    int64_t bad_t0 = 0, bad_t1 = 0;
    int32_t method = 3;    // 1 TD, 2 BU, 3 both
    int32_t kind = 0;      // 0: a search whose windows are results; 1: an iSYCOS trial run (Alg. 3 l.3-4)
    int32_t auto_id = -1;  // trial runs: index of the pair's selection state
    int32_t slot = -1;  // index into the active PairPtrs table
    int32_t pair_id = 0;
    PairPtrs ptrs{};
    PairCache cache;
    std::vector<TdJob> td;
    std::vector<BuJob> bu;
    bool finished() const {
        for (auto& j : td)
            if (!j.done) return false;
        for (auto& j : bu)
            if (!j.done) return false;
        return true;
    }
};

// A finished pair's share of the output: result windows (merged per method unless chunks are selected),
// algorithm counters, Alg. 3 trial counts, and the distinct windows its algorithms consumed.
struct Retired {
    AlgStats ps;
    std::vector<isycos_result_window> res;
    int64_t nL_td = 0, nS_bu = 0;
    int64_t dw = 0, dpp = 0;
};

void retire_pair(PairWork& pw, Retired& R, const SearchParams& P, bool chunk_sel) {
    pw.cache.pending.clear();  // leftover speculative requests of discarded climbs
    for (int m = 1; m <= 2; ++m) {
        std::vector<isycos_result_window> per;
        if (m == 1)
            for (auto& j : pw.td) {
                per.insert(per.end(), j.results.begin(), j.results.end());
                R.ps.add(j.stats);
            }
        else
            for (auto& j : pw.bu) {
                per.insert(per.end(), j.results.begin(), j.results.end());
                R.ps.add(j.stats);
            }
        if (!(pw.method & m)) continue;
        if (pw.kind == 1) {  // trial run: countWindows, |w| <= rho * s_max is small
            const double rho = P.auto_rho > 0.0 ? P.auto_rho : 0.5;
            for (const auto& r : per) {
                const bool small = (double)(r.t1 - r.t0) <= rho * (double)P.s_max;
                if (m == 1 && !small) R.nL_td += 1;
                if (m == 2 && small) R.nS_bu += 1;
            }
            continue;
        }
        if (chunk_sel) {  // merged by isycos_merge_windows once every chunk is gathered
            R.res.insert(R.res.end(), per.begin(), per.end());
            continue;
        }
        auto merged = merge_windows(per);
        R.res.insert(R.res.end(), merged.begin(), merged.end());
    }
    pw.cache.map.for_each([&](const Entry& en) {
        if (en.consumed) {
            const int64_t w = key_w(en.key);
            R.dw += 1;
            R.dpp += w * (w - 1);
            R.ps.eval_cost += wcost(w);
        }
    });
}

// Retires finished searches off the critical path: counts, merges and frees each pair's cache on its own
// thread; the outputs are collected in retire order when the search ends.
class Reaper {
public:
    Reaper(const SearchParams& P, bool chunk_sel) : P_(P), sel_(chunk_sel), th_([this] { loop(); }) {}
    ~Reaper() { finish(); }
    void push(std::unique_ptr<PairWork> pw) {
        {
            std::lock_guard<std::mutex> lk(mu_);
            q_.push_back(std::move(pw));
            out_.emplace_back();
        }
        cv_.notify_one();
    }
    std::deque<Retired>& finish() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_one();
        if (th_.joinable()) th_.join();
        return out_;
    }

private:
    void loop() {
        size_t next = 0;
        for (;;) {
            std::unique_ptr<PairWork> pw;
            Retired* slot = nullptr;
            {
                std::unique_lock<std::mutex> lk(mu_);
                cv_.wait(lk, [&] { return stop_ || next < out_.size(); });
                if (next >= out_.size()) return;
                pw = std::move(q_[next]);
                slot = &out_[next];  // deque: element addresses are stable under push_back
                ++next;
            }
            retire_pair(*pw, *slot, P_, sel_);
            pw.reset();
        }
    }
    const SearchParams& P_;
    bool sel_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::deque<std::unique_ptr<PairWork>> q_;
    std::deque<Retired> out_;
    bool stop_ = false;
    std::thread th_;
};

}  // namespace

Status run_search(Engine* eng, const std::vector<PairPtrs>& pair_ptrs, const std::vector<int32_t>& pair_ids,
                  int64_t n, const SearchParams& P, cudaStream_t st, std::vector<isycos_result_window>* out,
                  isycos_search_stats* stats) {
    const int32_t n_pairs = (int32_t)pair_ptrs.size();
    auto plan = chunks_of(n, std::max(1, P.n_chunks), P.s_max);
    const bool chunk_sel = P.chunk_end > P.chunk_begin;  // (pair, chunk) units: these chunks only, unmerged
    if (chunk_sel) {
        if (P.chunk_begin < 0 || P.chunk_end > (int32_t)plan.size())
            return make_err(ISYCOS_E_INVAL, "chunk range outside the plan");
        plan = std::vector<std::pair<int64_t, int64_t>>(plan.begin() + P.chunk_begin, plan.begin() + P.chunk_end);
    }
    // pairs (units) searched concurrently: every round batches the requests of all of them
    int max_active = 64;
    if (const char* ma = std::getenv("ISYCOS_MAX_ACTIVE")) max_active = std::max(1, std::atoi(ma));
    AlgStats total;
    BatchStats bs;
    int64_t distinct_w = 0, distinct_pp = 0;
    std::vector<isycos_result_window> all;
    std::vector<std::unique_ptr<PairWork>> active;
    // work units: a (pair, method, ranges) search; AUTO (iSYCOS, Alg. 3) pairs first queue 2m trial units
    // (SYCOS_TD and SYCOS_BU alone on each sampled partition, own window cache each, like the oracle's
    // fresh Searcher per trial), then, when the last trial retires, the chosen method over the full series
    struct Unit {
        int32_t pair_idx, method, kind, auto_id;
        std::vector<std::pair<int64_t, int64_t>> ranges;
    };
    struct AutoState {
        int32_t pair_idx, left;
        int64_t cost_td = 0, cost_bu = 0, nL_td = 0, nS_bu = 0;
        double nscore_td = 0.0, nscore_bu = 0.0;
        int32_t chosen = 0;
    };
    std::deque<Unit> queue;
    std::vector<AutoState> autos;
    int n_threads = P.host_threads;
    if (n_threads <= 0) n_threads = (int)std::min<unsigned>(16u, std::max(1u, std::thread::hardware_concurrency()));
    // one pair: its BU climbs may spread over the pool instead (ISYCOS_PAR_CLIMBS=1; measured 2x slower on
    // configs[1] — per-round dispatch and shard-lock traffic exceed the ~25 us of climb work per round — so off)
    bool par_climbs = false;
    if (const char* pc = std::getenv("ISYCOS_PAR_CLIMBS"))
        par_climbs = std::atoi(pc) != 0 && n_pairs == 1 && P.method != 4 && (P.method & 2) && P.n_chunks <= 1;
    if (n_pairs <= 1 && P.method != 4 && !par_climbs) n_threads = 1;  // one pair: nothing to spread
    HostPool pool(n_threads);
    Reaper reaper(P, chunk_sel);
    const int32_t aM = P.auto_M > 0 ? P.auto_M : 20, am = P.auto_m > 0 ? P.auto_m : 6;
    for (int32_t p = 0; p < n_pairs; ++p) {
        if (P.method != 4) {
            queue.push_back(Unit{p, P.method, 0, -1, plan});
            continue;
        }
        // Alg. 3 line 1, randomSampling(M): partial Fisher-Yates on a SplitMix64 stream keyed by (seed, pair)
        const int64_t Lp = n / aM;
        std::vector<int32_t> idx(aM);
        for (int32_t i = 0; i < aM; ++i) idx[i] = i;
        Rng rng{P.seed ^ ((uint64_t)(uint32_t)pair_ids[p] * 0x9E3779B97F4A7C15ull) ^ 0xA0761D6478BD642Full};
        for (int32_t i = 0; i < am; ++i) {
            const int32_t j = i + (int32_t)((rng.next() >> 32) % (uint64_t)(aM - i));
            std::swap(idx[i], idx[j]);
        }
        const int32_t aid = (int32_t)autos.size();
        autos.push_back(AutoState{p, 2 * am});
        for (int32_t i = 0; i < am; ++i) {
            const int64_t lo = (int64_t)idx[i] * Lp;
            queue.push_back(Unit{p, 1, 1, aid, {{lo, lo + Lp}}});
            queue.push_back(Unit{p, 2, 1, aid, {{lo, lo + Lp}}});
        }
    }
    // the round's batch: grown, never re-initialised (a value-initialising resize of a 10^7-window TD round
    // costs more host time than the copy itself)
    std::unique_ptr<KsgWin[]> batches[2];  // one per group: an asynchronous submit may still read the other
    int64_t batch_caps[2] = {0, 0}, batch_n = 0;
    using clk = std::chrono::steady_clock;
    const auto t_start = clk::now();
    auto t_last = t_start;
    double eval_ms = 0.0, adv_ms = 0.0, wait_ms = 0.0, dlv_ms = 0.0, ret_ms = 0.0, asm_ms = 0.0;
    int64_t round_no = 0;
    std::FILE* trace = nullptr;
    if (const char* tp = std::getenv("ISYCOS_TRACE")) trace = std::fopen(tp, "a");
    struct Closer {
        std::FILE*& f;
        ~Closer() {
            if (f) std::fclose(f);
        }
    } closer{trace};

    // Two batches in flight (P.pipeline): while the GPU evaluates one group's batch, the host advances
    // the other group's jobs and submits its batch, so host time and GPU time overlap.  Group 0 = TD jobs
    // + even BU climbs, group 1 = odd BU climbs.  Results never depend on this schedule: every decision
    // reads canonical cached records only.
    struct Flight {
        bool busy = false;
        std::vector<Entry*> owners;
        std::vector<PairWork*> pws;
        std::vector<int64_t> offs;  // batch offset of each pair in pws (+ end)
        int64_t n = 0;              // windows in flight (owners[0..n))
    };
    Flight fl[2];
    bool async_submit = P.pipeline;
    if (const char* a = std::getenv("ISYCOS_ASYNC_SUBMIT")) async_submit = async_submit && std::atoi(a) != 0;
    std::unique_ptr<Submitter> submitter;
    if (async_submit) submitter = std::make_unique<Submitter>(eng);
    // error exits leave no batch in flight: the slot's staging buffer and mapped records would otherwise be
    // reused by the next call while the old copies and kernels still run (queued submits run first)
    struct Drain {
        Engine* eng;
        Flight* fl;
        std::unique_ptr<Submitter>* sub;
        ~Drain() {
            for (int g = 0; g < 2; ++g)
                if (*sub) (*sub)->wait(g);
            for (int g = 0; g < 2; ++g)
                if (fl[g].busy) eng->collect(g, nullptr, nullptr);
            sub->reset();
        }
    } drain{eng, fl, &submitter};
    const int n_groups = P.pipeline ? 2 : 1;
    cudaStream_t sts[2] = {st, eng->second_stream()};
    if (n_groups == 2) {  // the second slot's stream starts after everything already queued on st
        Status s = eng->fork_second_stream(st);
        if (!s.ok()) return s;
    }
    auto deliver = [&](int g) -> Status {
        Flight& F = fl[g];
        if (!F.busy) return Status{};
        const KsgRec* recs = nullptr;
        const auto t_ev = clk::now();
        bool profiled = false;
        if (submitter) {
            Status ss = submitter->wait(g);
            if (!ss.ok()) {
                F.busy = false;  // the slot never launched (or its submit failed part-way: the Drain syncs it)
                return ss;
            }
        }
        Status s = eng->collect_view(g, &recs, &bs, false, &profiled);
        const double wms = std::chrono::duration<double, std::milli>(clk::now() - t_ev).count();
        eval_ms += wms;
        wait_ms += wms;
        if (!s.ok()) return s;
        const auto t_dl = clk::now();
        // records -> entries, pairs in parallel for big batches (each pair's records are a contiguous slice),
        // read straight from the pinned records; the per-pair scan-step sums feed the kernel stats
        const bool par = F.n >= 512;
        std::vector<unsigned long long> steps(par ? F.pws.size() : 1, 0ull), reuse(steps.size(), 0ull);
        pool.run(par ? (int)F.pws.size() : 1, [&](int p) {
            const int64_t i0 = par ? F.offs[p] : 0, i1 = par ? F.offs[p + 1] : F.n;
            unsigned long long st = 0, ru = 0;
            for (int64_t i = i0; i < i1; ++i) {
                Entry& e = *F.owners[i];
                e.e = Eval{recs[i].mi, recs[i].h, recs[i].nmi};
                e.ready = true;
                st += recs[i].steps;
                ru += (unsigned)recs[i].reused;
            }
            steps[par ? p : 0] = st;
            reuse[par ? p : 0] = ru;
        });
        for (unsigned long long v : steps) {
            bs.scan_steps += (int64_t)v;
            if (profiled) bs.prof_scan_steps += (int64_t)v;
        }
        for (unsigned long long v : reuse) bs.eps_reused += (int64_t)v;
        for (PairWork* pw : F.pws) pw->inflight -= 1;
        dlv_ms += std::chrono::duration<double, std::milli>(clk::now() - t_dl).count();
        F.busy = false;
        F.n = 0;
        F.pws.clear();
        F.offs.clear();
        return Status{};
    };

    for (;;) {
        bool progress = false;  // any delivery, admission, retirement or submission this cycle
        for (int g = 0; g < n_groups; ++g) {
            if (fl[g].busy) {
                Status s = deliver(g);
                if (!s.ok()) return s;
                progress = true;
            }
            // admit pairs
            while ((int)active.size() < max_active && !queue.empty()) {
                Unit u = std::move(queue.front());
                queue.pop_front();
                auto pw = std::make_unique<PairWork>();
                pw->pair_id = pair_ids[u.pair_idx];
                pw->ptrs = pair_ptrs[u.pair_idx];
                pw->method = u.method;
                pw->kind = u.kind;
                pw->auto_id = u.auto_id;
                for (auto [lo, hi] : u.ranges) {
                    if (u.method & 1) {
                        TdJob j;
                        j.P = &P;
                        j.cache = &pw->cache;
                        j.pair_id = pw->pair_id;
                        j.lo = lo;
                        j.hi = hi;
                        pw->td.push_back(std::move(j));
                    }
                    if (u.method & 2) {
                        BuJob j;
                        j.P = &P;
                        j.cache = &pw->cache;
                        j.pair_id = pw->pair_id;
                        j.lo_c = lo;
                        j.hi = hi;
                        pw->bu.push_back(std::move(j));
                    }
                }
                for (auto& j : pw->td) {
                    j.cache = &pw->cache;
                    j.init();
                }
                if (par_climbs && pool.size() > 1) {
                    pw->cache.map.make_concurrent(n);
                    for (auto& j : pw->bu)
                        j.par_for = [&pool](int cnt, const std::function<void(int)>& f) { pool.run(cnt, f); };
                }
                for (auto& j : pw->bu) {
                    j.cache = &pw->cache;
                    j.init();
                }
                active.push_back(std::move(pw));
                progress = true;
            }
            // advance this group's jobs (pairs in parallel on the host pool)
            const auto t_adv = clk::now();
            pool.run((int)active.size(), [&](int i) {
                PairWork* pw = active[i].get();
                if (g == 0)
                    for (auto& j : pw->td) j.advance();
                for (auto& j : pw->bu) j.advance(n_groups == 1 ? -1 : g);
                // stage the pair's requests for the batch (finished pairs: leftovers dropped)
                pw->stage_w.clear();
                pw->stage_o.clear();
                if (!pw->finished()) {
                    for (Entry* en : pw->cache.pending) {
                        const uint64_t k = en->key;
                        const int64_t t0 = key_t0(k), w = key_w(k);
                        if (t0 < 0 || t0 + w > n || w <= P.k) {  // never hand the kernels an out-of-range window
                            pw->stage_bad = true;
                            pw->bad_t0 = t0;
                            pw->bad_t1 = t0 + w;
                        }
                        pw->stage_w.push_back(KsgWin{t0, (int32_t)w, -1, -1});
                        pw->stage_o.push_back(en);
                    }
                }
                pw->cache.pending.clear();
            });
            adv_ms += std::chrono::duration<double, std::milli>(clk::now() - t_adv).count();
            // retire finished pairs (none of their entries may be in flight): the per-pair work (result merge,
            // distinct-window count over the pair's cache, freeing the cache) runs on the host pool; the
            // bookkeeping that orders results and feeds Alg. 3 stays sequential in admission order
            const auto t_ret = clk::now();
            std::vector<int32_t> fin;
            for (size_t i = 0; i < active.size(); ++i)
                if (active[i]->finished() && active[i]->inflight == 0) fin.push_back((int32_t)i);
            // searches (kind 0) retire on the reaper thread, off the round's critical path; Alg. 3 trial runs
            // (kind 1) retire here, their costs decide the method of the pair's next unit
            std::vector<int32_t> sync_fin;
            for (int32_t i : fin) {
                if (active[i]->kind == 0)
                    reaper.push(std::move(active[i]));
                else
                    sync_fin.push_back(i);
            }
            std::vector<Retired> rt(sync_fin.size());
            pool.run((int)sync_fin.size(), [&](int f) { retire_pair(*active[sync_fin[f]], rt[f], P, chunk_sel); });
            for (size_t f = 0; f < sync_fin.size(); ++f) {
                PairWork* pw = active[sync_fin[f]].get();
                Retired& R = rt[f];
                distinct_w += R.dw;
                distinct_pp += R.dpp;
                total.add(R.ps);
                AutoState& A = autos[pw->auto_id];
                A.nL_td += R.nL_td;
                A.nS_bu += R.nS_bu;
                (pw->method == 1 ? A.cost_td : A.cost_bu) += R.ps.eval_cost;
                if (--A.left == 0) {
                    // Alg. 3 lines 6-15, Eqs. 6-9 (fixed fp64 op order, as the oracle)
                    const double alpha = P.auto_alpha > 0.0 ? P.auto_alpha : 0.5;
                    const double tbar_td = (double)A.cost_td / (double)am;
                    const double tbar_bu = (double)A.cost_bu / (double)am;
                    const double tt_td = tbar_td / (tbar_bu + tbar_td);
                    const double tt_bu = tbar_bu / (tbar_bu + tbar_td);
                    double nl = 0.5, ns = 0.5;
                    if (A.nS_bu + A.nL_td > 0) {
                        nl = (double)A.nL_td / (double)(A.nS_bu + A.nL_td);
                        ns = (double)A.nS_bu / (double)(A.nS_bu + A.nL_td);
                    }
                    const double beta = 1.0 - alpha;
                    A.nscore_td = alpha * (1.0 / tt_td) + beta * nl;
                    A.nscore_bu = alpha * (1.0 / tt_bu) + beta * ns;
                    A.chosen = A.nscore_td > A.nscore_bu ? 1 : 2;
                    queue.push_front(Unit{A.pair_idx, A.chosen, 0, -1, plan});
                }
            }
            if (!fin.empty()) {
                std::vector<std::unique_ptr<PairWork>> dead;
                size_t keep = 0, fi = 0;
                for (size_t i = 0; i < active.size(); ++i) {
                    if (fi < fin.size() && (int32_t)i == fin[fi]) {
                        if (active[i]) dead.push_back(std::move(active[i]));
                        ++fi;
                    } else {
                        active[keep++] = std::move(active[i]);
                    }
                }
                active.resize(keep);
                pool.run((int)dead.size(), [&](int i) { dead[i].reset(); });  // free the caches in parallel
                progress = true;
            }
            const auto t_asm = clk::now();
            ret_ms += std::chrono::duration<double, std::milli>(t_asm - t_ret).count();
            // one batch of every pending window of every active pair (finished pairs: leftovers dropped)
            std::vector<PairPtrs> table;
            batch_n = 0;
            Flight& F = fl[g];
            int64_t tot = 0;
            for (auto& pw : active) {
                if (pw->stage_bad)
                    return make_err(ISYCOS_E_RANGE, "internal: search requested window [" +
                                                        std::to_string(pw->bad_t0) + ", " + std::to_string(pw->bad_t1) +
                                                        ")");
                if (pw->stage_w.empty()) continue;
                pw->slot = (int32_t)table.size();
                table.push_back(pw->ptrs);
                F.offs.push_back(tot);
                tot += (int64_t)pw->stage_w.size();
                pw->inflight += 1;
                F.pws.push_back(pw.get());
            }
            // each pair copies its staged requests to its slice of the batch (in parallel when large)
            auto& batch = batches[g];
            if (batch_caps[g] < tot) {
                batch_caps[g] = std::max<int64_t>(tot, batch_caps[g] * 2);
                batch.reset(new KsgWin[batch_caps[g]]);
            }
            batch_n = tot;
            if ((int64_t)F.owners.size() < tot) F.owners.resize(std::max<int64_t>(tot, 2 * (int64_t)F.owners.size()));
            F.n = tot;
            pool.run(tot >= 512 ? (int)F.pws.size() : 1, [&](int p) {
                const int p0 = tot >= 512 ? p : 0, p1 = tot >= 512 ? p + 1 : (int)F.pws.size();
                for (int q = p0; q < p1; ++q) {
                    PairWork* pw = F.pws[q];
                    int64_t o = F.offs[q];
                    for (size_t i = 0; i < pw->stage_w.size(); ++i, ++o) {
                        batch[o] = pw->stage_w[i];
                        batch[o].pair = pw->slot;
                        F.owners[o] = pw->stage_o[i];
                    }
                    pw->stage_w.clear();
                    pw->stage_o.clear();
                }
            });
            if (batch_n == 0) {
                F.offs.clear();
                continue;
            }
            F.offs.push_back(batch_n);
            const auto t_ev = clk::now();
            asm_ms += std::chrono::duration<double, std::milli>(t_ev - t_asm).count();
            // kernel timing samples every profile_every-th round (event records are host time per round)
            uint32_t fl_round = P.flags;
            if ((fl_round & ISYCOS_F_PROFILE) && P.profile_every > 1 && (round_no % P.profile_every) != 0)
                fl_round &= ~ISYCOS_F_PROFILE;
            if (submitter) {
                Submitter::Job j;
                j.g = g;
                j.table = std::move(table);
                j.wins = batch.get();
                j.n = batch_n;
                j.k = P.k;
                j.variant = P.variant;
                j.st = sts[g];
                j.flags = fl_round;
                submitter->post(std::move(j));
            } else {
                Status s = eng->submit(g, table.data(), (int32_t)table.size(), batch.get(), batch_n, P.k,
                                       P.variant, DebugOut{}, sts[g], fl_round, &bs);
                if (!s.ok()) return s;
            }
            const double ev_ms = std::chrono::duration<double, std::milli>(clk::now() - t_ev).count();
            eval_ms += ev_ms;
            F.busy = true;
            progress = true;
            if (trace) {  // per-round trace (ISYCOS_TRACE=<path>): round, host ms since last submit, submit ms, batch
                int64_t sw2 = 0, wmax = 0;
                for (int64_t bi = 0; bi < batch_n; ++bi) {
                    const KsgWin& kw = batch[bi];
                    sw2 += (int64_t)kw.w * kw.w;
                    wmax = std::max<int64_t>(wmax, kw.w);
                }
                const double host = std::chrono::duration<double, std::milli>(t_ev - t_last).count();
                const double adv_r = std::chrono::duration<double, std::milli>(t_ret - t_adv).count();
                const double asm_r = std::chrono::duration<double, std::milli>(t_ev - t_asm).count();
                std::fprintf(trace, "%lld %.4f %.4f %lld %lld %lld %.4f %.4f\n", (long long)round_no, host, ev_ms,
                             (long long)batch_n, (long long)sw2, (long long)wmax, adv_r, asm_r);
            }
            ++round_no;
            t_last = clk::now();
        }
        if (active.empty() && queue.empty() && !fl[0].busy && !fl[1].busy) break;
        if (!progress) return make_err(ISYCOS_E_CUDA, "search driver stalled (internal error)");
    }
    if (n_groups == 2) {
        Status s = eng->join_second_stream(st);
        if (!s.ok()) return s;
    }
    for (Retired& R : reaper.finish()) {  // retire order (deterministic: it follows the rounds)
        all.insert(all.end(), R.res.begin(), R.res.end());
        distinct_w += R.dw;
        distinct_pp += R.dpp;
        total.add(R.ps);
    }
    std::stable_sort(all.begin(), all.end(), [](const isycos_result_window& a, const isycos_result_window& b) {
        if (a.pair != b.pair) return a.pair < b.pair;
        if (a.method != b.method) return a.method < b.method;
        return a.t0 < b.t0;
    });
    *out = std::move(all);
    if (stats) {
        stats->td_windows = total.td_windows;
        stats->td_noise_checks = total.td_noise_checks;
        stats->td_skips = total.td_skips;
        stats->td_accepted = total.td_accepted;
        stats->bu_climbs = total.bu_climbs;
        stats->bu_iterations = total.bu_iterations;
        stats->bu_neighbors = total.bu_neighbors;
        stats->bu_noise_checks = total.bu_noise_checks;
        stats->bu_prunes = total.bu_prunes;
        stats->bu_accepted = total.bu_accepted;
        stats->distinct_windows = distinct_w;
        stats->distinct_pairs = distinct_pp;
        stats->eval_cost = total.eval_cost;
        stats->auto_td = stats->auto_bu = 0;
        stats->auto_nscore_td = stats->auto_nscore_bu = 0.0;
        for (const AutoState& A : autos) {  // pair order (the oracle's summation order)
            (A.chosen == 1 ? stats->auto_td : stats->auto_bu) += 1;
            stats->auto_nscore_td += A.nscore_td;
            stats->auto_nscore_bu += A.nscore_bu;
        }
        const double wall = std::chrono::duration<double, std::milli>(clk::now() - t_start).count();
        if (submitter) bs.h2d_bytes += submitter->bs.h2d_bytes;  // every posted submit has run (all delivered)
        bs.wall_ms = wall;
        bs.host_ms = wall - eval_ms;
        bs.add_to(&stats->kernel);
        if (trace)
            std::fprintf(trace, "# host: advance %.3f ms (%d threads), other %.3f ms (deliver %.3f, retire %.3f, "
                         "assemble %.3f), eval %.3f ms (collect wait %.3f), rounds %lld\n", adv_ms, pool.size(),
                         wall - eval_ms - adv_ms, dlv_ms, ret_ms, asm_ms, eval_ms, wait_ms, (long long)round_no);
        if (trace)
            std::fprintf(trace, "# engine submit (cumulative): binning %.3f ms, block plan %.3f ms, other prep %.3f ms, "
                         "packing %.3f ms, launches %.3f ms\n", eng->sub_ms[0], eng->sub_ms[1], eng->sub_ms[2],
                         eng->sub_ms[3], eng->sub_ms[4]);
    }
    return Status{};
}

}  // namespace isy
