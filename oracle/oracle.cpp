// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, single-threaded C++17 CPU implementation of what the iSYCOS
// hot path computes (arXiv 2204.09131, /root/reference/PAPER.md = "P:<line>").
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load it.  It shares NO code with the CUDA path
// (paper_2204_09131_b200/csrc): no headers, no tables, no helpers.  Every
// formula below is written out from the paper and the readings recorded in
// DESIGN.md §"Readings".
//
// Build: g++ -O2 -std=c++17 -ffp-contract=off -fno-fast-math -shared -fPIC
//   (no FMA contraction: float differences and fp64 op sequences must be the
//   plain IEEE round-to-nearest results the definitions name).
//
// Contents
//   psi table / canonical LN / q32       §8(c).3 canonical numerics
//   window estimator KSG-1 (default)     Kraskov alg. 1 (north star)
//   window estimator KSG-2 (flag)        Eq. 2 literal
//   entropy + normalized MI              Eq. 12-13, KL reading
//   SYCOS_TD                             Alg. 1 (§5.1.2)
//   SYCOS_BU                             Alg. 2 (Defs 5.2-5.3)
//   noise predicate + pruning            Def 6.2, §6.2, §6.3
//   chunks + merge                       Alg. 4 line 14
//   iSYCOS selection (method 4, AUTO)    Alg. 3, Eqs. 4-9; readings R24-R26
//
// Parity status: every function is pinned by tests/test_oracle_*.py except the
// search readings the paper leaves open (RNG, delta, h, p, T_maxIdle, tie
// rules): "parity unpinned" against the paper's own implementation for those
// (DESIGN.md §"Parity status").

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <set>
#include <thread>
#include <utility>
#include <vector>

namespace {

// ------------------------------------------------------------------------------------
// §8(c).3 canonical numerics
// ------------------------------------------------------------------------------------

// digamma on positive integers: psi(1) = -gamma; psi(m+1) = psi(m) + 1/m  (recurrence).
std::vector<double> g_psi;

void ensure_psi(int64_t m_max) {
    if ((int64_t)g_psi.size() > m_max) return;
    int64_t old = (int64_t)g_psi.size();
    g_psi.resize(m_max + 1);
    if (old < 2) {
        g_psi[0] = NAN;                       // psi(0) is a pole
        g_psi[1] = -0.57721566490153286061;   // -Euler-Mascheroni
        old = 2;
    }
    for (int64_t m = old - 1; m < m_max; ++m) {
        double inv = 1.0 / (double)m;
        g_psi[m + 1] = g_psi[m] + inv;
    }
}

double psi(int64_t m) { ensure_psi(m); return g_psi[m]; }

// q(v) = round-half-even(v * 2^32) as int64.
int64_t q32(double v) { return (int64_t)std::llrint(std::ldexp(v, 32)); }

// canonical natural log: frexp, reduce to [sqrt(1/2), sqrt(2)), 2*atanh series to s^19.
double canon_ln(double v) {
    int e = 0;
    double m = std::frexp(v, &e);           // v = m * 2^e, m in [0.5, 1)
    if (m < 0.70710678118654752440) { m = m * 2.0; e = e - 1; }
    double s = (m - 1.0) / (m + 1.0);
    double z = s * s;
    double c[10];
    for (int j = 1; j <= 9; ++j) c[j] = 1.0 / (double)(2 * j + 1);
    double p = c[9];
    for (int j = 8; j >= 1; --j) { p = p * z; p = p + c[j]; }
    double two_s = 2.0 * s;
    double tail = two_s * z;
    tail = tail * p;
    double r = two_s + tail;
    double el = (double)e * 0.69314718055994530942;
    return el + r;
}

const double kTwoPowMinus32 = 2.3283064365386962890625e-10;  // 2^-32 exactly

// ------------------------------------------------------------------------------------
// Window estimators (Defs 4.1-4.2: MI of the empirical window distribution)
// ------------------------------------------------------------------------------------

struct WinResult {
    double mi = 0, h = 0, nmi = 0;       // canonical
    double mi_plain = 0, h_plain = 0;    // plain fp64 sums (self-check of the canonical form)
    int64_t s_psi = 0, s_log = 0;
    int32_t zero_eps = 0;
};

// Chebyshev (max-norm, footnote P:671) distance with float32 differences.
inline float dist(float xi, float yi, float xj, float yj) {
    float dx = std::fabs(xi - xj);
    float dy = std::fabs(yi - yj);
    return dx > dy ? dx : dy;
}

// eps_i = k-th smallest of the multiset {d_ij : j in W, j != i}.
// eps_method 0: nth_element;  1: full sort (two independent ways).
float kth_distance(const float* x, const float* y, int64_t w, int64_t i, int k, int eps_method,
                   std::vector<float>& buf) {
    buf.clear();
    for (int64_t j = 0; j < w; ++j)
        if (j != i) buf.push_back(dist(x[i], y[i], x[j], y[j]));
    if (eps_method == 1) {
        std::sort(buf.begin(), buf.end());
    } else {
        std::nth_element(buf.begin(), buf.begin() + (k - 1), buf.end());
    }
    return buf[k - 1];
}

// Normalized MI, Eq. 12 with the degenerate rule of SURVEY §8(c).1.
double normalized(double mi, double h, int32_t zero_eps) {
    if (zero_eps > 0 || !(h > 1e-6)) return mi > 1e-6 ? 1.0 : 0.0;
    double r = mi / h;
    if (r < 0.0) return 0.0;
    if (r > 1.0) return 1.0;
    return r;
}

// Point i of a window: eps_i (KSG-1 radius, both variants) and the variant's marginal counts.
void point_eval(const float* x, const float* y, int64_t w, int64_t i, int k, int variant, int eps_method,
                std::vector<float>& buf, std::vector<std::pair<float, int64_t>>& dj, float* eps_o,
                int64_t* nx_o, int64_t* ny_o) {
    float eps = kth_distance(x, y, w, i, k, eps_method, buf);
    int64_t nx = 0, ny = 0;
    if (variant == 0) {
        // KSG-1: n_x(i) = #{j != i : |x_i - x_j| < eps_i}  (strict; north star)
        for (int64_t j = 0; j < w; ++j) {
            if (j == i) continue;
            if (std::fabs(x[i] - x[j]) < eps) ++nx;
            if (std::fabs(y[i] - y[j]) < eps) ++ny;
        }
    } else {
        // KSG-2 (Eq. 2): the k nearest in ascending (d_ij, j) order; per-dimension
        // d_x, d_y = max over them; n_x = #{j != i : |x_i - x_j| <= d_x}.
        dj.clear();
        for (int64_t j = 0; j < w; ++j)
            if (j != i) dj.push_back({dist(x[i], y[i], x[j], y[j]), j});
        std::sort(dj.begin(), dj.end());
        float dxk = 0.0f, dyk = 0.0f;
        for (int m = 0; m < k; ++m) {
            int64_t j = dj[m].second;
            float ax = std::fabs(x[i] - x[j]);
            float ay = std::fabs(y[i] - y[j]);
            if (ax > dxk) dxk = ax;
            if (ay > dyk) dyk = ay;
        }
        for (int64_t j = 0; j < w; ++j) {
            if (j == i) continue;
            if (std::fabs(x[i] - x[j]) <= dxk) ++nx;
            if (std::fabs(y[i] - y[j]) <= dyk) ++ny;
        }
    }
    *eps_o = eps;
    *nx_o = nx;
    *ny_o = ny;
}

// Optional worker threads for the per-point loop of large windows (env ORACLE_THREADS, default 1; used
// only to precompute the full-size golden files).  The points are independent and every sum below runs
// sequentially in point order, so the results do not depend on the thread count.
int oracle_threads() {
    static int t = [] {
        const char* e = std::getenv("ORACLE_THREADS");
        int v = e ? std::atoi(e) : 1;
        return v < 1 ? 1 : v;
    }();
    return t;
}

// KSG-1 (north star) or KSG-2 (Eq. 2 literal) MI of one window of w points, plus the
// Kozachenko-Leonenko joint entropy H from the same eps_i (Eq. 13 reading).
int window_estimate(const float* x, const float* y, int64_t w, int k, int variant, int eps_method,
                    WinResult* out, float* eps_out, int32_t* nx_out, int32_t* ny_out) {
    if (w <= k || k < 1) return -3;
    ensure_psi(w + 1);
    std::vector<float> E(w);
    std::vector<int64_t> NX(w), NY(w);
    auto run = [&](int64_t i0, int64_t i1) {
        std::vector<float> buf;
        buf.reserve(w);
        std::vector<std::pair<float, int64_t>> dj;
        for (int64_t i = i0; i < i1; ++i) point_eval(x, y, w, i, k, variant, eps_method, buf, dj, &E[i], &NX[i], &NY[i]);
    };
    const int T = w >= 2048 ? oracle_threads() : 1;
    if (T > 1) {
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t) th.emplace_back(run, w * t / T, w * (t + 1) / T);
        for (auto& h : th) h.join();
    } else {
        run(0, w);
    }
    int64_t s_psi = 0, s_log = 0;
    int32_t zeros = 0;
    double plain_psi = 0.0, plain_log = 0.0;
    for (int64_t i = 0; i < w; ++i) {
        const float eps = E[i];
        const int64_t nx = NX[i], ny = NY[i];
        if (variant == 0) {
            int64_t a = nx + 1, b = ny + 1;
            s_psi += q32(psi(a)) + q32(psi(b));
            plain_psi += psi(a) + psi(b);
        } else {
            s_psi += q32(psi(nx)) + q32(psi(ny));
            plain_psi += psi(nx) + psi(ny);
        }
        if (eps > 0.0f) {
            double v = 2.0 * (double)eps;
            s_log += q32(canon_ln(v));
            plain_log += std::log(v);
        } else {
            ++zeros;
        }
        if (eps_out) eps_out[i] = eps;
        if (nx_out) nx_out[i] = (int32_t)nx;
        if (ny_out) ny_out[i] = (int32_t)ny;
    }
    double dw = (double)w;
    double mean_q = ((double)s_psi * kTwoPowMinus32) / dw;
    double mi;
    if (variant == 0) {
        double a = psi(k) + psi(w);
        mi = a - mean_q;                                  // psi(k)+psi(w)-<psi(nx+1)+psi(ny+1)>
    } else {
        double a = psi(k) - 1.0 / (double)k;
        a = a + psi(w);
        mi = a - mean_q;                                  // psi(k)-1/k+psi(n)-<psi(nx)+psi(ny)>
    }
    double h;
    if (zeros > 0) {
        h = -INFINITY;                                    // ln(0) term in the KL sum
    } else {
        double a = psi(w) - psi(k);
        double m = ((double)s_log * kTwoPowMinus32) / dw;
        h = a + 2.0 * m;                                  // psi(w)-psi(k)+(2/w) sum ln(2 eps_i)
    }
    out->mi = mi;
    out->h = h;
    out->nmi = normalized(mi, h, zeros);
    out->s_psi = s_psi;
    out->s_log = s_log;
    out->zero_eps = zeros;
    out->mi_plain = (variant == 0 ? psi(k) + psi(w) : psi(k) - 1.0 / k + psi(w)) - plain_psi / dw;
    out->h_plain = zeros > 0 ? -INFINITY : psi(w) - psi(k) + 2.0 * plain_log / dw;
    return 0;
}

// ------------------------------------------------------------------------------------
// Search (Alg. 1, Alg. 2, §6, Alg. 4), generic over an MI provider
// ------------------------------------------------------------------------------------

struct Eval { double mi, h, nmi; };
using Provider = std::function<int(int64_t t0, int64_t t1, Eval* out)>;

}  // namespace

extern "C" {

struct OParams {
    int32_t k, variant, method, noise;     // method: 1 TD, 2 BU, 3 BOTH, 4 AUTO (iSYCOS, Alg. 3)
    int32_t p, h, t_max_idle, n_chunks;
    int64_t s_min, s_max, delta_td, delta_bu;   // 0 => defaults s/4, s_min/3
    double sigma, tau_ratio;
    uint64_t seed;
    const int64_t* sizes;                  // explicit TD layer sizes or NULL (halving)
    int32_t n_sizes, _pad;
    int32_t auto_M, auto_m;                // Alg. 3: M partitions, m sampled (0 => 20, 6)
    double auto_alpha, auto_rho;           // Eqs. 4-9 weight alpha, small/large cut rho (0 => 0.5, 0.5)
    int32_t chunk_begin, chunk_end;        // 0,0: every chunk, merged; else chunks [begin,end) only, unmerged
};

struct OResult {
    int32_t pair, method;
    int64_t t0, t1;
    double mi, h, nmi;
};

struct OStats {
    int64_t td_windows, td_noise_checks, td_skips, td_accepted;
    int64_t bu_climbs, bu_iterations, bu_neighbors, bu_noise_checks, bu_prunes, bu_accepted;
    int64_t distinct_windows, distinct_pairs;   // per pair, union over chunks/methods
    int64_t eval_cost;                     // sum over distinct windows of w * ceil(log2 w) (Alg. 3 runtime proxy)
    int64_t auto_td, auto_bu;              // AUTO: pairs for which Alg. 3 chose TD / BU
    double auto_nscore_td, auto_nscore_bu; // AUTO: sums over pairs of nscore_TD, nscore_BU (Eqs. 8-9)
};

}  // extern "C"

namespace {

// LAHC history index draw (Alg. 2 line 11 "random.get(L_h)"): tests may pass the draws in as inputs
// (called with the climb start lo and the iteration number; a value outside [0, h) aborts the search).
using Draw = std::function<int(int64_t lo, int64_t it)>;

struct Searcher {
    const OParams& P;
    Provider provider;
    int32_t pair_id;
    OStats* st;
    std::map<std::pair<int64_t, int64_t>, Eval> memo;   // distinct windows consumed
    int err = 0;
    Draw draw;                                           // null: the SplitMix64 stream (reading R14)

    Searcher(const OParams& p, Provider prov, int32_t id, OStats* s)
        : P(p), provider(std::move(prov)), pair_id(id), st(s) {}

    // Computing the MI of a window costs t_w ~ w log w; a run computes each distinct window once
    // (this memo); the sum over them is the deterministic runtime proxy of Alg. 3 (reading R24).
    static int64_t clog2(int64_t w) {
        int64_t L = 0;
        while ((int64_t(1) << L) < w) ++L;
        return L;
    }
    Eval I(int64_t t0, int64_t t1) {
        auto key = std::make_pair(t0, t1);
        auto it = memo.find(key);
        if (it != memo.end()) return it->second;
        Eval e{0, 0, 0};
        int rc = provider(t0, t1, &e);
        if (rc != 0 && err == 0) err = rc;
        memo[key] = e;
        st->distinct_windows += 1;
        st->eval_cost += (t1 - t0) * clog2(t1 - t0);
        st->distinct_pairs += (t1 - t0) * (t1 - t0 - 1);
        return e;
    }

    double tau() const { return P.tau_ratio * P.sigma; }

    std::vector<int64_t> schedule() const {
        std::vector<int64_t> s;
        if (P.sizes && P.n_sizes > 0) {
            for (int i = 0; i < P.n_sizes; ++i) s.push_back(P.sizes[i]);
            return s;
        }
        s.push_back(P.s_max);               // S:348 geometric halving s_max -> s_min
        while (s.back() > P.s_min) s.push_back(std::max(P.s_min, s.back() / 2));
        return s;
    }

    // SYCOS_TD (Alg. 1) on [lo,hi), with §6.2 noise pruning.
    void td(int64_t lo, int64_t hi, std::vector<OResult>& R) {
        std::vector<std::pair<int64_t, int64_t>> parts{{lo, hi}};
        for (int64_t s : schedule()) {
            std::vector<std::pair<int64_t, int64_t>> next;
            int64_t delta = P.delta_td > 0 ? P.delta_td : std::max<int64_t>(1, s / 4);
            for (auto [a, b] : parts) {
                if (b - a < s) { next.push_back({a, b}); continue; }
                int64_t t = a, pend = a;
                int streak = 0;
                bool shifted = false;
                while (t + s <= b) {                                        // Alg.1 l.5
                    st->td_windows += 1;
                    Eval e = I(t, t + s);                                   // l.6
                    if (e.nmi >= P.sigma) {                                 // l.7
                        R.push_back({pair_id, 1, t, t + s, e.mi, e.h, e.nmi});
                        st->td_accepted += 1;
                        if (t > pend) next.push_back({pend, t});            // P:243 truncate
                        t = t + s;                                          // l.9 next window
                        pend = t;
                        streak = 0;
                        shifted = false;
                        continue;
                    }
                    if (P.noise && shifted && delta > P.k && s - delta > P.k) {
                        // w1 = wo (.) wd; wd noise w.r.t. wo iff I~(wd) < tau ^ I(w1) < I(wo), I(wo) > 0
                        st->td_noise_checks += 1;
                        Eval wo = I(t, t + s - delta);
                        Eval wd = I(t + s - delta, t + s);
                        bool v = wd.nmi < tau() && e.mi < wo.mi && wo.mi > 0.0;
                        streak = v ? streak + 1 : 0;
                        if (streak >= P.p) {
                            st->td_skips += 1;
                            t = t + s;
                            streak = 0;
                            shifted = false;
                            continue;
                        }
                    }
                    t = t + delta;                                          // l.11 shiftWindow
                    shifted = true;
                }
                if (pend < b) next.push_back({pend, b});
            }
            parts.clear();
            for (auto& q : next)
                if (q.second - q.first >= P.s_min) parts.push_back(q);
        }
    }

    // LAHC random stream per climb, keyed by (seed, pair, lo)  (SURVEY §8(c).2 reading).
    struct Rng {
        uint64_t state;
        uint64_t next() {
            state += 0x9E3779B97F4A7C15ull;
            uint64_t z = state;
            z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
            z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
            return z ^ (z >> 31);
        }
    };

    // SYCOS_BU (Alg. 2) on [lo_c,hi), with §6.3 noise pruning.
    void bu(int64_t lo_c, int64_t hi, std::vector<OResult>& R) {
        const int64_t smin = P.s_min, smax = P.s_max;
        const int64_t d = P.delta_bu > 0 ? P.delta_bu : std::max<int64_t>(1, smin / 3);
        int64_t lo = lo_c;
        while (lo + smin <= hi) {                                           // l.1
            st->bu_climbs += 1;
            int64_t t0 = lo, t1 = lo + smin;                                // l.2
            double Iw = I(t0, t1).mi;                                       // l.3
            std::vector<double> L(P.h, Iw);                                 // l.4
            int idle = 0;                                                   // l.5
            int64_t it = 0;
            int streak[2] = {0, 0};
            bool pruned[2] = {false, false};                                // 0 LEFT, 1 RIGHT
            Rng rng{P.seed ^ ((uint64_t)(uint32_t)pair_id * 0x9E3779B97F4A7C15ull) ^
                    ((uint64_t)lo * 0xD1B54A32D192ED03ull)};
            while (idle <= P.t_max_idle) {                                  // l.6
                // l.7: N1 = the 8 delta-neighbours (Def 5.2-5.3), in (t0,t1) order
                int64_t bt0 = 0, bt1 = 0;
                double bI = 0.0;
                bool have = false;
                for (int da = -1; da <= 1; ++da) {
                    for (int db = -1; db <= 1; ++db) {
                        if (da == 0 && db == 0) continue;
                        if (da == -1 && pruned[0]) continue;
                        if (db == 1 && pruned[1]) continue;
                        int64_t c0 = t0 + da * d, c1 = t1 + db * d;
                        if (c0 < lo || c1 > hi) continue;
                        int64_t sz = c1 - c0;
                        if (sz < smin || sz > smax) continue;
                        st->bu_neighbors += 1;
                        double v = I(c0, c1).mi;                            // l.8
                        if (!have || v > bI) { have = true; bI = v; bt0 = c0; bt1 = c1; }  // l.10
                    }
                }
                if (!have) break;
                st->bu_iterations += 1;
                if (P.noise && d > P.k) {
                    for (int dir = 0; dir < 2; ++dir) {
                        if (pruned[dir]) continue;
                        int64_t e0, e1, m0, m1;
                        if (dir == 0) { e0 = t0 - d; e1 = t0; m0 = t0 - d; m1 = t1; }
                        else { e0 = t1; e1 = t1 + d; m0 = t0; m1 = t1 + d; }
                        if (e0 < lo || e1 > hi || m1 - m0 > smax) continue;
                        st->bu_noise_checks += 1;
                        Eval ext = I(e0, e1);
                        Eval mix = I(m0, m1);
                        bool v = ext.nmi < tau() && mix.mi < Iw && Iw > 0.0;
                        streak[dir] = v ? streak[dir] + 1 : 0;
                        if (streak[dir] >= P.p) { pruned[dir] = true; st->bu_prunes += 1; }
                    }
                }
                int r = (int)((rng.next() >> 32) % (uint64_t)P.h);          // l.11 random get
                if (draw) {
                    r = draw(lo, it);
                    if (r < 0 || r >= P.h) { if (err == 0) err = -1; return; }
                }
                it += 1;
                double Ih = L[r];
                if (bI > Ih || bI > Iw) {                                   // l.12 (strict, G4)
                    t0 = bt0; t1 = bt1; Iw = bI; idle = 0;                  // l.13-14
                } else {
                    idle += 1;                                              // l.17
                }
                if (Iw > Ih) L[r] = Iw;                                     // l.19-20
            }
            Eval fin = I(t0, t1);
            if (fin.nmi >= P.sigma) {                                       // l.23
                R.push_back({pair_id, 2, t0, t1, fin.mi, fin.h, fin.nmi});
                st->bu_accepted += 1;
                lo = std::max(t1, lo + smin);
            } else {
                lo = lo + smin;
            }
        }
    }
};

// Alg. 4 line 14, clipped (G10): chunk c = [max(0, cL - s_max), min(n, (c+1)L)).
std::vector<std::pair<int64_t, int64_t>> chunk_plan(int64_t n, int32_t n_p, int64_t s_max) {
    std::vector<std::pair<int64_t, int64_t>> c;
    int64_t L = (n + n_p - 1) / n_p;
    for (int32_t i = 0; i < n_p; ++i) {
        int64_t a = (int64_t)i * L;
        if (a >= n) break;
        c.push_back({std::max<int64_t>(0, a - s_max), std::min<int64_t>(n, a + L)});
    }
    return c;
}

// Merge: greedy by desc nmi, desc mi, asc (t0,t1); keep if disjoint; sort by t0.
std::vector<OResult> merge(std::vector<OResult> all) {
    std::sort(all.begin(), all.end(), [](const OResult& a, const OResult& b) {
        if (a.nmi != b.nmi) return a.nmi > b.nmi;
        if (a.mi != b.mi) return a.mi > b.mi;
        if (a.t0 != b.t0) return a.t0 < b.t0;
        return a.t1 < b.t1;
    });
    std::vector<OResult> kept;
    for (auto& r : all) {
        bool ok = true;
        for (auto& q : kept)
            if (r.t0 < q.t1 && q.t0 < r.t1) { ok = false; break; }
        if (ok) kept.push_back(r);
    }
    std::sort(kept.begin(), kept.end(), [](const OResult& a, const OResult& b) { return a.t0 < b.t0; });
    return kept;
}

int run_pair(const OParams& P, Provider prov, int32_t pair_id, int64_t n, OStats* st,
             std::vector<OResult>& out, Draw draw = nullptr);

void add_stats(OStats* a, const OStats& b) {
    a->td_windows += b.td_windows; a->td_noise_checks += b.td_noise_checks; a->td_skips += b.td_skips;
    a->td_accepted += b.td_accepted; a->bu_climbs += b.bu_climbs; a->bu_iterations += b.bu_iterations;
    a->bu_neighbors += b.bu_neighbors; a->bu_noise_checks += b.bu_noise_checks; a->bu_prunes += b.bu_prunes;
    a->bu_accepted += b.bu_accepted; a->distinct_windows += b.distinct_windows;
    a->distinct_pairs += b.distinct_pairs; a->eval_cost += b.eval_cost;
}

// Eqs. 6-9: average runtimes t_bar over the m trials, normalized t~ (Eq. 6), n~ (Eq. 7),
// nscore = alpha / t~ + (1 - alpha) n~ (Eqs. 8-9).  No windows at all: n~ = 0.5 each.
void auto_scores(int64_t cost_td, int64_t cost_bu, int32_t m, int64_t nL_td, int64_t nS_bu, double alpha,
                 double* nscore_td, double* nscore_bu) {
    const double tbar_td = (double)cost_td / (double)m;
    const double tbar_bu = (double)cost_bu / (double)m;
    const double tt_td = tbar_td / (tbar_bu + tbar_td);
    const double tt_bu = tbar_bu / (tbar_bu + tbar_td);
    double nl = 0.5, ns = 0.5;
    if (nS_bu + nL_td > 0) {
        nl = (double)nL_td / (double)(nS_bu + nL_td);
        ns = (double)nS_bu / (double)(nS_bu + nL_td);
    }
    const double beta = 1.0 - alpha;
    *nscore_td = alpha * (1.0 / tt_td) + beta * nl;
    *nscore_bu = alpha * (1.0 / tt_bu) + beta * ns;
}

// iSYCOS (Alg. 3; Eqs. 4-9), with the deterministic readings R24-R26:
//   random sampling (§5.3.1): M partitions of length floor(N/M); m of them drawn without replacement by a
//     partial Fisher-Yates shuffle on a SplitMix64 stream keyed by (seed, pair id);
//   runtime t_TD^i, t_BU^i := eval_cost of SYCOS_TD / SYCOS_BU run alone on partition i (a fresh window
//     memo per run), the sum of w*ceil(log2 w) over the run's MI requests (t_w ~ O(w log w));
//   countWindows: |w| <= rho * s_max is small, else large.
// The trial runs' counters are included in the pair's stats; their windows are not results.
int run_auto(const OParams& P, Provider prov, int32_t pair_id, int64_t n, OStats* st, std::vector<OResult>& out) {
    const int32_t M = P.auto_M > 0 ? P.auto_M : 20;
    const int32_t m = P.auto_m > 0 ? P.auto_m : 6;
    const double alpha = P.auto_alpha > 0.0 ? P.auto_alpha : 0.5;
    const double rho = P.auto_rho > 0.0 ? P.auto_rho : 0.5;
    const int64_t Lp = n / M;
    // line 1: randomSampling(M)
    std::vector<int32_t> idx(M);
    for (int32_t i = 0; i < M; ++i) idx[i] = i;
    Searcher::Rng rng{P.seed ^ ((uint64_t)(uint32_t)pair_id * 0x9E3779B97F4A7C15ull) ^ 0xA0761D6478BD642Full};
    for (int32_t i = 0; i < m; ++i) {
        const int32_t j = i + (int32_t)((rng.next() >> 32) % (uint64_t)(M - i));
        std::swap(idx[i], idx[j]);
    }
    // lines 2-5: SYCOS_TD and SYCOS_BU on each sampled partition
    int64_t cost_td = 0, cost_bu = 0, nL_td = 0, nS_bu = 0;
    for (int32_t i = 0; i < m; ++i) {
        const int64_t lo = (int64_t)idx[i] * Lp, hi = lo + Lp;
        for (int meth = 1; meth <= 2; ++meth) {
            OStats ts{};
            Searcher S(P, prov, pair_id, &ts);
            std::vector<OResult> R;
            if (meth == 1) S.td(lo, hi, R); else S.bu(lo, hi, R);
            if (S.err) return S.err;
            add_stats(st, ts);
            for (auto& r : R) {
                const bool small = (double)(r.t1 - r.t0) <= rho * (double)P.s_max;
                if (meth == 1 && !small) nL_td += 1;
                if (meth == 2 && small) nS_bu += 1;
            }
            (meth == 1 ? cost_td : cost_bu) += ts.eval_cost;
        }
    }
    // lines 6-10: Eqs. 6-9
    double nscore_td, nscore_bu;
    auto_scores(cost_td, cost_bu, m, nL_td, nS_bu, alpha, &nscore_td, &nscore_bu);
    st->auto_nscore_td += nscore_td;
    st->auto_nscore_bu += nscore_bu;
    // lines 11-15: strict ">" selects TD; ties select BU
    OParams Q = P;
    Q.method = nscore_td > nscore_bu ? 1 : 2;
    (Q.method == 1 ? st->auto_td : st->auto_bu) += 1;
    return run_pair(Q, prov, pair_id, n, st, out);
}

int run_pair(const OParams& P, Provider prov, int32_t pair_id, int64_t n, OStats* st,
             std::vector<OResult>& out, Draw draw) {
    if (P.method == 4) return run_auto(P, prov, pair_id, n, st, out);
    Searcher S(P, std::move(prov), pair_id, st);
    S.draw = std::move(draw);
    auto chunks = chunk_plan(n, P.n_chunks < 1 ? 1 : P.n_chunks, P.s_max);
    const bool sel = P.chunk_end > P.chunk_begin;   // one shard's (pair, chunk) units: merged by the caller
    if (sel) {
        if (P.chunk_begin < 0 || P.chunk_end > (int32_t)chunks.size()) return -1;
        chunks = std::vector<std::pair<int64_t, int64_t>>(chunks.begin() + P.chunk_begin, chunks.begin() + P.chunk_end);
    }
    for (int m = 1; m <= 2; ++m) {
        if (!(P.method & m)) continue;
        std::vector<OResult> all;
        for (auto [lo, hi] : chunks) {
            std::vector<OResult> R;
            if (m == 1) S.td(lo, hi, R); else S.bu(lo, hi, R);
            if (S.err) return S.err;
            all.insert(all.end(), R.begin(), R.end());
        }
        if (sel) {
            out.insert(out.end(), all.begin(), all.end());
            continue;
        }
        auto merged = merge(all);
        out.insert(out.end(), merged.begin(), merged.end());
    }
    return S.err;
}

bool params_ok(const OParams& P, int64_t n) {
    if (P.k < 1 || P.k > 16) return false;
    if (P.s_min < 2 || P.s_min > P.s_max || P.s_max > n) return false;
    if (P.k >= P.s_min) return false;
    if (!(P.sigma > 0.0 && P.sigma <= 1.0)) return false;
    if (!(P.tau_ratio >= 0.0 && P.tau_ratio < 1.0)) return false;
    if (P.h < 1 || P.p < 1 || P.t_max_idle < 0) return false;
    if (P.method < 1 || P.method > 4) return false;
    if (P.method == 4) {
        const int32_t M = P.auto_M > 0 ? P.auto_M : 20, m = P.auto_m > 0 ? P.auto_m : 6;
        if (m > M || n / M < P.s_min) return false;
        if (P.auto_alpha < 0.0 || P.auto_alpha > 1.0 || P.auto_rho < 0.0 || P.auto_rho > 1.0) return false;
    }
    return true;
}

}  // namespace

extern "C" {

int oracle_abi_version(void) { return 1; }

int oracle_psi(int64_t m_max, double* out) {
    if (m_max < 1 || !out) return -1;
    ensure_psi(m_max);
    for (int64_t m = 0; m <= m_max; ++m) out[m] = g_psi[m];
    return 0;
}

double oracle_ln(double v) { return canon_ln(v); }
int64_t oracle_q32(double v) { return q32(v); }

// One window of w points (x, y already sliced).  out6 = {mi, h, nmi, mi_plain, h_plain};
// out3 = {s_psi, s_log, zero_eps}.  eps/nx/ny optional per-point outputs.
int oracle_window(const float* x, const float* y, int64_t w, int32_t k, int32_t variant,
                  int32_t eps_method, double* out6, int64_t* out3, float* eps, int32_t* nx,
                  int32_t* ny) {
    WinResult r;
    int rc = window_estimate(x, y, w, k, variant, eps_method, &r, eps, nx, ny);
    if (rc) return rc;
    if (out6) { out6[0] = r.mi; out6[1] = r.h; out6[2] = r.nmi; out6[3] = r.mi_plain; out6[4] = r.h_plain; }
    if (out3) { out3[0] = r.s_psi; out3[1] = r.s_log; out3[2] = r.zero_eps; }
    return 0;
}

// Batch of windows [t0,t1) over series (x, y) of length n.  windows = 2*nw int64.
int oracle_mi_batch(const float* x, const float* y, int64_t n, const int64_t* windows, int64_t nw,
                    int32_t k, int32_t variant, double* mi, double* h, double* nmi, int64_t* s_psi,
                    int64_t* s_log, int32_t* zero_eps) {
    for (int64_t q = 0; q < nw; ++q) {
        int64_t t0 = windows[2 * q], t1 = windows[2 * q + 1];
        if (t0 < 0 || t1 > n || t0 >= t1) return -2;
        WinResult r;
        int rc = window_estimate(x + t0, y + t0, t1 - t0, k, variant, 0, &r, nullptr, nullptr, nullptr);
        if (rc) return rc;
        if (mi) mi[q] = r.mi;
        if (h) h[q] = r.h;
        if (nmi) nmi[q] = r.nmi;
        if (s_psi) s_psi[q] = r.s_psi;
        if (s_log) s_log[q] = r.s_log;
        if (zero_eps) zero_eps[q] = r.zero_eps;
    }
    return 0;
}

// Full search over pairs (pairs = 3*n_pairs int32: xs, ys, id).  Results sorted by (pair, method, t0).
int oracle_search(const float* const* series, int32_t n_series, int64_t n, const int32_t* pairs,
                  int32_t n_pairs, const OParams* P, OResult* out, int64_t cap, int64_t* count,
                  OStats* stats) {
    if (!series || !pairs || !P || !count || !params_ok(*P, n)) return -1;
    OStats local{};
    OStats* st = stats ? stats : &local;
    std::memset(st, 0, sizeof(OStats));
    std::vector<OResult> all;
    for (int32_t q = 0; q < n_pairs; ++q) {
        int32_t xs = pairs[3 * q], ys = pairs[3 * q + 1], id = pairs[3 * q + 2];
        if (xs < 0 || ys < 0 || xs >= n_series || ys >= n_series) return -1;
        const float* x = series[xs];
        const float* y = series[ys];
        Provider prov = [&](int64_t t0, int64_t t1, Eval* e) {
            WinResult r;
            int rc = window_estimate(x + t0, y + t0, t1 - t0, P->k, P->variant, 0, &r, nullptr,
                                     nullptr, nullptr);
            e->mi = r.mi; e->h = r.h; e->nmi = r.nmi;
            return rc;
        };
        std::vector<OResult> res;
        int rc = run_pair(*P, prov, id, n, st, res);
        if (rc) return rc;
        all.insert(all.end(), res.begin(), res.end());
    }
    std::stable_sort(all.begin(), all.end(), [](const OResult& a, const OResult& b) {
        if (a.pair != b.pair) return a.pair < b.pair;
        if (a.method != b.method) return a.method < b.method;
        return a.t0 < b.t0;
    });
    *count = (int64_t)all.size();
    int64_t m = std::min<int64_t>(cap, (int64_t)all.size());
    for (int64_t i = 0; i < m; ++i) out[i] = all[i];
    return (int64_t)all.size() > cap ? -4 : 0;
}

// Same search for one pair of length n, with a table-driven MI provider callback (tests).
typedef int (*oracle_mi_fn)(void* ctx, int64_t t0, int64_t t1, double* mi, double* h, double* nmi);

int oracle_search_mock(oracle_mi_fn fn, void* ctx, int64_t n, const OParams* P, OResult* out,
                       int64_t cap, int64_t* count, OStats* stats) {
    if (!fn || !P || !count) return -1;
    OStats local{};
    OStats* st = stats ? stats : &local;
    std::memset(st, 0, sizeof(OStats));
    Provider prov = [&](int64_t t0, int64_t t1, Eval* e) { return fn(ctx, t0, t1, &e->mi, &e->h, &e->nmi); };
    std::vector<OResult> res;
    int rc = run_pair(*P, prov, 0, n, st, res);
    *count = (int64_t)res.size();
    int64_t m = std::min<int64_t>(cap, (int64_t)res.size());
    for (int64_t i = 0; i < m; ++i) out[i] = res[i];
    if (rc) return rc;
    return (int64_t)res.size() > cap ? -4 : 0;
}

// The mock search with the LAHC history draws passed in as inputs (tests: hand-traced Alg. 2 runs).
typedef int (*oracle_draw_fn)(void* ctx, int64_t lo, int64_t it);

int oracle_search_mock_draws(oracle_mi_fn fn, oracle_draw_fn dfn, void* ctx, int64_t n, const OParams* P,
                             OResult* out, int64_t cap, int64_t* count, OStats* stats) {
    if (!fn || !dfn || !P || !count) return -1;
    OStats local{};
    OStats* st = stats ? stats : &local;
    std::memset(st, 0, sizeof(OStats));
    Provider prov = [&](int64_t t0, int64_t t1, Eval* e) { return fn(ctx, t0, t1, &e->mi, &e->h, &e->nmi); };
    Draw draw = [&](int64_t lo, int64_t it) { return dfn(ctx, lo, it); };
    std::vector<OResult> res;
    int rc = run_pair(*P, prov, 0, n, st, res, draw);
    *count = (int64_t)res.size();
    int64_t m = std::min<int64_t>(cap, (int64_t)res.size());
    for (int64_t i = 0; i < m; ++i) out[i] = res[i];
    if (rc) return rc;
    return (int64_t)res.size() > cap ? -4 : 0;
}

// One point i of a window (sampled checks at sizes where the full window is too slow):
// out_eps = eps_i (KSG-1 radius), out_n = {n_x, n_y} of the chosen variant.
int oracle_point(const float* x, const float* y, int64_t w, int64_t i, int32_t k, int32_t variant,
                 float* out_eps, int32_t* out_n) {
    if (w <= k || k < 1 || i < 0 || i >= w) return -3;
    std::vector<float> buf;
    float eps = kth_distance(x, y, w, i, k, 0, buf);
    int64_t nx = 0, ny = 0;
    if (variant == 0) {
        for (int64_t j = 0; j < w; ++j) {
            if (j == i) continue;
            if (std::fabs(x[i] - x[j]) < eps) ++nx;
            if (std::fabs(y[i] - y[j]) < eps) ++ny;
        }
    } else {
        std::vector<std::pair<float, int64_t>> dj;
        for (int64_t j = 0; j < w; ++j)
            if (j != i) dj.push_back({dist(x[i], y[i], x[j], y[j]), j});
        std::sort(dj.begin(), dj.end());
        float dxk = 0.0f, dyk = 0.0f;
        for (int m = 0; m < k; ++m) {
            int64_t j = dj[m].second;
            dxk = std::max(dxk, std::fabs(x[i] - x[j]));
            dyk = std::max(dyk, std::fabs(y[i] - y[j]));
        }
        for (int64_t j = 0; j < w; ++j) {
            if (j == i) continue;
            if (std::fabs(x[i] - x[j]) <= dxk) ++nx;
            if (std::fabs(y[i] - y[j]) <= dyk) ++ny;
        }
    }
    *out_eps = eps;
    out_n[0] = (int32_t)nx;
    out_n[1] = (int32_t)ny;
    return 0;
}

// Per-point canonical terms (q(psi(a)) + q(psi(b)), q(LN(2 eps)) or 0) and the window finish
// from the canonical sums: out3 = {mi, h, nmi}.
int64_t oracle_point_psi_q(int32_t nx, int32_t ny, int32_t variant) {
    int64_t a = variant == 0 ? nx + 1 : nx, b = variant == 0 ? ny + 1 : ny;
    ensure_psi(std::max(a, b));
    return q32(psi(a)) + q32(psi(b));
}
int64_t oracle_point_log_q(float eps) { return eps > 0.0f ? q32(canon_ln(2.0 * (double)eps)) : 0; }

int oracle_finish(int64_t s_psi, int64_t s_log, int32_t zeros, int64_t w, int32_t k, int32_t variant,
                  double* out3) {
    ensure_psi(w + 1);
    double dw = (double)w;
    double mean_q = ((double)s_psi * kTwoPowMinus32) / dw;
    double mi;
    if (variant == 0) {
        double a = psi(k) + psi(w);
        mi = a - mean_q;
    } else {
        double a = psi(k) - 1.0 / (double)k;
        a = a + psi(w);
        mi = a - mean_q;
    }
    double h;
    if (zeros > 0) {
        h = -INFINITY;
    } else {
        double a = psi(w) - psi(k);
        double m = ((double)s_log * kTwoPowMinus32) / dw;
        h = a + 2.0 * m;
    }
    out3[0] = mi;
    out3[1] = h;
    out3[2] = normalized(mi, h, zeros);
    return 0;
}

// Alg. 3 pieces for tests: Eqs. 6-9 on given trial totals; the sampled partition indices of a pair.
int oracle_auto_scores(int64_t cost_td, int64_t cost_bu, int32_t m, int64_t nL_td, int64_t nS_bu, double alpha,
                       double* out2) {
    if (m < 1 || cost_td < 0 || cost_bu < 0 || cost_td + cost_bu == 0 || !out2) return -1;
    auto_scores(cost_td, cost_bu, m, nL_td, nS_bu, alpha, &out2[0], &out2[1]);
    return out2[0] > out2[1] ? 1 : 2;
}
int oracle_auto_sample(int32_t M, int32_t m, uint64_t seed, int32_t pair_id, int32_t* out) {
    if (m < 1 || m > M || !out) return -1;
    std::vector<int32_t> idx(M);
    for (int32_t i = 0; i < M; ++i) idx[i] = i;
    Searcher::Rng rng{seed ^ ((uint64_t)(uint32_t)pair_id * 0x9E3779B97F4A7C15ull) ^ 0xA0761D6478BD642Full};
    for (int32_t i = 0; i < m; ++i) {
        const int32_t j = i + (int32_t)((rng.next() >> 32) % (uint64_t)(M - i));
        std::swap(idx[i], idx[j]);
    }
    for (int32_t i = 0; i < m; ++i) out[i] = idx[i];
    return 0;
}

int oracle_chunk_plan(int64_t n, int32_t n_p, int64_t s_max, int64_t* out, int32_t cap) {
    auto c = chunk_plan(n, n_p, s_max);
    for (int32_t i = 0; i < (int32_t)c.size() && i < cap; ++i) { out[2 * i] = c[i].first; out[2 * i + 1] = c[i].second; }
    return (int)c.size();
}

}  // extern "C"
