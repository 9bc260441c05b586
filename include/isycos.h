/*
 * isycos.h — C ABI of libisycos.so, the B200-native (sm_100a) hot path of iSYCOS
 * (Ho et al., "A Unified Approach for Multi-Scale Synchronous Correlation Search in
 * Big Time Series", arXiv 2204.09131; citations "P:<line>" are lines of the paper's
 * LaTeX source, "S:<line>" of SPEC.md, "§8(x)" of SURVEY.md).
 *
 * The library evaluates the KSG k-nearest-neighbour mutual information (Eq. 2,
 * P:148-157; default estimator KSG-1, see below) of many candidate windows [t0,t1)
 * of a synchronous series pair (Defs 3.2-3.4, 4.2) on the GPU,
 * and drives the paper's searches — SYCOS_TD (Alg. 1), SYCOS_BU (Alg. 2,
 * P:389-431), MI-based noise pruning (Def 6.2 and §6.2-6.3) and the
 * overlapping-chunk plan of Alg. 4 — by batching the windows each search step
 * needs.  Every arithmetic step runs in CUDA kernels; there is no CPU fallback: a
 * missing or failing GPU returns ISYCOS_E_CUDA.
 *
 * Conventions (all entry points)
 *   - Return value: ISYCOS_OK (0) or a negative ISYCOS_E_* code.  A human-readable
 *     message for the last failure on the calling thread is isycos_last_error().
 *   - Pointers may be host or device (current device) memory; the library detects
 *     which with cudaPointerGetAttributes.  All buffers are caller-owned; the library
 *     keeps no reference after return.  Calls are blocking: they return after every
 *     output has been written (on `stream` when one is given).
 *   - Windows are half-open [t0, t1); the paper's closed [t_s, t_e] maps to
 *     [t_s, t_e + 1).  Window size w = t1 - t0 must satisfy k < w <= ISYCOS_MAX_W.
 *   - Inputs must be finite; ties are never an error.
 *   - One device per calling thread (the current CUDA device).  Not re-entrant on the
 *     same device from several threads at once.
 *
 * Estimator (per window W of w points, float32 inputs)
 *   d_ij  = max(|fl(x_i - x_j)|, |fl(y_i - y_j)|)             (max norm, P:671 footnote)
 *   eps_i = k-th smallest of { d_ij : j in W, j != i }          (multiset order statistic)
 *   KSG-1 (variant 0, default; north star):
 *     n_x(i) = #{ j != i : |fl(x_i - x_j)| < eps_i },  n_y likewise (strict)
 *     I = psi(k) + psi(w) - < psi(n_x + 1) + psi(n_y + 1) >
 *   KSG-2 (variant 1, Eq. 2 literal, text P:669, example P:671):
 *     kNN(i) = the first k of j != i in ascending (d_ij, j) order (tie: smaller index)
 *     d_x(i) = max_{j in kNN(i)} |fl(x_i - x_j)|,  d_y likewise
 *     n_x(i) = #{ j != i : |fl(x_i - x_j)| <= d_x(i) },  n_y likewise (closed, >= k)
 *     I = psi(k) - 1/k + psi(w) - < psi(n_x) + psi(n_y) >
 *     (H and nmi use the KSG-1 radius eps_i for both variants; dbg_nx/dbg_ny report
 *     the variant's own counts.)
 *   Entropy (Eq. 13 read as the Kozachenko-Leonenko joint entropy, G2):
 *     H = psi(w) - psi(k) + (2/w) * sum_i ln(2 eps_i);  H = -inf if any eps_i == 0
 *   Normalized MI (Eq. 12): nmi = clamp(I/H, 0, 1); if any eps_i == 0 or
 *     H <= 1e-6 then nmi = (I > 1e-6) ? 1 : 0.
 *   Canonical numerics (DESIGN.md §Canonical numerics): the per-point digamma terms
 *   are summed exactly as int64 fixed point (Q = 2^32) and finished with a fixed fp64
 *   operation sequence, so I, H and nmi are bit-reproducible and agree with the oracle.
 */
#ifndef ISYCOS_H
#define ISYCOS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ISYCOS_ABI_VERSION 3
#define ISYCOS_MAX_K 16
#define ISYCOS_MAX_W 262144 /* 2^18: int64 fixed-point bound of the digamma sums */

enum {
    ISYCOS_OK = 0,
    ISYCOS_E_INVAL = -1,   /* null pointer, n < 2, k outside [1,16], non-finite input, bad params */
    ISYCOS_E_RANGE = -2,   /* window not 0 <= t0 < t1 <= n, or w > ISYCOS_MAX_W */
    ISYCOS_E_TOO_FEW = -3, /* w <= k */
    ISYCOS_E_TRUNC = -4,   /* out_capacity too small; *out_count = required */
    ISYCOS_E_CUDA = -5,    /* CUDA error or no usable sm_100 device */
    ISYCOS_E_NOMEM = -6,   /* device or pinned host allocation failed */
    ISYCOS_E_NCCL = -7     /* reserved: collectives live in the Python layer (torch.distributed) */
};

/* flags */
#define ISYCOS_F_PROFILE 1u /* record CUDA events around every KSG kernel; fills *_kernel_ms */
#define ISYCOS_F_BRUTE 2u   /* route every window to the brute-force kernels (no sorted-marginal path);
                               results are bit-identical either way — an A/B and test knob */
#define ISYCOS_F_PROFILE_SORTED_ONLY 8u /* with ISYCOS_F_PROFILE: events around sorted-path launches only */
#define ISYCOS_F_PROFILE_BRUTE_ONLY 16u  /* with ISYCOS_F_PROFILE: events around brute-force launches only */
#define ISYCOS_F_NO_BLOCK 32u /* no NEXT-3 shared-block sorts (every sorted-path window sorted from scratch)
                                 and no incremental radii; A/B knob, results identical */
#define ISYCOS_F_INCREMENTAL 64u /* NEXT-3 incremental radii and counts along block-grid chains (KSG-1; results
                                    identical; off by default: measured time-neutral on B200) */
#define ISYCOS_F_UNFUSED 4u /* sorted-marginal windows always take the throughput form (sort kernel, then
                               scan kernel), never the fused latency kernel; results identical */

/* Half-open window [t0, t1) of a series pair (Defs 3.2, 3.4). */
typedef struct {
    int64_t t0, t1;
} isycos_window;

/* Kernel-level counters of one call (filled when the caller passes a pointer). */
typedef struct {
    int64_t windows;       /* windows evaluated by kernels (including speculative ones in a search) */
    int64_t point_pairs;   /* sum over those windows of w*(w-1) ordered point pairs */
    int64_t launches;      /* kernels launched by the library (all kinds) */
    int64_t ksg_launches;  /* launches of the KSG window kernels */
    int64_t rounds;        /* host<->device rounds (batches) */
    double kernel_ms;      /* sum of KSG kernel durations (CUDA events; ISYCOS_F_PROFILE only) */
    int64_t h2d_bytes, d2h_bytes;
    double host_ms;        /* host time spent forming batches and replaying decisions (search) */
    double wall_ms;        /* wall time of the call */
    int64_t scan_steps;    /* sorted-marginal path: outward k-NN scan steps executed (algorithmic work) */
    int64_t sorted_windows, sorted_points; /* windows / points evaluated on the sorted-marginal path */
    int64_t brute_point_pairs; /* ordered point pairs of windows evaluated by the brute-force kernels */
    int64_t search_probes; /* sorted path: binary-search probes (5 searches x ceil(log2 w) per point) */
    double sorted_kernel_ms, brute_kernel_ms; /* ISYCOS_F_PROFILE: per-path share of kernel_ms */
    /* isycos_search with ISYCOS_F_PROFILE times every ISYCOS_PROFILE_EVERY-th round (env, default 1):
     * the work of the profiled rounds, to divide by the *_kernel_ms above */
    int64_t profiled_rounds, prof_brute_point_pairs, prof_scan_steps, prof_search_probes;
    /* NEXT-3 (incremental MI, GPU analogue): windows whose sorted layout was merged from shared
     * beta-blocks (each block sorted once per batch), and the block points sorted */
    int64_t block_windows, block_points;
    /* NEXT-3 incremental radii: windows that followed their predecessor on a grid chain, and the points of
     * those windows whose k-NN radius carried over (no removed / inserted point could change it) */
    int64_t inc_windows, eps_reused_points;
} isycos_kernel_stats;

/*
 * isycos_mi_batch — KSG-1 MI of each window (north star: isycos_mi_batch(x, y, n,
 * windows[], k, out_mi)).
 *   x, y       series pair, n float32 samples each (host or device)
 *   windows    n_windows half-open windows (host or device)
 *   k          neighbours, 1 <= k <= 16, k < every window size
 *   out_mi     n_windows doubles (host or device)
 * Errors: E_INVAL (null, n < 2, k out of range, non-finite sample), E_RANGE, E_TOO_FEW,
 *   E_CUDA, E_NOMEM.  On error no output is guaranteed.
 */
int isycos_mi_batch(const float* x, const float* y, int64_t n, const isycos_window* windows,
                    int64_t n_windows, int32_t k, double* out_mi);

/* Optional outputs / controls of isycos_mi_batch_ex.  Zero-initialise, then set fields. */
typedef struct {
    int32_t variant;        /* 0 = KSG-1 (default), 1 = KSG-2; anything else: E_INVAL */
    uint32_t flags;         /* ISYCOS_F_* */
    void* stream;           /* cudaStream_t to run on; NULL = the library's own stream */
    double* out_h;          /* [n_windows] KL joint entropy H (nats) */
    double* out_nmi;        /* [n_windows] normalized MI */
    int64_t* out_sum_psi_q; /* [n_windows] sum_i q(psi(n_x+1)) + q(psi(n_y+1)) (KSG-2: q(psi(n_x)) + q(psi(n_y))), q(v) = rint(v*2^32) */
    int64_t* out_sum_log_q; /* [n_windows] sum_{eps_i>0} q(LN(2 eps_i)) */
    int32_t* out_zero_eps;  /* [n_windows] #{i : eps_i == 0} */
    float* dbg_eps;         /* [sum w] per-point eps_i, windows concatenated in input order */
    int32_t* dbg_nx;        /* [sum w] per-point n_x(i) */
    int32_t* dbg_ny;        /* [sum w] per-point n_y(i) */
    isycos_kernel_stats* stats;
} isycos_mi_opts;

int isycos_mi_batch_ex(const float* x, const float* y, int64_t n, const isycos_window* windows,
                       int64_t n_windows, int32_t k, const isycos_mi_opts* opts, double* out_mi);

/* A series pair for the search: indices into series[], plus the pair id used to tag
 * results and key the LAHC random stream (keep it stable when sharding across GPUs). */
typedef struct {
    int32_t xs, ys, id;
} isycos_pair;

/* Scale bounds (Table 1).  sizes == NULL => TD layers halve s_max -> s_min
 * (last layer = s_min).  BU windows range over [s_min, s_max] (Def 5.2). */
typedef struct {
    int64_t s_min, s_max;
    const int64_t* sizes; /* optional explicit TD layer sizes, strictly decreasing */
    int32_t n_sizes;
} isycos_scales;

/* MI-based noise pruning (Def 6.2; §6.2-6.3).  tau = tau_ratio * sigma
 * (eps/sigma = 0.25); p = consecutive noise verdicts before pruning. */
typedef struct {
    int32_t enabled;
    double tau_ratio;
    int32_t p;
} isycos_noise;

typedef struct {
    double sigma;         /* correlation threshold on normalized MI (default 0.2) */
    int32_t method;       /* 1 = TD, 2 = BU, 3 = both (results tagged per method), 4 = AUTO (below) */
    int32_t variant;      /* 0 = KSG-1 (default), 1 = KSG-2 (Eq. 2 literal) */
    int64_t delta_td;     /* TD sliding step; 0 => max(1, s/4) per layer */
    int64_t delta_bu;     /* BU neighbour step; 0 => max(1, s_min/3) */
    int32_t t_max_idle;   /* Alg. 2 idle budget (loop while idle <= T_maxIdle, G5) */
    int32_t h;            /* LAHC history length L_h */
    int32_t n_chunks;     /* Alg. 4 overlapping chunks per pair (>= 1) */
    int32_t lookahead;    /* BU speculative climbs per chain (0 => default 32) */
    uint64_t seed;        /* LAHC random streams: SplitMix64 keyed by (seed, pair id, climb start) */
    uint32_t flags;       /* ISYCOS_F_* */
    void* stream;         /* cudaStream_t; NULL = the library's own stream */
    /* method 4 (AUTO, iSYCOS Alg. 3): M partitions of floor(n/M) samples, m of them sampled
     * (SplitMix64 keyed by (seed, pair id)); SYCOS_TD and SYCOS_BU run alone on each; runtime proxy
     * t = eval_cost of the run; windows small iff |w| <= rho * s_max; Eqs. 6-9 with weight alpha;
     * TD iff nscore_TD > nscore_BU; the chosen method then runs on the whole series (results tagged
     * with it).  Zero => defaults M = 20, m = 6, alpha = 0.5, rho = 0.5.  Needs m <= M, n / M >= s_min. */
    int32_t auto_M, auto_m;
    double auto_alpha, auto_rho;
    /* (pair, chunk) work units for multi-GPU sharding (Alg. 4 line 14): 0, 0 => every
     * chunk of the n_chunks plan, merged per (pair, method).  Otherwise only chunks [chunk_begin,
     * chunk_end) of the plan run and their windows are returned UNMERGED (per chunk, each chunk's windows
     * disjoint); isycos_merge_windows applies the merge once all chunks of a pair are gathered.  The
     * per-chunk searches are independent, so the merged result equals the all-chunks call.  Not with
     * method 4. */
    int32_t chunk_begin, chunk_end;
} isycos_search_opts;

/* One accepted window (Def 3.5).  Records are sorted by (pair, method, t0); per (pair,
 * method) they are pairwise disjoint, s_min <= t1 - t0 <= s_max and nmi >= sigma. */
typedef struct {
    int32_t pair, method;
    int64_t t0, t1;
    double mi, h, nmi;
} isycos_result_window;

/* Algorithm-level counters: identical to the oracle's for the same inputs (they count
 * what the sequential algorithms consume, not what the GPU speculated). */
typedef struct {
    int64_t td_windows, td_noise_checks, td_skips, td_accepted;
    int64_t bu_climbs, bu_iterations, bu_neighbors, bu_noise_checks, bu_prunes, bu_accepted;
    int64_t distinct_windows, distinct_pairs; /* per pair, union over chunks and methods */
    int64_t eval_cost;      /* sum over distinct windows computed of w * ceil(log2 w) (t_w ~ w log w) */
    int64_t auto_td, auto_bu;               /* method AUTO: pairs for which Alg. 3 chose TD / BU */
    double auto_nscore_td, auto_nscore_bu;  /* method AUTO: sums over pairs of nscore_TD / nscore_BU (Eqs. 8-9) */
    isycos_kernel_stats kernel;
} isycos_search_stats;

/*
 * isycos_search — SYCOS search over series pairs (north star: isycos_search(series, pairs,
 * scale bounds, k, noise params, out_windows)).
 *   series       n_series pointers to n float32 samples each (host or device, all alike)
 *   pairs        n_pairs pairs (host memory)
 *   scales, noise, opts   host structs (see above); noise may be NULL (= disabled)
 *   out_windows  out_capacity records (host memory)
 *   out_count    number of records found (also set on E_TRUNC)
 *   out_stats    optional counters
 * Errors: E_INVAL (bad params: 2 <= s_min <= s_max <= n, k < s_min, 0 < sigma <= 1,
 *   0 <= tau_ratio < 1, h >= 1, p >= 1, t_max_idle >= 0, method in 1..4, n_chunks >= 1; AUTO:
 *   m <= M, n / M >= s_min, alpha and rho in [0, 1]),
 *   E_TRUNC (first out_capacity records written, *out_count = required), E_CUDA, E_NOMEM.
 */
int isycos_search(const float* const* series, int32_t n_series, int64_t n, const isycos_pair* pairs,
                  int32_t n_pairs, const isycos_scales* scales, int32_t k, const isycos_noise* noise,
                  const isycos_search_opts* opts, isycos_result_window* out_windows,
                  int64_t out_capacity, int64_t* out_count, isycos_search_stats* out_stats);

/*
 * isycos_merge_windows — the chunk merge of Alg. 4 (the paper is silent on the rule, reading R20):
 * per (pair, method), greedy by (nmi desc, mi desc, t0 asc, t1 asc), a window is kept iff it is disjoint
 * from every window kept before it; output sorted by (pair, method, t0).
 *   in       n records (host memory, any order); out  out_capacity records (host memory, may not alias in)
 * Errors: E_INVAL (null pointers, n < 0), E_TRUNC (first out_capacity written, *out_count = required).
 */
int isycos_merge_windows(const isycos_result_window* in, int64_t n, isycos_result_window* out,
                         int64_t out_capacity, int64_t* out_count);

/* Message for the last non-OK return on this thread ("" if none).  Valid until the next call. */
const char* isycos_last_error(void);

/* ISYCOS_ABI_VERSION of the loaded library. */
int isycos_abi_version(void);

/* Release the library's cached device / pinned buffers on the current device. */
int isycos_release_cache(void);

#ifdef __cplusplus
}
#endif

#endif /* ISYCOS_H */
