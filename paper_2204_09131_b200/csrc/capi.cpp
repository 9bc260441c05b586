// C ABI of libisycos.so (include/isycos.h): validation, host/device pointer handling, error codes.
// All arithmetic of the path runs in the ksg_*.cu kernels; this file only marshals.

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "engine.h"

using namespace isy;

namespace {

// Device memory (or managed memory) the kernels can read directly?  Device memory of ANOTHER device is an
// argument error (kernels would fault with a sticky illegal-address error): *other_dev is set and the
// callers return ISYCOS_E_INVAL.  Host memory (pageable, pinned or mapped) is staged by the library.
bool is_device_ptr(const void* p, bool* other_dev = nullptr) {
    if (other_dev) *other_dev = false;
    if (!p) return false;
    cudaPointerAttributes a;
    cudaError_t e = cudaPointerGetAttributes(&a, p);
    if (e != cudaSuccess) {
        cudaGetLastError();  // clear: unregistered host memory on some drivers
        return false;
    }
    if (a.type == cudaMemoryTypeManaged) return true;
    if (a.type != cudaMemoryTypeDevice) return false;
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && a.device != cur && other_dev) *other_dev = true;
    return true;
}

Status check_ptr(const void* p, const char* what) {
    bool other = false;
    is_device_ptr(p, &other);
    if (other)
        return make_err(ISYCOS_E_INVAL, std::string(what) + " is device memory of another GPU than the current "
                                                              "device (call cudaSetDevice / torch.cuda.set_device)");
    return Status{};
}

int fail(const Status& s) {
    set_last_error(s);
    return s.code;
}

int ok() {
    set_last_error(Status{});
    return ISYCOS_OK;
}

// A series resident on the device in the layout the kernels need (16-B aligned, readable up to a
// multiple of 4 floats).  Caller-owned device series that already satisfy this are used in place.
struct DevSeries {
    DevSeries() = default;
    DevSeries(const DevSeries&) = delete;
    DevSeries& operator=(const DevSeries&) = delete;
    Engine* eng = nullptr;
    const float* ptr = nullptr;
    float* owned = nullptr;
    ~DevSeries() {
        if (owned) eng->free_series(owned);
    }
    Status make(Engine* e, const float* src, int64_t n, cudaStream_t st, BatchStats* bs) {
        eng = e;
        const bool dev = is_device_ptr(src);
        if (dev && (reinterpret_cast<uintptr_t>(src) % 16 == 0) && (n % 4 == 0)) {
            ptr = src;
            return Status{};
        }
        Status s = e->upload_series(src, n, dev, &owned, st, bs);
        ptr = owned;
        return s;
    }
};

// copy `bytes` from a host buffer to a caller pointer that may be host or device
Status put_out(void* dst, const void* src, size_t bytes, cudaStream_t st) {
    if (!dst || bytes == 0) return Status{};
    if (is_device_ptr(dst)) {
        cudaError_t e = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        return cuda_err(e, "copy output to device");
    }
    std::memcpy(dst, src, bytes);
    return Status{};
}

}  // namespace

extern "C" int isycos_abi_version(void) { return ISYCOS_ABI_VERSION; }

extern "C" int isycos_release_cache(void) {
    release_engine_for_current_device();
    return ok();
}

extern "C" int isycos_mi_batch_ex(const float* x, const float* y, int64_t n, const isycos_window* windows,
                                  int64_t n_windows, int32_t k, const isycos_mi_opts* opts, double* out_mi) {
    if (!x || !y || (!windows && n_windows > 0) || (!out_mi && n_windows > 0))
        return fail(make_err(ISYCOS_E_INVAL, "null pointer argument"));
    if (n < 2) return fail(make_err(ISYCOS_E_INVAL, "n must be >= 2"));
    if (k < 1 || k > ISYCOS_MAX_K) return fail(make_err(ISYCOS_E_INVAL, "k must be in [1, 16]"));
    if (n_windows < 0) return fail(make_err(ISYCOS_E_INVAL, "n_windows < 0"));
    isycos_mi_opts o{};
    if (opts) o = *opts;
    if (o.variant != 0 && o.variant != 1)
        return fail(make_err(ISYCOS_E_INVAL, "variant must be 0 (KSG-1) or 1 (KSG-2)"));
    if (n_windows == 0) return ok();

    Status s;
    for (auto [p, what] : {std::pair<const void*, const char*>{x, "x"}, {y, "y"}, {windows, "windows"},
                           {out_mi, "out_mi"}, {o.out_h, "out_h"}, {o.out_nmi, "out_nmi"},
                           {o.out_sum_psi_q, "out_sum_psi_q"}, {o.out_sum_log_q, "out_sum_log_q"},
                           {o.out_zero_eps, "out_zero_eps"}, {o.dbg_eps, "dbg_eps"}, {o.dbg_nx, "dbg_nx"},
                           {o.dbg_ny, "dbg_ny"}})
        if (!(s = check_ptr(p, what)).ok()) return fail(s);
    Engine* eng = engine_for_current_device(&s);
    if (!eng) return fail(s);
    cudaStream_t st = o.stream ? static_cast<cudaStream_t>(o.stream) : eng->own_stream();
    BatchStats bs;

    // windows to host
    std::vector<isycos_window> wh(n_windows);
    if (is_device_ptr(windows)) {
        cudaError_t e = cudaMemcpyAsync(wh.data(), windows, n_windows * sizeof(isycos_window),
                                        cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return fail(cuda_err(e, "copy windows to host"));
        bs.d2h_bytes += n_windows * (int64_t)sizeof(isycos_window);
    } else {
        std::memcpy(wh.data(), windows, n_windows * sizeof(isycos_window));
    }
    int64_t total_pts = 0;
    for (int64_t i = 0; i < n_windows; ++i) {
        const int64_t t0 = wh[i].t0, t1 = wh[i].t1;
        if (t0 < 0 || t1 > n || t0 >= t1)
            return fail(make_err(ISYCOS_E_RANGE, "window " + std::to_string(i) + " = [" + std::to_string(t0) + ", " +
                                                     std::to_string(t1) + ") outside [0, n)"));
        if (t1 - t0 > ISYCOS_MAX_W) return fail(make_err(ISYCOS_E_RANGE, "window larger than ISYCOS_MAX_W"));
        if (t1 - t0 <= k)
            return fail(make_err(ISYCOS_E_TOO_FEW, "window " + std::to_string(i) + " has w <= k"));
        total_pts += t1 - t0;
    }

    DevSeries dx, dy;
    if (!(s = dx.make(eng, x, n, st, &bs)).ok()) return fail(s);
    if (!(s = dy.make(eng, y, n, st, &bs)).ok()) return fail(s);
    bool fin_x = false, fin_y = false;
    if (!(s = eng->check_finite(dx.ptr, n, st, &fin_x)).ok()) return fail(s);
    if (!(s = eng->check_finite(dy.ptr, n, st, &fin_y)).ok()) return fail(s);
    bs.launches += 2;
    if (!fin_x || !fin_y) return fail(make_err(ISYCOS_E_INVAL, "non-finite sample in x or y"));

    // debug outputs: kernels write device memory; stage through device temporaries if needed
    const bool want_dbg = o.dbg_eps || o.dbg_nx || o.dbg_ny;
    DebugOut dbg;
    std::vector<void*> tmp_dev;
    auto dev_target = [&](void* user, size_t elem, void** devp) -> Status {
        if (!user) {
            *devp = nullptr;
            return Status{};
        }
        if (is_device_ptr(user)) {
            *devp = user;
            return Status{};
        }
        void* p = nullptr;
        cudaError_t e = cudaMalloc(&p, total_pts * elem);
        if (e != cudaSuccess) return cuda_err(e, "cudaMalloc debug buffer");
        tmp_dev.push_back(p);
        *devp = p;
        return Status{};
    };
    void *de = nullptr, *dnx = nullptr, *dny = nullptr;
    auto cleanup = [&] {
        for (void* p : tmp_dev) cudaFree(p);
    };
    if (want_dbg) {
        if (!(s = dev_target(o.dbg_eps, 4, &de)).ok() || !(s = dev_target(o.dbg_nx, 4, &dnx)).ok() ||
            !(s = dev_target(o.dbg_ny, 4, &dny)).ok()) {
            cleanup();
            return fail(s);
        }
        dbg.eps = static_cast<float*>(de);
        dbg.nx = static_cast<int32_t*>(dnx);
        dbg.ny = static_cast<int32_t*>(dny);
    }

    PairPtrs pp{dx.ptr, dy.ptr};
    std::vector<KsgWin> wins(n_windows);
    int64_t off = 0;
    for (int64_t i = 0; i < n_windows; ++i) {
        const int32_t w = (int32_t)(wh[i].t1 - wh[i].t0);
        wins[i] = KsgWin{wh[i].t0, w, 0, want_dbg ? off : -1};
        off += w;
    }
    std::vector<KsgRec> recs(n_windows);
    s = eng->evaluate(&pp, 1, wins.data(), n_windows, k, o.variant, recs.data(), dbg, st,
                      o.flags, &bs);
    if (!s.ok()) {
        cleanup();
        return fail(s);
    }
    // debug arrays back to host targets
    auto dbg_back = [&](void* user, void* devp) -> Status {
        if (!user || user == devp) return Status{};
        cudaError_t e = cudaMemcpyAsync(user, devp, total_pts * 4, cudaMemcpyDeviceToHost, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        return cuda_err(e, "copy debug output");
    };
    if (want_dbg) {
        if (!(s = dbg_back(o.dbg_eps, de)).ok() || !(s = dbg_back(o.dbg_nx, dnx)).ok() ||
            !(s = dbg_back(o.dbg_ny, dny)).ok()) {
            cleanup();
            return fail(s);
        }
    }
    cleanup();

    std::vector<double> col(n_windows);
    auto put_d = [&](double* dst, auto getter) -> Status {
        if (!dst) return Status{};
        for (int64_t i = 0; i < n_windows; ++i) col[i] = getter(recs[i]);
        return put_out(dst, col.data(), n_windows * sizeof(double), st);
    };
    if (!(s = put_d(out_mi, [](const KsgRec& r) { return r.mi; })).ok()) return fail(s);
    if (!(s = put_d(o.out_h, [](const KsgRec& r) { return r.h; })).ok()) return fail(s);
    if (!(s = put_d(o.out_nmi, [](const KsgRec& r) { return r.nmi; })).ok()) return fail(s);
    if (o.out_sum_psi_q || o.out_sum_log_q) {
        std::vector<int64_t> c(n_windows);
        if (o.out_sum_psi_q) {
            for (int64_t i = 0; i < n_windows; ++i) c[i] = recs[i].s_psi;
            if (!(s = put_out(o.out_sum_psi_q, c.data(), n_windows * 8, st)).ok()) return fail(s);
        }
        if (o.out_sum_log_q) {
            for (int64_t i = 0; i < n_windows; ++i) c[i] = recs[i].s_log;
            if (!(s = put_out(o.out_sum_log_q, c.data(), n_windows * 8, st)).ok()) return fail(s);
        }
    }
    if (o.out_zero_eps) {
        std::vector<int32_t> c(n_windows);
        for (int64_t i = 0; i < n_windows; ++i) c[i] = recs[i].zero_eps;
        if (!(s = put_out(o.out_zero_eps, c.data(), n_windows * 4, st)).ok()) return fail(s);
    }
    if (o.stats) bs.add_to(o.stats);
    return ok();
}

extern "C" int isycos_mi_batch(const float* x, const float* y, int64_t n, const isycos_window* windows,
                               int64_t n_windows, int32_t k, double* out_mi) {
    return isycos_mi_batch_ex(x, y, n, windows, n_windows, k, nullptr, out_mi);
}

extern "C" int isycos_search(const float* const* series, int32_t n_series, int64_t n, const isycos_pair* pairs,
                             int32_t n_pairs, const isycos_scales* scales, int32_t k, const isycos_noise* noise,
                             const isycos_search_opts* opts, isycos_result_window* out_windows,
                             int64_t out_capacity, int64_t* out_count, isycos_search_stats* out_stats) {
    if (!series || !pairs || !scales || !opts || !out_count || (!out_windows && out_capacity > 0))
        return fail(make_err(ISYCOS_E_INVAL, "null pointer argument"));
    if (n_series < 1 || n_pairs < 0 || n < 2) return fail(make_err(ISYCOS_E_INVAL, "bad n_series / n_pairs / n"));
    SearchParams P;
    P.k = k;
    P.variant = opts->variant;
    P.method = opts->method;
    P.auto_M = opts->auto_M;
    P.auto_m = opts->auto_m;
    P.auto_alpha = opts->auto_alpha;
    P.auto_rho = opts->auto_rho;
    P.s_min = scales->s_min;
    P.s_max = scales->s_max;
    if (scales->sizes && scales->n_sizes > 0) P.sizes.assign(scales->sizes, scales->sizes + scales->n_sizes);
    P.noise = noise && noise->enabled;
    P.tau_ratio = noise ? noise->tau_ratio : 0.25;
    P.p = noise ? noise->p : 3;
    P.sigma = opts->sigma;
    P.delta_td = opts->delta_td;
    P.delta_bu = opts->delta_bu;
    P.t_max_idle = opts->t_max_idle;
    P.h = opts->h;
    P.n_chunks = opts->n_chunks;
    P.lookahead = opts->lookahead > 0 ? opts->lookahead : 32;
    P.seed = opts->seed;
    P.flags = opts->flags;
    P.chunk_begin = opts->chunk_begin;
    P.chunk_end = opts->chunk_end;
    // speculation tuning knobs (do not change results)
    if (const char* e = std::getenv("ISYCOS_BU_DEPTH")) P.bu_depth = std::atoi(e);
    if (const char* e = std::getenv("ISYCOS_TREND_DEPTH")) P.trend_depth = std::atoi(e);
    if (const char* e = std::getenv("ISYCOS_PIPELINE")) P.pipeline = std::atoi(e) != 0;
    if (const char* e = std::getenv("ISYCOS_RING_RANK")) P.ring_rank = std::atoi(e);
    if (const char* e = std::getenv("ISYCOS_HOST_THREADS")) P.host_threads = std::atoi(e);
    if (const char* e = std::getenv("ISYCOS_PROFILE_EVERY")) P.profile_every = std::max(1, std::atoi(e));
    if (const char* e = std::getenv("ISYCOS_ANCHOR")) P.anchor_lookahead = std::atoi(e);
    if (const char* e = std::getenv("ISYCOS_SPEC_CAP")) P.spec_cap_mult = std::atoi(e);
    if (const char* e = std::getenv("ISYCOS_LOOKAHEAD")) P.lookahead = std::atoi(e);
    auto bad = [&](const char* m) { return fail(make_err(ISYCOS_E_INVAL, m)); };
    if (k < 1 || k > ISYCOS_MAX_K) return bad("k must be in [1, 16]");
    if (P.variant != 0 && P.variant != 1) return bad("variant must be 0 (KSG-1) or 1 (KSG-2)");
    if (P.s_min < 2 || P.s_min > P.s_max || P.s_max > n) return bad("need 2 <= s_min <= s_max <= n");
    if (P.s_max > ISYCOS_MAX_W) return bad("s_max > ISYCOS_MAX_W");
    if (k >= P.s_min) return bad("need k < s_min");
    if (!(P.sigma > 0.0 && P.sigma <= 1.0)) return bad("need 0 < sigma <= 1");
    if (!(P.tau_ratio >= 0.0 && P.tau_ratio < 1.0)) return bad("need 0 <= tau_ratio < 1");
    if (P.h < 1 || P.p < 1 || P.t_max_idle < 0) return bad("need h >= 1, p >= 1, t_max_idle >= 0");
    if (P.method < 1 || P.method > 4) return bad("method must be 1 (TD), 2 (BU), 3 (both) or 4 (AUTO)");
    if (P.method == 4) {
        const int32_t M = P.auto_M > 0 ? P.auto_M : 20, m = P.auto_m > 0 ? P.auto_m : 6;
        if (m > M) return bad("AUTO: auto_m must be <= auto_M");
        if (n / M < P.s_min) return bad("AUTO: partitions floor(n / auto_M) shorter than s_min");
        if (P.auto_alpha < 0.0 || P.auto_alpha > 1.0 || P.auto_rho < 0.0 || P.auto_rho > 1.0)
            return bad("AUTO: auto_alpha and auto_rho must be in [0, 1]");
    }
    if (P.n_chunks < 1) return bad("n_chunks must be >= 1");
    if (P.chunk_begin != 0 || P.chunk_end != 0) {
        if (P.method == 4) return bad("chunk selection is not available with method 4 (AUTO)");
        const int32_t n_plan = (int32_t)chunks_of(n, P.n_chunks, P.s_max).size();
        if (P.chunk_begin < 0 || P.chunk_end <= P.chunk_begin || P.chunk_end > n_plan)
            return bad("need 0 <= chunk_begin < chunk_end <= number of chunks");
    }
    if (P.delta_td < 0 || P.delta_bu < 0) return bad("delta must be >= 0");
    for (size_t i = 0; i < P.sizes.size(); ++i) {
        if (P.sizes[i] <= k || P.sizes[i] > P.s_max || P.sizes[i] < P.s_min || (i && P.sizes[i] >= P.sizes[i - 1]))
            return bad("sizes must be strictly decreasing within [s_min, s_max] and > k");
    }
    for (int32_t i = 0; i < n_pairs; ++i) {
        if (pairs[i].xs < 0 || pairs[i].ys < 0 || pairs[i].xs >= n_series || pairs[i].ys >= n_series)
            return bad("pair index out of range");
    }

    Status s;
    for (int32_t i = 0; i < n_series; ++i)
        if (!(s = check_ptr(series[i], "a series pointer")).ok()) return fail(s);
    Engine* eng = engine_for_current_device(&s);
    if (!eng) return fail(s);
    cudaStream_t st = opts->stream ? static_cast<cudaStream_t>(opts->stream) : eng->own_stream();
    BatchStats bs;

    // series used by any pair -> device layout; finiteness checked on the device
    std::vector<char> used(n_series, 0);
    for (int32_t i = 0; i < n_pairs; ++i) used[pairs[i].xs] = used[pairs[i].ys] = 1;
    std::vector<DevSeries> dev(n_series);
    for (int32_t i = 0; i < n_series; ++i) {
        if (!used[i]) continue;
        if (!series[i]) return bad("null series pointer");
        if (!(s = dev[i].make(eng, series[i], n, st, &bs)).ok()) return fail(s);
        bool fin = false;
        if (!(s = eng->check_finite(dev[i].ptr, n, st, &fin)).ok()) return fail(s);
        bs.launches += 1;
        if (!fin) return fail(make_err(ISYCOS_E_INVAL, "non-finite sample in series " + std::to_string(i)));
    }
    std::vector<PairPtrs> pp(n_pairs);
    std::vector<int32_t> ids(n_pairs);
    for (int32_t i = 0; i < n_pairs; ++i) {
        pp[i] = PairPtrs{dev[pairs[i].xs].ptr, dev[pairs[i].ys].ptr};
        ids[i] = pairs[i].id;
    }
    std::vector<isycos_result_window> res;
    isycos_search_stats local{};
    s = run_search(eng, pp, ids, n, P, st, &res, &local);
    if (!s.ok()) return fail(s);
    bs.add_to(&local.kernel);
    if (out_stats) *out_stats = local;
    *out_count = (int64_t)res.size();
    const int64_t m = std::min<int64_t>(out_capacity, (int64_t)res.size());
    if (m > 0) std::memcpy(out_windows, res.data(), m * sizeof(isycos_result_window));
    if ((int64_t)res.size() > out_capacity)
        return fail(make_err(ISYCOS_E_TRUNC, "out_capacity too small: need " + std::to_string(res.size())));
    return ok();
}

extern "C" int isycos_merge_windows(const isycos_result_window* in, int64_t n, isycos_result_window* out,
                                    int64_t out_capacity, int64_t* out_count) {
    if ((!in && n > 0) || !out_count || (!out && out_capacity > 0) || n < 0 || out_capacity < 0)
        return fail(make_err(ISYCOS_E_INVAL, "null pointer or negative count"));
    std::vector<isycos_result_window> all(in, in + n);
    std::stable_sort(all.begin(), all.end(), [](const isycos_result_window& a, const isycos_result_window& b) {
        return a.pair != b.pair ? a.pair < b.pair : a.method < b.method;
    });
    std::vector<isycos_result_window> res;
    for (size_t i = 0; i < all.size();) {
        size_t j = i;
        while (j < all.size() && all[j].pair == all[i].pair && all[j].method == all[i].method) ++j;
        auto m = merge_windows(std::vector<isycos_result_window>(all.begin() + i, all.begin() + j));
        res.insert(res.end(), m.begin(), m.end());
        i = j;
    }
    *out_count = (int64_t)res.size();
    const int64_t m = std::min<int64_t>(out_capacity, (int64_t)res.size());
    if (m > 0) std::memcpy(out, res.data(), m * sizeof(isycos_result_window));
    if ((int64_t)res.size() > out_capacity)
        return fail(make_err(ISYCOS_E_TRUNC, "out_capacity too small: need " + std::to_string(res.size())));
    return ok();
}
