"""ctypes binding of libisycos.so (include/isycos.h).  Argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; if the library is missing
or the GPU is unusable, these functions raise — there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# ISYCOS_LIB: an alternative in-tree build of the same library (kernel A/B measurements only)
LIB_PATH = os.environ.get("ISYCOS_LIB") or os.path.join(HERE, "libisycos.so")

ISYCOS_OK, E_INVAL, E_RANGE, E_TOO_FEW, E_TRUNC, E_CUDA, E_NOMEM, E_NCCL = 0, -1, -2, -3, -4, -5, -6, -7
F_PROFILE = 1
F_BRUTE = 2   # force the brute-force kernels (A/B and test knob; results identical)
F_UNFUSED = 4  # sorted path in its throughput form only (no fused latency kernel)
F_PROFILE_SORTED_ONLY = 8
F_PROFILE_BRUTE_ONLY = 16
F_NO_BLOCK = 32  # no NEXT-3 shared-block sorts nor incremental radii (A/B knob; results identical)
F_INCREMENTAL = 64  # NEXT-3 incremental radii / counts along block-grid chains (off by default; results identical)
MAX_K = 16
MAX_W = 262144
ERROR_NAMES = {0: "OK", -1: "E_INVAL", -2: "E_RANGE", -3: "E_TOO_FEW", -4: "E_TRUNC", -5: "E_CUDA",
               -6: "E_NOMEM", -7: "E_NCCL"}

# symbols declared in include/isycos.h (checked by tests/test_abi.py)
EXPORTS = ["isycos_mi_batch", "isycos_mi_batch_ex", "isycos_search", "isycos_merge_windows",
           "isycos_last_error", "isycos_abi_version", "isycos_release_cache"]


class IsycosError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code


class Window(C.Structure):
    _fields_ = [("t0", C.c_int64), ("t1", C.c_int64)]


class KernelStats(C.Structure):
    _fields_ = [("windows", C.c_int64), ("point_pairs", C.c_int64), ("launches", C.c_int64),
                ("ksg_launches", C.c_int64), ("rounds", C.c_int64), ("kernel_ms", C.c_double),
                ("h2d_bytes", C.c_int64), ("d2h_bytes", C.c_int64), ("host_ms", C.c_double),
                ("wall_ms", C.c_double), ("scan_steps", C.c_int64), ("sorted_windows", C.c_int64),
                ("sorted_points", C.c_int64), ("brute_point_pairs", C.c_int64), ("search_probes", C.c_int64),
                ("sorted_kernel_ms", C.c_double), ("brute_kernel_ms", C.c_double), ("profiled_rounds", C.c_int64),
                ("prof_brute_point_pairs", C.c_int64), ("prof_scan_steps", C.c_int64),
                ("prof_search_probes", C.c_int64), ("block_windows", C.c_int64), ("block_points", C.c_int64),
                ("inc_windows", C.c_int64), ("eps_reused_points", C.c_int64)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class MiOpts(C.Structure):
    _fields_ = [("variant", C.c_int32), ("flags", C.c_uint32), ("stream", C.c_void_p),
                ("out_h", C.c_void_p), ("out_nmi", C.c_void_p), ("out_sum_psi_q", C.c_void_p),
                ("out_sum_log_q", C.c_void_p), ("out_zero_eps", C.c_void_p), ("dbg_eps", C.c_void_p),
                ("dbg_nx", C.c_void_p), ("dbg_ny", C.c_void_p), ("stats", C.POINTER(KernelStats))]


class Pair(C.Structure):
    _fields_ = [("xs", C.c_int32), ("ys", C.c_int32), ("id", C.c_int32)]


class Scales(C.Structure):
    _fields_ = [("s_min", C.c_int64), ("s_max", C.c_int64), ("sizes", C.POINTER(C.c_int64)),
                ("n_sizes", C.c_int32)]


class Noise(C.Structure):
    _fields_ = [("enabled", C.c_int32), ("tau_ratio", C.c_double), ("p", C.c_int32)]


class SearchOpts(C.Structure):
    _fields_ = [("sigma", C.c_double), ("method", C.c_int32), ("variant", C.c_int32),
                ("delta_td", C.c_int64), ("delta_bu", C.c_int64), ("t_max_idle", C.c_int32),
                ("h", C.c_int32), ("n_chunks", C.c_int32), ("lookahead", C.c_int32), ("seed", C.c_uint64),
                ("flags", C.c_uint32), ("stream", C.c_void_p), ("auto_M", C.c_int32), ("auto_m", C.c_int32),
                ("auto_alpha", C.c_double), ("auto_rho", C.c_double), ("chunk_begin", C.c_int32),
                ("chunk_end", C.c_int32)]


class ResultWindow(C.Structure):
    _fields_ = [("pair", C.c_int32), ("method", C.c_int32), ("t0", C.c_int64), ("t1", C.c_int64),
                ("mi", C.c_double), ("h", C.c_double), ("nmi", C.c_double)]


RESULT_DTYPE = np.dtype([("pair", np.int32), ("method", np.int32), ("t0", np.int64), ("t1", np.int64),
                         ("mi", np.float64), ("h", np.float64), ("nmi", np.float64)])
assert RESULT_DTYPE.itemsize == C.sizeof(ResultWindow)


SEARCH_STAT_FIELDS = ["td_windows", "td_noise_checks", "td_skips", "td_accepted", "bu_climbs",
                      "bu_iterations", "bu_neighbors", "bu_noise_checks", "bu_prunes", "bu_accepted",
                      "distinct_windows", "distinct_pairs", "eval_cost", "auto_td", "auto_bu"]
SEARCH_STAT_FIELDS_F = ["auto_nscore_td", "auto_nscore_bu"]


class SearchStats(C.Structure):
    _fields_ = ([(f, C.c_int64) for f in SEARCH_STAT_FIELDS] + [(f, C.c_double) for f in SEARCH_STAT_FIELDS_F]
                + [("kernel", KernelStats)])

    def as_dict(self):
        d = {f: getattr(self, f) for f in SEARCH_STAT_FIELDS + SEARCH_STAT_FIELDS_F}
        d["kernel"] = self.kernel.as_dict()
        return d


_lib = None


def lib():
    """Load libisycos.so (raise if it was not built: no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2204_09131_b200.build` "
                              "(or __graft_entry__.build()); there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        L.isycos_last_error.restype = C.c_char_p
        L.isycos_abi_version.restype = C.c_int
        L.isycos_mi_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32,
                                      C.c_void_p]
        L.isycos_mi_batch_ex.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32,
                                         C.POINTER(MiOpts), C.c_void_p]
        L.isycos_search.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.POINTER(Pair), C.c_int32,
                                    C.POINTER(Scales), C.c_int32, C.POINTER(Noise), C.POINTER(SearchOpts),
                                    C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.POINTER(SearchStats)]
        L.isycos_merge_windows.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
        _lib = L
    return _lib


def isycos_last_error() -> str:
    return lib().isycos_last_error().decode()


def isycos_abi_version() -> int:
    return lib().isycos_abi_version()


def isycos_release_cache() -> None:
    lib().isycos_release_cache()


def _check(rc: int):
    if rc != ISYCOS_OK:
        raise IsycosError(rc, isycos_last_error())


# ------------------------------------------------------------------ buffer marshalling
class _Buf:
    """A pointer to host (numpy) or device (torch CUDA tensor) memory, kept alive.

    CUDA tensors are passed through as they are, so they must already have the dtype the C ABI expects and
    live on the current device (no silent reinterpretation, no cross-device pointers); host inputs are
    converted.  Output buffers (output=True) are written in place, so they must match exactly."""

    def __init__(self, obj, dtype, output: bool = False, name: str = "buffer"):
        self.obj = obj
        self.device = False
        try:
            import torch

            if isinstance(obj, torch.Tensor):
                want = {np.float32: torch.float32, np.float64: torch.float64, np.int64: torch.int64,
                        np.int32: torch.int32}[np.dtype(dtype).type]
                if obj.is_cuda:
                    if obj.dtype != want:
                        raise TypeError(f"{name}: CUDA tensor of dtype {obj.dtype}, expected {want}")
                    if obj.device.index != torch.cuda.current_device():
                        raise ValueError(f"{name}: tensor on {obj.device}, but the current device is "
                                         f"cuda:{torch.cuda.current_device()} (torch.cuda.set_device)")
                    if not obj.is_contiguous():
                        raise ValueError(f"{name}: device tensors must be contiguous")
                    self.device = True
                    self.ptr = obj.data_ptr()
                    self.n = obj.numel()
                    return
                if output and (obj.dtype != want or not obj.is_contiguous()):
                    raise TypeError(f"{name}: output tensor must be contiguous {want}")
                obj = obj.detach().numpy()
        except ImportError:  # pragma: no cover
            pass
        if output:
            if not (isinstance(obj, np.ndarray) and obj.dtype == np.dtype(dtype) and obj.flags.c_contiguous
                    and obj.flags.writeable):
                raise TypeError(f"{name}: output buffer must be a writeable C-contiguous {np.dtype(dtype)} array")
            self.obj = obj
        else:
            self.obj = np.ascontiguousarray(obj, dtype=dtype)
        self.ptr = self.obj.ctypes.data
        self.n = self.obj.size


def _stream_ptr(stream):
    if stream is None:
        return None
    if isinstance(stream, int):
        return stream
    return stream.cuda_stream  # torch.cuda.Stream


def isycos_mi_batch(x, y, windows, k: int = 4):
    """KSG-1 MI of each window [t0,t1) of (x, y).  Returns a float64 numpy array."""
    out = isycos_mi_batch_ex(x, y, windows, k)
    return out["mi"]


def isycos_mi_batch_ex(x, y, windows, k: int = 4, *, outputs=("mi", "h", "nmi", "s_psi", "s_log", "zero_eps"),
                       debug: bool = False, profile: bool = False, stream=None, out=None, variant: int = 0,
                       brute: bool = False, unfused: bool = False, no_block: bool = False,
                       incremental: bool = False):
    """Full per-window records (and optional per-point eps/n_x/n_y).  variant 0 = KSG-1, 1 = KSG-2.

    x, y: float32 numpy arrays or torch tensors (CPU or CUDA); windows: (n, 2) int64 array/tensor.
    out: optional dict of caller-provided output buffers (e.g. CUDA tensors) keyed like `outputs`.
    """
    bx, by = _Buf(x, np.float32, name="x"), _Buf(y, np.float32, name="y")
    if bx.n != by.n:
        raise ValueError("x and y must have the same length")
    bw = _Buf(windows, np.int64, name="windows")
    nw = bw.n // 2
    res = {}
    o = MiOpts()
    o.variant = int(variant)
    o.flags = ((F_PROFILE if profile else 0) | (F_BRUTE if brute else 0) | (F_UNFUSED if unfused else 0)
               | (F_NO_BLOCK if no_block else 0) | (F_INCREMENTAL if incremental else 0))
    o.stream = _stream_ptr(stream)
    keep = []

    def target(name, dtype, count):
        if out is not None and name in out:
            b = _Buf(out[name], dtype, output=True, name=f"out[{name!r}]")
            if b.n < count:
                raise ValueError(f"out[{name!r}] holds {b.n} elements, needs {count}")
            keep.append(b)
            res[name] = out[name]
            return b.ptr
        a = np.empty(count, dtype)
        res[name] = a
        return a.ctypes.data

    mi_ptr = target("mi", np.float64, nw)
    if "h" in outputs:
        o.out_h = target("h", np.float64, nw)
    if "nmi" in outputs:
        o.out_nmi = target("nmi", np.float64, nw)
    if "s_psi" in outputs:
        o.out_sum_psi_q = target("s_psi", np.int64, nw)
    if "s_log" in outputs:
        o.out_sum_log_q = target("s_log", np.int64, nw)
    if "zero_eps" in outputs:
        o.out_zero_eps = target("zero_eps", np.int32, nw)
    if debug:
        W = np.asarray(windows.cpu() if hasattr(windows, "cpu") else windows, np.int64).reshape(-1, 2)
        tot = int((W[:, 1] - W[:, 0]).sum()) if nw else 0
        o.dbg_eps = target("eps", np.float32, tot)
        o.dbg_nx = target("nx", np.int32, tot)
        o.dbg_ny = target("ny", np.int32, tot)
    st = KernelStats()
    o.stats = C.pointer(st)
    rc = lib().isycos_mi_batch_ex(bx.ptr, by.ptr, bx.n, bw.ptr, nw, int(k), C.byref(o), mi_ptr)
    _check(rc)
    res["stats"] = st.as_dict()
    return res


def isycos_search(series, pairs, *, s_min: int, s_max: int, k: int = 4, sizes=None, noise: bool = True,
                  tau_ratio: float = 0.25, p: int = 3, sigma: float = 0.2, method: int = 3, delta_td: int = 0,
                  delta_bu: int = 0, t_max_idle: int = 3, h: int = 5, n_chunks: int = 1, lookahead: int = 0,
                  seed: int = 0, variant: int = 0, profile: bool = False, brute: bool = False,
                  unfused: bool = False, stream=None, capacity: int | None = None, auto_M: int = 0, auto_m: int = 0,
                  auto_alpha: float = 0.0, auto_rho: float = 0.0, profile_only: str | None = None,
                  chunks: tuple | None = None, no_block: bool = False, incremental: bool = False):
    """SYCOS search over series pairs.  Returns (results, stats).

    series: list of float32 arrays / tensors (host or CUDA, all alike, same length)
    pairs:  list of (xs, ys) or (xs, ys, id)
    results: list of tuples (pair, method, t0, t1, mi, h, nmi) sorted by (pair, method, t0)
    """
    bufs = [_Buf(s, np.float32, name=f"series[{i}]") for i, s in enumerate(series)]
    n = bufs[0].n
    if not all(b.n == n for b in bufs):
        raise ValueError("all series must have the same length")
    ptrs = (C.c_void_p * len(bufs))(*[b.ptr for b in bufs])
    pr = (Pair * max(1, len(pairs)))()
    for i, q in enumerate(pairs):
        pr[i].xs, pr[i].ys = int(q[0]), int(q[1])
        pr[i].id = int(q[2]) if len(q) > 2 else i
    sc = Scales()
    sc.s_min, sc.s_max = int(s_min), int(s_max)
    if sizes:
        arr = (C.c_int64 * len(sizes))(*[int(v) for v in sizes])
        sc.sizes = C.cast(arr, C.POINTER(C.c_int64))
        sc.n_sizes = len(sizes)
    nz = Noise()
    nz.enabled, nz.tau_ratio, nz.p = int(bool(noise)), float(tau_ratio), int(p)
    o = SearchOpts()
    o.sigma, o.method, o.variant = float(sigma), int(method), int(variant)
    o.delta_td, o.delta_bu, o.t_max_idle, o.h = int(delta_td), int(delta_bu), int(t_max_idle), int(h)
    o.n_chunks, o.lookahead, o.seed = int(n_chunks), int(lookahead), int(seed) & ((1 << 64) - 1)
    o.auto_M, o.auto_m, o.auto_alpha, o.auto_rho = int(auto_M), int(auto_m), float(auto_alpha), float(auto_rho)
    if chunks is not None:  # (pair, chunk) units: chunks [begin, end) of the plan, windows unmerged
        o.chunk_begin, o.chunk_end = int(chunks[0]), int(chunks[1])
    o.flags = ((F_PROFILE if profile else 0) | (F_BRUTE if brute else 0) | (F_UNFUSED if unfused else 0)
               | (F_NO_BLOCK if no_block else 0) | (F_INCREMENTAL if incremental else 0))
    if profile and profile_only:  # events around one path's launches only ("sorted" or "brute")
        o.flags |= F_PROFILE_SORTED_ONLY if profile_only == "sorted" else F_PROFILE_BRUTE_ONLY
    o.stream = _stream_ptr(stream)
    # results per pair and method are disjoint windows of >= s_min samples: at most n // s_min each.  The
    # buffer is np.empty (untouched pages cost nothing), so the bound never forces a second search.
    n_methods = 2 if int(method) in (3, 4) else 1
    if capacity is None:
        capacity = min(max(1, n_methods * len(pairs) * (n // max(1, int(s_min)))), 1 << 24)
    while True:
        outw = np.empty(max(1, capacity), dtype=RESULT_DTYPE)
        cnt = C.c_int64(0)
        st = SearchStats()
        rc = lib().isycos_search(C.cast(ptrs, C.c_void_p), len(bufs), n, pr, len(pairs), C.byref(sc), int(k),
                                 C.byref(nz), C.byref(o), outw.ctypes.data, capacity, C.byref(cnt),
                                 C.byref(st))
        if rc == E_TRUNC:  # only when the caller passed a smaller capacity
            capacity = int(cnt.value)
            continue
        _check(rc)
        break
    res = [tuple(r) for r in outw[:cnt.value].tolist()]
    return res, st.as_dict()


def isycos_merge_windows(results):
    """Alg. 4 chunk merge (reading R20) of gathered per-chunk result tuples; sorted by (pair, method, t0)."""
    arr = np.array([tuple(r) for r in results], dtype=RESULT_DTYPE) if len(results) else np.empty(0, RESULT_DTYPE)
    out = np.empty(max(1, len(arr)), dtype=RESULT_DTYPE)
    cnt = C.c_int64(0)
    _check(lib().isycos_merge_windows(arr.ctypes.data if len(arr) else None, len(arr), out.ctypes.data, len(arr),
                                      C.byref(cnt)))
    return [tuple(r) for r in out[:cnt.value].tolist()]


def search_workload(wl, *, series=None, pairs=None, **kw):
    """isycos_search with a datagen.Workload's search configuration (series may be device tensors)."""
    sc = wl.search
    args = dict(s_min=sc.s_min, s_max=sc.s_max, k=sc.k, sizes=list(sc.sizes) or None, noise=sc.noise,
                tau_ratio=sc.tau_ratio, p=sc.p, sigma=sc.sigma, method=sc.method, delta_td=sc.delta_td,
                delta_bu=sc.delta_bu, t_max_idle=sc.t_max_idle, h=sc.h, n_chunks=sc.n_chunks, seed=sc.seed,
                auto_M=sc.auto_M, auto_m=sc.auto_m, auto_alpha=sc.auto_alpha, auto_rho=sc.auto_rho)
    args.update(kw)
    return isycos_search(series if series is not None else wl.series,
                         pairs if pairs is not None else wl.pairs, **args)
