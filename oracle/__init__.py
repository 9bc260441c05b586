"""ctypes loader for the ORACLE (oracle/oracle.cpp) — TEST INFRASTRUCTURE ONLY.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_2204_09131_b200``) never imports it: it has no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import hashlib
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
CXXFLAGS = ["-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-shared", "-fPIC", "-pthread"]


def _digest() -> str:  # content hash of the source and flags (an mtime can lie after a copy)
    with open(_SRC, "rb") as fh:
        return hashlib.sha256(fh.read() + " ".join(CXXFLAGS).encode()).hexdigest()


def build(force: bool = False) -> str:
    stamp = _LIB + ".sha256"
    fresh = os.path.exists(_LIB) and os.path.exists(stamp) and open(stamp).read().strip() == _digest()
    if force or not fresh:
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", *CXXFLAGS, "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
        with open(stamp, "w") as fh:
            fh.write(_digest() + "\n")
    return _LIB


class OParams(C.Structure):
    _fields_ = [
        ("k", C.c_int32), ("variant", C.c_int32), ("method", C.c_int32), ("noise", C.c_int32),
        ("p", C.c_int32), ("h", C.c_int32), ("t_max_idle", C.c_int32), ("n_chunks", C.c_int32),
        ("s_min", C.c_int64), ("s_max", C.c_int64), ("delta_td", C.c_int64), ("delta_bu", C.c_int64),
        ("sigma", C.c_double), ("tau_ratio", C.c_double), ("seed", C.c_uint64),
        ("sizes", C.POINTER(C.c_int64)), ("n_sizes", C.c_int32), ("_pad", C.c_int32),
        ("auto_M", C.c_int32), ("auto_m", C.c_int32), ("auto_alpha", C.c_double), ("auto_rho", C.c_double),
        ("chunk_begin", C.c_int32), ("chunk_end", C.c_int32),
    ]


class OResult(C.Structure):
    _fields_ = [("pair", C.c_int32), ("method", C.c_int32), ("t0", C.c_int64), ("t1", C.c_int64),
                ("mi", C.c_double), ("h", C.c_double), ("nmi", C.c_double)]


STAT_FIELDS = ["td_windows", "td_noise_checks", "td_skips", "td_accepted", "bu_climbs",
               "bu_iterations", "bu_neighbors", "bu_noise_checks", "bu_prunes", "bu_accepted",
               "distinct_windows", "distinct_pairs", "eval_cost", "auto_td", "auto_bu"]
STAT_FIELDS_F = ["auto_nscore_td", "auto_nscore_bu"]


class OStats(C.Structure):
    _fields_ = [(f, C.c_int64) for f in STAT_FIELDS] + [(f, C.c_double) for f in STAT_FIELDS_F]


MIFN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_double),
                   C.POINTER(C.c_double), C.POINTER(C.c_double))
DRAWFN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int64, C.c_int64)

_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        L = _lib
        L.oracle_ln.restype = C.c_double
        L.oracle_ln.argtypes = [C.c_double]
        L.oracle_q32.restype = C.c_int64
        L.oracle_q32.argtypes = [C.c_double]
        L.oracle_psi.argtypes = [C.c_int64, C.c_void_p]
        L.oracle_window.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.oracle_mi_batch.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int32,
                                      C.c_int32] + [C.c_void_p] * 6
        L.oracle_search.argtypes = [C.c_void_p, C.c_int32, C.c_int64, C.c_void_p, C.c_int32,
                                    C.POINTER(OParams), C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                    C.POINTER(OStats)]
        L.oracle_search_mock.argtypes = [MIFN, C.c_void_p, C.c_int64, C.POINTER(OParams), C.c_void_p,
                                         C.c_int64, C.POINTER(C.c_int64), C.POINTER(OStats)]
        L.oracle_search_mock_draws.argtypes = [MIFN, DRAWFN, C.c_void_p, C.c_int64, C.POINTER(OParams),
                                               C.c_void_p, C.c_int64, C.POINTER(C.c_int64), C.POINTER(OStats)]
        L.oracle_point.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int64, C.c_int32, C.c_int32,
                                   C.c_void_p, C.c_void_p]
        L.oracle_point_psi_q.restype = C.c_int64
        L.oracle_point_psi_q.argtypes = [C.c_int32, C.c_int32, C.c_int32]
        L.oracle_point_log_q.restype = C.c_int64
        L.oracle_point_log_q.argtypes = [C.c_float]
        L.oracle_finish.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_void_p]
        L.oracle_chunk_plan.argtypes = [C.c_int64, C.c_int32, C.c_int64, C.c_void_p, C.c_int32]
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def psi_table(m_max: int) -> np.ndarray:
    out = np.zeros(m_max + 1, np.float64)
    assert lib().oracle_psi(m_max, _p(out)) == 0
    return out


def ln(v: float) -> float:
    return lib().oracle_ln(float(v))


def q32(v: float) -> int:
    return lib().oracle_q32(float(v))


@dataclass
class WindowOut:
    mi: float
    h: float
    nmi: float
    mi_plain: float
    h_plain: float
    s_psi: int
    s_log: int
    zero_eps: int
    eps: np.ndarray
    nx: np.ndarray
    ny: np.ndarray


def window(x, y, k: int = 4, variant: int = 0, eps_method: int = 0) -> WindowOut:
    """KSG estimate of one window (the arrays ARE the window)."""
    x = np.ascontiguousarray(x, np.float32)
    y = np.ascontiguousarray(y, np.float32)
    w = len(x)
    o6 = np.zeros(5, np.float64)
    o3 = np.zeros(3, np.int64)
    eps = np.zeros(w, np.float32)
    nx = np.zeros(w, np.int32)
    ny = np.zeros(w, np.int32)
    rc = lib().oracle_window(_p(x), _p(y), w, k, variant, eps_method, _p(o6), _p(o3), _p(eps), _p(nx), _p(ny))
    if rc != 0:
        raise ValueError(f"oracle_window rc={rc}")
    return WindowOut(o6[0], o6[1], o6[2], o6[3], o6[4], int(o3[0]), int(o3[1]), int(o3[2]), eps, nx, ny)


def mi_batch(x, y, windows, k: int = 4, variant: int = 0):
    """Records for windows [t0,t1) of series (x,y): dict of arrays mi, h, nmi, s_psi, s_log, zero_eps."""
    x = np.ascontiguousarray(x, np.float32)
    y = np.ascontiguousarray(y, np.float32)
    W = np.ascontiguousarray(np.asarray(windows, np.int64).reshape(-1, 2))
    nw = len(W)
    out = {"mi": np.zeros(nw), "h": np.zeros(nw), "nmi": np.zeros(nw),
           "s_psi": np.zeros(nw, np.int64), "s_log": np.zeros(nw, np.int64),
           "zero_eps": np.zeros(nw, np.int32)}
    rc = lib().oracle_mi_batch(_p(x), _p(y), len(x), _p(W), nw, k, variant, _p(out["mi"]), _p(out["h"]),
                               _p(out["nmi"]), _p(out["s_psi"]), _p(out["s_log"]), _p(out["zero_eps"]))
    if rc != 0:
        raise ValueError(f"oracle_mi_batch rc={rc}")
    return out


def make_params(sc=None, **kw) -> OParams:
    d = dict(k=4, variant=0, method=3, noise=1, p=3, h=5, t_max_idle=3, n_chunks=1, s_min=64,
             s_max=512, delta_td=0, delta_bu=0, sigma=0.2, tau_ratio=0.25, seed=0, sizes=None,
             auto_M=0, auto_m=0, auto_alpha=0.0, auto_rho=0.0, chunk_begin=0, chunk_end=0)
    if sc is not None:
        d.update(k=sc.k, method=sc.method, noise=int(sc.noise), p=sc.p, h=sc.h, t_max_idle=sc.t_max_idle,
                 n_chunks=sc.n_chunks, s_min=sc.s_min, s_max=sc.s_max, delta_td=sc.delta_td,
                 delta_bu=sc.delta_bu, sigma=sc.sigma, tau_ratio=sc.tau_ratio, seed=sc.seed,
                 sizes=list(sc.sizes) or None, auto_M=sc.auto_M, auto_m=sc.auto_m, auto_alpha=sc.auto_alpha,
                 auto_rho=sc.auto_rho)
    d.update(kw)
    P = OParams()
    sizes = d.pop("sizes")
    for key, v in d.items():
        setattr(P, key, v)
    if sizes:
        arr = (C.c_int64 * len(sizes))(*sizes)
        P.sizes = C.cast(arr, C.POINTER(C.c_int64))
        P.n_sizes = len(sizes)
        P._keep = arr  # keep alive
    return P


def _results(buf, count):
    return [(r.pair, r.method, r.t0, r.t1, r.mi, r.h, r.nmi) for r in buf[:count]]


def search(series, pairs, params: OParams, cap: int = 1 << 16):
    """Full oracle search.  pairs: list of (xs, ys) or (xs, ys, id).  Returns (results, stats)."""
    arrs = [np.ascontiguousarray(s, np.float32) for s in series]
    n = len(arrs[0])
    ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    pr = []
    for i, p in enumerate(pairs):
        pr += [p[0], p[1], p[2] if len(p) > 2 else i]
    P3 = np.asarray(pr, np.int32)
    out = (OResult * cap)()
    count = C.c_int64(0)
    st = OStats()
    rc = lib().oracle_search(C.cast(ptrs, C.c_void_p), len(arrs), n, _p(P3), len(pairs), C.byref(params),
                             C.cast(out, C.c_void_p), cap, C.byref(count), C.byref(st))
    if rc != 0:
        raise ValueError(f"oracle_search rc={rc}")
    return _results(out, count.value), {f: getattr(st, f) for f in STAT_FIELDS + STAT_FIELDS_F}


def search_mock(fn, n: int, params: OParams, cap: int = 1 << 14):
    """Search one pair of length n with a Python MI provider fn(t0, t1) -> (mi, h, nmi)."""
    calls = []

    def cb(ctx, t0, t1, mi, h, nmi):
        calls.append((t0, t1))
        a, b, c = fn(t0, t1)
        mi[0], h[0], nmi[0] = a, b, c
        return 0

    cfn = MIFN(cb)
    out = (OResult * cap)()
    count = C.c_int64(0)
    st = OStats()
    rc = lib().oracle_search_mock(cfn, None, n, C.byref(params), C.cast(out, C.c_void_p), cap,
                                  C.byref(count), C.byref(st))
    if rc != 0:
        raise ValueError(f"oracle_search_mock rc={rc}")
    return _results(out, count.value), {f: getattr(st, f) for f in STAT_FIELDS + STAT_FIELDS_F}, calls


def search_mock_draws(fn, draws, n: int, params: OParams, cap: int = 1 << 14):
    """search_mock with the LAHC history-index draws (Alg. 2 line 11) passed in as inputs: draws is a
    dict {climb start lo: [r_0, r_1, ...]} (one entry per iteration with a non-empty neighbourhood) or a
    list used for every climb.  Asking for a draw beyond the list aborts the search (ValueError)."""
    calls = []
    asked = []

    def cb(ctx, t0, t1, mi, h, nmi):
        calls.append((t0, t1))
        a, b, c = fn(t0, t1)
        mi[0], h[0], nmi[0] = a, b, c
        return 0

    def dcb(ctx, lo, it):
        asked.append((lo, it))
        seq = draws.get(lo, []) if isinstance(draws, dict) else draws
        return seq[it] if it < len(seq) else -1

    cfn, dfn = MIFN(cb), DRAWFN(dcb)
    out = (OResult * cap)()
    count = C.c_int64(0)
    st = OStats()
    rc = lib().oracle_search_mock_draws(cfn, dfn, None, n, C.byref(params), C.cast(out, C.c_void_p), cap,
                                        C.byref(count), C.byref(st))
    if rc != 0:
        raise ValueError(f"oracle_search_mock_draws rc={rc} (draws asked: {asked[-3:]})")
    return _results(out, count.value), {f: getattr(st, f) for f in STAT_FIELDS + STAT_FIELDS_F}, calls


def point(x, y, i: int, k: int = 4, variant: int = 0):
    """(eps_i, n_x(i), n_y(i)) of point i of the window (x, y)."""
    x = np.ascontiguousarray(x, np.float32)
    y = np.ascontiguousarray(y, np.float32)
    e = np.zeros(1, np.float32)
    nn = np.zeros(2, np.int32)
    rc = lib().oracle_point(_p(x), _p(y), len(x), int(i), k, variant, _p(e), _p(nn))
    if rc != 0:
        raise ValueError(f"oracle_point rc={rc}")
    return float(e[0]), int(nn[0]), int(nn[1])


def point_terms(nx: int, ny: int, eps: float, variant: int = 0):
    """Canonical per-point terms (q(psi) pair sum, q(LN(2 eps)) or 0)."""
    return lib().oracle_point_psi_q(int(nx), int(ny), variant), lib().oracle_point_log_q(float(eps))


def finish(s_psi: int, s_log: int, zeros: int, w: int, k: int = 4, variant: int = 0):
    """(mi, h, nmi) from the canonical sums (the window finish of §8(c).3)."""
    o = np.zeros(3)
    lib().oracle_finish(int(s_psi), int(s_log), int(zeros), int(w), k, variant, _p(o))
    return float(o[0]), float(o[1]), float(o[2])


def chunk_plan(n: int, n_p: int, s_max: int):
    out = np.zeros(2 * max(n_p, 1), np.int64)
    c = lib().oracle_chunk_plan(n, n_p, s_max, _p(out), n_p)
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(c)]


def auto_scores(cost_td: int, cost_bu: int, m: int, nL_td: int, nS_bu: int, alpha: float = 0.5):
    """Eqs. 6-9 (iSYCOS, Alg. 3): returns (chosen method 1 TD / 2 BU, nscore_TD, nscore_BU)."""
    L = lib()
    L.oracle_auto_scores.argtypes = [C.c_int64, C.c_int64, C.c_int32, C.c_int64, C.c_int64, C.c_double,
                                     C.POINTER(C.c_double)]
    out = (C.c_double * 2)()
    rc = L.oracle_auto_scores(int(cost_td), int(cost_bu), int(m), int(nL_td), int(nS_bu), float(alpha), out)
    if rc < 0:
        raise ValueError("oracle_auto_scores")
    return rc, out[0], out[1]


def auto_sample(M: int, m: int, seed: int, pair_id: int):
    """Alg. 3 line 1: the m partition indices sampled from M for a pair."""
    L = lib()
    L.oracle_auto_sample.argtypes = [C.c_int32, C.c_int32, C.c_uint64, C.c_int32, C.POINTER(C.c_int32)]
    out = (C.c_int32 * max(1, m))()
    if L.oracle_auto_sample(M, m, seed & ((1 << 64) - 1), pair_id, out) != 0:
        raise ValueError("oracle_auto_sample")
    return list(out[:m])
