"""Build/load the CPU driver harness (tests only): product search driver + oracle-backed stub engine."""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
SRCS = [os.path.join(HERE, "driver_harness.cpp"),
        os.path.join(ROOT, "paper_2204_09131_b200", "csrc", "search.cpp"),
        os.path.join(ROOT, "oracle", "oracle.cpp")]
LIB = os.path.join(HERE, "libdriverharness.so")


def build():
    deps = SRCS + [os.path.join(ROOT, "paper_2204_09131_b200", "csrc", "engine.h"),
                   os.path.join(ROOT, "include", "isycos.h")]
    if os.path.exists(LIB) and all(os.path.getmtime(LIB) >= os.path.getmtime(f) for f in deps):
        return LIB
    tmp = LIB + f".tmp{os.getpid()}"
    subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared", "-fPIC",
                           "-I", os.path.join(ROOT, "include"), "-I",
                           os.path.join(ROOT, "paper_2204_09131_b200", "csrc"), "-I", "/usr/local/cuda/include",
                           "-o", tmp, *SRCS])
    os.replace(tmp, LIB)
    return LIB


class HarnessParams(C.Structure):
    _fields_ = [(f, C.c_int32) for f in ("k", "method", "noise", "p", "h", "t_max_idle", "n_chunks", "lookahead",
                                         "bu_depth", "anchor", "spec_cap", "trend", "pipeline", "ring_rank")] + \
               [("s_min", C.c_int64), ("s_max", C.c_int64), ("delta_td", C.c_int64), ("delta_bu", C.c_int64),
                ("sigma", C.c_double), ("tau_ratio", C.c_double), ("seed", C.c_uint64),
                ("sizes", C.POINTER(C.c_int64)), ("n_sizes", C.c_int64), ("auto_M", C.c_int32), ("auto_m", C.c_int32),
                ("auto_alpha", C.c_double), ("auto_rho", C.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        from paper_2204_09131_b200._capi import ResultWindow, SearchStats

        _lib.harness_use_cache.argtypes = [C.c_int]
        _lib.harness_parallel.argtypes = [C.c_int]
        _lib.harness_search.argtypes = [C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.POINTER(HarnessParams),
                                        C.POINTER(ResultWindow), C.c_int64, C.POINTER(C.c_int64),
                                        C.POINTER(SearchStats), C.POINTER(C.c_double), C.POINTER(C.c_int64)]
    return _lib


def search(series, pairs, sc, **kw):
    """The product driver on CPU (oracle-evaluated windows).  Returns (results, stats, eval_ms, evaluated)."""
    from paper_2204_09131_b200._capi import ResultWindow, SearchStats

    arrs = [np.ascontiguousarray(s, np.float32) for s in series]
    ptrs = (C.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
    pr = []
    for i, p in enumerate(pairs):
        pr += [p[0], p[1], p[2] if len(p) > 2 else i]
    P3 = np.asarray(pr, np.int32)
    hp = HarnessParams()
    d = dict(k=sc.k, method=sc.method, noise=int(sc.noise), p=sc.p, h=sc.h, t_max_idle=sc.t_max_idle,
             n_chunks=sc.n_chunks, lookahead=0, bu_depth=0, anchor=-1, spec_cap=-1, trend=-1, pipeline=-1, ring_rank=0, s_min=sc.s_min, s_max=sc.s_max,
             delta_td=sc.delta_td, delta_bu=sc.delta_bu, sigma=sc.sigma, tau_ratio=sc.tau_ratio, seed=sc.seed,
             auto_M=sc.auto_M, auto_m=sc.auto_m, auto_alpha=sc.auto_alpha, auto_rho=sc.auto_rho)
    d.update(kw)
    for key, v in d.items():
        setattr(hp, key, v)
    sizes = list(sc.sizes or [])
    arr = (C.c_int64 * max(1, len(sizes)))(*sizes)
    if sizes:
        hp.sizes = C.cast(arr, C.POINTER(C.c_int64))
        hp.n_sizes = len(sizes)
    cap = 1 << 15
    out = (ResultWindow * cap)()
    cnt = C.c_int64(0)
    st = SearchStats()
    ems = C.c_double(0)
    ev = C.c_int64(0)
    rc = lib().harness_search(C.cast(ptrs, C.c_void_p), len(arrs[0]), P3.ctypes.data, len(pairs), C.byref(hp),
                              out, cap, C.byref(cnt), C.byref(st), C.byref(ems), C.byref(ev))
    assert rc == 0, rc
    res = [(r.pair, r.method, r.t0, r.t1, r.mi, r.h, r.nmi) for r in out[:cnt.value]]
    return res, st.as_dict(), ems.value, ev.value
