"""CPU-side checks of the C ABI: the library loads, exports every symbol include/isycos.h declares,
and rejects bad arguments before touching the GPU.  No compute calls (no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def capi():
    from paper_2204_09131_b200 import build

    build.build()
    from paper_2204_09131_b200 import _capi

    _capi.lib()
    return _capi


def header_functions():
    src = open(os.path.join(ROOT, "include", "isycos.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(isycos_[a-z_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    fns = header_functions()
    assert "isycos_mi_batch" in fns and "isycos_search" in fns


def test_library_exports_every_declared_symbol(capi):
    fns = header_functions()
    for f in fns:
        assert hasattr(capi.lib(), f), f
    out = subprocess.check_output(["nm", "-D", "--defined-only", capi.LIB_PATH], text=True)
    exported = set(re.findall(r" T (isycos_\w+)", out))
    assert set(fns) <= exported
    assert set(capi.EXPORTS) == set(fns)


def test_library_is_sm100a_only(capi):
    out = subprocess.check_output(["cuobjdump", "--list-elf", capi.LIB_PATH], text=True)
    assert "sm_100a" in out


def test_kernels_use_bulk_copy(capi):
    sass = subprocess.check_output(["cuobjdump", "-sass", capi.LIB_PATH], text=True)
    assert "UBLKCP" in sass  # cp.async.bulk (TMA engine) staging in the tile kernel
    assert "HMMA" not in sass and "UTCHMMA" not in sass  # no tensor cores: compare/count work


def test_abi_version(capi):
    assert capi.isycos_abi_version() == 3


def test_validation_before_gpu(capi):
    L = capi.lib()
    x = np.zeros(16, np.float32)
    w = np.array([[0, 8]], np.int64)
    out = np.zeros(1)
    p = lambda a: a.ctypes.data
    assert L.isycos_mi_batch(None, p(x), 16, p(w), 1, 4, p(out)) == capi.E_INVAL
    assert L.isycos_mi_batch(p(x), p(x), 1, p(w), 1, 4, p(out)) == capi.E_INVAL
    assert L.isycos_mi_batch(p(x), p(x), 16, p(w), 1, 0, p(out)) == capi.E_INVAL
    assert L.isycos_mi_batch(p(x), p(x), 16, p(w), 1, 17, p(out)) == capi.E_INVAL
    assert "k must be" in capi.isycos_last_error()
    assert L.isycos_mi_batch(p(x), p(x), 16, p(w), 0, 4, p(out)) == capi.ISYCOS_OK
    o = capi.MiOpts()
    o.variant = 2  # 0 = KSG-1, 1 = KSG-2; nothing else
    assert L.isycos_mi_batch_ex(p(x), p(x), 16, p(w), 1, 4, C.byref(o), p(out)) == capi.E_INVAL
    assert "variant" in capi.isycos_last_error()


def test_search_param_validation(capi):
    x = np.zeros(256, np.float32)
    bad = [dict(s_min=1, s_max=64), dict(s_min=64, s_max=32), dict(s_min=8, s_max=64, k=8),
           dict(s_min=16, s_max=512), dict(s_min=16, s_max=64, sigma=0.0), dict(s_min=16, s_max=64, tau_ratio=1.0),
           dict(s_min=16, s_max=64, method=4), dict(s_min=16, s_max=64, h=0), dict(s_min=16, s_max=64, n_chunks=0),
           dict(s_min=16, s_max=64, sizes=[64, 64])]
    for kw in bad:
        with pytest.raises(capi.IsycosError) as ei:
            capi.isycos_search([x, x], [(0, 1)], **kw)
        assert ei.value.code == capi.E_INVAL, kw


def test_product_path_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2204_09131_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"\boracle\b\s*(import|\.)|import\s+oracle|from\s+oracle", src), f
                assert "oracle.cpp" not in src and "liboracle" not in src, f


def test_merge_windows_rule(capi):
    """isycos_merge_windows (Alg. 4 chunk merge, reading R20): per (pair, method), greedy by (nmi desc,
    mi desc, t0 asc, t1 asc), keep if disjoint; host logic, no GPU needed."""
    R = [(0, 1, 32, 96, 1.0, 2.0, 0.9), (0, 1, 36, 100, 5.0, 9.0, 0.5),   # higher nmi wins
         (0, 2, 32, 96, 2.0, 2.0, 1.0), (0, 2, 36, 100, 3.0, 3.0, 1.0),   # nmi tie: higher mi
         (1, 1, 36, 100, 2.0, 2.0, 1.0), (1, 1, 32, 96, 2.0, 2.0, 1.0),   # full tie: smaller t0
         (1, 1, 100, 164, 0.5, 1.0, 0.3), (1, 1, 10, 20, 0.1, 1.0, 0.2)]  # disjoint ones kept
    got = capi.isycos_merge_windows(R)
    assert [(r[0], r[1], r[2], r[3]) for r in got] == [(0, 1, 32, 96), (0, 2, 36, 100), (1, 1, 10, 20),
                                                        (1, 1, 32, 96), (1, 1, 100, 164)]
    assert capi.isycos_merge_windows([]) == []


def test_chunk_selection_validation(capi):
    x = np.zeros(256, np.float32)
    for kw in (dict(chunks=(0, 3)), dict(chunks=(1, 1)), dict(chunks=(-1, 1)), dict(chunks=(0, 1), method=4)):
        with pytest.raises(capi.IsycosError) as ei:
            capi.isycos_search([x, x], [(0, 1)], s_min=16, s_max=64, n_chunks=2, **kw)
        assert ei.value.code == capi.E_INVAL, kw


def test_binding_rejects_mismatched_buffers(capi):
    x = np.zeros(64, np.float32)
    w = np.array([[0, 32]], np.int64)
    with pytest.raises(TypeError):   # an output buffer of the wrong dtype would be written past its end
        capi.isycos_mi_batch_ex(x, x, w, 4, out={"mi": np.zeros(1, np.float32)})
    with pytest.raises(ValueError):
        capi.isycos_mi_batch_ex(x, x, w, 4, out={"mi": np.zeros(0)})
    with pytest.raises(ValueError):
        capi.isycos_mi_batch_ex(x, np.zeros(63, np.float32), w, 4)
