"""NEXT-3: the GPU analogue of the paper's incremental MI (IR/IMR).

Windows of one (pair, size) whose starts sit on a common grid share their beta-point blocks: every block
is sorted once per batch and each window's sorted layout is merged from its blocks (a delta-shifted window
reuses the sorted state of the blocks it shares with its neighbours).  The layouts are the same keys in the
same total order, so results must be bit-identical to the oracle and to the from-scratch sort.
"""
import numpy as np
import pytest

import datagen

pytestmark = pytest.mark.gpu
FIELDS = ("mi", "h", "nmi", "s_psi", "s_log", "zero_eps")


@pytest.fixture(scope="module")
def isy():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2204_09131_b200 import build

    build.build()
    import paper_2204_09131_b200 as isy

    return isy


def grid_windows(n, start, step, sizes, count):
    out = []
    for w in sizes:
        for i in range(count):
            t = start + i * step
            if t + w <= n:
                out.append((t, t + w))
    return np.asarray(out, np.int64)


@pytest.mark.parametrize("variant", [0, 1])
def test_block_merged_windows_bitwise(isy, orc, variant):
    wl = datagen.cfg3()
    x, y = wl.series
    x, y = x[:60_000], y[:60_000]
    # grids: step 256 from 37 (beta = 256: 2, 3, 4, 8 blocks), step 1024 from 5000 (XL 12,288 = 1.5 segments)
    W = np.concatenate([grid_windows(len(x), 37, 256, [512, 768, 1024, 2048], 5),
                        grid_windows(len(x), 5000, 1024, [4096, 12288], 3)])
    got = isy.isycos_mi_batch_ex(x, y, W, 4, variant=variant, unfused=True, debug=True)
    assert got["stats"]["block_windows"] == len(W) and got["stats"]["block_points"] > 0
    ref = orc.mi_batch(x, y, W, 4, variant=variant)
    for f in FIELDS:
        assert np.array_equal(np.asarray(got[f]), ref[f]), f
    scratch = isy.isycos_mi_batch_ex(x, y, W, 4, variant=variant, unfused=True, debug=True, no_block=True)
    assert scratch["stats"]["block_windows"] == 0
    for f in FIELDS + ("eps", "nx", "ny"):
        assert np.array_equal(np.asarray(got[f]), np.asarray(scratch[f])), f
    off = 0
    for j, (a, b) in enumerate(W):  # per point on a few windows
        if j % 9 == 0:
            o = orc.window(x[a:b], y[a:b], k=4, variant=variant)
            assert np.array_equal(got["eps"][off:off + b - a], o.eps)
            assert np.array_equal(got["nx"][off:off + b - a], o.nx)
            assert np.array_equal(got["ny"][off:off + b - a], o.ny)
        off += b - a


def test_block_merge_with_ties(isy, orc):
    """Integer-valued data (many equal x): ties are ordered by the sample index inside and across blocks."""
    st = datagen.Stream(9, 1)
    x = np.floor(st.uniform(20_000) * 16).astype(np.float32)
    y = np.floor(st.uniform(20_000) * 16).astype(np.float32)
    W = grid_windows(len(x), 3, 512, [1024, 1536, 2048], 6)
    got = isy.isycos_mi_batch_ex(x, y, W, 4, unfused=True)
    assert got["stats"]["block_windows"] == len(W)
    ref = orc.mi_batch(x, y, W, 4)
    for f in FIELDS:
        assert np.array_equal(np.asarray(got[f]), ref[f]), f


def test_search_block_mode_identical(isy):
    """A TD+BU search (configs[1]: layers 4,096 / 2,048 / 1,024 have delta >= 256) with and without shared
    blocks: identical windows and counters; the block path engaged."""
    wl = datagen.cfg2()
    a, sa = isy.search_workload(wl, unfused=True)
    b, sb = isy.search_workload(wl, unfused=True, no_block=True)
    assert a == b
    ka, kb = sa.pop("kernel"), sb.pop("kernel")
    assert sa == sb
    assert ka["block_windows"] > 0 and kb["block_windows"] == 0


def test_latency_split_kernel_small_windows(isy, orc):
    """Latency-mode small windows (classes of < 592 windows) run on the 8-lanes-per-point kernel (ksg_lat.cu):
    per-point eps / n_x / n_y and the records bitwise equal the oracle, ragged sizes and integer ties."""
    wl = datagen.cfg2()
    x, y = wl.series
    W = np.array([(100 + 300 * i, 100 + 300 * i + w) for i, w in enumerate([5, 6, 17, 31, 32, 33, 63, 64, 65, 97,
                                                                            128, 129, 200, 255, 256])], np.int64)
    got = isy.isycos_mi_batch_ex(x, y, W, 4, debug=True)
    ref = orc.mi_batch(x, y, W, 4)
    for f in FIELDS:
        assert np.array_equal(np.asarray(got[f]), ref[f]), f
    off = 0
    for a, b in W:
        o = orc.window(x[a:b], y[a:b], k=4)
        assert np.array_equal(got["eps"][off:off + b - a], o.eps) and np.array_equal(got["nx"][off:off + b - a], o.nx)
        assert np.array_equal(got["ny"][off:off + b - a], o.ny)
        off += b - a
    st = datagen.Stream(4, 2)
    xi = np.floor(st.uniform(4000) * 6).astype(np.float32)
    yi = np.floor(st.uniform(4000) * 6).astype(np.float32)
    W2 = np.array([(40 * i, 40 * i + 24 + 9 * i) for i in range(25)], np.int64)
    g2 = isy.isycos_mi_batch_ex(xi, yi, W2, 3)
    r2 = orc.mi_batch(xi, yi, W2, 3)
    for f in FIELDS:
        assert np.array_equal(np.asarray(g2[f]), r2[f]), f


@pytest.mark.parametrize("k", [1, 2, 4, 8])
def test_latency_split_kernel_merge_networks(isy, orc, k):
    """ksg_lat: self's 0 is dropped from the lane that scanned it and the 8 partial k-lists merge by bitonic
    networks (k = 4, 8) or insertions (other k).  Per-point outputs bitwise equal the oracle with integer ties and
    duplicated points, where the dropped 0 competes with other zero distances."""
    st = datagen.Stream(11, 5)
    n = 6000
    xs = {"int": (np.floor(st.uniform(n) * 5).astype(np.float32), np.floor(st.uniform(n) * 5).astype(np.float32)),
          "dup": (np.repeat(datagen.f32(st.normal(n // 3)), 3)[:n], np.repeat(datagen.f32(st.normal(n // 3)), 3)[:n]),
          "gauss": (datagen.f32(st.normal(n)), datagen.f32(st.normal(n)))}
    sizes = [w for w in (k + 1, 9, 16, 31, 33, 64, 100, 128, 200, 256) if w > k]
    W = np.array([(170 * i, 170 * i + w) for i, w in enumerate(sizes * 3)], np.int64)
    for name, (x, y) in xs.items():
        got = isy.isycos_mi_batch_ex(x, y, W, k, debug=True)
        ref = orc.mi_batch(x, y, W, k)
        for f in FIELDS:
            assert np.array_equal(np.asarray(got[f]), ref[f]), (name, f)
        off = 0
        for a, b in W:
            o = orc.window(x[a:b], y[a:b], k=k)
            for f, r in (("eps", o.eps), ("nx", o.nx), ("ny", o.ny)):
                assert np.array_equal(got[f][off:off + b - a], r), (name, f, a, b)
            off += b - a


@pytest.mark.parametrize("variant", [0, 1])
def test_incremental_radii_chains(isy, orc, variant):
    """NEXT-3 incremental radii (IR): windows that follow their predecessor by one 512-block (w = 4,096
    and 16,384, as in the configs[2] sweep) reuse the predecessor's eps where the removed / inserted block cannot
    change it.  Records and per-point outputs equal the from-scratch scan and the oracle (sampled windows)."""
    wl = datagen.cfg3()
    x, y = wl.series
    x, y = x[200_000:260_000], y[200_000:260_000]
    W = np.concatenate([grid_windows(len(x), 0, 512, [4096], 40), grid_windows(len(x), 1024, 512, [16384], 20)])
    got = isy.isycos_mi_batch_ex(x, y, W, 4, variant=variant, unfused=True, debug=True, incremental=True)
    st = got["stats"]
    if variant == 0:  # KSG-2 windows are scanned from scratch (its kNN thresholds are not carried)
        assert st["inc_windows"] > 0 and st["eps_reused_points"] > 0.5 * st["inc_windows"] * 4096
    ref = isy.isycos_mi_batch_ex(x, y, W, 4, variant=variant, unfused=True, debug=True)
    assert ref["stats"]["inc_windows"] == 0
    for f in FIELDS + ("eps", "nx", "ny"):
        assert np.array_equal(np.asarray(got[f]), np.asarray(ref[f])), f
    sel = [0, 1, 17, 39, 41, 59]
    o = orc.mi_batch(x, y, W[sel], 4, variant=variant)
    for f in FIELDS:
        assert np.array_equal(np.asarray(got[f])[sel], o[f]), f


def test_incremental_radii_ties(isy, orc):
    """Integer data: radii with many ties; a removed point at distance exactly eps forces a rescan."""
    st = datagen.Stream(12, 1)
    x = np.floor(st.uniform(30_000) * 24).astype(np.float32)
    y = np.floor(st.uniform(30_000) * 24).astype(np.float32)
    W = grid_windows(len(x), 100, 256, [2048, 4096], 30)
    got = isy.isycos_mi_batch_ex(x, y, W, 3, unfused=True, debug=True, incremental=True)
    assert got["stats"]["inc_windows"] > 0
    ref = orc.mi_batch(x, y, W, 3)
    for f in FIELDS:
        assert np.array_equal(np.asarray(got[f]), ref[f]), f
    scratch = isy.isycos_mi_batch_ex(x, y, W, 3, unfused=True, debug=True, no_block=True)
    for f in ("eps", "nx", "ny"):
        assert np.array_equal(got[f], scratch[f]), f
