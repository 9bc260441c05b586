"""GPU parity of the KSG window kernels against the oracle (run on a B200: pytest -m gpu).

Bar (north star): per-point eps_i, n_x(i), n_y(i) bit-exact; per-window MI within 1e-9 of the
oracle — here bit-exact, because both sides implement the canonical int64 fixed-point sums and
the fixed fp64 finish (DESIGN.md §Canonical numerics).  Every comparison below is `==`.
"""
import math

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


def assert_records_equal(got, ref, label=""):
    for f in FIELDS:
        g = np.asarray(got[f])
        r = np.asarray(ref[f])
        if f in ("mi", "h", "nmi"):
            same = (g == r) | (np.isinf(g) & np.isinf(r) & (np.sign(g) == np.sign(r)))
        else:
            same = g == r
        bad = np.flatnonzero(~same)
        assert bad.size == 0, f"{label} field {f}: {bad.size} mismatches, first {bad[:5]}: {g[bad[:5]]} vs {r[bad[:5]]}"
    assert np.max(np.abs(np.asarray(got["mi"]) - np.asarray(ref["mi"]))) <= 1e-9


def check_windows(isy, orc, x, y, W, k, debug=False, label="", variant=0, brute=False, unfused=False):
    W = np.asarray(W, np.int64).reshape(-1, 2)
    got = isy.isycos_mi_batch_ex(x, y, W, k, debug=debug, variant=variant, brute=brute, unfused=unfused)
    ref = orc.mi_batch(x, y, W, k, variant=variant)
    assert_records_equal(got, ref, label)
    if debug:
        off = 0
        for (a, b) in W:
            o = orc.window(x[a:b], y[a:b], k=k, variant=variant)
            w = b - a
            assert np.array_equal(got["eps"][off:off + w], o.eps), f"{label} eps [{a},{b})"
            assert np.array_equal(got["nx"][off:off + w], o.nx), f"{label} nx [{a},{b})"
            assert np.array_equal(got["ny"][off:off + w], o.ny), f"{label} ny [{a},{b})"
            off += w
    return got


def test_cfg1_sweep_bitwise(isy, orc):
    wl = datagen.cfg1()
    x, y = wl.series
    W = datagen.sweep_windows(len(x), wl.sweep["sizes"], wl.sweep["stride"])
    assert len(W) == 908
    check_windows(isy, orc, x, y, W, 4, label="cfg1 sweep")


def test_debug_points_bitwise(isy, orc):
    wl = datagen.cfg1()
    x, y = wl.series
    W = [(0, 64), (3, 100), (500, 756), (1201, 1713), (1, 1300)]
    check_windows(isy, orc, x, y, W, 4, debug=True, label="debug")


# size classes: warp R=1,2,4,8 (w<=256), tile R=2 (<=512), tile R=4 multi i-tile (>1024),
# multi j-tile (> 4096 = kTileJ), ragged tails everywhere, misaligned t0, array ends.
SIZES = [5, 17, 32, 33, 64, 65, 100, 128, 129, 255, 256, 257, 300, 512, 513, 777, 1024, 1025, 2047,
         4096, 4097, 5003, 8191]


@pytest.mark.parametrize("k", [1, 3, 4, 8, 16])
@pytest.mark.parametrize("path", ["default", "unfused", "brute"])
def test_size_classes_random_windows(isy, orc, k, path):
    """Every kernel family: warp brute force (w <= 64), warp-sorted (65..256), fused / throughput sorted
    (257..4096; 'unfused' forces the throughput form), XL runs + merge; 'brute' forces the brute force."""
    wl = datagen.cfg2(n=20_000)
    x, y = wl.series
    rng = np.random.default_rng(k)
    W = []
    for w in SIZES:
        if w <= k:
            continue
        t0 = int(rng.integers(0, len(x) - w))
        W.append((t0, t0 + w))
    n = len(x)
    W += [(0, 37), (n - 41, n), (n - 4100, n), (1, 1 + 4099), (2, 2 + 515), (3, 3 + 130)]
    W = [(a, b) for (a, b) in W if b - a > k]
    check_windows(isy, orc, x, y, W, k, debug=(k == 4), label=f"k={k} {path}", unfused=path == "unfused",
                  brute=path == "brute")


def test_tie_torture(isy, orc):
    st = datagen.Stream(99, 1)
    n = 6000
    xi = np.floor(st.uniform(n) * 8).astype(np.float32)       # integer values 0..7
    yi = np.floor(st.uniform(n) * 8).astype(np.float32)
    xc = xi.copy()
    yc = yi.copy()
    xc[1000:1400] = 3.0                                        # constant segment (eps = 0, degenerate)
    yc[1000:1400] = -2.0
    xd = np.repeat(datagen.f32(st.normal(n // 4)), 4)[:n]      # every point duplicated 4x
    yd = np.repeat(datagen.f32(st.normal(n // 4)), 4)[:n]
    W = [(0, 64), (10, 300), (100, 1100), (0, 4500), (1000, 1400), (990, 1500), (1100, 1200), (1, 5000)]
    for k in (1, 4, 8):
        for uf in (False, True):
            check_windows(isy, orc, xi, yi, W, k, debug=(k == 4), label=f"int k={k} uf={uf}", unfused=uf)
            check_windows(isy, orc, xc, yc, W, k, label=f"const k={k} uf={uf}", unfused=uf)
            check_windows(isy, orc, xd, yd, W, k, debug=(k == 4), label=f"dup k={k} uf={uf}", unfused=uf)


def test_extreme_magnitudes(isy, orc):
    st = datagen.Stream(5, 1)
    n = 3000
    base = st.normal(n)
    for scale in (1e-30, 1e-6, 1e6, 1e30):
        x = datagen.f32(base * scale)
        y = datagen.f32(st.normal(n) * scale)
        check_windows(isy, orc, x, y, [(0, 200), (7, 1500), (100, 2999)], 4, label=f"scale {scale}")
    # subnormal differences
    x = (np.arange(n, dtype=np.float32) * np.float32(1e-44)).astype(np.float32)
    y = datagen.f32(st.normal(n))
    check_windows(isy, orc, x, y, [(0, 300), (5, 1200)], 4, label="subnormal")


def test_device_tensors_and_outputs(isy, orc):
    import torch

    wl = datagen.cfg1()
    x, y = wl.series
    W = datagen.sweep_windows(len(x), [64, 512], 64)
    ref = orc.mi_batch(x, y, W, 4)
    dx, dy = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    dW = torch.from_numpy(W).cuda()
    out = {"mi": torch.empty(len(W), dtype=torch.float64, device="cuda"),
           "nmi": torch.empty(len(W), dtype=torch.float64, device="cuda")}
    got = isy.isycos_mi_batch_ex(dx, dy, dW, 4, outputs=("mi", "nmi"), out=out,
                                 stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    assert np.array_equal(out["mi"].cpu().numpy(), ref["mi"])
    assert np.array_equal(out["nmi"].cpu().numpy(), ref["nmi"])
    # misaligned device view (offset 1 float): the library re-stages it
    W2 = W[W[:, 1] < len(x) - 1]
    got2 = isy.isycos_mi_batch(dx[1:], dy[1:], W2, 4)
    ref2 = orc.mi_batch(x[1:], y[1:], W2, 4)
    assert np.array_equal(got2, ref2["mi"])


def test_errors(isy):
    x = np.zeros(100, np.float32)
    y = np.zeros(100, np.float32)
    with pytest.raises(isy.IsycosError) as e:
        isy.isycos_mi_batch(x, y, [(0, 4)], 4)
    assert e.value.code == -3  # w <= k
    with pytest.raises(isy.IsycosError) as e:
        isy.isycos_mi_batch(x, y, [(90, 101)], 4)
    assert e.value.code == -2
    bad = x.copy()
    bad[50] = np.nan
    with pytest.raises(isy.IsycosError) as e:
        isy.isycos_mi_batch(bad, y, [(0, 64)], 4)
    assert e.value.code == -1
    bad[50] = np.inf
    with pytest.raises(isy.IsycosError):
        isy.isycos_mi_batch(x, bad, [(0, 64)], 4)


def test_sorted_path_segment_boundaries(isy, orc):
    """Windows at the sorted path's segment boundary (8,192 = one SMEM sort; 8,193+ = runs + rank merge),
    with heavy x ties (integer-rounded x) so the run merge must order equal keys consistently."""
    wl = datagen.cfg2(n=60_000)
    x, y = wl.series
    xr = np.round(x * 2).astype(np.float32)
    W = [(100, 100 + 16384), (7, 7 + 16385), (30_001, 30_001 + 20_001), (50, 50 + 8192), (3, 3 + 8193)]
    check_windows(isy, orc, x, y, W, 4, debug=True, label="segments")
    check_windows(isy, orc, xr, y, W[1:], 3, debug=True, label="segments ties")


def test_large_window_sampled(isy, orc):
    """Full-size XL window (cfg5 s_max = 65,536): sampled per-point outputs against the oracle's
    one-point definition, and the window record against the oracle finish of the GPU's own sums
    (which must equal the sum of the per-point canonical terms)."""
    wl = datagen.cfg5(n=200_000, n_series=2)
    x, y = wl.series[0], wl.series[1]
    t0, w = 12_345, 65_536
    got = isy.isycos_mi_batch_ex(x, y, [(t0, t0 + w)], 4, debug=True)
    xs, ys = x[t0:t0 + w], y[t0:t0 + w]
    rng = np.random.default_rng(0)
    for i in list(rng.integers(0, w, 24)) + [0, 1, w - 2, w - 1]:
        e, nx, ny = orc.point(xs, ys, int(i), 4)
        assert (got["eps"][i], got["nx"][i], got["ny"][i]) == (np.float32(e), nx, ny), i
    sp = sl = 0
    for i in range(0, w):
        a, b = orc.point_terms(got["nx"][i], got["ny"][i], got["eps"][i])
        sp += a
        sl += b
    assert sp == got["s_psi"][0] and sl == got["s_log"][0]
    mi, h, nmi = orc.finish(sp, sl, int((got["eps"] == 0).sum()), w, 4)
    assert (mi, h, nmi) == (got["mi"][0], got["h"][0], got["nmi"][0])


def test_cfg3_subsample_bitwise(isy, orc):
    """configs[2] sweep: every 97th window per (k, w) at w = 1024, 4096 (the oracle's budget), plus two
    w = 16384 windows."""
    wl = datagen.cfg3()
    x, y = wl.series
    for k in wl.sweep["ks"]:
        for w in (1024, 4096):
            W = datagen.sweep_windows(len(x), [w], wl.sweep["stride"])[::97 if w == 1024 else 389]
            check_windows(isy, orc, x, y, W, k, label=f"cfg3 k={k} w={w}")
    check_windows(isy, orc, x, y, [(512 * 37, 512 * 37 + 16384), (999_000 - 16384, 999_000)], 4,
                  label="cfg3 w=16384")


# ---------------------------------------------------------------- brute-force path for w >= 257 (ISYCOS_F_BRUTE)
def test_brute_path_large_windows(isy, orc):
    """The tile kernel (multi i-tile, multi j-tile) is the default only when the sorted path is off; the
    flag routes every window there.  Same bitwise bar."""
    wl = datagen.cfg2(n=20_000)
    x, y = wl.series
    W = [(3, 3 + 257), (100, 612), (7, 7 + 1025), (1000, 1000 + 4097), (n0 := 11_111, n0 + 8191)]
    check_windows(isy, orc, x, y, W, 4, debug=True, label="brute", brute=True)
    check_windows(isy, orc, x, y, W[:3], 8, label="brute k=8", brute=True)


# ---------------------------------------------------------------- KSG-2 (paper's literal Eq. 2; NEXT-1)
@pytest.mark.parametrize("k", [1, 4, 8])
@pytest.mark.parametrize("brute", [False, True, "unfused"])
def test_ksg2_size_classes(isy, orc, k, brute):
    """KSG-2 through every kernel: warp (w <= 256), tile (brute), sorted (w >= 257) incl. a multi-j-tile
    window; per-point eps, n_x, n_y bit-exact (n = the closed <= d_x counts)."""
    wl = datagen.cfg2(n=20_000)
    x, y = wl.series
    rng = np.random.default_rng(100 + k)
    W = []
    for w in [9, 32, 33, 100, 128, 129, 256, 257, 513, 1025, 4097, 5003]:
        if w <= k:
            continue
        t0 = int(rng.integers(0, len(x) - w))
        W.append((t0, t0 + w))
    check_windows(isy, orc, x, y, W, k, debug=True, label=f"ksg2 k={k} brute={brute}", variant=1,
                  brute=brute is True, unfused=brute == "unfused")


def test_ksg2_ties(isy, orc):
    """Ties decide KSG-2's kNN set ((d, j) order, smaller index first) and its closed counts: integer
    data, duplicated points, a constant segment (eps = 0: d_x = d_y = 0, counts of exact duplicates)."""
    st = datagen.Stream(77, 1)
    n = 5000
    xi = np.floor(st.uniform(n) * 6).astype(np.float32)
    yi = np.floor(st.uniform(n) * 6).astype(np.float32)
    xd = np.repeat(datagen.f32(st.normal(n // 3 + 1)), 3)[:n]
    yd = np.repeat(datagen.f32(st.normal(n // 3 + 1)), 3)[:n]
    xc, yc = xi.copy(), yi.copy()
    xc[2000:2300] = 1.0
    yc[2000:2300] = 2.0
    W = [(0, 40), (5, 200), (50, 700), (0, 4500), (2000, 2300), (1990, 2400)]
    for k in (1, 3, 4):
        for brute in (False, True, "unfused"):
            lab = f"k={k} brute={brute}"
            kw = dict(debug=True, variant=1, brute=brute is True, unfused=brute == "unfused")
            check_windows(isy, orc, xi, yi, W, k, label="ksg2 int " + lab, **kw)
            check_windows(isy, orc, xd, yd, W, k, label="ksg2 dup " + lab, **kw)
            check_windows(isy, orc, xc, yc, W, k, label="ksg2 const " + lab, **kw)


def test_ksg2_cfg1_sweep_and_xl(isy, orc):
    wl = datagen.cfg1()
    x, y = wl.series
    W = datagen.sweep_windows(len(x), wl.sweep["sizes"], wl.sweep["stride"])
    check_windows(isy, orc, x, y, W, 4, label="ksg2 cfg1 sweep", variant=1)
    wl2 = datagen.cfg2(n=60_000)
    x2, y2 = wl2.series
    check_windows(isy, orc, x2, y2, [(7, 7 + 16385)], 4, debug=True, label="ksg2 xl", variant=1)


@pytest.mark.parametrize("variant", [0, 1])
def test_warp_sorted_dense_batches(isy, orc, variant):
    """Batches dense enough (>= 592 windows per class) for the warp-per-window sorted kernel (64 < w <= 256;
    sparser classes take the latency-mode tile kernel), per-point outputs included."""
    wl = datagen.cfg2(n=40_000)
    x, y = wl.series
    rng = np.random.default_rng(7 + variant)
    W = []
    for w, cnt in ((65, 600), (100, 650), (128, 600), (129, 600), (200, 620), (256, 600)):
        t0 = rng.integers(0, len(x) - w, cnt)
        W += [(int(a), int(a) + w) for a in t0]
    check_windows(isy, orc, x, y, W, 4, debug=True, label=f"wsorted v{variant}", variant=variant)
    xi = np.floor(datagen.Stream(3, 1).uniform(len(x)) * 5).astype(np.float32)  # heavy ties
    check_windows(isy, orc, xi, y, W[::2] + W[1::2][:700], 3, debug=True, label=f"wsorted ties v{variant}",
                  variant=variant)


def test_maximum_window_and_empty_batch(isy, orc):
    """ISYCOS_MAX_W = 2^18 (the int64 fixed-point bound): sampled per-point outputs against the oracle's
    one-point definition and the record against the oracle finish of the per-point terms; an empty batch
    is a no-op; one point over the maximum is E_RANGE."""
    n = 300_000
    st = datagen.Stream(17, 1)
    x = datagen.f32(st.normal(n))
    y = datagen.f32(0.6 * x.astype(np.float64) + 0.8 * st.normal(n))
    w = 1 << 18
    t0 = 11
    got = isy.isycos_mi_batch_ex(x, y, [(t0, t0 + w)], 4, debug=True)
    xs, ys = x[t0:t0 + w], y[t0:t0 + w]
    rng = np.random.default_rng(1)
    for i in list(rng.integers(0, w, 12)) + [0, w - 1]:
        e, nx, ny = orc.point(xs, ys, int(i), 4)
        assert (got["eps"][i], got["nx"][i], got["ny"][i]) == (np.float32(e), nx, ny), i
    sp = sl = 0
    for i in range(w):
        a, b = orc.point_terms(got["nx"][i], got["ny"][i], got["eps"][i])
        sp += a
        sl += b
    assert sp == got["s_psi"][0] and sl == got["s_log"][0]
    assert orc.finish(sp, sl, int((got["eps"] == 0).sum()), w, 4) == (got["mi"][0], got["h"][0], got["nmi"][0])
    assert len(isy.isycos_mi_batch(x, y, np.zeros((0, 2), np.int64), 4)) == 0
    with pytest.raises(isy.IsycosError) as e:
        isy.isycos_mi_batch(x, y, [(0, w + 1)], 4)
    assert e.value.code == -2


@pytest.mark.parametrize("k", [1, 4, 8])
def test_pair_loads_odd_layouts(isy, orc, k):
    """Phase A's 16-byte pair loads (throughput scan, w >= 2,048): aligned blocks with self masked in the first
    block of one side, so both parities of every position are exercised; odd window sizes before and after the
    large ones give odd scratch offsets (rounded up to even by the engine), plus a tied series."""
    wl = datagen.cfg2(n=40_000)
    x, y = wl.series
    sizes = [257, 999, 2049, 3001, 4095, 2048, 8191, 8193, 12289, 301, 2051]
    W = [(3 + 7 * i, 3 + 7 * i + w) for i, w in enumerate(sizes)] + [(len(x) - 4097, len(x))]
    check_windows(isy, orc, x, y, W, k, debug=True, label=f"pairs k={k}", unfused=True)
    st = datagen.Stream(21, 2)
    xi = np.floor(st.uniform(len(x)) * 9).astype(np.float32)
    check_windows(isy, orc, xi, y, W, k, debug=True, label=f"pairs ties k={k}", unfused=True)
