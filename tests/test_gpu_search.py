"""GPU search parity: isycos_search (batched, speculative) vs the oracle's sequential search.

Bar: the selected window set is bit-exact (north star) and the algorithm-level counters are
identical (they count what the sequential algorithms consume, not what the GPU speculated).
"""
import numpy as np
import pytest

import datagen

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def isy():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2204_09131_b200 import build

    build.build()
    import paper_2204_09131_b200 as isy

    return isy


def run_both(isy, orc, wl, series=None, pairs=None, **kw):
    series = wl.series if series is None else series
    pairs = wl.pairs if pairs is None else pairs
    ores, ost = orc.search(series, pairs, orc.make_params(wl.search, **kw))
    gres, gst = isy.search_workload(wl, series=series, pairs=pairs, **kw)
    return ores, ost, gres, gst


def assert_same(ores, ost, gres, gst, label=""):
    assert gres == ores, f"{label}: result sets differ\nGPU {gres}\nORC {ores}"
    for f, v in ost.items():
        assert gst[f] == v, f"{label}: stat {f} GPU {gst[f]} oracle {v}"


@pytest.mark.parametrize("method", [1, 2, 3])
@pytest.mark.parametrize("noise", [0, 1])
def test_cfg1_search(isy, orc, method, noise):
    wl = datagen.cfg1()
    ores, ost, gres, gst = run_both(isy, orc, wl, method=method, noise=noise)
    assert_same(ores, ost, gres, gst, f"cfg1 m={method} noise={noise}")
    assert len(gres) > 0


@pytest.mark.parametrize("lookahead", [1, 3, 1000])
def test_bu_speculation_invariance(isy, orc, lookahead):
    wl = datagen.cfg1()
    ores, ost = orc.search(wl.series, wl.pairs, orc.make_params(wl.search, method=2))
    gres, gst = isy.search_workload(wl, method=2, lookahead=lookahead)
    assert_same(ores, ost, gres, gst, f"lookahead={lookahead}")


def test_cfg1_chunks_and_params(isy, orc):
    wl = datagen.cfg1()
    for kw in (dict(n_chunks=4), dict(n_chunks=3, method=1), dict(t_max_idle=0, h=1, method=2),
               dict(delta_td=24, delta_bu=7), dict(sizes=[512, 200, 64], method=1), dict(p=1, seed=77),
               dict(k=8, sigma=0.3), dict(k=1)):
        ores, ost, gres, gst = run_both(isy, orc, wl, **kw)
        assert_same(ores, ost, gres, gst, f"cfg1 {kw}")


def test_cfg2_full_search(isy, orc):
    """configs[1] exactly: n=100,000 AR(1) + 4 planted relations, scales 32..4096, TD+BU, noise on."""
    wl = datagen.cfg2()
    ores, ost, gres, gst = run_both(isy, orc, wl)
    assert_same(ores, ost, gres, gst, "cfg2")
    # planted recovery (reported by the oracle tests too): every planted block is covered >= 0.8 by TD
    for (a, b, _) in wl.planted[0]:
        cov = set()
        for r in gres:
            if r[1] == 1:
                cov.update(range(max(a, r[2]), min(b, r[3])))
        assert len(cov) / (b - a) >= 0.8, (a, b)


def test_cfg4_instance(isy, orc):
    """configs[3] recipe on a reduced instance (6 series x 60,000 samples, scales 64..4096) that the
    oracle finishes in seconds; all 15 pairs, TD+BU with noise pruning; pair ids kept."""
    wl = datagen.cfg4(n=60_000, n_series=6, n_planted=2)
    pairs = [(a, b, 100 + i) for i, (a, b) in enumerate(wl.pairs)]
    ores, ost, gres, gst = run_both(isy, orc, wl, pairs=pairs, s_max=4096)
    assert_same(ores, ost, gres, gst, "cfg4 instance")


def test_cfg5_instance(isy, orc):
    """configs[4] recipe on a reduced instance (2 series x 120,000, scales 128..8192, 4 chunks, TD,
    noise on) — the chunked Alg. 4 path with merge."""
    wl = datagen.cfg5(n=120_000, n_series=2, n_chunks=4)
    ores, ost, gres, gst = run_both(isy, orc, wl, s_max=8192)
    assert_same(ores, ost, gres, gst, "cfg5 instance")


def test_device_series_input(isy, orc):
    import torch

    wl = datagen.cfg1()
    ores, ost = orc.search(wl.series, wl.pairs, orc.make_params(wl.search))
    ds = [torch.from_numpy(s).cuda() for s in wl.series]
    gres, gst = isy.search_workload(wl, series=ds)
    assert_same(ores, ost, gres, gst, "device series")


@pytest.mark.parametrize("method", [1, 2])
def test_cfg1_search_ksg2(isy, orc, method):
    """The search driven by KSG-2 (paper's literal Eq. 2) instead of KSG-1: same bitwise bar."""
    wl = datagen.cfg1()
    ores, ost, gres, gst = run_both(isy, orc, wl, method=method, variant=1)
    assert_same(ores, ost, gres, gst, f"cfg1 ksg2 m={method}")


@pytest.mark.parametrize("kw", [dict(auto_M=4, auto_m=2), dict(auto_M=8, auto_m=8, auto_alpha=0.2, auto_rho=0.3)])
def test_cfg1_auto_selection(isy, orc, kw):
    """iSYCOS (Alg. 3): sampled trial runs, Eqs. 6-9, then the chosen method — results, counters (incl.
    eval_cost, the runtime proxy) and the nscore sums bit-exact against the oracle."""
    wl = datagen.cfg1()
    ores, ost, gres, gst = run_both(isy, orc, wl, method=4, **kw)
    assert_same(ores, ost, gres, gst, f"cfg1 auto {kw}")
    assert gst["auto_td"] + gst["auto_bu"] == 1


@pytest.mark.parametrize("kind", ["dense", "sparse"])
def test_scenario_auto_selection(isy, orc, kind):
    wl = datagen.scenario(kind, seed=0)
    ores, ost, gres, gst = run_both(isy, orc, wl)
    assert_same(ores, ost, gres, gst, f"scenario {kind}")
    assert (gst["auto_td"], gst["auto_bu"]) == ((1, 0) if kind == "dense" else (0, 1))


def test_multi_pair_auto_selection(isy, orc):
    wl = datagen.cfg4(n=8000, n_series=4, n_planted=1)
    pairs = [(a, b, 40 + i) for i, (a, b) in enumerate(wl.pairs)]
    ores, ost, gres, gst = run_both(isy, orc, wl, pairs=pairs, s_max=1024, method=4, auto_M=5, auto_m=2)
    assert_same(ores, ost, gres, gst, "cfg4 auto")
    assert gst["auto_td"] + gst["auto_bu"] == len(pairs)


# ---------------------------------------------------------------- BASELINE.json full sizes (sampled outputs)
def _check_result_windows(orc, series, pairs, res, sc, n_check=6):
    """Properties every result set must have at any size: per (pair, method) pairwise
    disjoint, s_min <= |w| <= s_max, nmi >= sigma, sorted by (pair, method, t0); and a sample of the
    windows re-evaluated one by one by the oracle, bitwise (mi, h, nmi)."""
    assert res == sorted(res, key=lambda r: (r[0], r[1], r[2]))
    by = {}
    for r in res:
        by.setdefault((r[0], r[1]), []).append(r)
        assert sc.s_min <= r[3] - r[2] <= sc.s_max and r[6] >= sc.sigma
    for lst in by.values():
        for a, b in zip(lst, lst[1:]):
            assert a[3] <= b[2], (a, b)
    pid = {p[2] if len(p) > 2 else i: p for i, p in enumerate(pairs)}
    for r in sorted(res, key=lambda r: r[3] - r[2])[:n_check]:  # the cheapest ones for the O(w^2) oracle
        xs, ys = pid[r[0]][0], pid[r[0]][1]
        ref = orc.mi_batch(series[xs], series[ys], np.asarray([[r[2], r[3]]], np.int64), sc.k)
        assert (r[4], r[5], r[6]) == (ref["mi"][0], ref["h"][0], ref["nmi"][0]), r


def test_full_size_cfg4_pairs(isy, orc):
    """configs[3] at full size (n = 1,000,000, scales 64..16,384, TD+BU, noise on) on three of its pairs
    (two planted, one background); sampled result windows against the oracle, properties on all."""
    wl = datagen.cfg4()
    planted = sorted(wl.planted)[:2]
    pairs = [tuple(wl.pairs[i]) + (i,) for i in planted] + [tuple(wl.pairs[5]) + (5,)]
    res, st = isy.search_workload(wl, pairs=pairs)
    _check_result_windows(orc, wl.series, pairs, res, wl.search)
    for i in planted:  # each planted relation is found (union coverage >= 0.5 by either method)
        (a, b, _), = wl.planted[i]
        cov = set()
        for r in res:
            if r[0] == i:
                cov.update(range(max(a, r[2]), min(b, r[3])))
        assert len(cov) >= 0.5 * (b - a), (i, a, b, len(cov))


def test_full_size_cfg5_pair(isy, orc):
    """configs[4] at full size for one pair (n = 10,000,000, scales 128..65,536, 16 chunks, TD + noise
    pruning): XL windows, the chunk plan and the merge; sampled windows against the oracle."""
    wl = datagen.cfg5(n_series=2)
    res, st = isy.search_workload(wl, pairs=[(0, 1, 0)])
    _check_result_windows(orc, wl.series, [(0, 1, 0)], res, wl.search, n_check=4)
    assert st["td_windows"] > 0
