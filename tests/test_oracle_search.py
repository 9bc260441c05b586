"""Pins for the oracle's search (Alg. 1 SYCOS_TD, Alg. 2 SYCOS_BU, §6 noise pruning, Alg. 4 chunks).

The control logic is pinned with a table-driven mock MI provider against the
paper's worked examples and the SPEC examples
(S:329-341), then against invariants and planted-window
recovery on the real estimator (cfg1).
"""
import numpy as np
import pytest

import datagen

pytestmark = pytest.mark.timeout(300)  # a broken LAHC history can climb forever


def P(orc, **kw):
    base = dict(k=2, method=1, noise=0, s_min=16, s_max=16, sigma=0.2, tau_ratio=0.25, p=3, h=5,
                t_max_idle=3, n_chunks=1, seed=0)
    base.update(kw)
    return orc.make_params(**base)


# ------------------------------------------------------------------ TD worked examples
def test_td_worked_example_p238(orc):
    # w0=[0,16), w1=[4,20) uncorrelated; w2=[8,24) correlated -> S={w2}; partition [ts0, ts2)
    # passed down; w3 starts at te2 = 24.
    def fn(t0, t1):
        return (1.0, 1.0, 1.0) if (t0, t1) == (8, 24) else (0.0, 1.0, 0.0)

    res, st, calls = orc.search_mock(fn, 64, P(orc, s_max=16, s_min=4, sizes=[16, 4]))
    assert [(r[2], r[3]) for r in res] == [(8, 24)]
    assert calls[:4] == [(0, 16), (4, 20), (8, 24), (24, 40)]
    layer2 = [c for c in calls if c[1] - c[0] == 4]
    covered = set()
    for (a, b) in layer2:
        covered.update(range(a, b))
    assert covered == set(range(0, 8)) | set(range(24, 64))  # partitions [0,8) and [24,64)


def test_td_worked_example_p3009(orc):
    # w1..w4 uncorrelated, w5 correlated -> left-out list [ts1, ts5); w6 starts right after te5.
    def fn(t0, t1):
        return (1.0, 1.0, 1.0) if (t0, t1) == (16, 32) else (0.0, 1.0, 0.0)

    res, st, calls = orc.search_mock(fn, 64, P(orc, s_max=16, s_min=4, sizes=[16, 4]))
    assert [(r[2], r[3]) for r in res] == [(16, 32)]
    assert calls[:6] == [(0, 16), (4, 20), (8, 24), (12, 28), (16, 32), (32, 48)]
    layer2 = {c for c in calls if c[1] - c[0] == 4}
    assert (12, 16) in layer2 and (32, 36) in layer2 and not any(16 <= a < 32 for a, _ in layer2)


def test_td_fully_correlated_single_window(orc):
    # fully correlated pair with s_max = N -> {[0, N)} after layer 1
    res, st, calls = orc.search_mock(lambda a, b: (2.0, 1.0, 1.0), 256, P(orc, s_max=256, s_min=16))
    assert [(r[2], r[3]) for r in res] == [(0, 256)] and st["td_windows"] == 1


def test_td_independent_empty_and_full_coverage(orc):
    # independent pair -> {}; every sample ends in a bottom-layer partition
    res, st, calls = orc.search_mock(lambda a, b: (0.0, 1.0, 0.0), 200, P(orc, s_max=64, s_min=16))
    assert res == []
    bottom = [c for c in calls if c[1] - c[0] == 16]
    covered = set()
    for a, b in bottom:
        covered.update(range(a, b))
    assert covered == set(range(200))
    # layer schedule: halving 64 -> 32 -> 16; delta = s/4
    assert {c[1] - c[0] for c in calls} == {64, 32, 16}
    assert (4, 20) in calls and (8, 40) in calls and (16, 80) in calls


def _noise_mock(s, delta, clean_tails=()):
    # main windows: uncorrelated (nmi 0.1 < sigma), mi 0.5; overlap (size s-delta): mi 0.6 > main;
    # tail (size delta): nmi 0.01 < tau = 0.05 -> noise, unless listed in clean_tails.
    def fn(t0, t1):
        size = t1 - t0
        if size == s:
            return (0.5, 1.0, 0.1)
        if size == s - delta:
            return (0.6, 1.0, 0.1)
        if size == delta:
            return (0.0, 1.0, 0.5 if (t0, t1) in clean_tails else 0.01)
        return (0.0, 1.0, 0.0)
    return fn


def test_td_noise_p1_skips_immediately(orc):
    # p=1, verdict noise -> skip past w1
    res, st, calls = orc.search_mock(_noise_mock(16, 4), 64, P(orc, noise=1, p=1, s_min=16, s_max=16, k=2))
    mains = [c for c in calls if c[1] - c[0] == 16]
    assert mains == [(0, 16), (4, 20), (20, 36), (24, 40), (40, 56), (44, 60)]
    assert st["td_noise_checks"] == 3 and st["td_skips"] == 3 and st["td_windows"] == 6


def test_td_noise_streak_p3(orc):
    res, st, calls = orc.search_mock(_noise_mock(16, 4), 64, P(orc, noise=1, p=3, s_min=16, s_max=16, k=2))
    mains = [c for c in calls if c[1] - c[0] == 16]
    # checks at t=4,8,12 -> skip to 28; checks at 32,36,40 -> skip to 56 (56+16 > 64)
    assert mains == [(0, 16), (4, 20), (8, 24), (12, 28), (28, 44), (32, 48), (36, 52), (40, 56)]
    assert st["td_skips"] == 2


def test_td_noise_streak_reset(orc):
    # p=3, verdicts noise, noise, clean -> streak reset, no skip at t=12
    fn = _noise_mock(16, 4, clean_tails={(24, 28)})
    res, st, calls = orc.search_mock(fn, 64, P(orc, noise=1, p=3, s_min=16, s_max=16, k=2))
    mains = [c for c in calls if c[1] - c[0] == 16]
    # t=4 s1, t=8 s2, t=12 clean -> 0, t=16 s1, t=20 s2, t=24 s3 -> skip to 40; 40: no check; 44: s1; 48: s2
    assert mains[:9] == [(0, 16), (4, 20), (8, 24), (12, 28), (16, 32), (20, 36), (24, 40), (40, 56), (44, 60)]
    assert st["td_skips"] == 1


def test_noise_predicate_stated_values(orc):
    # S:275-276 with the split reading: tail nmi 0.03 < tau=0.05 and mix mi < base mi -> noise;
    # tail nmi 0.10 >= tau -> not noise regardless of the mixture.
    for tail_nmi, expect_skip in ((0.03, True), (0.10, False)):
        def fn(t0, t1, tail_nmi=tail_nmi):
            size = t1 - t0
            if size == 16:
                return (0.20, 1.0, 0.10)   # mixture w1 (normalized below sigma)
            if size == 12:
                return (0.30, 1.0, 0.30)   # base w_o
            return (0.0, 1.0, tail_nmi)    # extension w_delta
        res, st, _ = orc.search_mock(fn, 32, P(orc, noise=1, p=1, s_min=16, s_max=16, k=2))
        assert (st["td_skips"] > 0) == expect_skip


# ------------------------------------------------------------------ BU
def test_bu_constant_landscape_iterations(orc):
    # constant MI: every iteration rejects (strict '>', G4) -> T_maxIdle+1 iterations per climb
    for T in (0, 3):
        res, st, _ = orc.search_mock(lambda a, b: (0.3, 1.0, 0.1), 640,
                                     P(orc, method=2, s_min=32, s_max=128, t_max_idle=T, k=4))
        assert res == []
        assert st["bu_climbs"] == 20                 # lo = 0, 32, ..., 608
        # S:384 (T=0 stops at the first non-improvement); the last climb [608,640) has an empty
        # neighbourhood (every delta-neighbour leaves [lo,hi) or the size bounds) and stops at once.
        assert st["bu_iterations"] == 19 * (T + 1)


def test_bu_climbs_to_unimodal_peak(orc):
    d = 10
    a, b = 50, 50 + 32 + 3 * d   # peak window; s_min=32, delta_bu=10

    def fn(t0, t1):
        v = 1.0 - (abs(t0 - a) + abs(t1 - b)) / 1000.0
        return (v, 1.0, 0.5 if (t0, t1) == (a, b) else 0.05)

    res, st, calls = orc.search_mock(fn, 400, P(orc, method=2, s_min=32, s_max=200, delta_bu=d, k=4))
    assert [(r[2], r[3]) for r in res] == [(a, b)]
    assert res[0][1] == 2


def test_bu_noise_prunes_right_p1(orc):
    # smaller windows score higher; every extension is noise (nmi 0 < tau) and every mix (larger)
    # has lower MI than the base -> with p=1 the applicable direction is pruned after one verdict.
    fn = lambda t0, t1: (1.0 / (t1 - t0), 1.0, 0.0)
    base = P(orc, method=2, s_min=32, s_max=128, k=4, t_max_idle=1)
    _, st0, _ = orc.search_mock(fn, 320, base)
    _, st1, _ = orc.search_mock(fn, 320, P(orc, method=2, s_min=32, s_max=128, k=4, t_max_idle=1, noise=1, p=1))
    assert st1["bu_prunes"] >= st1["bu_climbs"] - 1   # the last climb has no neighbourhood
    assert st1["bu_neighbors"] < st0["bu_neighbors"]


# ------------------------------------------------------------------ LAHC acceptance + history (Alg. 2 l.11-21)
# Hand traces of Alg. 2 with the history draws r of line 11 passed in as inputs (the paper's
# "random policy"; tests may fix random numbers).  Landscapes live on the line t0 = lo: windows
# starting elsewhere score -1, so the best neighbour of (0, t1) is the better of (0, t1 - d), (0, t1 + d).
def _line(f, good):
    def fn(t0, t1):
        if t0 != 0:
            return (-1.0, 1.0, 0.0)
        return (f[t1], 1.0, 1.0 if t1 == good else 0.0)
    return fn


def _bu(orc, **kw):
    base = dict(method=2, s_min=32, s_max=200, delta_bu=10, k=4, t_max_idle=0, h=2)
    base.update(kw)
    return P(orc, **base)


def test_lahc_late_acceptance_crosses_a_dip(orc):
    """l.12 "I_best > I_h or I_best > I_w": the history lets the climb accept a worse window and cross a dip.
    f(t1) = 0.1, 0.3, 0.5, 0.4, 0.9, 0.2, 0.2 at t1 = 32..92; L = [0.1, 0.1]; draws r = 0, 0, 1, 0, 1.
      it1 r=0: best (0,42) 0.3 > L0 0.1: accept; I_w 0.3 > I_h -> L0 = 0.3
      it2 r=0: best (0,52) 0.5 > 0.3: accept; L0 = 0.5
      it3 r=1: best (0,62) 0.4 (the dip) > L1 0.1: accept although 0.4 < I_w 0.5; L1 = 0.4
      it4 r=0: best (0,72) 0.9 > 0.5: accept; L0 = 0.9
      it5 r=1: best (0,62) 0.4, not > L1 0.4, not > 0.9: reject; idle 1 > T_maxIdle 0: stop at (0,72).
    With "and" (or plain hill climbing, I_best > I_w only) it3 rejects and the climb stops on the 0.5 peak
    (0,52), whose normalized MI is below sigma: no result."""
    f = {32: 0.1, 42: 0.3, 52: 0.5, 62: 0.4, 72: 0.9, 82: 0.2, 92: 0.2}
    res, st, _ = orc.search_mock_draws(_line(f, 72), {0: [0, 0, 1, 0, 1]}, 100, _bu(orc))
    assert [(r[2], r[3]) for r in res] == [(0, 72)]
    assert st["bu_iterations"] == 5 and st["bu_climbs"] == 1   # lo = 72 next: 72 + 32 > 100


def test_lahc_accepts_above_current_below_history(orc):
    """The "or I_best > I_w" half: after the dip, the way back up is better than the current window but not
    than the history entry drawn.  Same trace to it3 (L = [0.5, 0.4], w = (0,62) 0.4), then
      it4 r=0: best (0,52) 0.5: not > L0 0.5, but > I_w 0.4: accept; I_w 0.5 not > I_h 0.5: no update
      it5 r=1: best (0,62) 0.4: reject; stop at (0,52).
    Dropping the I_w test rejects at it4 and stops at (0,62) (normalized MI below sigma): no result."""
    f = {32: 0.1, 42: 0.3, 52: 0.5, 62: 0.4, 72: 0.2, 82: 0.2, 92: 0.2}
    res, st, _ = orc.search_mock_draws(_line(f, 52), {0: [0, 0, 1, 0, 1]}, 80, _bu(orc))
    assert [(r[2], r[3]) for r in res] == [(0, 52)]
    assert st["bu_iterations"] == 5 and st["bu_climbs"] == 1   # lo = 52 next: 52 + 32 > 80


def test_lahc_history_update_writes_current_value(orc):
    """l.19-20 "if I_w > I_wh then I_wh := I_w" (the current solution's value, not the rejected candidate's).
    2-D landscape, d = 10, s_min 30, s_max 60, [lo, hi) = [0, 70), h = 3, T_maxIdle = 2,
    draws r = 1, 2, 0, 1, 2, 2, 2, 0, 1:
      start (0,30) 0.2, L = [.2 .2 .2]
      it1 r=1: N = (0,40) .5, (10,40) .2 -> (0,40) .5 > .2 accept;  L = [.2 .5 .2]
      it2 r=2: best (0,50) .3 > L2 .2: accept (late, downhill);       L = [.2 .5 .3]
      it3 r=0: best (0,60) .7: accept;                                 L = [.7 .5 .3]
      it4 r=1: best (10,60) .5 = L1, < .7: reject, idle 1; .7 > .5 -> L1 = .7 (the rejected .5 would stay)
      it5 r=2: (10,60) .5 > L2 .3: accept, idle 0;                     L = [.7 .7 .5]
      it6 r=2: best (20,70) .8: accept;                                L = [.7 .7 .8]
      it7 r=2: best (30,60) .6 < .8: reject, idle 1
      it8 r=0: .6 < L0 .7: reject, idle 2; L0 = .8
      it9 r=1: .6 < L1 .7: reject, idle 3 > 2: stop at (20,70) after 9 iterations.
    Writing I_best instead leaves L1 = .5 at it4, so it9 accepts (30,60) and the climb runs 13 iterations."""
    vals = {(0, 30): .2, (0, 40): .5, (0, 50): .3, (0, 60): .7, (10, 40): .2, (10, 50): .1, (10, 60): .5,
            (10, 70): .1, (20, 50): .2, (20, 60): .3, (20, 70): .8, (30, 60): .6, (30, 70): .5, (40, 70): .3}

    def fn(t0, t1):
        return (vals.get((t0, t1), -1.0), 1.0, 1.0 if (t0, t1) == (20, 70) else 0.0)

    res, st, _ = orc.search_mock_draws(fn, {0: [1, 2, 0, 1, 2, 2, 2, 0, 1]}, 70,
                                       _bu(orc, s_min=30, s_max=60, h=3, t_max_idle=2))
    assert [(r[2], r[3]) for r in res] == [(20, 70)]
    assert st["bu_iterations"] == 9 and st["bu_climbs"] == 1


def test_bu_restart_after_accept(orc):
    """Line 25 / S:407: after an accepted window the next climb starts at its end (max(t1, lo + s_min));
    after a rejected climb at lo + s_min.  The unimodal climb of test_bu_climbs_to_unimodal_peak accepts
    (50, 112) from lo = 0, so the climbs start at 0, 112, 144, ..., 368 (368 + 32 <= 400): 10 climbs
    (restarting at lo + s_min instead would give 12, starting at 0, 32, ..., 352)."""
    d = 10
    a, b = 50, 50 + 32 + 3 * d

    def fn(t0, t1):
        v = 1.0 - (abs(t0 - a) + abs(t1 - b)) / 1000.0
        return (v, 1.0, 0.5 if (t0, t1) == (a, b) else 0.05)

    res, st, calls = orc.search_mock(fn, 400, P(orc, method=2, s_min=32, s_max=200, delta_bu=d, k=4))
    assert [(r[2], r[3]) for r in res] == [(a, b)]
    assert st["bu_climbs"] == 10
    assert (112, 144) in calls and (368, 400) in calls


def test_bu_seed_determinism(orc):
    wl = datagen.cfg1()
    p = orc.make_params(wl.search, method=2)
    r1, s1 = orc.search(wl.series, wl.pairs, p)
    r2, s2 = orc.search(wl.series, wl.pairs, p)
    assert r1 == r2 and s1 == s2


# ------------------------------------------------------------------ chunks (Alg. 4)
def test_chunk_plan_s511(orc):
    assert orc.chunk_plan(1000, 4, 100) == [(0, 250), (150, 500), (400, 750), (650, 1000)]
    assert orc.chunk_plan(1000, 1, 100) == [(0, 1000)]


def test_chunks_np1_equals_plain(orc):
    wl = datagen.cfg1()
    a = orc.search(wl.series, wl.pairs, orc.make_params(wl.search))
    b = orc.search(wl.series, wl.pairs, orc.make_params(wl.search, n_chunks=1))
    assert a == b


def _chunk_mock(a, b):
    """n = 200, n_p = 2, s_max = s_min = 64 (TD, one layer, delta 16): chunks [0,100) and [36,200) (Alg. 4
    line 14).  Chunk 0 scans t = 0, 16, 32 and accepts (32,96); chunk 1 scans t = 36 and accepts
    (36,100), then 100, 116, 132.  The two results overlap: the merge keeps one (reading R20)."""
    def fn(t0, t1):
        if (t0, t1) == (32, 96):
            return a
        if (t0, t1) == (36, 100):
            return b
        return (0.0, 1.0, 0.0)
    return fn


@pytest.mark.parametrize("a,b,keep", [
    ((1.0, 2.0, 0.9), (5.0, 9.0, 0.5), (32, 96)),     # higher normalized MI first, whatever the raw MI
    ((2.0, 2.0, 1.0), (3.0, 3.0, 1.0), (36, 100)),    # normalized tie (saturated at 1): higher raw MI
    ((2.0, 2.0, 1.0), (2.0, 2.0, 1.0), (32, 96)),     # full tie: smaller (t0, t1)
    ((3.0, 3.0, 1.0), (2.0, 2.0, 1.0), (32, 96)),
])
def test_chunk_merge_priority(orc, a, b, keep):
    """R20: greedy by (normalized MI desc, raw MI desc, t0 asc, t1 asc), keep if disjoint, sort by t0."""
    p = P(orc, method=1, s_min=64, s_max=64, n_chunks=2)
    res, st, calls = orc.search_mock(_chunk_mock(a, b), 200, p)
    assert (32, 96) in calls and (36, 100) in calls and st["td_accepted"] == 2
    assert [(r[2], r[3]) for r in res] == [keep]
    got = res[0]
    assert (got[4], got[5], got[6]) == (a if keep == (32, 96) else b)


def test_chunks_interior_windows_preserved(orc):
    # windows far from chunk boundaries appear identically in the n_p=2 run (TD)
    wl = datagen.cfg1()
    a, _ = orc.search(wl.series, wl.pairs, orc.make_params(wl.search, method=1))
    b, _ = orc.search(wl.series, wl.pairs, orc.make_params(wl.search, method=1, n_chunks=2))
    for w in b:
        assert all(not (w[2] < q[3] and q[2] < w[3]) or q == w for q in b)  # disjoint
    interior_a = [w for w in a if w[3] <= 1024 - 512]
    assert all(w in b for w in interior_a)


# ------------------------------------------------------------------ invariants + planted recovery
def _coverage(res, block):
    a, b = block
    cov = set()
    for r in res:
        cov.update(range(max(a, r[2]), min(b, r[3])))
    return len(cov) / (b - a)


@pytest.mark.parametrize("noise", [0, 1])
def test_cfg1_search_invariants_and_recovery(orc, noise):
    wl = datagen.cfg1()
    sc = wl.search
    res, st = orc.search(wl.series, wl.pairs, orc.make_params(sc, noise=noise))
    x, y = wl.series
    for method in (1, 2):
        rs = [r for r in res if r[1] == method]
        # disjoint, sorted, size bounds, sigma re-verified from scratch
        for i, r in enumerate(rs):
            assert sc.s_min <= r[3] - r[2] <= sc.s_max
            if i:
                assert rs[i - 1][3] <= r[2]
            w = orc.window(x[r[2]:r[3]], y[r[2]:r[3]], k=sc.k)
            assert w.nmi >= sc.sigma and w.mi == r[4] and w.nmi == r[6]
        # planted recovery: union coverage >= 0.8 per planted block (S:331 form)
        for (a, b, _) in wl.planted[0]:
            assert _coverage(rs, (a, b)) >= 0.8, (method, a, b, rs)


# ------------------------------------------------------------------ iSYCOS selection (Alg. 3, Eqs. 4-9)
def test_auto_scores_worked_example(orc):
    # SPEC S:455-457 (Eqs. 6-8 arithmetic): equal runtimes -> t~ = 0.5 each; alpha = 0.5, n~L_TD = 3/5 = 0.6
    # -> nscore_TD = 0.5 * (1/0.5) + 0.5 * 0.6 = 1.3, nscore_BU = 0.5 * 2 + 0.5 * 0.4 = 1.2 -> TD.
    chosen, td, bu = orc.auto_scores(1000, 1000, 6, 3, 2, 0.5)
    assert chosen == 1
    assert td == pytest.approx(1.3, abs=1e-15) and bu == pytest.approx(1.2, abs=1e-15)
    # Eq. 6 symmetry: equal runtimes give equal runtime terms (alpha * 2)
    c2, td2, bu2 = orc.auto_scores(777, 777, 3, 0, 0, 0.3)
    assert td2 == bu2 == pytest.approx(0.3 * 2 + 0.7 * 0.5, abs=1e-15)


def test_auto_scores_rules(orc):
    # ties select BU (Alg. 3 line 11 is a strict ">")
    assert orc.auto_scores(500, 500, 6, 4, 4)[0] == 2
    # no windows at all: n~ = 0.5 each, the runtime alone decides
    c, td, bu = orc.auto_scores(100, 300, 6, 0, 0, 0.5)
    assert c == 1 and td == pytest.approx(0.5 * 4 + 0.25) and bu == pytest.approx(0.5 / 0.75 + 0.25)
    # monotonicity: decreasing t_TD strictly increases nscore_TD, windows fixed
    prev = -1.0
    for cost_td in (5000, 2000, 1000, 500, 100):
        _, td, _ = orc.auto_scores(cost_td, 1000, 6, 3, 5, 0.5)
        assert td > prev
        prev = td
    # alpha-robustness on extremes: TD faster AND more large windows -> TD for alpha in 0.2..0.8
    for a in (0.2, 0.4, 0.5, 0.6, 0.8):
        assert orc.auto_scores(100, 900, 6, 9, 1, a)[0] == 1
        assert orc.auto_scores(900, 100, 6, 1, 9, a)[0] == 2


def test_auto_sampling(orc):
    # m = M -> every partition exactly once; fixed seed reproduces; m of M distinct
    assert sorted(orc.auto_sample(20, 20, 123, 7)) == list(range(20))
    assert orc.auto_sample(20, 6, 5, 3) == orc.auto_sample(20, 6, 5, 3)
    s = orc.auto_sample(10, 4, 0, 0)
    assert len(set(s)) == 4 and all(0 <= i < 10 for i in s)
    # streams are keyed by (seed, pair): different pairs draw different samples (w.h.p.)
    assert len({tuple(orc.auto_sample(50, 5, 1, p)) for p in range(8)}) == 8


def test_auto_runs_the_chosen_method(orc):
    """AUTO's windows are those of the chosen method run alone on the whole series; its counters are the
    trial runs' plus that run's; TD trial counters equal TD run on the sampled partitions alone."""
    wl = datagen.cfg1()
    x, y = wl.series
    M, m = 4, 2
    pa = orc.make_params(wl.search, method=4, auto_M=M, auto_m=m)
    res, st = orc.search(wl.series, wl.pairs, pa)
    chosen = 1 if st["auto_td"] == 1 else 2
    assert st["auto_td"] + st["auto_bu"] == 1
    ref, rst = orc.search(wl.series, wl.pairs, orc.make_params(wl.search, method=chosen))
    assert res == ref
    # TD on each sampled partition alone (TD has no random stream: position-shift invariant counters)
    L = len(x) // M
    td = dict(td_windows=0, td_noise_checks=0, td_skips=0, td_accepted=0)
    for i in orc.auto_sample(M, m, wl.search.seed, 0):
        _, s = orc.search([x[i * L:(i + 1) * L], y[i * L:(i + 1) * L]], [(0, 1)],
                          orc.make_params(wl.search, method=1))
        for f in td:
            td[f] += s[f]
    for f in td:
        assert st[f] == td[f] + (rst[f] if chosen == 1 else 0), f


def test_auto_scenarios(orc):
    """Fig. 1 scenarios: long dense correlated stretches favour SYCOS_TD (cheap large accepts,
    many large windows); short sparse relations favour SYCOS_BU (many small windows)."""
    chosen = {"dense": [], "sparse": []}
    for seed in range(4):
        for kind in ("dense", "sparse"):
            wl = datagen.scenario(kind, seed=seed)
            _, st = orc.search(wl.series, wl.pairs, orc.make_params(wl.search))
            chosen[kind].append(1 if st["auto_td"] else 2)
    assert chosen["dense"].count(1) >= 3, chosen
    assert chosen["sparse"].count(2) >= 3, chosen
