"""Pins for the oracle's window estimator (KSG-1 default, KSG-2 flag, KL entropy, normalized MI).

Each pin is something the paper or the mathematics fixes, not a re-typing of
the oracle: closed forms on hand-derivable point sets, the
paper's worked example, brute force by a different algorithm on tiny
windows, exact invariants, and statistical closed forms (north star: MI of a
bivariate Gaussian -> -1/2 ln(1-rho^2)).
"""
import itertools
import math

import numpy as np
import pytest

import datagen


def H(n):  # harmonic number H_n = psi(n+1) - psi(1)
    return sum(1.0 / i for i in range(1, n + 1))


def psi_int(m):  # digamma at positive integers, from harmonic numbers (independent of the table)
    return -0.57721566490153286061 + H(m - 1)


# ---------------------------------------------------------------- closed forms
@pytest.mark.parametrize("w", [8, 64, 257])
def test_diagonal_k1_closed_form(orc, w):
    x = np.arange(w, dtype=np.float32)
    r = orc.window(x, x, k=1)
    # eps_i = 1, n_x = n_y = 0  =>  I = psi(1) + psi(w) - 2 psi(1) = H_{w-1}
    assert np.all(r.eps == 1.0) and np.all(r.nx == 0) and np.all(r.ny == 0)
    assert abs(r.mi - H(w - 1)) < 1e-9
    # KL entropy: psi(w) - psi(1) + (2/w) sum ln 2 = H_{w-1} + 2 ln 2
    assert abs(r.h - (H(w - 1) + 2 * math.log(2))) < 1e-9


@pytest.mark.parametrize("w", [8, 64, 300])
def test_diagonal_k4_closed_form(orc, w):
    x = np.arange(w, dtype=np.float32)
    r = orc.window(x, x, k=4)
    ends = [0, 1, w - 2, w - 1]
    exp_eps = np.full(w, 2.0, np.float32)
    exp_eps[[0, w - 1]] = 4.0
    exp_eps[[1, w - 2]] = 3.0
    exp_n = np.full(w, 2)
    exp_n[ends] = 3
    assert np.array_equal(r.eps, exp_eps)
    assert np.array_equal(r.nx, exp_n) and np.array_equal(r.ny, exp_n)
    closed = psi_int(4) + psi_int(w) - (4 * 2 * psi_int(4) + (w - 4) * 2 * psi_int(3)) / w
    assert abs(r.mi - closed) < 1e-9


def test_grid_4x4_closed_form(orc):
    # points (i mod 4, i div 4): corners eps=2, n=7; edges/interior eps=1, n=3 (k=4)
    pts = [(i % 4, i // 4) for i in range(16)]
    x = np.array([p[0] for p in pts], np.float32)
    y = np.array([p[1] for p in pts], np.float32)
    r = orc.window(x, y, k=4)
    corners = [0, 3, 12, 15]
    assert np.all(r.eps[corners] == 2.0)
    assert np.all(np.delete(r.eps, corners) == 1.0)
    assert np.all(r.nx[corners] == 7) and np.all(np.delete(r.nx, corners) == 3)
    closed = psi_int(4) + psi_int(16) - (4 * 2 * psi_int(8) + 12 * 2 * psi_int(4)) / 16
    assert abs(r.mi - closed) < 1e-9
    # k=1 on the same grid: eps = 1, n = 3 everywhere
    r1 = orc.window(x, y, k=1)
    assert abs(r1.mi - (psi_int(1) + psi_int(16) - 2 * psi_int(4))) < 1e-9


def test_constant_series_degenerate(orc):
    w, k = 50, 4
    x = np.full(w, 3.25, np.float32)
    r = orc.window(x, x, k=k)
    # every eps = 0; strict counts are 0; Z = w => degenerate normalized MI
    assert np.all(r.eps == 0) and np.all(r.nx == 0) and r.zero_eps == w
    assert abs(r.mi - (psi_int(k) + psi_int(w) - 2 * psi_int(1))) < 1e-9
    assert r.h == -math.inf and r.nmi == 1.0


def test_duplicated_points_eps_zero(orc):
    # every point has >= k exact duplicates -> eps_i = 0 for all i
    base = np.array([0, 1, 2, 3, 5, 7], np.float32)
    x = np.repeat(base, 5)
    y = np.repeat(base[::-1].copy(), 5)
    r = orc.window(x, y, k=4)
    assert np.all(r.eps == 0) and r.zero_eps == len(x)


# ---------------------------------------------------------------- the paper's worked example
def test_ksg2_worked_example_p671(orc):
    # k=2, p1's nearest are p2, p3; n_x = 3 (p2, p3, p5), n_y = 3 (p2, p3, p4).
    # Coordinates constructed to satisfy the figure's description (the figure itself is missing).
    pts = [(0.0, 0.0), (1.0, 0.5), (-0.5, -0.75), (5.0, 0.25), (0.25, 6.0), (4.0, 4.0), (-3.0, 3.0)]
    x = np.array([p[0] for p in pts], np.float32)
    y = np.array([p[1] for p in pts], np.float32)
    r2 = orc.window(x, y, k=2, variant=1)
    assert r2.nx[0] == 3 and r2.ny[0] == 3
    # KSG-1 on the same points: strict counts inside eps_1 = 1 exclude p2 (|dx| = 1 = eps)
    r1 = orc.window(x, y, k=2, variant=0)
    assert r1.eps[0] == 1.0 and r1.nx[0] == 2 and r1.ny[0] == 3


# ---------------------------------------------------------------- brute force (different algorithm)
def _brute_ksg1(x, y, k):
    x = x.astype(np.float32)
    y = y.astype(np.float32)
    dx = np.abs(x[:, None] - x[None, :])  # float32 differences, full matrix
    dy = np.abs(y[:, None] - y[None, :])
    d = np.maximum(dx, dy)
    w = len(x)
    eps = np.empty(w, np.float32)
    nx = np.empty(w, np.int64)
    ny = np.empty(w, np.int64)
    for i in range(w):
        row = np.sort(np.concatenate([d[i, :i], d[i, i + 1:]]))
        eps[i] = row[k - 1]
        nx[i] = int(np.sum(dx[i] < eps[i])) - (1 if eps[i] > 0 else 0)
        ny[i] = int(np.sum(dy[i] < eps[i])) - (1 if eps[i] > 0 else 0)
    mi = psi_int(k) + psi_int(w) - sum(psi_int(a + 1) + psi_int(b + 1) for a, b in zip(nx, ny)) / w
    return eps, nx, ny, mi


@pytest.mark.parametrize("seed,w,k,kind", [(0, 12, 1, "normal"), (1, 20, 3, "normal"), (2, 33, 4, "int"),
                                           (3, 40, 8, "int"), (4, 17, 16, "normal"), (5, 64, 4, "mixed")])
def test_brute_force_tiny_windows(orc, seed, w, k, kind):
    rng = np.random.default_rng(seed)
    if kind == "normal":
        x, y = rng.normal(size=w), rng.normal(size=w)
    elif kind == "int":
        x, y = rng.integers(0, 8, w), rng.integers(0, 8, w)
    else:
        x, y = rng.normal(size=w), rng.integers(0, 4, w)
    x = x.astype(np.float32)
    y = y.astype(np.float32)
    eps, nx, ny, mi = _brute_ksg1(x, y, k)
    r = orc.window(x, y, k=k)
    assert np.array_equal(r.eps, eps)
    assert np.array_equal(r.nx, nx) and np.array_equal(r.ny, ny)
    assert abs(r.mi - mi) < 1e-9


def test_eps_two_methods_agree(orc):
    x, y = datagen.gaussian_pair(300, 0.6, seed=9)
    xi = np.round(x * 4).astype(np.float32)  # heavy ties
    for xx, yy in ((x, y), (xi, y), (xi, np.round(y).astype(np.float32))):
        a = orc.window(xx, yy, k=4, eps_method=0)
        b = orc.window(xx, yy, k=4, eps_method=1)
        assert np.array_equal(a.eps, b.eps) and a.s_psi == b.s_psi and a.mi == b.mi


def test_canonical_vs_plain_within_1e9(orc):
    for rho, seed in ((0.0, 1), (0.9, 2)):
        x, y = datagen.gaussian_pair(2048, rho, seed=seed)
        r = orc.window(x, y)
        assert abs(r.mi - r.mi_plain) <= 1e-9
        assert abs(r.h - r.h_plain) <= 1e-9


def _ksg2_brute(x, y, k):
    # KSG-2 by full (d, j) sorting on a tiny window
    w = len(x)
    nx = []
    ny = []
    for i in range(w):
        cand = sorted((max(abs(np.float32(x[i] - x[j])), abs(np.float32(y[i] - y[j]))), j) for j in range(w) if j != i)
        knn = [j for _, j in cand[:k]]
        dxk = max(abs(np.float32(x[i] - x[j])) for j in knn)
        dyk = max(abs(np.float32(y[i] - y[j])) for j in knn)
        nx.append(sum(1 for j in range(w) if j != i and abs(np.float32(x[i] - x[j])) <= dxk))
        ny.append(sum(1 for j in range(w) if j != i and abs(np.float32(y[i] - y[j])) <= dyk))
    mi = psi_int(k) - 1.0 / k + psi_int(w) - sum(psi_int(a) + psi_int(b) for a, b in zip(nx, ny)) / w
    return np.array(nx), np.array(ny), mi


@pytest.mark.parametrize("seed,w,k", [(0, 15, 2), (1, 30, 4), (2, 24, 3)])
def test_ksg2_brute_force(orc, seed, w, k):
    rng = np.random.default_rng(seed)
    x = rng.integers(0, 6, w).astype(np.float32)
    y = rng.normal(size=w).astype(np.float32)
    nx, ny, mi = _ksg2_brute(x, y, k)
    r = orc.window(x, y, k=k, variant=1)
    assert np.array_equal(r.nx, nx) and np.array_equal(r.ny, ny)
    assert abs(r.mi - mi) < 1e-9
    assert np.all(r.nx >= k) and np.all(r.ny >= k)


# ---------------------------------------------------------------- exact invariants (bitwise)
def test_invariances_bitwise(orc):
    x, y = datagen.gaussian_pair(257, 0.7, seed=3)
    base = orc.window(x, y, k=4)
    # symmetry MI(x,y) = MI(y,x) (north star)
    assert orc.window(y, x, k=4).mi == base.mi
    # negation of either marginal
    assert orc.window(-x, y, k=4).mi == base.mi
    assert orc.window(x, -y, k=4).mi == base.mi
    # permutation of the points inside the window
    perm = np.random.default_rng(0).permutation(len(x))
    assert orc.window(x[perm], y[perm], k=4).mi == base.mi
    # joint scaling by 2^j is exact in float32 (normal range)
    for j in (-3, 5):
        s = np.float32(2.0 ** j)
        r = orc.window(x * s, y * s, k=4)
        assert r.mi == base.mi
        assert abs(r.h - (base.h + 2 * j * math.log(2))) < 1e-9  # KL entropy shifts by d*j*ln2


def test_integer_translation_invariance(orc):
    rng = np.random.default_rng(4)
    x = rng.integers(-50, 50, 200).astype(np.float32)
    y = rng.integers(-50, 50, 200).astype(np.float32)
    a = orc.window(x, y, k=3)
    b = orc.window(x + np.float32(1000), y - np.float32(77), k=3)
    assert a.mi == b.mi and a.s_psi == b.s_psi


# ---------------------------------------------------------------- statistical closed forms
@pytest.mark.parametrize("rho", [0.0, 0.5, 0.9])
def test_gaussian_convergence_to_closed_form(orc, rho):
    vals, hs = [], []
    for s in range(5):
        x, y = datagen.gaussian_pair(4096, rho, seed=100 + s)
        r = orc.window(x, y, k=4)
        vals.append(r.mi)
        hs.append(r.h)
    closed = -0.5 * math.log(1 - rho * rho)
    assert abs(np.mean(vals) - closed) <= 0.03
    # KL joint entropy of a unit-variance bivariate Gaussian: ln(2 pi e) + 1/2 ln(1 - rho^2)
    assert abs(np.mean(hs) - (math.log(2 * math.pi * math.e) + 0.5 * math.log(1 - rho * rho))) <= 0.04


def test_independent_near_zero(orc):
    for s in range(3):
        st = datagen.Stream(50 + s, 3)
        x = datagen.f32(st.uniform(1000))
        y = datagen.f32(st.uniform(1000))
        r = orc.window(x, y, k=4)
        assert abs(r.mi) < 0.05
        # S:148 normalized MI of an independent pair; on O(1)-scale data (KL H ~ 2.8 nats).
        # On the unit square H ~ 0 and I/H is meaningless: the scale hazard of reading R5.
        xn, yn = datagen.gaussian_pair(1000, 0.0, seed=60 + s)
        assert orc.window(xn, yn, k=4).nmi < 0.05


def test_entropy_uniform_square(orc):
    # uniform on [0,1]^2 -> 0 nats; on [0,e]^2 -> 2 nats (+-0.15)
    st = datagen.Stream(7, 3)
    u = st.uniform(4000).reshape(2, -1)
    r = orc.window(datagen.f32(u[0]), datagen.f32(u[1]))
    assert abs(r.h) < 0.15
    r = orc.window(datagen.f32(u[0] * math.e), datagen.f32(u[1] * math.e))
    assert abs(r.h - 2.0) < 0.15


RELATIONS = ["linear", "quadratic", "diamond", "circle", "sine", "cross", "quartic", "sqrt"]


@pytest.mark.parametrize("kind", RELATIONS)
def test_table2_relations_flagged(orc, kind):
    # Table 2: every relation family is correlated at sigma = 0.2 on normalized MI.
    x, y = datagen.table2_relation(kind, 1000, seed=1)
    assert orc.window(x, y, k=4).nmi >= 0.2


def test_table2_independent_not_flagged(orc):
    x, y = datagen.table2_relation("independent", 1000, seed=1)
    assert orc.window(x, y, k=4).nmi < 0.2


@pytest.mark.xfail(reason="KL entropy normalizer is scale dependent: y=0.01^(x+u) spans 40 decades, "
                          "H ~ 21.6 nats so I/H < sigma (DESIGN.md reading R5 hazard)", strict=True)
def test_table2_exponential_flagged(orc):
    x, y = datagen.table2_relation("exponential", 1000, seed=1)
    assert orc.window(x, y, k=4).nmi >= 0.2


def test_theorem1_mixture_direction(orc):
    # Theorem 1 / Eq. 18 with independently drawn labels (G9): I(Z;W) ~ theta*eta*I(X;Y).
    st = datagen.Stream(31, 1)
    n = 4000
    x, y = datagen.gaussian_pair(n, 0.9, seed=31)
    ixy = orc.window(x, y).mi
    # contaminants on a support disjoint from (X, Y), as the proof's range split assumes
    u = datagen.f32(st.uniform(n) * 4 + 10)
    v = datagen.f32(st.uniform(n) * 4 + 10)
    th = st.uniform(n) < 0.5
    et = st.uniform(n) < 0.5
    z = np.where(th, x, u).astype(np.float32)
    w = np.where(et, y, v).astype(np.float32)
    izw = orc.window(z, w).mi
    assert izw < ixy
    assert 0.1 <= izw / ixy <= 0.4  # Eq. 18 predicts 0.25


def test_table2_alternative_reading_evaluated(orc):
    """Reading R5 evaluation: the scale-free alternative normalizer I~_L = 1 - exp(-2 MI)
    (Linfoot's informational coefficient, squared) flags all ten Table 2 relations incl. the exponential
    family and not the independent pair -- but it also flags pure-background windows of configs[0]
    at w = 64 (KSG's small-w bias: MI up to ~0.12 nats on independent data), which would break the planted-
    recovery pins; so the KL normalizer stays and test_table2_exponential_flagged stays a strict xfail."""
    lin = lambda mi: 1.0 - math.exp(-2.0 * max(mi, 0.0))
    for kind in RELATIONS + ["exponential"]:
        x, y = datagen.table2_relation(kind, 1000, seed=1)
        assert lin(orc.window(x, y, k=4).mi) >= 0.2, kind
    x, y = datagen.table2_relation("independent", 1000, seed=1)
    assert lin(orc.window(x, y, k=4).mi) < 0.2
    wl = datagen.cfg1()
    x, y = wl.series
    W = [(a, b) for a, b in datagen.sweep_windows(len(x), [64], 8)            # configs[0] sweep, w = 64,
         if b <= 500 or (a >= 800 and b <= 1200) or a >= 1500]               # background windows only
    r = orc.mi_batch(x, y, W, 4)
    assert max(lin(v) for v in r["mi"]) >= 0.2   # a background false positive under the alternative
    assert max(r["nmi"]) < 0.2                   # none under the KL reading
