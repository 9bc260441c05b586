"""Seeded synthetic inputs shaped like the paper's workloads (BASELINE.json configs[0..4]).

This module is shared by the oracle tests, the GPU parity tests, ``smoke()`` and
``bench.py``.  It holds NONE of the method's arithmetic (no distances, no
neighbour search, no digamma, no search logic): only random numbers and the
planted-relation formulas that define each synthetic workload.  The recipe for
every config is restated in DESIGN.md §"Input recipe".

Random numbers: SplitMix64 (Steele et al.) keyed by (seed, stream id); 53-bit
uniforms; N(0,1) by Box-Muller (cos branch) in fp64; Laplace by inverse CDF;
all arithmetic in fp64, cast to float32 (round to nearest) at the end.

The paper's own datasets (NYC Open Data taxi/weather/traffic, an NDA wind-farm
dataset, a Kaggle energy dataset; §8.2) are not available;
these generators stand in for them.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

_GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
_MASK64 = (1 << 64) - 1


def _mix(z: np.ndarray) -> np.ndarray:
    z = (z ^ (z >> np.uint64(30))) * _M1
    z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def stream_key(seed: int, stream: int) -> int:
    """Initial SplitMix64 state of stream ``stream`` under ``seed``."""
    return (int(seed) ^ ((int(stream) * 0x9E3779B97F4A7C15) & _MASK64)) & _MASK64


class Stream:
    """A SplitMix64 stream; draws are position-addressed so blocks are reproducible."""

    def __init__(self, seed: int, stream: int):
        self.state = np.uint64(stream_key(seed, stream))
        self.pos = 0  # number of 64-bit outputs consumed

    def u64(self, count: int) -> np.ndarray:
        idx = np.arange(self.pos + 1, self.pos + 1 + count, dtype=np.uint64)
        self.pos += count
        with np.errstate(over="ignore"):
            return _mix(self.state + idx * _GAMMA)

    def uniform(self, count: int) -> np.ndarray:
        """U[0,1) with 53 random bits."""
        return (self.u64(count) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)

    def uniform_open(self, count: int) -> np.ndarray:
        """U(0,1]: 1 - U[0,1)."""
        return 1.0 - self.uniform(count)

    def normal(self, count: int) -> np.ndarray:
        u1 = self.uniform_open(count)
        u2 = self.uniform(count)
        return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)

    def laplace(self, count: int, b: float) -> np.ndarray:
        u = self.uniform_open(count) - 0.5  # (-0.5, 0.5]
        u = np.where(u >= 0.5, 0.4999999999999999, u)
        return -b * np.sign(u) * np.log1p(-2.0 * np.abs(u))

    def integer(self, lo: int, hi: int) -> int:
        """Uniform integer in [lo, hi] (inclusive)."""
        span = hi - lo + 1
        return lo + int(self.uniform(1)[0] * span)

    def scalar(self) -> float:
        return float(self.uniform(1)[0])


def ar1(stream: Stream, n: int, phi: float, innov_std: float = 1.0) -> np.ndarray:
    """Stationary AR(1): x0 ~ N(0, s^2/(1-phi^2)), x_t = phi x_{t-1} + e_t (fp64)."""
    e = stream.normal(n) * innov_std
    e[0] = e[0] / math.sqrt(1.0 - phi * phi)
    try:
        from scipy.signal import lfilter

        return lfilter([1.0], [1.0, -phi], e)
    except Exception:  # pragma: no cover - scipy is in the image
        x = np.empty(n)
        acc = 0.0
        for t in range(n):
            acc = phi * acc + e[t] if t else e[0]
            x[t] = acc
        return x


def f32(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64).astype(np.float32))


# --------------------------------------------------------------------------------------
# Per-config search parameters (BASELINE.json configs; SURVEY §8(c).2 / §8(d) readings)
# --------------------------------------------------------------------------------------
@dataclass
class SearchConfig:
    k: int = 4
    s_min: int = 64
    s_max: int = 512
    sigma: float = 0.2
    tau_ratio: float = 0.25
    p: int = 3
    h: int = 5
    t_max_idle: int = 3
    delta_td: int = 0  # 0 => max(1, s/4) per layer
    delta_bu: int = 0  # 0 => max(1, s_min/3)
    n_chunks: int = 1
    method: int = 3  # 1 TD, 2 BU, 3 BOTH, 4 AUTO (iSYCOS, Alg. 3)
    noise: bool = True
    seed: int = 0
    sizes: list = field(default_factory=list)  # explicit TD layer sizes; [] => halving
    auto_M: int = 0  # AUTO: partitions (0 => 20)
    auto_m: int = 0  # AUTO: sampled partitions (0 => 6)
    auto_alpha: float = 0.0  # AUTO: runtime weight (0 => 0.5)
    auto_rho: float = 0.0  # AUTO: small-window cut rho * s_max (0 => 0.5)


@dataclass
class Workload:
    name: str
    series: list  # list of float32 arrays (all the same length)
    pairs: list  # list of (xs, ys)
    search: SearchConfig
    sweep: dict | None = None  # {"sizes": [...], "stride": s, "ks": [...]}
    planted: dict = field(default_factory=dict)  # pair index -> list of (t0, t1, kind)


def cfg1(seed: int = 0, n: int = 2048) -> Workload:
    """configs[0]: n=2048, x,y iid N(0,1); y = x^2 + 0.1e on [500,800), y = -x + 0.1e on [1200,1500)."""
    st = Stream(seed, 1)
    x = st.normal(n)
    y = st.normal(n)
    e = st.normal(n)
    y = y.copy()
    y[500:800] = x[500:800] ** 2 + 0.1 * e[500:800]
    y[1200:1500] = -x[1200:1500] + 0.1 * e[1200:1500]
    sc = SearchConfig(k=4, s_min=64, s_max=512, seed=seed)
    return Workload(
        name="cfg1",
        series=[f32(x), f32(y)],
        pairs=[(0, 1)],
        search=sc,
        sweep={"sizes": [64, 128, 256, 512], "stride": 8, "ks": [4]},
        planted={0: [(500, 800, "quadratic"), (1200, 1500, "neg-linear")]},
    )


def cfg2(seed: int = 2, n: int = 100_000) -> Workload:
    """configs[1]: AR(1) phi=0.9 background + linear/quadratic/sine/circle planted at 4 scales."""
    st = Stream(seed, 1)
    x = ar1(st, n, 0.9)
    y = ar1(st, n, 0.9)
    e = st.normal(n) * 0.2
    planted = []
    spans = [
        (10_000, 200, "linear"),
        (30_000, 2_000, "quadratic"),
        (50_000, 8_000, "sine"),
        (70_000, 20_000, "circle"),
    ]
    for (a, L, kind) in spans:
        if a + L > n:
            continue
        s = slice(a, a + L)
        if kind == "linear":
            y[s] = 2.0 * x[s] + e[s]
        elif kind == "quadratic":
            y[s] = x[s] ** 2 + e[s]
        elif kind == "sine":
            y[s] = np.sin(3.0 * x[s]) + e[s]
        else:
            u = st.uniform(L) * (2.0 * math.pi)
            x[s] = np.cos(u)
            y[s] = np.sin(u)
        planted.append((a, a + L, kind))
    sc = SearchConfig(k=4, s_min=32, s_max=4096, seed=seed, noise=True, method=3)
    return Workload(name="cfg2", series=[f32(x), f32(y)], pairs=[(0, 1)], search=sc,
                    planted={0: planted})


def cfg3(seed: int = 3, n_segments: int = 20, seg_len: int = 50_000) -> Workload:
    """configs[2]: 20 bivariate-Gaussian segments, rho_s = 0.05 s (SURVEY G11 reading)."""
    st = Stream(seed, 1)
    xs, ys = [], []
    for s in range(n_segments):
        rho = 0.05 * s
        z1 = st.normal(seg_len)
        z2 = st.normal(seg_len)
        xs.append(z1)
        ys.append(rho * z1 + math.sqrt(1.0 - rho * rho) * z2)
    x = np.concatenate(xs)
    y = np.concatenate(ys)
    return Workload(
        name="cfg3",
        series=[f32(x), f32(y)],
        pairs=[(0, 1)],
        search=SearchConfig(k=4, seed=seed),
        sweep={"sizes": [1024, 4096, 16384], "stride": 512, "ks": [3, 4, 8], "seg_len": seg_len},
    )


def cfg4(seed: int = 4, n: int = 1_000_000, n_series: int = 64, n_planted: int = 10) -> Workload:
    """configs[3]: 64 sensor-like series (AR(1) 0.95 + daily sinusoid + N(0,0.3^2)); 10 planted pairs."""
    st = Stream(seed, 1)
    t = np.arange(n, dtype=np.float64)
    daily = np.sin(2.0 * math.pi * t / 1440.0)
    series = []
    for i in range(n_series):
        si = Stream(seed, 100 + i)
        a = ar1(si, n, 0.95)
        series.append(a + daily + 0.3 * si.normal(n))
    # planted pairs (2m, 2m+1), m without replacement from 0..n_series/2-1
    ms = list(range(n_series // 2))
    chosen = []
    for _ in range(min(n_planted, len(ms))):
        j = st.integer(0, len(ms) - 1)
        chosen.append(ms.pop(j))
    planted = {}
    for m in chosen:
        L = int(round(math.exp(math.log(500.0) + st.scalar() * (math.log(50_000.0) - math.log(500.0)))))
        L = min(L, n)
        a = st.integer(0, n - L)
        xi, yi = 2 * m, 2 * m + 1
        e = st.normal(L) * 0.3
        series[yi][a:a + L] = np.exp(series[xi][a:a + L] / 2.0) + e
        planted[(xi, yi)] = [(a, a + L, "exp")]
    pairs = [(i, j) for i in range(n_series) for j in range(i + 1, n_series)]
    pl = {pairs.index(k): v for k, v in planted.items()}
    sc = SearchConfig(k=4, s_min=64, s_max=16384, seed=seed, method=3, noise=True)
    return Workload(name="cfg4", series=[f32(s) for s in series], pairs=pairs, search=sc, planted=pl)


def cfg5(seed: int = 5, n: int = 10_000_000, n_series: int = 16, n_chunks: int = 16) -> Workload:
    """configs[4]: random walks with 30% Laplace/impulse noise segments; planted linear/quadratic/step."""
    st = Stream(seed, 1)
    series = []
    noise_segs = []
    for i in range(n_series):
        si = Stream(seed, 100 + i)
        r = np.cumsum(si.normal(n))
        r = r - r[0]  # r[0] = 0
        segs = []
        covered = 0
        target = 0.3 * n
        tries = 0
        lo_len, hi_len = min(1000, n // 10), min(100_000, n // 4)
        while covered < target and tries < 10_000:
            tries += 1
            L = int(round(math.exp(math.log(lo_len) + si.scalar() * (math.log(hi_len) - math.log(lo_len)))))
            a = si.integer(0, n - L)
            if any(a < b1 and b0 < a + L for (b0, b1, _) in segs):
                continue
            kind = "laplace" if si.scalar() < 0.5 else "impulse"
            if kind == "laplace":
                r[a:a + L] = si.laplace(L, 2.0)
            else:
                spikes = si.uniform(L) < 0.01
                sign = np.where(si.uniform(L) < 0.5, -1.0, 1.0)
                r[a:a + L] = r[a:a + L] + np.where(spikes, 20.0 * sign, 0.0)
            segs.append((a, a + L, kind))
            covered += L
        series.append(r)
        noise_segs.append(sorted(segs))
    planted = {}
    pairs = [(i, j) for i in range(n_series) for j in range(i + 1, n_series)]
    for m in range(n_series // 2):
        xi, yi = 2 * m, 2 * m + 1
        placed = []
        for kind in ("linear", "quadratic", "step"):
            for _ in range(1000):
                L = int(round(math.exp(math.log(min(1000, n // 20)) + st.scalar()
                                       * (math.log(min(65_536, n // 8)) - math.log(min(1000, n // 20))))))
                a = st.integer(0, n - L)
                clash = any(a < b1 and b0 < a + L for (b0, b1, _) in noise_segs[yi]) or any(
                    a < b1 and b0 < a + L for (b0, b1, _) in placed)
                if not clash:
                    break
            else:
                continue
            xw = series[xi][a:a + L]
            u = (xw - xw.mean()) / (xw.std() if xw.std() > 0 else 1.0)
            e = st.normal(L) * 0.2
            if kind == "linear":
                series[yi][a:a + L] = 2.0 * u + e
            elif kind == "quadratic":
                series[yi][a:a + L] = u * u + e
            else:
                series[yi][a:a + L] = np.sign(u) + e
            placed.append((a, a + L, kind))
        planted[pairs.index((xi, yi))] = sorted(placed)
    sc = SearchConfig(k=4, s_min=128, s_max=65_536, seed=seed, method=1, noise=True, n_chunks=n_chunks)
    return Workload(name="cfg5", series=[f32(s) for s in series], pairs=pairs, search=sc, planted=planted)


def scenario(kind: str, seed: int = 0, n: int = 8192) -> Workload:
    """Fig. 1 scenarios (the figures are missing, the text defines them): "dense" = large
    correlated windows located close or next to each other (the top-down case); "sparse" = small
    correlated windows sparsely distributed (the bottom-up case).  x, e ~ N(0,1); outside the planted
    windows y ~ N(0,1) independent; inside y = x + 0.3 e.  Search: s_min 64, s_max 1024, method AUTO with
    M = 8 partitions of 1024 samples, m = 4 sampled."""
    st = Stream(seed, 21 if kind == "dense" else 22)
    x = st.normal(n)
    y = st.normal(n)
    e = st.normal(n)
    planted = []
    if kind == "dense":      # blocks of 1024-2048 separated by gaps of 64-192 samples
        t = st.integer(0, 128)
        while True:
            L = st.integer(1024, 2048)
            if t + L > n:
                break
            planted.append((t, t + L))
            t += L + st.integer(64, 192)
    elif kind == "sparse":   # windows of 64-128 samples, 600-1000 apart
        t = st.integer(100, 400)
        while True:
            L = st.integer(64, 128)
            if t + L > n:
                break
            planted.append((t, t + L))
            t += L + st.integer(600, 1000)
    else:
        raise ValueError(kind)
    for (a, b) in planted:
        y[a:b] = x[a:b] + 0.3 * e[a:b]
    sc = SearchConfig(k=4, s_min=64, s_max=1024, seed=seed, method=4, auto_M=8, auto_m=4)
    return Workload(name=f"scenario-{kind}", series=[f32(x), f32(y)], pairs=[(0, 1)], search=sc,
                    planted={0: [(a, b, "linear") for (a, b) in planted]})


def sweep_windows(n: int, sizes, stride: int):
    """All windows [t, t+w) with t on the stride grid, for each size (the config sweeps)."""
    out = []
    for w in sizes:
        for t in range(0, n - w + 1, stride):
            out.append((t, t + w))
    return np.asarray(out, dtype=np.int64).reshape(-1, 2)


# Table 2 relation families, u ~ U(0,1).  Used only as statistical fixtures.
def table2_relation(kind: str, n: int, seed: int = 0):
    st = Stream(seed, 7)
    u = st.uniform(n)
    if kind == "independent":
        y = st.normal(n)
        x = 3.0 + 5.0 * st.normal(n)
        return f32(x), f32(y)
    ranges = {
        "linear": (0, 10), "exponential": (-10, 10), "quadratic": (-4, 4), "diamond": (4, 8),
        "circle": (-3, 3), "sine": (0, 10), "cross": (-5, 5), "quartic": (-1, 3), "sqrt": (0, 25),
    }
    a, b = ranges[kind]
    x = np.sort(a + (b - a) * st.uniform(n))
    br = st.uniform(n)
    if kind == "linear":
        y = 2 * x + u
    elif kind == "exponential":
        y = 0.01 ** (x + u)
    elif kind == "quadratic":
        y = x * x + u
    elif kind == "diamond":
        q = (br * 4).astype(int)
        y = np.choose(q, [x + u, 8 - x + u, -4 + x + u, 12 - x + u])
    elif kind == "circle":
        y = np.where(br < 0.5, 1.0, -1.0) * np.sqrt(np.maximum(9.0 - x * x + u, 0.0))
    elif kind == "sine":
        y = 2 * np.sin(x) + u
    elif kind == "cross":
        y = np.where(br < 0.5, x + u, -x + u)
    elif kind == "quartic":
        y = x ** 4 - 4 * x ** 3 + 4 * x ** 2 + x + u
    elif kind == "sqrt":
        y = np.sqrt(x)
    else:
        raise ValueError(kind)
    return f32(x), f32(y)


def gaussian_pair(n: int, rho: float, seed: int = 0, stream: int = 11):
    st = Stream(seed, stream)
    z1 = st.normal(n)
    z2 = st.normal(n)
    return f32(z1), f32(rho * z1 + math.sqrt(1.0 - rho * rho) * z2)


CONFIGS = {"cfg1": cfg1, "cfg2": cfg2, "cfg3": cfg3, "cfg4": cfg4, "cfg5": cfg5}
