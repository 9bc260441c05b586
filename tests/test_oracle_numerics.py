"""Pins for the oracle's canonical numerics (DESIGN.md §Canonical numerics).

The digamma table and the canonical log are pinned to things other than
themselves: scipy's digamma, the digamma asymptotic series, Python's libm log,
and exact identities.
"""
import math

import numpy as np
import pytest


def test_psi_recurrence_identities(orc):
    t = orc.psi_table(100)
    # S:118 digamma(1) = -gamma;  S:119 digamma(2) = digamma(1) + 1 exactly
    assert t[1] == -0.57721566490153286061
    assert t[2] == t[1] + 1.0
    assert math.isnan(t[0])


def test_psi_vs_scipy_digamma(orc):
    from scipy.special import digamma

    m_max = 1 << 18
    t = orc.psi_table(m_max)
    ms = np.array([1, 2, 3, 4, 5, 8, 17, 100, 1000, 4097, 65536, 65537, m_max])
    err = np.abs(t[ms] - digamma(ms.astype(np.float64)))
    assert err.max() < 5e-13, err


def test_psi_vs_asymptotic_series(orc):
    # psi(m) = ln m - 1/(2m) - 1/(12 m^2) + 1/(120 m^4) - 1/(252 m^6) + ...
    t = orc.psi_table(5000)
    for m in (20, 100, 1000, 5000):
        series = math.log(m) - 1 / (2 * m) - 1 / (12 * m**2) + 1 / (120 * m**4) - 1 / (252 * m**6)
        assert abs(t[m] - series) < 1e-11


def _ulp_diff(a, b):
    ia = np.frombuffer(np.float64(a).tobytes(), np.int64)[0]
    ib = np.frombuffer(np.float64(b).tobytes(), np.int64)[0]
    return abs(int(ia) - int(ib))


def test_canonical_ln_within_2ulp_of_libm(orc):
    rng = np.random.default_rng(1)
    # float32 radii across the whole range, doubled (v = 2*eps exact in double)
    e = rng.uniform(-120, 120, 4000)
    eps = (2.0 ** e).astype(np.float32)
    special = np.array([1e-45, 1.17549435e-38, 1e-30, 0.5, 1.0, 1.5, 2.0, 3.4028235e38 / 2], np.float32)
    for v in np.concatenate([eps, special]):
        if v <= 0:
            continue
        d = 2.0 * float(v)
        got = orc.ln(d)
        ref = math.log(d)
        if ref == 0.0:
            assert got == 0.0
        else:
            assert _ulp_diff(got, ref) <= 2, (v, got, ref)


def test_canonical_ln_exact_points(orc):
    assert orc.ln(1.0) == 0.0
    assert orc.ln(2.0) == 0.69314718055994530942
    assert orc.ln(0.5) == -0.69314718055994530942


def test_q32_round_half_even(orc):
    u = 2.0 ** -32
    assert orc.q32(0.5 * u) == 0
    assert orc.q32(1.5 * u) == 2
    assert orc.q32(2.5 * u) == 2
    assert orc.q32(-0.5 * u) == 0
    assert orc.q32(-1.5 * u) == -2
    assert orc.q32(1.0) == 1 << 32
    assert orc.q32(-0.57721566490153286061) == round(-0.57721566490153286061 * 2**32)
