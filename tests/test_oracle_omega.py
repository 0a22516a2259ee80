"""Pins for the oracle's Ω generator (oracle/omega.py), independent of the oracle itself:
Random123 known-answer vectors, correctly rounded references (mpmath), distribution tests,
and the sharding/blocking contract of DESIGN.md §3.3 (readings R14, R15)."""
import json
import os

import mpmath
import numpy as np
import pytest
from scipy import stats

from oracle import omega

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_worked_examples.json")))


def test_philox_known_answers():
    for case in GOLD["philox4x32_10_kat"]["cases"]:
        ctr = [int(h, 16) for h in case["ctr"]]
        key = [int(h, 16) for h in case["key"]]
        out = omega.philox4x32_10(*ctr, *key)
        assert [int(v) for v in out] == [int(h, 16) for h in case["out"]]


def test_philox_vectorised_equals_scalar():
    rng = np.random.default_rng(3)
    c = rng.integers(0, 2**32, size=(4, 64), dtype=np.uint64).astype(np.uint32)
    k = rng.integers(0, 2**32, size=(2, 64), dtype=np.uint64).astype(np.uint32)
    vec = omega.philox4x32_10(*c, *k)
    for i in range(64):
        one = omega.philox4x32_10(*(int(x[i]) for x in c), *(int(x[i]) for x in k))
        assert [int(v[i]) for v in vec] == [int(v) for v in one]


def _ulp_err(got, ref):
    ref = float(ref)
    if ref == 0.0:
        return 0.0 if got == 0.0 else np.inf
    return abs(got - ref) / np.spacing(abs(ref))


def test_coefficients_are_correctly_rounded():
    mpmath.mp.prec = 200
    for k in range(11):
        s = (-1) ** k * mpmath.pi ** (2 * k + 1) / mpmath.factorial(2 * k + 1)
        c = (-1) ** k * mpmath.pi ** (2 * k) / mpmath.factorial(2 * k)
        assert omega.SINPI_C[k] == float(s)
        assert omega.COSPI_C[k] == float(c)
    mpmath.mp.prec = 200
    ln2 = mpmath.log(2)
    assert abs(mpmath.mpf(omega.LN2_HI) + mpmath.mpf(omega.LN2_LO) - ln2) < mpmath.mpf(2) ** -100
    assert float.fromhex("0x1p+43") * omega.LN2_HI == float(mpmath.mpf(2) ** 43 * mpmath.mpf(omega.LN2_HI))


def test_spec_log_within_2ulp():
    mpmath.mp.prec = 120
    rng = np.random.default_rng(5)
    x = np.concatenate([rng.random(1500), 2.0 ** -rng.integers(1, 53, 300) * (1 + rng.random(300)) / 2,
                        [1.0, 2.0 ** -53, 0.5, omega.SQRT2 / 2, np.nextafter(omega.SQRT2 / 2, 0), 0.75]])
    x = x[(x > 0) & (x <= 1)]
    got = omega.spec_log(x)
    worst = max(_ulp_err(g, mpmath.log(mpmath.mpf(float(v)))) for g, v in zip(got, x))
    assert worst <= 2.0
    assert omega.spec_log(np.array([1.0]))[0] == 0.0


def test_spec_sincospi_within_1ulp():
    mpmath.mp.prec = 120
    rng = np.random.default_rng(6)
    t = np.concatenate([rng.random(1500) * 2, [0.0, 0.25, 0.5, 0.75, 1.0, 1.25, 1.5, 1.75,
                                               2 - 2.0 ** -52, 2.0 ** -52, 0.125, 1.875]])
    s, c = omega.spec_sincospi(t)
    for ti, si, ci in zip(t, s, c):
        S = float(mpmath.sinpi(mpmath.mpf(float(ti))))
        C = float(mpmath.cospi(mpmath.mpf(float(ti))))
        assert abs(si - S) <= np.spacing(max(abs(S), 2.0 ** -60))
        assert abs(ci - C) <= np.spacing(max(abs(C), 2.0 ** -60))


def test_gaussian_distribution():
    O = omega.omega_panel(seed=7, n=200_001, col0=3, w=5)
    x = O.ravel()
    N = x.size
    assert abs(x.mean()) < 5 / np.sqrt(N)
    assert abs(x.var() - 1.0) < 5 * np.sqrt(2.0 / N)
    assert stats.kstest(x, "norm").pvalue > 1e-4
    # independent columns and independent even/odd rows
    assert abs(np.corrcoef(O[:, 0], O[:, 1])[0, 1]) < 5 / np.sqrt(O.shape[0])
    assert abs(np.corrcoef(O[0::2, 2][:100_000], O[1::2, 2][:100_000])[0, 1]) < 5 / np.sqrt(100_000)


def test_box_muller_radius_relation():
    # Ω(2p)^2 + Ω(2p+1)^2 = -2 ln U1 with U1 = (a + 1) 2^-53 from the counter's first word pair
    p = np.arange(50, dtype=np.uint64)
    e, o = omega.gaussian_pairs(11, p, np.uint64(4))
    x, y, _, _ = omega.philox4x32_10(p & np.uint64(0xFFFFFFFF), np.zeros(50, np.uint64), 4, 0, 11, 0)
    a = ((x.astype(np.uint64) << np.uint64(32)) | y.astype(np.uint64)) >> np.uint64(11)
    u1 = (a + np.uint64(1)).astype(np.float64) * 2.0 ** -53
    np.testing.assert_allclose(e * e + o * o, -2.0 * np.log(u1), rtol=1e-13, atol=1e-300)


@pytest.mark.parametrize("row0,row1", [(0, 1001), (1, 1001), (7, 500), (500, 501), (999, 1001), (2, 4)])
def test_row_shards_bitwise(row0, row1):
    full = omega.omega_panel(3, 1001, 10, 6)
    part = omega.omega_panel(3, 1001, 10, 6, row0, row1)
    assert np.array_equal(full[row0:row1], part)


def test_columns_depend_only_on_global_index():
    wide = omega.omega_panel(9, 333, 0, 40)
    for c0, w in [(0, 5), (5, 10), (17, 23), (39, 1)]:
        assert np.array_equal(wide[:, c0:c0 + w], omega.omega_panel(9, 333, c0, w))
    assert not np.array_equal(omega.omega_panel(9, 333, 0, 4), omega.omega_panel(10, 333, 0, 4))
