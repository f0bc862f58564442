"""Pins of the oracle's noise primitives (NUMERICS N1–N5) against things other than itself:
published Philox known-answer vectors, exhaustive comparison with double-precision libm over the
complete 2^23-point input domains, and the statistics of N(0,1)."""
import json
import os

import numpy as np
import pytest
from scipy import stats

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_philox_known_answers(orc):
    kat = json.load(open(os.path.join(GOLD, "philox_kat.json")))
    for v in kat["vectors"]:
        out = orc.philox([int(h, 16) for h in v["ctr"]], [int(h, 16) for h in v["key"]])
        assert [f"{o:08x}" for o in out] == v["out"]


def _all_mantissas():
    return np.arange(2 ** 23, dtype=np.uint32)


def test_uniforms_exhaustive(orc):
    # u_a, u_b are exactly 1 - m 2^-23 and m 2^-23 for every 23-bit mantissa m (N3).
    lib = orc.lib()
    rng = np.random.default_rng(0)
    for m in list(rng.integers(0, 2 ** 23, 20000)) + [0, 1, 2 ** 23 - 1]:
        o = int(m) << 9 | int(rng.integers(0, 512))
        assert lib.orc_u_a(o) == 1.0 - int(m) * 2.0 ** -23
        assert lib.orc_u_b(o) == int(m) * 2.0 ** -23


def test_ln_exhaustive_vs_libm(orc):
    m = _all_mantissas().astype(np.float64)
    ua = (1.0 - m * 2.0 ** -23).astype(np.float32)          # every value u_a can take
    got = orc.ln(ua).astype(np.float64)
    ref = np.log(ua.astype(np.float64))
    assert got[0] == 0.0                                      # ln 1 = 0 exactly
    ulp = np.spacing(np.abs(ref).astype(np.float32)).astype(np.float64)
    err = np.abs(got - ref)[1:] / ulp[1:]
    assert err.max() <= 1.5, err.max()
    # and on general normal floats across many binades (the function is used only on u_a, but
    # a wrong exponent term would show here)
    rng = np.random.default_rng(1)
    u = np.exp2(rng.uniform(-120, 0, 200000)).astype(np.float32)
    got = orc.ln(u).astype(np.float64)
    ref = np.log(u.astype(np.float64))
    assert (np.abs(got - ref) / np.spacing(np.abs(ref).astype(np.float32))).max() <= 1.5


def test_sincos2pi_exhaustive_vs_libm(orc):
    ub = (_all_mantissas().astype(np.float64) * 2.0 ** -23).astype(np.float32)
    c, s = orc.sincos2pi(ub)
    th = 2 * np.pi * ub.astype(np.float64)
    for got, ref in ((c, np.cos(th)), (s, np.sin(th))):
        got = got.astype(np.float64)
        assert np.abs(got - ref).max() <= 1.0e-7
        big = np.abs(ref) >= 2.0 ** -6
        ulp = np.spacing(np.abs(ref[big]).astype(np.float32)).astype(np.float64)
        assert (np.abs(got[big] - ref[big]) / ulp).max() <= 2.0
    # exact special values
    c0, s0 = orc.sincos2pi(np.array([0.0, 0.25, 0.5, 0.75], np.float32))
    assert list(np.abs(c0)) == [1.0, 0.0, 1.0, 0.0] and list(np.abs(s0)) == [0.0, 1.0, 0.0, 1.0]
    assert c0[2] == -1.0 and s0[3] == -1.0


def test_sincos2pi_general_floats(orc):
    # Rastrigin feeds frac(|x|)/2, an arbitrary float in [0, 0.5)
    rng = np.random.default_rng(2)
    u = np.concatenate([rng.uniform(0, 0.5, 500000), np.exp2(rng.uniform(-60, -1, 100000))])
    u = u.astype(np.float32)
    c, s = orc.sincos2pi(u)
    th = 2 * np.pi * u.astype(np.float64)
    assert np.abs(c - np.cos(th)).max() <= 1.0e-7
    assert np.abs(s - np.sin(th)).max() <= 1.0e-7
    tiny = u < 1e-6                                  # relative accuracy of sin near 0
    assert np.all(np.abs(s[tiny] / np.sin(th[tiny]) - 1) < 3e-7)


def test_normals_distribution(orc):
    n = 4_000_000
    z = orc.normals(12345, 3, 7, 0, n).astype(np.float64)
    se = 1 / np.sqrt(n)
    assert abs(z.mean()) < 5 * se
    assert abs(z.var() - 1) < 5 * np.sqrt(2.0) * se
    assert abs(stats.kurtosis(z, fisher=False) - 3) < 5 * np.sqrt(24.0) * se
    assert abs(stats.skew(z)) < 5 * np.sqrt(6.0) * se
    assert stats.kstest(z[:1_000_000], "norm").pvalue > 1e-4
    assert np.abs(z).max() <= np.sqrt(-2 * np.log(2.0 ** -23)) + 1e-5   # Box–Muller tail bound


def test_streams_independent(orc):
    n = 400_000
    a = orc.normals(1, 0, 0, 0, n)
    b = orc.normals(1, 0, 0, 1, n)     # other tag
    c = orc.normals(2, 0, 0, 0, n)     # other seed
    d = orc.normals(1, 1, 0, 0, n)     # other direction
    e = orc.normals(1, 0, 1, 0, n)     # other generation
    for other in (b, c, d, e):
        assert abs(np.corrcoef(a, other)[0, 1]) < 5 / np.sqrt(n)
    # counter-based: the same (seed, i, t) regenerates the same row, independently of D
    z1 = orc.direction(9, 5, 3, 37)
    z2 = orc.direction(9, 5, 3, 1000)[:37]
    assert np.array_equal(z1.view(np.uint32), z2.view(np.uint32))
    assert np.array_equal(z1.view(np.uint32), orc.normals(9, 5, 3, 0, 37).view(np.uint32))


def test_sinpi_half_vs_libm(orc):
    """NUMERICS N7 Rastrigin factor S = sin(pi b), b in [0, 1/2]: <= 3 ulp and 2e-7 absolute against
    double libm over 4M points plus every float in [0, 2^-10)."""
    b = np.concatenate([np.linspace(0, 0.5, 4_000_001),
                        np.exp2(np.random.default_rng(3).uniform(-126, -10, 1_000_000))])
    b = b.astype(np.float32)
    got = orc.sinpi_half(b).astype(np.float64)
    ref = np.sin(np.pi * b.astype(np.float64))
    assert np.abs(got - ref).max() <= 2e-7
    nz = ref > 0
    assert (np.abs(got[nz] - ref[nz]) / np.spacing(ref[nz].astype(np.float32))).max() <= 3.0
    assert orc.sinpi_half(np.array([0.0, 0.5], np.float32))[0] == 0.0
