"""Pins of the oracle's fitness (N7), ranking (N9–N10) and weights (N11) against hand values the
SPEC prints, textbook formulas evaluated independently in numpy, brute force and closed forms."""
import json
import os

import numpy as np
import pytest

import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")
FN = {"sphere": W.SPHERE, "rosenbrock": W.ROSENBROCK, "rastrigin": W.RASTRIGIN}


def test_bbob_hand_values(orc):
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for ex in g["bbob"]:
        assert orc.evaluate(FN[ex["fn"]], np.array(ex["x"], np.float32))[0] == ex["f"], ex


def _textbook(fn, x):
    x = x.astype(np.float64)
    if fn == W.SPHERE:
        return (x * x).sum(1)
    if fn == W.ROSENBROCK:
        return (100 * (x[:, 1:] - x[:, :-1] ** 2) ** 2 + (1 - x[:, :-1]) ** 2).sum(1)
    return 10 * x.shape[1] + (x * x - 10 * np.cos(2 * np.pi * x)).sum(1)   # textbook Rastrigin


@pytest.mark.parametrize("fn", [W.SPHERE, W.ROSENBROCK, W.RASTRIGIN])
@pytest.mark.parametrize("D", [1, 2, 7, 100, 1000])
def test_bbob_vs_textbook(orc, fn, D):
    rng = np.random.default_rng(D * 10 + fn)
    x = W.random_population(rng, 64, D, scale=2.5)
    got = orc.evaluate(fn, x).astype(np.float64)
    ref = _textbook(fn, x)
    tol = 2e-6 if fn != W.RASTRIGIN else 1e-5   # Rastrigin textbook form cancels in double
    assert np.all(np.abs(got - ref) <= tol * np.maximum(np.abs(ref), 1e-3)), np.abs(got - ref).max()
    assert np.all(got >= 0)


def test_bbob_optima(orc):
    assert orc.evaluate(W.SPHERE, np.zeros((1, 50), np.float32))[0] == 0
    assert orc.evaluate(W.RASTRIGIN, np.zeros((1, 50), np.float32))[0] == 0
    assert orc.evaluate(W.ROSENBROCK, np.ones((1, 50), np.float32))[0] == 0
    # Rastrigin: integer points give sum x^2 exactly
    x = np.array([[-3.0, 2.0, 5.0, -1.0]], np.float32)
    assert orc.evaluate(W.RASTRIGIN, x)[0] == 39.0


def _brute_rank(f):
    """O(N^2) rank of each member under "lower fitness first, NaN last, -0 == +0"."""
    N = len(f)
    f64 = f.astype(np.float64)
    nan = np.isnan(f64)
    s = np.empty(N, np.int64)
    e = np.empty(N, np.int64)
    for j in range(N):
        if nan[j]:
            less = (~nan).sum()
            eq = nan.sum()
        else:
            less = ((f64 < f64[j]) & ~nan).sum()
            eq = (f64 == f64[j]).sum()
        s[j], e[j] = less, less + eq - 1
    return s, e


def test_rank_brute_force(orc):
    rng = np.random.default_rng(3)
    for N in [2, 3, 16, 255, 256, 1000]:
        for ties, nans, infs in [(0, 0, 0), (N // 4, 0, 0), (3, 2, 2)]:
            f = W.random_fitness(rng, N, ties=ties, nans=nans, infs=infs)
            s, e, perm = orc.rank(f)
            bs, be = _brute_rank(f)
            assert np.array_equal(s, bs) and np.array_equal(e, be)
            assert sorted(perm) == list(range(N))
            # perm lists members by position; ties ordered by index
            for p in range(N - 1):
                a, b = perm[p], perm[p + 1]
                if s[a] == s[b]:
                    assert a < b


def test_centered_rank_examples_and_invariants(orc):
    g = json.load(open(os.path.join(GOLD, "spec_examples.json")))
    for ex in g["centered_rank"]:
        assert list(orc.centered_rank(np.array(ex["f"], np.float32))) == ex["c"]
    rng = np.random.default_rng(4)
    for N in [2, 16, 256, 4096, 65536]:
        f = W.random_fitness(rng, N, ties=N // 8)
        c = orc.centered_rank(f)
        s, e, _ = orc.rank(f)
        assert (s + e - (N - 1)).sum() == 0                       # numerators sum to 0 exactly
        assert c.min() >= -0.5 and c.max() <= 0.5
        if len(np.unique(f)) == N:
            assert c.min() == -0.5 and c.max() == 0.5
        # rank invariance under a strictly increasing transform, and row permutation
        g2 = (np.exp(np.clip(f.astype(np.float64), -80, 80) / 50.0) + 7).astype(np.float32)
        if len(np.unique(g2)) == len(np.unique(f)):
            assert np.array_equal(orc.centered_rank(g2), c)
        pi = rng.permutation(N)
        assert np.array_equal(orc.centered_rank(f[pi]), c[pi])


def test_snes_weights_closed_form(orc):
    for N, beta in [(16, 12.0), (256, 12.0), (256, 32.0), (1000, 16.0)]:
        run = orc.Run(W.SNES, N, 5, temperature=beta)
        w = run.wpos.astype(np.float64)
        assert abs(w.sum() - 1) < 1e-5
        ratio = w[:-1] / w[1:]                                    # geometric: e^{beta/N}
        assert np.allclose(ratio, np.exp(beta / N), rtol=1e-5)
    run = orc.Run(W.SNES, 8, 3, temperature=0.0)
    assert np.all(run.wpos == np.float32(1 / 8))


def test_sepcma_weights(orc):
    for N, er in [(256, 0.4), (256, 0.5), (16, 0.5), (10, 0.2)]:
        run = orc.Run(W.SEP_CMA_ES, N, 10, elite_ratio=er)
        w = run.wpos.astype(np.float64)
        mu = int(np.floor(np.float64(np.float32(er)) * N))
        assert run.mu == mu
        assert abs(w.sum() - 1) < 1e-6
        assert np.all(w[:mu] > 0) and np.all(w[mu:] == 0)
        assert np.all(np.diff(w[:mu]) < 0)
        assert np.isclose(run.mueff, 1 / (w ** 2).sum(), rtol=1e-5)
    # Hansen's default weights at elite ratio 0.5 (mu = N/2): w_p ∝ ln((N+1)/2) - ln(p+1)
    run = orc.Run(W.SEP_CMA_ES, 256, 1000, elite_ratio=0.4)
    assert abs(run.mueff - 63.98) < 0.01       # SURVEY App. A worked value


def test_member_weights_ties(orc):
    wpos = np.array([0.4, 0.3, 0.2, 0.1], np.float32)
    f = np.array([2.0, 1.0, 2.0, 3.0], np.float32)       # members 0 and 2 tie at positions 1..2
    w = orc.member_weights(wpos, f)
    assert w[1] == np.float32(0.4) and w[3] == np.float32(0.1)
    assert w[0] == w[2] == (np.float32(0.3) + np.float32(0.2)) / np.float32(2)
