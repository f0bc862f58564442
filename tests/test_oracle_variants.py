"""Pins of the §8(f) row f3 variants in the oracle: z-score shaping, SGD with momentum
(S:199-207), ClipUp and ARS, against the SPEC's worked
examples (golden) and the relations the methods define."""
import json
import os

import numpy as np
import pytest

import workloads as W

G = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def mk(orc, algo, N, D, seed=0, **kw):
    return orc.Run(algo, N, D, **W.run_params(algo, seed, **kw))


def test_zscore_golden_and_invariants(orc):
    ex = G["zscore"][0]
    assert np.allclose(orc.zscore(np.array(ex["f"], np.float32)), ex["z"], atol=ex["tol"])
    assert np.all(orc.zscore(np.full(7, 3.5, np.float32)) == 0)          # constant -> zeros
    f = np.random.default_rng(0).standard_normal(1000).astype(np.float32) * 30 + 5
    z = orc.zscore(f).astype(np.float64)
    assert abs(z.mean()) < 1e-6 and abs(z.std() - 1) < 1e-5
    ref = (f.astype(np.float64) - f.mean(dtype=np.float64)) / (f.std(dtype=np.float64) + 1e-8)
    assert np.allclose(z, ref, rtol=0, atol=1e-6)


def test_zscore_shaping_in_the_tell(orc):
    """OpenAI-ES with z-score shaping = raw-fitness OpenAI-ES fed the z-scored fitness."""
    a = mk(orc, W.OPENAI_ES, 32, 17, seed=3, shaping=2)
    b = mk(orc, W.OPENAI_ES, 32, 17, seed=3, shaping=1)
    f = orc.evaluate(W.RASTRIGIN, a.ask())
    assert np.array_equal(a.reduce(f), b.reduce(orc.zscore(f)))


def _grad(run, f):
    return (run.reduce(f)[0] / (run.popsize * run.sigma)).astype(np.float32)


def test_sgd_momentum_relation(orc):
    ex = G["sgd_momentum"][0]
    run = mk(orc, W.OPENAI_ES, 16, 5, seed=2, optimizer=W.SGD, momentum=ex["momentum"],
             lrate_decay=1.0, sigma_decay=1.0)
    v = np.zeros(5, np.float32)
    for _ in range(3):
        m0 = run.mean.copy()
        x = run.ask()
        f = orc.evaluate(W.SPHERE, x)
        g = _grad(run, f)
        run.tell(f)
        v = (np.float32(ex["momentum"]) * v + g).astype(np.float32)      # S:206 recursion
        assert np.allclose(run.mean - m0, -np.float32(0.01) * v, rtol=1e-5, atol=1e-9)
    # the SPEC example in isolation: v1 = g1, v2 = mu v1 + g2 -> updates -lr v
    mu, lr = ex["momentum"], ex["lr"]
    v1 = ex["grads"][0]
    v2 = mu * v1 + ex["grads"][1]
    assert [-lr * v1, -lr * v2] == pytest.approx(ex["updates"])


def test_clipup_relation_and_speed_limit(orc):
    ex = G["clipup"][0]
    g = np.array(ex["grad"])
    assert np.allclose(-ex["lr"] * g / np.linalg.norm(g), ex["update"])     # S:225 by hand
    run = mk(orc, W.OPENAI_ES, 32, 9, seed=4, optimizer=W.CLIPUP, momentum=0.9, max_speed=0.015,
             lrate_init=0.01, lrate_decay=1.0)
    m0 = run.mean.copy()
    f = orc.evaluate(W.SPHERE, run.ask())
    g1 = _grad(run, f)
    run.tell(f)
    step = run.mean - m0
    assert np.allclose(step, -0.01 * g1 / np.linalg.norm(g1.astype(np.float64)), rtol=1e-5)
    for _ in range(50):                                          # velocity norm <= max_speed
        run.tell(orc.evaluate(W.SPHERE, run.ask()))
        assert np.linalg.norm(run.vec[2].astype(np.float64)) <= 0.015 * (1 + 1e-6)


def test_ars_golden_and_guard(orc):
    ex = G["ars"][0]
    run = mk(orc, W.ARS, 2, 1, seed=6, elite_ratio=0.5, lrate_init=ex["alpha"], lrate_decay=1.0)
    m0 = float(run.mean[0])
    run.ask()
    z = float(orc.direction(6, 0, 0, 1)[0])
    run.tell(np.array([ex["f_plus"], ex["f_minus"]], np.float32))
    assert run.mean[0] == pytest.approx(m0 + ex["step_over_z"] * z, rel=1e-6)
    # all pairs tied: sigma_R = 0 -> no update
    run2 = mk(orc, W.ARS, 8, 3, seed=7)
    mm = run2.mean.copy()
    run2.ask()
    run2.tell(np.full(8, 1.5, np.float32))
    assert np.array_equal(run2.mean, mm)


def test_ars_linear_descent_and_convergence(orc):
    a = np.array([1.0, -2.0, 0.5])
    run = mk(orc, W.ARS, 64, 3, seed=8, sigma_init=0.1, lrate_init=0.05, elite_ratio=0.25)
    proj = []
    for _ in range(200):
        m0 = run.mean.astype(np.float64).copy()
        x = run.ask()
        run.tell((x.astype(np.float64) @ a).astype(np.float32))
        proj.append((run.mean - m0) @ a)
    assert np.mean(proj) < 0 and np.mean(np.array(proj) < 0) > 0.9      # descends a^T x
    run = mk(orc, W.ARS, 32, 10, seed=1, sigma_init=0.05, lrate_init=0.02)
    for _ in range(400):
        run.tell(orc.evaluate(W.SPHERE, run.ask()))
    assert run.best_f < 1e-2


# ------------------------------------------------------------------ weight decay
def test_weight_decay_golden_and_invariants(orc):
    ex = G["weight_decay"][0]
    out = orc.weight_decay(np.array(ex["f"], np.float32), np.array(ex["x"], np.float32), ex["coef"])
    assert np.allclose(out, ex["out"], atol=ex["tol"])
    rng = np.random.default_rng(11)
    f = rng.standard_normal(50).astype(np.float32)
    x = rng.standard_normal((50, 33)).astype(np.float32)
    assert np.array_equal(orc.weight_decay(f, x, 0.0), f)                      # coef 0: identity
    c = float(np.float32(0.03))
    ref = f.astype(np.float64) + c * np.einsum("jd,jd->j", x.astype(np.float64), x.astype(np.float64))
    got = orc.weight_decay(f, x, c)
    assert np.all(np.abs(got - ref) <= np.spacing(np.abs(got)))      # correctly rounded, ±1 ulp
    big = orc.weight_decay(np.zeros(2, np.float32), np.stack([x[0], 2 * x[0]]), 0.1)
    assert big[1] > big[0]                                                      # monotone in ||x||


@pytest.mark.parametrize("algo", [W.OPENAI_ES, W.PGPE, W.SNES, W.SEP_CMA_ES, W.ARS])
def test_weight_decay_in_the_tell(orc, algo):
    """tell(f) with weight decay == tell(f + coef ||x||^2) without it (the penalty computed here
    with numpy from the asked population), best tracking included (reading R-WD)."""
    a = mk(orc, algo, 16, 21, seed=12, weight_decay=0.05)
    b = mk(orc, algo, 16, 21, seed=12)
    for _ in range(3):
        x = a.ask()
        assert np.array_equal(x, b.ask())
        f = orc.evaluate(W.RASTRIGIN, x)
        fw = (f.astype(np.float64) + float(np.float32(0.05)) * (x.astype(np.float64) ** 2).sum(1)
              ).astype(np.float32)
        a.tell(f)
        b.tell(fw)
        assert np.allclose(a.vec, b.vec, rtol=1e-6, atol=1e-7) and a.best_f == b.best_f
        assert a.best_f == fw.min() or a.best_f < fw.min()


# ------------------------------------------------------------------ box bounds
@pytest.mark.parametrize("algo", [W.OPENAI_ES, W.PGPE, W.SNES, W.SEP_CMA_ES, W.ARS])
def test_box_clipping_at_ask(orc, algo):
    """Members are clipped into [lo, hi]; the distribution is not truncated, so with the same
    fitness the clipped and unclipped runs reach the same mean / σ (best_x differs: it is a
    clipped member)."""
    lo, hi = -0.3, 0.25
    a = mk(orc, algo, 16, 30, seed=13, clip_min=lo, clip_max=hi)
    b = mk(orc, algo, 16, 30, seed=13)
    xa, xb = a.ask(), b.ask()
    assert np.array_equal(xa, np.clip(xb, np.float32(lo), np.float32(hi)))
    assert xa.min() >= np.float32(lo) and xa.max() <= np.float32(hi) and (xb < lo).any()
    f = orc.evaluate(W.SPHERE, xb)
    a.tell(f)
    b.tell(f)
    keep = [i for i in range(a.vec.shape[0]) if i != 7]                     # all but best_x
    assert np.array_equal(a.vec[keep], b.vec[keep])
    j = int(np.argmin(f))
    assert np.array_equal(a.vec[7], xa[j])


# ------------------------------------------------------------------ PGPE elite pairs (Q13b)
def _mk_pgpe(orc, elite, N=32, D=11, **kw):
    return mk(orc, W.PGPE, N, D, seed=14, elite_ratio=elite, **kw)


@pytest.mark.parametrize("elite", [0.1, 0.25, 0.5, 0.9])
def test_pgpe_elite_direction_sums_brute_force(orc, elite):
    """G0, G1 over the k pairs of best min(f+, f-) (stable numpy argsort: ties by pair index)."""
    N, D = 32, 11
    run = _mk_pgpe(orc, elite, N, D)
    run.ask()
    rng = np.random.default_rng(15)
    f = W.random_fitness(rng, N, ties=6)
    f[np.isnan(f)] = 1.0
    P = N // 2
    k = max(1, min(P, int(np.floor(elite * P + 0.5))))
    mn = np.minimum(f[0::2], f[1::2])
    sel = np.argsort(mn, kind="stable")[:k]
    sh = orc.centered_rank(f).astype(np.float64)
    b = sh.mean()
    G0, G1 = np.zeros(D), np.zeros(D)
    for i in sel:
        z = orc.direction(run.p.seed, int(i), 0, D).astype(np.float64)
        G0 += (sh[2 * i] - sh[2 * i + 1]) * z
        G1 += ((sh[2 * i] + sh[2 * i + 1]) / 2 - b) * (z * z - 1)
    G = run.reduce(f)
    assert run.num_entries(f) == k
    assert np.allclose(G[0], G0, rtol=1e-12, atol=1e-12)
    assert np.allclose(G[1], G1, rtol=1e-12, atol=1e-12)


def test_pgpe_elite_normalisation(orc):
    """Mean and σ steps divide by the 2k members / k pairs used (SGD, momentum 0)."""
    run = _mk_pgpe(orc, 0.25, optimizer=W.SGD, momentum=0.0, lrate_decay=1.0)
    sig0, m0 = run.sigma_d.copy(), run.mean.copy()
    f = orc.evaluate(W.SPHERE, run.ask())
    G = run.reduce(f)
    k = 4
    run.tell(f)
    gm = (sig0 * G[0].astype(np.float32)) / np.float32(2 * k)
    assert np.allclose(run.mean, m0 - np.float32(0.01) * gm, rtol=1e-6, atol=1e-9)
    gs = (sig0 * G[1].astype(np.float32)) / np.float32(k)
    st = np.clip(sig0 - np.float32(0.2) * gs, np.float32(0.8) * sig0, np.float32(1.2) * sig0)
    assert np.allclose(run.sigma_d, np.maximum(st * np.float32(0.999), np.float32(0.01)), rtol=1e-6)


def test_pgpe_elite_one_is_every_pair(orc):
    a = _mk_pgpe(orc, 1.0)
    f = orc.evaluate(W.SPHERE, a.ask())
    assert a.num_entries(f) == 16
    G = a.reduce(f)
    sh = orc.centered_rank(f).astype(np.float64)
    G0 = sum((sh[2 * i] - sh[2 * i + 1]) * orc.direction(a.p.seed, i, 0, 11).astype(np.float64)
             for i in range(16))
    assert np.allclose(G[0], G0, rtol=1e-12, atol=1e-12)
