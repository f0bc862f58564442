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
