"""Pins of the full-covariance CMA-ES oracle (oracle/cma_oracle.py) against things
other than itself: the SPEC's identity-factor example and 2-D sphere acceptance criterion, a
Monte-Carlo check of the sampling covariance, the D = 1 reduction to the C oracle's Sep-CMA-ES
(the two algorithms coincide there: A = √C and the separable boost (D+2)/3 = 1), symmetry and
positive definiteness of C over 1000 random tells, rank invariance, and convergence."""
import numpy as np
import pytest

import workloads as W


@pytest.fixture(scope="module")
def cma(orc):
    from oracle import cma_oracle
    return cma_oracle


def test_identity_factor_samples_m_plus_z(cma, orc):
    """SPEC cma_ask example: C = I, σ = 1 → x_j = m + z_j exactly."""
    run = cma.CMARun(12, 7, seed=3, sigma_init=1.0, init_min=-2, init_max=2)
    x = run.ask()
    Z = np.stack([orc.direction(3, j, 0, 7) for j in range(12)]).astype(np.float64)
    assert np.array_equal(x, (run.m[None, :] + Z).astype(np.float32))


def test_sampling_covariance_monte_carlo(cma):
    """Sample covariance of x over 40,000 draws within 5 % (Frobenius) of σ²C (SPEC)."""
    D = 4
    run = cma.CMARun(20_000, D, seed=5, sigma_init=0.5, init_min=0, init_max=0)
    rng = np.random.default_rng(1)
    B = rng.standard_normal((D, D))
    C = B @ B.T + 0.5 * np.eye(D)
    run.C, run.A = C, np.linalg.cholesky(C)
    xs = []
    for _ in range(2):
        xs.append(run.ask().astype(np.float64))
        run.t += 1                                  # a fresh generation of noise
    x = np.concatenate(xs)
    S = np.cov(x.T, bias=True)
    assert np.linalg.norm(S - 0.25 * C) <= 0.05 * np.linalg.norm(0.25 * C)
    assert np.abs(x.mean(0)).max() < 5 * 0.5 * np.sqrt(np.diag(C).max() / len(x))


def test_d1_reduces_to_sep_cma(cma, orc):
    """At D = 1 full and separable CMA-ES are the same algorithm (SPEC sep_cma_tell example):
    fed the same fitness, their means, σ and C agree over 60 generations."""
    N, seed = 16, 9
    p = W.run_params(W.SEP_CMA_ES, seed, init_min=-3, init_max=3, sigma_init=0.3, elite_ratio=0.5)
    sep = orc.Run(W.SEP_CMA_ES, N, 1, **p)
    full = cma.CMARun(N, 1, seed=seed, sigma_init=0.3, elite_ratio=0.5, init_min=-3, init_max=3)
    assert full.k_refresh == 1
    for g in range(60):
        xs = sep.ask()
        xf = full.ask()
        assert np.allclose(xf, xs, rtol=1e-5, atol=1e-7), g
        f = orc.evaluate(W.SPHERE, xs) + np.float32(0.1)
        sep.tell(f)
        full.tell(f)
        assert abs(full.m[0] - sep.mean[0]) <= 1e-5 * max(1.0, abs(full.m[0])), g
        assert abs(full.sigma - sep.sigma) <= 1e-5 * full.sigma, g
        assert abs(full.C[0, 0] - sep.vec[6][0]) <= 1e-5 * full.C[0, 0], g
        assert abs(full.p_sigma[0] - sep.vec[4][0]) <= 1e-5 * max(1.0, abs(full.p_sigma[0]))


def test_two_d_sphere_acceptance(cma, orc):
    """SPEC acceptance: 2-D sphere, N = 8, m0 = (3, 3), σ0 = 1 → f < 1e-8 within 200 gens."""
    run = cma.CMARun(8, 2, seed=0, sigma_init=1.0, init_min=3, init_max=3)
    assert np.array_equal(run.m, [3.0, 3.0])
    for g in range(200):
        run.tell(orc.evaluate(W.SPHERE, run.ask()))
        if run.best_f < 1e-8:
            break
    assert run.best_f < 1e-8, run.best_f


def test_rosenbrock_convergence(cma, orc):
    """Rotation-dependent valley: needs the full covariance (Sep-CMA-ES is much slower here)."""
    run = cma.CMARun(16, 5, seed=2, sigma_init=0.5, init_min=-1, init_max=1)
    for _ in range(1500):
        run.tell(orc.evaluate(W.ROSENBROCK, run.ask()))
    assert run.best_f < 1e-6, run.best_f


def test_covariance_symmetric_positive_definite(cma):
    """C stays symmetric and positive definite over 1000 tells of random fitness (SPEC)."""
    run = cma.CMARun(10, 6, seed=4, sigma_init=0.2)
    rng = np.random.default_rng(0)
    for _ in range(1000):
        run.ask()
        run.tell(rng.standard_normal(10).astype(np.float32))
    assert np.abs(run.C - run.C.T).max() <= 1e-12 * np.abs(run.C).max()
    assert np.linalg.eigvalsh(0.5 * (run.C + run.C.T)).min() > 0
    assert np.allclose(run.A @ run.A.T, 0.5 * (run.C + run.C.T), rtol=1e-6) or \
        run.t % run.k_refresh != 0


def test_rank_invariance_and_weights(cma, orc):
    a = cma.CMARun(12, 5, seed=6, sigma_init=0.3)
    b = cma.CMARun(12, 5, seed=6, sigma_init=0.3)
    assert a.wpos.sum() == pytest.approx(1.0, abs=1e-6) and np.all(np.diff(a.wpos[:a.mu]) < 0)
    for _ in range(5):
        f = orc.evaluate(W.RASTRIGIN, a.ask())
        b.ask()
        a.tell(f)
        b.tell((np.exp(f.astype(np.float64) / 50.0) + 7).astype(np.float32))   # increasing map
        assert np.array_equal(a.m, b.m) and np.array_equal(a.C, b.C) and a.sigma == b.sigma


def test_zero_step_when_parents_equal_mean(cma):
    """SPEC cma_tell example: selected parents at m (y = 0) and zero paths → m unchanged and σ
    shrinks by exp(−c_σ/d_σ)."""
    run = cma.CMARun(8, 3, seed=7, sigma_init=0.4)
    run.ask()
    run.Y[:] = 0.0
    run.Z[:] = 0.0
    m0, s0 = run.m.copy(), run.sigma
    run.tell(np.arange(8, dtype=np.float32))
    assert np.array_equal(run.m, m0)
    assert run.sigma == pytest.approx(s0 * np.exp(-run.c_sigma / run.d_sigma), rel=1e-12)
