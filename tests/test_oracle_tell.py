"""Pins of the oracle's ask/tell (NUMERICS N6, N12) against closed forms and the definitions of the
cited methods: the FD-gradient expectation on linear f by brute-force sampling, the exact
antithetic identity on quadratics, weighted recombination (SNES/Sep-CMA mean updates),
Adam's textbook recursion, schedules, PGPE's clip, and convergence."""
import json
import os

import numpy as np
import pytest

import workloads as W

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def mk(orc, algo, N, D, seed=0, **kw):
    return orc.Run(algo, N, D, **W.run_params(algo, seed, **kw))


# ---------------------------------------------------------------- ask (N6)
@pytest.mark.parametrize("algo", [W.OPENAI_ES, W.PGPE])
def test_antithetic_pairs(orc, algo):
    run = mk(orc, algo, 64, 37, seed=5)
    x = run.ask().astype(np.float64)
    m = run.mean.astype(np.float64)
    # x_{2i} + x_{2i+1} = 2m up to one rounding of each member
    dev = np.abs(x[0::2] + x[1::2] - 2 * m)
    assert dev.max() <= 2 * np.spacing(np.abs(m).astype(np.float32)).max()
    # z is the same for the pair: (x+ - m) = -(x- - m) approximately, and differs between pairs
    assert not np.allclose(x[0], x[2])


def test_sigma_zero_gives_mean(orc):
    for algo in (W.OPENAI_ES, W.PGPE, W.SNES, W.SEP_CMA_ES):
        run = mk(orc, algo, 8, 13, sigma_init=0.0)
        assert np.array_equal(run.ask(), np.broadcast_to(run.mean, (8, 13)))


def test_init_mean_uniform(orc):
    run = mk(orc, W.SNES, 4, 200000, seed=3, init_min=-5.12, init_max=5.12)
    from scipy import stats
    m = run.mean.astype(np.float64)
    assert m.min() >= -5.12 and m.max() < 5.12
    assert stats.kstest((m + 5.12) / 10.24, "uniform").pvalue > 1e-4


def test_ask_distribution_matches_sigma(orc):
    run = mk(orc, W.SEP_CMA_ES, 4096, 8, seed=2, sigma_init=0.3)
    z = (run.ask().astype(np.float64) - run.mean) / 0.3
    assert abs(z.std() - 1) < 0.02 and abs(z.mean()) < 0.02


# ---------------------------------------------------------------- FD gradient
def test_openai_fd_gradient_linear_expectation(orc):
    """E[g] = a for f(x) = a^T x (raw-fitness mode), brute force over 10^6 antithetic pairs."""
    D, P = 3, 1_000_000
    a = np.array([0.7, -1.3, 0.4])
    run = mk(orc, W.OPENAI_ES, 2 * P, D, seed=11, shaping=1, sigma_init=0.05)
    x = run.ask().astype(np.float64)
    f = (x @ a).astype(np.float32)
    g = run.reduce(f)[0] / (2 * P * 0.05)
    se = np.sqrt((a @ a + a ** 2) / P)
    assert np.all(np.abs(g - a) < 5 * se), (g, a, se)


def test_openai_quadratic_exact_identity(orc):
    """Antithetic FD on f(x)=x^2 in D=1: g = 2m * mean_i(z_i^2) exactly (S:290 generalised)."""
    N = 64
    run = mk(orc, W.OPENAI_ES, N, 1, seed=4, shaping=1, sigma_init=0.1)
    x = run.ask().astype(np.float64)[:, 0]
    f = (x * x).astype(np.float32)
    g = run.reduce(f)[0][0] / (N * 0.1)
    z = np.array([orc.direction(4, i, 0, 1)[0] for i in range(N // 2)], np.float64)
    m = float(run.mean[0])
    assert abs(g - 2 * m * np.mean(z * z)) < 1e-5 * abs(g) + 1e-7


def test_pgpe_linear_expectation(orc):
    """PGPE raw mode, f = a^T x: E[g^m_d] = sigma_d^2 a_d (eps = sigma z)."""
    D, P = 2, 1_000_000
    a = np.array([1.5, -0.5])
    run = mk(orc, W.PGPE, 2 * P, D, seed=12, shaping=1, sigma_init=0.2)
    x = run.ask().astype(np.float64)
    f = (x @ a).astype(np.float32)
    G = run.reduce(f)
    gm = 0.2 * G[0] / (2 * P)
    assert np.all(np.abs(gm - 0.04 * a) < 5 * 0.04 * np.sqrt((a @ a + a ** 2) / P))


# ---------------------------------------------------------------- updates
def test_adam_first_step_is_lr_sign(orc):
    for algo in (W.OPENAI_ES, W.PGPE):
        run = mk(orc, algo, 32, 50, seed=1, init_min=-2, init_max=2)
        m0 = run.mean.copy()
        x = run.ask()
        f = W_eval(orc, x)
        G = run.reduce(f)[0]
        run.tell(f)
        dm = run.mean.astype(np.float64) - m0
        big = np.abs(G) > 1e-3
        # |step| = lr * |g|/(|g|+eps), then one rounding of the fp32 mean
        g = G[big] / (32 * 0.05) if algo == W.OPENAI_ES else 0.025 * G[big] / 32
        tol = 2 * np.spacing(np.abs(m0[big])) + 0.01 * 1e-8 / np.abs(g) + 1e-9
        assert np.all(np.abs(np.abs(dm[big]) - 0.01) <= tol)
        assert np.all(np.sign(dm[big]) == -np.sign(G[big]))


def W_eval(orc, x):
    return orc.evaluate(W.SPHERE, x)


def test_adam_textbook_recursion(orc):
    """5 generations of OpenAI-ES vs. a textbook Adam (Kingma & Ba) in double driven by the same
    gradients; agreement to fp32 rounding."""
    N, D = 16, 10
    run = mk(orc, W.OPENAI_ES, N, D, seed=0, lrate_decay=0.999, sigma_decay=0.999)
    mean = run.mean.astype(np.float64)
    m = np.zeros(D)
    v = np.zeros(D)
    lr, sig = 0.01, 0.05
    for t in range(1, 6):
        x = run.ask()
        f = W_eval(orc, x)
        g = run.reduce(f)[0] / (N * sig)
        run.tell(f)
        m = 0.9 * m + 0.1 * g
        v = 0.999 * v + 0.001 * g * g
        mean = mean - lr * (m / (1 - 0.9 ** t)) / (np.sqrt(v / (1 - 0.999 ** t)) + 1e-8)
        lr, sig = max(lr * 0.999, 0.0), max(sig * 0.999, 0.0)
        assert np.allclose(run.mean, mean, rtol=0, atol=2e-6 * t)
        assert abs(run.lr - lr) < 1e-8 and abs(run.sigma - sig) < 1e-8


def test_schedule_golden_and_floor(orc):
    ex = json.load(open(os.path.join(GOLD, "spec_examples.json")))["exp_decay"][0]
    run = mk(orc, W.OPENAI_ES, 4, 3, lrate_init=ex["value"], lrate_decay=ex["decay"],
             lrate_limit=ex["floor"], sigma_decay=0.5, sigma_limit=0.01)
    x = run.ask()
    run.tell(W_eval(orc, x))
    assert abs(run.lr - ex["out"]) < 1e-9
    for _ in range(20):
        run.tell(W_eval(orc, run.ask()))
    assert run.sigma == np.float32(0.01)           # sigma floor reached and held


def test_pgpe_sigma_clip_and_pair_symmetry(orc):
    run = mk(orc, W.PGPE, 64, 40, seed=3)
    for _ in range(5):
        s0 = run.sigma_d.copy()
        x = run.ask()
        run.tell(W.random_fitness(np.random.default_rng(run.t), 64))
        ratio = run.sigma_d / s0
        assert np.all(ratio >= 0.8 * 0.999 - 1e-6) and np.all(ratio <= 1.2 * 0.999 + 1e-6)
    # equal fitness inside every pair: a_i = 0 -> mean unchanged exactly
    m0 = mk(orc, W.PGPE, 64, 40, seed=4)
    mean0 = m0.mean.copy()
    f = np.repeat(np.random.default_rng(0).standard_normal(32).astype(np.float32), 2)
    m0.ask()
    m0.tell(f)
    assert np.array_equal(m0.mean, mean0)


def _recombination_weights(orc, run, f):
    """omega_j computed independently: numpy double closed-form position weights + brute ranks."""
    N = len(f)
    order = np.argsort(f, kind="stable")
    p = np.empty(N, int)
    p[order] = np.arange(N)
    if run.algo == W.SNES:
        beta = run.p.temperature
        u = beta * ((N - 1 - np.arange(N)) / N - 0.5)
        w = np.exp(u - u.max())
        w /= w.sum()
    else:
        mu = run.mu
        w = np.where(np.arange(N) < mu, np.log((N + 1) / 2) - np.log(np.arange(N) + 1.0), 0.0)
        w /= w.sum()
    return w[p]


@pytest.mark.parametrize("algo", [W.SNES, W.SEP_CMA_ES])
def test_mean_is_weighted_recombination(orc, algo):
    """With sum(w)=1 and eta_m = c_m = 1: m' = sum_j w_j x_j (SNES P:369; Sep-CMA)."""
    N, D = 32, 25
    run = mk(orc, algo, N, D, seed=8, sigma_init=0.3)
    x = run.ask()
    f = orc.evaluate(W.RASTRIGIN, x)
    assert len(np.unique(f)) == N
    omega = _recombination_weights(orc, run, f)
    expect = omega @ x.astype(np.float64)
    run.tell(f)
    assert np.allclose(run.mean, expect, rtol=0, atol=1e-5)


def test_snes_sigma_natural_gradient(orc):
    """SNES sigma' = sigma * exp(eta_sigma/2 * sum_j w_j (s_j^2 - 1)), s_j = (x_j - m)/sigma."""
    N, D = 32, 12
    run = mk(orc, W.SNES, N, D, seed=9, sigma_init=0.3)
    m, s = run.mean.astype(np.float64), run.sigma_d.astype(np.float64)
    x = run.ask().astype(np.float64)
    f = orc.evaluate(W.SPHERE, x.astype(np.float32))
    omega = _recombination_weights(orc, run, f)
    sk = (x - m) / s
    eta = (3 + np.log(D)) / (5 * np.sqrt(D))
    expect = s * np.exp(eta / 2 * (omega @ (sk * sk - 1)))
    run.tell(f)
    assert np.allclose(run.sigma_d, expect, rtol=2e-5)


def test_sepcma_positivity_and_random_selection(orc):
    """Under random selection (fitness independent of x) the CSA path is stationary N(0, I), so
    E||p_sigma||^2 = D (Hansen's tutorial; checks c_sigma, the sqrt(c(2-c) mu_eff) factor and the
    recombination of z), while C_d > 0 and sigma > 0 always."""
    D = 10
    run = mk(orc, W.SEP_CMA_ES, 16, D, seed=21, elite_ratio=0.5)
    norms, logs = [], []
    for t in range(2000):
        run.ask()
        run.tell(orc.synth_fitness(21, t, 16))       # fitness independent of x
        norms.append(float((run.vec[4].astype(np.float64) ** 2).sum()))
        logs.append(np.log(run.sigma))
        assert np.all(run.vec[6] > 0) and run.sigma > 0
    assert abs(np.mean(norms[100:]) / D - 1) < 0.15
    assert abs((logs[-1] - logs[100]) / 1900) < 0.01


@pytest.mark.parametrize("algo,thresh,gens", [(W.OPENAI_ES, 1e-2, 600), (W.SNES, 1e-3, 300),
                                              (W.SEP_CMA_ES, 1e-3, 300), (W.PGPE, 1e-1, 600)])
def test_convergence_sphere10(orc, algo, thresh, gens):
    """S:790 behavioural acceptance: 10-D sphere from U[-1,1]."""
    kw = dict(sigma_init=0.3) if algo in (W.SNES, W.SEP_CMA_ES) else {}
    run = mk(orc, algo, 16 if algo != W.SNES else 32, 10, seed=1, **kw)
    for _ in range(gens):
        x = run.ask()
        run.tell(orc.evaluate(W.SPHERE, x))
    assert run.best_f < thresh, run.best_f


def test_best_tracking(orc):
    run = mk(orc, W.SNES, 16, 6, seed=2, sigma_init=0.5)
    running = np.inf
    for _ in range(30):
        x = run.ask()
        f = orc.evaluate(W.RASTRIGIN, x)
        running = min(running, f.min())
        run.tell(f)
        assert run.best_f == np.float32(running)
        # best_x is regenerated, bit-identical to the asked member: its fitness reproduces best_f
        assert orc.evaluate(W.RASTRIGIN, run.vec[7])[0] == run.best_f


def test_determinism(orc):
    a = mk(orc, W.PGPE, 16, 9, seed=77)
    b = mk(orc, W.PGPE, 16, 9, seed=77)
    for _ in range(5):
        fa = orc.evaluate(W.ROSENBROCK, a.ask())
        fb = orc.evaluate(W.ROSENBROCK, b.ask())
        a.tell(fa)
        b.tell(fb)
    assert np.array_equal(a.vec, b.vec)


# ---------------------------------------------------------------- round-2 pins
def test_pgpe_sigma_gradient_expectation(orc):
    """PGPE sigma gradient (reading Q12: eps = sigma z, baseline = mean shaped fitness,
    divided by P) on f = sum_d a_d x_d^2 in raw mode: E[g^sigma_d] = sigma_d^2 dE[f]/dsigma_d =
    2 a_d sigma_d^3 (E f = sum a (m^2 + sigma^2)), brute force over 10^6 antithetic pairs, within 5
    analytic standard errors (Var[h (z_d^2-1)] = 56 a_d^2 sigma_d^4 + 4 sum_{e!=d} a_e^2 sigma_e^4,
    from the chi^2_1 central moments). Checked both on the raw direction sum and through the sigma
    step of the tell (sigma' = sigma - 0.2 g^sigma, no clip hit, no decay): sigma shrinks where
    a > 0 and grows where a < 0. A sign error, /N instead of /P, or a missing sigma factor fails."""
    D, P, s0 = 3, 1_000_000, 0.5
    a = np.array([1.0, 1.5, -0.5])
    run = mk(orc, W.PGPE, 2 * P, D, seed=31, shaping=1, sigma_init=s0, sigma_decay=1.0,
             sigma_limit=0.0, init_min=-0.1, init_max=0.1)
    x = run.ask().astype(np.float64)
    f = ((x * x) @ a).astype(np.float32)
    expect = 2 * a * s0 ** 3
    var = 56 * a ** 2 * s0 ** 4 + 4 * ((a ** 2 * s0 ** 4).sum() - a ** 2 * s0 ** 4)
    se = s0 * np.sqrt(var / P)
    gs = s0 * run.reduce(f)[1] / P
    assert np.all(np.abs(gs - expect) < 5 * se), (gs, expect, se)
    run.tell(f)
    g_tell = (s0 - run.sigma_d.astype(np.float64)) / 0.2
    assert np.all(np.abs(g_tell - expect) < 5 * se + 1e-6), (g_tell, expect)
    assert run.sigma_d[0] < s0 and run.sigma_d[1] < s0 and run.sigma_d[2] > s0


def test_sepcma_constants_vs_appendix_a(orc):
    """mu, mu_eff, c_sigma, d_sigma, c_c, c_1 (D+2)/3, c_mu (D+2)/3, chi_D against SURVEY App. A's
    table (tests/golden/sepcma_constants.json) at both elite ratios of the C2 variant and at D=10."""
    g = json.load(open(os.path.join(GOLD, "sepcma_constants.json")))
    for row in g["rows"]:
        run = mk(orc, W.SEP_CMA_ES, row["N"], row["D"], elite_ratio=row["elite"])
        assert run.mu == row["mu"]
        for k in ("mueff", "c_sigma", "d_sigma", "c_c", "c_1", "c_mu", "chi_d"):
            got = getattr(run, k)
            assert abs(got - row[k]) <= 5e-4 * abs(row[k]), (row, k, got)
    for row in g["snes_eta_sigma"]:
        run = mk(orc, W.SNES, 4, row["D"]) if row["D"] <= 100000 else None
        if run is not None:
            assert abs(run.eta_sigma - row["eta"]) <= 5e-4 * row["eta"], (row, run.eta_sigma)


def test_sepcma_zero_path_s438(orc):
    """S:438 zero-path limit on the C oracle's Sep-CMA-ES: every selected parent at m (Z^w = 0,
    Q = 0) from the initial zero paths -> m unchanged, p_sigma = p_c = 0, sigma shrinks by exactly
    exp(-c_sigma/d_sigma) (||p_sigma|| = 0 < threshold so h_sigma = 1), and
    C' = (1 - c_1 - c_mu) C (no rank-one or rank-mu contribution)."""
    for D, N, er in ((10, 16, 0.5), (1000, 256, 0.4)):
        run = mk(orc, W.SEP_CMA_ES, N, D, seed=3, elite_ratio=er, sigma_init=0.05)
        m0 = run.mean.copy()
        f = np.arange(N, dtype=np.float32)
        run.tell_apply(f, np.zeros((2, D)))
        assert np.array_equal(run.mean, m0)
        assert np.all(run.vec[4] == 0) and np.all(run.vec[5] == 0)
        expect = 0.05 * np.exp(-run.c_sigma / run.d_sigma)
        assert abs(run.sigma - expect) <= 2 * np.spacing(np.float32(expect)), (run.sigma, expect)
        cexp = 1.0 - run.c_1 - run.c_mu
        assert np.allclose(run.vec[6], cexp, rtol=1e-7, atol=0), (run.vec[6][:3], cexp)
        assert run.t == 1
