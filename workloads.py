"""Seeded synthetic workloads shared by the tests and bench.py.

Holds NONE of the method's arithmetic: only hyperparameter tables (App. B), the
BASELINE.json config shapes, and numpy-seeded generators of arbitrary test inputs (fitness
vectors, populations). Both the oracle side and the CUDA side receive these as plain inputs.
"""
from __future__ import annotations

import numpy as np

OPENAI_ES, PGPE, SNES, SEP_CMA_ES, ARS, CMA_ES = 0, 1, 2, 3, 4, 5
ALGO_NAMES = {OPENAI_ES: "openai_es", PGPE: "pgpe", SNES: "snes", SEP_CMA_ES: "sep_cma_es",
              ARS: "ars", CMA_ES: "cma_es"}
ADAM, SGD, CLIPUP = 0, 1, 2
SPHERE, ROSENBROCK, RASTRIGIN, MLP, MLP16 = 0, 1, 2, 3, 4
FN_NAMES = {SPHERE: "sphere", ROSENBROCK: "rosenbrock", RASTRIGIN: "rastrigin", MLP: "mlp", MLP16: "mlp16"}

# PAPER.md Appendix B, "Ant" column.
ANT = {
    OPENAI_ES: dict(sigma_init=0.05, sigma_decay=0.999, sigma_limit=0.01,
                    lrate_init=0.01, lrate_decay=0.999, lrate_limit=0.001),
    PGPE: dict(sigma_init=0.025, sigma_decay=0.999, sigma_limit=0.01,
               lrate_init=0.01, lrate_decay=0.999, lrate_limit=0.001,
               sigma_lrate=0.2, sigma_max_change=0.2, elite_ratio=1.0),   # Q13: every pair
    SNES: dict(sigma_init=0.05, temperature=12.0),
    SEP_CMA_ES: dict(sigma_init=0.05, elite_ratio=0.4),
    # ARS has no App. B column (Table 1 row only): OpenAI-ES-like schedules, top-50 % pairs
    ARS: dict(sigma_init=0.05, sigma_decay=0.999, sigma_limit=0.01, lrate_init=0.01,
              lrate_decay=0.999, lrate_limit=0.001, elite_ratio=0.5),
    # full CMA-ES (f4) has no App. B column: Hansen's defaults (μ = N/2), σ0 a quarter of the
    # [-2, 2] init box
    CMA_ES: dict(sigma_init=0.5, elite_ratio=0.5),
}
# The four App. B columns (Ant, Fetch, HalfCheetah, Humanoid) for the hyperparameter-vmap variant.
SEP_CMA_COLUMNS = [(0.05, 0.4), (0.125, 0.2), (0.05, 0.5), (0.1, 0.2)]
SNES_COLUMNS = [(0.05, 12.0), (0.075, 12.0), (0.05, 16.0), (0.075, 32.0)]

BASE = dict(init_min=-1.0, init_max=1.0, sigma_init=0.05, sigma_decay=1.0, sigma_limit=0.0,
            lrate_init=0.01, lrate_decay=1.0, lrate_limit=0.0, beta1=0.9, beta2=0.999, eps=1e-8,
            sigma_lrate=0.2, sigma_max_change=0.2, temperature=12.0, elite_ratio=0.5, shaping=0,
            optimizer=0, momentum=0.9, max_speed=0.02, weight_decay=0.0, clip_min=-np.inf,
            clip_max=np.inf)


def run_params(algo, seed, **over):
    """Hyperparameters of one run: BASE <- App. B Ant column <- overrides."""
    p = dict(BASE)
    p.update(ANT[algo])
    p.update(over)
    p["seed"] = int(seed)
    return p


# BASELINE.json configs (SURVEY.md §8(d) concrete definitions).
CONFIGS = {
    "c1": dict(name="openai_es-sphere-D10-N16-R1", algo=OPENAI_ES, fn=SPHERE, D=10, N=16, R=1,
               gens=100, init=(-1.0, 1.0)),
    "c2_sepcma": dict(name="sep_cma_es-rastrigin-D1000-N256-R512", algo=SEP_CMA_ES, fn=RASTRIGIN,
                      D=1000, N=256, R=512, gens=100, init=(-5.12, 5.12)),
    "c2_snes": dict(name="snes-rastrigin-D1000-N256-R512", algo=SNES, fn=RASTRIGIN, D=1000, N=256,
                    R=512, gens=100, init=(-5.12, 5.12)),
    "c3": dict(name="pgpe-rosenbrock-D100000-N256-R1", algo=PGPE, fn=ROSENBROCK, D=100_000, N=256,
               R=1, gens=1000, init=(-2.0, 2.0)),
    "c4": dict(name="openai_es-mlp-D985216-N4096-R1", algo=OPENAI_ES, fn=MLP, D=985_216, N=4096,
               R=1, gens=100, init=(-0.04, 0.04)),
    # SURVEY 8(f) f4 (no BASELINE config): full-covariance CMA-ES at "moderate D", the paper's
    # population 256, 8 runs batched
    "c6": dict(name="cma_es-rosenbrock-D1024-N256-R8", algo=CMA_ES, fn=ROSENBROCK, D=1024, N=256,
               R=8, gens=100, init=(-2.0, 2.0)),
}


def config_params(cfg, r, seed_offset=0, hyper_vmap=False):
    """Run r's params for a config; hyper_vmap=True cycles the four App. B columns."""
    algo = cfg["algo"]
    lo, hi = cfg["init"]
    over = dict(init_min=lo, init_max=hi)
    if hyper_vmap and algo == SEP_CMA_ES:
        s, e = SEP_CMA_COLUMNS[r % 4]
        over.update(sigma_init=s, elite_ratio=e)
    if hyper_vmap and algo == SNES:
        s, b = SNES_COLUMNS[r % 4]
        over.update(sigma_init=s, temperature=b)
    return run_params(algo, seed_offset + r, **over)


def random_fitness(rng: np.random.Generator, N, ties=0, nans=0, infs=0):
    """Arbitrary fitness vector with a controllable number of exact ties / NaN / inf."""
    f = rng.standard_normal(N).astype(np.float32) * np.float32(rng.uniform(0.1, 100.0))
    for _ in range(ties):
        a, b = rng.integers(0, N, size=2)
        f[b] = f[a]
    for k in rng.choice(N, size=min(nans, N), replace=False):
        f[k] = np.nan
    for k in rng.choice(N, size=min(infs, N), replace=False):
        f[k] = np.inf if rng.random() < 0.5 else -np.inf
    if N > 3 and rng.random() < 0.5:
        f[rng.integers(0, N)] = -0.0
        f[rng.integers(0, N)] = 0.0
    return f


def random_population(rng: np.random.Generator, n, D, scale=3.0):
    return (rng.standard_normal((n, D)) * scale).astype(np.float32)
