"""B200-native hot path of evosax (arXiv:2212.04180): batched diagonal-Gaussian ES generations
(OpenAI-ES, PGPE, SNES, Sep-CMA-ES, ARS; full-covariance CMA-ES) on hand-written sm_100a kernels behind the C ABI include/es.h.
"""
from ._lib import (ADAM, ARS, CLIPUP, CMA_ES, MLP, MLP16, OPENAI_ES, PGPE, RASTRIGIN, ROSENBROCK, SEP_CMA_ES, SGD,
                   SNES, SPHERE, ESError, lib)

__all__ = ["OPENAI_ES", "PGPE", "SNES", "SEP_CMA_ES", "ARS", "CMA_ES", "ADAM", "SGD", "CLIPUP", "SPHERE", "ROSENBROCK", "RASTRIGIN", "MLP", "MLP16",
           "ESError", "lib", "Strategy", "eval_bbob"]


def __getattr__(name):
    if name in ("Strategy", "eval_bbob"):
        from . import strategy
        return getattr(strategy, name)
    raise AttributeError(name)
