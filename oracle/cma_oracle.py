"""Full-covariance CMA-ES oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference legs may import this
module; the product never does. Plain numpy in binary64, one run at a time, every step in the
order of Hansen's CMA-ES tutorial as the paper cites it ("weighted recombination-based mean
updates and iterative covariance matrix estimation ... evolution paths", Table 1 row P:177,
Listing 1), with the reparametrisation the paper names for sampling, "the Cholesky
decomposition of a covariance matrix". Readings (R-CMA):

* x_j = m + σ·A·z_j, A = chol(C) (lower, positive diagonal) refreshed after every k-th tell,
  k = max(1, ⌊1 / (10·D·(c_1 + c_μ))⌋) (SPEC's staleness rule); z_j the member's N2 normals
  (counter (⌊d/4⌋, j, t, ASK), the same stream SNES / Sep-CMA-ES use).
* weights w′_p = ln((N+1)/2) − ln(p+1) for p < μ = ⌊elite_ratio·N⌋, normalised (as Sep-CMA-ES),
  stored as fp32 position weights and averaged over tie groups (N11).
* p_σ is driven by z̄ = Σ w_j z_j (= A⁻¹ȳ with the cached factor — the Cholesky analogue of
  C^{-1/2}ȳ with a cached eigendecomposition); everything else is the tutorial's update with
  c_m = 1 and the (1 − h_σ) correction, no σ decay. Constants: tutorial defaults (no separable
  (D+2)/3 boost).
* Numerical repair (SPEC): if the factorisation fails, add 1e-14·tr(C)/D to the diagonal once;
  if it still fails, keep the previous factor.
* State in binary64; x rounded to fp32 once (then clipped into the box, as N6 for the others).

Parity status: pinned in tests/test_oracle_cma.py (SPEC C = I example, Monte-Carlo covariance,
D = 1 reduction to the C oracle's Sep-CMA-ES, SPEC 2-D sphere acceptance, symmetry / positive
definiteness over 1000 random tells, Rosenbrock convergence, rank invariance).
"""
from __future__ import annotations

import math

import numpy as np

from . import oracle as O

SEP_CMA_ES = 3


class CMARun:
    """One full-covariance CMA-ES run (binary64 state)."""

    def __init__(self, N, D, seed, sigma_init=0.05, elite_ratio=0.5, init_min=-1.0,
                 init_max=1.0, clip_min=-np.inf, clip_max=np.inf, **_ignored):
        self.N, self.D, self.seed = int(N), int(D), int(seed)
        self.clip = (np.float32(clip_min), np.float32(clip_max))
        # mean_0 from the INIT stream exactly as every other algorithm (N6, C oracle)
        init = O.Run(SEP_CMA_ES, max(N, 4), D, seed=seed, init_min=init_min, init_max=init_max,
                     sigma_init=sigma_init, elite_ratio=0.5)
        self.m = init.mean.astype(np.float64).copy()
        self.best_x = init.mean.astype(np.float32).copy()
        self.best_f = np.float32(np.inf)
        self.sigma = float(np.float32(sigma_init))
        # weights and constants (Hansen's tutorial; μ from the elite ratio as Sep-CMA-ES)
        mu = int(math.floor(float(np.float32(elite_ratio)) * N))
        if mu < 1:
            raise ValueError("floor(elite_ratio*N) < 1")
        w = np.zeros(N)
        w[:mu] = math.log((N + 1) / 2.0) - np.log(np.arange(1, mu + 1, dtype=np.float64))
        w /= w.sum()
        self.mu = mu
        self.wpos = w.astype(np.float32)
        self.mueff = 1.0 / float((w ** 2).sum())
        Dd, me = float(D), self.mueff
        self.c_sigma = (me + 2.0) / (Dd + me + 5.0)
        self.d_sigma = 1.0 + 2.0 * max(0.0, math.sqrt((me - 1.0) / (Dd + 1.0)) - 1.0) + self.c_sigma
        self.c_c = (4.0 + me / Dd) / (Dd + 4.0 + 2.0 * me / Dd)
        self.c_1 = 2.0 / ((Dd + 1.3) ** 2 + me)
        self.c_mu = min(1.0 - self.c_1, 2.0 * (me - 2.0 + 1.0 / me) / ((Dd + 2.0) ** 2 + me))
        self.chi_d = math.sqrt(Dd) * (1.0 - 1.0 / (4.0 * Dd) + 1.0 / (21.0 * Dd * Dd))
        self.k_refresh = max(1, int(math.floor(1.0 / (10.0 * Dd * (self.c_1 + self.c_mu)))))
        self.C = np.eye(D)
        self.A = np.eye(D)
        self.p_sigma = np.zeros(D)
        self.p_c = np.zeros(D)
        self.t = 0
        self.Z = self.Y = self.X = None

    # ask: x_j = m + σ A z_j
    def ask(self):
        Z = np.stack([O.direction(self.seed, j, self.t, self.D) for j in range(self.N)])
        self.Z = Z.astype(np.float64)
        self.Y = self.Z @ self.A.T
        X = (self.m[None, :] + self.sigma * self.Y).astype(np.float32)
        self.X = np.clip(X, self.clip[0], self.clip[1])
        return self.X.copy()

    # tell: tutorial update in order
    def tell(self, f):
        f = np.ascontiguousarray(f, dtype=np.float32)
        s, e, perm = O.rank(f)
        jb = int(perm[0])
        if f[jb] < self.best_f:                        # strict, NaN never improves
            self.best_f = f[jb]
            self.best_x = self.X[jb].copy()
        w = O.member_weights(self.wpos, f).astype(np.float64)     # N11, ties averaged
        ybar = w @ self.Y
        zbar = w @ self.Z
        self.m = self.m + self.sigma * ybar
        cs, cc, me = self.c_sigma, self.c_c, self.mueff
        self.p_sigma = (1.0 - cs) * self.p_sigma + math.sqrt(cs * (2.0 - cs) * me) * zbar
        norm = float(np.linalg.norm(self.p_sigma))
        hs = norm / math.sqrt(1.0 - (1.0 - cs) ** (2.0 * (self.t + 1))) < \
            (1.4 + 2.0 / (self.D + 1.0)) * self.chi_d
        self.p_c = (1.0 - cc) * self.p_c + (math.sqrt(cc * (2.0 - cc) * me) if hs else 0.0) * ybar
        a = 1.0 - self.c_1 - self.c_mu + (0.0 if hs else 1.0) * self.c_1 * cc * (2.0 - cc)
        rank_mu = (self.Y * w[:, None]).T @ self.Y
        self.C = a * self.C + self.c_1 * np.outer(self.p_c, self.p_c) + self.c_mu * rank_mu
        self.sigma = self.sigma * math.exp((cs / self.d_sigma) * (norm / self.chi_d - 1.0))
        self.t += 1
        if self.t % self.k_refresh == 0:
            self.A = self.factor(self.C, self.A)

    @staticmethod
    def factor(C, prev):
        """Cholesky factor of the symmetrised C; one diagonal repair, else keep prev (SPEC)."""
        Cs = 0.5 * (C + C.T)
        try:
            return np.linalg.cholesky(Cs)
        except np.linalg.LinAlgError:
            pass
        try:
            return np.linalg.cholesky(Cs + 1e-14 * np.trace(Cs) / Cs.shape[0] * np.eye(Cs.shape[0]))
        except np.linalg.LinAlgError:
            return prev
