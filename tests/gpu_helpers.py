"""Side-by-side drivers for the GPU parity tests: the CUDA path through the C ABI (via the thin
Python binding) and the CPU oracle, fed the same seeded inputs (workloads.py)."""
from __future__ import annotations

import numpy as np
import torch

import workloads as W
from oracle import oracle as O

VEC_FIELDS = ["mean", "sigma_d", "adam_m", "adam_v", "p_sigma", "p_c", "C", "best_x"]
KEPT = {
    W.OPENAI_ES: ["mean", "adam_m", "adam_v", "best_x"],
    W.PGPE: ["mean", "sigma_d", "adam_m", "adam_v", "best_x"],
    W.SNES: ["mean", "sigma_d", "best_x"],
    W.SEP_CMA_ES: ["mean", "p_sigma", "p_c", "C", "best_x"],
    W.ARS: ["mean", "best_x"],
}
HAS_SIGMA = (W.OPENAI_ES, W.SEP_CMA_ES, W.ARS)
HAS_LRATE = (W.OPENAI_ES, W.PGPE, W.ARS)


def q24(a, b):
    """max_d |a_d - b_d| / max(|b_d|, 2^-10 ||b||_inf)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    if b.size == 0:
        return 0.0
    floor = max(np.abs(b).max() * 2.0 ** -10, 1e-30)
    return float((np.abs(a - b) / np.maximum(np.abs(b), floor)).max())


def bits(a):
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def es_state(es, algo, r, dims=None):
    """Run r's state of any GPU context (sharded ones included) in the oracle's field names."""
    st = {f: es.get(f)[r].cpu().numpy() for f in KEPT[algo]}
    st["best_f"] = float(es.get("best_f")[r])
    if algo in HAS_SIGMA:
        st["sigma"] = float(es.get("sigma")[r])
    if algo in HAS_LRATE:
        st["lrate"] = float(es.get("lrate")[r])
    st["gen"] = int(es.get("gen")[r])
    if dims is not None:
        for f in KEPT[algo]:
            st[f] = st[f][dims]
    return st


def oracle_state(o, algo):
    st = {f: o.vec[VEC_FIELDS.index(f)].copy() for f in KEPT[algo]}
    st["best_f"] = float(o.best_f)
    if algo in HAS_SIGMA:
        st["sigma"] = float(o.sigma)
    if algo in HAS_LRATE:
        st["lrate"] = float(o.lr)
    st["gen"] = int(o.t)
    return st


def compare_to_oracle(es, algo, r, o, tol, dims=None, d0=0):
    """Q24 distance of run r of GPU context `es` (optionally a D-shard whose state starts at global
    dim d0) to oracle run `o`, per field; asserts <= tol and returns the worst."""
    g = es_state(es, algo, r)
    ref = oracle_state(o, algo)
    worst = 0.0
    for k in g:
        a, b = np.atleast_1d(g[k]), np.atleast_1d(ref[k])
        if k in KEPT[algo] and a.size != b.size:       # a D-shard holds the dims [d0, d0 + n)
            b = b[d0:d0 + a.size]
        e = q24(a, b)
        assert e <= tol, (k, r, e)
        worst = max(worst, e)
    return worst


class Pair:
    """R runs of one algorithm on the GPU and R oracle runs with identical parameters."""

    def __init__(self, algo, N, D, params, dims=None):
        from paper_2212_04180_b200 import strategy as S
        self.algo, self.N, self.D, self.R = algo, N, D, len(params)
        self.params = params
        self.gpu = S.Strategy(algo, N, D, params)
        self.orc = [O.Run(algo, N, D, dims=dims, **p) for p in params]
        self.dims = dims

    def gpu_state(self, r):
        st = {f: self.gpu.get(f)[r].cpu().numpy() for f in KEPT[self.algo]}
        st["best_f"] = float(self.gpu.get("best_f")[r])
        if self.algo in HAS_SIGMA:
            st["sigma"] = float(self.gpu.get("sigma")[r])
        if self.algo in HAS_LRATE:
            st["lrate"] = float(self.gpu.get("lrate")[r])
        st["gen"] = int(self.gpu.get("gen")[r])
        if self.dims is not None:
            for f in KEPT[self.algo]:
                st[f] = st[f][self.dims]
        return st

    def orc_state(self, r):
        o = self.orc[r]
        st = {f: o.vec[VEC_FIELDS.index(f)].copy() for f in KEPT[self.algo]}
        st["best_f"] = float(o.best_f)
        if self.algo in HAS_SIGMA:
            st["sigma"] = float(o.sigma)
        if self.algo in HAS_LRATE:
            st["lrate"] = float(o.lr)
        st["gen"] = int(o.t)
        return st

    def compare(self, r, tol):
        g, o = self.gpu_state(r), self.orc_state(r)
        worst = 0.0
        exact = True
        for k in g:
            e = q24(np.atleast_1d(g[k]), np.atleast_1d(o[k]))
            if not np.array_equal(bits(np.atleast_1d(g[k])), bits(np.atleast_1d(o[k]))):
                exact = False
            assert e <= tol, (k, r, e)
            worst = max(worst, e)
        return worst, exact

    def close(self):
        self.gpu.close()


def cuda_ok():
    return torch.cuda.is_available()
