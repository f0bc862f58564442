"""GPU parity of the full-covariance CMA-ES against oracle/cma_oracle.py.

The sampling y = A·z and the rank-μ update are dense contractions accumulated in fp32 (in a tile
order), against the oracle's binary64: x, C, A and the paths agree to a derived tolerance, not bit
for bit. Derivation: every contraction is a sum of ≤ D products of O(1) fp32 values, so its
rounding error is ≤ D·2⁻²⁴ relative to Σ|terms| (≈ 6e-5 at D = 1024, typically √D·2⁻²⁴ ≈ 2e-6);
the factorisation adds κ(C)·that. The bar is Q24 ≤ 1e-5 after one generation (teacher-forced on
the GPU's fitness) and, after 100 teacher-forced generations, ≤ 1e-3, both NORMWISE (‖Δ‖∞/‖ref‖∞).
The tensor-core sampling (kind::tf32, 3-pass split) represents each operand to ≈ 2⁻²³ (one fp32
ulp) and accumulates in fp32, so y carries absolute errors of ≈ 1 ulp of |z|·|A|: bounded normwise
— an elementwise metric with a small floor (Q24) would turn a 1e-7 absolute error on an entry near
zero into a large relative one. After 100 generations:
the GPU keeps m, C and A in fp32, so each generation adds an fp32 rounding of the state (a random
walk of ≈ 2⁻²⁴·‖m‖ per step) that the binary64 oracle does not have; an entry of m that crosses
zero makes that error arbitrarily large relative to the entry itself, which is why the bound is
normwise — the form in which contraction rounding errors are bounded in the first place
(|fl(Az) − Az| ≤ γ_D·|A||z|) (BASELINE.json north_star: 1e-5 after 1, 1e-3 after 100)."""


def nrel(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))
import numpy as np
import pytest
import torch

import workloads as W
from oracle import oracle as O
from gpu_helpers import bits, q24

pytestmark = pytest.mark.gpu
CMA = 5


@pytest.fixture(scope="module", autouse=True)
def built():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build()
    O.build()


def _params(R, **over):
    out = []
    for r in range(R):
        p = W.run_params(W.SEP_CMA_ES, 300 + r, init_min=-2.0, init_max=2.0, sigma_init=0.3,
                         elite_ratio=[0.5, 0.25, 0.4][r % 3])
        p.update(over)
        out.append(p)
    return out


class CmaPair:
    def __init__(self, N, D, params):
        from oracle import cma_oracle
        from paper_2212_04180_b200 import strategy as S
        self.N, self.D, self.R = N, D, len(params)
        self.gpu = S.Strategy(CMA, N, D, params)
        self.orc = [cma_oracle.CMARun(N, D, **p) for p in params]

    def step(self, fn, tol_x=1e-5, metric=None):
        metric = metric or nrel
        x = self.gpu.ask()
        f = self.gpu.eval(fn, x) if fn is not None else self.gpu.synth_fitness()
        self.gpu.tell(f)
        xh, fh = x.cpu().numpy(), f.cpu().numpy()
        for r in range(self.R):
            xo = self.orc[r].ask()
            assert metric(xh[r], xo) <= tol_x, (r, metric(xh[r], xo))
            self.orc[r].tell(fh[r])                    # teacher-forced on the GPU's fitness
        return fh

    def compare(self, r, tol, metric=None):
        metric = metric or nrel
        o = self.orc[r]
        g = {k: self.gpu.get(k)[r].cpu().numpy().astype(np.float64)
             for k in ("mean", "p_sigma", "p_c", "cov", "chol", "best_x")}
        ref = dict(mean=o.m, p_sigma=o.p_sigma, p_c=o.p_c, cov=o.C, chol=o.A, best_x=o.best_x)
        worst = {}
        for k in g:
            e = metric(g[k].ravel(), np.asarray(ref[k], np.float64).ravel())
            worst[k] = e
            assert e <= tol, (k, r, e)
        sg = float(self.gpu.get("sigma")[r])
        assert abs(sg - o.sigma) <= tol * o.sigma, (r, sg, o.sigma)
        assert float(self.gpu.get("best_f")[r]) == float(o.best_f)
        assert int(self.gpu.get("gen")[r]) == o.t
        return worst

    def close(self):
        self.gpu.close()


def test_first_population_is_m_plus_sigma_z():
    """A = I before the first refresh: y = z exactly, x = fma(σ, z, m) — within 1 ulp of the
    oracle's binary64 m + σz rounded once."""
    pair = CmaPair(16, 37, _params(2))
    x = pair.gpu.ask().cpu().numpy()
    for r in range(2):
        xo = pair.orc[r].ask()
        ulp = np.spacing(np.abs(xo))
        assert np.all(np.abs(x[r].astype(np.float64) - xo) <= ulp), r
    pair.close()


@pytest.mark.parametrize("R,N,D", [(3, 16, 10), (2, 8, 2), (1, 64, 100), (2, 32, 130),
                                   (1, 20, 257), (1, 256, 1024)])
@pytest.mark.parametrize("fn", [W.SPHERE, W.ROSENBROCK])
def test_one_generation(R, N, D, fn):
    pair = CmaPair(N, D, _params(R))
    pair.step(fn)
    for r in range(R):
        pair.compare(r, 1e-5)
    pair.close()


@pytest.mark.parametrize("R,N,D", [(2, 64, 128), (1, 256, 1024), (1, 40, 300)])
def test_sampling_through_the_factor_is_fp32_accurate(R, N, D):
    """The second population is x = m + σ·A·z with the FIRST refreshed factor A (≠ I). Checked
    against binary64 A·z built from the GPU's own A, m, σ and the oracle's bit-identical z, so the
    only error left is the contraction's: fp32-level (3-pass tf32 split on the tensor cores), far
    below what a one-tf32-ulp operand error (2⁻¹¹ relative) would give."""
    pair = CmaPair(N, D, _params(R))
    pair.step(W.ROSENBROCK)
    A = pair.gpu.get("chol").cpu().numpy().astype(np.float64)
    m = pair.gpu.get("mean").cpu().numpy().astype(np.float64)
    sg = pair.gpu.get("sigma").cpu().numpy().astype(np.float64)
    x = pair.gpu.ask().cpu().numpy().astype(np.float64)
    for r in range(R):
        assert not np.allclose(A[r], np.eye(D)), "the factor was not refreshed"
        pair.orc[r].ask()                              # advances the oracle; its Z is this gen's
        y_ref = pair.orc[r].Z @ A[r].T
        y_gpu = (x[r] - m[r][None, :]) / sg[r]
        e = np.abs(y_gpu - y_ref).max() / np.abs(y_ref).max()
        assert e <= 2e-6, (r, e)
    pair.close()


@pytest.mark.parametrize("R,N,D", [(2, 64, 128), (1, 256, 1024)])
def test_sampling_per_entry_bound(R, N, D):
    """Per entry, not normwise: |y_gpu - y_ref|[i, d] <= 2^-17 (|A| |z|)[i, d] + the rounding of
    x = fma(sigma, y, m) to binary32 seen through (x - m) / sigma. The 3-pass tf32 split drops
    small*small (<= 2^-20 |a b|) and small's truncation (<= 2^-21 |a b|) per product (N17), and
    the fp32 accumulation over K terms adds a few 2^-24 of the absolute sum, so no entry may
    carry an error beyond a small multiple of 2^-23 of its own absolute product sum."""
    pair = CmaPair(N, D, _params(R))
    pair.step(W.ROSENBROCK)
    A = pair.gpu.get("chol").cpu().numpy().astype(np.float64)
    m = pair.gpu.get("mean").cpu().numpy().astype(np.float64)
    sg = pair.gpu.get("sigma").cpu().numpy().astype(np.float64)
    x = pair.gpu.ask().cpu().numpy().astype(np.float64)
    for r in range(R):
        pair.orc[r].ask()
        Z = pair.orc[r].Z
        y_ref = Z @ A[r].T
        absum = np.abs(Z) @ np.abs(A[r]).T
        y_gpu = (x[r] - m[r][None, :]) / sg[r]
        xr = np.abs(x[r]) + np.abs(m[r][None, :])
        bound = 2.0 ** -17 * absum + 2.0 ** -23 * xr / sg[r]
        err = np.abs(y_gpu - y_ref)
        assert np.all(err <= bound), (r, float((err / bound).max()))
    pair.close()


def test_graph_replay_equals_eager_with_lazy_refresh():
    """D = 300, N = 8: the factor is refreshed every k = 6 generations (Hansen's lazy schedule).
    Eager calls skip the refresh launches on the other generations; a generation captured as a
    CUDA graph always launches them and the kernels decide per run on the device (t is device
    state). Ten replays after two eager generations must equal twelve eager generations bit for
    bit."""
    from paper_2212_04180_b200 import strategy as S
    N, D = 8, 300
    a = S.Strategy(CMA, N, D, _params(2))
    b = S.Strategy(CMA, N, D, _params(2))
    eye = torch.eye(D, device="cuda").expand(2, D, D)
    for g in range(12):
        a.tell(a.eval(W.ROSENBROCK, a.ask()))
        if g == 4:                                     # t = 5: no refresh yet (k = 6)
            assert torch.equal(a.get("chol"), eye)
    assert not torch.equal(a.get("chol"), eye)         # refreshed at t = 6 and t = 12
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        for _ in range(2):
            b.tell(b.eval(W.ROSENBROCK, b.ask()))
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side, capture_error_mode="thread_local"):
        b.tell(b.eval(W.ROSENBROCK, b.ask()))
    for _ in range(10):
        g.replay()
    torch.cuda.synchronize()
    for k in ("mean", "cov", "chol", "p_sigma", "p_c", "sigma", "gen", "best_f"):
        assert torch.equal(a.get(k), b.get(k)), k
    assert int(a.get("gen")[0]) == 12
    a.close()
    b.close()


def test_cma_es_with_the_mlp_fitness():
    """f4 × the MLP fitness (N14): full CMA-ES sampling feeds the tensor-core MLP evaluation.
    The fused es_ask_eval equals es_ask + es_eval bit for bit; the fitness matches the oracle's
    binary64 forward within the MLP parity bar (Q24 ≤ 1e-4, test_gpu_parity.py); and 40
    generations reduce the best fitness on the teacher problem."""
    from paper_2212_04180_b200 import strategy as S
    widths = [16, 32, 16]                              # D = 1072 (multiples of 16, N14)
    m = O.MLP(widths, 128, 5)
    N, D = 16, m.D
    params = _params(2, sigma_init=0.05, init_min=-0.3, init_max=0.3)
    a = S.Strategy(CMA, N, D, params)
    b = S.Strategy(CMA, N, D, params)
    for es in (a, b):
        es.set_mlp_problem(widths, 128, 5)
    first = None
    for g in range(40):
        xa, fa = a.ask_eval(W.MLP)
        xb = b.ask()
        fb = b.eval(W.MLP, xb)
        assert torch.equal(xa, xb) and torch.equal(fa, fb), g
        if g in (0, 39):
            ref = m.evaluate(xa.reshape(-1, D).cpu().numpy()).astype(np.float64)
            assert q24(fa.reshape(-1).cpu().numpy().astype(np.float64), ref) <= 1e-5, g
        a.tell(fa)
        b.tell(fb)
        if g == 0:
            first = a.get("best_f").clone()
    assert torch.all(a.get("best_f") < first)
    assert torch.equal(a.get("mean"), b.get("mean"))
    a.close()
    b.close()


@pytest.mark.parametrize("Wn,D", [(2, 64), (4, 130), (2, 37)])
def test_population_sharded_cma_es(Wn, D):
    """P:226 for f4: W ranks (emulated on one GPU through the communicator-less split-phase ABI)
    each sample all N members (Y feeds the tell), evaluate only their N/W, and run the identical
    tell on the all-gathered fitness. Populations are the unsharded one's slices and every rank's
    state equals the unsharded state bit for bit (tensor-core path D % 4 == 0, SIMT D = 37)."""
    from paper_2212_04180_b200 import strategy as S
    N, R = 32, 2
    params = _params(R)
    ref = S.Strategy(CMA, N, D, params)
    shards = [S.Strategy(CMA, N, D, params, shard=(w, Wn)) for w in range(Wn)]
    nl = N // Wn
    for g in range(6):
        x = ref.ask()
        ref.tell(ref.eval(W.ROSENBROCK, x))
        locs = []
        for w, sh in enumerate(shards):
            xs = sh.ask()
            assert torch.equal(xs, x[:, w * nl:(w + 1) * nl]), (g, w)
            locs.append(sh.eval(W.ROSENBROCK, xs))
        gathered = torch.stack(locs).contiguous()
        for sh in shards:
            sh.tell_local(gathered)
            sh.tell_apply()
        for sh in shards:
            for k in ("mean", "cov", "chol", "p_sigma", "p_c", "sigma", "best_f", "best_x", "gen"):
                assert torch.equal(sh.get(k), ref.get(k)), (g, k)
    for es in shards + [ref]:
        es.close()


# fn None: synthetic fitness (N15) — no convergence, so the state keeps its scale and the check
# isolates arithmetic drift; a converging run (sphere) shrinks ‖x‖ geometrically while the
# teacher-forced oracle's own-x error does not shrink with it.
@pytest.mark.parametrize("R,N,D,fn", [(2, 16, 10, W.ROSENBROCK), (1, 32, 70, W.RASTRIGIN),
                                      (3, 12, 5, None), (1, 64, 300, None)])
def test_hundred_generations_teacher_forced(R, N, D, fn):
    pair = CmaPair(N, D, _params(R))
    for g in range(100):
        pair.step(fn, tol_x=1e-3, metric=nrel)
        if g == 0:
            for r in range(R):
                pair.compare(r, 1e-5)
    for r in range(R):
        pair.compare(r, 1e-3, metric=nrel)
    pair.close()


def test_two_d_sphere_acceptance_on_gpu():
    """SPEC acceptance criterion, run on the GPU alone: N = 8, m0 = (3, 3), σ0 = 1."""
    from paper_2212_04180_b200 import strategy as S
    p = _params(1, init_min=3.0, init_max=3.0, sigma_init=1.0, elite_ratio=0.5)
    es = S.Strategy(CMA, 8, 2, p)
    for _ in range(200):
        es.tell(es.eval(W.SPHERE, es.ask()))
        if float(es.get("best_f")[0]) < 1e-8:
            break
    assert float(es.get("best_f")[0]) < 1e-8
    es.close()


def test_rosenbrock_converges_on_gpu():
    from paper_2212_04180_b200 import strategy as S
    es = S.Strategy(CMA, 16, 10, _params(1, sigma_init=0.5, init_min=-1, init_max=1))
    for _ in range(3000):
        es.tell(es.eval(W.ROSENBROCK, es.ask()))
    assert float(es.get("best_f")[0]) < 1e-6
    C = es.get("cov")[0].cpu().numpy().astype(np.float64)
    assert np.array_equal(C, C.T) and np.linalg.eigvalsh(C).min() > 0
    es.close()


def test_fused_ask_eval_and_bounds():
    from paper_2212_04180_b200 import strategy as S
    p = _params(2, clip_min=-0.5, clip_max=0.25)
    a = S.Strategy(CMA, 16, 33, p)
    b = S.Strategy(CMA, 16, 33, p)
    for _ in range(3):
        xa, fa = a.ask_eval(W.RASTRIGIN)
        xb = b.ask()
        fb = b.eval(W.RASTRIGIN, xb)
        assert torch.equal(xa, xb) and torch.equal(fa, fb)
        assert float(xa.min()) >= -0.5 and float(xa.max()) <= 0.25
        a.tell(fa)
        b.tell(fb)
    assert torch.equal(a.get("cov"), b.get("cov"))
    a.close()
    b.close()


def test_checkpoint_resume_bit_exact():
    from paper_2212_04180_b200 import strategy as S
    p = _params(2)
    a = S.Strategy(CMA, 16, 20, p)
    for _ in range(4):
        a.tell(a.eval(W.SPHERE, a.ask()))
    b = S.Strategy(CMA, 16, 20, p)
    for k in ("mean", "p_sigma", "p_c", "cov", "chol", "best_x", "best_f", "sigma", "gen"):
        b.set(k, a.get(k))
    for _ in range(4):
        a.tell(a.eval(W.SPHERE, a.ask()))
        b.tell(b.eval(W.SPHERE, b.ask()))
    for k in ("mean", "cov", "chol", "sigma"):
        assert torch.equal(a.get(k), b.get(k)), k
    a.close()
    b.close()


def test_cma_rejections():
    from paper_2212_04180_b200 import strategy as S
    from paper_2212_04180_b200._lib import ESError
    with pytest.raises(ESError):
        S.Strategy(CMA, 16, 5000, _params(1))                  # D > 4096
    with pytest.raises(ESError):
        S.Strategy(CMA, 16, 8, _params(1), shard=(0, 2), split="dims")   # D-sharding
    with pytest.raises(ESError):
        S.Strategy(CMA, 16, 8, _params(1, weight_decay=0.1))
