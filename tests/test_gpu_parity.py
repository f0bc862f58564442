"""GPU parity of the CUDA path (through the C ABI) against the CPU oracle.

Bar (BASELINE.json north_star): noise / populations and ranks bit-exact; fitness and state within
1e-5 (Q24 metric) after one generation and 1e-3 after 100. Sizes span several tiles and ragged
tails (D not a multiple of 4, D not a multiple of the 128-quad block, direction ranges split across
CTAs); full BASELINE sizes are checked on sampled runs / dimensions."""
import ctypes as C

import numpy as np
import pytest
import torch

import workloads as W
from oracle import oracle as O
from gpu_helpers import KEPT, Pair, bits, compare_to_oracle, q24

pytestmark = pytest.mark.gpu

ALGOS = [W.OPENAI_ES, W.PGPE, W.SNES, W.SEP_CMA_ES]
FNS = [W.SPHERE, W.ROSENBROCK, W.RASTRIGIN]


@pytest.fixture(scope="module", autouse=True)
def built():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build()
    O.build()


def L():
    from paper_2212_04180_b200 import _lib
    return _lib.lib()


def _prim(which, inp, out):
    rc = L().es_debug_primitive(which, C.c_void_p(inp.data_ptr()), C.c_void_p(out.data_ptr()),
                                inp.shape[0], None)
    assert rc == 0
    torch.cuda.synchronize()
    return out


# ------------------------------------------------------------------------ N1–N5 primitives
def test_philox_kat_on_device():
    import json, os
    kat = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "philox_kat.json")))
    rows = [[int(h, 16) for h in v["ctr"] + v["key"]] for v in kat["vectors"]]
    inp = torch.tensor(np.array(rows, dtype=np.uint32).view(np.int32), device="cuda")
    out = _prim(0, inp, torch.empty((len(rows), 4), dtype=torch.int32, device="cuda"))
    got = out.cpu().numpy().view(np.uint32)
    for g, v in zip(got, kat["vectors"]):
        assert [f"{x:08x}" for x in g] == v["out"]


def test_ln_exhaustive_bit_exact():
    m = np.arange(2 ** 23, dtype=np.float64)
    ua = (1.0 - m * 2.0 ** -23).astype(np.float32)
    dev = _prim(1, torch.from_numpy(ua).cuda(), torch.empty(ua.size, device="cuda"))
    assert np.array_equal(bits(dev.cpu().numpy()), bits(O.ln(ua)))


def test_rho_exhaustive_bit_exact():
    """ρ = sqrt_rn(−2·LN(u_a)) on every one of the 2^23 values u_a can take: the branchless device
    square root equals the oracle's IEEE sqrtf (numpy float32 sqrt) bit for bit."""
    m = np.arange(2 ** 23, dtype=np.float64)
    ua = (1.0 - m * 2.0 ** -23).astype(np.float32)
    x = (np.float32(-2.0) * O.ln(ua)).astype(np.float32)
    dev = _prim(4, torch.from_numpy(x).cuda(), torch.empty(x.size, device="cuda"))
    assert np.array_equal(bits(dev.cpu().numpy()), bits(np.sqrt(x)))


def test_sinpi_half_bit_exact():
    b = np.concatenate([np.linspace(0, 0.5, 1 << 22), np.exp2(np.random.default_rng(5).uniform(-126, -1, 1 << 20))])
    b = b.astype(np.float32)
    dev = _prim(5, torch.from_numpy(b).cuda(), torch.empty(b.size, device="cuda"))
    assert np.array_equal(bits(dev.cpu().numpy()), bits(O.sinpi_half(b)))


def test_sincos_exhaustive_bit_exact():
    ub = (np.arange(2 ** 23, dtype=np.float64) * 2.0 ** -23).astype(np.float32)
    rng = np.random.default_rng(0)
    extra = np.concatenate([rng.uniform(0, 0.5, 1 << 20), np.exp2(rng.uniform(-60, -1, 1 << 18))])
    u = np.concatenate([ub, extra.astype(np.float32)])
    dev = _prim(2, torch.from_numpy(u).cuda(), torch.empty((u.size, 2), device="cuda")).cpu().numpy()
    c, s = O.sincos2pi(u)
    assert np.array_equal(bits(dev[:, 0]), bits(c)) and np.array_equal(bits(dev[:, 1]), bits(s))


def test_mlp_tanh_accuracy():
    """N14's activation: the device tanh (odd rational x p(x^2)/q(x^2), one MUFU rcp) is
    within 5e-7 relative of binary64 tanh over a dense sweep of [-12, 12], tiny and huge values
    (odd, saturating at +-1, tanh(0) = 0)."""
    rng = np.random.default_rng(11)
    x = np.concatenate([np.linspace(-12, 12, 1 << 22), rng.uniform(-0.7, 0.7, 1 << 20),
                        np.exp2(rng.uniform(-40, 3, 1 << 18)) * rng.choice([-1, 1], 1 << 18),
                        [0.0, -0.0, 0.625, -0.625, 0.62499997, 30.0, -30.0, 1e30, -1e30]])
    x = x.astype(np.float32)
    dev = _prim(6, torch.from_numpy(x).cuda(), torch.empty(x.size, device="cuda")).cpu().numpy()
    ref = np.tanh(x.astype(np.float64))
    rel = np.abs(dev.astype(np.float64) - ref) / np.maximum(np.abs(ref), 1e-30)
    assert rel.max() <= 5e-7, (rel.max(), x[rel.argmax()])
    assert np.all(dev[x == 0] == 0.0)


def test_mlp16_hidden_tanh():
    """N14′'s hidden-layer tanh (its value is rounded to binary16 next): within 3.5e-7 relative
    of binary64 tanh on |x| <= 4.6, and beyond the clamp its binary16 rounding is exactly +-1
    (as tanh's is: tanh(4.6) > 1 - 2^-12); odd, tanh(0) = 0."""
    rng = np.random.default_rng(12)
    x = np.concatenate([np.linspace(-12, 12, 1 << 22), rng.uniform(-0.7, 0.7, 1 << 20),
                        np.exp2(rng.uniform(-40, 3, 1 << 18)) * rng.choice([-1, 1], 1 << 18),
                        [0.0, 4.6, -4.6, 4.59999, 4.60001, 30.0, -30.0, 1e30, -1e30]])
    x = x.astype(np.float32)
    dev = _prim(7, torch.from_numpy(x).cuda(), torch.empty(x.size, device="cuda")).cpu().numpy()
    ref = np.tanh(x.astype(np.float64))
    inr = np.abs(x) <= np.float32(4.6)
    rel = np.abs(dev[inr].astype(np.float64) - ref[inr]) / np.maximum(np.abs(ref[inr]), 1e-30)
    assert rel.max() <= 3.5e-7, (rel.max(), x[inr][rel.argmax()])
    h = dev[~inr].astype(np.float16)
    assert np.array_equal(h, np.sign(x[~inr]).astype(np.float16)), h
    assert np.all(dev[x == 0] == 0.0)
    assert np.array_equal(dev[x == 4.6], -dev[x == -4.6])


@pytest.mark.parametrize("seed,i,t,tag", [(0, 0, 0, 0), (12345, 7, 3, 0), (2 ** 40 + 5, 99, 1000, 1),
                                          (77, 0, 0, 4)])
def test_normals_bit_exact(seed, i, t, tag):
    n4 = 1 << 20
    q = np.arange(n4, dtype=np.uint32)
    rows = np.stack([q, np.full(n4, i), np.full(n4, t), np.full(n4, tag),
                     np.full(n4, seed & 0xFFFFFFFF), np.full(n4, seed >> 32)], 1).astype(np.uint32)
    dev = _prim(3, torch.from_numpy(rows.view(np.int32)).cuda(),
                torch.empty((n4, 4), device="cuda")).cpu().numpy().reshape(-1)
    assert np.array_equal(bits(dev), bits(O.normals(seed, i, t, tag, 4 * n4)))


# ------------------------------------------------------------------------ ask
def _params(algo, R, hyper=False, **over):
    cfg = dict(algo=algo, init=(-2.0, 2.0))
    out = []
    for r in range(R):
        p = W.config_params(cfg, r, seed_offset=1000 * algo + 17, hyper_vmap=hyper)
        p.update(over)
        out.append(p)
    return out


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("N,D", [(16, 1), (16, 10), (64, 1000), (32, 4099), (8, 513)])
def test_ask_bit_exact(algo, N, D):
    pair = Pair(algo, N, D, _params(algo, 3, hyper=True))
    x = pair.gpu.ask().cpu().numpy()
    for r in range(pair.R):
        assert np.array_equal(bits(x[r]), bits(pair.orc[r].ask())), r
    pair.close()


# ------------------------------------------------------------------------ fitness
@pytest.mark.parametrize("fn", FNS)
@pytest.mark.parametrize("n,D", [(7, 1), (33, 2), (64, 7), (64, 1000), (12000, 21), (50, 6000), (16, 4097), (4, 70001),
                                 (3, 262144)])
def test_eval_parity(fn, n, D):
    from paper_2212_04180_b200 import strategy as S
    rng = np.random.default_rng(n * 7 + D + fn)
    x = W.random_population(rng, n, D, scale=2.5)
    got = S.eval_bbob(fn, torch.from_numpy(x).cuda()).cpu().numpy()
    ref = O.evaluate(fn, x)
    ulp = np.abs(bits(got).astype(np.int64) - bits(ref).astype(np.int64))
    assert ulp.max() <= 1 and (ulp > 0).sum() <= max(1, n // 1000), ulp


def test_rastrigin_special_values():
    """The Rastrigin kernel forms (double)S from S's bit pattern (NUMERICS N7 GPU detail): exact for
    normal S; S = 0 (integer x) and subnormal S (subnormal x) take ~2⁻¹²⁷-scale values whose squares
    cannot move the sum. Rows of integers, zeros, ±0, subnormals, halves and large values — alone
    and mixed — must still agree with the oracle's binary64 evaluation to ≤ 1 ulp."""
    from paper_2212_04180_b200 import strategy as S
    sub = np.float32(1e-40)
    rows = [np.zeros(64), -np.zeros(64), np.arange(-32, 32), np.full(64, sub),
            np.full(64, 0.5), np.full(64, -2.5), np.linspace(-5.12, 5.12, 64),
            np.concatenate([np.zeros(32), np.full(32, 1e-3)]),
            np.concatenate([np.arange(16), np.full(16, sub), np.full(32, 3.75)]),
            np.full(64, 1e10), np.full(64, 2.0 ** -20)]
    x = np.stack(rows).astype(np.float32)
    got = S.eval_bbob(W.RASTRIGIN, torch.from_numpy(x).cuda()).cpu().numpy()
    ref = O.evaluate(W.RASTRIGIN, x)
    ulp = np.abs(bits(got).astype(np.int64) - bits(ref).astype(np.int64))
    assert ulp.max() <= 1, (got, ref)
    assert got[0] == 0.0 and got[1] == 0.0 and got[2] == ref[2]


def test_eval_empty_and_host_buffers():
    n, D = 5, 37
    x = W.random_population(np.random.default_rng(1), n, D)
    f = np.zeros(n, np.float32)
    rc = L().es_eval_bbob(None, W.RASTRIGIN, x.ctypes.data_as(C.c_void_p), n, D,
                          f.ctypes.data_as(C.c_void_p), None)
    assert rc == 0
    assert np.array_equal(bits(f), bits(O.evaluate(W.RASTRIGIN, x)))
    assert L().es_eval_bbob(None, 0, x.ctypes.data_as(C.c_void_p), 0, D,
                            f.ctypes.data_as(C.c_void_p), None) == 0


# ------------------------------------------------------------------------ ranks
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("N,R", [(2, 3), (16, 3), (256, 3), (1000, 3), (4096, 3), (16384, 3),
                                 (16386, 3), (40000, 3), (65536, 3), (2, 1), (256, 20),
                                 (4096, 17), (300, 1), (4096, 1)])
def test_rank_and_shaping_bit_exact(algo, N, R):
    """R <= 16 and N <= 16384 rank by counting over many CTAs, other shapes by the per-run
    bitonic sort (and the hybrid global-memory sort above 16384): every path bit-exact."""
    if algo == W.SEP_CMA_ES and N < 16:
        pytest.skip("elite ratio 0.2 needs N >= 5")
    pair = Pair(algo, N, 6, _params(algo, R, hyper=True))
    rng = np.random.default_rng(N + algo)
    f = np.stack([W.random_fitness(rng, N, ties=N // 5 + 1, nans=min(3, N // 8), infs=min(2, N // 8))
                  for _ in range(R)])
    pair.gpu.ask()
    pair.gpu.tell(torch.from_numpy(f).cuda())
    S_, E_, P_, SH = (pair.gpu.get(k).cpu().numpy() for k in ("rank_s", "rank_e", "perm", "shaped"))
    for r in range(R):
        s, e, perm = O.rank(f[r])
        assert np.array_equal(S_[r], s) and np.array_equal(E_[r], e) and np.array_equal(P_[r], perm)
        if algo in (W.OPENAI_ES, W.PGPE):
            ref = O.centered_rank(f[r])
        else:
            ref = O.member_weights(pair.orc[r].wpos, f[r])
        assert np.array_equal(bits(SH[r]), bits(ref)), r
    pair.close()


# ------------------------------------------------------------------------ one generation
SHAPES = [(3, 16, 10), (2, 64, 1003), (1, 256, 5000), (2, 32, 130), (1, 2, 1), (2, 1030, 40), (2, 8200, 12)]


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("R,N,D", SHAPES)
@pytest.mark.parametrize("fn", [W.SPHERE, W.RASTRIGIN])
def test_one_generation(algo, R, N, D, fn):
    if algo == W.SEP_CMA_ES and N < 4:
        pytest.skip("elite needs N >= 4 at ratio 0.4")
    pair = Pair(algo, N, D, _params(algo, R, hyper=True))
    x = pair.gpu.ask()
    f = pair.gpu.eval(fn, x)
    pair.gpu.tell(f)
    fh = f.cpu().numpy()
    xh = x.cpu().numpy()
    for r in range(R):
        xo = pair.orc[r].ask()
        assert np.array_equal(bits(xh[r]), bits(xo))
        fo = O.evaluate(fn, xo)
        assert q24(fh[r], fo) <= 1e-5
        pair.orc[r].tell(fh[r])                  # teacher-forced on the GPU's fitness
        pair.compare(r, 1e-5)
    pair.close()


# ------------------------------------------------------------------------ 100 generations
@pytest.mark.parametrize("algo,fn,N,D,R", [
    (W.OPENAI_ES, W.SPHERE, 16, 10, 1),          # config 1, full size
    (W.PGPE, W.ROSENBROCK, 32, 200, 2),
    (W.SNES, W.RASTRIGIN, 32, 100, 3),
    (W.SEP_CMA_ES, W.RASTRIGIN, 32, 100, 3),
])
def test_hundred_generations(algo, fn, N, D, R):
    """Both sides run free (each evaluates its own population): 1e-5 after 1, 1e-3 after 100."""
    cfg = W.CONFIGS["c1"] if algo == W.OPENAI_ES else dict(algo=algo, init=(-5.12, 5.12))
    params = [W.config_params(cfg, r, seed_offset=0) for r in range(R)]
    pair = Pair(algo, N, D, params)
    for g in range(100):
        x = pair.gpu.ask()
        f = pair.gpu.eval(fn, x)
        pair.gpu.tell(f)
        for r in range(R):
            o = pair.orc[r]
            o.tell(O.evaluate(fn, o.ask()))
        if g == 0:
            for r in range(R):
                pair.compare(r, 1e-5)
    for r in range(R):
        pair.compare(r, 1e-3)
    pair.close()


# ------------------------------------------------------------------------ invariants
@pytest.mark.parametrize("algo", ALGOS)
def test_multirun_equals_solo(algo):
    """vmap semantics: run r of an R-batch is bit-identical to the same run alone."""
    from paper_2212_04180_b200 import strategy as S
    params = _params(algo, 5, hyper=True)
    batch = S.Strategy(algo, 32, 257, params)
    solo = S.Strategy(algo, 32, 257, [params[3]])
    for _ in range(5):
        for es in (batch, solo):
            es.tell(es.eval(W.RASTRIGIN, es.ask()))
    for f in KEPT[algo]:
        assert np.array_equal(bits(batch.get(f)[3].cpu().numpy()), bits(solo.get(f)[0].cpu().numpy()))
    batch.close()
    solo.close()


def test_tell_without_ask_is_bad_state():
    from paper_2212_04180_b200 import strategy as S
    from paper_2212_04180_b200._lib import ESError
    es = S.Strategy(W.SNES, 8, 4, _params(W.SNES, 1))
    with pytest.raises(ESError) as ei:
        es.tell(torch.zeros((1, 8), device="cuda"))
    assert ei.value.code == 2
    es.close()


@pytest.mark.parametrize("algo", ALGOS)
def test_checkpoint_resume(algo):
    """es_get / es_set round trip: a resumed run continues bit-identically."""
    from paper_2212_04180_b200 import strategy as S
    params = _params(algo, 2)
    a = S.Strategy(algo, 16, 50, params)
    for _ in range(3):
        a.tell(a.eval(W.SPHERE, a.ask()))
    b = S.Strategy(algo, 16, 50, params)
    names = KEPT[algo] + ["best_f", "gen"] + (["sigma"] if algo in (0, 3) else []) + \
        (["lrate"] if algo in (0, 1) else [])
    for nm in names:
        b.set(nm, a.get(nm))
    for es in (a, b):
        es.tell(es.eval(W.SPHERE, es.ask()))
    for nm in KEPT[algo]:
        assert np.array_equal(bits(a.get(nm).cpu().numpy()), bits(b.get(nm).cpu().numpy())), nm
    a.close()
    b.close()


def test_host_buffer_path_matches_device():
    from paper_2212_04180_b200 import strategy as S
    from paper_2212_04180_b200._lib import check
    params = _params(W.PGPE, 2)
    a = S.Strategy(W.PGPE, 16, 33, params)
    b = S.Strategy(W.PGPE, 16, 33, params)
    xa = a.ask()
    xb = torch.empty((2, 16, 33), dtype=torch.float32).pin_memory()
    check(L().es_ask(b.ctx, C.c_void_p(xb.data_ptr()), None), b.ctx)
    assert torch.equal(xa.cpu(), xb)
    fa = a.eval(W.SPHERE, xa)
    fb = fa.cpu().numpy().copy()
    a.tell(fa)
    check(L().es_tell(b.ctx, fb.ctypes.data_as(C.c_void_p), None), b.ctx)
    assert torch.equal(a.get("mean"), b.get("mean"))
    a.close()
    b.close()


# ------------------------------------------------------------------------ full BASELINE sizes
@pytest.mark.parametrize("key", ["c2_sepcma", "c2_snes"])
def test_config2_full_size_sampled_runs(key):
    cfg = W.CONFIGS[key]
    R, N, D = cfg["R"], cfg["N"], cfg["D"]
    params = [W.config_params(cfg, r, hyper_vmap=True) for r in range(R)]
    from paper_2212_04180_b200 import strategy as S
    es = S.Strategy(cfg["algo"], N, D, params)
    x = es.ask()
    f = es.eval(cfg["fn"], x)
    es.tell(f)
    xh, fh = x.cpu().numpy(), f.cpu().numpy()
    for r in (0, 1, 255, R - 1):
        o = O.Run(cfg["algo"], N, D, **params[r])
        xo = o.ask()
        assert np.array_equal(bits(xh[r]), bits(xo))
        assert q24(fh[r], O.evaluate(cfg["fn"], xo)) <= 1e-5
        o.tell(fh[r])
        for fld in KEPT[cfg["algo"]]:
            g = es.get(fld)[r].cpu().numpy()
            assert q24(g, o.vec[["mean", "sigma_d", "adam_m", "adam_v", "p_sigma", "p_c", "C",
                                 "best_x"].index(fld)]) <= 1e-5, fld
    es.close()


def test_config3_full_size():
    cfg = W.CONFIGS["c3"]
    params = [W.config_params(cfg, 0)]
    pair = Pair(cfg["algo"], cfg["N"], cfg["D"], params)
    x = pair.gpu.ask()
    f = pair.gpu.eval(cfg["fn"], x)
    pair.gpu.tell(f)
    xo = pair.orc[0].ask()
    assert np.array_equal(bits(x[0].cpu().numpy()), bits(xo))
    fo = O.evaluate(cfg["fn"], xo)
    assert q24(f[0].cpu().numpy(), fo) <= 1e-5
    pair.orc[0].tell(f[0].cpu().numpy())
    pair.compare(0, 1e-5)
    pair.close()


@pytest.mark.parametrize("N,D", [(4096, 985_216), (16384, 100_000), (256, 10_000_000),
                                 (65536, 1000), (32768, 10_000)])
def test_tell_full_size_sampled_dims(N, D):
    """Config 4 / sweep sizes: the tell on synthetic fitness (N15), checked on 64 sampled quads
    (incl. the first and last) by an oracle run restricted to those dimensions."""
    rng = np.random.default_rng(N)
    quads = np.unique(np.concatenate([[0, (D - 1) // 4], rng.integers(0, (D + 3) // 4, 62)]))
    dims = np.array([4 * q + k for q in quads for k in range(4) if 4 * q + k < D])
    params = [W.run_params(W.OPENAI_ES, 5, init_min=-0.04, init_max=0.04)]
    pair = Pair(W.OPENAI_ES, N, D, params, dims=dims)
    f = pair.gpu.synth_fitness()          # stands in for ask + evaluate (x never materialised)
    fo = O.synth_fitness(params[0]["seed"], 0, N)
    assert np.array_equal(bits(f[0].cpu().numpy()), bits(fo))
    pair.gpu.tell(f)
    pair.orc[0].tell(fo)
    pair.compare(0, 1e-5)
    pair.close()


# ------------------------------------------------------------------------ sharded population
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("Wn", [2, 4])
def test_emulated_shards_match_single_gpu(algo, Wn):
    """W communicator-less shards on one GPU, exchanging through the split-phase ABI exactly as
    es_tell does through NCCL (all-gather of fitness, binary64 sum of the direction sums in rank
    order): populations and ranks bit-identical to the unsharded run, state within 1e-6 of it —
    and every shard's state within 1e-5 of the ORACLE run fed the same fitness (teacher-forced)."""
    from paper_2212_04180_b200 import strategy as S
    N, D, R = 32, 301, 2
    params = _params(algo, R, hyper=True)
    ref = S.Strategy(algo, N, D, params)
    shards = [S.Strategy(algo, N, D, params, shard=(w, Wn)) for w in range(Wn)]
    orcs = [O.Run(algo, N, D, **p) for p in params]
    nl = N // Wn
    for gen in range(3):
        x = ref.ask()
        f = ref.eval(W.RASTRIGIN, x)
        ref.tell(f)
        fh = f.cpu().numpy()
        for r, o in enumerate(orcs):
            assert np.array_equal(bits(o.ask()), bits(x[r].cpu().numpy())), (gen, r)
            o.tell(fh[r])
        locs = []
        for w, sh in enumerate(shards):
            xs = sh.ask()
            assert torch.equal(xs, x[:, w * nl:(w + 1) * nl]), (gen, w)
            locs.append(sh.eval(W.RASTRIGIN, xs))
        gathered = torch.stack(locs).contiguous()                 # [W][R][N/W]
        for sh in shards:
            sh.tell_local(gathered)
        total = shards[0].get("dirsum")
        for sh in shards[1:]:
            total = total + sh.get("dirsum")
        for sh in shards:
            sh.set("dirsum", total)
            sh.tell_apply()
        for sh in shards:
            for k in ("perm", "shaped"):
                assert torch.equal(sh.get(k), ref.get(k)), k
            for fld in KEPT[algo]:
                assert q24(sh.get(fld).cpu().numpy(), ref.get(fld).cpu().numpy()) <= 1e-6, fld
            for r, o in enumerate(orcs):
                compare_to_oracle(sh, algo, r, o, 1e-5)
    for es in shards + [ref]:
        es.close()


@pytest.mark.parametrize("algo", ALGOS + [W.ARS])
def test_nccl_one_rank_collective_tell(algo):
    """The population-sharded data plane of es_tell executed for real on one GPU: a one-rank NCCL
    communicator makes es_tell run ncclAllGather of the fitness (a5), ncclAllReduce of the binary64
    direction sums (a8) and the separate update kernel. Ranks bit-exact and state within 1e-5 of
    the ORACLE after 1 generation, 1e-3 after 30 (north_star tolerances), and identical to the
    fused single-GPU tell up to the reduce/update split (1e-6)."""
    from paper_2212_04180_b200 import strategy as S
    N, D, R = 64, 203, 2
    params = _params(algo, R, hyper=True)
    es = S.Strategy(algo, N, D, params, single_comm=True)
    ref = S.Strategy(algo, N, D, params)
    orcs = [O.Run(algo, N, D, **p) for p in params]
    for gen in range(30):
        x = es.ask()
        f = es.eval(W.RASTRIGIN, x)
        es.tell(f)
        xr = ref.ask()
        assert torch.equal(x, xr), gen
        ref.tell(ref.eval(W.RASTRIGIN, xr))
        fh = f.cpu().numpy()
        for r, o in enumerate(orcs):
            assert np.array_equal(bits(o.ask()), bits(x[r].cpu().numpy())), (gen, r)
            o.tell(fh[r])
        assert torch.equal(es.get("perm"), ref.get("perm"))
        for r, o in enumerate(orcs):
            compare_to_oracle(es, algo, r, o, 1e-5 if gen == 0 else 1e-3)
        for fld in KEPT[algo]:
            assert q24(es.get(fld).cpu().numpy(), ref.get(fld).cpu().numpy()) <= 1e-6, (gen, fld)
    for e in (es, ref):
        e.close()


# ------------------------------------------------------------------------ MLP fitness (N14, tcgen05)
def _mlp_population(m, n, seed):
    theta = m.teacher()
    rng = np.random.default_rng(seed)
    scales = np.geomspace(1e-3, 0.5, n)
    return theta, np.stack([theta + s * rng.standard_normal(m.D) for s in scales]).astype(np.float32)


@pytest.mark.parametrize("widths,n", [([32, 64, 64, 64, 64, 16], 24), ([16, 32], 8),
                                      ([256, 512, 512, 512, 512, 128], 6),
                                      ([96, 160, 48], 10), ([48, 16, 32], 5)])
def test_mlp_fitness_parity(widths, n):
    """N14, the definition (fp32 parameters) on the fp32-accurate tcgen05 kernel
    (binary16 hi/lo split, three products summed in TMEM): within the north star's 1e-5 of the
    oracle's binary64 forward (Q24 metric over the population's fitness vector, and per member for
    f >= 1e-3); f(theta*) = 0 exactly (the GPU's own teacher targets)."""
    from paper_2212_04180_b200 import strategy as S
    m = O.MLP(widths, 128, 7)
    es = S.Strategy(W.OPENAI_ES, 16, m.D, [W.run_params(W.OPENAI_ES, 1, init_min=-0.04,
                                                       init_max=0.04)])
    es.set_mlp_problem(widths, 128, 7)
    theta, xs = _mlp_population(m, n, len(widths))
    f0 = es.eval(W.MLP, torch.from_numpy(theta[None]).cuda(), out=torch.empty(1, device="cuda"))
    assert float(f0[0]) == 0.0
    got = es.eval(W.MLP, torch.from_numpy(xs).cuda(), out=torch.empty(n, device="cuda"))
    got = got.cpu().numpy().astype(np.float64)
    ref = m.evaluate(xs).astype(np.float64)
    assert q24(got, ref) <= 1e-5, (got, ref)
    big = ref >= 1e-3
    assert np.all(np.abs(got[big] - ref[big]) <= 1e-5 * ref[big]), (got, ref)
    es.close()


@pytest.mark.parametrize("widths,n", [([32, 64, 64, 64, 64, 16], 24),
                                      ([256, 512, 512, 512, 512, 128], 6)])
def test_mlp16_approximation_bound(widths, n):
    """ES_FIT_MLP16 (N14', the fp16 parameter image) is a labelled approximation: (i) within the
    Q24 1e-4 of the oracle's model of it (binary16 operands, fp32 vs binary64 accumulation flips
    rare fp16 activation roundings) and (ii) within its derived distance to the
    definition, |f16 - f| <= |model - f| + 1e-4 |model| per member, both oracle-computed."""
    from paper_2212_04180_b200 import strategy as S
    m = O.MLP(widths, 128, 7)
    es = S.Strategy(W.OPENAI_ES, 16, m.D, [W.run_params(W.OPENAI_ES, 1)])
    es.set_mlp_problem(widths, 128, 7)
    theta, xs = _mlp_population(m, n, len(widths) + 1)
    f0 = es.eval(W.MLP16, torch.from_numpy(theta[None]).cuda(), out=torch.empty(1, device="cuda"))
    assert float(f0[0]) == 0.0
    got = es.eval(W.MLP16, torch.from_numpy(xs).cuda(), out=torch.empty(n, device="cuda"))
    got = got.cpu().numpy().astype(np.float64)
    model = m.evaluate_f16(xs).astype(np.float64)
    ref = m.evaluate(xs).astype(np.float64)
    assert q24(got, model) <= 1e-4, (got, model)
    bound = np.abs(model - ref) + 1e-4 * np.maximum(np.abs(model), 2 ** -10 * np.abs(model).max())
    assert np.all(np.abs(got - ref) <= bound), (got, ref, model)
    es.close()


def test_mlp_openai_es_generations_teacher_forced():
    """Config-4 path (es_ask_eval with the fp32-accurate MLP) at SURVEY §8(d)'s reduced size
    ([32, 64x4, 16], D = 15,632, N = 256) for 100 generations: ask bit-exact every generation, MLP
    fitness within 1e-5 (Q24) of the oracle on sampled generations, tell fed the GPU's fitness
    within 1e-5 after one generation and 1e-3 after 100."""
    from paper_2212_04180_b200 import strategy as S
    widths = [32, 64, 64, 64, 64, 16]
    m = O.MLP(widths, 128, 3)
    params = [W.run_params(W.OPENAI_ES, 9, init_min=-0.04, init_max=0.04)]
    pair = Pair(W.OPENAI_ES, 256, m.D, params)
    pair.gpu.set_mlp_problem(widths, 128, 3)
    for g in range(100):
        x, f = pair.gpu.ask_eval(W.MLP)
        xo = pair.orc[0].ask()
        assert np.array_equal(bits(x[0].cpu().numpy()), bits(xo)), g
        if g in (0, 50, 99):
            fo = m.evaluate(xo[:32])
            assert q24(f[0, :32].cpu().numpy(), fo) <= 1e-5, g
        pair.gpu.tell(f)
        pair.orc[0].tell(f[0].cpu().numpy())
        if g == 0:
            pair.compare(0, 1e-5)
    pair.compare(0, 1e-3)
    pair.close()


# ------------------------------------------------------------------------ fused ask + evaluate (f1)
@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("fn", FNS)
@pytest.mark.parametrize("N,D", [(16, 1), (16, 10), (64, 1000), (32, 4099), (8, 513), (256, 1000)])
def test_ask_eval_fused(algo, fn, N, D):
    """x bit-identical to es_ask, fitness within 1 ulp of the oracle (and bit-identical whether or
    not x is materialised), and the generation tells normally afterwards."""
    from paper_2212_04180_b200 import strategy as S
    params = _params(algo, 3, hyper=True)
    es = S.Strategy(algo, N, D, params)
    x1, f1 = es.ask_eval(fn)
    _, f2 = es.ask_eval(fn, write_x=False)
    x0 = es.ask()
    assert torch.equal(x1, x0)
    assert np.array_equal(bits(f1.cpu().numpy()), bits(f2.cpu().numpy()))
    xh, fh = x0.cpu().numpy(), f1.cpu().numpy()
    for r in range(3):
        ref = O.evaluate(fn, xh[r])
        ulp = np.abs(bits(fh[r]).astype(np.int64) - bits(ref).astype(np.int64))
        assert ulp.max() <= 1 and (ulp > 0).sum() <= max(1, N // 64), ulp
    es.tell(f1)
    es.close()


@pytest.mark.parametrize("widths,N", [([32, 64, 64, 64, 64, 16], 64),
                                      ([256, 512, 512, 512, 512, 128], 32), ([96, 160, 48], 16)])
def test_mlp_fused_fp16_image_path(widths, N):
    """N14′: es_ask_eval(ES_FIT_MLP16) — ask writes the fp16 image, the TMA-fed tcgen05 kernel
    evaluates it — gives x bit-identical to es_ask and fitness bit-identical to es_eval_bbob(MLP16)
    on the fp32 population (with or without materialising x), and within the Q24 1e-4 of the
    oracle's model of the approximation; es_ask_eval(ES_FIT_MLP) likewise equals es_eval_bbob(MLP)
    bit for bit (x given or internal)."""
    from paper_2212_04180_b200 import strategy as S
    m = O.MLP(widths, 128, 5)
    params = [W.run_params(W.OPENAI_ES, 3, init_min=-0.04, init_max=0.04)]
    es = S.Strategy(W.OPENAI_ES, N, m.D, params)
    es.set_mlp_problem(widths, 128, 5)
    x1, f1 = es.ask_eval(W.MLP16)
    _, f2 = es.ask_eval(W.MLP16, write_x=False)
    x0 = es.ask()
    f0 = es.eval(W.MLP16, x0)
    assert torch.equal(x1, x0)
    assert np.array_equal(bits(f1.cpu().numpy()), bits(f0.cpu().numpy()))
    assert np.array_equal(bits(f2.cpu().numpy()), bits(f0.cpu().numpy()))
    ref = m.evaluate_f16(x0[0].cpu().numpy())
    assert q24(f1[0].cpu().numpy(), ref) <= 1e-4
    x3, f3 = es.ask_eval(W.MLP)
    _, f4 = es.ask_eval(W.MLP, write_x=False)
    f5 = es.eval(W.MLP, x0)
    assert torch.equal(x3, x0)
    assert np.array_equal(bits(f3.cpu().numpy()), bits(f5.cpu().numpy()))
    assert np.array_equal(bits(f4.cpu().numpy()), bits(f5.cpu().numpy()))
    es.tell(f3)
    es.close()


def test_config4_full_size_sampled_members():
    """C4 in the launch configuration bench.py times (es_ask_eval with the fp32-accurate tcgen05
    MLP, N = 4096, D = 985,216): the oracle's MLP fitness (the definition) of sampled members
    (first, last, both members of a middle pair) within 1e-5; the fp16-image approximation of the
    same members within its model's 1e-4; one tell then moves sampled dims of the mean exactly as
    the oracle's dimension-subset run fed the GPU's fitness."""
    from paper_2212_04180_b200 import strategy as S
    widths = [256, 512, 512, 512, 512, 128]
    cfg = W.CONFIGS["c4"]
    m = O.MLP(widths, 128, 0)
    assert m.D == cfg["D"]
    params = [W.config_params(cfg, 0)]
    es = S.Strategy(W.OPENAI_ES, cfg["N"], cfg["D"], params)
    es.set_mlp_problem(widths, 128, 0)
    _, f16 = es.ask_eval(W.MLP16, write_x=False)
    _, f = es.ask_eval(W.MLP, write_x=False)
    fh, fh16 = f.cpu().numpy()[0], f16.cpu().numpy()[0]
    run = O.Run(W.OPENAI_ES, cfg["N"], cfg["D"], **params[0])
    for j in (0, 2048, 2049, cfg["N"] - 1):
        xo = run.member(j)
        fo = m.evaluate(xo)[0]
        assert abs(float(fh[j]) - float(fo)) <= 1e-5 * abs(float(fo)), (j, fh[j], fo)
        fm = m.evaluate_f16(xo)[0]
        assert abs(float(fh16[j]) - float(fm)) <= 1e-4 * abs(float(fm)), (j, fh16[j], fm)
    dims = np.sort(np.random.default_rng(3).choice(cfg["D"], 64, replace=False))
    sub = O.Run(W.OPENAI_ES, cfg["N"], cfg["D"], dims=dims, **params[0])
    es.tell(f)
    sub.tell(fh)
    got = es.get("mean")[0].cpu().numpy()[dims]
    assert q24(got, sub.mean) <= 1e-5
    es.close()


def _ranks_equal(gpu, r, f_orc):
    s, e, perm = O.rank(f_orc)
    return (np.array_equal(gpu.get("perm")[r].cpu().numpy(), perm) and
            np.array_equal(gpu.get("rank_s")[r].cpu().numpy(), s))


@pytest.mark.parametrize("key", ["c2_sepcma", "c2_snes"])
def test_config2_hundred_generations_sampled_runs(key):
    """SURVEY §8(d) parity protocol at full C2 size (R = 512 runs in the GPU batch): runs 0 and 511
    followed by free-running oracles (each side evaluates its own population) for 100 generations —
    populations bit-exact and ranks identical at every generation, state within 1e-5 after
    generation 1 and 1e-3 after 100."""
    cfg = W.CONFIGS[key]
    R, N, D = cfg["R"], cfg["N"], cfg["D"]
    params = [W.config_params(cfg, r, hyper_vmap=True) for r in range(R)]
    from paper_2212_04180_b200 import strategy as S
    es = S.Strategy(cfg["algo"], N, D, params)
    sample = (0, R - 1)
    orcs = {r: O.Run(cfg["algo"], N, D, **params[r]) for r in sample}
    names = ["mean", "sigma_d", "adam_m", "adam_v", "p_sigma", "p_c", "C", "best_x"]
    for g in range(100):
        x = es.ask()
        f = es.eval(cfg["fn"], x)
        es.tell(f)
        xh = x.cpu().numpy()
        for r, o in orcs.items():
            xo = o.ask()
            assert np.array_equal(bits(xh[r]), bits(xo)), (g, r)
            fo = O.evaluate(cfg["fn"], xo)
            o.tell(fo)
            assert _ranks_equal(es, r, fo), (g, r)
            if g in (0, 99):
                tol = 1e-5 if g == 0 else 1e-3
                for fld in KEPT[cfg["algo"]]:
                    assert q24(es.get(fld)[r].cpu().numpy(), o.vec[names.index(fld)]) <= tol, (g, fld)
    es.close()


def test_config3_hundred_generations():
    """C3 at full size (D = 1e5, N = 256) for 100 free-running generations: populations bit-exact
    and ranks identical every generation, state within 1e-3 at the end."""
    cfg = W.CONFIGS["c3"]
    params = [W.config_params(cfg, 0)]
    pair = Pair(cfg["algo"], cfg["N"], cfg["D"], params)
    o = pair.orc[0]
    for g in range(100):
        x = pair.gpu.ask()
        f = pair.gpu.eval(cfg["fn"], x)
        pair.gpu.tell(f)
        xo = o.ask()
        assert np.array_equal(bits(x[0].cpu().numpy()), bits(xo)), g
        fo = O.evaluate(cfg["fn"], xo)
        o.tell(fo)
        assert _ranks_equal(pair.gpu, 0, fo), g
        if g == 0:
            pair.compare(0, 1e-5)
    pair.compare(0, 1e-3)
    pair.close()


@pytest.mark.parametrize("N,D", [(256, 1000), (1024, 1000), (256, 10_000), (1024, 10_000)])
def test_config5_corner_full(N, D):
    """SURVEY §8(d) C5 corner (N ≤ 1024, D ≤ 1e4), the sweep's exact path: synthetic fitness
    (N15, bit-exact vs the oracle's generator) → rank → tell, compared over the full D for 5
    generations (ranks identical, state ≤ 1e-5 each generation)."""
    cfg = dict(algo=W.OPENAI_ES, init=(-0.04, 0.04))
    params = [W.config_params(cfg, 0)]
    pair = Pair(W.OPENAI_ES, N, D, params)
    o = pair.orc[0]
    for g in range(5):
        f = pair.gpu.synth_fitness()
        fo = O.synth_fitness(params[0]["seed"], o.t, N)
        assert np.array_equal(bits(f[0].cpu().numpy()), bits(fo)), g
        pair.gpu.tell(f)
        o.tell(fo)
        assert _ranks_equal(pair.gpu, 0, fo), g
        pair.compare(0, 1e-5)
    pair.close()
