"""GPU parity of the SURVEY §8(f) row f3 variants against the CPU oracle: ARS (Table 1),
z-score fitness shaping, and the SGD-with-momentum / ClipUp optimizers of the
OpenAI-ES / PGPE mean update. Same bar as the core path: populations bit-exact, state within 1e-5
(Q24) after one generation and 1e-3 after 100 (BASELINE.json north_star)."""
import numpy as np
import pytest
import torch

import workloads as W
from oracle import oracle as O
from gpu_helpers import KEPT, Pair, bits, compare_to_oracle, q24

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def built():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build()
    O.build()


def _params(algo, R, per_run=None, **over):
    cfg = dict(algo=algo, init=(-2.0, 2.0))
    out = []
    for r in range(R):
        p = W.config_params(cfg, r, seed_offset=5000 + 100 * algo)
        p.update(over)
        if per_run:
            p.update(per_run[r % len(per_run)])
        out.append(p)
    return out


def _one_gen(pair, fn, tol=1e-5):
    x = pair.gpu.ask()
    f = pair.gpu.eval(fn, x)
    pair.gpu.tell(f)
    xh, fh = x.cpu().numpy(), f.cpu().numpy()
    for r in range(pair.R):
        xo = pair.orc[r].ask()
        assert np.array_equal(bits(xh[r]), bits(xo)), r
        pair.orc[r].tell(fh[r])                                    # teacher-forced
        pair.compare(r, tol)


# ------------------------------------------------------------------------ ARS
ARS_ELITES = [dict(elite_ratio=0.5), dict(elite_ratio=0.1), dict(elite_ratio=1.0),
              dict(elite_ratio=0.26)]


@pytest.mark.parametrize("R,N,D", [(4, 16, 10), (2, 64, 1003), (1, 256, 5000), (4, 2, 1),
                                   (2, 40000, 9)])
@pytest.mark.parametrize("fn", [W.SPHERE, W.RASTRIGIN])
def test_ars_one_generation(R, N, D, fn):
    pair = Pair(W.ARS, N, D, _params(W.ARS, R, ARS_ELITES))
    _one_gen(pair, fn)
    pair.close()


@pytest.mark.parametrize("N", [16, 256, 4096, 40000])
def test_ars_selection_with_ties_and_nan(N):
    """Elite pairs chosen by (key(min(f+, f-)), pair index): with exact ties, ±0 and NaN in the
    fitness the GPU's direction sum over the selected pairs equals the oracle's (binary64, summed in
    a different order: 1e-12 relative)."""
    R, D = 4, 37
    pair = Pair(W.ARS, N, D, _params(W.ARS, R, ARS_ELITES))
    rng = np.random.default_rng(N)
    f = np.stack([W.random_fitness(rng, N, ties=N // 3, nans=min(3, N // 8), infs=0)
                  for _ in range(R)])
    for r in range(R):                 # also whole tied pairs (f+ == f-)
        f[r, 2:6] = f[r, 1]
    pair.gpu.ask()
    pair.gpu.tell_local(torch.from_numpy(f).cuda())
    G = pair.gpu.get("dirsum").cpu().numpy()
    for r in range(R):
        pair.orc[r].ask()
        Go = pair.orc[r].reduce(f[r])
        nan = np.isnan(Go[0])
        assert np.array_equal(np.isnan(G[0, r]), nan), r     # a selected NaN pair poisons both
        assert q24(G[0, r][~nan], Go[0][~nan]) <= 1e-12, r
    pair.gpu.tell_apply()
    pair.close()


def test_ars_constant_fitness_no_step():
    """σ_R = 0 (all selected fitness equal): the oracle takes no step; neither may the GPU."""
    pair = Pair(W.ARS, 16, 33, _params(W.ARS, 2))
    m0 = pair.gpu.get("mean").cpu().numpy()
    pair.gpu.ask()
    pair.gpu.tell(torch.full((2, 16), 3.0, device="cuda"))
    assert np.array_equal(bits(pair.gpu.get("mean").cpu().numpy()), bits(m0))
    for r in range(2):
        pair.orc[r].ask()
        pair.orc[r].tell(np.full(16, 3.0, np.float32))
        pair.compare(r, 0.0)
    pair.close()


# ------------------------------------------------------------------------ z-score shaping
@pytest.mark.parametrize("algo", [W.OPENAI_ES, W.PGPE])
@pytest.mark.parametrize("N", [2, 16, 1000, 40000])
def test_zscore_shaping(algo, N):
    """Shaped values within 2 ulp of the oracle's (the binary64 mean/variance are summed in another
    order, so the rounded float may differ in the last place)."""
    R = 3
    pair = Pair(algo, N, 5, _params(algo, R, shaping=2))
    rng = np.random.default_rng(N + 7)
    f = np.stack([W.random_fitness(rng, N, ties=N // 5 + 1) for _ in range(R)])
    pair.gpu.ask()
    pair.gpu.tell(torch.from_numpy(f).cuda())
    SH = pair.gpu.get("shaped").cpu().numpy()
    for r in range(R):
        ref = O.zscore(f[r])
        ulp = np.spacing(np.maximum(np.abs(ref), np.float32(1e-30))).astype(np.float64)
        assert (np.abs(SH[r].astype(np.float64) - ref) / ulp).max() <= 2.0, r
    pair.close()


@pytest.mark.parametrize("algo", [W.OPENAI_ES, W.PGPE])
@pytest.mark.parametrize("R,N,D", [(3, 16, 10), (2, 64, 1003), (1, 256, 5000)])
def test_zscore_one_generation(algo, R, N, D):
    pair = Pair(algo, N, D, _params(algo, R, shaping=2))
    _one_gen(pair, W.RASTRIGIN)
    pair.close()


# ------------------------------------------------------------------------ SGD / ClipUp
# Per-run optimizer mix inside one batch (vmap over hyperparameters): Adam, SGD, ClipUp
# unclipped, ClipUp clipped (max_speed below lr so the velocity norm limit binds).
OPT_MIX = [dict(optimizer=W.SGD, momentum=0.9), dict(optimizer=W.CLIPUP, max_speed=0.02),
           dict(optimizer=W.ADAM), dict(optimizer=W.CLIPUP, max_speed=0.004, momentum=0.5),
           dict(optimizer=W.SGD, momentum=0.0)]


@pytest.mark.parametrize("algo", [W.OPENAI_ES, W.PGPE])
@pytest.mark.parametrize("R,N,D", [(5, 16, 10), (5, 64, 1003), (2, 256, 5000), (5, 2, 1),
                                   (3, 32, 70001)])
def test_optimizers_one_generation(algo, R, N, D):
    pair = Pair(algo, N, D, _params(algo, R, OPT_MIX))
    _one_gen(pair, W.SPHERE)
    pair.close()


# ------------------------------------------------------------------------ 100 generations
@pytest.mark.parametrize("algo,fn,N,D,R,over", [
    (W.ARS, W.SPHERE, 16, 10, 4, None),
    (W.ARS, W.RASTRIGIN, 64, 100, 2, None),
    (W.OPENAI_ES, W.SPHERE, 32, 100, 5, "opt"),
    (W.PGPE, W.ROSENBROCK, 32, 200, 5, "opt"),
    (W.OPENAI_ES, W.RASTRIGIN, 32, 100, 2, "z"),
])
def test_variants_hundred_generations(algo, fn, N, D, R, over):
    per = ARS_ELITES if algo == W.ARS else (OPT_MIX if over == "opt" else None)
    extra = dict(shaping=2) if over == "z" else {}
    pair = Pair(algo, N, D, _params(algo, R, per, **extra))
    for g in range(100):
        pair.gpu.tell(pair.gpu.eval(fn, pair.gpu.ask()))
        for r in range(R):
            o = pair.orc[r]
            o.tell(O.evaluate(fn, o.ask()))
        if g == 0:
            for r in range(R):
                pair.compare(r, 1e-5)
    for r in range(R):
        pair.compare(r, 1e-3)
    pair.close()


# ------------------------------------------------------------------------ sharded (split phase)
@pytest.mark.parametrize("algo,per", [(W.ARS, ARS_ELITES), (W.OPENAI_ES, OPT_MIX),
                                      (W.PGPE, OPT_MIX)])
@pytest.mark.parametrize("Wn", [2, 4])
def test_variants_emulated_shards(algo, per, Wn):
    """As test_gpu_parity.test_emulated_shards_match_single_gpu: ARS's k selected directions and
    ClipUp's global norms split over W shards reproduce the unsharded run, and every shard's state
    is within 1e-5 of the oracle fed the same fitness."""
    from paper_2212_04180_b200 import strategy as S
    N, D, R = 32, 301, 4
    params = _params(algo, R, per)
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
            o.ask()
            o.tell(fh[r])
        locs = []
        for w, sh in enumerate(shards):
            xs = sh.ask()
            assert torch.equal(xs, x[:, w * nl:(w + 1) * nl]), (gen, w)
            locs.append(sh.eval(W.RASTRIGIN, xs))
        gathered = torch.stack(locs).contiguous()
        for sh in shards:
            sh.tell_local(gathered)
        total = shards[0].get("dirsum")
        for sh in shards[1:]:
            total = total + sh.get("dirsum")
        for sh in shards:
            sh.set("dirsum", total)
            sh.tell_apply()
        for sh in shards:
            for fld in KEPT[algo]:
                assert q24(sh.get(fld).cpu().numpy(), ref.get(fld).cpu().numpy()) <= 1e-6, fld
            for r, o in enumerate(orcs):
                compare_to_oracle(sh, algo, r, o, 1e-5)
    for es in shards + [ref]:
        es.close()


# ------------------------------------------------------------------------ argument checks
@pytest.mark.parametrize("algo,over", [
    (W.SNES, dict(optimizer=W.SGD)), (W.SEP_CMA_ES, dict(optimizer=W.CLIPUP)),
    (W.ARS, dict(optimizer=W.SGD)), (W.OPENAI_ES, dict(optimizer=3)),
    (W.OPENAI_ES, dict(optimizer=W.CLIPUP, max_speed=0.0)), (W.ARS, dict(shaping=2)),
    (W.SNES, dict(shaping=2)), (W.ARS, dict(elite_ratio=0.0)), (W.PGPE, dict(shaping=3)),
    (W.PGPE, dict(elite_ratio=0.0)), (W.PGPE, dict(elite_ratio=1.5)),
    (W.SNES, dict(weight_decay=-0.1)), (W.OPENAI_ES, dict(clip_min=1.0, clip_max=0.0)),
    (W.SEP_CMA_ES, dict(clip_min=float("nan"))),
])
def test_variant_argument_errors(algo, over):
    from paper_2212_04180_b200 import strategy as S
    from paper_2212_04180_b200._lib import ESError
    with pytest.raises(ESError):
        S.Strategy(algo, 16, 8, _params(algo, 1, **over))


def test_ars_odd_popsize_rejected():
    from paper_2212_04180_b200 import strategy as S
    from paper_2212_04180_b200._lib import ESError
    with pytest.raises(ESError):
        S.Strategy(W.ARS, 15, 8, _params(W.ARS, 1))


# ------------------------------------------------------------------------ PGPE elite pairs (Q13b)
PGPE_ELITES = [dict(elite_ratio=0.25), dict(elite_ratio=1.0), dict(elite_ratio=0.1),
               dict(elite_ratio=0.6)]


@pytest.mark.parametrize("R,N,D", [(4, 16, 10), (4, 64, 1003), (1, 256, 5000), (4, 2, 1),
                                   (2, 40000, 9)])
def test_pgpe_elite_one_generation(R, N, D):
    pair = Pair(W.PGPE, N, D, _params(W.PGPE, R, PGPE_ELITES))
    _one_gen(pair, W.RASTRIGIN)
    pair.close()


# ------------------------------------------------------------------------ weight decay
WDS = [dict(weight_decay=0.05), dict(weight_decay=0.0), dict(weight_decay=0.7)]


@pytest.mark.parametrize("algo", [W.OPENAI_ES, W.PGPE, W.SNES, W.SEP_CMA_ES, W.ARS])
@pytest.mark.parametrize("R,N,D", [(3, 16, 10), (3, 64, 1003), (1, 32, 70001)])
def test_weight_decay_one_generation(algo, R, N, D):
    pair = Pair(algo, N, D, _params(algo, R, WDS))
    x = pair.gpu.ask()
    f = pair.gpu.eval(W.RASTRIGIN, x)
    fw = pair.gpu.weight_decay(f).cpu().numpy()
    pair.gpu.tell(f)
    fh = f.cpu().numpy()
    for r in range(R):
        o = pair.orc[r]
        o.ask()
        ref = o.weight_decay(fh[r])
        assert np.all(np.abs(fw[r].astype(np.float64) - ref) <= np.spacing(np.abs(ref))), r
        if WDS[r % 3]["weight_decay"] == 0.0:
            assert np.array_equal(bits(fw[r]), bits(fh[r]))
        o.tell(fh[r])
        pair.compare(r, 1e-5)
    pair.close()


def test_weight_decay_host_buffers():
    pair = Pair(W.OPENAI_ES, 16, 33, _params(W.OPENAI_ES, 2, WDS))
    x = pair.gpu.ask()
    f = pair.gpu.eval(W.SPHERE, x)
    dev = pair.gpu.weight_decay(f).cpu()
    host = pair.gpu.weight_decay(f.cpu())
    assert torch.equal(dev, host)
    pair.gpu.tell(f)
    pair.close()


# ------------------------------------------------------------------------ box bounds
BOXES = [dict(clip_min=-0.5, clip_max=0.3), dict(), dict(clip_min=0.0),
         dict(clip_max=-0.25)]


@pytest.mark.parametrize("algo", [W.OPENAI_ES, W.PGPE, W.SNES, W.SEP_CMA_ES, W.ARS])
@pytest.mark.parametrize("R,N,D", [(4, 16, 10), (4, 64, 1003), (1, 32, 4099)])
def test_box_bounds_one_generation(algo, R, N, D):
    pair = Pair(algo, N, D, _params(algo, R, BOXES))
    _one_gen(pair, W.SPHERE)                      # x bit-exact (clipped) and state incl. best_x
    pair.close()


@pytest.mark.parametrize("algo", [W.OPENAI_ES, W.SNES])
@pytest.mark.parametrize("fn", [W.SPHERE, W.ROSENBROCK, W.RASTRIGIN])
def test_box_bounds_fused_ask_eval(algo, fn):
    """The fused ask+eval kernel evaluates the clipped members (Rosenbrock's cross-quad successor
    included)."""
    N, D, R = 16, 1003, 4
    pair = Pair(algo, N, D, _params(algo, R, BOXES))
    x, f = pair.gpu.ask_eval(fn, write_x=True)
    xh, fh = x.cpu().numpy(), f.cpu().numpy()
    for r in range(R):
        xo = pair.orc[r].ask()
        assert np.array_equal(bits(xh[r]), bits(xo))
        assert q24(fh[r], O.evaluate(fn, xo)) <= 1e-5
    pair.close()


# ------------------------------------------------------------------------ combined, 100 generations
@pytest.mark.parametrize("algo,per", [
    (W.PGPE, [dict(elite_ratio=0.25, weight_decay=0.01, clip_min=-1.0, clip_max=1.5),
              dict(elite_ratio=1.0, optimizer=W.CLIPUP, max_speed=0.05)]),
    (W.ARS, [dict(weight_decay=0.02, clip_min=-1.0), dict(elite_ratio=0.3)]),
    (W.SEP_CMA_ES, [dict(weight_decay=0.1, clip_max=1.0), dict()]),
])
def test_f3_combined_hundred_generations(algo, per):
    N, D, R = 32, 100, 2
    pair = Pair(algo, N, D, _params(algo, R, per))
    for g in range(100):
        pair.gpu.tell(pair.gpu.eval(W.RASTRIGIN, pair.gpu.ask()))
        for r in range(R):
            o = pair.orc[r]
            o.tell(O.evaluate(W.RASTRIGIN, o.ask()))
        if g == 0:
            for r in range(R):
                pair.compare(r, 1e-5)
    for r in range(R):
        pair.compare(r, 1e-3)
    pair.close()


@pytest.mark.parametrize("algo", [W.PGPE, W.SNES])
def test_weight_decay_emulated_shards(algo):
    """Split-phase tell with weight decay: each shard decays its own slice before the gather."""
    from paper_2212_04180_b200 import strategy as S
    N, D, R, Wn = 32, 301, 3, 2
    per = [dict(weight_decay=0.05, elite_ratio=0.5), dict(weight_decay=0.0),
           dict(weight_decay=0.3, clip_min=-0.5)]
    params = _params(algo, R, per)
    ref = S.Strategy(algo, N, D, params)
    shards = [S.Strategy(algo, N, D, params, shard=(w, Wn)) for w in range(Wn)]
    for gen in range(3):
        ref.tell(ref.eval(W.RASTRIGIN, ref.ask()))
        locs = []
        for sh in shards:
            xs = sh.ask()
            locs.append(sh.weight_decay(sh.eval(W.RASTRIGIN, xs)))
        gathered = torch.stack(locs).contiguous()
        for sh in shards:
            sh.tell_local(gathered)
        total = shards[0].get("dirsum") + shards[1].get("dirsum")
        for sh in shards:
            sh.set("dirsum", total)
            sh.tell_apply()
        for sh in shards:
            assert torch.equal(sh.get("perm"), ref.get("perm"))
            for fld in KEPT[algo]:
                assert q24(sh.get(fld).cpu().numpy(), ref.get(fld).cpu().numpy()) <= 1e-6, fld
    for es in shards + [ref]:
        es.close()


# ------------------------------------------------------------------------ f2 peer-memory tell
@pytest.mark.parametrize("algo,per", [(W.OPENAI_ES, [dict(), dict(optimizer=W.SGD)]),
                                      (W.OPENAI_ES, [dict(optimizer=W.CLIPUP, max_speed=0.05),
                                                     dict(), dict(optimizer=W.CLIPUP, max_speed=50.0)]),
                                      (W.PGPE, [dict(), dict(elite_ratio=0.5)]),
                                      (W.PGPE, [dict(optimizer=W.CLIPUP, max_speed=0.1,
                                                     momentum=0.5)]),
                                      (W.SNES, [dict()]), (W.ARS, ARS_ELITES),
                                      (W.SEP_CMA_ES, [dict(), dict(elite_ratio=0.25)])])
@pytest.mark.parametrize("Wn,D", [(2, 301), (4, 1003), (8, 4099), (3, 37)])
def test_p2p_fused_tell_matches_unsharded(algo, per, Wn, D):
    """W ranks emulated on one GPU, each running the SAME fused kernel it would
    run on its own GPU (peer pointers here are plain device pointers): after tell_local on every
    rank, tell_p2p_apply on each reads the W partial sums of its slice, updates it and writes the
    slice into every peer. Populations bit-identical to the unsharded run; mean / best_x / σ_d
    (all-gathered) on every rank and the owned optimizer-state slices within 1e-6."""
    from paper_2212_04180_b200 import strategy as S
    N, R = 48, 3                              # N/W even for W = 2, 3, 4, 8
    params = _params(algo, R, per)
    ref = S.Strategy(algo, N, D, params)
    shards = [S.Strategy(algo, N, D, params, shard=(w, Wn)) for w in range(Wn)]
    peers = [sh.p2p_export() for sh in shards]
    for sh in shards:
        sh.p2p_set_peers(peers)
    nl = N // Wn
    Q = (D + 3) // 4
    for gen in range(4):
        x = ref.ask()
        f = ref.eval(W.RASTRIGIN, x)
        ref.tell(f)
        locs = []
        for w, sh in enumerate(shards):
            xs = sh.ask()
            assert torch.equal(xs, x[:, w * nl:(w + 1) * nl]), (gen, w)
            locs.append(sh.eval(W.RASTRIGIN, xs))
        gathered = torch.stack(locs).contiguous()
        for sh in shards:
            sh.tell_local(gathered)
        for sh in shards:                      # after every rank's partial sums exist
            sh.tell_p2p_apply()
        for _ in range(shards[0].p2p_finish_phases()):   # Sep-CMA ‖p_σ'‖; ClipUp ‖g‖, ‖v'‖
            for sh in shards:                  # (a barrier between phases)
                sh.tell_p2p_finish()
        for w, sh in enumerate(shards):
            assert torch.equal(sh.get("perm"), ref.get("perm"))
            fields = ["mean", "best_x"] + (["sigma_d"] if algo in (W.PGPE, W.SNES) else []) + \
                (["C"] if algo == W.SEP_CMA_ES else [])
            if algo == W.SEP_CMA_ES:
                assert abs(float(sh.get("sigma")[0]) - float(ref.get("sigma")[0])) <= \
                    1e-6 * float(ref.get("sigma")[0])
            for fld in fields:
                assert q24(sh.get(fld).cpu().numpy(), ref.get(fld).cpu().numpy()) <= 1e-6, (fld, w)
            if algo in (W.OPENAI_ES, W.PGPE):   # the rank's own optimizer-state slice
                d0, d1 = 4 * (Q * w // Wn), min(D, 4 * (Q * (w + 1) // Wn))
                a = sh.get("adam_m")[:, d0:d1].cpu().numpy()
                b = ref.get("adam_m")[:, d0:d1].cpu().numpy()
                assert q24(a, b) <= 1e-6, w
    for es in shards + [ref]:
        es.close()


def test_p2p_rejections():
    from paper_2212_04180_b200 import strategy as S
    from paper_2212_04180_b200._lib import ESError
    a = [S.Strategy(W.OPENAI_ES, 16, 8, _params(W.OPENAI_ES, 1, optimizer=W.CLIPUP, max_speed=1.0),
                    shard=(w, 2)) for w in range(2)]
    a[0].p2p_set_peers([s.p2p_export() for s in a])
    assert a[0].p2p_finish_phases() == 2
    with pytest.raises(ESError):                          # no apply pending
        a[0].tell_p2p_finish()
    b = [S.Strategy(W.OPENAI_ES, 16, 8, _params(W.OPENAI_ES, 1), shard=(w, 2)) for w in range(2)]
    with pytest.raises(ESError):
        b[0].p2p_set_peers([b[0].p2p_export()])           # wrong world size
    b[0].ask()
    b[0].tell_local(torch.zeros(2, 1, 8, device="cuda"))
    with pytest.raises(ESError):
        b[0].tell_p2p_apply()                             # peers not set
    for s in a + b:
        s.close()


# ------------------------------------------------------------------------ f2 NVLS (multicast)
@pytest.mark.parametrize("algo", [W.OPENAI_ES, W.PGPE, W.SNES, W.ARS])
def test_nvls_tell_single_rank(algo):
    """The NVLS path on the one GPU available: a one-device multicast team. The fused kernel's
    multimem.ld_reduce then returns this rank's sums and multimem.st writes back through the
    switch alias — exercising the object lifecycle (VMM, bind, multicast mapping), the PTX and the
    buffer relocation; the result must equal the ordinary tell bit for bit."""
    from paper_2212_04180_b200 import strategy as S
    from paper_2212_04180_b200._lib import ESError
    N, D, R = 32, 1003, 3
    params = _params(algo, R)
    ref = S.Strategy(algo, N, D, params)
    es = S.Strategy(algo, N, D, params)
    try:
        es.nvls_open(True)
    except ESError as e:
        pytest.skip(f"no multicast on this box: {e}")
    es.nvls_bind()
    for gen in range(3):
        x = ref.ask()
        f = ref.eval(W.RASTRIGIN, x)
        ref.tell(f)
        assert torch.equal(es.ask(), x)
        es.tell_local(f)
        es.tell_nvls_apply()
        for fld in KEPT[algo]:
            assert torch.equal(es.get(fld), ref.get(fld)), (gen, fld)
    es.close()
    ref.close()
