"""SURVEY §8(f) f1, D-sharded mode: W contexts each owning a quad-aligned dimension range of every
member, exchanging only R·N binary64 partial fitness values (and, for Sep-CMA-ES, R doubles of
‖p_σ'‖²). Emulated on one GPU through the communicator-less split-phase ABI (the sum over ranks is
done here in rank order, exactly what the all-reduce computes); compared with the unsharded
context, which the core parity tests pin to the oracle."""
import numpy as np
import pytest
import torch

import workloads as W
from oracle import oracle as O
from gpu_helpers import KEPT, bits, compare_to_oracle, q24

pytestmark = pytest.mark.gpu

ALGOS = [W.OPENAI_ES, W.PGPE, W.SNES, W.SEP_CMA_ES, W.ARS]


@pytest.fixture(scope="module", autouse=True)
def built():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__
    __graft_entry__.build()
    O.build()


def _params(algo, R, per=None):
    cfg = dict(algo=algo, init=(-2.0, 2.0))
    out = []
    for r in range(R):
        p = W.config_params(cfg, r, seed_offset=7000 + 100 * algo, hyper_vmap=True)
        if per:
            p.update(per[r % len(per)])
        out.append(p)
    return out


def _run(algo, N, D, R, Wn, fn, gens, per=None):
    from paper_2212_04180_b200 import strategy as S
    params = _params(algo, R, per)
    ref = S.Strategy(algo, N, D, params)
    shards = [S.Strategy(algo, N, D, params, shard=(w, Wn), split="dims") for w in range(Wn)]
    # the shards tile [0, D) in quad-aligned ranges
    assert shards[0].d_begin == 0 and all(a.d_begin + a.x_dims == b.d_begin
                                          for a, b in zip(shards, shards[1:]))
    assert shards[-1].d_begin + shards[-1].x_dims == D
    orcs = [O.Run(algo, N, D, **p) for p in params]
    for g in range(gens):
        x, f_ref = ref.ask_eval(fn)
        parts = []
        for sh in shards:
            xs, p = sh.ask_eval_partial(fn, write_x=True)
            d0 = sh.d_begin
            assert torch.equal(xs, x[:, :, d0:d0 + sh.x_dims]), (g, d0)    # bit-exact slices
            parts.append(p)
        fsum = parts[0].clone()
        for p in parts[1:]:
            fsum += p                                                      # rank order
        f = fsum.float()
        # the split sum differs from the unsharded block order only in binary64 rounding
        assert q24(f.cpu().numpy(), f_ref.cpu().numpy()) <= 2 ** -23
        ref.tell(f)
        fh = f.cpu().numpy()
        for r, o in enumerate(orcs):          # the oracle fed the same (summed) fitness
            o.tell(fh[r])
        for sh in shards:
            if algo == W.SEP_CMA_ES:
                sh.tell_local(f)
            else:
                sh.tell(f)
        if algo == W.SEP_CMA_ES:
            n2 = shards[0].get("norm2")
            for sh in shards[1:]:
                n2 = n2 + sh.get("norm2")
            for sh in shards:
                sh.set("norm2", n2)
                sh.tell_apply()
        tol = 1e-6 if algo == W.SEP_CMA_ES else 0.0
        for sh in shards:
            d0, ds = sh.d_begin, sh.state_dims
            for fld in KEPT[algo]:
                a = sh.get(fld).cpu().numpy()
                b = ref.get(fld)[:, d0:d0 + ds].cpu().numpy()
                if tol == 0.0:
                    assert np.array_equal(bits(a), bits(b)), (g, fld, d0)   # halo included
                else:
                    assert q24(a, b) <= tol, (g, fld, d0)
            assert torch.equal(sh.get("perm"), ref.get("perm"))
            for r, o in enumerate(orcs):      # each shard's dims against the oracle's
                compare_to_oracle(sh, algo, r, o, 1e-5, d0=sh.d_begin)
    for es in shards + [ref]:
        es.close()


@pytest.mark.parametrize("algo", ALGOS)
@pytest.mark.parametrize("fn", [W.SPHERE, W.ROSENBROCK, W.RASTRIGIN])
@pytest.mark.parametrize("D,Wn", [(1003, 2), (1000, 4), (37, 3), (9, 2), (4099, 8)])
def test_dshard_matches_unsharded(algo, fn, D, Wn):
    _run(algo, 16, D, 3, Wn, fn, 3)


@pytest.mark.parametrize("algo,per", [
    (W.OPENAI_ES, [dict(shaping=2), dict(optimizer=W.SGD)]),
    (W.PGPE, [dict(elite_ratio=0.25, clip_min=-1.0, clip_max=1.0)]),
    (W.ARS, [dict(elite_ratio=0.3)]),
])
def test_dshard_variants(algo, per):
    _run(algo, 32, 301, 2, 3, W.ROSENBROCK, 3, per)


@pytest.mark.parametrize("algo,per", [
    (W.OPENAI_ES, [dict(optimizer=W.CLIPUP, max_speed=0.05), dict(weight_decay=0.05)]),
    (W.PGPE, [dict(optimizer=W.CLIPUP, max_speed=0.1, momentum=0.5, weight_decay=0.02)]),
    (W.SNES, [dict(weight_decay=0.1), dict()]),
    (W.SEP_CMA_ES, [dict(weight_decay=0.05, clip_max=1.0)]),
    (W.ARS, [dict(weight_decay=0.03, elite_ratio=0.5)]),
])
@pytest.mark.parametrize("D,Wn", [(301, 2), (1003, 3)])
def test_dshard_global_norms(algo, per, D, Wn):
    """f1 × f3: weight decay (‖x_j‖²) and ClipUp (‖g‖, ‖v'‖) on D-sharded contexts,
    whose norms are sums of the ranks' binary64 shares. Split-phase ABI, sums formed here in rank
    order (what the all-reduce computes): es_sqnorm_partial → es_weight_decay_apply →
    es_tell_local → per phase: sum ES_FIELD_NORM2, es_tell_apply. Equal to the unsharded run
    (which applies both itself) up to the binary64 summation order: perm bit-exact, state ≤ 1e-6."""
    from paper_2212_04180_b200 import strategy as S
    N, R, fn = 32, 2, W.RASTRIGIN
    params = _params(algo, R, per)
    ref = S.Strategy(algo, N, D, params)
    shards = [S.Strategy(algo, N, D, params, shard=(w, Wn), split="dims") for w in range(Wn)]
    has_n2 = algo == W.SEP_CMA_ES or any(p.get("optimizer") == W.CLIPUP for p in per)
    for g in range(4):
        x, f_ref = ref.ask_eval(fn)
        parts = [sh.ask_eval_partial(fn)[1] for sh in shards]
        f = sum(parts[1:], parts[0].clone()).float()
        ref.tell(f)                                      # applies weight decay / ClipUp itself
        sq = [sh.sqnorm_partial() for sh in shards]
        sq = sum(sq[1:], sq[0].clone())                  # rank order
        fw = [sh.weight_decay_apply(f, sq) for sh in shards]
        for a in fw[1:]:
            assert torch.equal(a, fw[0])
        for sh, fws in zip(shards, fw):
            sh.tell_local(fws)
        for _ in range(shards[0].tell_apply_phases()):
            if has_n2:
                n2 = [sh.get("norm2") for sh in shards]
                n2 = sum(n2[1:], n2[0].clone())
                for sh in shards:
                    sh.set("norm2", n2)
            for sh in shards:
                sh.tell_apply()
        for sh in shards:
            d0, ds = sh.d_begin, sh.state_dims
            assert torch.equal(sh.get("perm"), ref.get("perm")), g
            for fld in KEPT[algo]:
                a = sh.get(fld).cpu().numpy()
                b = ref.get(fld)[:, d0:d0 + ds].cpu().numpy()
                assert q24(a, b) <= 1e-6, (g, fld, d0)
    for es in shards + [ref]:
        es.close()


def test_dshard_single_rank_equals_plain():
    """W = 1 D-shard: es_ask_eval's partial → fitness path reproduces the plain context bit for bit."""
    from paper_2212_04180_b200 import strategy as S
    params = _params(W.SNES, 2)
    a = S.Strategy(W.SNES, 16, 257, params)
    b = S.Strategy(W.SNES, 16, 257, params, shard=(0, 1), split="dims")
    for _ in range(3):
        xa, fa = a.ask_eval(W.RASTRIGIN)
        xb, fb = b.ask_eval(W.RASTRIGIN)
        assert torch.equal(xa, xb) and torch.equal(fa, fb)
        a.tell(fa)
        b.tell(fb)
    assert torch.equal(a.get("mean"), b.get("mean"))
    a.close()
    b.close()


def test_dshard_rejections():
    from paper_2212_04180_b200 import strategy as S
    from paper_2212_04180_b200._lib import ESError
    p = _params(W.OPENAI_ES, 1)
    with pytest.raises(ESError):                      # ceil(D/4) < W
        S.Strategy(W.OPENAI_ES, 16, 5, p, shard=(0, 3), split="dims")
    wd = S.Strategy(W.OPENAI_ES, 16, 64, _params(W.OPENAI_ES, 1, [dict(weight_decay=0.1)]),
                    shard=(0, 2), split="dims")
    wd.ask_eval_partial(W.SPHERE)
    with pytest.raises(ESError):                      # weight decay needs the ranks' ‖x‖² sum
        wd.tell(torch.zeros(1, 16, device="cuda"))
    with pytest.raises(ESError):
        wd.weight_decay(torch.zeros(1, 16, device="cuda"))
    wd.close()
    sh = S.Strategy(W.OPENAI_ES, 16, 64, p, shard=(0, 2), split="dims")
    with pytest.raises(ESError):                      # no communicator: full fitness impossible
        sh.ask_eval(W.SPHERE)
    sh.close()
