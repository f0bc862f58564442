"""CPU checks of the C ABI: the library loads, exports every symbol include/es.h declares, the
host-only entry points work, and argument validation rejects bad input before touching a GPU."""
import ctypes as C
import json
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    import __graft_entry__
    __graft_entry__.build()
    from paper_2212_04180_b200 import _lib
    return _lib.lib()


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "es.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(es_[a-z0-9_]+)\s*\(", src)))


def test_exports_every_declared_symbol(L):
    syms = declared_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    from paper_2212_04180_b200 import _lib
    assert sorted(_lib.EXPORTS) == syms


def test_mlp_param_count_golden(L):
    g = json.load(open(os.path.join(ROOT, "tests", "golden", "spec_examples.json")))
    for ex in g["mlp_param_count"]:
        w = (C.c_int32 * len(ex["widths"]))(*ex["widths"])
        assert L.es_mlp_num_params(w, len(ex["widths"])) == ex["count"]     # P:270 → 6248
    w = (C.c_int32 * 6)(256, 512, 512, 512, 512, 128)
    assert L.es_mlp_num_params(w, 6) == 985_216                              # config 4 (Q21)


def test_status_strings_and_nccl_id(L):
    assert L.es_status_string(0) == b"success"
    assert L.es_status_string(1) == b"invalid argument"
    assert L.es_nccl_unique_id_size() == 128


def _init(L, algo=0, R=1, N=16, D=10, W=1, rank=0, **over):
    from paper_2212_04180_b200._lib import RunParams
    import workloads as Wl
    arr = (RunParams * R)()
    for r in range(R):
        p = Wl.run_params(algo if algo in Wl.ANT else 0, r, **over)
        for k, v in p.items():
            setattr(arr[r], k, v)
    ctx = C.c_void_p()
    uid = (C.c_uint8 * 128)() if W > 1 else None
    rc = L.es_init(C.byref(ctx), algo, R, N, D, arr, rank, W, uid, None)
    return rc, ctx


@pytest.mark.parametrize("kw", [dict(N=15), dict(N=1), dict(D=0), dict(R=0),
                                dict(N=16, W=3, rank=0), dict(N=12, W=4, rank=1),
                                dict(algo=3, N=16, elite_ratio=0.01), dict(sigma_init=-1.0),
                                dict(lrate_init=0.0), dict(algo=2, shaping=1), dict(rank=2, W=2),
                                dict(algo=7)])
def test_invalid_arguments_rejected(L, kw):
    rc, ctx = _init(L, **kw)
    assert rc == 1, (kw, L.es_last_error(None))
    assert not ctx.value


def test_unsupported_popsize(L):
    rc, _ = _init(L, N=1 << 21)
    assert rc == 6


def test_null_arguments(L):
    assert L.es_ask(None, None, None) == 1
    assert L.es_tell(None, None, None) == 1
    assert L.es_eval_bbob(None, 0, None, 1, 1, None, None) == 1
    assert L.es_eval_bbob(None, 9, C.c_void_p(8), 1, 1, C.c_void_p(8), None) == 1
    assert L.es_debug_primitive(7, None, None, 1, None) == 1
    assert L.es_destroy(None) == 0


def test_product_has_no_oracle_dependency():
    """The product package must not import, include, link or execute anything under oracle/."""
    pkg = os.path.join(ROOT, "paper_2212_04180_b200")
    bad = re.compile(r"(import\s+oracle|from\s+oracle|es_oracle|libes_oracle|oracle\.py|orc_)")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not bad.search(txt), f


def test_dshard_plan_tiles_quad_aligned():
    """f1 D-sharding plan (host-only): ranges tile [0, D), start on quads, halo = next dim."""
    import ctypes as C
    from paper_2212_04180_b200 import _lib
    L = _lib.lib()
    for D in (1, 4, 5, 37, 1000, 1003, 100_000, 985_216):
        for W in (1, 2, 3, 4, 8):
            if (D + 3) // 4 < W:                      # some rank would own no dims
                out = (C.c_int64 * 3)()
                assert any(L.es_dshard_plan(D, W, r, out) != 0 for r in range(W))
                continue
            prev = 0
            for r in range(W):
                out = (C.c_int64 * 3)()
                assert L.es_dshard_plan(D, W, r, out) == 0
                d0, d1, s1 = out[0], out[1], out[2]
                assert d0 == prev and d0 % 4 == 0 and d1 > d0 and s1 == min(d1 + 1, D)
                prev = d1
            assert prev == D
