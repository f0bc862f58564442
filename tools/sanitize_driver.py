"""Small run of every kernel family (all five diagonal strategies × 3 fitness functions × bounds /
weight decay, fused ask+eval, SGD / ClipUp, shared-memory and global sorts, peer-memory tell incl.
Sep-CMA and ClipUp phases, D-sharding, tcgen05 MLP, full CMA-ES on the tensor-core and SIMT
paths), with ragged sizes so the tails and masks run. Meant for compute-sanitizer
(`compute-sanitizer --tool memcheck python tools/sanitize_driver.py`); the GPU pool has it closed
(r18: "runs under it have left GPUs needing a reset"), so it serves as an all-kernel smoke, and
with ES_GUARD_ALLOCS=1 as an out-of-bounds-write check: every context's 256-B guard zones around
its allocations are verified before it is closed (tests/test_gpu_guards.py)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import workloads as W  # noqa: E402
from paper_2212_04180_b200 import strategy as S  # noqa: E402


GUARD = os.environ.get("ES_GUARD_ALLOCS") == "1"


def done(*ess):
    for es in ess:
        if GUARD:
            bad = es.check_guards()
            assert bad == 0, f"{bad} guard bytes overwritten (algo {es.algo}, D {es.num_dims})"
        es.close()


def params(algo, R, **over):
    out = []
    for r in range(R):
        p = W.run_params(algo, 11 + r, init_min=-2.0, init_max=2.0)
        p.update(over)
        out.append(p)
    return out


def diagonal_family():
    for algo in (W.OPENAI_ES, W.PGPE, W.SNES, W.SEP_CMA_ES, W.ARS):
        for D in (37, 64):
            for over in (dict(), dict(weight_decay=0.05, clip_min=-1.5, clip_max=1.5)):
                es = S.Strategy(algo, 24, D, params(algo, 2, **over))
                for fn in (W.SPHERE, W.ROSENBROCK, W.RASTRIGIN):
                    es.tell(es.eval(fn, es.ask()))
                x, f = es.ask_eval(W.RASTRIGIN)
                es.tell(f)
                done(es)
    for opt in (W.SGD, W.CLIPUP):
        es = S.Strategy(W.OPENAI_ES, 16, 37, params(W.OPENAI_ES, 2, optimizer=opt, max_speed=0.1))
        for _ in range(2):
            es.tell(es.eval(W.SPHERE, es.ask()))
        done(es)


def big_rank():
    es = S.Strategy(W.OPENAI_ES, 16384, 4, params(W.OPENAI_ES, 1))      # shared-memory sort
    es.tell(es.eval(W.SPHERE, es.ask()))
    done(es)
    es = S.Strategy(W.SNES, 20000, 4, params(W.SNES, 1))                 # global hybrid sort
    es.tell(es.eval(W.SPHERE, es.ask()))
    done(es)


def shards():
    N, D, R, Wn = 24, 61, 2, 2
    for algo, over in ((W.PGPE, dict()), (W.SEP_CMA_ES, dict()),
                       (W.OPENAI_ES, dict(optimizer=W.CLIPUP, max_speed=0.05))):
        sh = [S.Strategy(algo, N, D, params(algo, R, **over), shard=(w, Wn)) for w in range(Wn)]
        peers = [s.p2p_export() for s in sh]
        for s in sh:
            s.p2p_set_peers(peers)
        for _ in range(2):
            g = torch.stack([s.eval(W.RASTRIGIN, s.ask()) for s in sh]).contiguous()
            for s in sh:
                s.tell_local(g)
            for s in sh:
                s.tell_p2p_apply()
            for _ in range(sh[0].p2p_finish_phases()):
                for s in sh:
                    s.tell_p2p_finish()
        done(*sh)
    for algo in (W.SNES, W.SEP_CMA_ES):
        sh = [S.Strategy(algo, N, D, params(algo, R), shard=(w, Wn), split="dims")
              for w in range(Wn)]
        for _ in range(2):
            parts = [s.ask_eval_partial(W.ROSENBROCK, write_x=True)[1] for s in sh]
            f = (parts[0] + parts[1]).float()
            for s in sh:
                s.tell_local(f) if algo == W.SEP_CMA_ES else s.tell(f)
            if algo == W.SEP_CMA_ES:
                n2 = sh[0].get("norm2") + sh[1].get("norm2")
                for s in sh:
                    s.set("norm2", n2)
                    s.tell_apply()
        done(*sh)


def mlp():
    import ctypes as C
    from paper_2212_04180_b200._lib import lib
    widths = [32, 64, 64, 16]
    D = int(lib().es_mlp_num_params((C.c_int32 * len(widths))(*widths), len(widths)))
    es = S.Strategy(W.OPENAI_ES, 16, D, params(W.OPENAI_ES, 1, init_min=-0.05, init_max=0.05))
    es.set_mlp_problem(widths, 128, 3)
    es.tell(es.eval(W.MLP, es.ask()))
    x, f = es.ask_eval(W.MLP)
    es.tell(f)
    es.tell(es.eval(W.MLP16, es.ask()))
    x, f = es.ask_eval(W.MLP16)
    es.tell(f)
    _, f = es.ask_eval(W.MLP, write_x=False)
    es.tell(f)
    done(es)


def cma():
    for D in (64, 130, 37):            # tensor-core path (D % 4 == 0) and the SIMT fallback
        es = S.Strategy(5, 16, D, params(W.SEP_CMA_ES, 2, sigma_init=0.3))
        for _ in range(3):
            es.tell(es.eval(W.ROSENBROCK, es.ask()))
        done(es)


if __name__ == "__main__":
    for part in (sys.argv[1:] or ["diagonal_family", "big_rank", "shards", "mlp", "cma"]):
        globals()[part]()
        torch.cuda.synchronize()
        print("ok", part, flush=True)
