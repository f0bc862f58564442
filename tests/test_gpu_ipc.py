"""SURVEY §8(f) f2 through its real transport: two PROCESSES, each with its own population-shard
context, exchange CUDA IPC handles (es_p2p_ipc_export / es_p2p_ipc_open) over a gloo group and run
the fused peer-memory tell on mapped peer memory. The box has one GPU, so both processes use
cuda:0 (IPC mappings of another process's allocations on the same device). The kernels never
wait on one another: every barrier is host-side (device synchronize + gloo barrier), as the
profiling guide requires for ranks sharing a GPU. Result: each rank's state equals the unsharded
run's (mean / best_x / σ_d / C / σ all-gathered, the rank's own optimizer-state slice)."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch

import workloads as W
from gpu_helpers import q24
from oracle import oracle as O

pytestmark = pytest.mark.gpu

CASES = {
    "openai_es_adam": (W.OPENAI_ES, [dict(), dict(optimizer=W.SGD)]),
    "openai_es_clipup": (W.OPENAI_ES, [dict(optimizer=W.CLIPUP, max_speed=0.05), dict()]),
    "snes": (W.SNES, [dict()]),
    "sep_cma_es": (W.SEP_CMA_ES, [dict(), dict(elite_ratio=0.25)]),
}
N, D, R, GENS, WS = 32, 203, 2, 3, 2


def _params(algo, per):
    out = []
    for r in range(R):
        p = W.config_params(dict(algo=algo, init=(-2.0, 2.0)), r, seed_offset=7000 + 100 * algo)
        p.update(per[r % len(per)])
        out.append(p)
    return out


def _fields(algo):
    return ["mean", "best_x"] + (["sigma_d"] if algo in (W.PGPE, W.SNES) else []) + \
        (["C", "sigma"] if algo == W.SEP_CMA_ES else []) + \
        (["adam_m"] if algo in (W.OPENAI_ES, W.PGPE) else [])


def _worker(rank, port, case, outdir):
    import torch.distributed as dist
    from paper_2212_04180_b200 import strategy as S
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=WS)
    algo, per = CASES[case]
    es = S.Strategy(algo, N, D, _params(algo, per), shard=(rank, WS))
    es.p2p_connect(dist.group.WORLD)                     # CUDA IPC handles over gloo

    def barrier():
        torch.cuda.synchronize()
        dist.barrier()

    for _ in range(GENS):
        f = es.eval(W.RASTRIGIN, es.ask()).cpu()
        parts = [torch.empty_like(f) for _ in range(WS)]
        dist.all_gather(parts, f)
        es.tell_local(torch.stack(parts).contiguous().cuda())
        barrier()                                        # every rank's partial sums exist
        es.tell_p2p_apply()
        barrier()
        for _ in range(es.p2p_finish_phases()):          # Sep-CMA ‖p_σ'‖; ClipUp ‖g‖, ‖v'‖
            es.tell_p2p_finish()
            barrier()
    out = {k: es.get(k).cpu() for k in _fields(algo)}
    out["perm"] = es.get("perm").cpu()
    torch.save(out, os.path.join(outdir, f"rank{rank}.pt"))
    barrier()                                            # peers unmap only after everyone is done
    es.close()
    dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("case", sorted(CASES))
def test_p2p_ipc_two_processes(case):
    import torch.multiprocessing as mp
    from paper_2212_04180_b200 import strategy as S
    algo, per = CASES[case]
    with tempfile.TemporaryDirectory() as td:
        mp.start_processes(_worker, args=(_free_port(), case, td), nprocs=WS, join=True,
                           start_method="spawn")
        res = [torch.load(os.path.join(td, f"rank{w}.pt")) for w in range(WS)]
    ref = S.Strategy(algo, N, D, _params(algo, per))
    orcs = [O.Run(algo, N, D, **p) for p in _params(algo, per)]
    for _ in range(GENS):
        f = ref.eval(W.RASTRIGIN, ref.ask())
        ref.tell(f)
        for r, o in enumerate(orcs):                     # the oracle fed the same fitness
            o.ask()
            o.tell(f[r].cpu().numpy())
    Q = (D + 3) // 4
    for w, got in enumerate(res):
        assert torch.equal(got["perm"], ref.get("perm").cpu()), w
        for k in _fields(algo):
            a, b = got[k].numpy(), ref.get(k).cpu().numpy()
            if k == "adam_m":                            # the rank's own optimizer-state slice
                d0, d1 = 4 * (Q * w // WS), min(D, 4 * (Q * (w + 1) // WS))
                a, b = a[:, d0:d1], b[:, d0:d1]
            if k == "sigma":
                assert np.all(np.abs(a - b) <= 1e-6 * np.abs(b)), (k, w)
            else:
                assert q24(a, b) <= 1e-6, (k, w)
            # and against the oracle (each rank's copy of the all-gathered fields, its own
            # optimizer-state slice)
            vi = {"mean": 0, "sigma_d": 1, "adam_m": 2, "C": 6, "best_x": 7}
            for r, o in enumerate(orcs):
                if k == "sigma":
                    assert abs(float(a[r]) - float(o.sigma)) <= 1e-5 * abs(float(o.sigma)), (k, w)
                    continue
                ob = o.vec[vi[k]]
                ar = a[r]
                if k == "adam_m":
                    ob = ob[d0:d1]
                assert q24(ar, ob) <= 1e-5, (k, w, r)
    ref.close()
