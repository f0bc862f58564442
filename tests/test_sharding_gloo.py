"""World-size-2 CPU test of the population-sharding protocol over torch.distributed
gloo: each rank owns the members and tell entries the PRODUCT's es_shard_plan assigns it, evaluates
only its members, all-gathers fitness in the layout es_tell expects ([W][R][N/W]), reduces its share
of the direction sums (the oracle's range reduction), and all-reduces them. The result must equal the
unsharded computation: fitness exactly, direction sums to binary64 rounding."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, algos, R, D, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import workloads as W
        from oracle import oracle as O
        from paper_2212_04180_b200._lib import lib
        L = lib()
        plan = (C.c_int32 * 4)()
        for algo in algos:
            N = 16 if algo != 3 else 20
            _check_algo(L, O, W, plan, rank, world, algo, R, N, D)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _check_algo(L, O, W, plan, rank, world, algo, R, N, D):
    if True:
        assert L.es_shard_plan(N, N, world, rank, plan) == 0
        m0, m1 = plan[0], plan[1]
        runs = [O.Run(algo, N, D, **W.run_params(algo, 40 + r, init_min=-3, init_max=3))
                for r in range(R)]
        # each rank materialises and evaluates only its own members
        local = np.stack([O.evaluate(W.RASTRIGIN, np.stack([run.member(j) for j in range(m0, m1)]))
                          for run in runs]).astype(np.float32)            # [R][N/W]
        gathered = [torch.empty(R, N // world) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(local))
        fw = torch.stack(gathered).numpy()                                  # [W][R][N/W]
        f_all = fw.transpose(1, 0, 2).reshape(R, N)                         # run-major [R][N]
        for r, run in enumerate(runs):
            full = O.evaluate(W.RASTRIGIN, run.ask())
            assert np.array_equal(f_all[r].view(np.uint32), full.view(np.uint32))
            ne = run.num_entries(f_all[r])
            assert L.es_shard_plan(N, ne, world, rank, plan) == 0
            part = torch.from_numpy(run.reduce_range(f_all[r], plan[2], plan[3]))
            dist.all_reduce(part, op=dist.ReduceOp.SUM)
            ref = run.reduce(f_all[r])
            scale = np.abs(ref).max() + 1e-300
            assert np.abs(part.numpy() - ref).max() <= 1e-12 * scale


def test_two_rank_sharding_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, [0, 1, 2, 3], 2, 37, q))
             for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, "ok"), (1, "ok")], res


def test_shard_plan_partitions():
    import sys
    sys.path.insert(0, ROOT)
    from paper_2212_04180_b200._lib import lib
    L = lib()
    out = (C.c_int32 * 4)()
    for N, W_ in [(16, 2), (4096, 8), (256, 4), (6, 3)]:
        for ne in [0, 1, N // 2, N - 1, N, 7]:
            covered = []
            mem = []
            for r in range(W_):
                assert L.es_shard_plan(N, ne, W_, r, out) == 0
                mem += list(range(out[0], out[1]))
                covered += list(range(out[2], out[3]))
            assert mem == list(range(N)) and covered == list(range(ne))
    assert L.es_shard_plan(10, 4, 3, 0, out) == 1     # N not divisible by W


# ------------------------------------------------------------------ f1 D-sharding over gloo
def _dshard_worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import workloads as W
        from oracle import oracle as O
        from paper_2212_04180_b200._lib import lib
        L = lib()
        N, D = 16, 41
        plan = (C.c_int64 * 3)()
        assert L.es_dshard_plan(D, world, rank, plan) == 0
        d0, d1, s1 = plan[0], plan[1], plan[2]
        for algo in (0, 1, 2):                                   # dims-subset-exact algorithms
            for fn in (W.SPHERE, W.ROSENBROCK):
                p = W.run_params(algo, 90 + algo, init_min=-2, init_max=2)
                full = O.Run(algo, N, D, **p)
                mine = O.Run(algo, N, D, dims=np.arange(d0, s1), **p)   # owned dims + halo
                for _ in range(2):
                    xf, xm = full.ask(), mine.ask()
                    assert np.array_equal(xm.view(np.uint32), xf[:, d0:s1].view(np.uint32))
                    x = xm.astype(np.float64)
                    if fn == W.SPHERE:                           # this rank's terms, binary64
                        part = (x[:, :d1 - d0] ** 2).sum(1)
                    else:
                        a, b = x[:, :-1], x[:, 1:]
                        part = (100 * (b - a * a) ** 2 + (1 - a) ** 2)[:, :min(d1, D - 1) - d0].sum(1)
                    t = torch.from_numpy(np.ascontiguousarray(part))
                    dist.all_reduce(t, op=dist.ReduceOp.SUM)      # the one collective (R·N doubles)
                    f = O.evaluate(fn, xf)
                    assert np.allclose(t.numpy(), f, rtol=1e-6, atol=1e-6)
                    full.tell(f)
                    mine.tell(f)
                    for v in range(mine.vec.shape[0]):           # state slice, bit for bit
                        assert np.array_equal(mine.vec[v].view(np.uint32),
                                              full.vec[v][d0:s1].view(np.uint32)), (algo, v)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_two_rank_dshard_matches_unsharded():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_dshard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(0, "ok"), (1, "ok")], res
