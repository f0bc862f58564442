"""Python mirror of Listing 1: Strategy(...).ask() → eval → .tell(fitness).

Thin marshalling over include/es.h. torch is used for device memory and streams only; buffers are
handed to the library by data_ptr(). Population sharding uses a torch.distributed process
group to broadcast the ncclUniqueId; the collectives themselves run inside es_tell.
"""
from __future__ import annotations

import ctypes as C
import math

import torch

from . import _lib
from ._lib import FIELDS, RunParams, check, lib

DEFAULT_PARAMS = dict(init_min=-1.0, init_max=1.0, sigma_init=0.05, sigma_decay=1.0,
                      sigma_limit=0.0, lrate_init=0.01, lrate_decay=1.0, lrate_limit=0.0,
                      beta1=0.9, beta2=0.999, eps=1e-8, sigma_lrate=0.2, sigma_max_change=0.2,
                      temperature=12.0, elite_ratio=0.5, shaping=0, optimizer=0,
                      momentum=0.9, max_speed=0.02, weight_decay=0.0, clip_min=-math.inf,
                      clip_max=math.inf)
PGPE_ELITE_DEFAULT = 1.0    # DESIGN Q13: every pair unless elite_ratio is given


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def eval_bbob(fn, x, out=None, stream=None, ctx=None):
    """Batched BBOB fitness of the rows of x (float32 [n, D], CUDA) → float32 [n]."""
    assert x.is_cuda and x.dtype == torch.float32 and x.is_contiguous()
    n, D = x.shape
    f = out if out is not None else torch.empty(n, dtype=torch.float32, device=x.device)
    check(lib().es_eval_bbob(ctx, int(fn), _ptr(x), n, D, _ptr(f), _stream(stream)), ctx)
    return f


class Strategy:
    """R independent runs of one algorithm (vmap over seeds / hyperparameters)."""

    def __init__(self, algo, popsize, num_dims, params, device="cuda", group=None, stream=None,
                 shard=None, split="population", single_comm=False):
        """params: one dict per run (es_run_params_t fields; 'seed' required).
        group: torch.distributed group for sharding with NCCL inside the library.
        shard: (rank, world_size) for a communicator-less shard (split-phase exchange).
        split: "population" (es_init) or "dims" (f1 D-sharding, es_init_dshard).
        single_comm: without a group, give the context a ONE-rank NCCL communicator so es_tell
        runs the population-sharded data plane (all-gather, all-reduce, separate update) on one
        GPU."""
        if isinstance(params, dict):
            params = [params]
        self.algo, self.popsize, self.num_dims = int(algo), int(popsize), int(num_dims)
        self.R = len(params)
        self.device = torch.device(device)
        arr = (RunParams * self.R)()
        for r, p in enumerate(params):
            kw = dict(DEFAULT_PARAMS)
            if self.algo == 1:                                   # PGPE
                kw["elite_ratio"] = PGPE_ELITE_DEFAULT
            kw.update(p)
            for k, v in kw.items():
                setattr(arr[r], k, v)
        self.world_size, self.rank, uid = 1, 0, None
        if group is not None and torch.distributed.get_world_size(group) > 1:
            self.world_size = torch.distributed.get_world_size(group)
            self.rank = torch.distributed.get_rank(group)
            n = lib().es_nccl_unique_id_size()
            buf = torch.zeros(n, dtype=torch.uint8)
            if self.rank == 0:
                check(lib().es_nccl_get_unique_id(C.c_void_p(buf.data_ptr())))
            bbuf = buf.to(self.device) if torch.distributed.get_backend(group) == "nccl" else buf
            torch.distributed.broadcast(bbuf, src=torch.distributed.get_global_rank(group, 0),
                                        group=group)
            buf = bbuf.cpu()
            self._uid = buf
            uid = C.c_void_p(buf.data_ptr())
        elif single_comm:
            n = lib().es_nccl_unique_id_size()
            buf = torch.zeros(n, dtype=torch.uint8)
            check(lib().es_nccl_get_unique_id(C.c_void_p(buf.data_ptr())))
            self._uid = buf
            uid = C.c_void_p(buf.data_ptr())
        if shard is not None:
            self.rank, self.world_size = int(shard[0]), int(shard[1])
        self.split = split
        self.ctx = C.c_void_p()
        init = lib().es_init_dshard if split == "dims" else lib().es_init
        with torch.cuda.device(self.device):
            check(init(C.byref(self.ctx), self.algo, self.R, self.popsize, self.num_dims,
                       arr, self.rank, self.world_size, uid, _stream(stream)))
        self.local_popsize = self.popsize // self.world_size
        self.x_dims = self.state_dims = self.num_dims
        self.d_begin = 0
        if split == "dims":
            info = (C.c_int64 * 4)()
            check(lib().es_dshard_info(self.ctx, info), self.ctx)
            self.d_begin, d_end, s_end = info[0], info[1], info[2]
            self.x_dims, self.state_dims = d_end - self.d_begin, s_end - self.d_begin
            self.local_popsize = self.popsize

    # -- Listing 1 ------------------------------------------------------------------------------
    def ask(self, out=None, stream=None):
        x = out if out is not None else torch.empty(
            (self.R, self.local_popsize, self.x_dims), dtype=torch.float32, device=self.device)
        check(lib().es_ask(self.ctx, _ptr(x), _stream(stream)), self.ctx)
        return x

    def ask_eval(self, fn, out_x=None, out_f=None, write_x=True, stream=None):
        """Fused ask + BBOB evaluate (§8(f) f1). write_x=False never materialises x."""
        x = None
        if write_x:
            x = out_x if out_x is not None else torch.empty(
                (self.R, self.local_popsize, self.x_dims), dtype=torch.float32,
                device=self.device)
        f = out_f if out_f is not None else torch.empty(
            (self.R, self.local_popsize), dtype=torch.float32, device=self.device)
        check(lib().es_ask_eval(self.ctx, int(fn), _ptr(x) if x is not None else None, _ptr(f),
                                _stream(stream)), self.ctx)
        return x, f

    def eval(self, fn, x, out=None, stream=None):
        n = x.numel() // self.num_dims
        f = out if out is not None else torch.empty(
            (self.R, self.local_popsize), dtype=torch.float32, device=self.device)
        check(lib().es_eval_bbob(self.ctx, int(fn), _ptr(x), n, self.num_dims, _ptr(f),
                                 _stream(stream)), self.ctx)
        return f

    def tell(self, fitness, stream=None):
        check(lib().es_tell(self.ctx, _ptr(fitness), _stream(stream)), self.ctx)

    def tell_local(self, fitness_all, stream=None):
        """Split phase 1: rank the gathered fitness [W, R, N/W] and reduce this rank's entries."""
        check(lib().es_tell_local(self.ctx, _ptr(fitness_all), _stream(stream)), self.ctx)

    # -- f2: fused peer-memory tell -------------------------------------------------------------
    def p2p_export(self):
        out = _lib.PeerT()
        check(lib().es_p2p_export(self.ctx, C.byref(out)), self.ctx)
        return out

    def p2p_set_peers(self, peers):
        arr = (_lib.PeerT * len(peers))(*peers)
        check(lib().es_p2p_set_peers(self.ctx, arr, len(peers)), self.ctx)

    def tell_p2p_apply(self, stream=None):
        """After tell_local on every rank: reduce-scatter → update → all-gather in one kernel."""
        check(lib().es_tell_p2p_apply(self.ctx, _stream(stream)), self.ctx)

    def tell_p2p_finish(self, stream=None):
        """One global-norm phase after a barrier (Sep-CMA-ES: 1, ClipUp: 2; no-op otherwise)."""
        check(lib().es_tell_p2p_finish(self.ctx, _stream(stream)), self.ctx)

    def p2p_finish_phases(self):
        return int(lib().es_p2p_finish_phases(self.ctx))

    def check_guards(self):
        """ES_GUARD_ALLOCS=1 contexts: guard bytes overwritten so far (0 = no out-of-bounds write)."""
        n = C.c_int64(-1)
        check(lib().es_debug_check_guards(self.ctx, C.byref(n)), self.ctx)
        return int(n.value)

    def nvls_open(self, creator, handle=None):
        """f2 NVLS: create (creator) or join the multicast object; returns the 64-byte handle."""
        h = torch.zeros(64, dtype=torch.uint8)
        if handle is not None:
            h[:] = torch.frombuffer(bytearray(handle), dtype=torch.uint8)
        check(lib().es_nvls_open(self.ctx, C.c_void_p(h.data_ptr()), 1 if creator else 0),
              self.ctx)
        return bytes(h.numpy())

    def nvls_bind(self):
        check(lib().es_nvls_bind(self.ctx), self.ctx)

    def tell_nvls_apply(self, stream=None):
        check(lib().es_tell_nvls_apply(self.ctx, _stream(stream)), self.ctx)

    def nvls_connect(self, group):
        """Real multi-GPU: rank 0 creates the multicast object, the others join, all bind."""
        rank = torch.distributed.get_rank(group)
        h = self.nvls_open(True) if rank == 0 else None
        obj = [h]
        torch.distributed.broadcast_object_list(obj, src=torch.distributed.get_global_rank(group, 0),
                                                group=group)
        if rank != 0:
            self.nvls_open(False, obj[0])
        torch.distributed.barrier(group)
        self.nvls_bind()
        torch.distributed.barrier(group)

    def p2p_connect(self, group):
        """Real multi-GPU: exchange CUDA IPC handles over `group` and map the peers' buffers."""
        h = torch.zeros(10 * 64, dtype=torch.uint8)
        check(lib().es_p2p_ipc_export(self.ctx, C.c_void_p(h.data_ptr())), self.ctx)
        allh = [None] * torch.distributed.get_world_size(group)
        torch.distributed.all_gather_object(allh, bytes(h.numpy()), group=group)
        buf = torch.frombuffer(bytearray(b"".join(allh)), dtype=torch.uint8)
        check(lib().es_p2p_ipc_open(self.ctx, C.c_void_p(buf.data_ptr())), self.ctx)

    def weight_decay(self, fitness, out=None, stream=None):
        """f + weight_decay·‖x_j‖² for this rank's members of the asked generation (es_tell does
        this itself; split-phase callers apply it to their slice before gathering)."""
        o = out if out is not None else torch.empty_like(fitness)
        check(lib().es_weight_decay(self.ctx, _ptr(fitness), _ptr(o), _stream(stream)), self.ctx)
        return o

    def tell_apply(self, stream=None):
        """Split phase 2: apply the update from the (summed) 'dirsum' field (D-shard: from the
        summed 'norm2' shares; tell_apply_phases() calls)."""
        check(lib().es_tell_apply(self.ctx, _stream(stream)), self.ctx)

    def tell_apply_phases(self):
        return int(lib().es_tell_apply_phases(self.ctx))

    def sqnorm_partial(self, stream=None):
        """D-shard: this rank's binary64 Σ_{owned d} x² per member [R, N] of the asked generation."""
        out = torch.empty((self.R, self.local_popsize), dtype=torch.float64, device=self.device)
        check(lib().es_sqnorm_partial(self.ctx, _ptr(out), _stream(stream)), self.ctx)
        return out

    def weight_decay_apply(self, fitness, sqnorm, out=None, stream=None):
        """f + weight_decay·‖x‖² from squared norms summed over the D-shard ranks."""
        o = out if out is not None else torch.empty_like(fitness)
        check(lib().es_weight_decay_apply(self.ctx, _ptr(fitness), _ptr(sqnorm), _ptr(o),
                                          _stream(stream)), self.ctx)
        return o

    def synth_fitness(self, out=None, stream=None):
        f = out if out is not None else torch.empty(
            (self.R, self.local_popsize), dtype=torch.float32, device=self.device)
        check(lib().es_synth_fitness(self.ctx, _ptr(f), _stream(stream)), self.ctx)
        return f

    def set_mlp_problem(self, widths, batch=128, data_seed=0, stream=None):
        w = (C.c_int32 * len(widths))(*widths)
        check(lib().es_set_mlp_problem(self.ctx, w, len(widths), batch, data_seed,
                                       _stream(stream)), self.ctx)

    # -- state ----------------------------------------------------------------------------------
    def ask_eval_partial(self, fn, out_x=None, write_x=False, stream=None):
        """D-shard: this rank's binary64 partial fitness [R, N] (fused ask + evaluate)."""
        x = None
        if write_x:
            x = out_x if out_x is not None else torch.empty(
                (self.R, self.popsize, self.x_dims), dtype=torch.float32, device=self.device)
        p = torch.empty((self.R, self.popsize), dtype=torch.float64, device=self.device)
        check(lib().es_ask_eval_partial(self.ctx, int(fn), _ptr(x) if x is not None else None,
                                        _ptr(p), _stream(stream)), self.ctx)
        return x, p

    def _shape(self, name):
        R, N, D = self.R, self.popsize, self.state_dims
        if name in ("best_f", "sigma", "lrate", "gen", "norm2"):
            return (R,)
        if name in ("shaped", "rank_s", "rank_e", "perm", "fitness"):
            return (R, N)
        if name == "dirsum":
            return (2, R, D)
        if name in ("cov", "chol"):
            return (R, D, D)
        return (R, D)

    def get(self, name, stream=None):
        dt = {"gen": torch.int32, "rank_s": torch.int32, "rank_e": torch.int32,
              "perm": torch.int32, "dirsum": torch.float64,
              "norm2": torch.float64}.get(name, torch.float32)
        out = torch.empty(self._shape(name), dtype=dt, device=self.device)
        check(lib().es_get(self.ctx, FIELDS[name], _ptr(out), _stream(stream)), self.ctx)
        return out

    def set(self, name, value, stream=None):
        v = value.to(self.device).contiguous()
        check(lib().es_set(self.ctx, FIELDS[name], _ptr(v), _stream(stream)), self.ctx)

    def profile(self, on=True):
        check(lib().es_profile_enable(self.ctx, 1 if on else 0), self.ctx)

    def profile_read(self, max_kinds=16):
        names = C.create_string_buffer(32 * max_kinds)
        ms = (C.c_double * max_kinds)()
        cnt = (C.c_int64 * max_kinds)()
        n = lib().es_profile_read(self.ctx, names, ms, cnt, max_kinds)
        if n < 0:
            raise RuntimeError("es_profile_read failed")
        raw = names.raw
        return {raw[32 * k:32 * k + 32].split(b"\0")[0].decode(): (ms[k], cnt[k]) for k in range(n)}

    @property
    def kernel_launches(self):
        return lib().es_kernel_launches(self.ctx)

    def close(self):
        if getattr(self, "ctx", None) and self.ctx.value:
            lib().es_destroy(self.ctx)
            self.ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
