"""ctypes binding of libes_b200.so (include/es.h). Argument marshalling only: every step of the
hot path runs in the library's sm_100a kernels. There is no fallback — a missing library raises."""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libes_b200.so")

ES_SUCCESS = 0
STATUS = {0: "success", 1: "invalid argument", 2: "bad state", 3: "CUDA error", 4: "NCCL error",
          5: "out of device memory", 6: "unsupported"}

OPENAI_ES, PGPE, SNES, SEP_CMA_ES, ARS, CMA_ES = 0, 1, 2, 3, 4, 5
ADAM, SGD, CLIPUP = 0, 1, 2
SPHERE, ROSENBROCK, RASTRIGIN, MLP, MLP16 = 0, 1, 2, 3, 4
FIELDS = dict(mean=0, sigma_d=1, adam_m=2, adam_v=3, p_sigma=4, p_c=5, C=6, best_x=7, best_f=8,
              sigma=9, lrate=10, gen=11, shaped=12, rank_s=13, rank_e=14, perm=15, fitness=16,
              dirsum=17, norm2=18, cov=19, chol=20)

EXPORTS = ["es_init", "es_ask", "es_eval_bbob", "es_tell", "es_synth_fitness", "es_get", "es_set",
           "es_set_mlp_problem", "es_mlp_num_params", "es_shape", "es_kernel_launches",
           "es_destroy", "es_last_error", "es_status_string", "es_nccl_unique_id_size",
           "es_nccl_get_unique_id", "es_debug_primitive", "es_profile_enable", "es_profile_read",
           "es_tell_local", "es_tell_apply", "es_shard_plan", "es_ask_eval", "es_weight_decay",
           "es_init_dshard", "es_dshard_plan", "es_dshard_info", "es_ask_eval_partial",
           "es_p2p_export", "es_p2p_set_peers", "es_tell_p2p_apply", "es_p2p_ipc_export",
           "es_p2p_ipc_open", "es_tell_p2p_finish", "es_p2p_finish_phases", "es_debug_check_guards", "es_tell_apply_phases", "es_sqnorm_partial", "es_weight_decay_apply", "es_nvls_open", "es_nvls_bind", "es_tell_nvls_apply"]


class RunParams(C.Structure):
    """es_run_params_t (include/es.h)."""
    _fields_ = [("seed", C.c_uint64), ("init_min", C.c_float), ("init_max", C.c_float),
                ("sigma_init", C.c_float), ("sigma_decay", C.c_float), ("sigma_limit", C.c_float),
                ("lrate_init", C.c_float), ("lrate_decay", C.c_float), ("lrate_limit", C.c_float),
                ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("sigma_lrate", C.c_float), ("sigma_max_change", C.c_float),
                ("temperature", C.c_float), ("elite_ratio", C.c_float), ("shaping", C.c_int32),
                ("optimizer", C.c_int32), ("momentum", C.c_float), ("max_speed", C.c_float),
                ("weight_decay", C.c_float), ("clip_min", C.c_float), ("clip_max", C.c_float)]


class PeerT(C.Structure):
    """es_peer_t: a rank's direction-sum buffer and state-field device pointers (f2)."""
    _fields_ = [("dirsum", C.c_void_p), ("field", C.c_void_p * 8), ("norm2", C.c_void_p)]


class ESError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


_lib = None


def lib():
    """Load the CUDA library; raise loudly if it has not been built (no CPU fallback exists)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ "
                          f"as g; g.build()'` (the CUDA path has no fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i32, i64, u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
    sig = {
        "es_init": (i32, [C.POINTER(vp), i32, i32, i32, i64, C.POINTER(RunParams), i32, i32, vp, vp]),
        "es_ask": (i32, [vp, vp, vp]),
        "es_eval_bbob": (i32, [vp, i32, vp, i64, i64, vp, vp]),
        "es_tell": (i32, [vp, vp, vp]),
        "es_synth_fitness": (i32, [vp, vp, vp]),
        "es_get": (i32, [vp, i32, vp, vp]),
        "es_set": (i32, [vp, i32, vp, vp]),
        "es_set_mlp_problem": (i32, [vp, C.POINTER(i32), i32, i32, u64, vp]),
        "es_mlp_num_params": (i64, [C.POINTER(i32), i32]),
        "es_shape": (i32, [vp, C.POINTER(i64)]),
        "es_kernel_launches": (i64, [vp]),
        "es_destroy": (i32, [vp]),
        "es_last_error": (C.c_char_p, [vp]),
        "es_status_string": (C.c_char_p, [i32]),
        "es_nccl_unique_id_size": (i32, []),
        "es_nccl_get_unique_id": (i32, [vp]),
        "es_debug_primitive": (i32, [i32, vp, vp, i64, vp]),
        "es_profile_enable": (i32, [vp, i32]),
        "es_tell_local": (i32, [vp, vp, vp]),
        "es_ask_eval": (i32, [vp, i32, vp, vp, vp]),
        "es_tell_apply": (i32, [vp, vp]),
        "es_weight_decay": (i32, [vp, vp, vp, vp]),
        "es_init_dshard": (i32, [C.POINTER(vp), i32, i32, i32, i64, C.POINTER(RunParams), i32, i32,
                                 vp, vp]),
        "es_dshard_plan": (i32, [i64, i32, i32, C.POINTER(i64)]),
        "es_dshard_info": (i32, [vp, C.POINTER(i64)]),
        "es_ask_eval_partial": (i32, [vp, i32, vp, vp, vp]),
        "es_p2p_export": (i32, [vp, C.POINTER(PeerT)]),
        "es_p2p_set_peers": (i32, [vp, C.POINTER(PeerT), i32]),
        "es_tell_p2p_apply": (i32, [vp, vp]),
        "es_tell_p2p_finish": (i32, [vp, vp]),
        "es_p2p_finish_phases": (i32, [vp]),
        "es_debug_check_guards": (i32, [vp, vp]),
        "es_tell_apply_phases": (i32, [vp]),
        "es_sqnorm_partial": (i32, [vp, vp, vp]),
        "es_weight_decay_apply": (i32, [vp, vp, vp, vp, vp]),
        "es_p2p_ipc_export": (i32, [vp, vp]),
        "es_p2p_ipc_open": (i32, [vp, vp]),
        "es_nvls_open": (i32, [vp, vp, i32]),
        "es_nvls_bind": (i32, [vp]),
        "es_tell_nvls_apply": (i32, [vp, vp]),
        "es_shard_plan": (i32, [i32, i32, i32, i32, C.POINTER(i32)]),
        "es_profile_read": (i32, [vp, C.c_char_p, C.POINTER(C.c_double), C.POINTER(i64), i32]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    _lib = L
    return L


def check(code, ctx=None):
    if code != ES_SUCCESS:
        msg = lib().es_last_error(ctx)
        raise ESError(code, msg.decode() if msg else "")
