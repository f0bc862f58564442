"""ctypes binding of the C oracle (oracle/es_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg. The product package never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libes_oracle.so")
SRC = os.path.join(HERE, "es_oracle.c")
HDR = os.path.join(HERE, "es_oracle.h")

OPENAI_ES, PGPE, SNES, SEP_CMA_ES, ARS = 0, 1, 2, 3, 4
ADAM, SGD, CLIPUP = 0, 1, 2
SPHERE, ROSENBROCK, RASTRIGIN = 0, 1, 2
V_MEAN, V_SIGMA, V_ADAM_M, V_ADAM_V, V_PSIGMA, V_PC, V_C, V_BEST_X, NV = range(9)


def build(force: bool = False) -> str:
    """Compile the oracle with the flags NUMERICS.md fixes (no contraction, no fast-math)."""
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(SRC), os.path.getmtime(HDR))):
        return LIB_PATH
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c99", "-Wall", "-fPIC",
           "-shared", SRC, "-o", LIB_PATH, "-lm"]
    subprocess.check_call(cmd)
    return LIB_PATH


class Params(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("init_min", C.c_float), ("init_max", C.c_float),
                ("sigma_init", C.c_float), ("sigma_decay", C.c_float), ("sigma_limit", C.c_float),
                ("lrate_init", C.c_float), ("lrate_decay", C.c_float), ("lrate_limit", C.c_float),
                ("beta1", C.c_float), ("beta2", C.c_float), ("eps", C.c_float),
                ("sigma_lrate", C.c_float), ("sigma_max_change", C.c_float),
                ("temperature", C.c_float), ("elite_ratio", C.c_float), ("shaping", C.c_int32),
                ("optimizer", C.c_int32), ("momentum", C.c_float), ("max_speed", C.c_float),
                ("weight_decay", C.c_float), ("clip_min", C.c_float), ("clip_max", C.c_float)]


class RunT(C.Structure):
    _fields_ = [("algo", C.c_int32), ("popsize", C.c_int32), ("num_dims", C.c_int64),
                ("p", Params), ("t", C.c_uint32), ("lr", C.c_float), ("sigma", C.c_float),
                ("b1pow", C.c_double), ("b2pow", C.c_double), ("best_f", C.c_float),
                ("mu", C.c_int32), ("mueff", C.c_double), ("c_sigma", C.c_double),
                ("d_sigma", C.c_double), ("c_c", C.c_double), ("c_1", C.c_double),
                ("c_mu", C.c_double), ("chi_d", C.c_double), ("eta_sigma", C.c_double),
                ("vec", C.POINTER(C.c_float)), ("wpos", C.POINTER(C.c_float)),
                ("dims", C.POINTER(C.c_int64)), ("full_dims", C.c_int64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        fp, u32p = C.POINTER(C.c_float), C.POINTER(C.c_uint32)
        dp, i32p = C.POINTER(C.c_double), C.POINTER(C.c_int32)
        sig = {
            "orc_philox4x32_10": (None, [u32p, u32p, u32p]),
            "orc_u_a": (C.c_float, [C.c_uint32]),
            "orc_u_b": (C.c_float, [C.c_uint32]),
            "orc_ln": (C.c_float, [C.c_float]),
            "orc_ln_n": (None, [fp, fp, C.c_int64]),
            "orc_sincos2pi_n": (None, [fp, fp, fp, C.c_int64]),
            "orc_sinpi_half_n": (None, [fp, fp, C.c_int64]),
            "orc_normals_n": (None, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int64, fp]),
            "orc_direction": (None, [C.c_uint64, C.c_uint32, C.c_uint32, C.c_int64, fp]),
            "orc_init": (C.c_int, [C.POINTER(RunT)]),
            "orc_num_directions": (C.c_int, [C.POINTER(RunT)]),
            "orc_ask": (None, [C.POINTER(RunT), fp]),
            "orc_member": (None, [C.POINTER(RunT), C.c_int32, fp]),
            "orc_eval": (None, [C.c_int32, fp, C.c_int32, C.c_int64, fp]),
            "orc_key": (C.c_uint32, [C.c_float]),
            "orc_rank": (None, [fp, C.c_int32, i32p, i32p, i32p]),
            "orc_centered_rank": (None, [fp, C.c_int32, fp]),
            "orc_member_weights": (None, [fp, fp, C.c_int32, fp]),
            "orc_zscore": (None, [fp, C.c_int32, fp]),
            "orc_reduce": (None, [C.POINTER(RunT), fp, dp]),
            "orc_reduce_range": (None, [C.POINTER(RunT), fp, C.c_int32, C.c_int32, dp]),
            "orc_num_entries": (C.c_int, [C.POINTER(RunT), fp]),
            "orc_tell": (C.c_int, [C.POINTER(RunT), fp]),
            "orc_tell_apply": (C.c_int, [C.POINTER(RunT), fp, dp]),
            "orc_weight_decay": (None, [fp, fp, C.c_int32, C.c_int64, C.c_float, fp]),
            "orc_run_weight_decay": (None, [C.POINTER(RunT), fp, fp]),
            "orc_synth_fitness": (None, [C.c_uint64, C.c_uint32, C.c_int32, fp]),
            "orc_fp16": (C.c_float, [C.c_float]),
            "orc_mlp_create": (C.c_void_p, [i32p, C.c_int32, C.c_int32, C.c_uint64]),
            "orc_mlp_destroy": (None, [C.c_void_p]),
            "orc_mlp_dims": (C.c_int64, [C.c_void_p]),
            "orc_mlp_teacher": (None, [C.c_void_p, fp]),
            "orc_mlp_eval": (None, [C.c_void_p, fp, C.c_int32, fp]),
            "orc_mlp_eval_f16": (None, [C.c_void_p, fp, C.c_int32, fp]),
            "orc_mlp_targets": (dp, [C.c_void_p]),
            "orc_mlp_targets_f16": (fp, [C.c_void_p]),
            "orc_mlp_inputs": (fp, [C.c_void_p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype, f.argtypes = res, args
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_p(c, C.c_uint32), _p(k, C.c_uint32), _p(o, C.c_uint32))
    return o


def ln(u):
    u = np.ascontiguousarray(u, dtype=np.float32)
    out = np.empty_like(u)
    lib().orc_ln_n(_p(u, C.c_float), _p(out, C.c_float), u.size)
    return out


def sincos2pi(u):
    u = np.ascontiguousarray(u, dtype=np.float32)
    c, s = np.empty_like(u), np.empty_like(u)
    lib().orc_sincos2pi_n(_p(u, C.c_float), _p(c, C.c_float), _p(s, C.c_float), u.size)
    return c, s


def sinpi_half(b):
    b = np.ascontiguousarray(b, dtype=np.float32)
    out = np.empty_like(b)
    lib().orc_sinpi_half_n(_p(b, C.c_float), _p(out, C.c_float), b.size)
    return out


def normals(seed, i, t, tag, n):
    out = np.empty(n, dtype=np.float32)
    lib().orc_normals_n(seed, i, t, tag, n, _p(out, C.c_float))
    return out


def direction(seed, i, t, D):
    z = np.empty(D, dtype=np.float32)
    lib().orc_direction(seed, i, t, D, _p(z, C.c_float))
    return z


def key(f):
    return lib().orc_key(float(np.float32(f)))


def rank(f):
    f = np.ascontiguousarray(f, dtype=np.float32)
    N = f.size
    s, e, perm = (np.empty(N, dtype=np.int32) for _ in range(3))
    lib().orc_rank(_p(f, C.c_float), N, _p(s, C.c_int32), _p(e, C.c_int32), _p(perm, C.c_int32))
    return s, e, perm


def centered_rank(f):
    f = np.ascontiguousarray(f, dtype=np.float32)
    c = np.empty_like(f)
    lib().orc_centered_rank(_p(f, C.c_float), f.size, _p(c, C.c_float))
    return c


def weight_decay(f, x, coef):
    f = np.ascontiguousarray(f, dtype=np.float32)
    x = np.ascontiguousarray(x, dtype=np.float32).reshape(f.size, -1)
    out = np.empty_like(f)
    lib().orc_weight_decay(_p(f, C.c_float), _p(x, C.c_float), f.size, x.shape[1], coef,
                           _p(out, C.c_float))
    return out


def zscore(f):
    f = np.ascontiguousarray(f, dtype=np.float32)
    out = np.empty_like(f)
    lib().orc_zscore(_p(f, C.c_float), f.size, _p(out, C.c_float))
    return out


def member_weights(wpos, f):
    f = np.ascontiguousarray(f, dtype=np.float32)
    wpos = np.ascontiguousarray(wpos, dtype=np.float32)
    w = np.empty_like(f)
    lib().orc_member_weights(_p(wpos, C.c_float), _p(f, C.c_float), f.size, _p(w, C.c_float))
    return w


def evaluate(fn, x):
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim == 1:
        x = x[None]
    n, D = x.shape
    f = np.empty(n, dtype=np.float32)
    lib().orc_eval(fn, _p(x, C.c_float), n, D, _p(f, C.c_float))
    return f


def synth_fitness(seed, t, N):
    f = np.empty(N, dtype=np.float32)
    lib().orc_synth_fitness(seed, t, N, _p(f, C.c_float))
    return f


DEFAULTS = dict(init_min=-1.0, init_max=1.0, sigma_init=0.05, sigma_decay=0.999, sigma_limit=0.01,
                lrate_init=0.01, lrate_decay=0.999, lrate_limit=0.001, beta1=0.9, beta2=0.999,
                eps=1e-8, sigma_lrate=0.2, sigma_max_change=0.2, temperature=12.0,
                elite_ratio=0.5, shaping=0, optimizer=0, momentum=0.9, max_speed=0.02,
                weight_decay=0.0, clip_min=-np.inf, clip_max=np.inf)
PGPE_ELITE_DEFAULT = 1.0     # Q13: App. B has no PGPE elite ratio; every pair is kept


class Run:
    """One oracle run (state owned by numpy arrays)."""

    def __init__(self, algo, popsize, num_dims, seed=0, dims=None, **params):
        """dims: optional sorted global dimension indices (num_dims is then the full D)."""
        kw = dict(DEFAULTS)
        if algo == PGPE:
            kw["elite_ratio"] = PGPE_ELITE_DEFAULT
        kw.update(params)
        full = num_dims
        if dims is not None:
            self.dims = np.ascontiguousarray(dims, dtype=np.int64)
            num_dims = len(self.dims)
        self.vec = np.zeros((NV, num_dims), dtype=np.float32)
        self.wpos = np.zeros(popsize, dtype=np.float32)
        self.r = RunT()
        self.r.algo, self.r.popsize, self.r.num_dims = algo, popsize, num_dims
        self.r.p = Params(seed=seed, **kw)
        self.r.vec = _p(self.vec, C.c_float)
        self.r.wpos = _p(self.wpos, C.c_float)
        if dims is not None:
            self.r.dims = _p(self.dims, C.c_int64)
        self.r.full_dims = full
        if lib().orc_init(C.byref(self.r)) != 0:
            raise ValueError("oracle init rejected the arguments")

    # state views
    @property
    def mean(self):
        return self.vec[V_MEAN]

    @property
    def sigma_d(self):
        return self.vec[V_SIGMA]

    @property
    def num_directions(self):
        return lib().orc_num_directions(C.byref(self.r))

    def __getattr__(self, name):
        r = self.__dict__.get("r")
        if r is not None and name in dict(RunT._fields_):
            return getattr(r, name)
        raise AttributeError(name)

    def ask(self):
        x = np.empty((self.r.popsize, self.r.num_dims), dtype=np.float32)
        lib().orc_ask(C.byref(self.r), _p(x, C.c_float))
        return x

    def member(self, j):
        x = np.empty(self.r.num_dims, dtype=np.float32)
        lib().orc_member(C.byref(self.r), j, _p(x, C.c_float))
        return x

    def reduce(self, f):
        f = np.ascontiguousarray(f, dtype=np.float32)
        G = np.empty((2, self.r.num_dims), dtype=np.float64)
        lib().orc_reduce(C.byref(self.r), _p(f, C.c_float), _p(G, C.c_double))
        return G

    def reduce_range(self, f, e0, e1):
        f = np.ascontiguousarray(f, dtype=np.float32)
        G = np.empty((2, self.r.num_dims), dtype=np.float64)
        lib().orc_reduce_range(C.byref(self.r), _p(f, C.c_float), e0, e1, _p(G, C.c_double))
        return G

    def num_entries(self, f):
        f = np.ascontiguousarray(f, dtype=np.float32)
        return lib().orc_num_entries(C.byref(self.r), _p(f, C.c_float))

    def tell(self, f):
        f = np.ascontiguousarray(f, dtype=np.float32)
        lib().orc_tell(C.byref(self.r), _p(f, C.c_float))

    def tell_apply(self, f, G):
        """The update half of tell from direction sums G [2][D] (no best tracking), then t+1."""
        f = np.ascontiguousarray(f, dtype=np.float32)
        G = np.ascontiguousarray(G, dtype=np.float64).reshape(2, self.r.num_dims)
        lib().orc_tell_apply(C.byref(self.r), _p(f, C.c_float), _p(G, C.c_double))

    def weight_decay(self, f):
        """f_j + weight_decay ||x_j||^2 for the current members (what tell ranks)."""
        f = np.ascontiguousarray(f, dtype=np.float32)
        out = np.empty_like(f)
        lib().orc_run_weight_decay(C.byref(self.r), _p(f, C.c_float), _p(out, C.c_float))
        return out


class MLP:
    """N14 synthetic MLP regression problem (oracle side). evaluate() is the definition (binary64
    forward of the fp32 parameters); evaluate_f16() is the N14' fp16-image approximation model."""

    def __init__(self, widths, batch=128, seed=0):
        w = (C.c_int32 * len(widths))(*widths)
        self.widths, self.batch = list(widths), batch
        self.h = lib().orc_mlp_create(w, len(widths), batch, seed)
        if not self.h:
            raise ValueError("bad MLP problem")
        self.D = lib().orc_mlp_dims(self.h)

    def teacher(self):
        t = np.empty(self.D, dtype=np.float32)
        lib().orc_mlp_teacher(self.h, _p(t, C.c_float))
        return t

    def targets(self):
        p = lib().orc_mlp_targets(self.h)
        return np.ctypeslib.as_array(p, shape=(self.batch * self.widths[-1],)).reshape(
            self.batch, self.widths[-1]).copy()

    def targets_f16(self):
        p = lib().orc_mlp_targets_f16(self.h)
        return np.ctypeslib.as_array(p, shape=(self.batch * self.widths[-1],)).reshape(
            self.batch, self.widths[-1]).copy()

    def inputs(self):
        p = lib().orc_mlp_inputs(self.h)
        return np.ctypeslib.as_array(p, shape=(self.batch * self.widths[0],)).reshape(
            self.batch, self.widths[0]).copy()

    def _eval(self, fn, x):
        x = np.ascontiguousarray(x, dtype=np.float32).reshape(-1, self.D)
        f = np.empty(x.shape[0], dtype=np.float32)
        fn(self.h, _p(x, C.c_float), x.shape[0], _p(f, C.c_float))
        return f

    def evaluate(self, x):
        return self._eval(lib().orc_mlp_eval, x)

    def evaluate_f16(self, x):
        return self._eval(lib().orc_mlp_eval_f16, x)

    def __del__(self):
        try:
            lib().orc_mlp_destroy(self.h)
        except Exception:
            pass


def fp16(v):
    return np.array([lib().orc_fp16(float(a)) for a in np.ravel(v)], dtype=np.float32)
