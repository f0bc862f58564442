#!/usr/bin/env python
"""Benchmark of the B200 ES hot path (BASELINE.json metric: ES generations/s and N·D samples/s per
B200 at 1/2/4/8 GPUs, with the achieved fraction of the bounding roofline).

Default workload = BASELINE.json configs[1] ("c2"): Sep-CMA-ES and SNES on Rastrigin, D=1000,
N=256, 512 independent runs each (vmap over seeds). One step = one full generation
(ask -> evaluate -> tell) of BOTH 512-run batches. Multi-GPU: every rank runs its own 512+512 runs
(seeds offset by rank; "replicas only", no data-path collective) -> weak scaling.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c3|c5] [--impl reference]

Prints ONE JSON line (rank 0). See DESIGN.md "Measurement" for every field.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads as W  # noqa: E402

# NUMERICS.md N16: lane-ops of one normal (Philox ¼ + Box–Muller ½ pair), spec operation count.
NORMAL_OPS = 37
# consumer ops per normal: ask antithetic (2 FFMA), ask plain (1 FFMA); tell: F2F + DFMA(s)
ASK_USE = {W.OPENAI_ES: 2, W.PGPE: 2, W.SNES: 1, W.SEP_CMA_ES: 1}
TELL_USE = {W.OPENAI_ES: 2, W.PGPE: 5, W.SNES: 5, W.SEP_CMA_ES: 4}
STATE_BYTES = {W.OPENAI_ES: 24, W.PGPE: 32, W.SNES: 16, W.SEP_CMA_ES: 40}   # r+w per dim per tell
# N7 operations per evaluated element (fused ask+eval): conversions + binary64 accumulation (+ the
# Rastrigin sin(pi b) polynomial, Rosenbrock's double pair term)
EVAL_OPS = {W.SPHERE: 2, W.ROSENBROCK: 12, W.RASTRIGIN: 15}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return dict(hbm_gbs=d["hbm_gbs"], sm_max_mhz=d.get("sm_max_mhz", 1965.0),
                    bf16_tflops=d.get("bf16_tflops", 1590.0), src="measured")
    return dict(hbm_gbs=6650.0, sm_max_mhz=1965.0, bf16_tflops=1590.0, src="fallback")


def alu_peak(peaks, sms=148):
    # 4 SMSPs x 1 warp-instruction/clk x 32 lanes per SM (guide: 148 SMs, 1965 MHz max clock)
    return sms * 128 * peaks["sm_max_mhz"] * 1e6


# ----------------------------------------------------------------------------- workloads
def handles_for(cfg_key, rank):
    """(label, cfg dict, params list) per ES handle of the workload."""
    if cfg_key == "c2":
        out = []
        for key in ("c2_sepcma", "c2_snes"):
            cfg = W.CONFIGS[key]
            params = [W.config_params(cfg, r, seed_offset=rank * cfg["R"], hyper_vmap=True)
                      for r in range(cfg["R"])]
            out.append((key, cfg, params))
        return out
    if cfg_key in ("c1", "c3", "c6"):
        cfg = W.CONFIGS[cfg_key]
        return [(cfg_key, cfg, [W.config_params(cfg, r) for r in range(cfg["R"])])]
    if cfg_key == "c5":
        cfg = sweep_cfg(SWEEP["N"], SWEEP["D"])
        return [("c5", cfg, [W.config_params(cfg, r) for r in range(cfg["R"])])]
    if cfg_key == "c4":
        cfg = dict(W.CONFIGS["c4"], widths=MLP_WIDTHS, batch=128, data_seed=0,
                   fn=W.MLP16 if MLP_MODE["mode"] == "fp16" else W.MLP)
        return [("c4", cfg, [W.config_params(cfg, r) for r in range(cfg["R"])])]
    raise SystemExit(f"unknown config {cfg_key}")


SWEEP = {"N": 4096, "D": 985_216}     # the north-star tell point (config 4's shape)
# c4's MLP fitness: "fp32" = N14, the definition (fp32-accurate tcgen05 kernel); "fp16" = N14',
# the labelled fp16-parameter-image approximation
MLP_MODE = {"mode": "fp32"}
MLP_WIDTHS = [256, 512, 512, 512, 512, 128]   # config 4: D = 985,216


def sweep_cfg(N, D):
    """Config 5 cell: OpenAI-ES tell on synthetic fitness (N15); x is never materialised."""
    return dict(name=f"openai_es-tell-synthetic-D{D}-N{N}-R1", algo=W.OPENAI_ES, fn=None, D=D, N=N,
                R=1, init=(-0.04, 0.04))


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [c.strip() for c in line.split(",")]))

    def stop(self, t0=None, t1=None):
        """Samples inside the host window [t0, t1] of the timed region (±20 ms, one sampling
        period); if that window is shorter than a period and caught none, the nearest sample."""
        if self.proc is None:
            return None
        time.sleep(0.1)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.t.join(timeout=2)
        rows = [(ts, r) for ts, r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        if t0 is not None and rows:
            inside = [(ts, r) for ts, r in rows if t0 - 0.02 <= ts <= t1 + 0.02]
            rows = inside or [min(rows, key=lambda x: abs(x[0] - 0.5 * (t0 + t1)))]
        sm = [float(r[0]) for _, r in rows]
        mx = [float(r[1]) for _, r in rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for _, r in rows for k in range(4)
                          if r[3 + k].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(sm)}


# ----------------------------------------------------------------------------- CPU oracle
SWEEP_ORACLE_DIMS = 2048     # dimension subset of the oracle's tell-only sample (N15 sweeps)


def _oracle_gen(args):
    """`gens` generations of one oracle run (ask, evaluate, tell); returns (samples, seconds).
    Tell-only sweeps (fn None) run the oracle's tell on a subset of the dimensions."""
    algo, fn, N, D, params, gens = args
    from oracle import oracle as O
    if fn is None:
        dims = range(min(D, SWEEP_ORACLE_DIMS))
        run = O.Run(algo, N, D, dims=dims, **params)
        t0 = time.perf_counter()
        for _ in range(gens):
            run.tell(O.synth_fitness(params["seed"], run.t, N))
        return N * len(dims) * gens, time.perf_counter() - t0
    if fn in (W.MLP, W.MLP16):
        # config 4: ask + MLP fitness of `gens` members (the tell, a third of the oracle's
        # per-generation work, is excluded from this sample)
        mlp = O.MLP(MLP_WIDTHS, 128, 0)
        run = O.Run(algo, N, D, **params)
        ev = mlp.evaluate if fn == W.MLP else mlp.evaluate_f16
        t0 = time.perf_counter()
        for j in range(gens):
            ev(run.member(j % N))
        return D * gens, time.perf_counter() - t0
    if algo == W.CMA_ES:                     # f4: numpy binary64 oracle, one BLAS thread
        from oracle import cma_oracle
        from threadpoolctl import threadpool_limits
        with threadpool_limits(1):
            run = cma_oracle.CMARun(N, D, **params)
            t0 = time.perf_counter()
            for _ in range(gens):
                run.tell(O.evaluate(fn, run.ask()))
            return N * D * gens, time.perf_counter() - t0
    run = O.Run(algo, N, D, **params)
    t0 = time.perf_counter()
    for _ in range(gens):
        x = run.ask()
        run.tell(O.evaluate(fn, x))
    return N * D * gens, time.perf_counter() - t0


def host_description():
    """nproc, lscpu model / sockets / SMT of the host the oracle is timed on."""
    d = {"nproc": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        kv = {}
        for line in out.splitlines():
            if ":" in line:
                k, v = line.split(":", 1)
                kv[k.strip()] = v.strip()
        d.update(model=kv.get("Model name"), sockets=kv.get("Socket(s)"),
                 cores_per_socket=kv.get("Core(s) per socket"),
                 threads_per_core=kv.get("Thread(s) per core"))
    except (OSError, subprocess.SubprocessError):
        pass
    return d


def cpu_baseline(cfg_key, budget_s=15.0, procs=None):
    """The oracle as it stands, on the host cores, on a bounded sample of the same workload:
    (i) one thread (one process, run 0 of each handle) and (ii) all cores — independent runs in
    parallel processes (c2: one oracle run per process, as vmap over runs; single-run
    configs: one replica of the run per process, the same per-core work). The all-cores figure is
    `value`."""
    import multiprocessing as mp
    from oracle import oracle as O
    O.build()
    hs = handles_for(cfg_key, 0)
    procs = procs or (os.cpu_count() or 1)
    # (i) single thread: calibrate one generation of run 0 of each handle, then ~budget/3 seconds
    per_gen = []
    for _, cfg, params in hs:
        s, t = _oracle_gen((cfg["algo"], cfg["fn"], cfg["N"], cfg["D"], params[0], 1))
        per_gen.append(t)
    g1 = max(1, int(budget_s / 3 / (sum(per_gen) + 1e-9)))
    t0 = time.perf_counter()
    s1 = sum(_oracle_gen((cfg["algo"], cfg["fn"], cfg["N"], cfg["D"], params[0], g1))[0]
             for _, cfg, params in hs)
    w1 = time.perf_counter() - t0
    # (ii) all cores
    n_runs = min(procs, min(len(p) for _, _, p in hs))
    if hs[0][1]["fn"] in (W.MLP, W.MLP16) or len(hs[0][2]) == 1:
        n_runs = procs                     # one run: a replica per process
    gens = max(1, int(2 * budget_s / 3 / (sum(per_gen) * math.ceil(len(hs) * n_runs / procs) + 1e-9)))
    jobs = [(cfg["algo"], cfg["fn"], cfg["N"], cfg["D"], params[r % len(params)], gens)
            for _, cfg, params in hs for r in range(n_runs)]
    t0 = time.perf_counter()
    with mp.get_context("fork").Pool(procs) as pool:
        res = pool.map(_oracle_gen, jobs)
    wall = time.perf_counter() - t0
    samples = sum(s for s, _ in res)
    unit_desc = ("generations each (tell on synthetic fitness, first %d dims; samples = N x those "
                 "dims)" % SWEEP_ORACLE_DIMS if hs[0][1]["fn"] is None else
                 "members each (ask + MLP fitness; tell excluded)"
                 if hs[0][1]["fn"] in (W.MLP, W.MLP16) else "generations each (ask+eval+tell)")
    return {"value": samples / wall, "unit": "samples/s", "cores": min(procs, len(jobs)),
            "kind": "oracle",
            "sample": f"{n_runs} runs of each of {[h[0] for h in hs]}, {gens} {unit_desc}, "
                      f"{procs} processes, {wall:.1f} s wall",
            "single_thread": {"value": s1 / w1, "unit": "samples/s", "cores": 1,
                              "sample": f"run 0 of each handle, {g1} {unit_desc}, {w1:.1f} s"},
            "host": host_description()}


def run_reference(args):
    """--impl reference: the CPU oracle timed as the reference arm (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle as O
    O.build()
    import multiprocessing as mp
    hs = handles_for(args.config, 0)
    procs = os.cpu_count() or 1
    n_runs = min(procs, min(len(p) for _, _, p in hs))
    if hs[0][1]["fn"] in (W.MLP, W.MLP16):
        n_runs = procs
    jobs = [(cfg["algo"], cfg["fn"], cfg["N"], cfg["D"], params[r % len(params)], 1)
            for _, cfg, params in hs for r in range(n_runs)]
    with mp.get_context("fork").Pool(procs) as pool:
        for _ in range(args.warmup):
            pool.map(_oracle_gen, jobs)
        t0 = time.perf_counter()
        samples = 0
        for _ in range(args.steps):
            samples += sum(s for s, _ in pool.map(_oracle_gen, jobs))
        wall = time.perf_counter() - t0
    value = samples / wall
    sample = (f"each step: 1 generation of {n_runs} runs of each of {[h[0] for h in hs]} "
              f"({procs} processes)")
    line = {"metric": metric_name(args.config), "value": value, "unit": "samples/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1e3 * wall / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic", "impl": "reference",
            "config": config_block(args.config, 1),
            "cpu_baseline": {"value": value, "unit": "samples/s", "cores": procs, "kind": "oracle",
                             "sample": sample, "host": host_description()},
            "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def metric_name(cfg_key):
    return ("ES samples/sec (R*N*D per generation, summed over GPUs; generations/s alongside) "
            "and % of roofline")


def config_block(cfg_key, world):
    if cfg_key == "c2":
        a, b = W.CONFIGS["c2_sepcma"], W.CONFIGS["c2_snes"]
        return {"workload": "c2: Sep-CMA-ES and SNES on Rastrigin, D=1000, popsize=256, 512 "
                            "independent seeds each (App. B columns vmapped), one generation of "
                            "both per step",
                "R": a["R"], "N": a["N"], "D": a["D"], "handles": [a["name"], b["name"]],
                "parallelism": f"replicas x{world} (runs per GPU fixed, no collective)",
                "l2": "inputs larger than L2: x is 1.05 GB per step (2 x 524 MB), state 2 MB/run "
                      "array"}
    cfg = W.CONFIGS.get(cfg_key, {})
    if cfg_key == "c4":
        c = W.CONFIGS["c4"]
        return {"workload": "c4: OpenAI-ES + Adam on the synthetic tanh-MLP fitness "
                            f"{MLP_WIDTHS} (D=985,216), popsize 4096, batch 128",
                "R": 1, "N": c["N"], "D": c["D"],
                "parallelism": f"population sharded x{world}" if world > 1 else "1 GPU",
                "l2": ("inputs larger than L2: the MLP reads the population's split binary16 "
                       "image (hi and lo planes, 16.1 GB per step) the ask wrote; x itself is not "
                       "materialised in fp32" if MLP_MODE["mode"] == "fp32" else
                       "inputs larger than L2: the MLP reads the population's fp16 image (8.07 GB "
                       "per step) the ask wrote; x itself is not materialised in fp32")}
    if cfg_key == "c5":
        cfg = sweep_cfg(SWEEP["N"], SWEEP["D"])
        return {"workload": f"c5 cell: {cfg['name']} (tell only on synthetic fitness, the north-star "
                            f"D~1e6 N=4096 point)", "R": 1, "N": cfg["N"], "D": cfg["D"],
                "parallelism": f"population sharded x{world}" if world > 1 else "1 GPU",
                "l2": "x never materialised; state 12 MB resident in L2"}
    if cfg_key == "c6":
        return {"workload": "c6 (SURVEY 8(f) f4, not a BASELINE config): full-covariance CMA-ES on "
                            "Rosenbrock, D=1024, popsize 256, 8 runs; Cholesky factor refreshed "
                            "every generation (k = 1 at this D, N)", "R": cfg["R"], "N": cfg["N"],
                "D": cfg["D"], "parallelism": "1 GPU",
                "l2": "C, A, workspace 4 MB/run each; x, y, z 1 MB/run each (L2-resident)"}
    return {"workload": f"{cfg_key}: {cfg.get('name', '')}", "R": cfg.get("R"), "N": cfg.get("N"),
            "D": cfg.get("D"), "parallelism": f"population sharded x{world}" if world > 1 else "1 GPU",
            "l2": "state resident; x > L2 only for D*N*4 > 126 MB"}


# ----------------------------------------------------------------------------- sub-records
def sub_bench(cfg_key, world, sharded, steps, peaks, group=None):
    """One generation of a config timed on its own (warm-up, a profiled pass for per-kernel CUDA
    events, then `steps` timed steps, max over ranks): the north-star tell cell at W = 1 and the
    population-sharded C5 / C4 records at W > 1 (the path north_star scales)."""
    import torch
    import torch.distributed as dist
    from paper_2212_04180_b200 import strategy as S
    (label, cfg, params), = handles_for(cfg_key, 0)
    es = S.Strategy(cfg["algo"], cfg["N"], cfg["D"], params, group=group if sharded else None)
    nl = es.local_popsize
    f = torch.empty((cfg["R"], nl), dtype=torch.float32, device="cuda")
    if cfg["fn"] in (W.MLP, W.MLP16):
        es.set_mlp_problem(cfg["widths"], cfg["batch"], cfg["data_seed"])

    def step():
        if cfg["fn"] is None:
            es.synth_fitness(out=f)
        else:
            es.ask_eval(cfg["fn"], out_f=f, write_x=False)
        es.tell(f)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    es.profile(True)
    for _ in range(max(2, steps // 2)):
        step()
    torch.cuda.synchronize()
    prof = es.profile_read()
    es.profile(False)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    per_rank = [ms]
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        allt = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(allt, t)
        per_rank = [float(v.item()) for v in allt]
        ms = max(per_rank)
    kern = {k: round(t / max(n, 1), 4) for k, (t, n) in prof.items()}
    W_ = world if sharded else 1
    P = (cfg["N"] // W_) // (2 if cfg["algo"] in (W.OPENAI_ES, W.PGPE) else 1)
    out = {"workload": config_block(cfg_key, W_)["workload"], "N": cfg["N"], "D": cfg["D"],
           "ms_per_generation": ms, "generations_per_s": 1e3 / ms,
           "samples_per_s": cfg["R"] * cfg["N"] * cfg["D"] / (ms / 1e3),
           "kernel_ms_per_launch": kern}
    if world > 1:
        out["per_rank_ms"] = per_rank
        out["allgather_us"] = round(1e3 * kern.get("allgather", 0.0), 2)
        out["allreduce_us"] = round(1e3 * kern.get("allreduce", 0.0), 2)
    tk = "tell" if "tell" in kern else "tell_reduce"
    if tk in kern:
        ops = cfg["R"] * P * cfg["D"] * (NORMAL_OPS + TELL_USE[cfg["algo"]])
        ach = ops / (kern[tk] / 1e3) / 1e12
        out["tell_roofline"] = {"bound": "alu", "kernel": tk, "achieved": ach,
                                "peak": alu_peak(peaks) / 1e12, "unit": "Tlane-op/s",
                                "frac": ach / (alu_peak(peaks) / 1e12),
                                "traffic": ncu_traffic("c5", "tell") if cfg_key == "c5" else None}
    es.close()
    return out


# ----------------------------------------------------------------------------- GPU arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--fused", type=int, default=None,
                    help="1: es_ask_eval (BBOB: one fused kernel; MLP: ask writes the fp16 image "
                         "the TMA-fed tcgen05 kernel reads). Default: on for c4, off otherwise")
    ap.add_argument("--write-x", type=int, default=None,
                    help="with --fused 1: also materialise the fp32 population x (default: 0 for "
                         "c4, whose fitness reads the fp16 parameter image the ask writes; 1 "
                         "otherwise)")
    ap.add_argument("--graph", type=int, default=None,
                    help="1: time replays of one generation captured as a CUDA graph "
                         "(default on for the launch-bound c1/c3)")
    ap.add_argument("--split", default="population", choices=["population", "dims"],
                    help="multi-GPU c1/c3: shard the population (P:226) or the dimensions "
                         "(f1 D-sharding: only R*N partial fitness doubles are all-reduced)")
    ap.add_argument("--p2p", type=int, default=0,
                    help="population-sharded configs: 1 = fused peer-memory tell (f2: CUDA IPC "
                         "peer mappings, one reduce-scatter/update/all-gather kernel) instead of "
                         "the NCCL all-reduce of the direction sums")
    ap.add_argument("--streams", type=int, default=1,
                    help="run independent handles (c2's two algorithms) on separate streams")
    ap.add_argument("--mlp", default="fp32", choices=["fp32", "fp16"],
                    help="c4 MLP fitness: fp32 = N14 (the definition, fp32-accurate kernel); "
                         "fp16 = N14' (the fp16-parameter-image approximation)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--sub", type=int, default=1,
                    help="c2: add the north_star_tell record (W=1) or the population-sharded "
                         "c5/c4 records (W>1)")
    ap.add_argument("--N", type=int, default=SWEEP["N"], help="c5 popsize")
    ap.add_argument("--D", type=int, default=SWEEP["D"], help="c5 dimensions")
    args = ap.parse_args()
    SWEEP.update(N=args.N, D=args.D)
    MLP_MODE["mode"] = args.mlp
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        # communicator creation logged (INIT subsystem only, on stderr) so the NCCL INIT lines show
        # every rank's nranks; algorithm and protocol pinned for run-to-run determinism of the
        # binary64 direction-sum all-reduce
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        os.environ.setdefault("NCCL_ALGO", "Ring")
        os.environ.setdefault("NCCL_PROTO", "Simple")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import __graft_entry__
    if rank == 0:
        __graft_entry__.build()
    if world > 1:
        dist.barrier()
    from paper_2212_04180_b200 import strategy as S

    peaks = load_peaks()
    stream = torch.cuda.current_stream()
    sharded = world > 1 and args.config != "c2"       # population sharding
    dsplit = sharded and args.split == "dims"
    if dsplit and args.config not in ("c1", "c3"):
        raise SystemExit("--split dims needs a separable BBOB config (c1, c3)")
    hs = []
    for label, cfg, params in handles_for(args.config, 0 if sharded else rank):
        es = S.Strategy(cfg["algo"], cfg["N"], cfg["D"], params,
                        group=dist.group.WORLD if sharded else None,
                        split="dims" if dsplit else "population")
        if sharded and not dsplit and args.p2p:
            es.p2p_connect(dist.group.WORLD)
        nl = es.local_popsize
        x = (torch.empty((cfg["R"], nl, es.x_dims), dtype=torch.float32, device="cuda")
             if cfg["fn"] is not None else None)
        f = torch.empty((cfg["R"], nl), dtype=torch.float32, device="cuda")
        es.params = params
        if cfg["fn"] in (W.MLP, W.MLP16):
            es.set_mlp_problem(cfg["widths"], cfg["batch"], cfg["data_seed"])
        hs.append((label, cfg, es, x, f))

    fused = bool(args.fused) if args.fused is not None else args.config == "c4"
    fused = fused or dsplit                       # a D-shard evaluates inside es_ask_eval
    write_x = bool(args.write_x) if args.write_x is not None else args.config != "c4"

    # independent handles (c2: the Sep-CMA-ES and the SNES batch) run on their own streams, so
    # one's kernels fill the other's wave-quantisation tails; the step joins them on `stream`
    hstreams = [torch.cuda.Stream() for _ in hs] if (len(hs) > 1 and args.streams) else None

    def one(cfg, es, x, f, st):
        with torch.cuda.stream(st):
            if cfg["fn"] is None:            # tell-only sweep: synthetic fitness stands in
                es.synth_fitness(out=f, stream=st)
            elif fused:
                es.ask_eval(cfg["fn"], out_x=x if write_x else None, out_f=f, write_x=write_x,
                            stream=st)
            else:
                es.ask(out=x, stream=st)
                es.eval(cfg["fn"], x, out=f, stream=st)
            es.tell(f, stream=st)

    mode = {"streams": hstreams}

    def step():
        if mode["streams"] is None:
            for _, cfg, es, x, f in hs:
                one(cfg, es, x, f, torch.cuda.current_stream())
            return
        cur = torch.cuda.current_stream()
        for (_, cfg, es, x, f), st in zip(hs, mode["streams"]):
            st.wait_stream(cur)
            one(cfg, es, x, f, st)
        for st in hstreams:
            cur.wait_stream(st)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    use_graph = args.graph if args.graph is not None else (args.config in ("c1", "c3", "c6")
                                                           and world == 1)
    graph = None
    if use_graph:
        # one generation captured once and replayed: the per-run scalars live on the device, so
        # replays advance t, lr, sigma exactly like eager calls (NCCL calls would be capturable too)
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(cs):
            step()
        torch.cuda.current_stream().wait_stream(cs)
        with torch.cuda.graph(graph, stream=cs, capture_error_mode="thread_local"):
            step()
        graph.replay()
        torch.cuda.synchronize()
    # profiled pass: per-kernel CUDA events (es_profile), handles serialised on one stream so that
    # every kernel's bracket holds only that kernel — these durations feed the roofline
    launches0 = sum(h[2].kernel_launches for h in hs)
    for h in hs:
        h[2].profile(True)
    mode["streams"] = None
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    mode["streams"] = hstreams
    launches = sum(h[2].kernel_launches for h in hs) - launches0
    prof = {}
    for label, cfg, es, _, _ in hs:
        for k, (t, n) in es.profile_read().items():
            prof.setdefault(k, []).append((label, cfg, t, n))
        es.profile(False)
    # timed pass: exactly K steps (graph replays, or eager with the handles on their streams)
    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)                     # the sampler is running before the timed region starts
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tw0 = time.time()
    e0.record(stream)
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            step()
    e1.record(stream)
    torch.cuda.synchronize()
    tw1 = time.time()
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        dist.barrier()
    clk = clocks.stop(tw0, tw1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())

    samples_per_step = sum(cfg["R"] * cfg["N"] * cfg["D"] for _, cfg, _, _, _ in hs) * \
        (1 if sharded else world)
    value = samples_per_step / (ms / 1e3)
    W_ = world if sharded else 1      # the work model below is per rank

    # --- roofline of the dominant kernel kind (algorithmic work / measured duration)
    pk_alu, pk_hbm = alu_peak(peaks), peaks["hbm_gbs"] * 1e9
    kinds = {}
    elite = {label: sum(math.floor(float(p["elite_ratio"]) * cfg["N"]) for p in es.params) /
             len(es.params) for label, cfg, es, _, _ in hs}
    for k, lst in prof.items():
        tot_ms = sum(t for _, _, t, _ in lst)
        ops = byt = flops = 0.0
        for label, cfg, t, n in lst:
            R, N, D, algo = cfg["R"], cfg["N"] // W_, cfg["D"], cfg["algo"]
            if dsplit:                                   # all members, this rank's dims
                N, D = cfg["N"], hs[0][2].x_dims
            P = N // 2 if algo in (W.OPENAI_ES, W.PGPE) else N          # this rank's directions
            if k == "ask":
                ops += n * R * P * D * (NORMAL_OPS + ASK_USE[algo])
                byt += n * (4.0 * R * N * D + 8.0 * R * D)
            elif k == "ask16":                 # ask + fp16 parameter image (N14′)
                ops += n * R * P * D * (NORMAL_OPS + ASK_USE[algo])
                byt += n * ((4.0 if write_x else 0.0) * R * N * D + 2.0 * R * N * D + 8.0 * R * D)
            elif k == "ask_eval":
                ops += n * (R * P * D * (NORMAL_OPS + ASK_USE[algo]) +
                            R * N * D * EVAL_OPS[cfg["fn"]])
                byt += n * (4.0 * R * N * D + 8.0 * R * D)
            elif k == "eval_bbob":
                byt += n * (4.0 * R * N * D + 4.0 * R * N)
            elif k in ("tell", "tell_reduce"):
                # Sep-CMA regenerates only the mu weighted members (no ties in continuous fitness)
                E = elite[label] / (1 if dsplit else W_) if algo == W.SEP_CMA_ES else P
                ops += n * R * E * D * (NORMAL_OPS + TELL_USE[algo])
                byt += n * R * D * STATE_BYTES[algo]
            elif k == "cma_ask":                # z (N2) + y = A z (triangular FFMA) + x epilogue
                ops += n * R * N * D * (NORMAL_OPS / 1.0 + D / 2.0 + 1.0)
                byt += n * (12.0 * R * N * D + 2.0 * R * D * D)
            elif k == "cma_tell":               # ȳ, z̄ + rank-μ (lower) + Cholesky (D³/6 FFMA)
                mu = elite[label]
                ops += n * R * (2.0 * mu * D + mu * D * D / 2.0 + D ** 3 / 6.0)
                byt += n * R * (8.0 * mu * D + 12.0 * D * D)
            elif k == "rank":
                byt += n * R * cfg["N"] * 40.0
            elif k in ("eval_mlp", "eval_mlp16"):
                # N14 reads the fp32 parameters; N14' the fp16 image when fused
                byt += n * ((2.0 if fused and k == "eval_mlp16" else 4.0) * R * N * D + 4.0 * R * N)
                wd = cfg["widths"]
                flops += n * R * N * 2.0 * cfg["batch"] * sum(wd[i] * wd[i + 1]
                                                              for i in range(len(wd) - 1))
        kinds[k] = dict(ms=tot_ms, ops=ops, bytes=byt, flops=flops,
                        launches=sum(n for _, _, _, n in lst))
    dom = max(kinds, key=lambda k: kinds[k]["ms"])
    d = kinds[dom]
    secs = d["ms"] / 1e3
    t_alu, t_hbm = d["ops"] / pk_alu, d["bytes"] / pk_hbm
    t_tc = d["flops"] / (peaks["bf16_tflops"] * 1e12)
    if t_tc > max(t_alu, t_hbm):
        achieved = d["flops"] / secs / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": peaks["bf16_tflops"],
                "unit": "TFLOP/s", "frac": achieved / peaks["bf16_tflops"]}
    elif t_alu >= t_hbm:
        achieved = d["ops"] / secs / 1e12
        roof = {"bound": "alu", "achieved": achieved, "peak": pk_alu / 1e12,
                "unit": "Tlane-op/s", "frac": achieved / (pk_alu / 1e12)}
    else:
        achieved = d["bytes"] / secs / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": achieved / peaks["hbm_gbs"]}
    src = peaks["src"]
    if roof["bound"] == "alu":   # derived, not measured: unit counts x the max SM clock
        src = (f"derived: 148 SMs x 4 SMSPs x 32 lanes x {peaks['sm_max_mhz']:.0f} MHz "
               f"(clock from MEASURED_PEAKS.json)" if src == "measured" else
               "derived: 148 SMs x 4 SMSPs x 32 lanes x 1965 MHz (B200_PROFILING.md)")
    roof.update(kernel=dom, launches=d["launches"], peak_source=src,
                traffic=ncu_traffic(args.config, dom))
    extra = {}
    for k, v in kinds.items():
        if v["ms"] > 0:
            extra[k] = {"GB/s": round(v["bytes"] / (v["ms"] / 1e3) / 1e9, 1),
                        "Tlane-op/s": round(v["ops"] / (v["ms"] / 1e3) / 1e12, 2),
                        "TFLOP/s": round(v["flops"] / (v["ms"] / 1e3) / 1e12, 1)}
    tot_k = sum(v["ms"] for v in kinds.values()) or 1.0
    share = {k: round(v["ms"] / tot_k, 4) for k, v in kinds.items()}   # of the serialised pass
    kernels_ms = {k: round(v["ms"] / max(v["launches"], 1), 4) for k, v in kinds.items()}
    by_handle = {}
    for k, lst in prof.items():
        for label, _, t, n in lst:
            by_handle.setdefault(label, {})[k] = round(t / max(n, 1), 4)

    # --- end to end through the C ABI with HOST buffers (fitness read back and fed to tell)
    e2e = e2e_run(hs, args, 1 if sharded else world, fused, write_x)

    cb = config_block(args.config, world)
    if dsplit:
        cb["parallelism"] = f"dimensions sharded x{world} (R*N partial-fitness all-reduce only)"
    elif sharded and args.p2p:
        cb["parallelism"] = f"population sharded x{world}, fused peer-memory tell (f2)"
    if hs[0][1]["fn"] is None:
        cb["path"] = "synthetic fitness, tell"
    elif fused and hs[0][1]["fn"] == W.MLP16:
        cb["path"] = ("es_ask_eval: ask writes " + ("x and " if write_x else "") +
                      "the fp16 parameter image (N14', a labelled approximation of N14), "
                      "TMA-fed tcgen05 MLP fitness, then tell")
    elif fused and hs[0][1]["fn"] == W.MLP:
        cb["path"] = ("es_ask_eval: the ask writes the population's split binary16 image (N14: hi "
                      "and lo parts of x*2^8" + (", and x" if write_x else "; x not materialised") +
                      "), the fp32-accurate tcgen05 MLP fitness streams it (2-CTA pair MMAs, three "
                      "products summed in TMEM), then tell")
    elif fused:
        cb["path"] = "fused ask+evaluate kernel" + (" (x written)" if write_x else "") + ", tell"
    else:
        cb["path"] = "ask, evaluate, tell kernels"
    line = {"metric": metric_name(args.config), "value": value, "unit": "samples/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong" if sharded else "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic", "config": cb,
            "generations_per_s": 1e3 / ms, "roofline": roof, "e2e": e2e,
            "gpu_launches": launches, "clocks": clk, "kernel_share": share,
            "kernel_ms_per_launch": kernels_ms, "kernel_ms_by_handle": by_handle,
            "kernel_rates": extra,
            "timing": "CUDA-graph replays of one generation" if graph is not None else
                      "eager C-ABI calls, CUDA events on the stream"}
    for h in hs:
        h[2].close()
    hs = []
    if args.config == "c2" and args.sub:
        if world == 1:
            # the north star's own target (fused tell >= 70 % of the ALU roofline at D ~ 1e6,
            # N = 4096) measured under the same clock as the headline
            line["north_star_tell"] = sub_bench("c5", 1, False, 10, peaks)
        else:
            # the path north_star scales: one population sharded over the ranks
            line["sharded"] = {"c5": sub_bench("c5", world, True, 10, peaks, dist.group.WORLD),
                               "c4": sub_bench("c4", world, True, 3, peaks, dist.group.WORLD),
                               "nccl": {k: os.environ.get(k) for k in
                                        ("NCCL_ALGO", "NCCL_PROTO", "NCCL_DEBUG_SUBSYS")}}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args.config, args.cpu_budget)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def ncu_traffic(cfg_key, kernel):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(cfg_key, {}).get(kernel)


def e2e_run(hs, args, world, fused=False, write_x=True):
    """Same metric through the public API with host buffers: per step and handle, ask on the
    device, evaluate, copy the fitness into PINNED HOST memory (D2H), tell from that host buffer
    (H2D), and read best_fitness back (D2H)."""
    import torch
    fh = [torch.empty((cfg["R"], es.local_popsize), dtype=torch.float32).pin_memory()
          for _, cfg, es, _, _ in hs]
    fd = [torch.empty((cfg["R"], es.local_popsize), dtype=torch.float32, device="cuda")
          for _, cfg, es, _, _ in hs]
    bh = [torch.empty(cfg["R"], dtype=torch.float32).pin_memory() for _, cfg, _, _, _ in hs]
    from paper_2212_04180_b200._lib import check, lib
    import ctypes as C

    # independent handles on their own streams (as a user driving two batches would): every
    # handle's ask, evaluation and fitness D2H copy (cudaMemcpyAsync into pinned memory) is
    # queued first; then, handle by handle, the host waits for that handle's copy and tells from
    # the host buffer (the library's H2D), so the GPU queue never drains while the host waits;
    # best_fitness last
    streams = [torch.cuda.Stream() for _ in hs] if len(hs) > 1 else [torch.cuda.current_stream()]
    ss = [C.c_void_p(st.cuda_stream) for st in streams]
    evs = [torch.cuda.Event() for _ in hs]

    def step():
        for (label, cfg, es, x, _), f, d, s, st, ev in zip(hs, fh, fd, ss, streams, evs):
            n = cfg["R"] * es.local_popsize
            if cfg["fn"] is None:
                check(lib().es_synth_fitness(es.ctx, C.c_void_p(d.data_ptr()), s), es.ctx)
            elif fused:
                check(lib().es_ask_eval(es.ctx, cfg["fn"],
                                        C.c_void_p(x.data_ptr()) if write_x else None,
                                        C.c_void_p(d.data_ptr()), s), es.ctx)
            else:
                es.ask(out=x, stream=st)
                check(lib().es_eval_bbob(es.ctx, cfg["fn"], C.c_void_p(x.data_ptr()), n,
                                         cfg["D"], C.c_void_p(d.data_ptr()), s), es.ctx)
            with torch.cuda.stream(st):
                f.copy_(d, non_blocking=True)                  # D2H into pinned host memory
                ev.record(st)
        for (label, cfg, es, x, _), f, s, ev in zip(hs, fh, ss, evs):
            ev.synchronize()                                   # this handle's fitness on the host
            check(lib().es_tell(es.ctx, C.c_void_p(f.data_ptr()), s), es.ctx)
        for (label, cfg, es, x, _), b, s in zip(hs, bh, ss):
            check(lib().es_get(es.ctx, 8, C.c_void_p(b.data_ptr()), s), es.ctx)

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    steps = max(3, args.steps // 2)
    t0 = time.perf_counter()
    for _ in range(steps):
        step()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([dt], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t.item())
    samples = sum(cfg["R"] * cfg["N"] * cfg["D"] for _, cfg, _, _, _ in hs) * world
    return {"value": samples / dt, "unit": "samples/s", "ms_per_step": dt * 1e3,
            "h2d_bytes_per_step": sum(4 * cfg["R"] * es.local_popsize for _, cfg, es, _, _ in hs),
            "d2h_bytes_per_step": sum(4 * cfg["R"] * es.local_popsize + 4 * cfg["R"]
                                      for _, cfg, es, _, _ in hs),
            "timing": "host wall clock (host syncs are part of the API path)"}


if __name__ == "__main__":
    sys.exit(main())
