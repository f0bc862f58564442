"""Config-5 sweep: OpenAI-ES tell throughput over popsize x dimension (BASELINE.json configs[4]).
Runs bench.py --config c5 per cell (on the GPU box) and writes profiles/<tag>_c5_sweep.{json,md}."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TAG = sys.argv[1] if len(sys.argv) > 1 else "sweep"
NS = [256, 1024, 4096, 16384, 65536]
DS = [1_000, 10_000, 100_000, 1_000_000, 10_000_000]
rows = []
for N in NS:
    for D in DS:
        work = N // 2 * D
        steps = max(3, min(30, int(4e10 / work)))
        cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "c5", "--N", str(N),
               "--D", str(D), "--steps", str(steps), "--warmup", "3", "--no-cpu-baseline",
               "--graph", "1"]
        out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT)
        try:
            d = json.loads(out.stdout.strip().splitlines()[-1])
        except Exception:
            rows.append(dict(N=N, D=D, error=(out.stderr or out.stdout)[-400:]))
            print(N, D, "ERROR", file=sys.stderr)
            continue
        tell = d["kernel_ms_per_launch"].get("tell")
        rows.append(dict(N=N, D=D, ms_per_gen=d["ms_per_step"], tell_ms=tell,
                         gens_per_s=d["generations_per_s"], samples_per_s=d["value"],
                         normals_per_s=(N // 2) * D / (tell / 1e3) if tell else None,
                         alu_frac=d["kernel_rates"].get("tell", {}).get("Tlane-op/s", 0) /
                         d["roofline"]["peak"] if d["roofline"]["bound"] == "alu" else None,
                         clocks=d.get("clocks")))
        print(N, D, rows[-1]["ms_per_gen"], rows[-1]["alu_frac"], file=sys.stderr, flush=True)
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(rows, open(os.path.join(ROOT, "gpurun_out", f"{TAG}_c5_sweep.json"), "w"), indent=1)
with open(os.path.join(ROOT, "gpurun_out", f"{TAG}_c5_sweep.md"), "w") as f:
    f.write("| N \\\\ D | " + " | ".join(f"{D:.0e}" for D in DS) + " |\n")
    f.write("|---" * (len(DS) + 1) + "|\n")
    for N in NS:
        cells = []
        for D in DS:
            r = next(x for x in rows if x["N"] == N and x["D"] == D)
            if "error" in r:
                cells.append("err")
            else:
                fr = f"{100 * r['alu_frac']:.0f}%" if r["alu_frac"] else "-"
                cells.append(f"{r['ms_per_gen']:.3g} ms ({fr})")
        f.write(f"| {N} | " + " | ".join(cells) + " |\n")
