mkdir -p gpurun_out
T=${TAG:-r2final5}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench_default.log 2>&1; echo bench default rc=$?; tail -1 gpurun_out/${T}_bench_default.log | cut -c1-300
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref.log 2>&1; echo bench ref rc=$?; tail -1 gpurun_out/${T}_bench_ref.log | cut -c1-200
for c in c1 c3 c5 c4 c6; do
  timeout 600 python bench.py --config $c --no-cpu-baseline > gpurun_out/${T}_bench_$c.log 2>&1; echo "bench $c rc=$?"
  tail -1 gpurun_out/${T}_bench_$c.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), json.dumps(d.get("kernel_ms_by_handle")))'
done
timeout 600 python bench.py --config c4 --mlp fp16 --no-cpu-baseline > gpurun_out/${T}_bench_c4fp16.log 2>&1; echo "bench c4 fp16 rc=$?"
tail -1 gpurun_out/${T}_bench_c4fp16.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))'
TAG=$T bash tools/runs/_prof_final.sh
