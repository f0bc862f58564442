mkdir -p gpurun_out
T=${TAG:-r2bk}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
timeout 400 python -m pytest tests -m gpu -q -x -k "eval or bbob or fitness or rosen" > gpurun_out/${T}_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${T}_tests.log; grep -E "^FAILED|Error" gpurun_out/${T}_tests.log | head
for c in "--steps 20 --warmup 5 --no-cpu-baseline" "--config c3 --steps 50 --warmup 5 --no-cpu-baseline" "--config c1 --steps 50 --warmup 5 --no-cpu-baseline"; do
  timeout 300 python bench.py $c > /tmp/o.log 2>&1; echo "bench $c rc=$?"
  tail -1 /tmp/o.log >> gpurun_out/${T}_bench.jsonl
  tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), json.dumps(d.get("kernel_ms_by_handle")))'
done
