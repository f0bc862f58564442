mkdir -p gpurun_out
T=${TAG:-r2ai}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
timeout 300 python -m pytest tests -m gpu -q -x -k "mlp or tanh" > gpurun_out/${T}_t1.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/${T}_t1.log; grep -E "^FAILED|Error" gpurun_out/${T}_t1.log | head -5
for c in "--config c4 --steps 5 --warmup 3 --no-cpu-baseline --mlp fp16" "--config c4 --steps 5 --warmup 3 --no-cpu-baseline" "--config c3 --steps 50 --warmup 5 --no-cpu-baseline" "--config c1 --steps 50 --warmup 5 --no-cpu-baseline"; do
  timeout 200 python bench.py $c > /tmp/o.log 2>&1
  echo "$c: $(tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))')"
done
