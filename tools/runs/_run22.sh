mkdir -p gpurun_out
T=${TAG:-r2be}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "mlp or tanh or ask or fused or clip or bound" > gpurun_out/${T}_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/${T}_tests.log; grep -E "^FAILED" gpurun_out/${T}_tests.log | head
for a in "--config c4"; do
  timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline $a > /tmp/o.log 2>&1; echo "bench [$a] rc=$?"
  tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))'
done
