python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "ask_eval or dshard or weight_decay or fused" > /tmp/t.log 2>&1; echo tests rc=$?; tail -2 /tmp/t.log; grep -E "^FAILED|Error" /tmp/t.log | head -5
for a in "--fused 1" "--fused 1 --write-x 0" "--config c3 --fused 1" "--config c3 --fused 1 --write-x 0"; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline $a > /tmp/o.log 2>&1; echo "bench [$a] rc=$?"
  tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), json.dumps(d.get("kernel_ms_by_handle")))'
done
