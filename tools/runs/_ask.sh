python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "ask" > /tmp/t.log 2>&1; echo tests rc=$?; tail -1 /tmp/t.log
for c in "--steps 20 --warmup 5 --no-cpu-baseline" "--config c4 --mlp fp16 --steps 3 --warmup 3 --no-cpu-baseline"; do
  timeout 300 python bench.py $c > /tmp/o.log 2>&1; echo "bench $c rc=$?"
  tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), d["roofline"]["kernel"], round(d["roofline"]["frac"],4), json.dumps(d.get("kernel_ms_by_handle")))'
done
