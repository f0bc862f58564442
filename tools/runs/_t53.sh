python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "tanh or mlp" > /tmp/t.log 2>&1; echo tests rc=$?; tail -1 /tmp/t.log; grep -E "^FAILED|assert rel" -A3 /tmp/t.log | head -8
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > /tmp/o.log 2>&1; tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))'
