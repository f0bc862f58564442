python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "rank or shap or sep or snes or tell" > /tmp/t.log 2>&1; echo tests rc=$?; tail -1 /tmp/t.log; grep -E "^FAILED" /tmp/t.log | head -3
for p in 1 0 1 0; do
ES_COUNT_MANY=$p timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > /tmp/o.log 2>&1; echo "many=$p rc=$?"
tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))'
done
