python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
ES_EVAL_2ROWS=1 timeout 600 python -m pytest tests -m gpu -q -x -k "eval or bbob" > /tmp/t.log 2>&1; echo tests rc=$?; tail -1 /tmp/t.log
for p in 1 0 1 0; do
ES_EVAL_2ROWS=$p timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > /tmp/o.log 2>&1
echo "2rows=$p $(tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))')"
done
