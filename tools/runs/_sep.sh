python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "sep or cma or p2p or ipc or dshard" > /tmp/t.log 2>&1; echo tests rc=$?; tail -1 /tmp/t.log; grep -E "^FAILED" /tmp/t.log | head -3
for i in 1 2; do
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > /tmp/o.log 2>&1; echo "bench rc=$?"
tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))'
done
