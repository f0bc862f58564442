python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "rank or shap" > /tmp/t.log 2>&1; echo tests-default rc=$?; tail -1 /tmp/t.log; grep -E "^FAILED" /tmp/t.log | head -3
ES_RADIX_MIN_N=2 timeout 600 python -m pytest tests -m gpu -q -x -k "rank or shap" > /tmp/t2.log 2>&1; echo tests-radix rc=$?; tail -1 /tmp/t2.log; grep -E "^FAILED" /tmp/t2.log | head -3
for N in 256 1024 2048 4096 8192 16384; do
  for m in 4097 2; do
    ES_RADIX_MIN_N=$m timeout 120 python bench.py --config c5 --N $N --D 10000 --steps 20 --warmup 3 --no-cpu-baseline --graph 1 > /tmp/o.log 2>&1
    echo "N=$N min=$m $(tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))' 2>&1 | tail -1)"
  done
done
