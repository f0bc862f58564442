python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for p in 0 1 2 0 1 2; do
ES_BENCH_PRIO=$p timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline > /tmp/o.log 2>&1; echo "prio=$p rc=$?"
tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4))'
done
