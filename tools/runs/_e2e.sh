python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for a in "" "--config c5" "--config c3" "--config c4"; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline $a > /tmp/o.log 2>&1; echo "bench [$a] rc=$?"
  tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("e2e")))'
done
