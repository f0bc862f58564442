python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2212_04180_b200/lib/libes_b200.so /tmp/keep.so
for v in base oes10 oes12 base oes10; do
  if [ $v != base ]; then cp exp/libes_$v.so paper_2212_04180_b200/lib/libes_b200.so; else cp /tmp/keep.so paper_2212_04180_b200/lib/libes_b200.so; fi
  timeout 300 python bench.py --config c5 --steps 10 --warmup 3 --no-cpu-baseline > /tmp/o.log 2>&1
  echo "$v c5 $(tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), round(d["roofline"]["frac"],4))')"
done
for v in base ahead2 base ahead2; do
  if [ $v != base ]; then cp exp/libes_$v.so paper_2212_04180_b200/lib/libes_b200.so; else cp /tmp/keep.so paper_2212_04180_b200/lib/libes_b200.so; fi
  timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > /tmp/o.log 2>&1
  echo "$v c4 $(tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))')"
done
cp /tmp/keep.so paper_2212_04180_b200/lib/libes_b200.so
