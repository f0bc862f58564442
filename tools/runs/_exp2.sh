mkdir -p gpurun_out
T=${TAG:-r2ao}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
for v in normal bulk normal bulk; do
  cp paper_2212_04180_b200/lib/libes_b200.so /tmp/keep.so
  [ $v = bulk ] && cp exp/libes_bulk.so paper_2212_04180_b200/lib/libes_b200.so
  timeout 200 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > /tmp/o.log 2>&1; echo "bench c4 $v rc=$?"
  cp /tmp/keep.so paper_2212_04180_b200/lib/libes_b200.so
  tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))'
done
