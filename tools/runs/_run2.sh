mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2i_build.log 2>&1 || { tail gpurun_out/r2i_build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -q --maxfail=20 > gpurun_out/r2i_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/r2i_tests.log
grep -E "^FAILED|^ERROR" gpurun_out/r2i_tests.log | head -20
for c in "--steps 20 --warmup 5 --no-cpu-baseline" "--config c5 --steps 10 --warmup 3 --no-cpu-baseline" "--config c3 --steps 50 --warmup 5 --no-cpu-baseline" "--config c1 --steps 50 --warmup 5 --no-cpu-baseline"; do
  timeout 600 python bench.py $c > /tmp/o.log 2>&1; echo "bench $c rc=$?"
  tail -1 /tmp/o.log >> gpurun_out/r2i_bench.jsonl
  tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), json.dumps(d.get("kernel_ms_by_handle")))'
done
