mkdir -p gpurun_out
T=${TAG:-r2bg}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "not mlp and not cma" > gpurun_out/${T}_tests.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/${T}_tests.log; grep -E "^FAILED|Error" gpurun_out/${T}_tests.log | head -5
for p in 1 0; do
for c in "--steps 20 --warmup 5 --no-cpu-baseline" "--config c3 --steps 50 --warmup 5 --no-cpu-baseline" "--config c1 --steps 50 --warmup 5 --no-cpu-baseline"; do
  ES_RANK_IN_TELL=$p timeout 300 python bench.py $c > /tmp/o.log 2>&1; echo "RIT=$p bench $c rc=$?"
  tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))'
done; done
