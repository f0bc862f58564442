mkdir -p gpurun_out
T=${TAG:-r2o}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
timeout 300 python -m pytest tests -m gpu -q -x -k "mlp or tanh" > gpurun_out/${T}_tests_mlp.log 2>&1; echo mlp tests rc=$?; tail -2 gpurun_out/${T}_tests_mlp.log; grep -E "^FAILED|Error" gpurun_out/${T}_tests_mlp.log | head
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > /tmp/o.log 2>&1; echo "bench c4 rc=$?"
tail -1 /tmp/o.log >> gpurun_out/${T}_bench.jsonl
tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), json.dumps(d.get("kernel_ms_by_handle")))'
cp paper_2212_04180_b200/lib/libes_b200.so /tmp/keep.so
cp exp/libes_trace.so paper_2212_04180_b200/lib/libes_b200.so
timeout 300 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_trace_c4.log 2>&1; echo trace rc=$?
cp /tmp/keep.so paper_2212_04180_b200/lib/libes_b200.so
grep "mlp32 trace" gpurun_out/${T}_trace_c4.log | tail -4
timeout 300 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline --mlp fp16 > /tmp/o.log 2>&1; echo "bench c4 fp16 rc=$?"
tail -1 /tmp/o.log >> gpurun_out/${T}_bench.jsonl
tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), json.dumps(d.get("kernel_ms_by_handle")))'
