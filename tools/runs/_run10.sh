mkdir -p gpurun_out
T=${TAG:-r2am}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
timeout 240 python -m pytest tests -m gpu -q -x -k "mlp_fitness_parity" > gpurun_out/${T}_t1.log 2>&1; rc=$?; echo t1 rc=$rc; tail -3 gpurun_out/${T}_t1.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 400 python -m pytest tests -m gpu -q -x -k "mlp or tanh" > gpurun_out/${T}_tests_mlp.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${T}_tests_mlp.log; grep -E "^FAILED|Error" gpurun_out/${T}_tests_mlp.log | head
cp paper_2212_04180_b200/lib/libes_b200.so /tmp/keep.so
cp exp/libes_trace.so paper_2212_04180_b200/lib/libes_b200.so
timeout 120 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_trace_c4.log 2>&1; echo trace rc=$?
cp /tmp/keep.so paper_2212_04180_b200/lib/libes_b200.so
grep "mlp32 trace" gpurun_out/${T}_trace_c4.log | tail -4
timeout 200 python bench.py --config c4 --steps 3 --warmup 3 --no-cpu-baseline > /tmp/o.log 2>&1; echo "bench c4 rc=$?"
tail -1 /tmp/o.log >> gpurun_out/${T}_bench.jsonl
tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), json.dumps(d.get("kernel_ms_by_handle")))'
timeout 200 python bench.py --config c4 --mlp fp16 --steps 3 --warmup 3 --no-cpu-baseline > /tmp/o.log 2>&1; echo "bench c4 fp16 rc=$?"
tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))'
