mkdir -p gpurun_out
T=${TAG:-r2l}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
timeout 300 python -m pytest tests -m gpu -q -x -k "mlp or tanh" > gpurun_out/${T}_tests_mlp.log 2>&1; echo mlp tests rc=$?; tail -2 gpurun_out/${T}_tests_mlp.log; grep -E "^FAILED|Error" gpurun_out/${T}_tests_mlp.log | head
timeout 1200 python -m pytest tests -m gpu -q --maxfail=10 -k "not mlp" > gpurun_out/${T}_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${T}_tests.log; grep -E "^FAILED|Error" gpurun_out/${T}_tests.log | head
for c in "--steps 20 --warmup 5 --no-cpu-baseline --sub 0" "--config c5 --steps 10 --warmup 3 --no-cpu-baseline" "--config c4 --steps 3 --warmup 3 --no-cpu-baseline" "--config c4 --steps 3 --warmup 3 --no-cpu-baseline --mlp fp16"; do
  timeout 300 python bench.py $c > /tmp/o.log 2>&1; echo "bench $c rc=$?"
  tail -1 /tmp/o.log >> gpurun_out/${T}_bench.jsonl
  tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), json.dumps(d.get("kernel_ms_by_handle")))'
done
timeout 300 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_plain4.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mlp32_kernel" -s 1 -c 1 -o gpurun_out/${T}_mlp32 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu32.log 2>&1; echo ncu32 rc=$?
timeout 300 python bench.py --config c4 --mlp fp16 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_plain16.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mlp_kernel" -s 1 -c 1 -o gpurun_out/${T}_mlp16 python bench.py --config c4 --mlp fp16 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu16.log 2>&1; echo ncu16 rc=$?
