mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2j_build.log 2>&1 || { tail gpurun_out/r2j_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -x -k "rank or eval or generation or rastrigin" > gpurun_out/r2j_tests.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/r2j_tests.log
for c in "--steps 20 --warmup 5 --no-cpu-baseline --sub 0" "--config c3 --steps 50 --warmup 5 --no-cpu-baseline" "--config c4 --steps 3 --warmup 3 --no-cpu-baseline --mlp fp16"; do
  timeout 600 python bench.py $c > /tmp/o.log 2>&1; echo "bench $c rc=$?"
  tail -1 /tmp/o.log >> gpurun_out/r2j_bench.jsonl
  tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), json.dumps(d.get("kernel_ms_by_handle")))'
done
python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mlp32_kernel|mlp_kernel" -c 1 -o gpurun_out/r2j_mlp32 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_ncu32.log 2>&1; echo ncu32 rc=$?
python bench.py --config c4 --mlp fp16 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_plain16.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mlp_kernel" -c 1 -o gpurun_out/r2j_mlp16 python bench.py --config c4 --mlp fp16 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_ncu16.log 2>&1; echo ncu16 rc=$?
