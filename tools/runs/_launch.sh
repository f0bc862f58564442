mkdir -p gpurun_out
T=${TAG:-r2t}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python -m pytest tests -m gpu -q -x -k "mlp" > gpurun_out/${T}_tests_mlp.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/${T}_tests_mlp.log
for c in c3 c5 c1; do
timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_plain_$c.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_$c.log 2>&1; echo ncu $c rc=$?
done
for c in "--config c4 --steps 3 --warmup 3 --no-cpu-baseline" "--config c4 --steps 3 --warmup 3 --no-cpu-baseline --mlp fp16"; do
  timeout 300 python bench.py $c > /tmp/o.log 2>&1; echo "bench $c rc=$?"
  tail -1 /tmp/o.log >> gpurun_out/${T}_bench.jsonl
  tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), d["roofline"]["kernel"], round(d["roofline"]["frac"],3), json.dumps(d.get("kernel_ms_by_handle")))'
done
