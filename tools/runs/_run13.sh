mkdir -p gpurun_out
T=${TAG:-r2ag}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
timeout 240 python -m pytest tests -m gpu -q -x -k "rank" > gpurun_out/${T}_t1.log 2>&1; rc=$?; echo rank tests rc=$rc; tail -2 gpurun_out/${T}_t1.log; grep -E "^FAILED|Error" gpurun_out/${T}_t1.log | head -5
if [ $rc -ne 0 ]; then exit 1; fi
timeout 900 python -m pytest tests -m gpu -q -k "generation or sweep or c5 or tell or sharded or nccl or graph" > gpurun_out/${T}_t2.log 2>&1; echo tests rc=$?; tail -2 gpurun_out/${T}_t2.log; grep -E "^FAILED|Error" gpurun_out/${T}_t2.log | head -5
for nn in 4096 8200 16384 40000 65536; do
  timeout 200 python bench.py --config c5 --N $nn --D 10000 --steps 10 --warmup 3 --no-cpu-baseline > /tmp/o.log 2>&1
  echo "c5 N=$nn D=1e4: $(tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))')"
done
timeout 300 python bench.py --config c5 --N 65536 --D 10000 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launch_rank.csv python bench.py --config c5 --N 65536 --D 10000 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo launch rc=$?
for nn in 1024 4096; do
  ES_RADIX_MIN_N=2 timeout 200 python bench.py --config c5 --N $nn --D 10000 --steps 10 --warmup 3 --no-cpu-baseline > /tmp/o.log 2>&1
  echo "radix c5 N=$nn D=1e4: $(tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))')"
done
ES_RADIX_MIN_N=2 timeout 200 python bench.py --config c3 --steps 50 --warmup 5 --no-cpu-baseline > /tmp/o.log 2>&1
echo "radix c3: $(tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))')"
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2212_04180_b200/lib/libes_b200.so /tmp/keep.so
cp exp/libes_rtrace.so paper_2212_04180_b200/lib/libes_b200.so
ES_RADIX_MIN_N=2 timeout 120 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/rtrace_c3.log 2>&1; echo rc=$?
timeout 120 python bench.py --config c5 --N 65536 --D 1000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/rtrace_c5.log 2>&1; echo rc=$?
cp /tmp/keep.so paper_2212_04180_b200/lib/libes_b200.so
grep "radix trace" gpurun_out/rtrace_c3.log | tail -2
grep "radix trace" gpurun_out/rtrace_c5.log | tail -2; grep "radix cta" gpurun_out/rtrace_c5.log | tail -32 | sort -k5 -n | tail -6
