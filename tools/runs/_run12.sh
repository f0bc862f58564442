mkdir -p gpurun_out
T=${TAG:-r2ab}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
timeout 400 python -m pytest tests -m gpu -q -x -k "mlp or tanh" > gpurun_out/${T}_tests_mlp.log 2>&1; echo tests rc=$?; tail -1 gpurun_out/${T}_tests_mlp.log
cp paper_2212_04180_b200/lib/libes_b200.so /tmp/keep.so
for v in default a0; do
  if [ $v != default ]; then cp exp/libes_$v.so paper_2212_04180_b200/lib/libes_b200.so; fi
  for c in "--config c4 --steps 3 --warmup 3 --no-cpu-baseline" "--config c4 --steps 3 --warmup 3 --no-cpu-baseline --mlp fp16"; do
    timeout 200 python bench.py $c > /tmp/o.log 2>&1
    echo "$v $c: $(tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))')"
  done
  cp /tmp/keep.so paper_2212_04180_b200/lib/libes_b200.so
done
for nn in 4096 16384 65536; do
  timeout 200 python bench.py --config c5 --N $nn --D 10000 --steps 10 --warmup 3 --no-cpu-baseline > /tmp/o.log 2>&1
  echo "c5 N=$nn D=1e4: $(tail -1 /tmp/o.log | python -c 'import json,sys; d=json.load(sys.stdin); print(round(d["ms_per_step"],4), json.dumps(d.get("kernel_ms_by_handle")))')"
done
timeout 300 python bench.py --config c5 --N 4096 --D 10000 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launch_rank.csv python bench.py --config c5 --N 65536 --D 10000 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo launch rc=$?
