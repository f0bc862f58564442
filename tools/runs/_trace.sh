mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2212_04180_b200/lib/libes_b200.so /tmp/keep.so
cp exp/libes_trace.so paper_2212_04180_b200/lib/libes_b200.so
timeout 300 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/trace_c4.log 2>&1; echo rc=$?
cp /tmp/keep.so paper_2212_04180_b200/lib/libes_b200.so
grep "mlp32 trace" gpurun_out/trace_c4.log | tail -12
