mkdir -p gpurun_out
T=${TAG:-r2aq}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${T}_build.log 2>&1 || { tail gpurun_out/${T}_build.log; exit 1; }
cp paper_2212_04180_b200/lib/libes_b200.so /tmp/keep.so
cp exp/libes_trace.so paper_2212_04180_b200/lib/libes_b200.so
timeout 120 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_trace_c4.log 2>&1; echo trace rc=$?
timeout 120 python bench.py --config c4 --mlp fp16 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_trace_c4_16.log 2>&1; echo trace16 rc=$?
cp /tmp/keep.so paper_2212_04180_b200/lib/libes_b200.so
grep "trace" gpurun_out/${T}_trace_c4.log | tail -6
grep "trace" gpurun_out/${T}_trace_c4_16.log | tail -6
