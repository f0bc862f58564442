mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2212_04180_b200/lib/libes_b200.so /tmp/keep.so
cp exp/libes_rtrace.so paper_2212_04180_b200/lib/libes_b200.so
ES_RADIX_MIN_N=2 timeout 120 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/rtrace_c3.log 2>&1; echo rc=$?
timeout 120 python bench.py --config c5 --N 65536 --D 1000 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/rtrace_c5.log 2>&1; echo rc=$?
cp /tmp/keep.so paper_2212_04180_b200/lib/libes_b200.so
grep "radix trace" gpurun_out/rtrace_c3.log | tail -2
grep "radix trace" gpurun_out/rtrace_c5.log | tail -2; grep "radix cta" gpurun_out/rtrace_c5.log | tail -32 | sort -k5 -n | tail -6
