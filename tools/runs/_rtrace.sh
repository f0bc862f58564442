python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
cp paper_2212_04180_b200/lib/libes_b200.so /tmp/keep.so; cp exp/libes_rtrace.so paper_2212_04180_b200/lib/libes_b200.so
timeout 120 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline --graph 0 2>&1 | grep "rank trace" | tail -3
timeout 120 python bench.py --config c1 --steps 3 --warmup 3 --no-cpu-baseline --graph 0 2>&1 | grep "rank trace" | tail -3
cp /tmp/keep.so paper_2212_04180_b200/lib/libes_b200.so
