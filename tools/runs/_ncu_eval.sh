mkdir -p gpurun_out
T=${TAG:-r2av}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"eval_" -s 3 -c 1 -o gpurun_out/${T}_c3eval python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu.log 2>&1; echo ncu rc=$?
