mkdir -p gpurun_out
T=${TAG:-r2as}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python bench.py --config c3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_plain_c3.log 2>&1; echo plain rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c3.csv python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_launch_c3.log 2>&1; echo launch rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -s 20 -c 12 -o gpurun_out/${T}_c3 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_c3.log 2>&1; echo ncu rc=$?
