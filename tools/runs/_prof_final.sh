mkdir -p gpurun_out
T=${TAG:-r2final2}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sub 0 > gpurun_out/${T}_plain_c2.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --sub 0 > gpurun_out/${T}_ncu_launch_c2.log 2>&1; echo launch c2 rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"ask_kernel|eval_warp|tell_kernel|rank_kernel|sepcma" -c 9 -o gpurun_out/${T}_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --sub 0 > gpurun_out/${T}_ncu_c2.log 2>&1; echo ncu c2 rc=$?
timeout 300 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_plain4.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"mlp32_kernel|ask_kernel" -s 2 -c 2 -o gpurun_out/${T}_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_c4.log 2>&1; echo ncu c4 rc=$?
timeout 300 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_plain5.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"tell_kernel|rank_count" -s 2 -c 2 -o gpurun_out/${T}_c5 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/${T}_ncu_c5.log 2>&1; echo ncu c5 rc=$?
