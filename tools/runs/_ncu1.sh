mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2g_build.log 2>&1
python bench.py --steps 1 --warmup 3 --no-cpu-baseline --sub 0 > gpurun_out/r2g_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ask_kernel|eval_warp|tell_kernel|rank|sepcma" -c 10 -o gpurun_out/r2g_c2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --sub 0 > gpurun_out/r2g_ncu_c2.log 2>&1; echo ncu c2 rc=$?
python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_plain4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"mlp|ask" -c 2 -o gpurun_out/r2g_c4 python bench.py --config c4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_ncu_c4.log 2>&1; echo ncu c4 rc=$?
python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_plain5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"rank" -c 2 -o gpurun_out/r2g_c5 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2g_ncu_c5.log 2>&1; echo ncu c5 rc=$?
